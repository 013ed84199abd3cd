# A/B of compile-time variants on cfg1 / cfg2 benches: bash tools/gpu_variant_ab2.sh "" "-DX" ...
for v in "$@"; do
  echo "=== variant '$v'"
  TF_NVCC_EXTRA="$v" python -m paper_2011_03910_b200._build --force > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  for cfg in cfg1 cfg2; do
    timeout 300 python bench.py --no-cpu --no-cfg4 --config $cfg --steps 10 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); ph=d.get('assoc_phases_us_per_frame') or {}; c=d.get('assoc_counters_per_frame') or {}
print('$cfg', round(d['value']), 'whole', round(ph.get('whole_frame',0),2), 'lap', round(ph.get('lap',0),2), 'full', round(ph.get('lap.full_restatement',0),2), 'ties', c.get('tie_fallback'), 'parity', (d.get('parity') or {}).get('ids_exact'))"
  done
done
