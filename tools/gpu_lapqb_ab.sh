# A/B of the shared-memory warp LAP's load batching (TF_LAP_QB; 1 = one position at a time):
# config 2 over all 300 frames, per-solve cost of the full-matrix tie solves, cfg1 headline
for v in "-DTF_LAP_QB=1" "" "-DTF_LAP_QB=8" "-DTF_LAP_QB=1" ""; do
  echo "=== variant '$v'"
  TF_NVCC_EXTRA="$v" python -m paper_2011_03910_b200._build --force > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  for args in "--config cfg2 --steps 34 --warmup 3" "--steps 20 --warmup 5"; do
    timeout 600 python bench.py --no-cpu --no-cfg4 $args 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); ph=d.get('assoc_phases_us_per_frame') or {}; c=d.get('assoc_counters_per_frame') or {}
print('$args', round(d['value']), 'step_us', round(d['ms_per_step']*1000,1), 'whole', round(ph.get('whole_frame',0),2), 'lap', round(ph.get('lap',0),2), 'full', round(ph.get('lap.full_restatement',0),2), 'ties', c.get('tie_fallback'), 'parity', (d.get('parity') or {}).get('ids_exact'))"
  done
  timeout 600 python tools/tie_probe.py cfg2 2>/dev/null | tail -1
done
timeout 900 python -m pytest tests/test_gpu_units.py tests/test_gpu_ties.py -q -x 2>&1 | tail -2
