# A/B of the speculative association prologue (default) vs the serial one (-DTF_SERIAL_PROLOGUE):
# cfg1 B = 32 / 4 / 1 (long runs at small B), cfg2, config-4 shard probes (512 and 64 streams)
T=${1:-r02s}
for v in "-DTF_SERIAL_PROLOGUE" "" "-DTF_SERIAL_PROLOGUE" ""; do
  echo "=== variant '$v'"
  TF_NVCC_EXTRA="$v" python -m paper_2011_03910_b200._build --force > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  for args in "--steps 20 --warmup 5" "--batch 4 --steps 160 --warmup 20" "--batch 1 --steps 600 --warmup 50" "--config cfg2 --steps 10 --warmup 3"; do
    timeout 300 python bench.py --no-cpu --no-cfg4 $args 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); ph=d.get('assoc_phases_us_per_frame') or {}
print('$args', round(d['value']), 'step_us', round(d['ms_per_step']*1000,1), 'assoc_us', round(d['kernels']['associate_kernel']['ms_per_launch']*1000,1), 'whole', round(ph.get('whole_frame',0),2), 'pro', round(ph.get('launch.prologue',0),3), 'parity', (d.get('parity') or {}).get('ids_exact'))"
  done
  timeout 300 python tools/shard_probe.py 512 4 | cut -c1-200
  timeout 300 python tools/shard_probe.py 64 6 | cut -c1-200
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/${T}_pytest.log
