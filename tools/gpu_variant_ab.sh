# A/B of compile-time variants on the shard probes and a short cfg1 bench:
#   bash tools/gpu_variant_ab.sh "" "-DX" ...   (results in gpurun_out/vab.log)
for v in "$@"; do
  echo "=== variant '$v'"
  TF_NVCC_EXTRA="$v" python -m paper_2011_03910_b200._build --force > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  timeout 300 python tools/shard_probe.py 64 6
  timeout 300 python tools/shard_probe.py 512 4
  timeout 300 python bench.py --no-cpu --no-cfg4 --config cfg1 --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg1', round(d['value']), d.get('assoc_phases_us_per_frame',{}).get('cost'), d.get('assoc_phases_us_per_frame',{}).get('whole_frame'))"
done
