timeout 900 python -m pytest tests/test_gpu_heads.py tests/test_gpu_tracker.py -q -x -m gpu 2>&1 | tail -2
for env in "" "TF_NO_SPLIT=1"; do
  echo "== $env"
  env $env timeout 300 python tools/shard_probe.py 512 4 | cut -c1-200
  env $env timeout 300 python tools/shard_probe.py 64 6 | cut -c1-200
  env $env timeout 300 python bench.py --no-cpu --no-cfg4 --config cfg3 --steps 6 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3', round(d['value']), d['kernels']['frame_heads_kernel'])"
done
