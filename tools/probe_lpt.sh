echo "== LPT 512"; timeout 300 python tools/stream_clock_probe.py 512 4
echo "== NO_LPT 512"; TF_NO_LPT=1 timeout 300 python tools/stream_clock_probe.py 512 3
echo "== shard 512 LPT"; timeout 300 python tools/shard_probe.py 512 4
echo "== shard 512 NO_LPT"; TF_NO_LPT=1 timeout 300 python tools/shard_probe.py 512 4
timeout 900 python -m pytest tests/test_gpu_heads.py -q -x -m gpu 2>&1 | tail -3
