echo "== shard 512 default"; timeout 300 python tools/shard_probe.py 512 4
echo "== shard 512 overlap (opt-in)"; TF_OVERLAP=1 timeout 300 python tools/shard_probe.py 512 4
echo "== clocks 512 overlap"; timeout 300 python tools/stream_clock_probe.py 512 3
