set -x
timeout 300 python tools/shard_probe.py 64 >> gpurun_out/shard64b.txt 2>&1
