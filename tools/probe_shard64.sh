set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for env in "" "TF_CLUSTER=1" "TF_ASSOC_NARROW=1"; do
  echo "== $env"; env $env timeout 300 python tools/shard_probe.py 64 6
done
echo "== 512"; timeout 300 python tools/shard_probe.py 512 3
