# A/B of compile-time variants on the cfg4 shard probes: bash tools/gpu_variant_ab3.sh "" "-DX" ...
for v in "$@"; do
  echo "=== variant '$v'"
  TF_NVCC_EXTRA="$v" python -m paper_2011_03910_b200._build --force > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  timeout 300 python tools/shard_probe.py 512 4 | cut -c1-330
  TF_CLUSTER=1 timeout 300 python tools/shard_probe.py 64 6 | cut -c1-330
done
