# config sweep: bench lines for cfg1 (B = 1, 4, 32), cfg2, cfg3, cfg4 (no CPU legs), tag in $TAG
set -x
TAG=${TAG:-sweep}
for c in "cfg1" "cfg1 --batch 1" "cfg1 --batch 4" "cfg2" "cfg3" "cfg4"; do
  n=$(echo $c | tr -d ' -')
  timeout 600 python bench.py --no-cpu --no-cfg4 --config $c ${SWEEP_ARGS} > gpurun_out/${TAG}_$n.json 2> gpurun_out/${TAG}_$n.err; echo $n=$?
done
