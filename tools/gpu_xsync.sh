# Race bisection for the 128-thread association variant: extra barriers at the
# transitions in TF_XSYNC_MASK, RUNS cfg4 runs each. usage: MASK=255 RUNS=40 bash tools/gpu_xsync.sh
TF_NVCC_EXTRA="-DTF_XSYNC_MASK=${MASK:-0}" python -m paper_2011_03910_b200._build --force > /dev/null 2>&1 || { echo build failed; exit 1; }
fail=0
for i in $(seq 1 ${RUNS:-40}); do
  TF_ASSOC_NARROW=1 CUDA_LAUNCH_BLOCKING=1 timeout 300 python bench.py --no-cpu --config cfg4 --steps 3 --warmup 3 > /dev/null 2> gpurun_out/xs_$i.err || fail=$((fail+1))
done
echo "mask=${MASK:-0} runs=${RUNS:-40} failures=$fail"
