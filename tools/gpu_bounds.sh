# Repeat a config under the TF_BOUNDS debug build until a bounds check prints (bad-index hunt; no sanitizer on the pool)
TF_NVCC_EXTRA="-DTF_BOUNDS" python -m paper_2011_03910_b200._build --force > /dev/null 2>&1 || { echo build failed; exit 1; }
for i in $(seq 1 ${RUNS:-8}); do
  CUDA_LAUNCH_BLOCKING=1 timeout 300 python bench.py --no-cpu --config ${CFG:-cfg4} --steps 3 --warmup 3 > gpurun_out/bd_$i.out 2> gpurun_out/bd_$i.err
  rc=$?
  n=$(grep -c TFBOUND gpurun_out/bd_$i.out)
  echo run$i rc=$rc bounds=$n
  if [ $rc -ne 0 ] || [ $n -gt 0 ]; then grep TFBOUND gpurun_out/bd_$i.out | head -20; tail -3 gpurun_out/bd_$i.err; fi
done
