# Shared-memory overrun hunt: 64 canary words past the association plan, checked at every phase mark
TF_NVCC_EXTRA="-DTF_CANARY" python -m paper_2011_03910_b200._build --force > /dev/null 2>&1 || { echo build failed; exit 1; }
for i in $(seq 1 ${RUNS:-10}); do
  env ${ENVS} CUDA_LAUNCH_BLOCKING=1 timeout 300 python bench.py --no-cpu --config ${CFG:-cfg4} --steps 3 --warmup 3 > gpurun_out/cy_$i.out 2> gpurun_out/cy_$i.err
  rc=$?
  n=$(grep -c TFCANARY gpurun_out/cy_$i.out)
  echo run$i rc=$rc canary=$n
  if [ $n -gt 0 ]; then grep TFCANARY gpurun_out/cy_$i.out | head -12; fi
  if [ $rc -ne 0 ]; then tail -2 gpurun_out/cy_$i.err; fi
done
