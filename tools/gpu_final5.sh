# round-2 closing captures for the final build (tag $1): ncu --set full of both hot kernels at
# cfg1 and cfg4 (each only after the same command exited 0 without ncu), then a short repeat
# campaign (fresh process per run) on cfg4 and cfg1 counting failures
set -x
T=${1:-r02t}
python bench.py --no-cpu --no-cfg4 --steps 2 --warmup 3 > gpurun_out/${T}_pb1.json 2> gpurun_out/${T}_pb1.err; echo pb1=$?
python bench.py --no-cpu --no-cfg4 --config cfg4 --steps 1 --warmup 3 > gpurun_out/${T}_pb4.json 2> gpurun_out/${T}_pb4.err; echo pb4=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:associate_kernel -s 5 -c 1 \
  -o gpurun_out/${T}_assoc -f python bench.py --no-cpu --no-cfg4 --steps 2 --warmup 3 > gpurun_out/${T}_ncu_assoc.log 2>&1; echo assoc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:frame_heads_kernel -s 5 -c 1 \
  -o gpurun_out/${T}_frame -f python bench.py --no-cpu --no-cfg4 --steps 2 --warmup 3 > gpurun_out/${T}_ncu_frame.log 2>&1; echo frame=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:associate_kernel -s 3 -c 1 \
  -o gpurun_out/${T}_c4assoc -f python bench.py --no-cpu --no-cfg4 --config cfg4 --steps 1 --warmup 3 > gpurun_out/${T}_ncu_c4assoc.log 2>&1; echo c4assoc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:frame_heads_kernel -s 3 -c 1 \
  -o gpurun_out/${T}_c4frame -f python bench.py --no-cpu --no-cfg4 --config cfg4 --steps 1 --warmup 3 > gpurun_out/${T}_ncu_c4frame.log 2>&1; echo c4frame=$?
for cfg in cfg4 cfg1 cfg2; do
  fail=0
  for i in $(seq 1 ${RUNS:-15}); do
    timeout 300 python bench.py --no-cpu --no-cfg4 --config $cfg --steps 3 --warmup 3 > /dev/null 2> gpurun_out/${T}_rp_${cfg}_$i.err || fail=$((fail+1))
  done
  echo "repeat cfg=$cfg runs=${RUNS:-15} failures=$fail" | tee -a gpurun_out/${T}_repeat.txt
done
