# round-2 final measurement set (tag $1, default r02f): tests, smoke, bench + reference arm,
# config sweep, ncu launch list and full captures of the two kernels (cfg1 and cfg4)
set -x
T=${1:-r02z}
timeout 1500 python -m pytest tests -m gpu -q -rA --durations=10 > gpurun_out/${T}_pytest.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo bench=$?
timeout 600 python bench.py --impl reference > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err; echo ref=$?
for c in "cfg0" "cfg1 --batch 1" "cfg1 --batch 4" "cfg1 --batch 8" "cfg1 --batch 16" "cfg2" "cfg3" "cfg4" "cfg1 --dtype f16" "cfg1 --jde"; do
  n=$(echo $c | tr -d ' -')
  timeout 600 python bench.py --no-cpu --no-cfg4 --config $c > gpurun_out/${T}_$n.json 2> gpurun_out/${T}_$n.err; echo $n=$?
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"frame_heads|associate" \
  --csv --log-file gpurun_out/${T}_launches.csv python bench.py --no-cpu --no-cfg4 --steps 20 --warmup 5 > gpurun_out/${T}_ncu_launch.log 2>&1; echo launches=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:associate_kernel -s 5 -c 1 \
  -o gpurun_out/${T}_assoc -f python bench.py --no-cpu --no-cfg4 --steps 2 --warmup 3 > gpurun_out/${T}_ncu_assoc.log 2>&1; echo assoc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:frame_heads_kernel -s 5 -c 1 \
  -o gpurun_out/${T}_frame -f python bench.py --no-cpu --no-cfg4 --steps 2 --warmup 3 > gpurun_out/${T}_ncu_frame.log 2>&1; echo frame=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:associate_kernel -s 3 -c 1 \
  -o gpurun_out/${T}_c4assoc -f python bench.py --no-cpu --no-cfg4 --config cfg4 --steps 1 --warmup 3 > gpurun_out/${T}_ncu_c4assoc.log 2>&1; echo c4assoc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:frame_heads_kernel -s 3 -c 1 \
  -o gpurun_out/${T}_c4frame -f python bench.py --no-cpu --no-cfg4 --config cfg4 --steps 1 --warmup 3 > gpurun_out/${T}_ncu_c4frame.log 2>&1; echo c4frame=$?
