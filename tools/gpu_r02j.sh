set -x
timeout 900 python -m pytest tests/test_gpu_heads.py tests/test_gpu_tracker.py tests/test_gpu_units.py tests/test_gpu_ties.py tests/test_gpu_detfile.py -q -x > gpurun_out/r02j_tests.log 2>&1; echo tests=$?
for c in "cfg1" "cfg2" "cfg4" "cfg1 --batch 1"; do
  n=$(echo $c | tr -d ' -')
  timeout 600 python bench.py --no-cpu --no-cfg4 --config $c > gpurun_out/r02j_$n.json 2> gpurun_out/r02j_$n.err; echo $n=$?
done
