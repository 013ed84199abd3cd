set -x
timeout 900 python -m pytest tests/test_gpu_heads.py tests/test_gpu_tracker.py tests/test_gpu_units.py tests/test_gpu_ties.py tests/test_gpu_detfile.py -q -x > gpurun_out/r02k_tests.log 2>&1; echo tests=$?
timeout 300 python tools/b1_probe.py 1 300 > gpurun_out/r02k_b1.txt 2>&1
for c in "cfg1" "cfg1 --batch 1" "cfg1 --batch 4" "cfg4" "cfg3"; do
  n=$(echo $c | tr -d ' -')
  timeout 600 python bench.py --no-cpu --no-cfg4 --config $c > gpurun_out/r02k_$n.json 2> gpurun_out/r02k_$n.err; echo $n=$?
done
