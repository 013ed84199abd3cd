set -x
timeout 900 python -m pytest tests/test_gpu_heads.py tests/test_gpu_tracker.py tests/test_gpu_detfile.py tests/test_gpu_ties.py -q -x > gpurun_out/r02i_tests.log 2>&1; echo tests=$?
timeout 300 python tools/host_probe.py 1 > gpurun_out/r02i_host_b1.txt 2>&1
for c in "cfg1" "cfg1 --batch 1" "cfg1 --batch 4" "cfg4"; do
  n=$(echo $c | tr -d ' -')
  timeout 600 python bench.py --no-cpu --no-cfg4 --config $c > gpurun_out/r02i_$n.json 2> gpurun_out/r02i_$n.err; echo $n=$?
done
