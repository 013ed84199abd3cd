# quick GPU check: micro-benchmarks (optional), gpu tests, bench (no cpu leg)
set -x
[ -x tools/micro/lat ] && tools/micro/lat > gpurun_out/micro_lat.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q_pytest.log 2>&1; echo pytest=$?
timeout 600 python bench.py --no-cpu ${BENCH_ARGS} > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err; echo bench=$?
