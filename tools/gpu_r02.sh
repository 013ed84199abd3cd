# round-2 GPU session: gpu tests (incl. the reference's own suite), smoke, bench, reference arm
set -x
mkdir -p gpurun_out
T0=$(date +%s)
timeout 1500 python -m pytest tests -m gpu -q -rA --durations=15 ${PYTEST_ARGS} > gpurun_out/r2_pytest.log 2>&1; echo pytest=$? $(( $(date +%s) - T0 ))s
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo bench=$? $(( $(date +%s) - T0 ))s
timeout 600 python bench.py --impl reference ${BENCH_ARGS} > gpurun_out/r2_ref.json 2> gpurun_out/r2_ref.err; echo ref=$? $(( $(date +%s) - T0 ))s
