# round-2 closing set (tag $1): pytest -m gpu (with the reference suite staged), smoke, bench, reference arm
set -x
T=${1:-r02o}
timeout 1500 python -m pytest tests -m gpu -q -rA --durations=10 > gpurun_out/${T}_pytest.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo bench=$?
timeout 600 python bench.py --impl reference > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err; echo ref=$?
