# Full round measurement: tests, smoke, default bench (with CPU baseline), reference arm, ncu launch list + full captures.
set -x
tag=${1:-full}
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo bench=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${tag}_ref.json 2> gpurun_out/${tag}_ref.err; echo ref=$?
bash tools/gpu_profile.sh ${tag}
