set -x
timeout 900 python -m pytest tests/test_gpu_heads.py -q -x -k "cfg4 or cluster or narrow or pooled or replay" > gpurun_out/r02h_tests.log 2>&1; echo tests=$?
timeout 600 python bench.py --no-cpu --no-cfg4 --config cfg4 > gpurun_out/r02h_cfg4.json 2> gpurun_out/r02h_cfg4.err; echo cfg4=$?
