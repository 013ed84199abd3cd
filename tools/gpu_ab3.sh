set -x
python -m paper_2011_03910_b200._build --force > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_ties.py tests/test_gpu_heads.py -q -x -k "ties or cfg1 or cfg2 or dense or replay or cluster" > gpurun_out/ab3_tests.log 2>&1; echo tests=$?
ORDER="base exp base" bash tools/gpu_ab2.sh
