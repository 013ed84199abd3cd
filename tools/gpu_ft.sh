set -x
TF_NVCC_EXTRA=-DTF_FRAME_TIMERS python -m paper_2011_03910_b200._build --force > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 300 python tools/b1_probe.py 1 40 > gpurun_out/ft_b1.txt 2>&1
python -m paper_2011_03910_b200._build --force > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_units.py tests/test_gpu_heads.py tests/test_gpu_tracker.py -q -x > gpurun_out/ft_tests.log 2>&1; echo tests=$?
timeout 300 python tools/b1_probe.py 1 300 > gpurun_out/ft_b1b.txt 2>&1
timeout 600 python bench.py --no-cpu --no-cfg4 --config cfg1 --batch 1 > gpurun_out/ft_b1.json 2>/dev/null
timeout 600 python bench.py --no-cpu --no-cfg4 --config cfg4 > gpurun_out/ft_cfg4.json 2>/dev/null
