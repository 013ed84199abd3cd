# timing experiment: the cost phase without fp32->fp64 conversions (numerics wrong; phases only)
set -x
python -m paper_2011_03910_b200._build --force > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 600 python bench.py --no-cpu --no-cfg4 --config cfg4 > gpurun_out/nc_base.json 2> gpurun_out/nc_base.err; echo base=$?
TF_NVCC_EXTRA=-DTF_EXPERIMENT_NOCVT python -m paper_2011_03910_b200._build --force > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 600 python bench.py --no-cpu --no-cfg4 --config cfg4 > gpurun_out/nc_exp.json 2> gpurun_out/nc_exp.err; echo exp=$?
python -m paper_2011_03910_b200._build --force > /dev/null 2>&1
timeout 600 python tools/b1_probe.py 1 300 > gpurun_out/b1_probe.txt 2>&1; echo b1=$?
timeout 600 python tools/b1_probe.py 4 200 >> gpurun_out/b1_probe.txt 2>&1; echo b4=$?
timeout 900 python -m pytest tests/test_gpu_heads.py tests/test_gpu_ties.py -q -x > gpurun_out/nc_tests.log 2>&1; echo tests=$?
