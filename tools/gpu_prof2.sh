set -x
bash tools/gpu_profile.sh r02f --no-cfg4
bash tools/gpu_profile.sh r02f4 --no-cfg4 --config cfg4 --steps 1
timeout 300 python tools/host_probe.py 1 > gpurun_out/r02f_host_b1.txt 2>&1
