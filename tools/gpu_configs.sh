# bench the multi-stream configs on one GPU
set -x
timeout 900 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu > gpurun_out/cfg3.json 2> gpurun_out/cfg3.err; echo cfg3=$?
timeout 900 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu > gpurun_out/cfg4.json 2> gpurun_out/cfg4.err; echo cfg4=$?
timeout 900 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu > gpurun_out/cfg2.json 2> gpurun_out/cfg2.err; echo cfg2=$?
