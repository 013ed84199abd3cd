set -x
export TF_CLUSTER=1
python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/c1_bench.json 2> gpurun_out/c1_bench.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:associate_kernel -s 3 -c 1 \
  -o gpurun_out/c1_assoc -f python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/c1_ncu_assoc.log 2>&1
echo done
