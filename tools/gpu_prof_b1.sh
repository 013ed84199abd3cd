# ncu of the B = 1 kernels (one update's frame kernel and association)
set -x
args="--batch 1 --steps 30 --warmup 5 --no-cpu --no-cfg4"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:frame_heads_kernel -s 20 -c 1 \
  -o gpurun_out/b1_frame -f python bench.py $args > gpurun_out/b1_ncu_frame.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:associate_kernel -s 20 -c 1 \
  -o gpurun_out/b1_assoc -f python bench.py $args > gpurun_out/b1_ncu_assoc.log 2>&1
echo done
