# B = 1 with many steps (a 20-step B = 1 run times 20 frames): association cluster size
set -x
T=${1:-r02r}
for rep in 1 2; do
  for c in 16 8 4; do
    TF_CLUSTER=$c timeout 300 python bench.py --no-cpu --no-cfg4 --batch 1 --steps 600 --warmup 50 > gpurun_out/${T}_b1_c${c}_${rep}.json 2> gpurun_out/${T}_b1_c${c}_${rep}.err; echo b1 c$c=$?
  done
done
