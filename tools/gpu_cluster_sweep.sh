# cluster size of the association at small batches (TF_CLUSTER), cfg1 B = 1, 4, 8, 32
set -x
T=${1:-r02q}
timeout 600 python bench.py --no-cpu --no-cfg4 > gpurun_out/${T}_head.json 2> gpurun_out/${T}_head.err; echo head=$?
for b in 1 4 8; do
  for c in 16 8 4 2 1; do
    TF_CLUSTER=$c timeout 300 python bench.py --no-cpu --no-cfg4 --batch $b > gpurun_out/${T}_b${b}_c${c}.json 2> gpurun_out/${T}_b${b}_c${c}.err; echo b$b c$c=$?
  done
done
for c in 8 4; do
  TF_CLUSTER=$c timeout 300 python bench.py --no-cpu --no-cfg4 > gpurun_out/${T}_b32_c${c}.json 2> gpurun_out/${T}_b32_c${c}.err; echo b32 c$c=$?
done
