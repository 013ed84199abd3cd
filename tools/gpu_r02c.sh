set -x
for c in "cfg1" "cfg2" "cfg4"; do
  timeout 600 python bench.py --no-cpu --no-cfg4 --config $c > gpurun_out/r02c_$c.json 2> gpurun_out/r02c_$c.err; echo $c=$?
done
for i in 1 2 3; do TF_ASSOC_NARROW=1 timeout 300 python tools/narrow_fault.py 400 $i >> gpurun_out/r02c_narrow.txt 2>&1; echo narrow$i=$?; done
for i in 1 2 3; do TF_ASSOC_NARROW=1 TF_ZERO_SMEM=1 timeout 300 python tools/narrow_fault.py 400 $i >> gpurun_out/r02c_narrow_zero.txt 2>&1; echo zero$i=$?; done
