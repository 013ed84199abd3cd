# ncu --set full captures of both hot kernels at cfg1 and cfg4 for the final build (tag $1); the
# reports are exported to CSV on the box (raw + details pages) and removed, so gpurun_out stays
# under the 64 MiB merge limit (the four reports with source exceed it)
set -x
T=${1:-r02t}
cap() {  # name kernel skip bench-args...
  n=$1; k=$2; s=$3; shift 3
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -s $s -c 1 \
    -o gpurun_out/${T}_$n -f python bench.py --no-cpu --no-cfg4 "$@" > gpurun_out/${T}_ncu_$n.log 2>&1; echo $n=$?
  ncu -i gpurun_out/${T}_$n.ncu-rep --page raw --csv > gpurun_out/${T}_${n}_raw.csv 2>/dev/null
  ncu -i gpurun_out/${T}_$n.ncu-rep --page details --csv > gpurun_out/${T}_${n}_details.csv 2>/dev/null
  rm -f gpurun_out/${T}_$n.ncu-rep
}
python bench.py --no-cpu --no-cfg4 --steps 2 --warmup 3 > gpurun_out/${T}_pb1.json 2> gpurun_out/${T}_pb1.err; echo pb1=$?
python bench.py --no-cpu --no-cfg4 --config cfg4 --steps 1 --warmup 3 > gpurun_out/${T}_pb4.json 2> gpurun_out/${T}_pb4.err; echo pb4=$?
cap assoc associate_kernel 5 --steps 2 --warmup 3
cap frame frame_heads_kernel 5 --steps 2 --warmup 3
cap c4assoc associate_kernel 3 --config cfg4 --steps 1 --warmup 3
cap c4frame frame_heads_kernel 3 --config cfg4 --steps 1 --warmup 3
du -sh gpurun_out
