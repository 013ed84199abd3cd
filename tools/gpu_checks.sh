# repeat campaign on the cluster configurations (cfg1 single stream, cfg2 dense) and the
# smoke() launch list (which kernels a driver-side launch capture of smoke() sees)
set -x
fail=0
for i in $(seq 1 40); do timeout 120 python bench.py --no-cpu --no-cfg4 --config cfg1 --steps 3 --warmup 3 > /dev/null 2> gpurun_out/rc1_$i.err || fail=$((fail+1)); done
echo cfg1_fail=$fail
fail=0
for i in $(seq 1 20); do timeout 120 python bench.py --no-cpu --no-cfg4 --config cfg2 --steps 3 --warmup 3 --seed $i > /dev/null 2> gpurun_out/rc2_$i.err || fail=$((fail+1)); done
echo cfg2_fail=$fail
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/smoke_launches.csv \
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ncu.log 2>&1; echo smoke_ncu=$?
