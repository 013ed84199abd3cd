# round-2 closing set (tag $1): pytest -m gpu, smoke, bench + reference arm, the config sweep with
# small batches timed over >= 600 frames (a 20-step B = 1 run times 20 frames), ncu launch list
set -x
T=${1:-r02t}
timeout 1500 python -m pytest tests -m gpu -q -rA --durations=10 > gpurun_out/${T}_pytest.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo bench=$?
timeout 600 python bench.py --impl reference > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err; echo ref=$?
while read -r n args; do
  timeout 600 python bench.py --no-cpu --no-cfg4 $args > gpurun_out/${T}_$n.json 2> gpurun_out/${T}_$n.err; echo $n=$?
done <<'LIST'
cfg0 --config cfg0 --steps 95 --warmup 5
cfg1batch1 --batch 1 --steps 600 --warmup 50
cfg1batch4 --batch 4 --steps 160 --warmup 20
cfg1batch8 --batch 8 --steps 80 --warmup 10
cfg1batch16 --batch 16 --steps 40 --warmup 5
cfg2 --config cfg2 --steps 34 --warmup 3
cfg3 --config cfg3
cfg4 --config cfg4
cfg1dtypef16 --dtype f16
cfg1jde --jde
LIST
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"frame_heads|associate" \
  --csv --log-file gpurun_out/${T}_launches.csv python bench.py --no-cpu --no-cfg4 --steps 20 --warmup 5 > gpurun_out/${T}_ncu_launch.log 2>&1; echo launches=$?
