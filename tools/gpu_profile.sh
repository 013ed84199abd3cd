# ncu captures of the two hot kernels (run under gpurun, one GPU).
# usage: bash tools/gpu_profile.sh <tag> [bench args...]
set -x
tag=${1:-prof}; shift
args="--steps 2 --warmup 3 --no-cpu $*"
python bench.py $args > gpurun_out/${tag}_pbench.json 2> gpurun_out/${tag}_pbench.err || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"frame_heads|associate" \
  --csv --log-file gpurun_out/${tag}_launches.csv python bench.py $args > gpurun_out/${tag}_ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:associate_kernel -s 3 -c 1 \
  -o gpurun_out/${tag}_assoc -f python bench.py $args > gpurun_out/${tag}_ncu_assoc.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:frame_heads_kernel -s 3 -c 1 \
  -o gpurun_out/${tag}_frame -f python bench.py $args > gpurun_out/${tag}_ncu_frame.log 2>&1
echo done
