# A/B of compile-time variants on a bench config: CFG=cfg4 bash tools/gpu_cfg_ab.sh "-DX" ...
for v in "$@"; do
  tag=$(echo "$v" | tr -c 'A-Za-z0-9' '_')
  TF_NVCC_EXTRA="$v" python -m paper_2011_03910_b200._build --force > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  python bench.py --no-cpu --config ${CFG:-cfg4} --steps 3 --warmup 3 > gpurun_out/cab_${tag}.json 2> gpurun_out/cab_${tag}.err
  python - "$v" gpurun_out/cab_${tag}.json <<'PY'
import json, sys
d = json.load(open(sys.argv[2]))
k = d["kernels"]
print(repr(sys.argv[1]), round(d["value"]), "frame ms", round(k["frame_heads_kernel"]["ms_per_launch"], 4),
      "assoc ms", round(k["associate_kernel"]["ms_per_launch"], 4))
PY
done
