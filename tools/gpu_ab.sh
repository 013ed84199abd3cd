# A/B of compile-time variants: bash tools/gpu_ab.sh "-DVAR1" "-DVAR2" ...  (empty string = baseline)
for v in "$@"; do
  tag=$(echo "$v" | tr -c 'A-Za-z0-9' '_')
  TF_NVCC_EXTRA="$v" python -m paper_2011_03910_b200._build --force > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  python bench.py --no-cpu --steps 10 ${BENCH_ARGS} > gpurun_out/ab_${tag}.json 2> gpurun_out/ab_${tag}.err
  python - "$v" gpurun_out/ab_${tag}.json <<'PY'
import json, sys
d = json.load(open(sys.argv[2]))
ph = {k: round(v, 2) for k, v in d["assoc_phases_us_per_frame"].items()}
print(repr(sys.argv[1]), round(d["value"]), "e2e", round(d["e2e"]["value"] or 0), ph)
PY
done
