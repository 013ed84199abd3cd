# A/B of runtime env settings: bash tools/gpu_env_ab.sh "TF_CLUSTER=8" "TF_CLUSTER=16"
for v in "$@"; do
  tag=$(echo "$v" | tr -c 'A-Za-z0-9' '_')
  env $v python bench.py --no-cpu --steps 10 ${BENCH_ARGS} > gpurun_out/envab_${tag}.json 2> gpurun_out/envab_${tag}.err
  python - "$v" gpurun_out/envab_${tag}.json <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[2]))
except Exception as e:
    print(sys.argv[1], "failed", e); sys.exit()
ph = {k: round(v, 2) for k, v in d["assoc_phases_us_per_frame"].items() if not k.startswith("f.")}
print(repr(sys.argv[1]), round(d["value"]), "e2e", round(d["e2e"]["value"] or 0), ph)
PY
done
