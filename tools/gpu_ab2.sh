# A/B of a compile-time switch on the cfg1 headline: base vs TF_NVCC_EXTRA=$AB (3 runs each)
set -x
for v in ${ORDER:-base exp base exp base exp}; do
  if [ $v = exp ]; then TF_NVCC_EXTRA="$AB" python -m paper_2011_03910_b200._build --force > /dev/null 2>&1; else python -m paper_2011_03910_b200._build --force > /dev/null 2>&1; fi
  timeout 600 python bench.py --no-cpu --no-cfg4 --config cfg1 --steps 20 > gpurun_out/ab_$v.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['value']), round(d['assoc_phases_us_per_frame']['whole_frame'],2), round(d['assoc_phases_us_per_frame']['lap'],2), round(d['assoc_counters_per_frame']['multi_components'],3), round(d['assoc_counters_per_frame']['residual_entries'],3))" >> gpurun_out/ab_summary.txt
done
python -m paper_2011_03910_b200._build --force > /dev/null 2>&1
