# A/B of the JDE-extension instantiation: its two out-of-line phases inlined or not
for v in "-DTF_JDE_IOU_ATTR=__noinline__ -DTF_JDE_FUSE_ATTR=__noinline__" "-DTF_JDE_FUSE_ATTR=__noinline__" "-DTF_JDE_IOU_ATTR=__noinline__" ""; do
  echo "=== variant '$v'"
  TF_NVCC_EXTRA="$v" python -m paper_2011_03910_b200._build --force > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  grep -B1 "Used 255" paper_2011_03910_b200/csrc/tf_kernels.ptxas.txt | grep spill | sort | uniq -c
  for args in "--jde" "--jde" ""; do
    timeout 600 python bench.py --no-cpu --no-cfg4 $args 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); ph=d.get('assoc_phases_us_per_frame') or {}
print('$args', round(d['value']), 'whole', round(ph.get('whole_frame',0),2), 'upd', round(ph.get('update_ema',0),2), 'cost', round(ph.get('cost',0),2), 'lap', round(ph.get('lap',0),2))"
  done
done
