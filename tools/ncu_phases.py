"""Group ncu source-page stall samples of associate_kernel by phase (line ranges of tf_kernels.cu)."""
import csv, io, subprocess, sys
from collections import defaultdict
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
PH = [(1, 665, "prologue/helpers"), (666, 765, "setup"), (766, 818, "follower"), (819, 875, "load_predict"),
      (876, 926, "gate"), (927, 970, "csr"), (971, 993, "cost"), (994, 1265, "lap"), (1266, 1286, "match"),
      (1287, 1332, "update_ema"), (1333, 1459, "records"), (1460, 1490, "epilogue")]
fname = None; hdr = None
agg = defaultdict(lambda: defaultdict(int))
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if not hdr or r[0] in ("", "Function Name"): continue
    d = dict(zip(hdr[2:], r[2:]))
    ln = int(r[0])
    if fname == "tf_kernels.cu":
        ph = next((n for a, b, n in PH if a <= ln <= b), "other")
        if 518 <= ln <= 580: ph = "cost_work(shared)"
        if 595 <= ln <= 658: ph = "ema_work(shared)"
    elif fname == "tf_device.cuh":
        ph = "dev:" + ("lap" if ln >= 300 else "KF/misc" if ln >= 95 else "util")
    else:
        ph = "cluster_sync" if fname in ("sm_90_rt.hpp", "helpers.h", "cooperative_groups.h") else "intrinsics"
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k:
            try: agg[ph][k[6:]] += int(v)
            except ValueError: pass
    try:
        agg[ph]["_samples"] += int(d["Warp Stall Sampling (All Samples)"]); agg[ph]["_inst"] += int(d["Instructions Executed"])
    except ValueError: pass
tot = sum(a["_samples"] for a in agg.values())
for ph, a in sorted(agg.items(), key=lambda x: -x[1]["_samples"]):
    top = sorted(((v, k) for k, v in a.items() if not k.startswith("_")), reverse=True)[:4]
    print(f"{ph:20s} {100*a['_samples']/tot:5.1f}%  inst {a['_inst']:8d}  " + ", ".join(f"{k}={v}" for v, k in top))
