"""Group ncu source-page stall samples of associate_kernel by phase (line ranges of tf_kernels.cu)."""
import csv, io, subprocess, sys
from pathlib import Path
from collections import defaultdict
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
SRC = Path(__file__).resolve().parents[1] / "paper_2011_03910_b200" / "csrc" / "tf_kernels.cu"
MARKERS = [("__device__ void cost_work", "cost_work(shared)"), ("__device__ void ema_work", "ema_work(shared)"),
           ("associate_kernel(AssocArgs a", "setup"), ("  if (rank != 0) {", "follower"),
           ("// ---- Kalman predict", "load_predict"), ("// ---- gate (", "gate"), ("// ---- CSR of finite", "csr"),
           ("// ---- fp64 cosine cost", "cost"), ("// ---- exact LAP", "lap"), ("// ---- matches + max_cost", "match"),
           ("// ---- matched: Kalman update", "update_ema"), ("// ---- records: matched", "records"),
           ("// ---- release the follower", "epilogue"), ("__global__ void nms_sets_kernel", "stage kernels")]
lines = SRC.read_text().splitlines()
starts = sorted((next(i + 1 for i, l in enumerate(lines) if m in l), name) for m, name in MARKERS)
PH = [(a, (starts[k + 1][0] - 1) if k + 1 < len(starts) else 10 ** 9, n) for k, (a, n) in enumerate(starts)]
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
        ph = next((n for a, b, n in PH if a <= ln <= b), "frame/other")
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
