"""Per-GPU share of config 4 at N GPUs: S = 512 / N streams of cfg4 (B = 8) on
this GPU, steps timed alone (generation between steps), association phases.
Usage: [TF_CLUSTER=c] python tools/shard_probe.py S [steps]"""
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2011_03910_b200 as p  # noqa: E402
from paper_2011_03910_b200 import synth  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 64
K = int(sys.argv[2]) if len(sys.argv) > 2 else 4
gen = synth.make("cfg4", device="cuda", seed=7, streams=S)
cap = p.Capacity(streams=S, max_frames=S * 8, max_candidates=192, max_detections=96, max_tracks=160)
bt = p.BatchTracker(S, frames_per_update=8, capacity=cap)
for _ in range(3):
    b = gen.next_batch(8)
    bt.update(b)
    del b
lib = bt.engine.lib
lib.tf_set_profiling(bt.engine.ctx, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ms = 0.0
flag = torch.zeros(1, dtype=torch.int32).pin_memory()
stream = torch.cuda.current_stream()
for _ in range(K):
    b = gen.next_batch(8)
    torch.cuda.synchronize()
    flag.zero_()
    lib.tf_stream_hold(flag.data_ptr(), stream.cuda_stream)   # time the device work, not the host's submission
    e0.record()
    try:
        bt.update(b, sync=False)
        e1.record()
    finally:
        flag.fill_(1)
    e1.synchronize()
    ms += e0.elapsed_time(e1)
    del b
tl = np.zeros(6 * 64)
ntl = C.c_int32()
lib.tf_timeline(bt.engine.ctx, tl.ctypes.data, 64, C.byref(ntl))
tl = tl[:6 * min(ntl.value, 64)].reshape(-1, 6)
fr, asc, n = C.c_double(), C.c_double(), C.c_int64()
lib.tf_kernel_times(bt.engine.ctx, C.byref(fr), C.byref(asc), C.byref(n))
th, cl = C.c_int32(), C.c_int32()
lib.tf_launch_info(bt.engine.ctx, C.byref(th), C.byref(cl))
lib.tf_set_profiling(bt.engine.ctx, 2)
b = gen.next_batch(8)
bt.update(b)
ph = np.zeros(40, np.int64)
lib.tf_phase_stats(bt.engine.ctx, ph.ctypes.data)
names = ["load_predict", "gate", "csr", "cost", "lap", "match", "update_ema", "records_births"]
print(json.dumps({"streams": S, "threads": th.value, "cluster": cl.value, "ms_per_step": ms / K,
                  "frames_per_s": S * 8 * K / (ms / 1e3), "frame_ms": fr.value / max(n.value, 1),
                  "assoc_ms": asc.value / max(n.value, 1),
                  "phases_us": {nm: round(float(ph[i]) / max(ph[11], 1) / 1965, 2) for i, nm in enumerate(names)},
                  "whole_us": round(float(ph[31]) / max(ph[11], 1) / 1965, 2),
                  "timeline_us": [[round(1e3 * (v - row[4]), 1) for v in row[:4]] for row in tl[:4]]}))
