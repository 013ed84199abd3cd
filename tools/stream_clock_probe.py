"""Per-stream association clocks (tf_stream_clocks) for S streams of cfg4 (B = 8):
when each stream's leader CTA starts, how long its prologue and its frames take,
and when it exits. Usage: [env knobs] python tools/stream_clock_probe.py S [updates]"""
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
U = int(sys.argv[2]) if len(sys.argv) > 2 else 3
gen = synth.make("cfg4", device="cuda", seed=7, streams=S)
cap = p.Capacity(streams=S, max_frames=S * 8, max_candidates=192, max_detections=96, max_tracks=160)
bt = p.BatchTracker(S, frames_per_update=8, capacity=cap)
for _ in range(3):
    b = gen.next_batch(8)
    bt.update(b)
    del b
lib = bt.engine.lib
out = []
for u in range(U):
    b = gen.next_batch(8)
    lib.tf_set_profiling(bt.engine.ctx, 4)
    torch.cuda.synchronize()
    bt.update(b)
    torch.cuda.synchronize()
    clk = np.zeros(4 * S, np.int64)
    assert lib.tf_stream_clocks(bt.engine.ctx, clk.ctypes.data, S) == 0
    lib.tf_set_profiling(bt.engine.ctx, 0)
    clk = clk.reshape(S, 4).astype(np.float64) / 1e3   # us
    t0 = clk[:, 0].min()
    ent, pro, frm, epi = clk[:, 0] - t0, clk[:, 1] - clk[:, 0], clk[:, 2] - clk[:, 1], clk[:, 3] - clk[:, 2]
    q = lambda x: [round(float(v), 1) for v in np.percentile(x, [0, 50, 90, 100])]
    out.append({"update": u, "entry_us_p0_50_90_100": q(ent), "prologue_us": q(pro), "frames_us": q(frm),
                "epilogue_us": q(epi), "end_us_max": round(float((clk[:, 3] - t0).max()), 1),
                "slowest_stream": int(np.argmax(clk[:, 3])), "late_entries": int((ent > 5).sum())})
    del b
th, cl = C.c_int32(), C.c_int32()
lib.tf_launch_info(bt.engine.ctx, C.byref(th), C.byref(cl))
print(json.dumps({"streams": S, "threads": th.value, "cluster": cl.value, "updates": out}))
