"""Host submission latency of one streamed update at S streams (cfg4 shapes):
time from e0 (recorded before update()) to the first kernel, host wall time of
update(), and the device span (first mark to association end) vs the event
span. Usage: python tools/submit_probe.py S [steps]"""
import ctypes as C
import cProfile
import pstats
import sys
import time
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
PROF = int(sys.argv[3]) if len(sys.argv) > 3 else 1
lib.tf_set_profiling(bt.engine.ctx, PROF)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev_ms, host_us = [], []
prof = cProfile.Profile()
for _ in range(K):
    b = gen.next_batch(8)
    torch.cuda.synchronize()
    e0.record()
    t0 = time.perf_counter()
    prof.enable()
    bt.update(b, sync=False)
    prof.disable()
    host_us.append(1e6 * (time.perf_counter() - t0))
    e1.record()
    e1.synchronize()
    ev_ms.append(e0.elapsed_time(e1))
    del b
tl = np.zeros(6 * 64)
ntl = C.c_int32()
lib.tf_timeline(bt.engine.ctx, tl.ctypes.data, 64, C.byref(ntl))
tl = tl[:6 * ntl.value].reshape(-1, 6)
span = [float(r[3] - min(r[0], r[4])) for r in tl] or [float("nan")]
print(f"S={S}: event span {np.mean(ev_ms):.3f} ms, device span (first mark -> association end) "
      f"{np.mean(span):.3f} ms, host update() {np.mean(host_us):.0f} us")
pstats.Stats(prof).sort_stats("cumulative").print_stats(12)
