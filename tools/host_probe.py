"""Host-side cost of one BatchTracker.update call (device-resident inputs).

python tools/host_probe.py [B]  -> us per update call (host wall time, calls
enqueue only), GPU us per update, and the top cProfile entries.
"""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2011_03910_b200 as p  # noqa: E402
from paper_2011_03910_b200 import synth  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
N = 300
gen = synth.make("cfg1", device="cuda", seed=0, streams=1)
batches = [gen.next_batch(B) for _ in range(N + 10)]
cap = p.Capacity(streams=1, max_frames=B, max_candidates=512, max_detections=256, max_tracks=256)
bt = p.BatchTracker(1, frames_per_update=B, capacity=cap, pipeline=True)
for i in range(10):
    bt.update(batches[i], sync=False)
bt.join()
torch.cuda.synchronize()
t0 = time.perf_counter()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
for i in range(10, 10 + N // 2):
    bt.update(batches[i], sync=False)
t1 = time.perf_counter()
bt.join()
ev1.record()
torch.cuda.synchronize()
print(f"B={B}: host {1e6 * (t1 - t0) / (N // 2):.1f} us per update call, "
      f"GPU {1e3 * ev0.elapsed_time(ev1) / (N // 2):.1f} us per update")
# time spent inside the C entry point alone
lib0 = bt.engine.lib
orig = lib0.tf_update_heads
acc = [0.0, 0]


def timed(*args):
    t = time.perf_counter()
    r = orig(*args)
    acc[0] += time.perf_counter() - t
    acc[1] += 1
    return r


lib0.tf_update_heads = timed
for i in range(10, 10 + N // 2):
    bt.update(batches[i], sync=False)
bt.join()
lib0.tf_update_heads = orig
print(f"inside tf_update_heads: {1e6 * acc[0] / max(acc[1], 1):.1f} us per call")
pr = cProfile.Profile()
pr.enable()
for i in range(10 + N // 2, 10 + N):
    bt.update(batches[i], sync=False)
pr.disable()
bt.join()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)

# timeline of a few pipelined updates (kernel events only)
import ctypes as C  # noqa: E402
import numpy as np  # noqa: E402
lib = bt.engine.lib
lib.tf_set_profiling(bt.engine.ctx, 1)
for i in range(10, 18):
    bt.update(batches[i], sync=False)
bt.join()
tl = np.zeros(6 * 8)
n = C.c_int32()
lib.tf_timeline(bt.engine.ctx, tl.ctypes.data, 8, C.byref(n))
print("timeline (us): frame start/end, assoc start/end, copy start/end")
for row in tl.reshape(-1, 6)[: n.value]:
    print("  " + "  ".join(f"{1e3 * v:8.1f}" for v in row))
lib.tf_set_profiling(bt.engine.ctx, 0)
