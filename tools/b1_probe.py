"""Small-batch timeline probe: cfg1 with B frames per update (default 1),
pipelined; prints the host time per update call, the device time per update,
and the first updates' kernel timeline (tf_timeline)."""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2011_03910_b200 as p  # noqa: E402
from paper_2011_03910_b200 import synth  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
N = int(sys.argv[2]) if len(sys.argv) > 2 else 200
gen = synth.make("cfg1", device="cuda", seed=0)
batches = [gen.next_batch(B) for _ in range(N)]
bt = p.BatchTracker(1, frames_per_update=B, pipeline=True)
lib = bt.engine.lib
for b in batches[:10]:
    bt.update(b, sync=False)
bt.finish()
lib.tf_set_profiling(bt.engine.ctx, 1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
t0 = time.perf_counter()
for b in batches[10:]:
    bt.update(b, sync=False)
t1 = time.perf_counter()
bt.join()
e1.record()
e1.synchronize()
n = N - 10
print(f"B={B} host_us_per_update={1e6 * (t1 - t0) / n:.1f} device_us_per_update={1e3 * e0.elapsed_time(e1) / n:.1f}")
tl = np.zeros(6 * 64)
ntl = C.c_int32()
lib.tf_timeline(bt.engine.ctx, tl.ctypes.data, 64, C.byref(ntl))
tl = tl[:6 * min(ntl.value, 64)].reshape(-1, 6)
for row in tl[:12]:
    print(" ".join(f"{1e3 * v:8.1f}" for v in row[:4]))
