"""Config 4 step as G pipelined stream groups: the decode of group g+1 (caller's
stream) overlaps the association of group g (context stream).
Usage: python tools/group_probe.py S G [steps]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2011_03910_b200 as p  # noqa: E402
from paper_2011_03910_b200 import synth  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 512
G = int(sys.argv[2]) if len(sys.argv) > 2 else 2
K = int(sys.argv[3]) if len(sys.argv) > 3 else 4
B = 8
gen = synth.make("cfg4", device="cuda", seed=7, streams=S)
cap = p.Capacity(streams=S, max_frames=S * B, max_candidates=192, max_detections=96, max_tracks=160)
bt = p.BatchTracker(S, frames_per_update=B, capacity=cap, pipeline=G > 1)
sg = S // G


def step(b):
    for g in range(G):
        sub = p.HeadOutputs(tuple(h[g * sg * B:(g + 1) * sg * B] for h in b.heads),
                            tuple(e[g * sg * B:(g + 1) * sg * B] for e in b.embs))
        bt.update(sub, stream_begin=g * sg, n_streams=sg, sync=False)
    bt.join()


for _ in range(3):
    b = gen.next_batch(B)
    step(b)
    torch.cuda.synchronize()
    del b
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ms = 0.0
for _ in range(K):
    b = gen.next_batch(B)
    torch.cuda.synchronize()
    e0.record()
    step(b)
    e1.record()
    e1.synchronize()
    ms += e0.elapsed_time(e1)
    del b
bt.finish()
print(f"S={S} G={G} ms_per_step={ms / K:.3f} frames_per_s={S * B * K / (ms / 1e3):.0f}")
