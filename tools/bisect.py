import sys, torch
sys.path.insert(0, '.')
import paper_2011_03910_b200 as p
from paper_2011_03910_b200 import synth
mc, md, mt, steps = (int(x) for x in sys.argv[1:5])
gen = synth.make("cfg2", device="cuda")
cap = p.Capacity(streams=1, max_frames=8, max_candidates=mc, max_detections=md, max_tracks=mt)
bt = p.BatchTracker(1, frames_per_update=8, capacity=cap)
for i in range(steps):
    r = bt.update(gen.next_batch(8), trace=True)
    tr = bt.trace(8)
    print(i, "cand", tr["cand_count"].tolist(), "det", tr["det_count"].tolist(), "T", bt.export(0)["count"], flush=True)
print("OK", mc, md, mt)
