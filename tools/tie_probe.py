"""Why the association falls back to the full scipy-order solve (config 2 by
default): counters per frame from the phase statistics.
Usage: python tools/tie_probe.py [cfg] [updates] [B]"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2011_03910_b200 as p  # noqa: E402
from paper_2011_03910_b200 import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
U = int(sys.argv[2]) if len(sys.argv) > 2 else 25
B = int(sys.argv[3]) if len(sys.argv) > 3 else 8
gen = synth.make(cfg, device="cuda", seed=0)
cap = p.Capacity(streams=1, max_frames=B, max_candidates=512, max_detections=256, max_tracks=512)
bt = p.BatchTracker(1, frames_per_update=B, capacity=cap)
lib = bt.engine.lib
lib.tf_set_profiling(bt.engine.ctx, 2)
for _ in range(U):
    bt.update(gen.next_batch(B))
ph = np.zeros(40, np.int64)
lib.tf_phase_stats(bt.engine.ctx, ph.ctypes.data)
fr = max(int(ph[11]), 1)
print(json.dumps({"cfg": cfg, "frames": int(ph[11]), "full_solves": int(ph[8]),
                  "undecided_gt32_active_rows": int(ph[32]), "alternative_found": int(ph[33]),
                  "star_runner_up": int(ph[34]), "edge_lists_overflow": int(ph[35]),
                  "full_restatement_us_per_solve": round(float(ph[20]) / max(int(ph[8]), 1) / 1965, 1),
                  "tracks_per_frame": round(float(ph[12]) / fr, 1), "dets_per_frame": round(float(ph[13]) / fr, 1)}))
