"""Per-frame comparison of GPU tracker output against the CPU oracle.

TEST INFRASTRUCTURE ONLY: used by ``tests/`` (strict: the first difference
fails the test) and by ``bench.py``'s CPU-baseline leg (counting: the bench
line reports how many of the timed frames matched).

What is compared for one frame (north-star tolerances):

* bit-exact: candidates past the confidence test (count), kept detection
  indices (global anchor codes after NMS), detection -> track id for matches
  and births, record ids (sorted, ``min_hits`` gate);
* within 1e-4 relative: record boxes (posterior tlwh), objectness, match costs
  (the gated cosine cost of tf/assoc.py:34-57).
"""

from __future__ import annotations

import numpy as np

TOL = 1e-4


class FrameCompare:
    """Accumulates per-frame comparisons; ``strict`` raises on the first difference."""

    def __init__(self, strict: bool = True):
        self.strict = strict
        self.frames = 0
        self.records = 0
        self.matches = 0
        self.max_box_rel = 0.0
        self.max_obj_rel = 0.0
        self.max_cost_rel = 0.0
        self.bad_frames: list[tuple[int, str]] = []
        self.kept_exact = self.ids_exact = self.pairs_exact = self.cand_exact = True

    def _fail(self, f, what: str) -> None:
        if self.strict:
            raise AssertionError(f"{what} at frame {f}")
        self.bad_frames.append((int(f), what))

    def check(self, f, trace, gpu_records, gpu_codes, gpu_tracks, gpu_costs, gpu_matched, codes,
              gpu_cand_count=None) -> None:
        """trace: the oracle's StepTrace of this frame; codes: the oracle's
        candidate anchor codes; gpu_*: this frame's GPU outputs as numpy."""
        self.frames += 1
        if gpu_cand_count is not None and int(gpu_cand_count) != len(codes):
            self.cand_exact = False
            self._fail(f, f"candidate count {int(gpu_cand_count)} vs {len(codes)}")
        kept_codes = codes[trace.kept] if len(trace.kept) else np.zeros(0, np.int64)
        if not np.array_equal(np.asarray(gpu_codes, np.int64), kept_codes):
            self.kept_exact = False
            self._fail(f, "kept detections differ")
            return
        want_ids = [r[0] for r in trace.records]
        got_ids = [r[0] for r in gpu_records]
        if got_ids != want_ids:
            self.ids_exact = False
            self._fail(f, f"record ids differ: {got_ids[:8]} vs {want_ids[:8]}")
            return
        for (_, gbox, gobj), (_, wbox, wobj) in zip(gpu_records, trace.records):
            g = np.asarray(gbox.as_tlwh() if hasattr(gbox, "as_tlwh") else gbox, np.float64)
            w = np.asarray(wbox, np.float64)
            rel = float(np.max(np.abs(g - w) / np.maximum(np.abs(w), 1.0)))
            self.max_box_rel = max(self.max_box_rel, rel)
            self.max_obj_rel = max(self.max_obj_rel, abs(gobj - wobj) / max(abs(wobj), 1e-300))
            self.records += 1
        matched = {pos: (tid, cost) for tid, pos, cost in trace.matches}
        births = set(trace.births)
        for k in range(len(trace.kept)):
            if k in matched:
                tid, cost = matched[k]
                if not (gpu_matched[k] == 1 and gpu_tracks[k] == tid):
                    self.pairs_exact = False
                    self._fail(f, f"det {k}: match differs")
                    return
                self.max_cost_rel = max(self.max_cost_rel, abs(gpu_costs[k] - cost) / max(abs(cost), 1e-12))
                self.matches += 1
            elif not (gpu_matched[k] == 0 and int(gpu_tracks[k]) in births):
                self.pairs_exact = False
                self._fail(f, f"det {k}: birth differs")
                return
        for name, v in (("box", self.max_box_rel), ("cost", self.max_cost_rel), ("objectness", self.max_obj_rel)):
            if v > TOL:
                self._fail(f, f"{name} rel err {v:.3e} > {TOL}")

    def summary(self) -> dict:
        return {"frames": self.frames, "records": self.records, "matches": self.matches,
                "candidates_exact": self.cand_exact, "kept_exact": self.kept_exact, "ids_exact": self.ids_exact,
                "pairs_exact": self.pairs_exact, "max_box_rel": self.max_box_rel,
                "max_cost_rel": self.max_cost_rel, "max_obj_rel": self.max_obj_rel, "tolerance": TOL,
                "bad_frames": len(self.bad_frames), "first_bad": self.bad_frames[:3]}
