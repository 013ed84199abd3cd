"""Helpers that run the CPU oracle on exactly the tensors the GPU consumed."""

from __future__ import annotations

import numpy as np

from oracle import heads as oh
from oracle import tracker as ot


def host_frames(out, frames):
    """Copy frames of a HeadOutputs batch to numpy (per-scale [24,H,W] / [D,H,W])."""
    heads = [h.detach().cpu().numpy() for h in out.heads]
    embs = [e.detach().cpu().contiguous().numpy() for e in out.embs]
    return [([h[f] for h in heads], [e[f] for e in embs]) for f in frames]


def oracle_settings(cfg, quantize=False) -> ot.Settings:
    n = cfg.motion_noise
    return ot.Settings(conf_threshold=cfg.conf_threshold, nms_iou=cfg.nms_iou, max_cost=cfg.max_cost,
                       gate_threshold=cfg.gate_threshold, gate_metric=cfg.gate_metric,
                       smoothing_alpha=cfg.smoothing_alpha, max_lost=cfg.max_lost, min_hits=cfg.min_hits,
                       embedding_dim=cfg.embedding_dim, std_weight_position=n.std_weight_position,
                       std_weight_velocity=n.std_weight_velocity, std_aspect=n.std_aspect,
                       std_aspect_velocity=n.std_aspect_velocity,
                       std_aspect_measurement=n.std_aspect_measurement, quantize=quantize,
                       motion_lambda=getattr(cfg, "motion_lambda", 1.0), iou_stage=getattr(cfg, "iou_stage", False),
                       iou_threshold=getattr(cfg, "iou_threshold", 0.5))


class FrameCompare:
    """Accumulates per-frame comparisons of GPU output against the oracle."""

    def __init__(self):
        self.frames = 0
        self.records = 0
        self.max_box_rel = 0.0
        self.max_obj_rel = 0.0
        self.max_cost_rel = 0.0
        self.matches = 0

    def check(self, f, trace, gpu_records, gpu_codes, gpu_tracks, gpu_costs, gpu_matched, codes):
        """trace: oracle StepTrace; gpu_*: numpy arrays of this frame."""
        self.frames += 1
        kept_codes = codes[trace.kept] if len(trace.kept) else np.zeros(0, np.int64)
        assert np.array_equal(np.asarray(gpu_codes, np.int64), kept_codes), f"kept detections differ at frame {f}"
        want_ids = [r[0] for r in trace.records]
        got_ids = [r[0] for r in gpu_records]
        assert got_ids == want_ids, f"record ids differ at frame {f}: {got_ids[:8]} vs {want_ids[:8]}"
        for (gid, gbox, gobj), (_, wbox, wobj) in zip(gpu_records, trace.records):
            g = np.asarray(gbox.as_tlwh() if hasattr(gbox, "as_tlwh") else gbox, np.float64)
            w = np.asarray(wbox, np.float64)
            rel = np.max(np.abs(g - w) / np.maximum(np.abs(w), 1.0))
            self.max_box_rel = max(self.max_box_rel, float(rel))
            self.max_obj_rel = max(self.max_obj_rel, abs(gobj - wobj) / max(abs(wobj), 1e-300))
            self.records += 1
        # association pairs: detection k -> track id (matched or born), costs of matches
        matched = {pos: (tid, cost) for tid, pos, cost in trace.matches}
        births = set(trace.births)
        for k in range(len(trace.kept)):
            if k in matched:
                tid, cost = matched[k]
                assert gpu_matched[k] == 1 and gpu_tracks[k] == tid, f"frame {f} det {k}: match differs"
                self.max_cost_rel = max(self.max_cost_rel, abs(gpu_costs[k] - cost) / max(abs(cost), 1e-12))
                self.matches += 1
            else:
                assert gpu_matched[k] == 0 and int(gpu_tracks[k]) in births, f"frame {f} det {k}: birth differs"
        assert self.max_box_rel <= 1e-4, f"box rel err {self.max_box_rel}"
        assert self.max_cost_rel <= 1e-4, f"cost rel err {self.max_cost_rel}"
        assert self.max_obj_rel <= 1e-4, f"objectness rel err {self.max_obj_rel}"


def run_oracle_frame(trk: ot.OracleTracker, frame_index, heads, embs, quantize=False):
    codes, rows = oh.decode_frame(heads, embs, trk.s.conf_threshold)
    trace = trk.step(frame_index, ot.rows_to_dets(rows, trk.s.embedding_dim, quantize))
    return codes, trace
