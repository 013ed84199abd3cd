"""Helpers that run the CPU oracle on exactly the tensors the GPU consumed."""

from __future__ import annotations

import numpy as np

from oracle import heads as oh
from oracle import tracker as ot
from oracle.compare import FrameCompare   # noqa: F401  (re-exported for the tests)


def host_frames(out, frames):
    """Copy the given frames of a HeadOutputs batch to numpy (per-scale
    [24,H,W] / [D,H,W]); only those frames cross to the host, so full-size
    configs (512 streams) can be sampled."""
    import torch

    frames = list(frames)
    if not frames:
        return []
    idx = torch.as_tensor(frames, dtype=torch.long, device=out.heads[0].device)
    heads = [h.detach().index_select(0, idx).cpu().numpy() for h in out.heads]
    embs = [e.detach().index_select(0, idx).cpu().contiguous().numpy() for e in out.embs]
    return [([h[i] for h in heads], [e[i] for e in embs]) for i in range(len(frames))]


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


def run_oracle_frame(trk: ot.OracleTracker, frame_index, heads, embs, quantize=False):
    codes, rows = oh.decode_frame(heads, embs, trk.s.conf_threshold)
    trace = trk.step(frame_index, ot.rows_to_dets(rows, trk.s.embedding_dim, quantize))
    return codes, trace
