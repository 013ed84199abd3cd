"""Owner of one C-ABI context: device track tables for S streams plus the
device output buffers of an update. Everything here is plumbing around the
CUDA path; there is no host-side compute of tracking results.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _lib
from .errors import ConfigError


@dataclass(frozen=True)
class Capacity:
    """Fixed device capacities (tf_capacity). Overflow raises CapacityError."""

    streams: int = 1
    max_frames: int = 32           # frames per update (streams x B)
    max_candidates: int = 512      # per frame, after the confidence test
    max_detections: int = 256      # per frame, after NMS
    max_tracks: int = 256          # per stream, ACTIVE + LOST


GATE_METRICS = {"mahalanobis": 0, "euclidean": 1}


def make_config(cfg, quantize: bool = False) -> _lib.TfConfig:
    """TrackerConfig (tf/tracker.py:43-56) -> tf_config."""
    n = cfg.motion_noise
    return _lib.TfConfig(
        conf_threshold=float(cfg.conf_threshold), nms_iou=float(cfg.nms_iou), max_cost=float(cfg.max_cost),
        gate_threshold=float(cfg.gate_threshold), smoothing_alpha=float(cfg.smoothing_alpha),
        std_weight_position=float(n.std_weight_position), std_weight_velocity=float(n.std_weight_velocity),
        std_aspect=float(n.std_aspect), std_aspect_velocity=float(n.std_aspect_velocity),
        std_aspect_measurement=float(n.std_aspect_measurement),
        # unknown metric names are carried as 2 and rejected when gating is needed,
        # as the reference rejects them lazily in _gate_matrix (tf/tracker.py:161-170)
        gate_metric=GATE_METRICS.get(cfg.gate_metric, 2), max_lost=int(cfg.max_lost),
        min_hits=int(cfg.min_hits), embedding_dim=int(cfg.embedding_dim),
        quantize_binary16=int(bool(quantize)),
        # JDE extensions (off by default: the reference path)
        iou_stage=int(bool(getattr(cfg, "iou_stage", False))),
        motion_lambda=float(getattr(cfg, "motion_lambda", 1.0)),
        motion_weight=1.0 - float(getattr(cfg, "motion_lambda", 1.0)),
        iou_threshold=float(getattr(cfg, "iou_threshold", 0.5)))


class Engine:
    """tf_ctx wrapper with preallocated device record / trace buffers."""

    def __init__(self, cfg, capacity: Capacity, quantize: bool = False, device=None):
        torch = _lib.require_cuda()
        self.lib = _lib.load()
        if cfg.embedding_dim < 1:
            raise ConfigError(f"embedding_dim must be >= 1, got {cfg.embedding_dim}")
        self.torch = torch
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.cap = capacity
        self.dim = int(cfg.embedding_dim)
        self._cfg = make_config(cfg, quantize)
        ccap = _lib.TfCapacity(capacity.streams, capacity.max_frames, capacity.max_candidates,
                               capacity.max_detections, capacity.max_tracks, 0)
        handle = C.c_void_p()
        with torch.cuda.device(self.device):
            code = self.lib.tf_create(C.byref(self._cfg), C.byref(ccap), self.device.index, C.byref(handle))
        if code != 0:
            raise _lib.status_error(code, f"tf_create failed ({self.lib.tf_status_name(code).decode()}); "
                                          f"capacity {capacity} may not fit this device")
        self.ctx = handle
        F, R = capacity.max_frames, capacity.max_detections
        z = dict(device=self.device)
        self.rec_count = torch.zeros(F, dtype=torch.int32, **z)
        self.rec_id = torch.zeros(F, R, dtype=torch.int64, **z)
        self.rec_box = torch.zeros(F, R, 4, dtype=torch.float64, **z)
        self.rec_obj = torch.zeros(F, R, dtype=torch.float64, **z)
        self.tr_cand = torch.zeros(F, dtype=torch.int32, **z)
        self.tr_det = torch.zeros(F, dtype=torch.int32, **z)
        self.tr_code = torch.full((F, R), -1, dtype=torch.int32, **z)
        self.tr_track = torch.full((F, R), -1, dtype=torch.int64, **z)
        self.tr_cost = torch.zeros(F, R, dtype=torch.float64, **z)
        self.tr_matched = torch.zeros(F, R, dtype=torch.int32, **z)
        self.records = _lib.TfRecords(self.rec_count.data_ptr(), self.rec_id.data_ptr(), self.rec_box.data_ptr(),
                                      self.rec_obj.data_ptr(), R, 0)
        self.trace = _lib.TfTrace(self.tr_cand.data_ptr(), self.tr_det.data_ptr(), self.tr_code.data_ptr(),
                                  self.tr_track.data_ptr(), self.tr_cost.data_ptr(), self.tr_matched.data_ptr())

    def close(self):
        if getattr(self, "ctx", None) is not None and self.ctx.value:
            self.lib.tf_destroy(self.ctx)
            self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- calls ---------------------------------------------------------------
    def check(self, code: int, what: str) -> None:
        _lib.check(code, self.ctx, what)

    def finish(self, stream=None) -> None:
        self.check(self.lib.tf_finish(self.ctx, _lib.stream_handle(stream)), "update")

    def reset_stream(self, s: int) -> None:
        self.check(self.lib.tf_reset_stream(self.ctx, s, _lib.stream_handle()), "reset")

    def export(self, s: int) -> dict:
        """Host copy of stream s's track table (synchronising)."""
        import numpy as np

        T, D = self.cap.max_tracks, self.dim
        out = dict(track_id=np.zeros(T, np.int64), state=np.zeros(T, np.int32), hits=np.zeros(T, np.int32),
                   lost_since=np.zeros(T, np.int64), last_update_frame=np.zeros(T, np.int64),
                   mean=np.zeros((T, 8)), covariance=np.zeros((T, 8, 8)), embedding=np.zeros((T, D), np.float32))
        ex = _lib.TfTrackExport()
        for k in ("track_id", "state", "hits", "lost_since", "last_update_frame", "mean", "covariance",
                  "embedding"):
            setattr(ex, k, out[k].ctypes.data)
        self.check(self.lib.tf_export_tracks(self.ctx, s, C.byref(ex), _lib.stream_handle()), "export")
        n = ex.count
        res = {k: v[:n] for k, v in out.items()}
        res["count"], res["next_id"], res["last_frame"] = n, ex.next_id, ex.last_frame
        return res

    def import_(self, s: int, state: dict) -> None:
        """Make ``state`` (the dict ``export`` returns) stream s's track table
        (tf_import_tracks; synchronising)."""
        import numpy as np

        n = int(state["count"])
        D = self.dim
        arrs = dict(track_id=np.ascontiguousarray(state["track_id"][:n], np.int64),
                    state=np.ascontiguousarray(state["state"][:n], np.int32),
                    hits=np.ascontiguousarray(state["hits"][:n], np.int32),
                    lost_since=np.ascontiguousarray(state["lost_since"][:n], np.int64),
                    last_update_frame=np.ascontiguousarray(state["last_update_frame"][:n], np.int64),
                    mean=np.ascontiguousarray(np.reshape(state["mean"][:n], (n, 8)), np.float64),
                    covariance=np.ascontiguousarray(np.reshape(state["covariance"][:n], (n, 8, 8)), np.float64),
                    embedding=np.ascontiguousarray(np.reshape(state["embedding"][:n], (n, D)), np.float32))
        ex = _lib.TfTrackExport()
        ex.count, ex.next_id, ex.last_frame = n, int(state["next_id"]), int(state["last_frame"])
        for k, v in arrs.items():
            setattr(ex, k, v.ctypes.data)
        self.check(self.lib.tf_import_tracks(self.ctx, s, C.byref(ex), _lib.stream_handle()), "import")
