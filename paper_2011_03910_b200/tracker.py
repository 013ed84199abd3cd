"""Per-frame tracking step and track lifecycle (mirror of tf/tracker.py).

``Tracker`` keeps the reference API -- ``Tracker(config).step(frame_index,
detections) -> TrackerOutput``, ``.tracks``, ``.removed_ids`` -- while the
state lives on the GPU: each step uploads the frame's detections, runs
frame_dets_kernel (confidence filter + bitmask NMS) and associate_kernel
(predict, gate, fp64 cosine cost, exact LAP, max_cost threshold, Kalman
update, EMA, lifecycle, births, records) and reads the records back.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _lib
from .core import BoundingBox, Detection, EMBEDDING_DIM
from .engine import Capacity, Engine
from .errors import DegenerateEmbeddingError, DimensionError
from .motion import CHI2_GATE_95_4DOF, KalmanState, MotionNoise


class TrackState(Enum):
    """Lifecycle states (tf/tracker.py:24-27). The north-star's "new" state is
    ACTIVE with hits == 1: births are ACTIVE immediately."""

    ACTIVE = "active"
    LOST = "lost"
    REMOVED = "removed"


@dataclass
class Track:
    """One identity (tf/tracker.py:30-40); a host snapshot of the device row."""

    track_id: int
    state: TrackState
    kalman: KalmanState
    smooth_embedding: np.ndarray
    last_update_frame: int
    lost_since: int | None = None
    hits: int = 1


STrack = Track   # north-star vocabulary


@dataclass(frozen=True)
class TrackerConfig:
    """Thresholds and lifecycle knobs (tf/tracker.py:43-56)."""

    conf_threshold: float = 0.5
    nms_iou: float = 0.4
    max_cost: float = 0.7
    gate_threshold: float = CHI2_GATE_95_4DOF
    gate_metric: str = "mahalanobis"
    smoothing_alpha: float = 0.9
    max_lost: int = 30
    min_hits: int = 1
    embedding_dim: int = EMBEDDING_DIM
    motion_noise: MotionNoise = MotionNoise()
    # JDE extensions the reference does not have (off = the reference path):
    # lambda-fused cost lambda * cosine + (1 - lambda) * gate distance, and a
    # second association stage on 1 - IoU (tracks ACTIVE before the frame x
    # detections left unmatched, pairs above iou_threshold dissolved)
    motion_lambda: float = 1.0
    iou_stage: bool = False
    iou_threshold: float = 0.5


@dataclass(frozen=True)
class TrackerOutput:
    """Tracks updated in one frame, sorted by id (tf/tracker.py:59-64)."""

    frame_index: int
    records: tuple[tuple[int, BoundingBox, float], ...]


def smooth_embedding(old: np.ndarray, new: np.ndarray, alpha: float) -> np.ndarray:
    """normalize(alpha * old + (1 - alpha) * new) on the GPU (tf/tracker.py:67-71)."""
    if old.shape != new.shape:
        raise DimensionError(f"embedding shapes differ: {old.shape} vs {new.shape}")
    torch = _lib.require_cuda()
    o = torch.as_tensor(np.asarray(old, np.float32).reshape(1, -1)).cuda()
    q = torch.as_tensor(np.asarray(new, np.float32).reshape(1, -1)).cuda()
    out = torch.empty_like(o)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.check(_lib.load().tf_smooth_embedding(1, o.shape[1], o.data_ptr(), q.data_ptr(), float(alpha),
                                               out.data_ptr(), st.data_ptr(), _lib.stream_handle()))
    if int(st.item()):
        raise DegenerateEmbeddingError("smoothed embedding norm too small to normalize")
    return out.cpu().numpy()[0]


def records_from_device(count: int, ids: np.ndarray, boxes: np.ndarray, obj: np.ndarray):
    return tuple((int(ids[i]), BoundingBox(*(float(v) for v in boxes[i])), float(obj[i])) for i in range(count))


class Tracker:
    """Owns all tracks of one sequence; ``step`` must be called in frame order
    (tf/tracker.py:74-159). State is device resident."""

    def __init__(self, config: TrackerConfig | None = None, *, capacity: Capacity | None = None,
                 quantize: bool = False) -> None:
        self.config = config or TrackerConfig()
        cap = capacity or Capacity(streams=1, max_frames=1)
        self._engine = Engine(self.config, cap, quantize=quantize)
        self._snapshot = None

    # -- reference API ---------------------------------------------------------
    def step(self, frame_index: int, detections: list[Detection]) -> TrackerOutput:
        torch = self._engine.torch
        eng = self._engine
        n = len(detections)
        D = self.config.embedding_dim
        boxes = np.zeros((n, 4), np.float64)
        obj = np.zeros(n, np.float64)
        emb = np.zeros((n, D), np.float32)
        has = np.zeros(n, np.uint8)
        for i, d in enumerate(detections):
            boxes[i] = d.box.as_tlwh()
            obj[i] = d.objectness
            if d.embedding is not None:
                e = np.asarray(d.embedding)
                if e.shape != (D,):
                    raise DimensionError(f"embedding shape {e.shape} does not match embedding_dim {D}")
                emb[i] = e
                has[i] = 1
        dev = eng.device
        db = torch.as_tensor(boxes).to(dev, non_blocking=False)
        do = torch.as_tensor(obj).to(dev)
        de = torch.as_tensor(emb).to(dev)
        dh = torch.as_tensor(has).to(dev)
        eng.check(eng.lib.tf_step_detections(eng.ctx, 0, int(frame_index), n, db.data_ptr(), do.data_ptr(),
                                             de.data_ptr(), dh.data_ptr(), eng.records, eng.trace,
                                             _lib.stream_handle()), "step")
        eng.finish()
        self._snapshot = None
        cnt = int(eng.rec_count[0].item())
        if cnt == 0:
            return TrackerOutput(frame_index=frame_index, records=())
        ids = eng.rec_id[0, :cnt].cpu().numpy()
        bx = eng.rec_box[0, :cnt].cpu().numpy()
        ob = eng.rec_obj[0, :cnt].cpu().numpy()
        return TrackerOutput(frame_index=frame_index, records=records_from_device(cnt, ids, bx, ob))

    def _export(self) -> dict:
        if self._snapshot is None:
            self._snapshot = self._engine.export(0)
        return self._snapshot

    @property
    def tracks(self) -> list[Track]:
        """ACTIVE and LOST tracks, survivors first then births (tf/tracker.py:79)."""
        ex = self._export()
        out = []
        for i in range(ex["count"]):
            lost = int(ex["lost_since"][i])
            out.append(Track(
                track_id=int(ex["track_id"][i]),
                state=TrackState.LOST if ex["state"][i] else TrackState.ACTIVE,
                kalman=KalmanState(mean=ex["mean"][i].copy(), covariance=ex["covariance"][i].copy()),
                smooth_embedding=ex["embedding"][i].copy(),
                last_update_frame=int(ex["last_update_frame"][i]),
                lost_since=None if lost < 0 else lost,
                hits=int(ex["hits"][i])))
        return out

    def load_state(self, tracks: list[Track], *, next_id: int, last_frame: int | None) -> None:
        """Resume from a track table: the reference Tracker's ``tracks``,
        ``_next_id`` and ``_last_frame`` at some frame (tf/tracker.py:74-83)
        become this tracker's state (tf_import_tracks), so one frame can be
        re-run on the GPU from the reference's exact state."""
        n = len(tracks)
        D = self.config.embedding_dim
        state = dict(count=n, next_id=int(next_id),
                     last_frame=_lib.NO_FRAME if last_frame is None else int(last_frame),
                     track_id=np.array([t.track_id for t in tracks], np.int64),
                     state=np.array([1 if t.state.value == TrackState.LOST.value else 0 for t in tracks],
                                    np.int32),
                     hits=np.array([t.hits for t in tracks], np.int32),
                     lost_since=np.array([-1 if t.lost_since is None else t.lost_since for t in tracks],
                                         np.int64),
                     last_update_frame=np.array([t.last_update_frame for t in tracks], np.int64),
                     mean=np.array([np.asarray(t.kalman.mean, np.float64) for t in tracks]).reshape(n, 8),
                     covariance=np.array([np.asarray(t.kalman.covariance, np.float64) for t in tracks]
                                         ).reshape(n, 8, 8),
                     embedding=np.array([np.asarray(t.smooth_embedding, np.float32) for t in tracks]
                                        ).reshape(n, D))
        for t in tracks:
            if t.state.value not in (TrackState.ACTIVE.value, TrackState.LOST.value):
                raise ValueError(f"track {t.track_id}: only ACTIVE and LOST tracks are held, got {t.state}")
            if np.shape(t.smooth_embedding) != (D,):
                raise DimensionError(f"track {t.track_id}: embedding shape {np.shape(t.smooth_embedding)} "
                                     f"does not match embedding_dim {D}")
        self._engine.import_(0, state)
        self._snapshot = None

    @classmethod
    def from_reference(cls, tracker, *, capacity: Capacity | None = None, quantize: bool = False) -> "Tracker":
        """A GPU tracker holding a reference ``trackforge.Tracker``'s current
        state (config, tracks, id counter, last frame)."""
        cfg = tracker.config
        kw = {f: getattr(cfg, f) for f in TrackerConfig.__dataclass_fields__ if hasattr(cfg, f)}
        if "motion_noise" in kw:
            mn = kw["motion_noise"]
            kw["motion_noise"] = MotionNoise(**{f: getattr(mn, f) for f in MotionNoise.__dataclass_fields__})
        mine = TrackerConfig(**kw)
        out = cls(mine, capacity=capacity, quantize=quantize)
        out.load_state(list(tracker.tracks), next_id=tracker._next_id, last_frame=tracker._last_frame)
        return out

    @property
    def removed_ids(self) -> set[int]:
        """Ids issued and no longer live: ids are never reused (tf/tracker.py:80, 139-140)."""
        ex = self._export()
        return set(range(1, int(ex["next_id"]))) - {int(v) for v in ex["track_id"]}
