"""CPU restatement of the reference tracker path (TEST INFRASTRUCTURE ONLY).

Follows ``trackforge`` 0.1.0 (``/root/reference/pkg/src/trackforge``; ``tf/``
below). The arithmetic uses the same numpy / scipy operations in the same
order as the reference, so on one machine this restatement reproduces the
reference bit for bit (pinned by ``tests/test_oracle_golden.py`` against
vectors the reference produced). The data model is different on purpose:
detections are plain tuples, tracks are ``_TrackRow`` records, and every step
returns the intermediate decisions (kept indices, gated cost entries,
matches) that the GPU parity tests compare.

Errors are raised as :class:`OracleError` whose ``kind`` names the reference
exception class (``tf/errors.py``), so tests can check that the GPU path
raises the matching class.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg
from scipy.optimize import linear_sum_assignment

ROW_PREFIX = 6                      # tf/postproc.py:16
CHI2_GATE_95_4DOF = 9.4877          # tf/motion.py:23
BINARY16_MAX = 65504.0              # tf/core.py:25


class OracleError(Exception):
    """Failure raised by the oracle; ``kind`` is the reference class name."""

    def __init__(self, kind: str, message: str) -> None:
        super().__init__(f"{kind}: {message}")
        self.kind = kind


@dataclass(frozen=True)
class Settings:
    """Mirror of ``TrackerConfig`` + ``MotionNoise`` (tf/tracker.py:43-56,
    tf/motion.py:28-41) plus the pipeline's MIXED switch
    (tf/pipeline.py:436-441)."""

    conf_threshold: float = 0.5
    nms_iou: float = 0.4
    max_cost: float = 0.7
    gate_threshold: float = CHI2_GATE_95_4DOF
    gate_metric: str = "mahalanobis"
    smoothing_alpha: float = 0.9
    max_lost: int = 30
    min_hits: int = 1
    embedding_dim: int = 512
    std_weight_position: float = 1.0 / 20
    std_weight_velocity: float = 1.0 / 160
    std_aspect: float = 1e-2
    std_aspect_velocity: float = 1e-5
    std_aspect_measurement: float = 1e-1
    quantize: bool = False
    # JDE extensions, NOT in the reference (SURVEY.md section 8 name map):
    # defaults are the reference path. Their semantics are defined by this
    # restatement (parity unpinned: no reference implementation exists).
    motion_lambda: float = 1.0          # cost = lambda * cosine + (1 - lambda) * gate distance
    iou_stage: bool = False             # second stage on 1 - IoU
    iou_threshold: float = 0.5


# ---------------------------------------------------------------------------
# tf/core.py
# ---------------------------------------------------------------------------

def check_box(x: float, y: float, w: float, h: float) -> tuple[float, float, float, float]:
    """BoundingBox validation, tf/core.py:37-43."""
    for v in (x, y, w, h):
        if not math.isfinite(v):
            raise OracleError("InvalidBoxError", f"non-finite box field {v!r}")
    if w <= 0 or h <= 0:
        raise OracleError("InvalidBoxError", f"non-positive size w={w} h={h}")
    return (x, y, w, h)


def box_iou(a, b) -> float:
    """tf/core.py:71-80 on (x, y, w, h) tuples; right/bottom/area as in
    tf/core.py:45-55."""
    ax, ay, aw, ah = a
    bx, by, bw, bh = b
    iw = min(ax + aw, bx + bw) - max(ax, bx)
    ih = min(ay + ah, by + bh) - max(ay, by)
    if iw <= 0 or ih <= 0:
        return 0.0
    inter = iw * ih
    union = aw * ah + bw * bh - inter
    return float(min(inter / union, 1.0))


def to_measurement(box) -> np.ndarray:
    """tf/core.py:83-88."""
    x, y, w, h = box
    return np.array([x + w / 2.0, y + h / 2.0, w / h, h], dtype=np.float64)


def from_measurement(m: np.ndarray) -> tuple[float, float, float, float]:
    """tf/core.py:91-97."""
    cx, cy, aspect, h = (float(v) for v in m)
    w = aspect * h
    if h <= 0 or w <= 0:
        raise OracleError("InvalidBoxError", f"measurement implies non-positive size a={aspect} h={h}")
    return check_box(cx - w / 2.0, cy - h / 2.0, w, h)


def unit_vector(values) -> np.ndarray:
    """tf/core.py:100-111: fp64 norm, fp32 result."""
    v = np.asarray(values, dtype=np.float64)
    if not np.all(np.isfinite(v)):
        raise OracleError("DegenerateEmbeddingError", "non-finite embedding")
    norm = float(np.linalg.norm(v))
    if norm < 1e-12:
        raise OracleError("DegenerateEmbeddingError", f"norm {norm!r}")
    return (v / norm).astype(np.float32)


def to_half(values) -> np.ndarray:
    """tf/core.py:124-136: fp32 -> binary16 (RNE) -> fp32."""
    v = np.asarray(values, dtype=np.float32)
    if not np.all(np.isfinite(v)):
        raise OracleError("PrecisionOverflowError", "non-finite value")
    if np.any(np.abs(v) > BINARY16_MAX):
        raise OracleError("PrecisionOverflowError", "beyond binary16 range")
    return v.astype(np.float16).astype(np.float32)


# ---------------------------------------------------------------------------
# tf/postproc.py  (+ the MIXED re-quantisation of tf/pipeline.py:436-441)
# ---------------------------------------------------------------------------

@dataclass
class Det:
    """A parsed detection: tlwh box, objectness, class score, fp32 embedding."""

    box: tuple[float, float, float, float]
    objectness: float
    class_score: float
    embedding: np.ndarray | None


def rows_to_dets(raw: np.ndarray, embedding_dim: int, quantize: bool = False) -> list[Det]:
    """tf/postproc.py:19-42 (+ tf/pipeline.py:436-441 when ``quantize``)."""
    raw = np.asarray(raw, dtype=np.float64)
    if raw.ndim != 2 or (raw.shape[0] > 0 and raw.shape[1] != ROW_PREFIX + embedding_dim):
        raise OracleError("LayoutError", f"bad raw shape {raw.shape}")
    out = []
    for row in raw:
        box = check_box(float(row[0]), float(row[1]), float(row[2]), float(row[3]))
        emb = unit_vector(row[ROW_PREFIX:]) if embedding_dim > 0 else None
        if quantize and emb is not None:
            emb = unit_vector(to_half(emb))
        out.append(Det(box, float(row[4]), float(row[5]), emb))
    return out


def confident(dets: list[Det], threshold: float) -> list[int]:
    """tf/postproc.py:61-65, returned as indices."""
    if not 0.0 <= threshold <= 1.0:
        raise OracleError("ConfigError", f"confidence threshold {threshold}")
    return [i for i, d in enumerate(dets) if d.objectness >= threshold]


def greedy_nms(boxes, scores, threshold: float) -> list[int]:
    """tf/postproc.py:68-89: kept positions in ascending (input) order."""
    if not 0.0 < threshold < 1.0:
        raise OracleError("ConfigError", f"NMS IoU threshold {threshold}")
    n = len(boxes)
    ranked = sorted(range(n), key=lambda i: (-scores[i], i))
    dead = [False] * n
    keep = []
    for k, i in enumerate(ranked):
        if dead[i]:
            continue
        keep.append(i)
        for j in ranked[k + 1:]:
            if not dead[j] and box_iou(boxes[i], boxes[j]) > threshold:
                dead[j] = True
    return sorted(keep)


# ---------------------------------------------------------------------------
# tf/motion.py
# ---------------------------------------------------------------------------

class Motion:
    """Constant-velocity filter of tf/motion.py:52-142 with its exact numpy /
    scipy operations (dense 8x8 matrices, Cholesky solves)."""

    def __init__(self, s: Settings) -> None:
        self.s = s
        self.F = np.eye(8)
        self.F[:4, 4:] = np.eye(4)
        self.H = np.eye(4, 8)

    def _q_std(self, h: float, init: bool) -> np.ndarray:
        s = self.s
        wp, wv = s.std_weight_position, s.std_weight_velocity
        if init:   # tf/motion.py:69-80
            return np.array([2 * wp * h, 2 * wp * h, s.std_aspect, 2 * wp * h,
                             10 * wv * h, 10 * wv * h, s.std_aspect_velocity, 10 * wv * h])
        return np.array([wp * h, wp * h, s.std_aspect, wp * h,   # tf/motion.py:87-98
                         wv * h, wv * h, s.std_aspect_velocity, wv * h])

    def initiate(self, z: np.ndarray):
        z = np.asarray(z, dtype=np.float64)
        h = float(z[3])
        if h <= 0:
            raise OracleError("InvalidMeasurementError", f"height {h}")
        return np.concatenate([z, np.zeros(4)]), np.diag(self._q_std(h, True) ** 2)

    def predict(self, mean, cov):
        h = float(mean[3])
        q = self._q_std(h, False)
        m = self.F @ mean
        p = self.F @ cov @ self.F.T + np.diag(q ** 2)
        return m, (p + p.T) / 2.0

    def project(self, mean, cov):
        h = float(mean[3])
        wp = self.s.std_weight_position
        r = np.array([wp * h, wp * h, self.s.std_aspect_measurement, wp * h])
        return self.H @ mean, self.H @ cov @ self.H.T + np.diag(r ** 2)

    def update(self, mean, cov, z):
        z = np.asarray(z, dtype=np.float64)
        pm, pc = self.project(mean, cov)
        try:
            chol = scipy.linalg.cho_factor(pc, lower=True, check_finite=False)
            gain = scipy.linalg.cho_solve(chol, (cov @ self.H.T).T, check_finite=False).T
        except scipy.linalg.LinAlgError as exc:
            raise OracleError("NumericError", str(exc)) from exc
        m = mean + gain @ (z - pm)
        p = cov - gain @ pc @ gain.T
        return m, (p + p.T) / 2.0

    def gate(self, mean, cov, zs):
        zs = np.atleast_2d(np.asarray(zs, dtype=np.float64))
        pm, pc = self.project(mean, cov)
        try:
            chol = np.linalg.cholesky(pc)
        except np.linalg.LinAlgError as exc:
            raise OracleError("NumericError", str(exc)) from exc
        x = scipy.linalg.solve_triangular(chol, (zs - pm).T, lower=True, check_finite=False)
        return np.sum(x * x, axis=0)


# ---------------------------------------------------------------------------
# tf/assoc.py
# ---------------------------------------------------------------------------

def cosine_costs(track_embs: list[np.ndarray], det_embs: list[np.ndarray]) -> np.ndarray:
    """tf/assoc.py:34-46."""
    if not track_embs or not det_embs:
        return np.zeros((len(track_embs), len(det_embs)), dtype=np.float64)
    shapes = {e.shape for e in track_embs} | {e.shape for e in det_embs}
    if len(shapes) != 1:
        raise OracleError("DimensionError", f"mixed embedding shapes {shapes}")
    t = np.stack(track_embs).astype(np.float64)
    d = np.stack(det_embs).astype(np.float64)
    return np.clip(1.0 - t @ d.T, 0.0, 2.0)


def solve_assignment(cost: np.ndarray):
    """tf/assoc.py:60-87: sentinel padding then scipy's LSAP.

    Returns (matches [(row, col, cost)], unmatched rows, unmatched cols)."""
    cost = np.asarray(cost, dtype=np.float64)
    nr, nc = cost.shape
    if nr == 0 or nc == 0:
        return [], list(range(nr)), list(range(nc))
    n = max(nr, nc)
    finite = cost[np.isfinite(cost)]
    amp = float(np.max(np.abs(finite))) if finite.size else 1.0
    sentinel = 2.0 * n * max(amp, 1.0) + 1.0
    padded = np.full((n, n), sentinel, dtype=np.float64)
    padded[:nr, :nc] = np.where(np.isfinite(cost), cost, sentinel)
    rows, cols = linear_sum_assignment(padded)
    matches = [(int(r), int(c), float(cost[r, c]))
               for r, c in zip(rows, cols)
               if r < nr and c < nc and np.isfinite(cost[r, c])]
    mr = {m[0] for m in matches}
    mc = {m[1] for m in matches}
    return matches, [r for r in range(nr) if r not in mr], [c for c in range(nc) if c not in mc]


def threshold_matches(matches, um_rows, um_cols, max_cost: float):
    """tf/assoc.py:90-107."""
    kept = []
    rows, cols = list(um_rows), list(um_cols)
    for r, c, v in matches:
        if v > max_cost:
            rows.append(r)
            cols.append(c)
        else:
            kept.append((r, c, v))
    return kept, sorted(rows), sorted(cols)


# ---------------------------------------------------------------------------
# tf/tracker.py
# ---------------------------------------------------------------------------

ACTIVE, LOST = "active", "lost"


@dataclass
class _TrackRow:
    track_id: int
    state: str
    mean: np.ndarray
    cov: np.ndarray
    emb: np.ndarray
    last_update_frame: int
    lost_since: int | None = None
    hits: int = 1


@dataclass
class StepTrace:
    """What one step decided, for parity checks against the device."""

    frame_index: int
    records: list                 # [(track_id, (x, y, w, h), objectness)] sorted by id
    kept: list                    # indices into the step's input detections after filter + NMS
    gated: np.ndarray             # gated cost matrix [T, K] (+inf where gated)
    matches: list                 # [(track_id, kept position, cost)] after max_cost
    births: list                  # track ids born this step
    removed: list                 # track ids removed this step


class OracleTracker:
    """Restatement of ``Tracker`` (tf/tracker.py:74-174)."""

    def __init__(self, settings: Settings | None = None) -> None:
        self.s = settings or Settings()
        self.motion = Motion(self.s)
        self.tracks: list[_TrackRow] = []
        self.removed_ids: set[int] = set()
        self.next_id = 1
        self.last_frame: int | None = None
        self.stage2_matches = 0                 # IoU-stage matches (extension), for tests

    def _gates(self, meas: np.ndarray) -> np.ndarray:
        """tf/tracker.py:161-170."""
        if self.s.gate_metric == "mahalanobis":
            return np.stack([self.motion.gate(t.mean, t.cov, meas) for t in self.tracks])
        if self.s.gate_metric == "euclidean":
            centers = np.stack([t.mean[:2] for t in self.tracks])
            delta = centers[:, None, :] - meas[None, :, :2]
            return np.sum(delta * delta, axis=2)
        raise OracleError("ConfigError", f"gate metric {self.s.gate_metric!r}")

    def _iou_stage(self, matches, ur, uc, meas):
        """JDE's IoU association (extension): tracks ACTIVE before this frame
        and unmatched by the first stage x detections still unmatched, both
        ascending; cost 1 - IoU of the predicted track box and the detection's
        box recovered from its measurement; the first stage's exact solve, then
        pairs above ``iou_threshold`` dissolved."""
        rows = [r for r in ur if self.tracks[r].state == ACTIVE]
        if not rows or not uc:
            return matches, ur, uc
        tb = [from_measurement(self.tracks[r].mean[:4]) for r in rows]
        db = [from_measurement(meas[c]) for c in uc]
        iou_cost = np.array([[1.0 - box_iou(a, b) for b in db] for a in tb], dtype=np.float64)
        m2, _, _ = solve_assignment(iou_cost)
        m2, _, _ = threshold_matches(m2, [], [], self.s.iou_threshold)
        self.stage2_matches += len(m2)
        got_r = {rows[i] for i, _, _ in m2}
        got_c = {uc[j] for _, j, _ in m2}
        matches = list(matches) + [(rows[i], uc[j], v) for i, j, v in m2]
        return (matches, [r for r in ur if r not in got_r], [c for c in uc if c not in got_c])

    def step(self, frame_index: int, dets: list[Det]) -> StepTrace:
        """tf/tracker.py:85-159."""
        s = self.s
        if self.last_frame is not None and frame_index <= self.last_frame:
            raise OracleError("OrderingError", f"frame {frame_index} after {self.last_frame}")
        self.last_frame = frame_index

        conf = confident(dets, s.conf_threshold)
        sub = [dets[i] for i in conf]
        kept_sub = greedy_nms([d.box for d in sub], [d.objectness for d in sub], s.nms_iou)
        kept = [conf[i] for i in kept_sub]
        live = [dets[i] for i in kept]
        for d in live:
            if d.embedding is None:
                raise OracleError("DimensionError", "detection without embedding")

        for t in self.tracks:
            t.mean, t.cov = self.motion.predict(t.mean, t.cov)

        meas = (np.stack([to_measurement(d.box) for d in live]) if live
                else np.zeros((0, 4), dtype=np.float64))
        cost = cosine_costs([t.emb for t in self.tracks], [d.embedding for d in live])
        if self.tracks and live:
            g = self._gates(meas)
            if s.motion_lambda != 1.0:                            # JDE fuse_motion (extension)
                cost = s.motion_lambda * cost + (1.0 - s.motion_lambda) * g
            cost = np.where(g > s.gate_threshold, np.inf, cost)   # tf/assoc.py:49-57
        m, ur, uc = solve_assignment(cost)
        matches, ur, uc = threshold_matches(m, ur, uc, s.max_cost)
        if s.iou_stage:
            matches, ur, uc = self._iou_stage(matches, ur, uc, meas)

        emitted = []
        match_ids = []
        for r, c, v in matches:
            t, d = self.tracks[r], live[c]
            t.mean, t.cov = self.motion.update(t.mean, t.cov, meas[c])
            if t.emb.shape != d.embedding.shape:   # tf/tracker.py:67-71
                raise OracleError("DimensionError", "embedding shapes differ")
            t.emb = unit_vector(s.smoothing_alpha * t.emb.astype(np.float64)
                                + (1.0 - s.smoothing_alpha) * d.embedding.astype(np.float64))
            t.state = ACTIVE
            t.lost_since = None
            t.last_update_frame = frame_index
            t.hits += 1
            match_ids.append((t.track_id, c, v))
            if t.hits >= s.min_hits:
                emitted.append((t.track_id, from_measurement(t.mean[:4]), d.objectness))

        for r in ur:
            t = self.tracks[r]
            if t.state == ACTIVE:
                t.state = LOST
                t.lost_since = frame_index

        survivors, removed = [], []
        for t in self.tracks:
            if t.state == LOST and frame_index - t.lost_since >= s.max_lost:
                self.removed_ids.add(t.track_id)
                removed.append(t.track_id)
            else:
                survivors.append(t)
        self.tracks = survivors

        births = []
        for c in uc:
            d = live[c]
            mean, cov = self.motion.initiate(meas[c])
            t = _TrackRow(self.next_id, ACTIVE, mean, cov, d.embedding.copy(), frame_index)
            self.next_id += 1
            self.tracks.append(t)
            births.append(t.track_id)
            if t.hits >= s.min_hits:
                emitted.append((t.track_id, from_measurement(t.mean[:4]), d.objectness))

        emitted.sort(key=lambda rec: rec[0])
        return StepTrace(frame_index, emitted, kept, cost, match_ids, births, removed)
