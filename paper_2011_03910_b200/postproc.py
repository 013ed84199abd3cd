"""Raw-output parsing, confidence filter and NMS (mirror of tf/postproc.py).

``parse_output`` normalises every embedding row on the GPU in one batched
launch; ``nms`` runs the bitmask NMS kernel (tf_nms_sets), the same device
routine the tracking path uses inside frame_heads_kernel. ``filter_confidence``
and ``serialize_detections`` are list bookkeeping kept on the host for API
compatibility (the tracking path applies the confidence test on the device).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .core import EMBEDDING_DIM, BoundingBox, Detection, normalize_rows
from .errors import ConfigError, LayoutError

ROW_PREFIX = 6  # 4 box values + objectness + class score (tf/postproc.py:16)


def parse_output(raw: np.ndarray, embedding_dim: int = EMBEDDING_DIM) -> list[Detection]:
    """(n, 6 + D) rows -> Detections with unit fp32 embeddings (tf/postproc.py:19-42)."""
    raw = np.asarray(raw, dtype=np.float64)
    if raw.ndim != 2 or (raw.shape[0] > 0 and raw.shape[1] != ROW_PREFIX + embedding_dim):
        raise LayoutError(f"expected rows of width {ROW_PREFIX + embedding_dim}, got shape {raw.shape}")
    if raw.shape[0] == 0:
        return []
    boxes = [BoundingBox(float(r[0]), float(r[1]), float(r[2]), float(r[3])) for r in raw]
    embs = normalize_rows(raw[:, ROW_PREFIX:]) if embedding_dim > 0 else [None] * raw.shape[0]
    return [Detection(box=b, objectness=float(r[4]), class_score=float(r[5]), embedding=e)
            for b, r, e in zip(boxes, raw, embs)]


def serialize_detections(detections: list[Detection], embedding_dim: int = EMBEDDING_DIM) -> np.ndarray:
    """Inverse of parse_output for normalized detections (tf/postproc.py:45-58)."""
    rows = np.zeros((len(detections), ROW_PREFIX + embedding_dim), dtype=np.float64)
    for i, det in enumerate(detections):
        rows[i, :4] = det.box.as_tlwh()
        rows[i, 4] = det.objectness
        rows[i, 5] = det.class_score
        if embedding_dim > 0:
            if det.embedding is None or det.embedding.shape != (embedding_dim,):
                raise LayoutError(f"detection {i} lacks a {embedding_dim}-dim embedding")
            rows[i, ROW_PREFIX:] = det.embedding
    return rows


def filter_confidence(detections: list[Detection], threshold: float) -> list[Detection]:
    """Keep objectness >= threshold, order preserved (tf/postproc.py:61-65)."""
    if not 0.0 <= threshold <= 1.0:
        raise ConfigError(f"confidence threshold must be in [0, 1], got {threshold}")
    return [d for d in detections if d.objectness >= threshold]


def nms_sets(boxes: np.ndarray, scores: np.ndarray, offsets, thresholds) -> np.ndarray:
    """Batched greedy NMS on the GPU over independent sets; returns keep flags."""
    torch = _lib.require_cuda()
    boxes = np.ascontiguousarray(boxes, dtype=np.float64).reshape(-1, 4)
    scores = np.ascontiguousarray(scores, dtype=np.float64).reshape(-1)
    off = np.ascontiguousarray(offsets, dtype=np.int32)
    thr = np.ascontiguousarray(thresholds, dtype=np.float64)
    n_sets = len(thr)
    if boxes.shape[0] == 0:
        return np.zeros(0, dtype=bool)
    db = torch.as_tensor(boxes).cuda()
    ds = torch.as_tensor(scores).cuda()
    dt = torch.as_tensor(thr).cuda()
    keep = torch.zeros(boxes.shape[0], dtype=torch.uint8, device="cuda")
    st = torch.zeros(n_sets, dtype=torch.int32, device="cuda")
    _lib.check(_lib.load().tf_nms_sets(n_sets, off.ctypes.data, db.data_ptr(), ds.data_ptr(), dt.data_ptr(),
                                        keep.data_ptr(), st.data_ptr(), _lib.stream_handle()), what="nms")
    status = st.cpu().numpy()
    if status.any():
        raise _lib.status_error(int(status[status != 0][0]), "nms set exceeds 1024 boxes")
    return keep.cpu().numpy().astype(bool)


def nms(detections: list[Detection], iou_threshold: float) -> list[Detection]:
    """Greedy NMS, ties to the lower index, survivors in input order (tf/postproc.py:68-89)."""
    if not 0.0 < iou_threshold < 1.0:
        raise ConfigError(f"NMS IoU threshold must be in (0, 1), got {iou_threshold}")
    if not detections:
        return []
    boxes = np.array([d.box.as_tlwh() for d in detections], dtype=np.float64)
    scores = np.array([d.objectness for d in detections], dtype=np.float64)
    keep = nms_sets(boxes, scores, [0, len(detections)], [iou_threshold])
    return [d for d, k in zip(detections, keep) if k]
