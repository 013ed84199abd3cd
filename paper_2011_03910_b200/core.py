"""Geometry / embedding primitives (mirror of tf/core.py).

``BoundingBox`` and ``Detection`` are plain host value types, as in the
reference (tf/core.py:28-68). The arithmetic helpers run on the GPU through
the C ABI (``iou`` -> tf_iou_pairs, ``normalize`` -> tf_normalize_rows,
``cosine_distance`` -> tf_cosine_cost, ``quantize_binary16`` ->
tf_quantize_binary16); the tracking path itself performs these operations
inside its kernels and never calls back into Python.
``box_to_measurement`` / ``measurement_to_box`` are value conversions kept on
the host for API compatibility; the device path has its own copies
(tf_device.cuh box_to_meas / meas_to_box).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import DegenerateEmbeddingError, DimensionError, InvalidBoxError, PrecisionOverflowError

EMBEDDING_DIM = 512
BINARY16_MAX = 65504.0


@dataclass(frozen=True)
class BoundingBox:
    """Axis-aligned tlwh box in pixels (tf/core.py:28-58)."""

    x: float
    y: float
    w: float
    h: float

    def __post_init__(self) -> None:
        for name in ("x", "y", "w", "h"):
            value = getattr(self, name)
            if not math.isfinite(value):
                raise InvalidBoxError(f"box field {name!r} is not finite: {value!r}")
        if self.w <= 0 or self.h <= 0:
            raise InvalidBoxError(f"box must have positive size, got w={self.w}, h={self.h}")

    @property
    def right(self) -> float:
        return self.x + self.w

    @property
    def bottom(self) -> float:
        return self.y + self.h

    @property
    def area(self) -> float:
        return self.w * self.h

    def as_tlwh(self) -> tuple[float, float, float, float]:
        return (self.x, self.y, self.w, self.h)


@dataclass(frozen=True, eq=False)
class Detection:
    """One detector output (tf/core.py:61-68)."""

    box: BoundingBox
    objectness: float
    class_score: float = 1.0
    embedding: np.ndarray | None = None


def _dev(a, dtype):
    torch = _lib.require_cuda()
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype).cuda()


def iou_pairs(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Batched iou over [n, 4] tlwh pairs on the GPU (tf/core.py:71-80)."""
    torch = _lib.require_cuda()
    a, b = np.asarray(a, np.float64).reshape(-1, 4), np.asarray(b, np.float64).reshape(-1, 4)
    n = a.shape[0]
    da, db = _dev(a, torch.float64), _dev(b, torch.float64)
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    _lib.check(_lib.load().tf_iou_pairs(n, da.data_ptr(), db.data_ptr(), out.data_ptr(), _lib.stream_handle()))
    return out.cpu().numpy()


def iou(a: BoundingBox, b: BoundingBox) -> float:
    """Intersection-over-union; 0.0 when disjoint (tf/core.py:71-80)."""
    return float(iou_pairs(np.array([a.as_tlwh()]), np.array([b.as_tlwh()]))[0])


def box_to_measurement(box: BoundingBox) -> np.ndarray:
    """(cx, cy, aspect, h) (tf/core.py:83-88)."""
    return np.array([box.x + box.w / 2.0, box.y + box.h / 2.0, box.w / box.h, box.h], dtype=np.float64)


def measurement_to_box(measurement: np.ndarray) -> BoundingBox:
    """Inverse of box_to_measurement (tf/core.py:91-97)."""
    cx, cy, aspect, h = (float(v) for v in measurement)
    w = aspect * h
    if h <= 0 or w <= 0:
        raise InvalidBoxError(f"measurement implies non-positive size: aspect={aspect}, h={h}")
    return BoundingBox(cx - w / 2.0, cy - h / 2.0, w, h)


def normalize_rows(rows: np.ndarray, quantize: bool = False) -> np.ndarray:
    """Row-wise normalize (tf/core.py:100-111) on the GPU; fp64 norm, fp32 out.
    ``quantize`` adds the MIXED binary16 round trip (tf/pipeline.py:436-441)."""
    torch = _lib.require_cuda()
    rows = np.asarray(rows)
    if rows.ndim != 2:
        raise DimensionError(f"expected a 2-D array, got shape {rows.shape}")
    n, d = rows.shape
    if n == 0:
        return np.zeros((0, d), np.float32)
    if d == 0:
        raise DegenerateEmbeddingError("embedding norm too small to normalize: 0.0")
    is64 = rows.dtype != np.float32
    src = _dev(rows, torch.float64 if is64 else torch.float32)
    out = torch.empty(n, d, dtype=torch.float32, device="cuda")
    st = torch.empty(n, dtype=torch.int32, device="cuda")
    _lib.check(_lib.load().tf_normalize_rows(n, d, src.data_ptr() if is64 else None,
                                              None if is64 else src.data_ptr(), d, int(quantize),
                                              out.data_ptr(), st.data_ptr(), _lib.stream_handle()))
    status = st.cpu().numpy()
    bad = np.nonzero(status)[0]
    if bad.size:
        raise _lib.status_error(int(status[bad[0]]), f"row {int(bad[0])} cannot be normalized")
    return out.cpu().numpy()


def normalize(values: np.ndarray) -> np.ndarray:
    """Scale a vector to unit norm, float32 (tf/core.py:100-111)."""
    v = np.asarray(values, dtype=np.float64).reshape(1, -1)
    return normalize_rows(v)[0]


def cosine_distance(a: np.ndarray, b: np.ndarray) -> float:
    """1 - dot(a, b) clipped to [0, 2], fp64 (tf/core.py:114-121)."""
    a, b = np.asarray(a), np.asarray(b)
    if a.shape != b.shape:
        raise DimensionError(f"embedding shapes differ: {a.shape} vs {b.shape}")
    torch = _lib.require_cuda()
    ta, tb = _dev(a.reshape(1, -1), torch.float32), _dev(b.reshape(1, -1), torch.float32)
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    _lib.check(_lib.load().tf_cosine_cost(1, 1, a.size, ta.data_ptr(), tb.data_ptr(), out.data_ptr(),
                                          _lib.stream_handle()))
    return float(out.item())


def quantize_binary16(values: np.ndarray) -> np.ndarray:
    """Round to binary16 (RNE) and widen to float32 (tf/core.py:124-136)."""
    torch = _lib.require_cuda()
    v = np.asarray(values, dtype=np.float32)
    flat = v.reshape(-1)
    if flat.size == 0:
        return v.copy()
    src = _dev(flat, torch.float32)
    out = torch.empty_like(src)
    st = torch.empty(flat.size, dtype=torch.int32, device="cuda")
    _lib.check(_lib.load().tf_quantize_binary16(flat.size, src.data_ptr(), out.data_ptr(), st.data_ptr(),
                                                 _lib.stream_handle()))
    if int(st.max().item()) != 0:
        bad = flat[np.abs(flat) > BINARY16_MAX] if np.all(np.isfinite(flat)) else flat
        raise PrecisionOverflowError(f"value {float(np.max(np.abs(bad)))!r} exceeds binary16 range "
                                     f"(max {BINARY16_MAX})")
    return out.cpu().numpy().reshape(v.shape)
