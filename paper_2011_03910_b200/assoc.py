"""Appearance cost, motion gate and assignment (mirror of tf/assoc.py).

``build_cost_matrix`` runs the fp64 cosine kernel (tf_cosine_cost) and
``hungarian_solve`` the on-device exact LAP (tf_lap_dense: one warp per
matrix, sentinel padding + shortest augmenting path with the reference
solver's tie rules). ``apply_gate`` and ``match_with_threshold`` are
elementwise / list bookkeeping kept on the host for API compatibility; the
tracking path performs both inside associate_kernel.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import DimensionError


@dataclass
class Assignment:
    """(track, detection, cost) triples plus leftovers (tf/assoc.py:21-31)."""

    matches: list[tuple[int, int, float]] = field(default_factory=list)
    unmatched_tracks: list[int] = field(default_factory=list)
    unmatched_detections: list[int] = field(default_factory=list)


def build_cost_matrix(track_embeddings: list[np.ndarray], detection_embeddings: list[np.ndarray]) -> np.ndarray:
    """clip(1 - E_t . E_d^T, 0, 2) in fp64 on the GPU (tf/assoc.py:34-46)."""
    nt, nd = len(track_embeddings), len(detection_embeddings)
    if nt == 0 or nd == 0:
        return np.zeros((nt, nd), dtype=np.float64)
    dims = {e.shape for e in track_embeddings} | {e.shape for e in detection_embeddings}
    if len(dims) != 1:
        raise DimensionError(f"mixed embedding shapes in cost matrix: {sorted(dims)}")
    torch = _lib.require_cuda()
    te = torch.as_tensor(np.stack(track_embeddings).astype(np.float32)).cuda()
    de = torch.as_tensor(np.stack(detection_embeddings).astype(np.float32)).cuda()
    out = torch.empty(nt, nd, dtype=torch.float64, device="cuda")
    _lib.check(_lib.load().tf_cosine_cost(nt, nd, te.shape[1], te.data_ptr(), de.data_ptr(), out.data_ptr(),
                                          _lib.stream_handle()))
    return out.cpu().numpy()


def apply_gate(cost: np.ndarray, gate_distances: np.ndarray, gate_threshold: float) -> np.ndarray:
    """+inf where gate > threshold (tf/assoc.py:49-57)."""
    cost = np.asarray(cost, dtype=np.float64)
    gate = np.asarray(gate_distances, dtype=np.float64)
    if cost.shape != gate.shape:
        raise DimensionError(f"cost shape {cost.shape} != gate shape {gate.shape}")
    return np.where(gate > gate_threshold, np.inf, cost)


def solve_batch(costs: list[np.ndarray]) -> list[np.ndarray]:
    """Exact min-cost max-cardinality assignment of many matrices in one launch.

    Returns, per matrix, the matched column of each row or -1."""
    torch = _lib.require_cuda()
    mats = [np.ascontiguousarray(c, dtype=np.float64) for c in costs]
    shapes = np.array([m.shape for m in mats], dtype=np.int32).reshape(-1, 2)
    sizes = np.array([m.size for m in mats], dtype=np.int64)
    coff = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    roff = np.concatenate([[0], np.cumsum(shapes[:, 0])[:-1]]).astype(np.int64)
    flat = np.concatenate([m.ravel() for m in mats]) if mats else np.zeros(0)
    dc = torch.as_tensor(flat if flat.size else np.zeros(1)).cuda()
    out = torch.full((max(int(shapes[:, 0].sum()), 1),), -1, dtype=torch.int32, device="cuda")
    st = torch.zeros(max(len(mats), 1), dtype=torch.int32, device="cuda")
    _lib.check(_lib.load().tf_lap_dense(len(mats), shapes.ctypes.data, coff.ctypes.data, dc.data_ptr(),
                                        roff.ctypes.data, out.data_ptr(), st.data_ptr(), _lib.stream_handle()),
               what="lap")
    status = st.cpu().numpy()
    if status.any():
        raise _lib.status_error(int(status[status != 0][0]), "assignment matrix too large")
    res = out.cpu().numpy()
    return [res[roff[i]:roff[i] + shapes[i, 0]].astype(np.int64) for i in range(len(mats))]


def hungarian_solve(cost: np.ndarray) -> Assignment:
    """Minimum-cost assignment with +inf forbidden edges (tf/assoc.py:60-87)."""
    cost = np.asarray(cost, dtype=np.float64)
    n_rows, n_cols = cost.shape
    if n_rows == 0 or n_cols == 0:
        return Assignment([], list(range(n_rows)), list(range(n_cols)))
    col = solve_batch([cost])[0]
    matches = [(r, int(col[r]), float(cost[r, col[r]])) for r in range(n_rows) if col[r] >= 0]
    mr = {m[0] for m in matches}
    mc = {m[1] for m in matches}
    return Assignment(matches=matches,
                      unmatched_tracks=[r for r in range(n_rows) if r not in mr],
                      unmatched_detections=[c for c in range(n_cols) if c not in mc])


def match_with_threshold(assignment: Assignment, cost: np.ndarray, max_cost: float) -> Assignment:
    """Dissolve matches costing more than max_cost (tf/assoc.py:90-107)."""
    kept, rows, cols = [], list(assignment.unmatched_tracks), list(assignment.unmatched_detections)
    for t, d, v in assignment.matches:
        if v > max_cost:
            rows.append(t)
            cols.append(d)
        else:
            kept.append((t, d, v))
    return Assignment(matches=kept, unmatched_tracks=sorted(rows), unmatched_detections=sorted(cols))
