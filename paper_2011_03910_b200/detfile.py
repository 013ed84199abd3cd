"""Detection-file source: MOT detection CSV + EMB1 embedding sidecar.

Mirrors the reference's file source (``tf/detgen.py:364-484``): the same
function names, file formats, normalisation and error classes. Parsing is
host I/O; the sidecar vectors are normalised on the GPU in one batched
``tf_normalize_rows`` call, and :func:`replay` pushes whole batches of frames
through ``tf_update_detections`` (NMS + association, one launch per batch)
instead of one ``Tracker.step`` per frame.
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from . import motfile
from .core import normalize_rows
from .errors import ConsistencyError, DimensionError, ParseError
from .tracker import TrackerConfig, TrackerOutput, records_from_device

SIDECAR_MAGIC = b"EMB1"


def load_mot_detections(path: str | Path) -> dict[int, np.ndarray]:
    """MOT detection file -> frame -> (n, 6) raw rows (tf/detgen.py:364-396).

    Rows are ``frame,id,bb_left,bb_top,bb_width,bb_height,conf,...``: the id
    field is not read, extra fields are allowed, frames become 0-indexed map
    keys in order of first appearance, the confidence is clamped into [0, 1]
    and the class-score column is 1.0. Errors (ParseError, InvalidBoxError)
    name the offending line (motfile.read_table)."""
    t = motfile.read_table(path, 7, with_id=False, with_conf=True)
    rows = np.empty((t.frame.size, 6), np.float64)
    rows[:, :4] = t.box
    rows[:, 4] = np.minimum(np.maximum(t.conf, 0.0), 1.0)
    rows[:, 5] = 1.0
    return {frame: rows[idx] for frame, idx in motfile.group_by_frame(t.frame)}


def _sidecar_dtype(dim: int) -> np.dtype:
    """One sidecar record: little-endian u32 frame, u32 det_index, dim x f32."""
    return np.dtype([("frame", "<u4"), ("det", "<u4"), ("v", "<f4", (dim,))])


def write_embedding_sidecar(path: str | Path, records: dict[tuple[int, int], np.ndarray], dim: int) -> None:
    """EMB1 sidecar (tf/detgen.py:401-417): magic, u32 dim, then the records in
    ascending (frame, det_index) order. Every vector must have shape (dim,)
    (DimensionError naming the first bad key)."""
    keys = sorted(records)
    vecs = [np.asarray(records[k], dtype=np.float32) for k in keys]
    bad = [k for k, v in zip(keys, vecs) if v.shape != (dim,)]
    if bad:
        raise DimensionError(f"record {bad[0]} has shape {np.shape(records[bad[0]])}, expected ({dim},)")
    table = np.zeros(len(keys), _sidecar_dtype(dim))
    if keys:
        table["frame"] = [k[0] for k in keys]
        table["det"] = [k[1] for k in keys]
        table["v"] = np.stack(vecs)
    Path(path).write_bytes(SIDECAR_MAGIC + struct.pack("<I", dim) + table.tobytes())


def load_embedding_sidecar(path: str | Path, detections: dict[int, np.ndarray], dim: int = 512) -> dict[int, np.ndarray]:
    """Attach normalised sidecar embeddings to a detection map (tf/detgen.py:420-471).

    Exactly one record per (frame, det_index) of the map: a duplicate, missing
    or extra key is a ConsistencyError naming the key, another declared
    dimension a DimensionError. Keys are matched as sorted u64 codes, and
    all vectors are normalised in one GPU call."""
    blob = Path(path).read_bytes()
    if blob[:4] != SIDECAR_MAGIC:
        raise ParseError(f"bad sidecar magic: {blob[:4]!r}")
    if len(blob) < 8:
        raise ParseError("sidecar truncated before the dimension field")
    declared = struct.unpack("<I", blob[4:8])[0]
    if declared != dim:
        raise DimensionError(f"sidecar declares dim={declared}, expected {dim}")
    dt = _sidecar_dtype(dim)
    if (len(blob) - 8) % dt.itemsize:
        raise ParseError(f"sidecar body size {len(blob) - 8} is not a multiple of {dt.itemsize}")
    rec = np.frombuffer(blob, dtype=dt, offset=8)
    code = (rec["frame"].astype(np.uint64) << np.uint64(32)) | rec["det"].astype(np.uint64)
    order = np.argsort(code, kind="stable")
    sc = code[order]
    dup = np.nonzero(sc[1:] == sc[:-1])[0]
    if dup.size:          # the duplicate met first in file order
        pos = int(np.min(order[dup + 1]))
        raise ConsistencyError(f"duplicate sidecar record for {(int(rec['frame'][pos]), int(rec['det'][pos]))}")
    frames = list(detections)
    need = np.concatenate([(np.uint64(f) << np.uint64(32)) + np.arange(detections[f].shape[0], dtype=np.uint64)
                           for f in frames]) if frames else np.zeros(0, np.uint64)
    missing = np.setdiff1d(need, sc)
    if missing.size:
        m = int(missing.min())
        raise ConsistencyError(f"sidecar missing record for {(m >> 32, m & 0xFFFFFFFF)}")
    extra = np.setdiff1d(sc, need)
    if extra.size:
        m = int(extra.min())
        raise ConsistencyError(f"sidecar has record {(m >> 32, m & 0xFFFFFFFF)} with no matching detection")
    # vector content last: the structure is checked before any vector is
    # normalised (the reference normalises while reading, so a file with both
    # a structural and a degenerate-vector fault may name the other one)
    units = normalize_rows(np.ascontiguousarray(rec["v"])) if rec.size else np.zeros((0, dim), np.float32)
    where = order[np.searchsorted(sc, need)]       # record of each needed key, map order
    attached: dict[int, np.ndarray] = {}
    start = 0
    for f in frames:
        n = detections[f].shape[0]
        out = np.empty((n, 6 + dim), np.float64)
        out[:, :6] = detections[f]
        out[:, 6:] = units[where[start:start + n]]
        attached[f] = out
        start += n
    return attached


def file_frames(detections: dict[int, np.ndarray], n_frames: int | None = None, row_width: int | None = None):
    """(frame_index, rows) for frames 0..n_frames-1 of a loaded map; frames
    with no detections give an empty (0, row_width) array (tf/detgen.py:474-484)."""
    n = (max(detections) + 1 if detections else 0) if n_frames is None else n_frames
    width = row_width if row_width is not None else (
        next(iter(detections.values())).shape[1] if detections else 6)
    none = np.zeros((0, width), dtype=np.float64)
    return ((f, detections[f] if f in detections else none) for f in range(n))


def replay(detections: dict[int, np.ndarray], config: TrackerConfig | None = None, *, n_frames: int | None = None,
           batch: int = 32, quantize: bool = False, max_tracks: int = 256) -> list[TrackerOutput]:
    """Track a loaded detection map (rows with embeddings, width 6 + D) and
    return one TrackerOutput per frame -- what the reference's pipeline gets by
    feeding ``file_frames`` through parse_output + Tracker.step
    (tf/pipeline.py:291-302) -- with ``batch`` frames per device launch."""
    from .engine import Capacity
    from .heads import BatchTracker

    config = config or TrackerConfig()
    width = 6 + config.embedding_dim
    frames = list(file_frames(detections, n_frames, width))
    most = max((r.shape[0] for _, r in frames), default=0)
    cap = Capacity(streams=1, max_frames=batch, max_candidates=max(most, 1), max_detections=max(most, 1),
                   max_tracks=max_tracks)
    bt = BatchTracker(1, config, frames_per_update=batch, capacity=cap, quantize=quantize)
    outputs: list[TrackerOutput] = []
    for start in range(0, len(frames), batch):
        chunk = frames[start:start + batch]
        res = bt.update_rows([r for _, r in chunk], np.array([f for f, _ in chunk], np.int64))
        count = res.count.cpu().numpy()
        ids, boxes, objs = res.track_id.cpu().numpy(), res.box.cpu().numpy(), res.objectness.cpu().numpy()
        for i, (f, _) in enumerate(chunk):
            n = int(count[i])
            outputs.append(TrackerOutput(frame_index=f, records=records_from_device(n, ids[i, :n], boxes[i, :n],
                                                                                     objs[i, :n]) if n else ()))
    return outputs
