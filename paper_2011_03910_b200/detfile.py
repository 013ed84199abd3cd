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

from .core import normalize_rows
from .errors import ConsistencyError, DimensionError, InvalidBoxError, ParseError
from .tracker import TrackerConfig, TrackerOutput, records_from_device

SIDECAR_MAGIC = b"EMB1"


def load_mot_detections(path: str | Path) -> dict[int, np.ndarray]:
    """Parse a MOT detection file into frame -> (n, 6) raw rows (tf/detgen.py:364-396).

    Rows are ``frame,id,bb_left,bb_top,bb_width,bb_height,conf,...``; frames
    are 1-indexed in the file and 0-indexed in the map (insertion order = first
    appearance), the id field is ignored, extra fields are allowed and the
    confidence is clamped into [0, 1]."""
    per_frame: dict[int, list[np.ndarray]] = {}
    with open(path, "r", encoding="utf-8") as handle:
        for lineno, line in enumerate(handle, start=1):
            line = line.strip()
            if not line:
                continue
            parts = line.split(",")
            if len(parts) < 7:
                raise ParseError(f"line {lineno}: expected at least 7 fields, got {len(parts)}")
            try:
                frame = int(float(parts[0]))
                x, y, w, h = (float(v) for v in parts[2:6])
                conf = float(parts[6])
            except ValueError as exc:
                raise ParseError(f"line {lineno}: non-numeric field ({exc})") from exc
            if frame < 1:
                raise ParseError(f"line {lineno}: frame index must be >= 1, got {frame}")
            if w <= 0 or h <= 0:
                raise InvalidBoxError(f"line {lineno}: non-positive box size w={w}, h={h}")
            conf = min(max(conf, 0.0), 1.0)
            per_frame.setdefault(frame - 1, []).append(np.array([x, y, w, h, conf, 1.0], dtype=np.float64))
    return {frame: np.stack(rows) for frame, rows in per_frame.items()}


def write_embedding_sidecar(path: str | Path, records: dict[tuple[int, int], np.ndarray], dim: int) -> None:
    """Magic, u32 dim, then (u32 frame, u32 det_index, dim x f32) records in key order (tf/detgen.py:401-417)."""
    keys = sorted(records)
    with open(path, "wb") as handle:
        handle.write(SIDECAR_MAGIC)
        handle.write(struct.pack("<I", dim))
        for frame, det_index in keys:
            vector = np.asarray(records[(frame, det_index)], dtype=np.float32)
            if vector.shape != (dim,):
                raise DimensionError(f"record ({frame}, {det_index}) has shape {vector.shape}, expected ({dim},)")
            handle.write(struct.pack("<II", frame, det_index))
            handle.write(vector.tobytes())


def load_embedding_sidecar(path: str | Path, detections: dict[int, np.ndarray], dim: int = 512) -> dict[int, np.ndarray]:
    """Attach normalised sidecar embeddings to a detection map (tf/detgen.py:420-471).

    Exactly one record per (frame, det_index) of the map: a missing, extra or
    duplicate key is a ConsistencyError, another declared dimension a
    DimensionError. All vectors are normalised in one GPU call."""
    blob = Path(path).read_bytes()
    if blob[:4] != SIDECAR_MAGIC:
        raise ParseError(f"bad sidecar magic: {blob[:4]!r}")
    if len(blob) < 8:
        raise ParseError("sidecar truncated before the dimension field")
    declared = struct.unpack("<I", blob[4:8])[0]
    if declared != dim:
        raise DimensionError(f"sidecar declares dim={declared}, expected {dim}")
    record_size = 8 + 4 * dim
    body = blob[8:]
    if len(body) % record_size != 0:
        raise ParseError(f"sidecar body size {len(body)} is not a multiple of {record_size}")
    n = len(body) // record_size
    rec = np.frombuffer(body, dtype=np.dtype([("frame", "<u4"), ("det", "<u4"), ("v", "<f4", (dim,))]), count=n)
    index: dict[tuple[int, int], int] = {}
    for i, (frame, det_index) in enumerate(zip(rec["frame"].tolist(), rec["det"].tolist())):
        key = (frame, det_index)
        if key in index:
            raise ConsistencyError(f"duplicate sidecar record for {key}")
        index[key] = i
    needed = {(frame, det_index) for frame, rows in detections.items() for det_index in range(rows.shape[0])}
    missing = needed - index.keys()
    if missing:
        raise ConsistencyError(f"sidecar missing record for {min(missing)}")
    extra = index.keys() - needed
    if extra:
        raise ConsistencyError(f"sidecar has record {min(extra)} with no matching detection")
    units = normalize_rows(np.ascontiguousarray(rec["v"])) if n else np.zeros((0, dim), np.float32)
    attached: dict[int, np.ndarray] = {}
    for frame, rows in detections.items():
        out = np.zeros((rows.shape[0], 6 + dim), dtype=np.float64)
        out[:, :6] = rows
        for det_index in range(rows.shape[0]):
            out[det_index, 6:] = units[index[(frame, det_index)]]
        attached[frame] = out
    return attached


def file_frames(detections: dict[int, np.ndarray], n_frames: int | None = None, row_width: int | None = None):
    """(frame_index, rows) over a loaded map; missing frames yield no rows (tf/detgen.py:474-484)."""
    if n_frames is None:
        n_frames = max(detections) + 1 if detections else 0
    if row_width is None:
        row_width = next(iter(detections.values())).shape[1] if detections else 6
    empty = np.zeros((0, row_width), dtype=np.float64)
    for frame_index in range(n_frames):
        yield frame_index, detections.get(frame_index, empty)


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
