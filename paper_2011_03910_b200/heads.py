"""Batched ``update(head_outputs) -> online_tracks`` over S streams x B frames.

This is the north-star entry point: the JDE/YOLO head tensors of a batch go
in (device tensors, or pinned host tensors for the end-to-end path), and the
per-frame online tracks come out, with per-frame semantics identical to
``parse_output`` + ``Tracker.step`` of the reference (tf/postproc.py:19-42,
tf/tracker.py:85-159, call site tf/pipeline.py:291-302).

Head layout (see oracle/heads.py for the pinned decode semantics):
  head[i]  [S*B, 24, H_i, W_i] fp32, channel 6a+k (k: tx, ty, tw, th, bg, fg)
  emb[i]   [S*B, D, H_i, W_i]  fp32, any strides (channels_last is the fast path)
with scales in candidate order (stride 32, 16, 8) and frames stream-major.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .engine import Capacity, Engine
from .errors import LayoutError
from .tracker import TrackerConfig, records_from_device

ROW_WIDTH = 6   # parse_output row prefix: tlwh, objectness, class score (tf/postproc.py:16)

INPUT_W, INPUT_H = 1088, 608
IMAGE_W, IMAGE_H = 1920, 1080
STRIDES = (32, 16, 8)
GRID = {32: (19, 34), 16: (38, 68), 8: (76, 136)}
ANCHORS = {
    8: ((8.0, 24.0), (11.0, 34.0), (16.0, 48.0), (23.0, 68.0)),
    16: ((32.0, 96.0), (45.0, 135.0), (64.0, 192.0), (90.0, 271.0)),
    32: ((128.0, 384.0), (180.0, 540.0), (256.0, 640.0), (512.0, 640.0)),
}
TOTAL_ANCHORS = sum(4 * h * w for h, w in GRID.values())   # 54,264
N_CELLS = sum(h * w for h, w in GRID.values())             # 13,566


def letterbox() -> tuple[float, float, float]:
    """(scale_inv, pad_x, pad_y) of the JDE letterbox 1920x1080 -> 1088x608."""
    ratio = min(INPUT_W / IMAGE_W, INPUT_H / IMAGE_H)
    new_w, new_h = round(IMAGE_W * ratio), round(IMAGE_H * ratio)
    return IMAGE_H / INPUT_H, (INPUT_W - new_w) / 2.0, (INPUT_H - new_h) / 2.0


@dataclass
class HeadOutputs:
    """Network outputs of one batch: three head tensors and three embedding maps."""

    heads: tuple   # 3 x torch.Tensor [N, 24, H, W]
    embs: tuple    # 3 x torch.Tensor [N, D, H, W]

    @property
    def frames(self) -> int:
        return int(self.heads[0].shape[0])

    def half(self) -> "HeadOutputs":
        """binary16 copy (the MIXED-precision input mode: heads emitted in fp16
        by the network), keeping each tensor's memory format."""
        import torch
        fmt = [torch.channels_last if e.is_contiguous(memory_format=torch.channels_last) and not e.is_contiguous()
               else torch.contiguous_format for e in self.embs]
        return HeadOutputs(tuple(h.half() for h in self.heads),
                           tuple(e.half().contiguous(memory_format=m) for e, m in zip(self.embs, fmt)))


@dataclass
class OnlineTracks:
    """Per-frame records of one update; device tensors plus host accessors."""

    count: object        # [F] int32
    track_id: object     # [F, R] int64
    box: object          # [F, R, 4] float64 tlwh
    objectness: object   # [F, R] float64
    frame_index: np.ndarray
    B: int

    def records(self, stream: int, b: int):
        f = stream * self.B + b
        n = int(self.count[f])
        return records_from_device(n, np.asarray(self.track_id[f, :n].cpu() if hasattr(self.track_id, "cpu")
                                                 else self.track_id[f, :n]),
                                   np.asarray(self.box[f, :n].cpu() if hasattr(self.box, "cpu") else self.box[f, :n]),
                                   np.asarray(self.objectness[f, :n].cpu() if hasattr(self.objectness, "cpu")
                                              else self.objectness[f, :n]))


def _dtype_code(t) -> int | None:
    """tf_heads.dtype of a head / embedding tensor: 0 fp32, 1 binary16 (the
    MIXED-precision input mode, network heads emitted in fp16); None otherwise."""
    return {"torch.float32": 0, "torch.float16": 1}.get(str(t.dtype))


def _scale_desc(head, emb, stride: int, dim: int) -> _lib.TfHeadScale:
    h, w = GRID[stride]
    if tuple(head.shape[1:]) != (24, h, w):
        raise LayoutError(f"head of stride {stride} must be [N, 24, {h}, {w}], got {tuple(head.shape)}")
    if tuple(emb.shape[2:]) != (h, w) or emb.shape[0] != head.shape[0]:
        raise LayoutError(f"embedding map of stride {stride} must be [N, D, {h}, {w}], got {tuple(emb.shape)}")
    # parse_output rejects rows whose width is not 6 + embedding_dim (tf/postproc.py:25-29)
    if emb.shape[1] != dim:
        raise LayoutError(f"embedding map of stride {stride} has {emb.shape[1]} channels, "
                          f"expected embedding_dim {dim}")
    if emb.device != head.device:
        raise LayoutError(f"head and embedding map of stride {stride} are on different devices "
                          f"({head.device} vs {emb.device})")
    hs = head.stride()
    if hs[3] != 1 or hs[2] != w:
        raise LayoutError("head planes must have contiguous H*W planes")
    if _dtype_code(head) is None or emb.dtype != head.dtype:
        raise LayoutError(f"heads and embedding maps must both be float32 or both float16, got {head.dtype}/{emb.dtype}")
    es = emb.stride()
    d = _lib.TfHeadScale(head=head.data_ptr(), head_stride_n=hs[0], head_stride_c=hs[1], emb=emb.data_ptr(),
                         emb_stride_n=es[0], emb_stride_c=es[1], emb_stride_h=es[2], emb_stride_w=es[3],
                         height=h, width=w, stride=stride, channels=int(emb.shape[1]))
    for a, (aw, ah) in enumerate(ANCHORS[stride]):
        d.anchors[2 * a] = aw
        d.anchors[2 * a + 1] = ah
    return d


def heads_descriptor(out: HeadOutputs, host_memory: bool, dim: int) -> _lib.TfHeads:
    devs = {t.device for t in (*out.heads, *out.embs)}
    if len(devs) != 1:
        raise LayoutError(f"all head tensors and embedding maps must be on one device, got {sorted(map(str, devs))}")
    desc = _lib.TfHeads()
    for i, s in enumerate(STRIDES):
        desc.scale[i] = _scale_desc(out.heads[i], out.embs[i], s, dim)
    desc.scale_inv, desc.pad_x, desc.pad_y = letterbox()
    desc.host_memory = int(host_memory)
    desc.dtype = _dtype_code(out.heads[0])
    return desc


class BatchTracker:
    """S independent trackers updated with B frames each per call."""

    def __init__(self, num_streams: int, config: TrackerConfig | None = None, *, frames_per_update: int = 8,
                 capacity: Capacity | None = None, quantize: bool = False, pipeline: bool = False):
        """``pipeline=True`` overlaps the decode of update i+1 with the
        association of update i (the paper's PP stage): the
        association runs on a context-owned CUDA stream; results are valid
        after ``finish()`` (``update(sync=True)`` calls it) or ``join()``."""
        self.config = config or TrackerConfig()
        self.S = int(num_streams)
        cap = capacity or Capacity(streams=self.S, max_frames=self.S * frames_per_update)
        if cap.streams < self.S:
            raise ValueError("capacity.streams < num_streams")
        self.engine = Engine(self.config, cap, quantize=quantize)
        self.frame = np.full(self.S, -1, np.int64)
        self._desc, self._desc_key, self._views = None, None, {}
        self.pipeline = bool(pipeline)
        if self.pipeline:
            self.engine.check(self.engine.lib.tf_set_pipeline(self.engine.ctx, 1), "pipeline")

    def join(self, stream=None) -> None:
        """Make ``stream`` (default: current) wait for all queued association work."""
        self.engine.check(self.engine.lib.tf_join(self.engine.ctx, _lib.stream_handle(stream)), "join")

    def finish(self) -> None:
        """Synchronise and raise the first device-side error of the queued updates."""
        self.engine.finish()

    def _frames(self, stream_begin: int, n_streams: int, B: int, frame_index) -> np.ndarray:
        if frame_index is None:
            if n_streams == 1:                     # (the host cost matters at small batches)
                start = int(self.frame[stream_begin]) + 1
                return np.arange(start, start + B, dtype=np.int64)
            last = self.frame[stream_begin:stream_begin + n_streams]
            return np.add.outer(last + 1, np.arange(B, dtype=np.int64)).reshape(-1)
        return np.ascontiguousarray(frame_index, dtype=np.int64).reshape(-1)

    def update(self, head_outputs: HeadOutputs, frame_index=None, *, stream_begin: int = 0,
               n_streams: int | None = None, trace: bool = False, sync: bool = True,
               host_out: dict | None = None) -> OnlineTracks:
        """Run decode + NMS + association for ``n_streams`` streams x B frames.

        Device tensors by default; pinned host tensors (``tensor.is_pinned()``)
        select the end-to-end path, whose records land in ``host_out`` (dict of
        pinned host tensors from :meth:`host_output`)."""
        eng = self.engine
        n_streams = self.S if n_streams is None else n_streams
        F = head_outputs.frames
        if F % n_streams:
            raise LayoutError(f"{F} frames do not split over {n_streams} streams")
        B = F // n_streams
        host = not head_outputs.heads[0].is_cuda
        if host and not all(t.is_pinned() for t in (*head_outputs.heads, *head_outputs.embs)):
            raise LayoutError("host inputs must be pinned (torch.Tensor.pin_memory())")
        if not host and head_outputs.heads[0].device != eng.device:
            raise LayoutError(f"head tensors are on {head_outputs.heads[0].device}, the tracker on {eng.device}")
        frames = self._frames(stream_begin, n_streams, B, frame_index)
        desc = self._descriptor(head_outputs, host)
        if host:
            if host_out is None:
                host_out = self.host_output(F)
            rec = _lib.TfRecords(host_out["count"].data_ptr(), host_out["track_id"].data_ptr(),
                                 host_out["box"].data_ptr(), host_out["objectness"].data_ptr(),
                                 eng.cap.max_detections, 0)
        else:
            rec = eng.records
        code = eng.lib.tf_update_heads(eng.ctx, C.byref(desc), stream_begin, n_streams, B, frames.ctypes.data,
                                       C.byref(rec), C.byref(eng.trace) if trace else None,
                                       _lib.stream_handle())
        eng.check(code, "update")
        if sync:
            eng.finish()
        self.frame[stream_begin:stream_begin + n_streams] = frames.reshape(n_streams, B)[:, -1]
        if host:
            return OnlineTracks(host_out["count"], host_out["track_id"], host_out["box"], host_out["objectness"],
                                frames, B)
        views = self._views.get(F)
        if views is None:
            views = self._views[F] = (eng.rec_count[:F], eng.rec_id[:F], eng.rec_box[:F], eng.rec_obj[:F])
        return OnlineTracks(*views, frames, B)

    def update_rows(self, rows, frame_index=None, *, stream_begin: int = 0, n_streams: int | None = None,
                    trace: bool = False, sync: bool = True) -> OnlineTracks:
        """Post-decode entry: ``rows[f]`` is frame f's ``[n, 6 + D]`` parse_output
        input (tlwh, objectness, class score, raw embedding; tf/postproc.py:19-42),
        frames stream-major. Replays detector output (the detection-file source,
        tf/detgen.py:366-484) through NMS and association in one launch per
        update instead of one ``Tracker.step`` per frame."""
        torch = self.engine.torch
        eng = self.engine
        n_streams = self.S if n_streams is None else n_streams
        F = len(rows)
        if F == 0 or F % n_streams:
            raise LayoutError(f"{F} frames do not split over {n_streams} streams")
        B = F // n_streams
        D = self.config.embedding_dim
        arrs = []
        for f, r in enumerate(rows):
            r = np.asarray(r, dtype=np.float64)
            if r.size == 0:
                r = np.zeros((0, ROW_WIDTH + D), np.float64)
            if r.ndim != 2 or r.shape[1] != ROW_WIDTH + D:
                raise LayoutError(f"frame {f}: expected rows of width {ROW_WIDTH + D}, got shape {r.shape}")
            arrs.append(r)
        offsets = np.zeros(F + 1, np.int32)
        offsets[1:] = np.cumsum([a.shape[0] for a in arrs])
        allr = np.concatenate(arrs) if offsets[-1] else np.zeros((0, ROW_WIDTH + D), np.float64)
        boxes = np.ascontiguousarray(allr[:, :4])
        # parse_output builds a BoundingBox per row (tf/core.py:37-43)
        bad = ~(np.isfinite(boxes).all(axis=1) & (boxes[:, 2] > 0) & (boxes[:, 3] > 0))
        if bad.any():
            i = int(np.nonzero(bad)[0][0])
            from .core import BoundingBox
            BoundingBox(*(float(v) for v in boxes[i]))      # raises the reference's InvalidBoxError
        emb64 = allr[:, ROW_WIDTH:]
        emb32 = emb64.astype(np.float32)
        normalized = 0
        if not np.array_equal(emb32.astype(np.float64), emb64):
            # raw values beyond fp32: parse_output's fp64 normalisation first (GPU)
            from .core import normalize_rows
            emb32 = normalize_rows(emb64)
            normalized = 1
        dev = eng.device
        db = torch.as_tensor(boxes).to(dev)
        do = torch.as_tensor(np.ascontiguousarray(allr[:, 4])).to(dev)
        de = torch.as_tensor(np.ascontiguousarray(emb32)).to(dev)
        frames = self._frames(stream_begin, n_streams, B, frame_index)
        code = eng.lib.tf_update_detections(eng.ctx, stream_begin, n_streams, B, frames.ctypes.data,
                                            offsets.ctypes.data, db.data_ptr() if allr.shape[0] else None,
                                            do.data_ptr() if allr.shape[0] else None,
                                            de.data_ptr() if allr.shape[0] else None, normalized,
                                            C.byref(eng.records), C.byref(eng.trace) if trace else None,
                                            _lib.stream_handle())
        eng.check(code, "update_rows")
        if sync:
            eng.finish()
        self.frame[stream_begin:stream_begin + n_streams] = frames.reshape(n_streams, B)[:, -1]
        views = self._views.get(F)
        if views is None:
            views = self._views[F] = (eng.rec_count[:F], eng.rec_id[:F], eng.rec_box[:F], eng.rec_obj[:F])
        return OnlineTracks(*views, frames, B)

    def _descriptor(self, out: HeadOutputs, host: bool) -> _lib.TfHeads:
        """heads_descriptor with the layout validated once per tensor layout:
        later updates with the same shapes / strides / dtype only swap the data
        pointers (the per-update host cost matters at small batches)."""
        key = (host,) + tuple((t.shape, t.stride(), t.dtype, t.device) for t in (*out.heads, *out.embs))
        if self._desc_key != key:           # (a changed layout, dtype or device: validate and rebuild)
            self._desc = heads_descriptor(out, host, self.config.embedding_dim)
            self._desc_key = key
            self._desc_scales = [self._desc.scale[i] for i in range(3)]   # views into the struct
            return self._desc
        for sc, h, e in zip(self._desc_scales, out.heads, out.embs):
            sc.head = h.data_ptr()
            sc.emb = e.data_ptr()
        return self._desc

    def host_output(self, frames: int) -> dict:
        torch = self.engine.torch
        R = self.engine.cap.max_detections
        return dict(count=torch.zeros(frames, dtype=torch.int32).pin_memory(),
                    track_id=torch.zeros(frames, R, dtype=torch.int64).pin_memory(),
                    box=torch.zeros(frames, R, 4, dtype=torch.float64).pin_memory(),
                    objectness=torch.zeros(frames, R, dtype=torch.float64).pin_memory())

    def trace(self, frames: int) -> dict:
        """Per-frame parity trace of the last traced update (device tensors)."""
        e = self.engine
        return dict(cand_count=e.tr_cand[:frames], det_count=e.tr_det[:frames], det_code=e.tr_code[:frames],
                    det_track=e.tr_track[:frames], det_cost=e.tr_cost[:frames], det_matched=e.tr_matched[:frames])

    def export(self, stream: int) -> dict:
        return self.engine.export(stream)

    def import_tracks(self, stream: int, state: dict) -> None:
        """Inverse of ``export``: resume ``stream`` from a track table
        (tf_import_tracks). Waits for the stream's pending updates."""
        self.engine.import_(stream, state)
        lf = int(state["last_frame"])
        self.frame[stream] = -1 if lf == _lib.NO_FRAME else lf
