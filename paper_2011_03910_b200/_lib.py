"""ctypes binding of libtrackforge_b200.so (the C ABI in include/trackforge_b200.h).

There is no CPU fallback: importing a compute entry point without the built
library, or calling it without a CUDA device, raises immediately.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

from . import errors as E

LIB_PATH = Path(__file__).resolve().parent / "libtrackforge_b200.so"

c_i32, c_i64, c_dbl, c_vp = C.c_int32, C.c_int64, C.c_double, C.c_void_p


class TfConfig(C.Structure):
    _fields_ = [
        ("conf_threshold", c_dbl), ("nms_iou", c_dbl), ("max_cost", c_dbl), ("gate_threshold", c_dbl),
        ("smoothing_alpha", c_dbl), ("std_weight_position", c_dbl), ("std_weight_velocity", c_dbl),
        ("std_aspect", c_dbl), ("std_aspect_velocity", c_dbl), ("std_aspect_measurement", c_dbl),
        ("gate_metric", c_i32), ("max_lost", c_i32), ("min_hits", c_i32), ("embedding_dim", c_i32),
        ("quantize_binary16", c_i32), ("iou_stage", c_i32),
        ("motion_lambda", c_dbl), ("motion_weight", c_dbl), ("iou_threshold", c_dbl),
    ]


class TfCapacity(C.Structure):
    _fields_ = [("streams", c_i32), ("max_frames", c_i32), ("max_candidates", c_i32),
                ("max_detections", c_i32), ("max_tracks", c_i32), ("reserved", c_i32)]


class TfHeadScale(C.Structure):
    _fields_ = [
        ("head", c_vp), ("head_stride_n", c_i64), ("head_stride_c", c_i64),
        ("emb", c_vp), ("emb_stride_n", c_i64), ("emb_stride_c", c_i64), ("emb_stride_h", c_i64),
        ("emb_stride_w", c_i64), ("height", c_i32), ("width", c_i32), ("stride", c_i32),
        ("channels", c_i32), ("anchors", C.c_float * 8),
    ]


class TfHeads(C.Structure):
    _fields_ = [("scale", TfHeadScale * 3), ("scale_inv", c_dbl), ("pad_x", c_dbl), ("pad_y", c_dbl),
                ("host_memory", c_i32), ("dtype", c_i32)]


class TfRecords(C.Structure):
    _fields_ = [("count", c_vp), ("track_id", c_vp), ("box", c_vp), ("objectness", c_vp),
                ("max_records", c_i32), ("reserved", c_i32)]


class TfTrace(C.Structure):
    _fields_ = [("cand_count", c_vp), ("det_count", c_vp), ("det_code", c_vp), ("det_track", c_vp),
                ("det_cost", c_vp), ("det_matched", c_vp)]


NO_FRAME = -(2 ** 63)  # tf_track_export.last_frame before the first step (_last_frame None)


class TfTrackExport(C.Structure):
    _fields_ = [("count", c_i32), ("reserved", c_i32), ("next_id", c_i64), ("last_frame", c_i64),
                ("track_id", c_vp), ("state", c_vp), ("hits", c_vp), ("lost_since", c_vp),
                ("last_update_frame", c_vp), ("mean", c_vp), ("covariance", c_vp), ("embedding", c_vp)]


# name -> (restype, argtypes)
_SIGS = {
    "tf_version": (c_i32, []),
    "tf_status_name": (C.c_char_p, [c_i32]),
    "tf_create": (c_i32, [C.POINTER(TfConfig), C.POINTER(TfCapacity), c_i32, C.POINTER(c_vp)]),
    "tf_destroy": (c_i32, [c_vp]),
    "tf_last_error": (C.c_char_p, [c_vp]),
    "tf_reset_stream": (c_i32, [c_vp, c_i32, c_vp]),
    "tf_update_heads": (c_i32, [c_vp, C.POINTER(TfHeads), c_i32, c_i32, c_i32, c_vp,
                                C.POINTER(TfRecords), C.POINTER(TfTrace), c_vp]),
    "tf_step_detections": (c_i32, [c_vp, c_i32, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp,
                                   C.POINTER(TfRecords), C.POINTER(TfTrace), c_vp]),
    "tf_finish": (c_i32, [c_vp, c_vp]),
    "tf_export_tracks": (c_i32, [c_vp, c_i32, C.POINTER(TfTrackExport), c_vp]),
    "tf_import_tracks": (c_i32, [c_vp, c_i32, C.POINTER(TfTrackExport), c_vp]),
    "tf_set_pipeline": (c_i32, [c_vp, c_i32]),
    "tf_join": (c_i32, [c_vp, c_vp]),
    "tf_set_profiling": (c_i32, [c_vp, c_i32]),
    "tf_kernel_times": (c_i32, [c_vp, C.POINTER(c_dbl), C.POINTER(c_dbl), C.POINTER(c_i64)]),
    "tf_copy_times": (c_i32, [c_vp, C.POINTER(c_dbl)]),
    "tf_launch_count": (c_i32, [c_vp, C.POINTER(c_i64)]),
    "tf_launch_info": (c_i32, [c_vp, C.POINTER(c_i32), C.POINTER(c_i32)]),
    "tf_timeline": (c_i32, [c_vp, c_vp, c_i32, C.POINTER(c_i32)]),
    "tf_mot_accumulate": (c_i32, [c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_i32, c_dbl,
                                  c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "tf_mot_coverage": (c_i32, [c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_dbl, c_vp, c_vp]),
    "tf_update_detections": (c_i32, [c_vp, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32,
                                     C.POINTER(TfRecords), C.POINTER(TfTrace), c_vp]),
    "tf_phase_stats": (c_i32, [c_vp, c_vp]),
    "tf_stream_clocks": (c_i32, [c_vp, c_vp, c_i32]),
    "tf_stream_hold": (c_i32, [c_vp, c_vp]),
    "tf_nms_sets": (c_i32, [c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "tf_lap_dense": (c_i32, [c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "tf_kalman": (c_i32, [c_i32, c_i32, C.POINTER(TfConfig), c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "tf_gating": (c_i32, [c_i32, c_vp, c_vp, c_i32, c_vp, c_i32, C.POINTER(TfConfig), c_vp, c_vp, c_vp]),
    "tf_cosine_cost": (c_i32, [c_i32, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "tf_normalize_rows": (c_i32, [c_i32, c_i32, c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_vp]),
    "tf_quantize_binary16": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_vp]),
    "tf_smooth_embedding": (c_i32, [c_i32, c_i32, c_vp, c_vp, c_dbl, c_vp, c_vp, c_vp]),
    "tf_iou_pairs": (c_i32, [c_i32, c_vp, c_vp, c_vp, c_vp]),
}

EXPORTED = tuple(_SIGS)

_lock = threading.Lock()
_lib: C.CDLL | None = None


def load() -> C.CDLL:
    """Load (once) and type the shared library. Raises if it was not built."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise ImportError(
                    f"{LIB_PATH.name} is not built; run `python -m paper_2011_03910_b200._build` "
                    "(there is no CPU fallback for the tracking path)")
            lib = C.CDLL(str(LIB_PATH))
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def status_error(code: int, message: str) -> Exception:
    cls = E.STATUS_TO_ERROR.get(int(code), E.TrackforgeError)
    return cls(message)


def check(code: int, ctx=None, what: str = "") -> None:
    if code == 0:
        return
    lib = load()
    name = lib.tf_status_name(code).decode()
    detail = lib.tf_last_error(ctx).decode() if ctx else ""
    raise status_error(code, f"{what}: {name}: {detail}" if what else f"{name}: {detail}")


def require_cuda():
    """The product path runs on the GPU only."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("trackforge_b200 needs a CUDA device (sm_100a); no CPU fallback exists")
    return torch


def stream_handle(torch_stream=None) -> int:
    """cudaStream_t of `torch_stream`, default torch's current stream on the
    current device (read through the raw accessor: this runs per update and
    its host cost shows at small batches)."""
    import torch

    if torch_stream is not None:
        return int(torch_stream.cuda_stream)
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return int(raw(torch._C._cuda_getDevice()))
    return int(torch.cuda.current_stream().cuda_stream)


def ptr(t) -> int | None:
    return None if t is None else int(t.data_ptr())
