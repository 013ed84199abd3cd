"""Decode oracle: JDE/YOLO head tensors -> the reference's raw rows.

TEST INFRASTRUCTURE ONLY.

The reference has no head decode (its synthetic source
emits already-decoded rows, ``tf/detgen.py:220-267``). This module pins the
decode the product implements, following BASELINE.json config 0 with the
SURVEY.md section 7 H1 decisions, and emits exactly the ``[n, 6 + D]`` rows
``parse_output`` consumes (``tf/postproc.py:19-42``; class score 1.0 as in
``tf/detgen.py:265``). Decode parity is pinned by this restatement only.

Layout (per frame, per scale s):

* head tensor ``[24, H_s, W_s]`` fp32, channel ``6a + k`` for anchor ``a``:
  k = 0..3 box deltas (tx, ty, tw, th), k = 4 background logit, k = 5
  foreground logit;
* embedding map ``[D, H_s, W_s]`` fp32 (any strides; channels_last on device).

Decisions:

* confidence = softmax over (bg, fg) = sigmoid(fg - bg); the keep test is done
  exactly in logit space, ``fg - bg >= logit(conf_threshold)`` with the
  difference taken in fp64 (exact for fp32 inputs), so CPU and GPU select
  identical candidates; the emitted objectness is ``1 / (1 + exp(-(fg - bg)))``;
* candidate order: scale (stride 32, 16, 8), then anchor, then y, then x;
* box: centre ``(cell + sigmoid(t)) * stride``, size ``anchor * exp(t)`` in the
  1088x608 letterboxed input, mapped back to 1920x1080 with
  ``(v - pad) * (1080 / 608)``; tlwh = centre - size / 2.
"""

from __future__ import annotations

import math

import numpy as np

INPUT_W, INPUT_H = 1088, 608
IMAGE_W, IMAGE_H = 1920, 1080
STRIDES = (32, 16, 8)                       # candidate order
GRID = {32: (19, 34), 16: (38, 68), 8: (76, 136)}   # (H, W)
ANCHORS = {
    8: ((8.0, 24.0), (11.0, 34.0), (16.0, 48.0), (23.0, 68.0)),
    16: ((32.0, 96.0), (45.0, 135.0), (64.0, 192.0), (90.0, 271.0)),
    32: ((128.0, 384.0), (180.0, 540.0), (256.0, 640.0), (512.0, 640.0)),
}
NUM_ANCHORS = 4
HEAD_CHANNELS = 6 * NUM_ANCHORS


def letterbox() -> tuple[float, float, float]:
    """(scale_inv, pad_x, pad_y) for 1920x1080 -> 1088x608 (JDE letterbox)."""
    ratio = min(INPUT_W / IMAGE_W, INPUT_H / IMAGE_H)
    new_w, new_h = round(IMAGE_W * ratio), round(IMAGE_H * ratio)
    pad_x, pad_y = (INPUT_W - new_w) / 2.0, (INPUT_H - new_h) / 2.0
    return IMAGE_H / INPUT_H, pad_x, pad_y


def scale_offsets() -> dict[int, int]:
    """First global anchor index of each scale in candidate order."""
    out, acc = {}, 0
    for s in STRIDES:
        h, w = GRID[s]
        out[s] = acc
        acc += NUM_ANCHORS * h * w
    return out


TOTAL_ANCHORS = sum(NUM_ANCHORS * h * w for h, w in GRID.values())   # 54,264


def logit_threshold(conf_threshold: float) -> float:
    """logit(p) in fp64; exactly 0.0 at p = 0.5, +-inf at the ends."""
    if conf_threshold <= 0.0:
        return -math.inf
    if conf_threshold >= 1.0:
        return math.inf
    return math.log(conf_threshold) - math.log1p(-conf_threshold)


def _sigmoid(t: float) -> float:
    return 1.0 / (1.0 + math.exp(-t))


def decode_frame(heads, embs, conf_threshold: float = 0.5):
    """Decode one frame.

    ``heads[i]`` is the ``[24, H, W]`` fp32 array and ``embs[i]`` the
    ``[D, H, W]`` fp32 array of scale ``STRIDES[i]``. Returns
    ``(codes int64 [C], rows float64 [C, 6 + D])`` with ``codes`` the global
    anchor index of each candidate (candidate order).
    """
    lim = logit_threshold(conf_threshold)
    inv_r, pad_x, pad_y = letterbox()
    offs = scale_offsets()
    dim = int(embs[0].shape[0])
    codes, rows = [], []
    for si, s in enumerate(STRIDES):
        head = np.asarray(heads[si], dtype=np.float32)
        emb = embs[si]
        h, w = GRID[s]
        assert head.shape == (HEAD_CHANNELS, h, w), head.shape
        bg = head[4::6].astype(np.float64)
        fg = head[5::6].astype(np.float64)
        logit = fg - bg
        a_idx, y_idx, x_idx = np.nonzero(logit >= lim)
        for a, y, x in zip(a_idx.tolist(), y_idx.tolist(), x_idx.tolist()):
            tx, ty, tw, th = (float(head[6 * a + k, y, x]) for k in range(4))
            aw, ah = ANCHORS[s][a]
            cx = (x + _sigmoid(tx)) * s
            cy = (y + _sigmoid(ty)) * s
            bw = aw * math.exp(tw)
            bh = ah * math.exp(th)
            cx = (cx - pad_x) * inv_r
            cy = (cy - pad_y) * inv_r
            bw = bw * inv_r
            bh = bh * inv_r
            row = np.empty(ROW_WIDTH_PREFIX + dim, dtype=np.float64)
            row[0] = cx - bw / 2.0
            row[1] = cy - bh / 2.0
            row[2] = bw
            row[3] = bh
            row[4] = _sigmoid(float(logit[a, y, x]))
            row[5] = 1.0
            row[6:] = np.asarray(emb[:, y, x], dtype=np.float32).astype(np.float64)
            codes.append(offs[s] + (a * h + y) * w + x)
            rows.append(row)
    if not rows:
        return np.zeros(0, dtype=np.int64), np.zeros((0, ROW_WIDTH_PREFIX + dim), dtype=np.float64)
    return np.asarray(codes, dtype=np.int64), np.stack(rows)


ROW_WIDTH_PREFIX = 6
