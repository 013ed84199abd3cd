"""Pin of the head decode against the generator's encoded truth (test helper).

The reference has no head decode, so GPU == oracle
alone proves only self-consistency. This helper supplies the independent
statement: with zero box-delta noise, synth.py encodes each visible object's
true box as t = logit(frac), ln(size / anchor) at its anchor cell, so a
correct decode must give back the truth box. Objects whose centre fraction
hit the generator's [1e-3, 1 - 1e-3] clamp at any stride are excluded (their
encoded centre is moved on purpose).
"""

from __future__ import annotations

import numpy as np

INPUT_W, INPUT_H, IMAGE_W, IMAGE_H = 1088, 608, 1920, 1080
STRIDES = (32, 16, 8)


def _clamped(truth_tlwh: np.ndarray) -> np.ndarray:
    r = INPUT_H / IMAGE_H
    pad_x = (INPUT_W - round(IMAGE_W * r)) / 2.0
    pad_y = (INPUT_H - round(IMAGE_H * r)) / 2.0
    cx = (truth_tlwh[:, 0] + truth_tlwh[:, 2] / 2.0) * r + pad_x
    cy = (truth_tlwh[:, 1] + truth_tlwh[:, 3] / 2.0) * r + pad_y
    bad = np.zeros(len(truth_tlwh), bool)
    for s in STRIDES:
        for c in (cx, cy):
            frac = c / s - np.floor(c / s)
            bad |= (frac < 1e-3) | (frac > 1 - 1e-3)
    return bad


def match_truth(decoded_tlwh: np.ndarray, truth_tlwh: np.ndarray, rtol: float = 1e-6) -> int:
    """Every decoded box of an encoded object equals the truth box whose
    centre is nearest (collisions keep the later object, whose centre is then
    the nearest at ~0 distance). Returns the number of boxes checked."""
    decoded_tlwh = np.asarray(decoded_tlwh, np.float64).reshape(-1, 4)
    truth_tlwh = np.asarray(truth_tlwh, np.float64).reshape(-1, 4)
    excluded = _clamped(truth_tlwh)
    tc = truth_tlwh[:, :2] + truth_tlwh[:, 2:] / 2.0
    checked = 0
    for box in decoded_tlwh:
        c = box[:2] + box[2:] / 2.0
        j = int(np.argmin(np.sum((tc - c) ** 2, axis=1)))
        if excluded[j]:
            continue
        want = truth_tlwh[j]
        scale = np.maximum(np.abs(want), want[3])
        err = np.abs(box - want) / scale
        assert np.all(err <= rtol), (box, want, err)
        checked += 1
    return checked
