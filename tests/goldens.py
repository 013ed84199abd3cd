"""Loaders for the committed golden vectors (tests/golden/*.npz)."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"
SEQUENCES = ["lanes16", "noisy16", "random64", "mixed64", "euclid16", "lifecycle16", "random512"]


def load_sequence(name: str) -> dict:
    z = np.load(GOLDEN / f"tracker_{name}.npz")
    data = {k: z[k] for k in z.files}
    data["config"] = json.loads(str(data["config"]))
    counts = data["counts"]
    offs = np.concatenate([[0], np.cumsum(counts)])
    data["frames"] = [
        np.concatenate([data["rows6"][offs[i]:offs[i + 1]],
                        data["emb"][offs[i]:offs[i + 1]].astype(np.float64)], axis=1)
        for i in range(len(counts))
    ]
    return data


def records_by_frame(data: dict) -> dict:
    out: dict[int, list] = {f: [] for f in range(len(data["counts"]))}
    for f, tid, box, obj in zip(data["rec_frame"], data["rec_id"], data["rec_box"], data["rec_obj"]):
        out[int(f)].append((int(tid), tuple(float(v) for v in box), float(obj)))
    return out


def load_units() -> dict:
    z = np.load(GOLDEN / "units.npz")
    return {k: z[k] for k in z.files}


def known_answers() -> dict:
    return json.loads((GOLDEN / "known_answers.json").read_text())
