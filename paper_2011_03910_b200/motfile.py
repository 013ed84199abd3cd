"""Column-wise reader of MOT text files (detections, ground truth, results).

One parser serves the detection-file source (``detfile.load_mot_detections``,
tf/detgen.py:366-397) and the tracking-result / ground-truth reader
(``moteval.load_mot_tracks``, tf/moteval.py:288-316). The file is split once,
the needed columns are converted as whole columns, and every per-line rule is
evaluated as a vector; the error reported is the one of the first offending
line, with that line's rules taken in the reference's order (field count,
numeric fields, frame index, box size, repeated id), so the exception class
and the ``line N`` in its message are the reference's.
"""

from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .errors import DuplicateIdError, InvalidBoxError, ParseError


@dataclass
class Table:
    """Parsed numeric columns of the non-blank lines, in file order."""

    line: np.ndarray        # 1-based line numbers
    frame: np.ndarray       # 0-based frame index (int64)
    ident: np.ndarray | None  # object / track id (int64), when requested
    box: np.ndarray         # [n, 4] tlwh float64
    conf: np.ndarray | None  # confidence column, when requested


def _column(values: list[str]):
    """float() of every entry (Python's parser: the reference's semantics);
    on failure, the index of the first bad entry and the error text."""
    try:
        return np.fromiter(map(float, values), dtype=np.float64, count=len(values)), None
    except ValueError:
        for i, v in enumerate(values):
            try:
                float(v)
            except ValueError as exc:
                return None, (i, str(exc))
    raise AssertionError("unreachable")


def read_table(path: str | Path, min_fields: int, with_id: bool, with_conf: bool) -> Table:
    """Parse the lines of a MOT file (``frame,id,x,y,w,h,conf,...``). With
    ``with_id`` (tracks) a repeated (frame, id) and a non-finite box are
    errors too, as BoundingBox construction makes them in the reference."""
    lines = Path(path).read_text(encoding="utf-8").split("\n")
    numbered = [(i + 1, ln.strip()) for i, ln in enumerate(lines)]
    numbered = [(n, ln) for n, ln in numbered if ln]
    line_no = np.fromiter((n for n, _ in numbered), dtype=np.int64, count=len(numbered))
    fields = [ln.split(",") for _, ln in numbered]
    n = len(fields)
    width = np.fromiter(map(len, fields), dtype=np.int64, count=n)
    # rule 1: field count (nothing after the first short line is ever read)
    short = np.nonzero(width < min_fields)[0]
    limit = int(short[0]) if short.size else n
    # rule 2: numeric fields, column by column
    cols = [0, 2, 3, 4, 5] + ([1] if with_id else []) + ([6] if with_conf else [])
    conv, bad_at, bad_msg = {}, limit, None
    for c in cols:
        vals, err = _column([f[c] for f in fields[:limit]])
        if err is not None and err[0] < bad_at:
            bad_at, bad_msg = err
        conv[c] = vals
    n_ok = bad_at                       # lines [0, n_ok) pass rules 1-2
    take = {c: (v[:n_ok] if v is not None else _column([f[c] for f in fields[:n_ok]])[0]) for c, v in conv.items()}
    frame = np.trunc(take[0]).astype(np.int64) if n_ok else np.zeros(0, np.int64)   # int(float(v))
    box = np.stack([take[c] for c in (2, 3, 4, 5)], axis=1) if n_ok else np.zeros((0, 4))
    ident = np.trunc(take[1]).astype(np.int64) if with_id and n_ok else np.zeros(0, np.int64)
    # rules 3-6 on those lines: the first failing line wins, its rules in order
    rules = [("frame", frame < 1), ("box", (box[:, 2] <= 0) | (box[:, 3] <= 0))]
    if with_id:
        seen = np.ones(n_ok, bool)
        if n_ok:
            seen[np.unique(np.stack([frame, ident], axis=1), axis=0, return_index=True)[1]] = False
        rules += [("dup", seen), ("finite", ~np.isfinite(box).all(axis=1))]
    first = None
    for kind, bad in rules:
        idx = np.nonzero(bad)[0]
        if idx.size and (first is None or int(idx[0]) < first[1]):
            first = (kind, int(idx[0]))
    if first is not None:
        kind, i = first
        ln = int(line_no[i])
        if kind == "frame":
            raise ParseError(f"line {ln}: frame index must be >= 1, got {int(frame[i])}")
        if kind == "box":
            raise InvalidBoxError(f"line {ln}: non-positive box size w={box[i, 2]}, h={box[i, 3]}")
        if kind == "dup":
            raise DuplicateIdError(f"line {ln}: id {int(ident[i])} repeats in frame {int(frame[i])}")
        raise InvalidBoxError(f"line {ln}: box is not finite: {tuple(box[i])}")
    if n_ok < n:
        ln = int(line_no[n_ok])
        if bad_msg is not None:
            raise ParseError(f"line {ln}: non-numeric field ({bad_msg})")
        raise ParseError(f"line {ln}: expected at least {min_fields} fields, got {int(width[n_ok])}")
    return Table(line_no, frame - 1, ident if with_id else None, box, take[6] if with_conf else None)


def group_by_frame(frame: np.ndarray):
    """(frame, row indices) per distinct frame, frames in order of first
    appearance, rows in file order."""
    if frame.size == 0:
        return []
    order = np.argsort(frame, kind="stable")
    uniq, start = np.unique(frame[order], return_index=True)
    bounds = list(start) + [frame.size]
    groups = [(int(u), order[bounds[k]:bounds[k + 1]]) for k, u in enumerate(uniq)]
    groups.sort(key=lambda g: int(g[1][0]))
    return groups
