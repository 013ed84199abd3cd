"""MOT result rows and the MOT file reader on the CPU against the reference's
files (tests/golden/files: gt.txt / res.txt written by tf/cli.py:56-70)."""

from pathlib import Path

import numpy as np
import pytest

from paper_2011_03910_b200 import moteval
from paper_2011_03910_b200.core import BoundingBox
from paper_2011_03910_b200.errors import DuplicateIdError, InvalidBoxError, ParseError
from paper_2011_03910_b200.tracker import TrackerOutput

GOLD = Path(__file__).resolve().parent / "golden" / "files"


def test_result_rows_byte_identical(tmp_path):
    exp = np.load(GOLD / "detfile_expected.npz")
    outs, frames = [], exp["rec_frame"]
    for f in np.unique(frames):
        sel = frames == f
        recs = tuple((int(i), BoundingBox(*b), float(o))
                     for i, b, o in zip(exp["rec_id"][sel], exp["rec_box"][sel], exp["rec_obj"][sel]))
        outs.append(TrackerOutput(frame_index=int(f), records=recs))
    moteval.write_mot_results(tmp_path / "res.txt", outs)
    assert (tmp_path / "res.txt").read_bytes() == (GOLD / "res.txt").read_bytes()


def test_load_mot_tracks_golden():
    gt = moteval.load_mot_tracks(GOLD / "gt.txt")
    lines = (GOLD / "gt.txt").read_text().splitlines()
    assert sum(len(v) for v in gt.values()) == len(lines)
    first = lines[0].split(",")
    tid, box = gt[int(first[0]) - 1][0]
    assert tid == int(first[1]) and box.as_tlwh() == tuple(float(v) for v in first[2:6])


@pytest.mark.parametrize("text,exc", [
    ("1,1,10,20,30\n", ParseError),
    ("1,1,10,20,-30,40,1\n", InvalidBoxError),
    ("0,1,10,20,30,40,1\n", ParseError),
    ("1,1,10,20,30,40,1\n1,1,11,20,30,40,1\n", DuplicateIdError),
])
def test_load_mot_tracks_errors(tmp_path, text, exc):
    (tmp_path / "t.txt").write_text(text)
    with pytest.raises(exc):
        moteval.load_mot_tracks(tmp_path / "t.txt")


def test_clear_mot_micro_scenario():
    """Hand case: gt 1 switches 10 -> 20, gt 2 is missed once then switches 20 -> 30."""
    C = moteval.FrameCorrespondence
    corr = [C(0, ((1, 10, 1.0), (2, 20, 1.0)), (), ()), C(1, ((1, 20, 1.0),), (2,), ()),
            C(2, ((1, 20, 0.9), (2, 30, 1.0)), (), (40,))]
    s = moteval.clear_mot(corr)
    assert (s.id_switches, s.fn, s.fp, s.true_positives, s.total_gt) == (2, 1, 1, 5, 6)
    assert s.mota == pytest.approx(1.0 - 4 / 6)
    assert s.fragmentations == 1
