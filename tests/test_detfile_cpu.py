"""Detection-file source on the CPU: the MOT detection parser and the sidecar
checks follow tf/detgen.py:366-484 and the reference's own tests
(tests/test_detgen.py:196-305); the parse of the golden file must equal the
reference's parse bit for bit (tests/golden/make_golden_files.py)."""

from pathlib import Path

import numpy as np
import pytest

from paper_2011_03910_b200 import detfile
from paper_2011_03910_b200.errors import ConsistencyError, DimensionError, InvalidBoxError, ParseError

GOLD = Path(__file__).resolve().parent / "golden" / "files"
DIM = 16


def test_golden_parse_bit_exact():
    exp = np.load(GOLD / "detfile_expected.npz")
    dets = detfile.load_mot_detections(GOLD / "det.txt")
    assert list(dets) == exp["parsed_frames"].tolist()          # insertion order of first appearance
    assert [dets[f].shape[0] for f in dets] == exp["parsed_counts"].tolist()
    np.testing.assert_array_equal(np.concatenate([dets[f] for f in dets]), exp["parsed_rows"])


def test_example_row(tmp_path):
    path = tmp_path / "det.txt"
    path.write_text("1,-1,10,20,30,40,0.9\n")
    frames = detfile.load_mot_detections(path)
    assert list(frames) == [0]
    np.testing.assert_allclose(frames[0], [[10, 20, 30, 40, 0.9, 1.0]])


def test_empty_file(tmp_path):
    path = tmp_path / "det.txt"
    path.write_text("")
    assert detfile.load_mot_detections(path) == {}


@pytest.mark.parametrize("text,exc,match", [
    ("1,-1,10,20,30,40,0.9\n1,-1,10,20,30\n", ParseError, "line 2"),
    ("1,-1,10,20,-5,40,0.9\n", InvalidBoxError, "line 1"),
    ("1,-1,ten,20,30,40,0.9\n", ParseError, "line 1"),
    ("0,-1,10,20,30,40,0.9\n", ParseError, "frame index must be >= 1"),
])
def test_bad_rows(tmp_path, text, exc, match):
    path = tmp_path / "det.txt"
    path.write_text(text)
    with pytest.raises(exc, match=match):
        detfile.load_mot_detections(path)


def test_confidence_clamped_and_extra_fields(tmp_path):
    path = tmp_path / "det.txt"
    path.write_text("1,-1,10,20,30,40,1.7,-1,-1,-1\n2,-1,10,20,30,40,-0.5\n")
    frames = detfile.load_mot_detections(path)
    assert frames[0][0, 4] == 1.0
    assert frames[1][0, 4] == 0.0


def _detections():
    return {0: np.array([[10.0, 20.0, 30.0, 40.0, 0.9, 1.0]]),
            2: np.array([[1.0, 2.0, 3.0, 4.0, 0.8, 1.0], [5.0, 6.0, 7.0, 8.0, 0.7, 1.0]])}


def _records(rng):
    return {k: rng.standard_normal(DIM).astype(np.float32) for k in [(0, 0), (2, 0), (2, 1)]}


def test_sidecar_golden_bytes_round_trip(tmp_path):
    """Our writer reproduces the reference-written sidecar byte for byte."""
    blob = (GOLD / "det.emb").read_bytes()
    n = (len(blob) - 8) // (8 + 4 * DIM)
    rec = np.frombuffer(blob[8:], dtype=np.dtype([("f", "<u4"), ("d", "<u4"), ("v", "<f4", (DIM,))]), count=n)
    records = {(int(f), int(d)): v for f, d, v in zip(rec["f"], rec["d"], rec["v"])}
    detfile.write_embedding_sidecar(tmp_path / "x.emb", records, DIM)
    assert (tmp_path / "x.emb").read_bytes() == blob


def test_sidecar_dimension_mismatch(tmp_path):
    path = tmp_path / "det.emb"
    detfile.write_embedding_sidecar(path, {(0, 0): np.ones(8, dtype=np.float32)}, 8)
    with pytest.raises(DimensionError):
        detfile.load_embedding_sidecar(path, _detections(), DIM)


def test_sidecar_missing_and_extra(tmp_path):
    rng = np.random.default_rng(1)
    records = _records(rng)
    del records[(2, 0)]
    detfile.write_embedding_sidecar(tmp_path / "a.emb", records, DIM)
    with pytest.raises(ConsistencyError, match=r"\(2, 0\)"):
        detfile.load_embedding_sidecar(tmp_path / "a.emb", _detections(), DIM)
    records = _records(rng)
    records[(9, 0)] = rng.standard_normal(DIM).astype(np.float32)
    detfile.write_embedding_sidecar(tmp_path / "b.emb", records, DIM)
    with pytest.raises(ConsistencyError, match=r"\(9, 0\)"):
        detfile.load_embedding_sidecar(tmp_path / "b.emb", _detections(), DIM)


def test_sidecar_duplicate_and_bad_magic(tmp_path):
    blob = b"EMB1" + np.uint32(DIM).tobytes()
    rec = np.uint32(0).tobytes() * 2 + np.ones(DIM, np.float32).tobytes()
    (tmp_path / "d.emb").write_bytes(blob + rec + rec)
    with pytest.raises(ConsistencyError, match="duplicate"):
        detfile.load_embedding_sidecar(tmp_path / "d.emb", {0: np.zeros((1, 6))}, DIM)
    (tmp_path / "m.emb").write_bytes(b"NOPE" + b"\x00" * 16)
    with pytest.raises(ParseError):
        detfile.load_embedding_sidecar(tmp_path / "m.emb", _detections(), DIM)
    (tmp_path / "t.emb").write_bytes(blob + rec[:-4])
    with pytest.raises(ParseError, match="not a multiple"):
        detfile.load_embedding_sidecar(tmp_path / "t.emb", {0: np.zeros((1, 6))}, DIM)


def test_file_frames_gaps():
    frames = dict(detfile.file_frames({1: np.ones((2, 6)), 3: np.ones((1, 6))}, n_frames=5))
    assert sorted(frames) == [0, 1, 2, 3, 4]
    assert frames[0].shape == (0, 6)
    assert frames[1].shape == (2, 6)
