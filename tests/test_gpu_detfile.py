"""Detection-file source on the GPU against the reference's own outputs
(tests/golden/files, written by tests/golden/make_golden_files.py): sidecar
normalisation, and the whole replay (tf_update_detections: NMS + association
per batch of frames) against the reference's parse_output + Tracker.step
records over the same files. Bit-exact ids; boxes / objectness 1e-4 relative."""

from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2011_03910_b200 import detfile                     # noqa: E402
from paper_2011_03910_b200.errors import DegenerateEmbeddingError   # noqa: E402

GOLD = Path(__file__).resolve().parent / "golden" / "files"
DIM = 16


def _loaded():
    dets = detfile.load_mot_detections(GOLD / "det.txt")
    return detfile.load_embedding_sidecar(GOLD / "det.emb", dets, DIM)


def test_sidecar_attach_matches_reference():
    exp = np.load(GOLD / "detfile_expected.npz")
    attached = _loaded()
    rows = np.concatenate([r for _, r in detfile.file_frames(attached, int(exp["frames"].size), 6 + DIM)])
    np.testing.assert_array_equal(rows[:, :6], exp["rows"][:, :6])
    np.testing.assert_allclose(rows[:, 6:], exp["rows"][:, 6:], rtol=0, atol=1e-7)


@pytest.mark.parametrize("batch", [1, 7, 40])
def test_replay_matches_reference_tracker(batch):
    import paper_2011_03910_b200 as p
    exp = np.load(GOLD / "detfile_expected.npz")
    outs = detfile.replay(_loaded(), p.TrackerConfig(embedding_dim=DIM), n_frames=int(exp["frames"].size),
                          batch=batch)
    assert [o.frame_index for o in outs] == exp["frames"].tolist()
    got = [(o.frame_index, tid, box.as_tlwh(), obj) for o in outs for tid, box, obj in o.records]
    assert [g[0] for g in got] == exp["rec_frame"].tolist()
    assert [g[1] for g in got] == exp["rec_id"].tolist()
    np.testing.assert_allclose(np.array([g[2] for g in got]), exp["rec_box"], rtol=1e-4, atol=1e-6)
    np.testing.assert_allclose(np.array([g[3] for g in got]), exp["rec_obj"], rtol=1e-12)


def test_update_rows_matches_tracker_step():
    """The batched rows entry and the per-frame Tracker.step agree (fp64 rows
    whose embeddings are not fp32 take the GPU fp64 normalisation first)."""
    import paper_2011_03910_b200 as p
    rng = np.random.default_rng(5)
    cfg = p.TrackerConfig(embedding_dim=DIM)
    frames = []
    base = rng.uniform(100, 1500, (6, 2))
    for f in range(12):
        n = 6
        rows = np.zeros((n, 6 + DIM))
        rows[:, 0:2] = base + f * 3.0 + rng.normal(0, 0.5, (n, 2))
        rows[:, 2:4] = [40.0, 90.0]
        rows[:, 4] = 0.9
        rows[:, 5] = 1.0
        rows[:, 6:] = np.eye(n, DIM) + rng.normal(0, 0.01, (n, DIM))   # fp64 values
        frames.append(rows)
    bt = p.BatchTracker(1, cfg, frames_per_update=4)
    got = []
    for s in range(0, 12, 4):
        res = bt.update_rows(frames[s:s + 4], np.arange(s, s + 4))
        got += [res.records(0, b) for b in range(4)]
    trk = p.Tracker(cfg)
    for f in range(12):
        want = trk.step(f, p.parse_output(frames[f], DIM)).records
        assert [r[0] for r in got[f]] == [r[0] for r in want]
        for (_, gb, go), (_, wb, wo) in zip(got[f], want):
            np.testing.assert_allclose(gb.as_tlwh(), wb.as_tlwh(), rtol=1e-9)


def test_zero_vector_rejected(tmp_path):
    rng = np.random.default_rng(3)
    records = {k: rng.standard_normal(DIM).astype(np.float32) for k in [(0, 0), (2, 0), (2, 1)]}
    records[(0, 0)] = np.zeros(DIM, dtype=np.float32)
    detfile.write_embedding_sidecar(tmp_path / "z.emb", records, DIM)
    dets = {0: np.array([[10.0, 20.0, 30.0, 40.0, 0.9, 1.0]]),
            2: np.array([[1.0, 2.0, 3.0, 4.0, 0.8, 1.0], [5.0, 6.0, 7.0, 8.0, 0.7, 1.0]])}
    with pytest.raises(DegenerateEmbeddingError):
        detfile.load_embedding_sidecar(tmp_path / "z.emb", dets, DIM)


def test_degenerate_raw_row_raises_like_parse_output():
    import paper_2011_03910_b200 as p
    rows = np.zeros((2, 6 + DIM))
    rows[:, 2:4] = 10.0
    rows[:, 4] = 0.9
    rows[0, 6] = 1.0                      # row 1 has a zero embedding
    bt = p.BatchTracker(1, p.TrackerConfig(embedding_dim=DIM), frames_per_update=1)
    with pytest.raises(DegenerateEmbeddingError):
        bt.update_rows([rows], np.array([0]))
