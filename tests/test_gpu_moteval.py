"""GPU MOT evaluation against the reference's moteval on the same files
(tests/golden/files/moteval_expected.json from tests/golden/make_golden_files.py):
per-frame correspondences (one-launch accumulate), identity metrics and the
full report are exact."""

import json
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2011_03910_b200 import detfile, moteval   # noqa: E402

GOLD = Path(__file__).resolve().parent / "golden" / "files"
EXP = json.loads((GOLD / "moteval_expected.json").read_text())


def _frames():
    return moteval.load_mot_tracks(GOLD / "gt.txt"), moteval.load_mot_tracks(GOLD / "res.txt")


@pytest.mark.parametrize("thr", [0.5, 0.3])
def test_accumulate_matches_reference(thr):
    gt, hyp = _frames()
    got = moteval.accumulate(gt, hyp, thr)
    exp = EXP[f"accumulate_{thr}"]
    assert len(got) == len(exp)
    for c, (f, matches, ug, uh) in zip(got, exp):
        assert c.frame_index == f
        assert [(g, h) for g, h, _ in c.matches] == [(m[0], m[1]) for m in matches]
        assert [o for _, _, o in c.matches] == [m[2] for m in matches]       # bit-exact IoU
        assert list(c.unmatched_gt) == ug and list(c.unmatched_hyp) == uh


def test_match_frame_agrees_with_accumulate():
    gt, hyp = _frames()
    prev = {}
    seq = moteval.accumulate(gt, hyp, 0.5)
    for c in seq[:10]:
        one = moteval.match_frame(gt.get(c.frame_index, []), hyp.get(c.frame_index, []), prev, 0.5, c.frame_index)
        assert one == c
        for g, h, _ in one.matches:
            prev[g] = h


def test_report_and_id_metrics_match_reference():
    gt, hyp = _frames()
    rep = moteval.evaluate(gt, hyp)
    assert dict(zip(moteval.MetricsReport.COLUMNS, rep.row())) == EXP["report"]
    assert list(moteval.id_metrics(gt, hyp, 0.5)) == EXP["id_metrics_0.5"]


def test_gpu_tracker_outputs_score_like_reference(tmp_path):
    """Detection file -> GPU replay -> MOT result file -> GPU evaluation == the
    reference's report on its own result file (rows rounded to 6 decimals alike)."""
    import paper_2011_03910_b200 as p
    dets = detfile.load_mot_detections(GOLD / "det.txt")
    outs = detfile.replay(detfile.load_embedding_sidecar(GOLD / "det.emb", dets, 16), p.TrackerConfig(embedding_dim=16),
                          n_frames=40)
    moteval.write_mot_results(tmp_path / "res.txt", outs)
    assert (tmp_path / "res.txt").read_bytes() == (GOLD / "res.txt").read_bytes()
    gt, _ = _frames()
    rep = moteval.evaluate(gt, moteval.load_mot_tracks(tmp_path / "res.txt"))
    assert dict(zip(moteval.MetricsReport.COLUMNS, rep.row())) == EXP["report"]
