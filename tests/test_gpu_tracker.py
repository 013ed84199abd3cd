"""GPU Tracker.step against the reference's own golden runs and semantics tests.

The golden sequences were produced by the reference Tracker on the reference's
own scenario generator (tests/golden/make_golden.py); the semantic tests
restate /root/reference/pkg/tests/test_tracker.py and test_acceptance.py
criterion 10 against the device tracker.
"""

import numpy as np
import pytest

pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from goldens import SEQUENCES, load_sequence, records_by_frame   # noqa: E402

DIM = 16


@pytest.fixture(scope="module")
def p():
    import paper_2011_03910_b200 as pkg
    return pkg


def unit(p, axis, dim=DIM):
    v = np.zeros(dim)
    v[axis] = 1.0
    return p.normalize(v)


def det(p, x, y, embedding, w=20.0, h=30.0, objectness=0.9):
    return p.Detection(box=p.BoundingBox(x, y, w, h), objectness=objectness, embedding=embedding)


def config(p, **kw):
    d = dict(embedding_dim=DIM)
    d.update(kw)
    return p.TrackerConfig(**d)


@pytest.mark.parametrize("name", SEQUENCES)
def test_golden_sequence(p, name):
    data = load_sequence(name)
    cfg = dict(data["config"])
    quant = cfg.pop("quantize", False)
    trk = p.Tracker(p.TrackerConfig(**cfg), capacity=p.Capacity(streams=1, max_frames=1, max_tracks=512),
                    quantize=False)
    want = records_by_frame(data)
    worst = 0.0
    for f, raw in enumerate(data["frames"]):
        dets = p.parse_output(raw, cfg["embedding_dim"])
        if quant:
            from paper_2011_03910_b200.core import normalize_rows
            if dets:
                # _quantize_detection (tf/pipeline.py:436-441): binary16 round trip, then normalize
                q = normalize_rows(p.quantize_binary16(np.stack([d.embedding for d in dets])))
                dets = [p.Detection(d.box, d.objectness, d.class_score, e) for d, e in zip(dets, q)]
        out = trk.step(f, dets)
        assert [r[0] for r in out.records] == [r[0] for r in want[f]], f"frame {f}"
        for (_, gb, go), (_, wb, wo) in zip(out.records, want[f]):
            g, w = np.array(gb.as_tlwh()), np.array(wb)
            worst = max(worst, float(np.max(np.abs(g - w) / np.maximum(np.abs(w), 1.0))))
            assert go == wo
    assert worst <= 1e-4
    tracks = trk.tracks
    assert [t.track_id for t in tracks] == data["trk_id"].tolist()
    assert [t.hits for t in tracks] == data["trk_hits"].tolist()
    assert [int(t.state is p.TrackState.LOST) for t in tracks] == data["trk_state"].tolist()
    assert [-1 if t.lost_since is None else t.lost_since for t in tracks] == data["trk_lost"].tolist()
    for t, m, c, e in zip(tracks, data["trk_mean"], data["trk_cov"], data["trk_emb"]):
        np.testing.assert_allclose(t.kalman.mean, m, rtol=1e-4, atol=1e-6)
        np.testing.assert_allclose(t.kalman.covariance, c, rtol=1e-4, atol=1e-9)
        np.testing.assert_allclose(t.smooth_embedding, e, rtol=1e-4, atol=1e-6)
    assert sorted(trk.removed_ids) == data["removed"].tolist()


def test_empty_step(p):
    t = p.Tracker(config(p))
    out = t.step(0, [])
    assert out.frame_index == 0 and out.records == () and t.tracks == []


def test_birth_then_rematch_keeps_id(p):
    t = p.Tracker(config(p))
    assert [r[0] for r in t.step(0, [det(p, 100, 100, unit(p, 0))]).records] == [1]
    assert [r[0] for r in t.step(1, [det(p, 103, 101, unit(p, 0))]).records] == [1]
    assert t.tracks[0].hits == 2


def test_new_track_box_equals_measurement(p):
    t = p.Tracker(config(p))
    _, box, conf = t.step(0, [det(p, 100, 100, unit(p, 0))]).records[0]
    assert box.x == pytest.approx(100.0, abs=1e-9) and box.w == pytest.approx(20.0, abs=1e-9)
    assert conf == 0.9


def test_unmatched_detections_spawn_fresh_ids(p):
    t = p.Tracker(config(p))
    t.step(0, [det(p, 0, 0, unit(p, 0)), det(p, 200, 0, unit(p, 1))])
    out = t.step(1, [det(p, 0, 0, unit(p, 0)), det(p, 200, 0, unit(p, 1)), det(p, 400, 0, unit(p, 2))])
    assert [r[0] for r in out.records] == [1, 2, 3]


def test_ordering_and_missing_embedding(p):
    t = p.Tracker(config(p))
    t.step(5, [])
    with pytest.raises(p.OrderingError):
        t.step(5, [])
    with pytest.raises(p.OrderingError):
        t.step(3, [])
    t2 = p.Tracker(config(p))
    with pytest.raises(p.DimensionError):
        t2.step(0, [det(p, 0, 0, None)])


def test_low_confidence_filtered(p):
    t = p.Tracker(config(p, conf_threshold=0.5))
    assert t.step(0, [det(p, 0, 0, unit(p, 0), objectness=0.4)]).records == ()
    assert t.tracks == []


def test_lifecycle(p):
    t = p.Tracker(config(p, max_lost=3))
    t.step(0, [det(p, 100, 100, unit(p, 0))])
    for f in range(1, 4):
        t.step(f, [])
        assert t.tracks and t.tracks[0].state is p.TrackState.LOST
        assert t.tracks[0].lost_since == 1
    t.step(4, [])
    assert t.tracks == [] and t.removed_ids == {1}
    assert [r[0] for r in t.step(5, [det(p, 100, 100, unit(p, 0))]).records] == [2]


def test_lost_track_rematches(p):
    t = p.Tracker(config(p, max_lost=5))
    t.step(0, [det(p, 100, 100, unit(p, 0))])
    t.step(1, [])
    t.step(2, [])
    assert [r[0] for r in t.step(3, [det(p, 100, 100, unit(p, 0))]).records] == [1]
    assert t.tracks[0].state is p.TrackState.ACTIVE and t.tracks[0].lost_since is None


def test_min_hits_delays_reporting(p):
    t = p.Tracker(config(p, min_hits=3))
    assert t.step(0, [det(p, 0, 0, unit(p, 0))]).records == ()
    assert t.step(1, [det(p, 1, 0, unit(p, 0))]).records == ()
    assert [r[0] for r in t.step(2, [det(p, 2, 0, unit(p, 0))]).records] == [1]


def test_euclidean_gate(p):
    t = p.Tracker(config(p, gate_metric="euclidean", gate_threshold=100.0))
    t.step(0, [det(p, 100, 100, unit(p, 0))])
    out = t.step(1, [det(p, 500, 500, unit(p, 0))])
    assert [r[0] for r in out.records] == [2]
    assert t.tracks[0].state is p.TrackState.LOST


def test_unknown_gate_metric_is_config_error(p):
    t = p.Tracker(config(p, gate_metric="cosine"))
    t.step(0, [det(p, 100, 100, unit(p, 0))])
    with pytest.raises(p.ConfigError):
        t.step(1, [det(p, 100, 100, unit(p, 0))])


def test_lifecycle_conformance_criterion_10(p):
    """tests/test_acceptance.py:289-347 restated on the device tracker."""
    rng = np.random.default_rng(30)
    max_lost = 4
    t = p.Tracker(p.TrackerConfig(embedding_dim=DIM, max_lost=max_lost, max_cost=0.5))
    known = set()
    for frame in range(80):
        dets = [p.Detection(p.BoundingBox(float(rng.uniform(0, 2000)), float(rng.uniform(0, 2000)), 20.0, 30.0),
                            objectness=0.9, embedding=p.normalize(rng.standard_normal(DIM)))
                for _ in range(int(rng.integers(0, 5)))]
        usable = len(p.nms(dets, t.config.nms_iou)) if dets else 0
        out = t.step(frame, dets)
        ids = {r[0] for r in out.records}
        assert len(out.records) == usable
        assert all(i > max(known, default=0) for i in ids - known)
        known |= ids
        for tr in t.tracks:
            if tr.state is p.TrackState.ACTIVE:
                assert tr.last_update_frame == frame and tr.lost_since is None
            else:
                assert tr.lost_since == tr.last_update_frame + 1 and frame - tr.lost_since < max_lost
        assert not ids & t.removed_ids
