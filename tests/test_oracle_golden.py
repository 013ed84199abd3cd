"""Pin the CPU oracle against vectors the reference produced (CPU only).

The oracle is only trusted as a parity checker because these tests show it
reproduces the reference's own outputs on the reference's own inputs
(``tests/golden/make_golden.py``) and its hand-derived known answers.
"""

import math

import numpy as np
import pytest

from goldens import SEQUENCES, known_answers, load_sequence, load_units, records_by_frame
from oracle import lap as olap
from oracle import tracker as ot


def _settings(cfg: dict) -> ot.Settings:
    kw = dict(cfg)
    quant = kw.pop("quantize", False)
    return ot.Settings(quantize=quant, **kw)


@pytest.mark.parametrize("name", SEQUENCES)
def test_oracle_tracker_matches_reference_golden(name):
    data = load_sequence(name)
    s = _settings(data["config"])
    trk = ot.OracleTracker(s)
    want = records_by_frame(data)
    for f, raw in enumerate(data["frames"]):
        trace = trk.step(f, ot.rows_to_dets(raw, s.embedding_dim, s.quantize))
        got = trace.records
        assert [r[0] for r in got] == [r[0] for r in want[f]], f"ids differ at frame {f}"
        for (gid, gbox, gobj), (_, wbox, wobj) in zip(got, want[f]):
            np.testing.assert_allclose(gbox, wbox, rtol=1e-12, atol=1e-9)
            assert gobj == wobj
    assert [t.track_id for t in trk.tracks] == data["trk_id"].tolist()
    assert [int(t.state == ot.LOST) for t in trk.tracks] == data["trk_state"].tolist()
    assert [t.hits for t in trk.tracks] == data["trk_hits"].tolist()
    assert [-1 if t.lost_since is None else t.lost_since for t in trk.tracks] == data["trk_lost"].tolist()
    for t, m, c, e in zip(trk.tracks, data["trk_mean"], data["trk_cov"], data["trk_emb"]):
        np.testing.assert_allclose(t.mean, m, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(t.cov, c, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(t.emb, e, rtol=1e-6, atol=1e-7)
    assert sorted(trk.removed_ids) == data["removed"].tolist()


def test_oracle_nms_matches_reference():
    u = load_units()
    off = u["nms_off"]
    for i, thr in enumerate(u["nms_thr"]):
        a, b = off[i], off[i + 1]
        boxes = [tuple(r) for r in u["nms_boxes"][a:b]]
        kept = ot.greedy_nms(boxes, list(u["nms_scores"][a:b]), float(thr))
        assert kept == np.nonzero(u["nms_keep"][a:b])[0].tolist()


def test_oracle_lap_matches_reference_and_scipy_ties():
    u = load_units()
    vals, off, pos = u["lap_vals"], u["lap_off"], 0
    for i, (nr, nc) in enumerate(u["lap_shapes"]):
        cost = vals[pos:pos + nr * nc].reshape(nr, nc)
        pos += nr * nc
        matches, _, _ = ot.solve_assignment(cost)
        want = [tuple(p) for p in u["lap_pairs"][off[i]:off[i + 1]]]
        assert [(r, c) for r, c, _ in matches] == want
        # restated shortest-augmenting-path solver picks the same optimum
        n = max(nr, nc)
        finite = cost[np.isfinite(cost)]
        amp = float(np.max(np.abs(finite))) if finite.size else 1.0
        sent = 2.0 * n * max(amp, 1.0) + 1.0
        pad = np.full((n, n), sent)
        pad[:nr, :nc] = np.where(np.isfinite(cost), cost, sent)
        col4row, _ = olap.solve_square(pad)
        mine = [(r, int(col4row[r])) for r in range(nr)
                if col4row[r] < nc and math.isfinite(cost[r, col4row[r]])]
        assert mine == want
        if nr <= 6 and nc <= 6:
            card, total = olap.brute_force(cost)
            assert len(want) == card
            assert sum(cost[r, c] for r, c in want) == pytest.approx(total, abs=1e-9)


def test_oracle_kalman_matches_reference():
    u = load_units()
    m = ot.Motion(ot.Settings())
    state = None
    gi = 0
    for op, z, mean, cov in zip(u["kf_ops"], u["kf_z"], u["kf_mean"], u["kf_cov"]):
        if op == 0:
            state = m.initiate(z)
        elif op == 1:
            state = m.predict(*state)
            g = m.gate(state[0], state[1], u["kf_gate_z"][gi][None, :])[0]
            assert g == u["kf_gate"][gi]
            gi += 1
        else:
            state = m.update(state[0], state[1], z)
        np.testing.assert_array_equal(state[0], mean)
        np.testing.assert_array_equal(state[1], cov)


def test_oracle_normalize_and_binary16():
    u = load_units()
    for a, b in zip(u["norm_in"], u["norm_out"]):
        np.testing.assert_array_equal(ot.unit_vector(a), b)
    np.testing.assert_array_equal(ot.to_half(u["fp16_in"]), u["fp16_out"])


def test_oracle_known_answers():
    ka = known_answers()
    assert ot.box_iou((0, 0, 2, 2), (1, 1, 2, 2)) == ka["iou_1_7"] == pytest.approx(1 / 7)
    assert ot.to_measurement((10, 20, 4, 8)).tolist() == ka["measurement"]
    assert float(ot.to_half(np.array([0.1]))[0]) == ka["fp16_0_1"] == 0.0999755859375
    cov = np.zeros((8, 8))
    cov[:4, :4] = np.diag([3.0, 3.0, 4.0 - 1e-2, 3.0])
    g = ot.Motion(ot.Settings()).gate(np.array([0.0, 0.0, 1.0, 20.0, 0, 0, 0, 0]), cov,
                                      np.array([[2.0, 0.0, 1.0, 20.0]]))
    assert g[0] == pytest.approx(ka["gate_scalar"], abs=1e-12)
    matches, _, _ = ot.solve_assignment(np.array([[1.0, 2.0], [2.0, 4.0]]))
    assert [[r, c] for r, c, _ in matches] == ka["lap_2x2"]


def test_oracle_errors_name_reference_classes():
    trk = ot.OracleTracker(ot.Settings(embedding_dim=8))
    trk.step(5, [])
    with pytest.raises(ot.OracleError) as e:
        trk.step(5, [])
    assert e.value.kind == "OrderingError"
    with pytest.raises(ot.OracleError) as e:
        ot.rows_to_dets(np.zeros((1, 13)), 8)
    assert e.value.kind == "LayoutError"
    with pytest.raises(ot.OracleError) as e:
        ot.unit_vector(np.zeros(8))
    assert e.value.kind == "DegenerateEmbeddingError"
    with pytest.raises(ot.OracleError) as e:
        ot.greedy_nms([], [], 1.0)
    assert e.value.kind == "ConfigError"
