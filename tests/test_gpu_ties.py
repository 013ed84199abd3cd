"""Exact ties through the whole device association (GPU): scipy's order decides.

Every track and detection embedding is drawn from 24 exactly representable
unit vectors in 4-d (the axis vectors +-e_i and the 16 vectors (+-1/2)^4), and
smoothing_alpha = 0 keeps the tracks' embeddings in that set, so every cosine
cost is exactly one of {0, 0.5, 1, 1.5, 2}: equal costs and equal sums of
distinct costs (a + d == b + c, two optima with four different costs) occur
in most frames. Boxes are packed so that gates overlap. Whatever the device's
decomposition (peeling, components, per-component solves), the finite pairs
must be the ones scipy's solve of the padded matrix returns (via the oracle,
which calls scipy.optimize.linear_sum_assignment like tf/assoc.py:76).
"""

import itertools

import numpy as np
import pytest

pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import tracker as ot   # noqa: E402

VECS = np.array([s * np.eye(4)[i] for i in range(4) for s in (1.0, -1.0)]
                + [np.array(sgn) * 0.5 for sgn in itertools.product((1.0, -1.0), repeat=4)])


def _scene(rng, n_obj, frames, width=100.0, height=20.0, jitter=3.0):
    cx = rng.uniform(400, 400 + width, n_obj)
    cy = rng.uniform(300, 300 + height, n_obj)
    emb = rng.integers(0, len(VECS), n_obj)
    out = []
    for _ in range(frames):
        cx = cx + rng.normal(0, jitter, n_obj)
        cy = cy + rng.normal(0, 1.0, n_obj)
        flip = rng.random(n_obj) < 0.3
        emb = np.where(flip, rng.integers(0, len(VECS), n_obj), emb)
        keep = rng.random(n_obj) > 0.1
        rows = []
        for i in np.nonzero(keep)[0]:
            w, h = 12.0, 30.0
            rows.append(np.concatenate([[cx[i] - w / 2, cy[i] - h / 2, w, h, 0.9, 1.0], VECS[emb[i]]]))
        out.append(np.array(rows).reshape(-1, 10))
    return out


@pytest.mark.parametrize("seed,n_obj,width,height", [(0, 40, 100.0, 20.0), (1, 40, 100.0, 20.0),
                                                     (2, 60, 200.0, 30.0), (3, 60, 200.0, 30.0)])
def test_exact_ties_follow_scipy_order(seed, n_obj, width, height):
    import paper_2011_03910_b200 as p

    rng = np.random.default_rng(seed)
    cfg = p.TrackerConfig(embedding_dim=4, smoothing_alpha=0.0, max_cost=1.6)
    trk = p.Tracker(cfg, capacity=p.Capacity(streams=1, max_frames=1, max_tracks=512))
    ora = ot.OracleTracker(ot.Settings(embedding_dim=4, smoothing_alpha=0.0, max_cost=1.6))
    matched = 0
    for f, rows in enumerate(_scene(rng, n_obj, 60, width, height)):
        got = trk.step(f, p.parse_output(rows, 4))
        want = ora.step(f, ot.rows_to_dets(rows, 4))
        assert [r[0] for r in got.records] == [r[0] for r in want.records], f"frame {f}"
        for (_, gb, _), (_, wb, _) in zip(got.records, want.records):
            np.testing.assert_allclose(gb.as_tlwh(), wb, rtol=1e-9, atol=1e-9)
        matched += len(want.matches)
    assert matched > 1000
