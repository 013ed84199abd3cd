"""The oracle's JDE extensions (lambda-fused cost, IoU second stage) on hand
cases. They are not in the reference: with their defaults the oracle is the
reference path (pinned by test_oracle_golden.py); these tests pin the
extension semantics the GPU parity tests then hold the kernels to."""

import numpy as np

from oracle import tracker as ot


def _unit(v):
    v = np.asarray(v, np.float64)
    return (v / np.linalg.norm(v)).astype(np.float32)


E1 = _unit([1.0, 0.0, 0.0, 0.0])
E2 = _unit([0.0, 1.0, 0.0, 0.0])        # orthogonal: cosine cost 1.0


def _det(box, emb):
    return ot.Det(box, 0.9, 1.0, emb)


def _tracker(**kw):
    return ot.OracleTracker(ot.Settings(embedding_dim=4, **kw))


def test_defaults_are_the_reference_path():
    s = ot.Settings()
    assert s.motion_lambda == 1.0 and not s.iou_stage


def test_iou_stage_rematches_an_overlapping_detection():
    for iou_stage, expect_match in ((False, False), (True, True)):
        trk = _tracker(iou_stage=iou_stage)
        trk.step(0, [_det((100.0, 100.0, 50.0, 100.0), E1)])
        out = trk.step(1, [_det((102.0, 101.0, 50.0, 100.0), E2)])
        if expect_match:
            assert [m[0] for m in out.matches] == [1] and out.births == []
            assert 0.0 <= out.matches[0][2] <= 0.5            # the IoU distance
            assert trk.stage2_matches == 1
        else:
            assert out.matches == [] and out.births == [2]


def test_iou_stage_respects_threshold_and_lost_tracks():
    trk = _tracker(iou_stage=True, iou_threshold=0.5)
    trk.step(0, [_det((100.0, 100.0, 50.0, 100.0), E1)])
    out = trk.step(1, [_det((140.0, 100.0, 50.0, 100.0), E2)])   # IoU 1/9: distance 8/9 > 0.5
    assert out.matches == [] and out.births == [2]
    # track 1 is LOST now: a LOST track is not offered to the IoU stage
    out = trk.step(2, [_det((100.0, 100.0, 50.0, 100.0), E2)])
    assert all(m[0] != 1 for m in out.matches)


def test_lambda_fused_cost_values():
    lam = 0.98
    trk = _tracker(motion_lambda=lam)
    trk.step(0, [_det((100.0, 100.0, 50.0, 100.0), E1)])
    ref = _tracker()
    ref.step(0, [_det((100.0, 100.0, 50.0, 100.0), E1)])
    d = [_det((101.0, 100.0, 50.0, 100.0), _unit([1.0, 0.1, 0.0, 0.0]))]
    fused = trk.step(1, d).gated
    plain = ref.step(1, d).gated
    t = ref.tracks[0]
    meas = np.stack([ot.to_measurement(x.box) for x in d])
    # gate distance of the predicted track (the reference's own gate)
    pm, pc = ref.motion.predict(*ref.motion.initiate(ot.to_measurement((100.0, 100.0, 50.0, 100.0))))
    g = ref.motion.gate(pm, pc, meas)
    assert np.isfinite(plain[0, 0]) and t.track_id == 1
    assert fused[0, 0] == lam * plain[0, 0] + (1.0 - lam) * g[0]
