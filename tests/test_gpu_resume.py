"""Resuming from a track table (tf_import_tracks, the inverse of tf_export_tracks).

Parity bisection: the reference Tracker's state at frame
k - ``tracks``, ``_next_id``, ``_last_frame`` (tf/tracker.py:74-83), captured
by tests/golden/make_golden_resume.py - is loaded into the GPU tracker, which
must then reproduce the reference's records of frames k.. exactly (ids,
objectness; boxes to the golden sequences' 1e-4). Export -> import between
two GPU trackers must be bit-exact, and invalid tables are refused with the
reference's error classes.
"""

import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from goldens import GOLDEN   # noqa: E402

RESUME = ["noisy16", "lifecycle16", "random64"]


@pytest.fixture(scope="module")
def p():
    import paper_2011_03910_b200 as pkg
    return pkg


def _tracks(p, z):
    out = []
    for i in range(len(z["mid_id"])):
        lost = int(z["mid_lost"][i])
        out.append(p.Track(track_id=int(z["mid_id"][i]),
                           state=p.TrackState.LOST if z["mid_state"][i] else p.TrackState.ACTIVE,
                           kalman=p.KalmanState(mean=z["mid_mean"][i].copy(), covariance=z["mid_cov"][i].copy()),
                           smooth_embedding=z["mid_emb"][i].copy(), last_update_frame=int(z["mid_last"][i]),
                           lost_since=None if lost < 0 else lost, hits=int(z["mid_hits"][i])))
    return out


@pytest.mark.parametrize("name", RESUME)
def test_resume_from_reference_state(p, name):
    from goldens import load_sequence
    z = dict(np.load(GOLDEN / f"resume_{name}.npz"))
    cfg = json.loads(str(z["config"]))
    cfg.pop("quantize", None)
    seq = load_sequence(name)
    k = int(z["k"])
    trk = p.Tracker(p.TrackerConfig(**cfg), capacity=p.Capacity(streams=1, max_frames=1, max_tracks=512))
    trk.load_state(_tracks(p, z), next_id=int(z["mid_next_id"]), last_frame=int(z["mid_last_frame"]))
    # the imported table reads back bit-exactly
    back = trk.tracks
    assert [t.track_id for t in back] == z["mid_id"].tolist()
    for t, m, c, e in zip(back, z["mid_mean"], z["mid_cov"], z["mid_emb"]):
        assert np.array_equal(t.kalman.mean, m) and np.array_equal(t.kalman.covariance, c)
        assert np.array_equal(t.smooth_embedding, e)
    with pytest.raises(p.OrderingError):
        trk.step(int(z["mid_last_frame"]), [])
    want: dict[int, list] = {}
    for f, tid, box, obj in zip(z["rec_frame"], z["rec_id"], z["rec_box"], z["rec_obj"]):
        want.setdefault(int(f), []).append((int(tid), box, float(obj)))
    worst = 0.0
    for f in range(k, len(seq["frames"])):
        out = trk.step(f, p.parse_output(seq["frames"][f], cfg["embedding_dim"]))
        assert [r[0] for r in out.records] == [r[0] for r in want.get(f, [])], f"frame {f}"
        for (_, gb, go), (_, wb, wo) in zip(out.records, want.get(f, [])):
            g = np.array(gb.as_tlwh())
            worst = max(worst, float(np.max(np.abs(g - wb) / np.maximum(np.abs(wb), 1.0))))
            assert go == wo
    assert worst <= 1e-4
    # and the end state is the uninterrupted reference run's
    assert [t.track_id for t in trk.tracks] == seq["trk_id"].tolist()
    assert sorted(trk.removed_ids) == seq["removed"].tolist()


def test_from_reference_tracker_object(p):
    """Tracker.from_reference reads a reference-shaped Tracker (config,
    tracks, _next_id, _last_frame)."""
    z = dict(np.load(GOLDEN / "resume_noisy16.npz"))

    class RefLike:
        config = p.TrackerConfig(embedding_dim=16)
        tracks = _tracks(p, z)
        _next_id = int(z["mid_next_id"])
        _last_frame = int(z["mid_last_frame"])

    trk = p.Tracker.from_reference(RefLike())
    assert [t.track_id for t in trk.tracks] == z["mid_id"].tolist()
    assert sorted(trk.removed_ids) == sorted(set(range(1, RefLike._next_id)) - set(z["mid_id"].tolist()))


def test_export_import_between_batch_trackers_bit_exact(p):
    """Stream state exported after update 1 and imported into a fresh
    BatchTracker continues bit-identically; per-stream updates with default
    frame indices (stream_begin > 0) follow each stream's own frame count."""
    from paper_2011_03910_b200 import synth
    S, B = 4, 8
    gen = synth.make("cfg3", device="cuda", seed=11, streams=S)
    batches = [gen.next_batch(B) for _ in range(3)]

    def snap(r):
        return [t.cpu().numpy().copy() for t in (r.count, r.track_id, r.box, r.objectness)]

    ref = p.BatchTracker(S, frames_per_update=B)
    want = [snap(ref.update(bb)) for bb in batches]

    first = p.BatchTracker(S, frames_per_update=B)
    got0 = snap(first.update(batches[0]))
    tables = [first.export(s) for s in range(S)]
    second = p.BatchTracker(S, frames_per_update=B)
    for s in range(S):
        second.import_tracks(s, tables[s])
    for s in range(S):
        a, b = second.export(s), tables[s]
        for key in ("track_id", "state", "hits", "lost_since", "last_update_frame", "mean", "covariance",
                    "embedding"):
            assert np.array_equal(a[key], b[key]), key
        assert (a["count"], a["next_id"], a["last_frame"]) == (b["count"], b["next_id"], b["last_frame"])
    got = [got0]
    for bb in batches[1:]:
        # streams 2..3 first, then 0..1: default frame indices are per stream
        halves = []
        for sb in (2, 0):
            sub = p.HeadOutputs(tuple(h[sb * B:(sb + 2) * B] for h in bb.heads),
                                tuple(e[sb * B:(sb + 2) * B] for e in bb.embs))
            halves.append((sb, snap(second.update(sub, stream_begin=sb, n_streams=2))))
        halves.sort()
        got.append([np.concatenate([halves[0][1][i], halves[1][1][i]]) for i in range(4)])
    for u, (g, w) in enumerate(zip(got, want)):
        assert np.array_equal(g[0], w[0]), f"update {u} counts"
        for f in range(S * B):
            n = int(w[0][f])
            for i in (1, 2, 3):
                assert np.array_equal(g[i][f, :n], w[i][f, :n]), f"update {u} frame {f}"


def test_import_rejects_invalid_tables(p):
    z = dict(np.load(GOLDEN / "resume_noisy16.npz"))
    mk = lambda: p.Tracker(p.TrackerConfig(embedding_dim=16),   # noqa: E731
                           capacity=p.Capacity(streams=1, max_frames=1, max_tracks=64))
    tr = _tracks(p, z)
    nid, lf = int(z["mid_next_id"]), int(z["mid_last_frame"])
    with pytest.raises(ValueError, match="duplicate"):
        mk().load_state(tr + [tr[0]], next_id=nid, last_frame=lf)
    with pytest.raises(ValueError, match="outside"):
        mk().load_state(tr, next_id=int(z["mid_id"].max()), last_frame=lf)
    bad = _tracks(p, z)
    bad[0].kalman.covariance[0, 1] = 1e-3
    bad[0].kalman.covariance[1, 0] = 1e-3
    with pytest.raises(ValueError, match="couples two axes"):
        mk().load_state(bad, next_id=nid, last_frame=lf)
    bad = _tracks(p, z)
    lost = [t for t in bad if t.state is p.TrackState.LOST][0]
    lost.lost_since = None
    with pytest.raises(ValueError, match="lost_since"):
        mk().load_state(bad, next_id=nid, last_frame=lf)
    small = p.Tracker(p.TrackerConfig(embedding_dim=16), capacity=p.Capacity(streams=1, max_frames=1, max_tracks=4))
    with pytest.raises(p.CapacityError):
        small.load_state(tr, next_id=nid, last_frame=lf)
    # a fresh state (no frame stepped yet) is accepted and steps from frame 0
    t = mk()
    t.load_state([], next_id=1, last_frame=None)
    assert t.step(0, []).records == ()
