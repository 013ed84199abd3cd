"""Generate golden vectors by running the reference itself.

Run in the build container only (it imports the read-only reference from
``/root/reference/pkg/src``; that tree does not exist on the GPU box):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py

Outputs (committed, small):

* ``tracker_*.npz`` - per-frame detection rows (from the reference's own
  scenario generator ``tf/detgen.py:161-258``) and the reference
  ``Tracker.step`` outputs (``tf/tracker.py:85-159``): records, final track
  table, removed ids.
* ``units.npz`` - NMS sets (``tests/test_acceptance.py:214-237`` recipe), LAP
  matrices (``tests/test_acceptance.py:160-178`` recipe), Kalman sequences
  (``tests/test_acceptance.py:181-211`` recipe), embeddings, fp16 values, with
  the reference's answers.
* ``known_answers.json`` - the hand-derived constants of the reference suite.
"""

from __future__ import annotations

import json
import os
import sys
from dataclasses import replace
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from trackforge.assoc import hungarian_solve                      # noqa: E402
from trackforge.core import (BoundingBox, Detection, iou, box_to_measurement,  # noqa: E402
                             normalize, quantize_binary16)
from trackforge.detgen import NoiseParams, generate_frame, make_scenario   # noqa: E402
from trackforge.motion import KalmanFilter, KalmanState             # noqa: E402
from trackforge.pipeline import _quantize_detection                 # noqa: E402
from trackforge.postproc import nms, parse_output                   # noqa: E402
from trackforge.tracker import Tracker, TrackerConfig, TrackState   # noqa: E402

OUT = Path(__file__).resolve().parent

# (name, scenario kwargs, noise, tracker overrides, frames, quantize)
SEQUENCES = [
    ("lanes16", dict(num_objects=10, seed=4, embedding_dim=16), NoiseParams(), {}, 60, False),
    ("noisy16", dict(num_objects=8, seed=2, embedding_dim=16),
     NoiseParams(p_miss=0.1, sigma_box=0.8, sigma_emb=0.03, lambda_fp=0.5), {}, 40, False),
    ("random64", dict(num_objects=25, seed=7, embedding_dim=64, layout="random"),
     NoiseParams(p_miss=0.05, sigma_box=1.0, sigma_emb=0.02, lambda_fp=1.5), {}, 80, False),
    ("mixed64", dict(num_objects=15, seed=29, embedding_dim=64, separation_margin=0.5),
     NoiseParams(sigma_box=0.8, sigma_emb=0.03), {}, 60, True),
    ("euclid16", dict(num_objects=12, seed=11, embedding_dim=16, layout="random"),
     NoiseParams(p_miss=0.1, sigma_box=1.5, sigma_emb=0.05, lambda_fp=1.0),
     dict(gate_metric="euclidean", gate_threshold=400.0), 50, False),
    ("lifecycle16", dict(num_objects=10, seed=5, embedding_dim=16, layout="random"),
     NoiseParams(p_miss=0.4, sigma_box=1.0, sigma_emb=0.05, lambda_fp=2.0),
     dict(max_lost=4, min_hits=3, max_cost=0.5), 70, False),
    ("random512", dict(num_objects=20, seed=13, embedding_dim=512, layout="random"),
     NoiseParams(p_miss=0.05, sigma_box=1.0, sigma_emb=0.1 / np.sqrt(512), lambda_fp=1.7),
     {}, 25, False),
]


def run_sequence(name, scen_kwargs, noise, overrides, frames, quantize):
    scen = make_scenario(frames=frames, noise=noise, **scen_kwargs)
    dim = scen.embedding_dim
    cfg = TrackerConfig(embedding_dim=dim, **overrides)
    tracker = Tracker(cfg)
    boxes, embs, counts = [], [], []
    rec_frame, rec_id, rec_box, rec_obj = [], [], [], []
    for f in range(frames):
        raw, _ = generate_frame(scen, f, seed=scen_kwargs["seed"] + 100)
        counts.append(raw.shape[0])
        boxes.append(raw[:, :6])
        embs.append(raw[:, 6:].astype(np.float32))
        assert np.array_equal(embs[-1].astype(np.float64), raw[:, 6:])
        dets = parse_output(raw, dim)
        if quantize:
            dets = [_quantize_detection(d) for d in dets]
        out = tracker.step(f, dets)
        for tid, box, obj in out.records:
            rec_frame.append(f)
            rec_id.append(tid)
            rec_box.append(box.as_tlwh())
            rec_obj.append(obj)
    tr = tracker.tracks
    np.savez_compressed(
        OUT / f"tracker_{name}.npz",
        config=json.dumps(dict(overrides, embedding_dim=dim, quantize=quantize)),
        counts=np.asarray(counts, np.int64),
        rows6=np.concatenate(boxes) if boxes else np.zeros((0, 6)),
        emb=np.concatenate(embs) if embs else np.zeros((0, dim), np.float32),
        rec_frame=np.asarray(rec_frame, np.int64),
        rec_id=np.asarray(rec_id, np.int64),
        rec_box=np.asarray(rec_box, np.float64).reshape(-1, 4),
        rec_obj=np.asarray(rec_obj, np.float64),
        trk_id=np.asarray([t.track_id for t in tr], np.int64),
        trk_state=np.asarray([t.state is TrackState.LOST for t in tr], np.int64),
        trk_hits=np.asarray([t.hits for t in tr], np.int64),
        trk_lost=np.asarray([-1 if t.lost_since is None else t.lost_since for t in tr], np.int64),
        trk_last=np.asarray([t.last_update_frame for t in tr], np.int64),
        trk_mean=np.asarray([t.kalman.mean for t in tr], np.float64).reshape(-1, 8),
        trk_cov=np.asarray([t.kalman.covariance for t in tr], np.float64).reshape(-1, 8, 8),
        trk_emb=np.asarray([t.smooth_embedding for t in tr], np.float32).reshape(-1, dim),
        removed=np.asarray(sorted(tracker.removed_ids), np.int64),
    )
    print(f"{name}: frames={frames} dets={sum(counts)} records={len(rec_id)} "
          f"live={len(tr)} removed={len(tracker.removed_ids)}")


def units():
    out = {}
    # NMS: tests/test_acceptance.py:214-237 recipe (coarse scores force ties).
    rng = np.random.default_rng(27)
    nb, ns, nt, nk, noff = [], [], [], [], [0]
    for _ in range(500):
        count = int(rng.integers(1, 41))
        dets = []
        for _ in range(count):
            w, h = rng.uniform(5, 40, 2)
            dets.append(Detection(BoundingBox(float(rng.uniform(0, 120)), float(rng.uniform(0, 120)),
                                              float(w), float(h)),
                                  objectness=float(rng.integers(1, 11)) / 10.0))
        thr = float(rng.uniform(0.2, 0.7))
        kept = nms(dets, thr)
        mask = np.zeros(count, np.int64)
        for d in kept:
            mask[dets.index(d)] = 1
        nb.append(np.asarray([d.box.as_tlwh() for d in dets]))
        ns.append(np.asarray([d.objectness for d in dets]))
        nk.append(mask)
        nt.append(thr)
        noff.append(noff[-1] + count)
    out.update(nms_boxes=np.concatenate(nb), nms_scores=np.concatenate(ns),
               nms_keep=np.concatenate(nk), nms_thr=np.asarray(nt), nms_off=np.asarray(noff))

    # LAP: tests/test_acceptance.py:160-178 recipe plus tie-heavy integer matrices.
    rng = np.random.default_rng(25)
    mats, shapes, pairs, poff = [], [], [], [0]
    for trial in range(1200):
        nr, nc = int(rng.integers(1, 7)), int(rng.integers(1, 7))
        if trial < 1000:
            c = rng.uniform(0.0, 10.0, (nr, nc))
            if trial % 2:
                c[rng.random((nr, nc)) < rng.uniform(0.0, 0.7)] = np.inf
        else:
            c = rng.integers(0, 3, (nr, nc)).astype(np.float64)
            c[rng.random((nr, nc)) < 0.3] = np.inf
        a = hungarian_solve(c)
        mats.append(c.ravel())
        shapes.append((nr, nc))
        pairs.extend((r, col) for r, col, _ in a.matches)
        poff.append(len(pairs))
    out.update(lap_vals=np.concatenate(mats), lap_shapes=np.asarray(shapes, np.int64),
               lap_pairs=np.asarray(pairs, np.int64).reshape(-1, 2), lap_off=np.asarray(poff))

    # Kalman: tests/test_acceptance.py:181-211 recipe; ops tape + reference states.
    kf = KalmanFilter()
    rng = np.random.default_rng(26)
    ops, zs, means, covs, gates, gz = [], [], [], [], [], []
    for _ in range(300):
        z0 = np.array([rng.uniform(-500, 500), rng.uniform(-500, 500),
                       rng.uniform(0.3, 3.0), rng.uniform(10, 300)])
        st = kf.initiate(z0)
        ops.append(0); zs.append(z0); means.append(st.mean); covs.append(st.covariance)
        for _ in range(int(rng.integers(2, 6))):
            st = kf.predict(st)
            ops.append(1); zs.append(np.zeros(4)); means.append(st.mean); covs.append(st.covariance)
            probe = st.mean[:4] + rng.normal(0, 3.0, 4) * np.array([1, 1, 0.05, 1])
            gz.append(probe)
            gates.append(kf.gating_distance(st, probe[None, :])[0])
            if rng.random() < 0.7:
                z = st.mean[:4] + rng.normal(0, 2.0, 4) * np.array([1, 1, 0.02, 1])
                z[3] = max(z[3], 1.0)
                st = kf.update(st, z)
                ops.append(2); zs.append(z); means.append(st.mean); covs.append(st.covariance)
    out.update(kf_ops=np.asarray(ops, np.int64), kf_z=np.asarray(zs), kf_mean=np.asarray(means),
               kf_cov=np.asarray(covs), kf_gate=np.asarray(gates), kf_gate_z=np.asarray(gz))

    # normalize / binary16 on random vectors.
    rng = np.random.default_rng(31)
    raw = rng.standard_normal((64, 512)) * rng.uniform(0.01, 100, (64, 1))
    out.update(norm_in=raw, norm_out=np.stack([normalize(r) for r in raw]))
    q = (rng.standard_normal(4096) * np.exp(rng.uniform(-20, 10, 4096))).astype(np.float32)
    q = q[np.abs(q) <= 65504.0]
    out.update(fp16_in=q, fp16_out=quantize_binary16(q))
    np.savez_compressed(OUT / "units.npz", **out)
    print("units written")


def known_answers():
    kf = KalmanFilter()
    cov = np.zeros((8, 8))
    cov[:4, :4] = np.diag([3.0, 3.0, 4.0 - 1e-2, 3.0])
    st = KalmanState(mean=np.array([0.0, 0.0, 1.0, 20.0, 0, 0, 0, 0]), covariance=cov)
    ka = {
        "iou_1_7": iou(BoundingBox(0, 0, 2, 2), BoundingBox(1, 1, 2, 2)),          # tests/test_core.py:57-60
        "measurement": box_to_measurement(BoundingBox(10, 20, 4, 8)).tolist(),    # tests/test_core.py:75-78
        "fp16_0_1": float(quantize_binary16(np.array([0.1]))[0]),                 # tests/test_core.py:157-159
        "gate_scalar": float(kf.gating_distance(st, np.array([[2.0, 0.0, 1.0, 20.0]]))[0]),  # tests/test_motion.py:124-131
        "lap_2x2": [list(m[:2]) for m in hungarian_solve(np.array([[1.0, 2.0], [2.0, 4.0]])).matches],  # tests/test_assoc.py:87-90
    }
    (OUT / "known_answers.json").write_text(json.dumps(ka, indent=1) + "\n")
    print("known answers", ka)


if __name__ == "__main__":
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    for seq in SEQUENCES:
        run_sequence(*seq)
    units()
    known_answers()
