"""Mid-sequence reference track tables, for the resume (tf_import_tracks) tests.

Run in the build container only (imports the read-only reference):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_resume.py

For each sequence below, the reference ``Tracker`` (``tf/tracker.py:74-159``)
is stepped over the first ``k`` frames of the same scenario make_golden.py
uses, and its state then - ``tracks`` (every field), ``_next_id``,
``_last_frame`` - is written to ``resume_<name>.npz`` together with the
records of frames k.. of the uninterrupted run. A tracker resumed from that
state must reproduce those records exactly.
"""

from __future__ import annotations

import json

import numpy as np

from make_golden import OUT, SEQUENCES, generate_frame, make_scenario, parse_output  # noqa: F401
from make_golden import Tracker, TrackerConfig, TrackState, _quantize_detection

RESUME = {"noisy16": 20, "lifecycle16": 35, "random64": 40}


def state_arrays(tracker, dim):
    tr = tracker.tracks
    return dict(
        mid_id=np.asarray([t.track_id for t in tr], np.int64),
        mid_state=np.asarray([t.state is TrackState.LOST for t in tr], np.int64),
        mid_hits=np.asarray([t.hits for t in tr], np.int64),
        mid_lost=np.asarray([-1 if t.lost_since is None else t.lost_since for t in tr], np.int64),
        mid_last=np.asarray([t.last_update_frame for t in tr], np.int64),
        mid_mean=np.asarray([t.kalman.mean for t in tr], np.float64).reshape(-1, 8),
        mid_cov=np.asarray([t.kalman.covariance for t in tr], np.float64).reshape(-1, 8, 8),
        mid_emb=np.asarray([t.smooth_embedding for t in tr], np.float32).reshape(-1, dim),
        mid_next_id=np.int64(tracker._next_id),
        mid_last_frame=np.int64(tracker._last_frame),
    )


def main():
    for name, scen_kwargs, noise, overrides, frames, quantize in SEQUENCES:
        if name not in RESUME:
            continue
        k = RESUME[name]
        scen = make_scenario(frames=frames, noise=noise, **scen_kwargs)
        dim = scen.embedding_dim
        tracker = Tracker(TrackerConfig(embedding_dim=dim, **overrides))
        snap = None
        rec_frame, rec_id, rec_box, rec_obj = [], [], [], []
        for f in range(frames):
            if f == k:
                snap = state_arrays(tracker, dim)
                n_lost = int(snap["mid_state"].sum())
            raw, _ = generate_frame(scen, f, seed=scen_kwargs["seed"] + 100)
            dets = parse_output(raw, dim)
            if quantize:
                dets = [_quantize_detection(d) for d in dets]
            out = tracker.step(f, dets)
            if f >= k:
                for tid, box, obj in out.records:
                    rec_frame.append(f)
                    rec_id.append(tid)
                    rec_box.append(box.as_tlwh())
                    rec_obj.append(obj)
        np.savez_compressed(
            OUT / f"resume_{name}.npz",
            config=json.dumps(dict(overrides, embedding_dim=dim, quantize=quantize)),
            k=np.int64(k),
            rec_frame=np.asarray(rec_frame, np.int64),
            rec_id=np.asarray(rec_id, np.int64),
            rec_box=np.asarray(rec_box, np.float64).reshape(-1, 4),
            rec_obj=np.asarray(rec_obj, np.float64),
            **snap,
        )
        print(f"{name}: resume at {k}: live={len(snap['mid_id'])} lost={n_lost} "
              f"next_id={int(snap['mid_next_id'])} records after={len(rec_id)}")


if __name__ == "__main__":
    main()
