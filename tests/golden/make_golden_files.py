"""Golden files for the detection-file source and MOT evaluation.

Run in the build container only (imports the read-only reference):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_files.py

Writes ``tests/golden/files/``:

* ``det.txt`` / ``det.emb`` - a MOT detection file and EMB1 sidecar written
  the way the reference's own CLI test does (``tests/test_cli.py:135-151``)
  from a reference scenario (``tf/detgen.py:161-258``);
* ``detfile_expected.npz`` - the reference's parse of both files
  (``load_mot_detections`` + ``load_embedding_sidecar``, ``tf/detgen.py:366-471``)
  and its tracker outputs over ``file_frames`` (parse_output + Tracker.step);
* ``gt.txt`` / ``res.txt`` - MOT ground truth of the scenario and the tracker
  result (``format_mot_row``, ``tf/cli.py:56-70``);
* ``moteval_expected.json`` - ``moteval.evaluate`` of res against gt
  (``tf/moteval.py:262-285``) plus the per-frame correspondences of
  ``moteval.accumulate`` for two iou_min values.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from trackforge import moteval                                            # noqa: E402
from trackforge.cli import format_mot_row                                 # noqa: E402
from trackforge.detgen import (NoiseParams, file_frames, load_embedding_sidecar,  # noqa: E402
                               load_mot_detections, make_scenario, scenario_frames,
                               scenario_ground_truth, write_embedding_sidecar)
from trackforge.postproc import parse_output                              # noqa: E402
from trackforge.tracker import Tracker, TrackerConfig                     # noqa: E402

OUT = Path(__file__).resolve().parent / "files"
DIM = 16


def main() -> None:
    OUT.mkdir(exist_ok=True)
    scen = make_scenario(num_objects=8, frames=40, seed=21, embedding_dim=DIM, layout="random",
                         noise=NoiseParams(p_miss=0.1, sigma_box=0.8, sigma_emb=0.03, lambda_fp=0.5))
    lines, sidecar = [], {}
    for frame_index, raw in scenario_frames(scen, seed=0):
        for det_index, row in enumerate(raw):
            x, y, w, h, conf = (float(v) for v in row[:5])
            lines.append(f"{frame_index + 1},-1,{x!r},{y!r},{w!r},{h!r},{conf!r}")
            sidecar[(frame_index, det_index)] = row[6:].astype(np.float32)
    (OUT / "det.txt").write_text("\n".join(lines) + "\n")
    write_embedding_sidecar(OUT / "det.emb", sidecar, DIM)

    dets = load_mot_detections(OUT / "det.txt")
    attached = load_embedding_sidecar(OUT / "det.emb", dets, DIM)
    tracker = Tracker(TrackerConfig(embedding_dim=DIM))
    frames, counts, rows = [], [], []
    rec = {"frame": [], "id": [], "box": [], "obj": []}
    res_lines = []
    for frame_index, r in file_frames(attached, scen.frames, 6 + DIM):
        frames.append(frame_index)
        counts.append(r.shape[0])
        rows.append(r)
        out = tracker.step(frame_index, parse_output(r, DIM))
        for tid, box, obj in out.records:
            rec["frame"].append(frame_index)
            rec["id"].append(tid)
            rec["box"].append(box.as_tlwh())
            rec["obj"].append(obj)
            res_lines.append(format_mot_row(frame_index, tid, box, obj))
    np.savez_compressed(
        OUT / "detfile_expected.npz",
        parsed_frames=np.asarray(list(dets), np.int64),
        parsed_counts=np.asarray([dets[f].shape[0] for f in dets], np.int64),
        parsed_rows=np.concatenate([dets[f] for f in dets]),
        frames=np.asarray(frames, np.int64), counts=np.asarray(counts, np.int64),
        rows=np.concatenate(rows), rec_frame=np.asarray(rec["frame"], np.int64),
        rec_id=np.asarray(rec["id"], np.int64), rec_box=np.asarray(rec["box"], np.float64).reshape(-1, 4),
        rec_obj=np.asarray(rec["obj"], np.float64))
    (OUT / "res.txt").write_text("".join(line + "\n" for line in res_lines))
    truth = scenario_ground_truth(scen)
    gt_lines = [format_mot_row(f, oid, box, 1.0) for f in sorted(truth) for oid, box in truth[f]]
    (OUT / "gt.txt").write_text("".join(line + "\n" for line in gt_lines))

    gt = moteval.load_mot_tracks(OUT / "gt.txt")
    hyp = moteval.load_mot_tracks(OUT / "res.txt")
    expected = {"report": dict(zip(moteval.MetricsReport.COLUMNS, moteval.evaluate(gt, hyp).row()))}
    for thr in (0.5, 0.3):
        corr = moteval.accumulate(gt, hyp, thr)
        expected[f"accumulate_{thr}"] = [[c.frame_index, [list(m) for m in c.matches], list(c.unmatched_gt),
                                          list(c.unmatched_hyp)] for c in corr]
    expected["id_metrics_0.5"] = list(moteval.id_metrics(gt, hyp, 0.5))
    (OUT / "moteval_expected.json").write_text(json.dumps(expected, indent=1) + "\n")
    print("detfile:", len(lines), "rows,", len(rec["id"]), "records; moteval:", expected["report"])


if __name__ == "__main__":
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    main()
