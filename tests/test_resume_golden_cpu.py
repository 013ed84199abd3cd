"""The mid-sequence reference states (tests/golden/resume_*.npz) against the
full golden runs: the records after the resume frame are the uninterrupted
run's, and every covariance is in the per-axis (position, velocity) form the
device filter stores and tf_import_tracks requires (tf/motion.py:61-126)."""

import json

import numpy as np
import pytest

from goldens import GOLDEN, load_sequence

RESUME = ["noisy16", "lifecycle16", "random64"]


@pytest.mark.parametrize("name", RESUME)
def test_resume_golden_is_a_suffix_of_the_full_run(name):
    z = np.load(GOLDEN / f"resume_{name}.npz")
    seq = load_sequence(name)
    k = int(z["k"])
    sel = seq["rec_frame"] >= k
    assert np.array_equal(z["rec_frame"], seq["rec_frame"][sel])
    assert np.array_equal(z["rec_id"], seq["rec_id"][sel])
    assert np.array_equal(z["rec_box"], seq["rec_box"][sel])
    assert np.array_equal(z["rec_obj"], seq["rec_obj"][sel])
    assert json.loads(str(z["config"])) == seq["config"]
    assert int(z["mid_last_frame"]) == k - 1
    assert z["mid_state"].sum() > 0          # LOST tracks are part of the resumed state


@pytest.mark.parametrize("name", RESUME)
def test_reference_covariances_are_per_axis_blocks(name):
    z = np.load(GOLDEN / f"resume_{name}.npz")
    for C8 in z["mid_cov"]:
        i, j = np.indices((8, 8))
        assert np.all(C8[(i % 4) != (j % 4)] == 0.0)
        assert np.array_equal(C8, C8.T)
    assert np.all(z["mid_id"] < int(z["mid_next_id"]))
    assert len(set(z["mid_id"].tolist())) == len(z["mid_id"])
    assert np.array_equal(z["mid_state"] == 1, z["mid_lost"] >= 0)
