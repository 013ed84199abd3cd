"""CPU checks of the drop-in boundary: the C-ABI library loads and exports every
symbol include/trackforge_b200.h declares; host-side logic without a GPU."""

import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "trackforge_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(tf_\w+)\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2011_03910_b200 import _build, _lib

    _build.build()
    lib = _lib.load()
    decl = declared_symbols()
    assert len(decl) >= 20
    for name in decl:
        assert hasattr(lib, name), name
    assert set(decl) == set(_lib.EXPORTED)
    assert lib.tf_version() == 3
    assert lib.tf_status_name(7) == b"ConfigError"
    assert lib.tf_status_name(8) == b"OrderingError"


def test_status_codes_map_to_reference_exceptions():
    import paper_2011_03910_b200 as p
    from paper_2011_03910_b200 import errors

    names = {1: "InvalidBoxError", 2: "InvalidMeasurementError", 3: "DimensionError",
             4: "DegenerateEmbeddingError", 5: "PrecisionOverflowError", 6: "LayoutError",
             7: "ConfigError", 8: "OrderingError", 9: "NumericError"}
    for code, name in names.items():
        assert errors.STATUS_TO_ERROR[code].__name__ == name
        assert issubclass(errors.STATUS_TO_ERROR[code], p.TrackforgeError)


def test_no_cpu_fallback_without_cuda():
    import torch

    import paper_2011_03910_b200 as p

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError, match="CUDA"):
        p.Tracker(p.TrackerConfig(embedding_dim=8))
    with pytest.raises(RuntimeError, match="CUDA"):
        p.normalize(np.ones(4))


def test_host_value_types_mirror_reference():
    import paper_2011_03910_b200 as p

    b = p.BoundingBox(10, 20, 4, 8)
    assert (b.right, b.bottom, b.area) == (14, 28, 32)
    assert p.box_to_measurement(b).tolist() == [12.0, 24.0, 0.5, 8.0]   # tests/test_core.py:75-78
    with pytest.raises(p.InvalidBoxError):
        p.BoundingBox(0, 0, -1, 4)
    with pytest.raises(p.ConfigError):
        p.filter_confidence([], 1.5)
    with pytest.raises(p.LayoutError):
        p.parse_output(np.zeros((1, 13)), embedding_dim=8)
    assert p.parse_output(np.zeros((0, 14)), embedding_dim=8) == []


def test_letterbox_and_anchor_geometry_match_oracle():
    from oracle import heads as oh
    from paper_2011_03910_b200 import heads as ph

    assert ph.letterbox() == oh.letterbox() == (1080 / 608, 3.5, 0.0)
    assert ph.TOTAL_ANCHORS == oh.TOTAL_ANCHORS == 54264
    assert ph.ANCHORS == oh.ANCHORS and ph.GRID == oh.GRID and ph.STRIDES == oh.STRIDES


def test_synthetic_generator_cpu_decode_oracle():
    """Generator + decode oracle + oracle tracker on the CPU: every visible object
    is decoded back to a candidate near its true box, and IDs persist."""
    from oracle import heads as oh
    from oracle import tracker as ot
    from paper_2011_03910_b200 import synth

    g = synth.make("cfg0", device="cpu", seed=3, p_miss=0.0)
    out = g.next_batch(4)
    trk = ot.OracleTracker(ot.Settings())
    for b in range(4):
        codes, rows = oh.decode_frame([h[b].numpy() for h in out.heads], [e[b].numpy() for e in out.embs])
        assert 18 <= len(codes) <= 26          # 20 objects (+ rare spurious / collisions)
        tr = trk.step(b, ot.rows_to_dets(rows, 512))
        if b > 0:
            assert len(tr.matches) >= 18
    assert trk.next_id <= 20 + 4 * 4    # 20 identities + a few spurious candidates per frame
