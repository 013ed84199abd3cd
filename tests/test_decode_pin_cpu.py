"""The decode oracle against the generator's encoded truth (no GPU).

oracle/heads.py is the builder's own statement of the decode (the reference
has none); this pins it to an independent one: synth.py's encoder. With zero
box-delta noise the decode of every encoded object must give back its truth
box (1e-6 relative, clamp-affected objects excluded; tests/decode_pin.py).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from decode_pin import match_truth   # noqa: E402
from oracle import heads as oh       # noqa: E402


@pytest.mark.parametrize("seed", [0, 1])
def test_oracle_decode_reproduces_generator_boxes(seed):
    from paper_2011_03910_b200 import synth

    gen = synth.make("cfg0", device="cpu", seed=seed, delta_sigma=0.0, dim=16)
    gen.record_truth()
    out = gen.next_batch(3)
    total = 0
    for b in range(3):
        heads = [h[b].numpy() for h in out.heads]
        embs = [e[b].numpy() for e in out.embs]
        codes, rows = oh.decode_frame(heads, embs)
        true_obj = rows[:, 4] == 1.0 / (1.0 + np.exp(-8.0))
        _, active, _, box = gen.truth[b]
        total += match_truth(rows[true_obj, :4], box[0][active[0]].numpy(), rtol=1e-6)
        # embeddings: the encoded identity vector (+ noise) lands at the object's cell
        assert np.all(np.isfinite(rows[:, 6:]))
    assert total >= 45, total


def test_decode_pin_detects_a_wrong_decode():
    """The pin is not vacuous: a decode off by one cell fails it."""
    from paper_2011_03910_b200 import synth

    gen = synth.make("cfg0", device="cpu", seed=3, delta_sigma=0.0, dim=16)
    gen.record_truth()
    out = gen.next_batch(1)
    _, rows = oh.decode_frame([h[0].numpy() for h in out.heads], [e[0].numpy() for e in out.embs])
    true_obj = rows[:, 4] == 1.0 / (1.0 + np.exp(-8.0))
    shifted = rows[true_obj, :4].copy()
    shifted[:, 0] += 8.0 * 1080 / 608
    _, active, _, box = gen.truth[0]
    with pytest.raises(AssertionError):
        match_truth(shifted, box[0][active[0]].numpy(), rtol=1e-6)
