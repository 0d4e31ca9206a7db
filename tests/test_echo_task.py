"""The NEXT-1 delayed-echo task generator (synth.echo_batch): the label of frame t is the input
symbol of frame t-3 (0 before), padded frames carry x = 0 and label 0, so the task has an exact
answer a causal model can learn."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1608_00895_b200 import synth  # noqa: E402


def test_labels_are_delayed_inputs():
    b = synth.echo_batch(T=50, B=7, D=40, seed=3)
    V, k = synth.ECHO_SYMBOLS, synth.ECHO_DELAY
    sym = np.argmax(b.x[:, :, :V], axis=2) + 1
    for bi in range(7):
        n = int(b.lengths[bi])
        assert np.all(b.mask[:n, bi] == 1) and np.all(b.mask[n:, bi] == 0)
        assert np.all(b.labels[:k, bi] == 0)
        assert np.array_equal(b.labels[k:n, bi], sym[:n - k, bi])
        assert np.all(b.labels[n:, bi] == 0) and np.all(b.x[n:, bi] == 0)
        assert np.all(b.x[:n, bi, :V].sum(axis=1) == 1.0)  # one-hot symbol
    assert b.labels.max() <= V and b.lengths.max() == 50


def test_deterministic_and_seed_dependent():
    a, b, c = (synth.echo_batch(20, 4, 16, s) for s in (1, 1, 2))
    assert np.array_equal(a.x, b.x) and np.array_equal(a.labels, b.labels)
    assert not np.array_equal(a.x, c.x)
