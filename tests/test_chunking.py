"""Chunked data pipeline (NEXT-4): the host planner
(paper_1608_00895_b200.data) and its oracle (oracle/chunking.py), pinned by SPEC's worked
examples and by the invariants the rule fixes (coverage, conservation, determinism)."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import chunking as ref  # noqa: E402
from paper_1608_00895_b200 import data  # noqa: E402


def test_spec_examples():
    # L=738, C=250, S=250 -> 3 chunks, valid lens (250, 250, 238)
    assert [c.valid_len for c in data.chunk_sequences([738], 250, 250)] == [250, 250, 238]
    assert [n for _, n in ref.chunk_starts(738, 250, 250)] == [250, 250, 238]
    # L=100 <= C=250 -> 1 chunk, valid_len=100
    assert [(c.start, c.valid_len) for c in data.chunk_sequences([100], 250, 250)] == [(0, 100)]
    # L=300, C=250, S=125 -> starts 0, 125, 250
    assert [c.start for c in data.chunk_sequences([300], 250, 125)] == [0, 125, 250]
    assert [s for s, _ in ref.chunk_starts(300, 250, 125)] == [0, 125, 250]


@pytest.mark.parametrize("C,S", [(250, 250), (250, 125), (7, 3), (5, 1), (1, 1)])
def test_coverage_and_agreement(C, S):
    g = np.random.default_rng(C * 31 + S)
    lengths = g.integers(1, 4 * C + 3, size=40)
    chunks = data.chunk_sequences(lengths, C, S)
    for s, L in enumerate(lengths):
        mine = [(c.start, c.valid_len) for c in chunks if c.seq == s]
        assert mine == ref.chunk_starts(int(L), C, S)
        cov = np.zeros(L, np.int32)
        for a, n in mine:
            assert 1 <= n <= C and a % S == 0
            cov[a:a + n] += 1
        assert cov.min() >= 1                      # every frame covered
        if S == C:
            assert cov.max() == 1                  # no overlap without overlap step
    if S == C:
        assert sum(c.valid_len for c in chunks) == lengths.sum()


def test_errors():
    with pytest.raises(ValueError):
        data.chunk_sequences([10], 5, 6)
    with pytest.raises(ValueError):
        data.chunk_sequences([10], 5, 0)
    with pytest.raises(ValueError):
        data.chunk_sequences([], 5, 5)


def test_make_batches():
    chunks = data.chunk_sequences([3, 2], 1, 1)  # 5 chunks
    bs = data.make_batches(chunks, 2, seed=7)
    assert [len(b) for b in bs] == [2, 2, 1]
    assert data.make_batches(chunks, 2, seed=7) == bs
    assert sorted((c.seq, c.start) for b in bs for c in b) == sorted((c.seq, c.start) for c in chunks)
    assert data.chunk_frames(bs) == 5          # conservation


def test_gather_chunks_golden():
    """Pin of oracle.chunking.gather_chunks (an off-by-one in seq_offset or a label written at
    padding fails): the hand-written batch of tests/golden/chunk_gather.txt."""
    rows = [list(map(float, ln.split())) for ln in open(os.path.join(os.path.dirname(__file__), "golden",
                                                                    "chunk_gather.txt"))
            if ln.strip() and not ln.startswith("#")]
    T, B, D = 4, 5, 2
    exp = np.array(rows)[:, 1:].reshape(T, B, 4)
    frames = np.array([[f + 1, -(f + 1)] for f in range(8)], np.float32)
    flabels = np.arange(10, 18, dtype=np.int32)
    seq_offset = [0, 5, 8]
    chunks = [(s, a, n) for s, L in enumerate((5, 3)) for a, n in ref.chunk_starts(L, 4, 2)]
    assert chunks == [(0, 0, 4), (0, 2, 3), (0, 4, 1), (1, 0, 3), (1, 2, 1)]
    x, mask, labels = ref.gather_chunks(frames, flabels, seq_offset, chunks, T)
    assert np.array_equal(x, exp[..., :D].astype(np.float32))
    assert np.array_equal(mask, exp[..., 2].astype(np.uint8))
    assert np.array_equal(labels, exp[..., 3].astype(np.int32))
