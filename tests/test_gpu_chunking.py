"""blstm_gather_chunks (NEXT-4) against the oracle's gather (oracle/chunking.py): bit-exact,
with overlapping chunks, partial last chunks, empty columns and a batch wider than the chunk
list."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle import chunking as ref  # noqa: E402
from paper_1608_00895_b200 import data  # noqa: E402


@pytest.mark.parametrize("C,S,D", [(250, 250, 40), (250, 125, 40), (17, 5, 3)])
def test_gather_bit_exact(C, S, D):
    dev = torch.device("cuda:0")
    g = np.random.default_rng(C + S + D)
    lengths = g.integers(1, 3 * C, size=13)
    xs = [g.normal(size=(L, D)).astype(np.float32) for L in lengths]
    ls = [g.integers(0, 1501, size=L).astype(np.int32) for L in lengths]
    corpus = data.DeviceCorpus(xs, ls, dev)
    chunks = data.chunk_sequences(lengths, C, S)
    B = 11
    for batch in data.make_batches(chunks, B, seed=3):
        x = torch.full((C, B, D), 7.0, device=dev)
        m = torch.full((C, B), 9, dtype=torch.uint8, device=dev)
        lab = torch.full((C, B), -1, dtype=torch.int32, device=dev)
        corpus.gather(batch, C, x, m, lab)
        off = np.concatenate([[0], np.cumsum(lengths)])
        rx, rm, rl = ref.gather_chunks(np.concatenate(xs), np.concatenate(ls), off,
                                       [(c.seq, c.start, c.valid_len) for c in batch] +
                                       [(0, 0, 0)] * (B - len(batch)), C)
        assert np.array_equal(x.cpu().numpy(), rx)
        assert np.array_equal(m.cpu().numpy(), rm)
        assert np.array_equal(lab.cpu().numpy(), rl)


def test_planned_epoch_equals_per_batch_gather():
    dev = torch.device("cuda:0")
    g = np.random.default_rng(5)
    lengths = g.integers(1, 600, size=9)
    xs = [g.normal(size=(L, 8)).astype(np.float32) for L in lengths]
    corpus = data.DeviceCorpus(xs, None, dev)
    batches = data.make_batches(data.chunk_sequences(lengths, 250, 100), 4, seed=1)
    corpus.plan_epoch(batches, 4, 250)
    for k, batch in enumerate(batches):
        a = torch.empty((250, 4, 8), device=dev)
        am = torch.empty((250, 4), dtype=torch.uint8, device=dev)
        b = torch.empty_like(a)
        bm = torch.empty_like(am)
        corpus.gather(batch, 250, a, am)
        corpus.gather_planned(k, b, bm)
        assert torch.equal(a, b) and torch.equal(am, bm)
