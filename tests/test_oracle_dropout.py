"""Pins of the oracle's input dropout (oracle.c ref_blstm_step_ex; "dropout on
the layer inputs of any layer"; R20):

* the keep draw: rate 1-p, independent across sites and seeds, p = 0 keeps everything;
* layer 0: the step with dropout equals the step WITHOUT dropout on the hand-masked input
  x~ = x * keep / (1-p) (masks recomputed here from ref_dropout_keep), and dX = dX~ * keep/(1-p);
* the whole stack (layer-1 input and head input dropped too): central finite differences of
  the loss with the masks held fixed (fixed seed) match the analytic gradient.
"""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle  # noqa: E402
from paper_1608_00895_b200 import synth  # noqa: E402


def _mask(seed, site, rows, Dl, p):
    return np.array([[oracle.dropout_keep(seed, site, r * Dl + j, p) for j in range(Dl)] for r in range(rows)],
                    np.float64)


def test_keep_rate_and_independence():
    p, n = 0.3, 40000
    a = np.array([oracle.dropout_keep(11, 0, i, p) for i in range(n)], np.float64)
    b = np.array([oracle.dropout_keep(11, 1, i, p) for i in range(n)], np.float64)
    c = np.array([oracle.dropout_keep(12, 0, i, p) for i in range(n)], np.float64)
    sd = np.sqrt(p * (1 - p) / n)
    for m in (a, b, c):
        assert abs(m.mean() - (1 - p)) < 5 * sd
    for u, v in ((a, b), (a, c)):  # different site / seed: uncorrelated
        assert abs(np.corrcoef(u, v)[0, 1]) < 5 / np.sqrt(n)
    assert all(oracle.dropout_keep(3, 2, i, 0.0) for i in range(1000))


def test_layer0_equals_masked_input():
    L, T, B, D, H = 1, 5, 3, 4, 3
    p, seed = 0.4, 77
    params = synth.stack_params(L, D, H, 0)
    theta = oracle.pack_params(params, L, D, H, 0)
    case = synth.random_small_case(5, T, B, D, H, lengths=np.array([5, 4, 2]))
    x = case["x"].astype(np.float64)
    mask = case["mask"]
    dy = synth.rng(3).standard_normal((T, B, 2 * H)) * mask[..., None]
    keep = _mask(seed, 0, T * B, D, p).reshape(T, B, D)
    xt = x * keep / (1 - p)
    a = oracle.blstm_step(theta, x, mask, L, H, 0, dy_top=dy, want_states=True, want_dx=True, dropout=p, seed=seed)
    b = oracle.blstm_step(theta, xt, mask, L, H, 0, dy_top=dy, want_states=True, want_dx=True)
    assert np.array_equal(a["grad"], b["grad"])
    assert np.array_equal(a["Ys"], b["Ys"])
    assert np.array_equal(a["dX1"], b["dX1"] * keep / (1 - p))
    assert 0 < keep.mean() < 1


def test_stack_with_dropout_central_fd():
    L, T, B, D, H, K = 2, 4, 3, 3, 3, 5
    p, seed = 0.3, 5
    params = synth.stack_params(L, D, H, K)
    batch = synth.speech_batch(T, B, D, K, np.array([4, 3, 2]), seed=9)
    theta = oracle.pack_params(params, L, D, H, K)
    g = synth.rng(4)
    theta = theta + 0.3 * g.standard_normal(theta.size)

    def step(th):
        return oracle.blstm_step(th, batch.x, batch.mask, L, H, K, labels=batch.labels, dropout=p, seed=seed)
    res = step(theta)
    ref = oracle.blstm_step(theta, batch.x, batch.mask, L, H, K, labels=batch.labels)
    assert res["loss"] != ref["loss"]  # dropout changes the step
    idx = g.choice(theta.size, size=60, replace=False)
    eps = 1e-4
    fd = np.array([(step(theta + eps * np.eye(1, theta.size, i)[0])["loss"]
                    - step(theta - eps * np.eye(1, theta.size, i)[0])["loss"]) / (2 * eps) for i in idx])
    an = res["grad"][idx]
    assert np.max(np.abs(fd - an) / np.maximum(1e-7, np.abs(fd) + np.abs(an))) <= 1e-5


def test_p_zero_is_no_dropout():
    L, T, B, D, H, K = 2, 4, 3, 3, 3, 5
    params = synth.stack_params(L, D, H, K)
    batch = synth.speech_batch(T, B, D, K, np.array([4, 3, 2]), seed=9)
    theta = oracle.pack_params(params, L, D, H, K)
    a = oracle.blstm_step(theta, batch.x, batch.mask, L, H, K, labels=batch.labels, dropout=0.0, seed=123)
    b = oracle.blstm_step(theta, batch.x, batch.mask, L, H, K, labels=batch.labels)
    assert a["loss"] == b["loss"] and np.array_equal(a["grad"], b["grad"])
