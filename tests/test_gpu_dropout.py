"""Input dropout in blstm_stack_fwd_bwd (NEXT-4, R20) against the
oracle's step with the same counter-based masks (oracle.c ref_blstm_step_ex): loss and every
gradient tensor within the path's tolerances, every site (layer 0 input, the inputs of layers
>= 1, the head input) exercised; the no-head path; p = 0 is bitwise the plain step; a new seed
gives a different step."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from paper_1608_00895_b200 import synth  # noqa: E402
from tests.gpu_util import GRAD_TOL, OUT_TOL, Stack, grad_errors  # noqa: E402


@pytest.mark.parametrize("L,H,K,p", [(2, 64, 17, 0.25), (3, 130, 11, 0.5), (2, 300, 9, 0.125)])
def test_stack_dropout_matches_oracle(L, H, K, p):
    D, T, B, seed = 40, 9, 7, 4242
    params = synth.stack_params(L, D, H, K)
    batch = synth.speech_batch(T, B, D, K, np.array([9, 8, 6, 9, 3, 2, 1]), seed=1002)
    theta = oracle.pack_params(params, L, D, H, K)
    pf = float(np.float32(p))  # the descriptor carries fp32
    got = Stack(L, D, H, K, T, B, dropout=pf, seed=seed).step(theta, batch, side_stream=True)
    ref = oracle.blstm_step(theta, batch.x, batch.mask, L, H, K, labels=batch.labels, dropout=pf, seed=seed)
    plain = oracle.blstm_step(theta, batch.x, batch.mask, L, H, K, labels=batch.labels)
    # the masks matter (at init the loss hardly depends on the inputs; the gradients do)
    assert np.linalg.norm(ref["grad"] - plain["grad"]) > 0.05 * np.linalg.norm(plain["grad"])
    assert abs(got["loss"] - ref["loss"]) / abs(ref["loss"]) < OUT_TOL
    errs = grad_errors(got["grad"], ref["grad"], L, D, H, K)
    assert max(errs.values()) < GRAD_TOL, errs


def test_no_head_dropout():
    L, D, H, T, B, p, seed = 2, 40, 64, 10, 5, 0.25, 9
    params = synth.stack_params(L, D, H, 0)
    batch = synth.speech_batch(T, B, D, 0, np.array([10, 7, 5, 10, 2]), seed=1001)
    dy = (synth.rng(3).standard_normal((T, B, 2 * H)) * batch.mask[..., None]).astype(np.float32)
    theta = oracle.pack_params(params, L, D, H, 0)
    got = Stack(L, D, H, 0, T, B, dropout=p, seed=seed).step(theta, batch, dy_top=dy)
    ref = oracle.blstm_step(theta, batch.x, batch.mask, L, H, 0, dy_top=dy, dropout=p, seed=seed)
    errs = grad_errors(got["grad"], ref["grad"], L, D, H, 0)
    assert max(errs.values()) < GRAD_TOL, errs


def test_p_zero_bitwise_and_seed_matters():
    L, D, H, K, T, B = 2, 40, 64, 17, 8, 5
    params = synth.stack_params(L, D, H, K)
    batch = synth.speech_batch(T, B, D, K, np.array([8, 6, 5, 3, 1]), seed=1000)
    theta = oracle.pack_params(params, L, D, H, K)
    a = Stack(L, D, H, K, T, B).step(theta, batch)
    b = Stack(L, D, H, K, T, B, dropout=0.0, seed=77).step(theta, batch)
    assert np.array_equal(a["grad"], b["grad"]) and a["loss"] == b["loss"]
    c = Stack(L, D, H, K, T, B, dropout=0.25, seed=1).step(theta, batch)
    d = Stack(L, D, H, K, T, B, dropout=0.25, seed=2).step(theta, batch)
    e = Stack(L, D, H, K, T, B, dropout=0.25, seed=2).step(theta, batch)
    assert c["loss"] != d["loss"]
    assert np.array_equal(d["grad"], e["grad"])  # reproducible for a fixed seed
