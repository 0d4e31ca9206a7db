"""The step-launched recurrence (rec_step.cu), the path for layers beyond the
persistent kernels' on-chip capacity: BASELINE C5's H = 1024 against the oracle, and the same
path forced at small sizes (BLSTM_FORCE_STEP=1) against the oracle and the persistent path."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from paper_1608_00895_b200 import synth  # noqa: E402
from tests.gpu_util import GRAD_TOL, OUT_TOL, Stack, grad_errors, norm_rel  # noqa: E402


@pytest.fixture
def force_step():
    os.environ["BLSTM_FORCE_STEP"] = "1"
    yield
    del os.environ["BLSTM_FORCE_STEP"]


def _check(L, D, H, K, T, lengths, side_stream=True, dropout=0.0):
    B = len(lengths)
    params = synth.stack_params(L, D, H, K)
    batch = synth.speech_batch(T, B, D, K, np.array(lengths), seed=1004)
    theta = oracle.pack_params(params, L, D, H, K)
    st = Stack(L, D, H, K, T, B, dropout=dropout, seed=5)
    got = st.step(theta, batch, side_stream=side_stream)
    ref = oracle.blstm_step(theta, batch.x, batch.mask, L, H, K, labels=batch.labels, want_states=True,
                            dropout=dropout, seed=5)
    assert abs(got["loss"] - ref["loss"]) / abs(ref["loss"]) < OUT_TOL
    errs = grad_errors(got["grad"], ref["grad"], L, D, H, K)
    assert max(errs.values()) < GRAD_TOL, errs
    if dropout == 0.0:
        Y, C = st.forward(theta, batch)
        for l in range(L):
            assert norm_rel(Y[l], ref["Ys"][l]) < OUT_TOL
            for d in range(2):
                assert norm_rel(C[l, d], ref["Cs"][l, d]) < OUT_TOL
    return got


def test_h1024_matches_oracle():
    """C5's width (H = 1024 > the persistent kernels' capacity): selected automatically."""
    _check(L=2, D=40, H=1024, K=17, T=6, lengths=[6, 5, 3, 6, 1])


def test_h1024_wide_batch():
    _check(L=1, D=40, H=1024, K=9, T=4, lengths=[4 - (i % 3) for i in range(130)])


@pytest.mark.parametrize("H", [64, 300])
def test_forced_step_small(force_step, H):
    _check(L=3, D=40, H=H, K=11, T=9, lengths=[9, 8, 6, 9, 3, 2, 1])


def test_forced_step_with_dropout(force_step):
    _check(L=2, D=40, H=130, K=11, T=7, lengths=[7, 5, 3, 7], dropout=0.25)


def test_forced_step_close_to_persistent():
    L, D, H, K, T = 2, 40, 130, 11, 9
    lengths = [9, 8, 6, 9, 3, 2, 1]
    params = synth.stack_params(L, D, H, K)
    batch = synth.speech_batch(T, len(lengths), D, K, np.array(lengths), seed=1004)
    theta = oracle.pack_params(params, L, D, H, K)
    a = Stack(L, D, H, K, T, len(lengths)).step(theta, batch, side_stream=True)
    os.environ["BLSTM_FORCE_STEP"] = "1"
    try:
        b = Stack(L, D, H, K, T, len(lengths)).step(theta, batch, side_stream=True)
    finally:
        del os.environ["BLSTM_FORCE_STEP"]
    assert abs(a["loss"] - b["loss"]) / abs(a["loss"]) < 1e-4
    errs = grad_errors(a["grad"], b["grad"], L, D, H, K)
    assert max(errs.values()) < GRAD_TOL, errs


@pytest.mark.parametrize("direction", [1, -1])
def test_single_layer_h1024(direction):
    """lstm_fwd / lstm_bwd beyond the persistent kernels' capacity (H = 1024) through the
    step-launched path, with h0 / c0 and the end-of-scan gradients dhT / dcT, against the oracle
    (y, c, hT, cT, dx, dW, dR, db, dh0, dc0)."""
    from tests.gpu_util import compare_layer, oracle_layer, run_layer
    case = synth.random_small_case(11, T=5, B=3, D=24, H=1024, lengths=np.array([5, 3, 0]))
    s = 1.0 / np.sqrt(1024)
    case["W"] = (case["W"] * s).astype(np.float32)
    case["R"] = (case["R"] * s).astype(np.float32)
    case["dy"] = (case["dy"] * case["mask"][..., None]).astype(np.float32)
    got = run_layer(case, direction, ldx_pad=3, ldy_pad=5)
    ref = oracle_layer(case, direction)
    compare_layer(got, ref, f"H=1024 dir={direction}")
    assert np.allclose(got["hT"][2], case["h0"][2], atol=1e-6)  # all-masked sequence carries h0


@pytest.mark.parametrize("direction,H", [(1, 1024), (-1, 1024), (1, 1000)])
def test_single_layer_persistent_bptt(direction, H):
    """lstm_bwd at H = 1024 and 1000 (Hq = 1024: padding units) through the persistent BPTT
    (rec_step.cu, ndir = 1): no launch per time step, ragged lengths with an empty sequence, row
    pitches wider than H, against the oracle."""
    from paper_1608_00895_b200 import blstm
    from tests.gpu_util import compare_layer, oracle_layer, run_layer
    T = 40
    rng = np.random.default_rng(13)
    lengths = rng.integers(1, T + 1, size=37)
    lengths[0], lengths[3] = T, 0
    case = synth.random_small_case(13, T=T, B=37, D=24, H=H, lengths=lengths)
    s = 1.0 / np.sqrt(H)
    case["W"] = (case["W"] * s).astype(np.float32)
    case["R"] = (case["R"] * s).astype(np.float32)
    case["dy"] = (case["dy"] * case["mask"][..., None]).astype(np.float32)
    n0 = blstm.blstm_launch_count()
    got = run_layer(case, direction, ldx_pad=3, ldy_pad=5)
    n = blstm.blstm_launch_count() - n0
    assert n < T, f"{n} launches for T = {T}: a per-step chain ran"
    compare_layer(got, oracle_layer(case, direction), f"persistent BPTT H={H} dir={direction}")


def test_forced_step_single_layer(force_step):
    from tests.gpu_util import compare_layer, oracle_layer, run_layer
    case = synth.random_small_case(12, T=9, B=5, D=7, H=70)
    s = 1.0 / np.sqrt(70)  # the paper-sized init scale of the layer tests (test_gpu_parity.py)
    case["W"] = (case["W"] * s).astype(np.float32)
    case["R"] = (case["R"] * s).astype(np.float32)
    case["dy"] = (case["dy"] * case["mask"][..., None]).astype(np.float32)
    for direction in (1, -1):
        compare_layer(run_layer(case, direction), oracle_layer(case, direction), f"forced dir={direction}")


@pytest.mark.parametrize("H,force", [(1024, False), (300, True)])
def test_persistent_forward_close_to_chain(H, force):
    """The persistent forward of the step path (B <= 128, Hq <= 1024; rec_step.cu) against the
    launched chain it replaces (BLSTM_STEP_PERSIST=1 forced vs =0): the same two K-half partial
    sums in the same order, but separately compiled gate math (FMA contraction may differ), so the
    outputs agree to rounding, not bit for bit."""
    L, D, K, T = 2, 40, 13, 7
    lengths = [7, 6, 2, 7, 1]
    params = synth.stack_params(L, D, H, K)
    batch = synth.speech_batch(T, len(lengths), D, K, np.array(lengths), seed=1006)
    theta = oracle.pack_params(params, L, D, H, K)
    out = {}
    if force:
        os.environ["BLSTM_FORCE_STEP"] = "1"
    try:
        for mode in ("0", "1"):
            os.environ["BLSTM_STEP_PERSIST"] = mode
            st = Stack(L, D, H, K, T, len(lengths))
            out[mode] = (st.forward(theta, batch), st.step(theta, batch, side_stream=True))
    finally:
        os.environ.pop("BLSTM_STEP_PERSIST", None)
        os.environ.pop("BLSTM_FORCE_STEP", None)
    (Y0, C0), g0 = out["0"]
    (Y1, C1), g1 = out["1"]
    for l in range(L):
        assert norm_rel(Y1[l], Y0[l]) < OUT_TOL
        for d in range(2):
            assert norm_rel(C1[l, d], C0[l, d]) < OUT_TOL
    assert abs(g1["loss"] - g0["loss"]) / abs(g0["loss"]) < 1e-4
    errs = grad_errors(g1["grad"], g0["grad"], L, D, H, K)
    assert max(errs.values()) < GRAD_TOL, errs


# ---------------------------------------------------------------------------------------------
# the persistent BPTT of the step path (rec_step.cu step_bwd_persist_kernel): R resident in TMEM +
# shared memory across 4-CTA clusters, no launch per time step
# ---------------------------------------------------------------------------------------------
def _launches_of_step(st, theta, batch):
    from paper_1608_00895_b200 import blstm
    n0 = blstm.blstm_launch_count()
    out = st.step(theta, batch, side_stream=True)
    return out, blstm.blstm_launch_count() - n0


@pytest.mark.parametrize("H,force", [(1024, False), (300, True)])
def test_persistent_bptt_matches_oracle(H, force):
    """Hq = 1024 (TMEM + shared-memory A operand) and Hq = 512 (TMEM only), ragged lengths with an
    empty sequence, B not a multiple of the 32-column ownership blocks."""
    if force:
        os.environ["BLSTM_FORCE_STEP"] = "1"
    try:
        rng = np.random.default_rng(3)
        T, B = 17, 37
        lengths = rng.integers(1, T + 1, size=B)
        lengths[0], lengths[5] = T, 0
        L, D, K = 2, 40, 13
        params = synth.stack_params(L, D, H, K)
        batch = synth.speech_batch(T, B, D, K, lengths, seed=1006)
        theta = oracle.pack_params(params, L, D, H, K)
        got, n = _launches_of_step(Stack(L, D, H, K, T, B), theta, batch)
        assert n < 2 * L * T, f"{n} launches: the per-step chain ran, not the persistent BPTT"
        ref = oracle.blstm_step(theta, batch.x, batch.mask, L, H, K, labels=batch.labels)
        assert abs(got["loss"] - ref["loss"]) / abs(ref["loss"]) < OUT_TOL
        errs = grad_errors(got["grad"], ref["grad"], L, D, H, K)
        assert max(errs.values()) < GRAD_TOL, errs
    finally:
        os.environ.pop("BLSTM_FORCE_STEP", None)


@pytest.mark.parametrize("H,B,force", [(1024, 128, False), (1024, 100, False), (300, 128, True)])
def test_persistent_bptt_close_to_chain(H, B, force):
    """Full 128-column batch (every owner block busy) over 40 steps: the persistent BPTT and the
    launched chain compute the same gradients up to rounding order (fp32 sums of fp16 products)."""
    if force:
        os.environ["BLSTM_FORCE_STEP"] = "1"
    try:
        T, L, D, K = 40, 2, 40, 11
        rng = np.random.default_rng(4)
        lengths = rng.integers(1, T + 1, size=B)
        lengths[0] = T
        params = synth.stack_params(L, D, H, K)
        batch = synth.speech_batch(T, B, D, K, lengths, seed=1007)
        theta = oracle.pack_params(params, L, D, H, K)
        a, na = _launches_of_step(Stack(L, D, H, K, T, B), theta, batch)
        os.environ["BLSTM_STEP_PERSIST_BWD"] = "0"
        try:
            b, nb = _launches_of_step(Stack(L, D, H, K, T, B), theta, batch)
        finally:
            del os.environ["BLSTM_STEP_PERSIST_BWD"]
        assert na < nb - L * T, (na, nb)
        assert abs(a["loss"] - b["loss"]) <= 1e-6 * abs(b["loss"])
        errs = grad_errors(a["grad"], b["grad"], L, D, H, K)
        assert max(errs.values()) < 2e-3, errs
    finally:
        os.environ.pop("BLSTM_FORCE_STEP", None)
