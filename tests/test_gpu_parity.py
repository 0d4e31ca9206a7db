"""GPU parity: the CUDA path through the C-ABI vs the fp64 oracle, element by
element on the same seeded inputs (tests/gpu_util.py states the tolerances)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a GPU", allow_module_level=True)

import oracle  # noqa: E402
from paper_1608_00895_b200 import blstm, synth  # noqa: E402
from tests.gpu_util import (GRAD_TOL, OUT_TOL, Stack, T_, compare_layer, dev, grad_errors, l2_rel,  # noqa: E402
                            norm_rel, np_, oracle_layer, run_layer)


# ----------------------------------------------------------------------------
# the tcgen05 GEMM (test hook) vs a plain PyTorch fp32 product of the same fp16 operands
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (300, 200, 130), (20250 // 50, 1501, 1024), (64, 40, 8),
                                   (1000, 2048, 512),
                                   # >= 74 tiles of 256 x 256: the CTA-pair kernel (M and N tails; exact)
                                   (4000, 1200, 320), (4096, 1280, 256),
                                   # long K: split-K on the single-CTA kernel, and on the pair kernel
                                   (500, 300, 8192), (4096, 1000, 12288)])
def test_gemm_tcgen05_matches_torch(a_mn, b_mn, M, N, K):
    g = torch.Generator(device="cpu").manual_seed(M * 7 + N * 3 + K)
    A = torch.randn(M, K, generator=g).half()
    Bm = torch.randn(N, K, generator=g).half()
    ref = (A.double() @ Bm.double().T).float()  # exact products, fp64 sums
    bias = torch.randn(N, generator=g)
    ref_b = 0.5 * ref + bias
    # fp32 accumulation over K terms (any order: TMEM, split-K partials): error ~ sqrt(K) ulps
    tol = 1e-5 * max(1.0, (K / 1024) ** 0.5)
    def padded(X):  # row stride a multiple of 8 elements (TMA: 16-byte strides)
        r, c = X.shape
        buf = torch.zeros(r, (c + 7) // 8 * 8, dtype=X.dtype)
        buf[:, :c] = X
        return buf.to(dev())[:, :c]

    Ad = padded(A.T.contiguous() if a_mn else A)
    Bd = padded(Bm.T.contiguous() if b_mn else Bm)
    C = torch.zeros(M, N, device=dev())
    blstm.blstm_gemm_f16(Ad, a_mn, Bd, b_mn, C, M, N, K, alpha=0.5, bias=bias.to(dev()))
    torch.cuda.synchronize()
    err = (C.cpu() - ref_b).abs().max().item() / ref_b.abs().max().item()
    assert err < tol, err
    # beta accumulate
    blstm.blstm_gemm_f16(Ad, a_mn, Bd, b_mn, C, M, N, K, alpha=1.0, beta=1)
    torch.cuda.synchronize()
    err2 = (C.cpu() - (ref_b + ref)).abs().max().item() / (ref_b + ref).abs().max().item()
    assert err2 < tol, err2


# ----------------------------------------------------------------------------
# one layer, one direction (lstm_fwd / lstm_bwd)
# ----------------------------------------------------------------------------
def _c1_case(state):
    """Config C1 (BASELINE.json configs[0]): D=4, H=8, B=2, T=10, lengths (10, 7)."""
    cfg, params, batch = synth.make_workload(synth.CONFIGS["C1"])
    p = params.layers[0][0]
    g = synth.rng(77)
    case = dict(x=batch.x, mask=batch.mask, W=p.W, R=p.R, b=p.b,
                h0=(0.5 * g.standard_normal((2, 8))).astype(np.float32) if state else np.zeros((2, 8), np.float32),
                c0=(0.5 * g.standard_normal((2, 8))).astype(np.float32) if state else np.zeros((2, 8), np.float32),
                dy=(g.standard_normal((10, 2, 8)) * batch.mask[..., None]).astype(np.float32),
                dhT=g.standard_normal((2, 8)).astype(np.float32), dcT=g.standard_normal((2, 8)).astype(np.float32))
    return case


@pytest.mark.parametrize("direction", [1, -1])
@pytest.mark.parametrize("state", [False, True])
def test_layer_c1(direction, state):
    case = _c1_case(state)
    got = run_layer(case, direction, with_state=state)
    ref = oracle_layer(case, direction, with_state=state)
    compare_layer(got, ref, f"C1 dir={direction} state={state}")
    assert np.all(got["y"][case["mask"] == 0] == 0)


@pytest.mark.parametrize("T,B,D,H,seed", [
    (1, 1, 3, 5, 0),        # single frame, single sequence
    (17, 5, 70, 130, 1),    # H not a multiple of the 32-unit CTA slice; Hq = 256 (2 M tiles)
    (9, 37, 16, 33, 2),     # batch padded to the MMA N granularity, several groups
    (40, 3, 40, 500, 3),    # the paper-sized layer width
    (25, 64, 8, 64, 4),
    (3, 300, 10, 300, 5),   # one direction, G = 9 groups of 34: MMA N = 64; ldy_pad makes c / dy repacked
])
@pytest.mark.parametrize("direction", [1, -1])
def test_layer_random_shapes(T, B, D, H, seed, direction):
    case = synth.random_small_case(seed, T, B, D, H, state_scale=0.5)
    # scale weights like the paper-sized init so activations stay in range
    s = 1.0 / np.sqrt(max(D, H))
    case["W"] = (case["W"] * s).astype(np.float32)
    case["R"] = (case["R"] * s).astype(np.float32)
    case["dy"] = (case["dy"] * case["mask"][..., None]).astype(np.float32)
    got = run_layer(case, direction, ldx_pad=3, ldy_pad=5)
    ref = oracle_layer(case, direction)
    compare_layer(got, ref, f"T={T} B={B} D={D} H={H} dir={direction}")
    assert np.all(got["y_pad"] == 7.0), "y row padding (ldy) must be untouched"
    assert np.all(got["dx_pad"] == 3.0), "dx row padding (ldx) must be untouched"


def test_layer_all_masked_column_and_empty_frames():
    case = synth.random_small_case(5, 8, 4, 6, 20, lengths=np.array([8, 0, 3, 1]))
    case["dy"] = (case["dy"] * case["mask"][..., None]).astype(np.float32)
    for direction in (1, -1):
        got = run_layer(case, direction)
        ref = oracle_layer(case, direction)
        compare_layer(got, ref, f"masked dir={direction}")
        # the all-masked sequence carries h0/c0 and has zero output / dx
        assert np.allclose(got["hT"][1], case["h0"][1], atol=1e-6)
        assert np.allclose(got["cT"][1], case["c0"][1], atol=1e-6)
        assert np.all(got["y"][:, 1] == 0) and np.all(got["dx"][:, 1] == 0)


@pytest.mark.parametrize("precision", [0, 1], ids=["fp16", "fp16x2w"])
@pytest.mark.parametrize("direction", [1, -1])
def test_layer_c2(direction, precision):
    """Config C2 (BASELINE.json configs[1]) per direction: H=500, D=40, B=32, T=500, masked; in both
    precision modes (blstm.h BLSTM_PREC_*)."""
    cfg, params, batch = synth.make_workload(synth.CONFIGS["C2"])
    p = params.layers[0][0 if direction > 0 else 1]
    H = cfg.H
    dy = batch.dy_top[..., (0 if direction > 0 else H):(H if direction > 0 else 2 * H)]
    case = dict(x=batch.x, mask=batch.mask, W=p.W, R=p.R, b=p.b, h0=np.zeros((cfg.B, H), np.float32),
                c0=np.zeros((cfg.B, H), np.float32), dy=np.ascontiguousarray(dy),
                dhT=np.zeros((cfg.B, H), np.float32), dcT=np.zeros((cfg.B, H), np.float32))
    got = run_layer(case, direction, with_state=False, precision=precision)
    ref = oracle_layer(case, direction, with_state=False)
    errs = compare_layer(got, ref, f"C2 dir={direction} precision={precision}")
    print("C2 errors", direction, precision, errs)


def test_layer_deterministic():
    case = synth.random_small_case(9, 30, 9, 20, 96)
    case["W"] = (case["W"] * 0.2).astype(np.float32)
    case["R"] = (case["R"] * 0.1).astype(np.float32)
    a = run_layer(case, -1)
    b = run_layer(case, -1)
    for k in a:
        assert np.array_equal(a[k], b[k]), k


# ----------------------------------------------------------------------------
# the BLSTM stack + CE head (blstm_stack_fwd_bwd)
# ----------------------------------------------------------------------------
def test_stack_small_with_head():
    L, D, H, K, T, B = 2, 40, 64, 17, 12, 5
    params = synth.stack_params(L, D, H, K)
    batch = synth.speech_batch(T, B, D, K, np.array([12, 9, 7, 3, 1]), seed=1000)
    theta = oracle.pack_params(params, L, D, H, K)
    st = Stack(L, D, H, K, T, B)
    got = st.step(theta, batch)
    ref = oracle.blstm_step(theta, batch.x, batch.mask, L, H, K, labels=batch.labels, want_states=True)
    assert abs(got["loss"] - ref["loss"]) / abs(ref["loss"]) < OUT_TOL
    errs = grad_errors(got["grad"], ref["grad"], L, D, H, K)
    assert max(errs.values()) < GRAD_TOL, errs
    Y, C = st.forward(theta, batch)
    for l in range(L):
        assert norm_rel(Y[l], ref["Ys"][l]) < OUT_TOL
        for d in range(2):
            assert norm_rel(C[l, d], ref["Cs"][l, d]) < OUT_TOL


@pytest.mark.parametrize("H,B", [(64, 300),    # Hq = 256 (one BPTT pair tile), G = 9 groups of 34 -> MMA N = 64
                                 (300, 140)])  # Hq = 512 (two pair tiles), G = 4 groups of 35 -> N = 64
def test_stack_wide_groups_n64(H, B):
    """The N = 64 instantiations of both recurrence kernels (4 K-split accumulators x 64 columns next
    to the resident R in TMEM) and their native layouts, through a full training step."""
    L, D, K, T = 1, 12, 7, 4
    params = synth.stack_params(L, D, H, K)
    lengths = np.array([T - (i % 3) for i in range(B)])
    batch = synth.speech_batch(T, B, D, K, lengths, seed=1003)
    theta = oracle.pack_params(params, L, D, H, K)
    st = Stack(L, D, H, K, T, B)
    got = st.step(theta, batch, side_stream=True)
    ref = oracle.blstm_step(theta, batch.x, batch.mask, L, H, K, labels=batch.labels, want_states=True)
    assert abs(got["loss"] - ref["loss"]) / abs(ref["loss"]) < OUT_TOL
    errs = grad_errors(got["grad"], ref["grad"], L, D, H, K)
    assert max(errs.values()) < GRAD_TOL, errs
    Y, C = st.forward(theta, batch)
    assert norm_rel(Y[0], ref["Ys"][0]) < OUT_TOL
    for d in range(2):
        assert norm_rel(C[0, d], ref["Cs"][0, d]) < OUT_TOL


def test_stack_side_stream_bitwise_equal():
    """Weight-gradient GEMMs on a side stream (overlapping BPTT) give bitwise the same step."""
    L, D, H, K, T, B = 3, 40, 130, 11, 9, 7
    params = synth.stack_params(L, D, H, K)
    batch = synth.speech_batch(T, B, D, K, np.array([9, 8, 6, 9, 3, 2, 1]), seed=1002)
    theta = oracle.pack_params(params, L, D, H, K)
    st = Stack(L, D, H, K, T, B)
    a = st.step(theta, batch)
    b = st.step(theta, batch, side_stream=True)
    assert np.array_equal(a["grad"], b["grad"]) and a["loss"] == b["loss"]
    ref = oracle.blstm_step(theta, batch.x, batch.mask, L, H, K, labels=batch.labels)
    errs = grad_errors(b["grad"], ref["grad"], L, D, H, K)
    assert max(errs.values()) < GRAD_TOL, errs


def test_stack_no_head_dy_top():
    L, D, H, T, B = 1, 40, 130, 20, 6
    params = synth.stack_params(L, D, H, 0)
    batch = synth.speech_batch(T, B, D, 0, np.array([20, 17, 9, 20, 4, 1]), seed=1001)
    dy = (synth.rng(3).standard_normal((T, B, 2 * H)) * batch.mask[..., None]).astype(np.float32)
    theta = oracle.pack_params(params, L, D, H, 0)
    got = Stack(L, D, H, 0, T, B).step(theta, batch, dy_top=dy)
    ref = oracle.blstm_step(theta, batch.x, batch.mask, L, H, 0, dy_top=dy)
    errs = grad_errors(got["grad"], ref["grad"], L, D, H, 0)
    assert max(errs.values()) < GRAD_TOL, errs


def test_sgd_update_matches_definition():
    n = 1000003
    th = torch.randn(n, device=dev())
    gr = torch.randn(n, device=dev())
    exp = (th.double() - 0.01 * gr.double()).float()
    blstm.sgd_update(th, gr, 0.01, zero_grad=True)
    torch.cuda.synchronize()
    assert torch.allclose(th, exp, rtol=0, atol=1e-6)
    assert torch.all(gr == 0)
