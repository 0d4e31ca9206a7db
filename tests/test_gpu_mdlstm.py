"""MDLSTM layer (NEXT-2; mdlstm.cu) against the oracle's four-direction MDLSTM
(oracle.c ref_mdlstm_fwd / ref_mdlstm_bwd behind oracle.mdlstm_multidir*), through the C-ABI:
outputs within the path's output tolerance (normwise 1e-3) and every gradient (dx, and W, Ru, Rv,
b of each direction) within rel-L2 1e-2, for both cells, ragged per-image rectangles and an
irregular mask, H not a multiple of the 16-unit padding, non-square grids."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from paper_1608_00895_b200 import blstm  # noqa: E402
from tests.gpu_util import GRAD_TOL, OUT_TOL, l2_rel, norm_rel  # noqa: E402


def _case(U, V, B, D, H, seed, irregular=False, scale=0.4, fbias=0.0):
    """fbias: added to the biases of both forget gates of the two-forget cell ([i, fu, fv, g, o]).
    On long grids (hundreds of anti-diagonals) the two-forget cell is only well conditioned when
    fu + fv < 1 (c(u, v) = fu c(u-1, v) + fv c(u, v-1) + ... grows like (fu + fv)^(u+v) otherwise,
    and fp32 / fp16 overflow); the stable cell is bounded (|c| <= u+v+1) at any scale."""
    g = np.random.default_rng(seed)
    scale = float(os.environ.get("MD_CASE_SCALE", scale))
    fbias = float(os.environ.get("MD_CASE_FBIAS", fbias))
    params = [(scale * g.standard_normal((D, 5 * H)), scale * g.standard_normal((H, 5 * H)),
               scale * g.standard_normal((H, 5 * H)), 0.5 * scale * g.standard_normal(5 * H)) for _ in range(4)]
    for ps in params:
        ps[3][H:3 * H] += fbias
    x = g.standard_normal((U, V, B, D)).astype(np.float32)
    mask = np.zeros((U, V, B), np.uint8)
    for b in range(B):  # top-left anchored image rectangles of varying size
        mask[:max(1, U - b), :max(1, V - 2 * b), b] = 1
    if irregular:
        mask[g.random((U, V, B)) < 0.15] = 0
    dy = (g.standard_normal((U, V, B, 4 * H)) * mask[..., None]).astype(np.float32)
    params = [tuple(p.astype(np.float32) for p in ps) for ps in params]
    theta = np.concatenate([np.concatenate([p.ravel() for p in ps]) for ps in params]).astype(np.float32)
    return params, theta, x, mask, dy


def _run(U, V, B, D, H, stable, irregular, seed=None, **kw):
    dev = torch.device("cuda:0")
    params, theta, x, mask, dy = _case(U, V, B, D, H, U * 100 + V if seed is None else seed, irregular, **kw)
    desc = blstm.mdlstm_desc(U, V, B, D, H, stable)
    n, wsb, rsb = blstm.mdlstm_sizes(desc)
    th = torch.tensor(theta, device=dev)
    xt, mt, dyt = (torch.tensor(a, device=dev) for a in (x, mask, dy))
    y = torch.zeros((U, V, B, 4 * H), device=dev)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    res = torch.empty(rsb, dtype=torch.uint8, device=dev)
    blstm.mdlstm_fwd(desc, th, xt, mt, y, res, ws)
    grad = torch.zeros_like(th)
    dx = torch.zeros_like(xt)
    blstm.mdlstm_bwd(desc, th, xt, mt, res, dyt, dx, grad, ws)
    torch.cuda.synchronize()
    return params, theta, x, mask, dy, y.cpu().numpy(), dx.cpu().numpy(), grad.cpu().numpy()


def _check(params, theta, x, mask, dy, y, dx, g, stable, tag=""):
    ref_y, fwds = oracle.mdlstm_multidir(x, mask, params, stable)
    ey = norm_rel(y, ref_y)
    assert ey < OUT_TOL, (tag, ey)
    ref_dx, ref_g = oracle.mdlstm_multidir_bwd(x, mask, params, fwds, dy, stable)
    errs = {"dx": l2_rel(dx, ref_dx)}
    P1 = theta.size // 4
    for k in range(4):
        o = k * P1
        for name, ref in zip(("W", "Ru", "Rv", "b"), ref_g[k]):
            got = g[o:o + ref.size].reshape(ref.shape)
            o += ref.size
            errs[f"{name}{k}"] = l2_rel(got, ref)
    assert max(errs.values()) < GRAD_TOL, (tag, errs)
    print(f"mdlstm parity {tag}: y {ey:.2e}, worst gradient {max(errs.values()):.2e}")
    return ey, errs


@pytest.mark.parametrize("wave", ["1", "single", "0"])
@pytest.mark.parametrize("U,V,B,D,H,stable,irregular", [
    (5, 7, 3, 6, 16, False, False),
    (6, 4, 2, 9, 5, True, False),
    (8, 9, 4, 3, 24, False, True),
    (3, 11, 2, 40, 32, True, True),
    (9, 5, 3, 7, 64, False, True),    # wavefront: 5 gate tiles, the largest Hp it takes
    (33, 6, 2, 5, 20, True, True),    # min(U, V) = 6 but U > 32: diagonals of <= 6 cells
    (4, 6, 2, 8, 100, False, True),   # 4 unit tiles in the persistent forward (141 KB of shared memory)
    (3, 4, 2, 8, 200, True, False),   # R tile beyond 200 KB: the per-diagonal forward
])
def test_mdlstm_matches_oracle(U, V, B, D, H, stable, irregular, wave, monkeypatch):
    """wave=1: the tensor-core wavefront where it applies (Hp <= 64, min(U, V) <= 32; CTA pairs for
    Hp in {32, 64}), else the CUDA-core kernels; single: the one-CTA tensor-core wavefront
    (BLSTM_MD_PAIR=0); wave=0 forces the CUDA-core kernels."""
    monkeypatch.setenv("BLSTM_MD_WAVE", "0" if wave == "0" else "1")
    monkeypatch.setenv("BLSTM_MD_PAIR", "0" if wave == "single" else "1")
    _check(*_run(U, V, B, D, H, stable, irregular), stable, f"{U}x{V} B={B} H={H} wave={wave}")


@pytest.mark.parametrize("H,stable,scale,fbias", [(64, False, 0.25, -1.5), (64, True, 0.4, 0.0), (30, False, 0.4, -2.0)])
def test_mdlstm_bench_grid(H, stable, scale, fbias):
    """The bench's handwriting-line grid (scripts/mdlstm_bench.py: 32 x 256, D = 16), two images
    (ragged rectangles + an irregular mask): 287 anti-diagonals of up to 32 cells through the
    tensor-core wavefront, every output and gradient against the fp64 oracle.  Parameters are
    well conditioned on this grid (_case: the two-forget cell with fu + fv < 1)."""
    _check(*_run(32, 256, 2, 16, H, stable, True, seed=77, scale=scale, fbias=fbias), stable, f"32x256 H={H}")


@pytest.mark.parametrize("H,stable", [(64, False), (32, True)])
def test_mdlstm_pair_close_to_single(H, stable, monkeypatch):
    """The CTA-pair wavefront (units split over a cluster of 2, h halves / partial P exchanged over
    DSMEM) and the one-CTA wavefront agree to ~fp32 rounding on the 32 x 256 grid."""
    outs = []
    for pair in ("1", "0"):
        monkeypatch.setenv("BLSTM_MD_PAIR", pair)
        outs.append(_run(32, 256, 2, 16, H, stable, True, seed=9, scale=0.25, fbias=-1.5)[5:])
    (y1, dx1, g1), (y0, dx0, g0) = outs
    assert norm_rel(y1, y0) < 2e-5, norm_rel(y1, y0)
    assert l2_rel(dx1, dx0) < 1e-4 and l2_rel(g1, g0) < 1e-4, (l2_rel(dx1, dx0), l2_rel(g1, g0))


def test_mdlstm_wave_close_to_cuda_cores(monkeypatch):
    """The tensor-core wavefront (3-term split products) and the fp32 CUDA-core kernels agree to
    ~fp32 rounding on a 32 x 40 grid."""
    outs = []
    for wave in ("1", "0"):
        monkeypatch.setenv("BLSTM_MD_WAVE", wave)
        outs.append(_run(32, 40, 3, 16, 48, False, True, seed=5, scale=0.3, fbias=-1.0)[5:])
    (y1, dx1, g1), (y0, dx0, g0) = outs
    assert norm_rel(y1, y0) < 2e-5, norm_rel(y1, y0)
    assert l2_rel(dx1, dx0) < 1e-4 and l2_rel(g1, g0) < 1e-4, (l2_rel(dx1, dx0), l2_rel(g1, g0))


def test_mdlstm_grad_accumulates_and_sizes():
    dev = torch.device("cuda:0")
    U, V, B, D, H = 4, 5, 2, 3, 8
    params, theta, x, mask, dy = _case(U, V, B, D, H, 3)
    desc = blstm.mdlstm_desc(U, V, B, D, H)
    n, wsb, rsb = blstm.mdlstm_sizes(desc)
    th = torch.tensor(theta, device=dev)
    xt, mt, dyt = (torch.tensor(a, device=dev) for a in (x, mask, dy))
    y = torch.zeros((U, V, B, 4 * H), device=dev)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    res = torch.empty(rsb, dtype=torch.uint8, device=dev)
    blstm.mdlstm_fwd(desc, th, xt, mt, y, res, ws)
    g1 = torch.zeros_like(th)
    blstm.mdlstm_bwd(desc, th, xt, mt, res, dyt, None, g1, ws)
    g2 = g1.clone()
    blstm.mdlstm_bwd(desc, th, xt, mt, res, dyt, None, g2, ws)
    torch.cuda.synchronize()
    assert torch.allclose(g2, 2 * g1, rtol=1e-6, atol=1e-7)  # += semantics, deterministic
    assert torch.all(y[mt == 0] == 0)                         # masked cells output 0
