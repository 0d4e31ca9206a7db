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


def _case(U, V, B, D, H, seed, irregular=False):
    g = np.random.default_rng(seed)
    params = [(0.4 * g.standard_normal((D, 5 * H)), 0.4 * g.standard_normal((H, 5 * H)),
               0.4 * g.standard_normal((H, 5 * H)), 0.2 * g.standard_normal(5 * H)) for _ in range(4)]
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


@pytest.mark.parametrize("U,V,B,D,H,stable,irregular", [
    (5, 7, 3, 6, 16, False, False),
    (6, 4, 2, 9, 5, True, False),
    (8, 9, 4, 3, 24, False, True),
    (3, 11, 2, 40, 32, True, True),
    (4, 6, 2, 8, 100, False, True),   # 4 unit tiles in the persistent forward (141 KB of shared memory)
    (3, 4, 2, 8, 200, True, False),   # R tile beyond 200 KB: the per-diagonal forward
])
def test_mdlstm_matches_oracle(U, V, B, D, H, stable, irregular):
    dev = torch.device("cuda:0")
    params, theta, x, mask, dy = _case(U, V, B, D, H, U * 100 + V, irregular)
    desc = blstm.mdlstm_desc(U, V, B, D, H, stable)
    n, wsb, rsb = blstm.mdlstm_sizes(desc)
    assert n == theta.size
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
    ref_y, fwds = oracle.mdlstm_multidir(x, mask, params, stable)
    assert norm_rel(y.cpu().numpy(), ref_y) < OUT_TOL
    ref_dx, ref_g = oracle.mdlstm_multidir_bwd(x, mask, params, fwds, dy, stable)
    assert l2_rel(dx.cpu().numpy(), ref_dx) < GRAD_TOL
    g = grad.cpu().numpy()
    P1 = theta.size // 4
    for k in range(4):
        o = k * P1
        for name, ref in zip(("W", "Ru", "Rv", "b"), ref_g[k]):
            got = g[o:o + ref.size].reshape(ref.shape)
            o += ref.size
            assert l2_rel(got, ref) < GRAD_TOL, (k, name, l2_rel(got, ref))


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
