"""Pins of the MDLSTM oracle (oracle.c ref_mdlstm_fwd / ref_mdlstm_bwd; §4.2 P:238-245,
SPEC S:256-306, R21), each independent of the oracle's own code:

* all-zero parameters give h = 0;
* a 1 x 1 grid is one step: c = s(a_i) tanh(a_g), h = s(a_o) tanh(c), written out here;
* a one-column grid (V = 1) of the unstable cell is the 1-D LSTM of the fwd gate blocks
  [i, f_u, g, o] (the v-predecessor never exists): checked against the 1-D oracle, itself pinned
  against torch.nn.LSTM (tests/test_oracle_pins.py);
* wavefront order: a diagonal-by-diagonal evaluation written here in numpy equals the raster
  oracle to 1e-12;
* central finite differences of the loss on U=3, V=3, B=2 for both cells;
* the stable cell's boundedness |c| <= u + v + 1;
* mask extension: padding the grid with masked rows / columns leaves the image's outputs and the
  gradients unchanged;
* four directions: direction k equals the single-direction oracle on the flipped grid.
"""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle  # noqa: E402


def _params(g, D, H, scale=0.5):
    return (scale * g.standard_normal((D, 5 * H)), scale * g.standard_normal((H, 5 * H)),
            scale * g.standard_normal((H, 5 * H)), scale * g.standard_normal(5 * H))


def _sig(z):
    return 1.0 / (1.0 + np.exp(-z))


def test_zero_params_zero_output():
    g = np.random.default_rng(0)
    x = g.standard_normal((3, 4, 2, 5))
    H = 3
    z = np.zeros((5, 5 * H)), np.zeros((H, 5 * H)), np.zeros((H, 5 * H)), np.zeros(5 * H)
    for stable in (False, True):
        f = oracle.mdlstm_fwd(x, np.ones((3, 4, 2)), *z, stable)
        assert np.all(f["h"] == 0)


@pytest.mark.parametrize("stable", [False, True])
def test_single_cell_closed_form(stable):
    g = np.random.default_rng(1)
    D, H = 4, 3
    W, Ru, Rv, b = _params(g, D, H)
    x = g.standard_normal((1, 1, 1, D))
    a = x[0, 0, 0] @ W + b
    i = _sig(a[:H])
    gb = 2 if stable else 3
    ob = 3 if stable else 4
    c = i * np.tanh(a[gb * H:(gb + 1) * H])
    h = _sig(a[ob * H:(ob + 1) * H]) * np.tanh(c)
    f = oracle.mdlstm_fwd(x, np.ones((1, 1, 1)), W, Ru, Rv, b, stable)
    assert np.allclose(f["c"][0, 0, 0], c, rtol=0, atol=1e-14)
    assert np.allclose(f["h"][0, 0, 0], h, rtol=0, atol=1e-14)


def test_one_column_is_1d_lstm():
    g = np.random.default_rng(2)
    U, B, D, H = 6, 3, 4, 5
    W, Ru, Rv, b = _params(g, D, H)
    x = g.standard_normal((U, 1, B, D))
    f = oracle.mdlstm_fwd(x, np.ones((U, 1, B)), W, Ru, Rv, b, False)
    # 1-D gate blocks (i, f, g, o) = MDLSTM blocks (i, f_u, g, o)
    sel = np.concatenate([np.arange(0, H), np.arange(H, 2 * H), np.arange(3 * H, 4 * H), np.arange(4 * H, 5 * H)])
    ref = oracle.lstm_fwd(x[:, 0], np.ones((U, B), np.uint8), W[:, sel], Ru[:, sel], b[sel])
    assert np.allclose(f["h"][:, 0], ref["y"], rtol=0, atol=1e-12)
    assert np.allclose(f["c"][:, 0], ref["C"], rtol=0, atol=1e-12)


def _wavefront(x, W, Ru, Rv, b, stable):
    """Diagonal-by-diagonal evaluation (all cells with u + v = d at once), numpy, no mask."""
    U, V, B, D = x.shape
    H = Ru.shape[0]
    h = np.zeros((U + 1, V + 1, B, H)); c = np.zeros((U + 1, V + 1, B, H))  # index 0 = out of grid
    for d in range(U + V - 1):
        cells = [(u, d - u) for u in range(U) if 0 <= d - u < V]
        uu = np.array([p[0] for p in cells]); vv = np.array([p[1] for p in cells])
        a = (np.einsum("nbk,kg->nbg", x[uu, vv], W) + np.einsum("nbk,kg->nbg", h[uu, vv + 1], Ru)
             + np.einsum("nbk,kg->nbg", h[uu + 1, vv], Rv) + b)
        s = _sig(a)
        cu, cv = c[uu, vv + 1], c[uu + 1, vv]
        if stable:
            cn = s[..., H:2 * H] * (s[..., 4 * H:] * cu + (1 - s[..., 4 * H:]) * cv) + s[..., :H] * np.tanh(a[..., 2 * H:3 * H])
            hn = s[..., 3 * H:4 * H] * np.tanh(cn)
        else:
            cn = s[..., H:2 * H] * cu + s[..., 2 * H:3 * H] * cv + s[..., :H] * np.tanh(a[..., 3 * H:4 * H])
            hn = s[..., 4 * H:] * np.tanh(cn)
        c[uu + 1, vv + 1] = cn
        h[uu + 1, vv + 1] = hn
    return h[1:, 1:], c[1:, 1:]


@pytest.mark.parametrize("stable", [False, True])
def test_wavefront_equals_raster(stable):
    g = np.random.default_rng(3)
    U, V, B, D, H = 4, 5, 2, 3, 4
    W, Ru, Rv, b = _params(g, D, H)
    x = g.standard_normal((U, V, B, D))
    f = oracle.mdlstm_fwd(x, np.ones((U, V, B)), W, Ru, Rv, b, stable)
    h, c = _wavefront(x, W, Ru, Rv, b, stable)
    assert np.allclose(f["h"], h, rtol=0, atol=1e-12) and np.allclose(f["c"], c, rtol=0, atol=1e-12)


@pytest.mark.parametrize("stable", [False, True])
def test_central_fd(stable):
    g = np.random.default_rng(4)
    U, V, B, D, H = 3, 3, 2, 3, 4
    W, Ru, Rv, b = _params(g, D, H)
    x = g.standard_normal((U, V, B, D))
    mask = np.ones((U, V, B)); mask[2, 2, 1] = 0; mask[2, :, 1] = 0  # image 1: 2 x 3
    dy = g.standard_normal((U, V, B, H))

    def loss(x=x, W=W, Ru=Ru, Rv=Rv, b=b):
        return np.sum(oracle.mdlstm_fwd(x, mask, W, Ru, Rv, b, stable)["h"] * dy)
    f = oracle.mdlstm_fwd(x, mask, W, Ru, Rv, b, stable)
    an = oracle.mdlstm_bwd(x, mask, W, Ru, Rv, f, dy, stable)
    eps = 1e-5
    worst = 0.0
    for name, key, base in (("x", "dx", x), ("W", "dW", W), ("Ru", "dRu", Ru), ("Rv", "dRv", Rv), ("b", "db", b)):
        fd = np.zeros_like(base)
        it = np.nditer(base, flags=["multi_index"])
        for _ in it:
            i = it.multi_index
            p = base.copy(); p[i] += eps
            m = base.copy(); m[i] -= eps
            fd[i] = (loss(**{name: p}) - loss(**{name: m})) / (2 * eps)
        worst = max(worst, np.max(np.abs(fd - an[key]) / np.maximum(1e-7, np.abs(fd) + np.abs(an[key]))))
    assert worst <= 1e-5, worst


def test_stable_cell_bounded():
    g = np.random.default_rng(5)
    U, V, B, D, H = 7, 6, 2, 3, 4
    W, Ru, Rv, b = _params(g, D, H, scale=3.0)
    x = g.standard_normal((U, V, B, D))
    f = oracle.mdlstm_fwd(x, np.ones((U, V, B)), W, Ru, Rv, b, True)
    uu, vv = np.meshgrid(np.arange(U), np.arange(V), indexing="ij")
    assert np.all(np.abs(f["c"]) <= (uu + vv + 1)[:, :, None, None] + 1e-12)


@pytest.mark.parametrize("stable", [False, True])
def test_mask_extension(stable):
    g = np.random.default_rng(6)
    U, V, B, D, H = 3, 4, 2, 3, 4
    W, Ru, Rv, b = _params(g, D, H)
    x = g.standard_normal((U, V, B, D))
    dy = g.standard_normal((U, V, B, H))
    f = oracle.mdlstm_fwd(x, np.ones((U, V, B)), W, Ru, Rv, b, stable)
    an = oracle.mdlstm_bwd(x, np.ones((U, V, B)), W, Ru, Rv, f, dy, stable)
    xp = np.zeros((U + 2, V + 3, B, D)); xp[:U, :V] = x; xp[U:, :] = 9.0; xp[:, V:] = -7.0
    mp = np.zeros((U + 2, V + 3, B)); mp[:U, :V] = 1
    dyp = np.zeros((U + 2, V + 3, B, H)); dyp[:U, :V] = dy
    fp = oracle.mdlstm_fwd(xp, mp, W, Ru, Rv, b, stable)
    ap = oracle.mdlstm_bwd(xp, mp, W, Ru, Rv, fp, dyp, stable)
    assert np.allclose(fp["h"][:U, :V], f["h"], rtol=0, atol=1e-12)
    assert np.all(fp["h"][U:] == 0) and np.all(fp["h"][:, V:] == 0)
    for k in ("dW", "dRu", "dRv", "db"):
        assert np.allclose(ap[k], an[k], rtol=0, atol=1e-12)
    assert np.allclose(ap["dx"][:U, :V], an["dx"], rtol=0, atol=1e-12) and np.all(ap["dx"][U:] == 0)


def test_four_directions_are_flipped_runs():
    g = np.random.default_rng(7)
    U, V, B, D, H = 3, 4, 2, 3, 2
    params = [_params(g, D, H) for _ in range(4)]
    x = g.standard_normal((U, V, B, D))
    mask = np.ones((U, V, B))
    y, _ = oracle.mdlstm_multidir(x, mask, params, False)
    # direction 3 (flip both) by hand
    f = oracle.mdlstm_fwd(x[::-1, ::-1].copy(), mask, *params[3], False)
    assert np.allclose(y[..., 3 * H:], f["h"][::-1, ::-1], rtol=0, atol=1e-14)
    assert np.allclose(y[..., :H], oracle.mdlstm_fwd(x, mask, *params[0], False)["h"], rtol=0, atol=1e-14)


@pytest.mark.parametrize("stable", [False, True])
def test_multidir_bwd_central_fd(stable):
    """Pin of oracle.mdlstm_multidir_bwd (the flips of dy into each direction's frame and of dx
    back out, and the sum of dx over directions): central finite differences of
    L = sum(y * dy) through all four directions, for dx and every direction's
    (W, Ru, Rv, b), on a non-square grid with an irregular mask so that a wrong flip fails."""
    g = np.random.default_rng(8)
    U, V, B, D, H = 3, 2, 2, 2, 2
    params = [_params(g, D, H) for _ in range(4)]
    x = g.standard_normal((U, V, B, D))
    mask = np.ones((U, V, B)); mask[2, 1, 0] = 0; mask[2, :, 1] = 0; mask[1, 1, 1] = 0
    dy = g.standard_normal((U, V, B, 4 * H))

    def loss(x=x, params=params):
        y, _ = oracle.mdlstm_multidir(x, mask, params, stable)
        return np.sum(y * dy)
    _, fwds = oracle.mdlstm_multidir(x, mask, params, stable)
    dx, grads = oracle.mdlstm_multidir_bwd(x, mask, params, fwds, dy, stable)
    eps = 1e-5

    def rel(fd, an):
        return np.max(np.abs(fd - an) / np.maximum(1e-7, np.abs(fd) + np.abs(an)))
    fd = np.zeros_like(x)
    for i in np.ndindex(x.shape):
        p = x.copy(); p[i] += eps
        m = x.copy(); m[i] -= eps
        fd[i] = (loss(x=p) - loss(x=m)) / (2 * eps)
    worst = rel(fd, dx)
    assert np.any(dx != 0)
    for k in range(4):
        for q in range(4):
            base = params[k][q]
            fd = np.zeros_like(base)
            for i in np.ndindex(base.shape):
                pp = [list(t) for t in params]; pm = [list(t) for t in params]
                a = base.copy(); a[i] += eps; pp[k][q] = a
                a = base.copy(); a[i] -= eps; pm[k][q] = a
                fd[i] = (loss(params=pp) - loss(params=pm)) / (2 * eps)
            worst = max(worst, rel(fd, grads[k][q]))
    assert worst <= 1e-5, worst
