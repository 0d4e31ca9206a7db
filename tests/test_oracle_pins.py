"""Pins of the fp64 oracle to things other than itself (CPU only).

Each test names what fixes the expected value: a closed form or worked example
(tests/golden/, cited there), a library routine (torch.nn.LSTM in float64 on
packed sequences — an independent implementation of the same LSTM variant),
central finite differences, or an invariant the paper / mathematics imposes.
"""
import json
import os

import numpy as np
import pytest

import oracle
from paper_1608_00895_b200 import synth


def _load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        return json.load(f)


# ----------------------------------------------------------------------------
# closed forms and worked examples
# ----------------------------------------------------------------------------

def test_closed_form_single_step(golden_dir):
    """T=1, W=R=0, b=[0|0|+20|0] -> h = 0.5 tanh(0.5)."""
    g = _load(golden_dir, "closed_form_single_step.json")
    H = 3
    x = np.zeros((1, 2, 2))
    b = np.zeros(4 * H)
    b[2 * H:3 * H] = 20.0
    out = oracle.lstm_fwd(x, np.ones((1, 2), np.uint8), np.zeros((2, 4 * H)),
                          np.zeros((H, 4 * H)), b)
    assert np.allclose(out["y"], g["h"], atol=g["tol"], rtol=0)
    assert np.allclose(out["C"], g["c"], atol=g["tol"], rtol=0)


def test_zero_parameters_give_zero_state():
    """all parameters zero -> h = c = 0 at every frame."""
    rng = synth.rng(3)
    x = rng.standard_normal((5, 3, 4))
    H = 6
    out = oracle.lstm_fwd(x, np.ones((5, 3), np.uint8), np.zeros((4, 4 * H)),
                          np.zeros((H, 4 * H)), np.zeros(4 * H))
    assert np.all(out["y"] == 0) and np.all(out["C"] == 0)


def test_worked_example_w1(golden_dir):
    g = _load(golden_dir, "w1_scalar_lstm.json")
    tol = g["tol"]
    x = np.array(g["x"]).reshape(2, 1, 1)
    W = np.array(g["W"]).reshape(1, 4)
    R = np.array(g["R"]).reshape(1, 4)
    b = np.array(g["b"])
    m = np.ones((2, 1), np.uint8)
    f = oracle.lstm_fwd(x, m, W, R, b)
    assert np.allclose(f["G"].reshape(2, 4), g["forward"]["gates"], atol=tol)
    assert np.allclose(f["C"].ravel(), g["forward"]["c"], atol=tol)
    assert np.allclose(f["y"].ravel(), g["forward"]["y"], atol=tol)
    r = oracle.lstm_fwd(x, m, W, R, b, direction=-1)
    assert np.allclose(r["y"].ravel(), g["reverse"]["y"], atol=tol)
    assert np.allclose(r["C"].ravel(), g["reverse"]["c"], atol=tol)
    gr = oracle.lstm_bwd(x, m, W, R, f, np.ones((2, 1, 1)))
    e = g["grad_sum_y_forward"]
    assert np.allclose(gr["dW"].ravel(), e["dW"], atol=tol)
    assert np.allclose(gr["dR"].ravel(), e["dR"], atol=tol)
    assert np.allclose(gr["db"], e["db"], atol=tol)
    assert np.allclose(gr["dx"].ravel(), e["dx"], atol=tol)
    assert abs(gr["dh0"].item() - e["dh0"]) < tol
    assert abs(gr["dc0"].item() - e["dc0"]) < tol
    # masked batch: two copies of the sequence, lengths (2, 1)
    mb = g["masked_batch"]
    x2 = np.repeat(x, 2, axis=1)
    m2 = synth.mask_from_lengths(2, np.array(mb["lengths"]))
    f2 = oracle.lstm_fwd(x2, m2, W, R, b)
    assert np.allclose(f2["y"][:, :, 0], mb["y"], atol=tol)
    assert np.allclose(f2["hT"].ravel(), mb["hT"], atol=tol)
    assert np.allclose(f2["cT"].ravel(), mb["cT"], atol=tol)
    g2 = oracle.lstm_bwd(x2, m2, W, R, f2, np.ones((2, 2, 1)))
    assert np.allclose(g2["dx"][:, :, 0], mb["dx"], atol=tol)
    assert np.allclose(g2["dW"].ravel(), mb["dW"], atol=tol)
    # bidirectional: reverse direction of the length-1 sequence starts at its own last frame
    r2 = oracle.lstm_fwd(x2, m2, W, R, b, direction=-1)
    bi = g["bidirectional_masked"]
    for key, (t, bb) in dict(y_t0_b0=(0, 0), y_t0_b1=(0, 1), y_t1_b0=(1, 0), y_t1_b1=(1, 1)).items():
        got = [f2["y"][t, bb, 0], r2["y"][t, bb, 0]]
        assert np.allclose(got, bi[key], atol=tol), key


def test_worked_example_w2(golden_dir):
    g = _load(golden_dir, "w2_two_unit_lstm.json")
    tol = g["tol"]
    x = np.array(g["x"], float).reshape(2, 1, 2)
    W, R, b = np.array(g["W"]), np.array(g["R"]), np.array(g["b"], float)
    m = np.ones((2, 1), np.uint8)
    f = oracle.lstm_fwd(x, m, W, R, b)
    assert np.allclose(f["y"][:, 0, :], g["y"], atol=tol)
    assert np.allclose(f["C"][:, 0, :], g["c"], atol=tol)
    gr = oracle.lstm_bwd(x, m, W, R, f, np.ones((2, 1, 2)))
    e = g["grad_sum_y"]
    assert np.allclose(gr["db"], e["db"], atol=tol)
    assert np.allclose(gr["dx"][:, 0, :], e["dx"], atol=tol)
    assert np.allclose(gr["dW"], e["dW"], atol=tol)
    assert np.allclose(gr["dR"], e["dR"], atol=tol)


# ----------------------------------------------------------------------------
# library-routine pin: torch.nn.LSTM (float64) on packed sequences
# ----------------------------------------------------------------------------

def _torch_layer(case, direction):
    import torch
    from torch.nn.utils.rnn import pack_padded_sequence, pad_packed_sequence
    x = torch.tensor(case["x"], dtype=torch.float64)
    T, B, D = x.shape
    H = case["R"].shape[0]
    lens = torch.tensor(case["lengths"], dtype=torch.int64)
    if direction < 0:  # per-sequence time reversal (§5 index tensor; reading R2)
        idx = torch.stack([torch.cat([torch.arange(n - 1, -1, -1), torch.arange(n, T)])
                           for n in lens.tolist()], 1)
        x = x[idx, torch.arange(B)[None, :]]
    x = x.detach().requires_grad_(True)
    lstm = torch.nn.LSTM(D, H, dtype=torch.float64)
    with torch.no_grad():
        lstm.weight_ih_l0.copy_(torch.tensor(case["W"].T))
        lstm.weight_hh_l0.copy_(torch.tensor(case["R"].T))
        lstm.bias_ih_l0.copy_(torch.tensor(case["b"]))
        lstm.bias_hh_l0.zero_()
    h0 = torch.tensor(case["h0"], dtype=torch.float64)[None].requires_grad_(True)
    c0 = torch.tensor(case["c0"], dtype=torch.float64)[None].requires_grad_(True)
    packed = pack_padded_sequence(x, lens, enforce_sorted=False)
    out, (hT, cT) = lstm(packed, (h0, c0))
    y, _ = pad_packed_sequence(out, total_length=T)
    if direction < 0:
        y = y[idx, torch.arange(B)[None, :]]
    dy = torch.tensor(case["dy"], dtype=torch.float64) * torch.tensor(case["mask"])[..., None]
    loss = (y * dy).sum() + (hT[0] * torch.tensor(case["dhT"])).sum() + \
        (cT[0] * torch.tensor(case["dcT"])).sum()
    loss.backward()
    dx = x.grad
    if direction < 0:
        dx = torch.zeros_like(dx).index_put_((idx, torch.arange(B)[None, :].expand(T, B)), dx)
    return dict(y=y.detach().numpy(), hT=hT[0].detach().numpy(), cT=cT[0].detach().numpy(),
                dW=lstm.weight_ih_l0.grad.numpy().T, dR=lstm.weight_hh_l0.grad.numpy().T,
                db=lstm.bias_ih_l0.grad.numpy(), dx=dx.numpy(),
                dh0=h0.grad[0].numpy(), dc0=c0.grad[0].numpy())


@pytest.mark.parametrize("direction", [1, -1])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_layer_matches_torch_lstm_float64(direction, seed):
    case = synth.random_small_case(seed, T=7, B=4, D=3, H=5, lengths=np.array([7, 5, 3, 1]))
    case = {k: (v.astype(np.float64) if isinstance(v, np.ndarray) and v.dtype == np.float32 else v)
            for k, v in case.items()}
    ref = _torch_layer(case, direction)
    f = oracle.lstm_fwd(case["x"], case["mask"], case["W"], case["R"], case["b"],
                        case["h0"], case["c0"], direction)
    g = oracle.lstm_bwd(case["x"], case["mask"], case["W"], case["R"], f, case["dy"],
                        case["dhT"], case["dcT"], direction)
    tol = 1e-12
    assert np.max(np.abs(f["y"] - ref["y"])) < tol
    assert np.max(np.abs(f["hT"] - ref["hT"])) < tol
    assert np.max(np.abs(f["cT"] - ref["cT"])) < tol
    for k in ("dW", "dR", "db", "dx", "dh0", "dc0"):
        assert np.max(np.abs(g[k] - ref[k])) < tol, k


def test_stack_with_ce_head_matches_torch_float64():
    """Full L-layer BLSTM + Linear + summed CE vs torch."""
    import torch
    from torch.nn.utils.rnn import pack_padded_sequence, pad_packed_sequence
    L, T, B, D, H, K = 3, 6, 4, 3, 5, 7
    lens = np.array([6, 5, 3, 1])
    params = synth.stack_params(L, D, H, K)
    batch = synth.speech_batch(T, B, D, K, lens, seed=5)
    theta = oracle.pack_params(params, L, D, H, K)
    res = oracle.blstm_step(theta, batch.x, batch.mask, L, H, K, labels=batch.labels,
                            want_states=True)
    lstm = torch.nn.LSTM(D, H, num_layers=L, bidirectional=True, dtype=torch.float64)
    lin = torch.nn.Linear(2 * H, K, dtype=torch.float64)
    with torch.no_grad():
        for l, (f, bw) in enumerate(params.layers):
            for sfx, p in (("", f), ("_reverse", bw)):
                getattr(lstm, f"weight_ih_l{l}{sfx}").copy_(torch.tensor(p.W.T, dtype=torch.float64))
                getattr(lstm, f"weight_hh_l{l}{sfx}").copy_(torch.tensor(p.R.T, dtype=torch.float64))
                getattr(lstm, f"bias_ih_l{l}{sfx}").copy_(torch.tensor(p.b, dtype=torch.float64))
                getattr(lstm, f"bias_hh_l{l}{sfx}").zero_()
        lin.weight.copy_(torch.tensor(params.W_out.T, dtype=torch.float64))
        lin.bias.copy_(torch.tensor(params.b_out, dtype=torch.float64))
    x = torch.tensor(batch.x, dtype=torch.float64)
    packed = pack_padded_sequence(x, torch.tensor(lens), enforce_sorted=False)
    out, _ = lstm(packed)
    Y, _ = pad_packed_sequence(out, total_length=T)
    logits = lin(Y)
    lab = torch.tensor(batch.labels, dtype=torch.int64)
    ce = torch.nn.functional.cross_entropy(logits.reshape(-1, K), lab.reshape(-1), reduction="none")
    m = torch.tensor(batch.mask, dtype=torch.float64).reshape(-1)
    loss = (ce * m).sum()
    loss.backward()
    assert abs(res["loss"] - loss.item()) < 1e-12 * max(1.0, abs(loss.item()))
    fe = int(((logits.argmax(-1) != lab).double() * torch.tensor(batch.mask)).sum().item())
    assert res["frame_errors"] == fe
    assert np.max(np.abs(res["Ys"][-1] - Y.detach().numpy())) < 1e-13
    grads = oracle.unpack(res["grad"], L, D, H, K)
    for l in range(L):
        for d, sfx in ((0, ""), (1, "_reverse")):
            assert np.max(np.abs(grads[(l, d, "W")] - getattr(lstm, f"weight_ih_l{l}{sfx}").grad.numpy().T)) < 1e-12
            assert np.max(np.abs(grads[(l, d, "R")] - getattr(lstm, f"weight_hh_l{l}{sfx}").grad.numpy().T)) < 1e-12
            assert np.max(np.abs(grads[(l, d, "b")] - getattr(lstm, f"bias_ih_l{l}{sfx}").grad.numpy())) < 1e-12
    assert np.max(np.abs(grads[("head", "W")] - lin.weight.grad.numpy().T)) < 1e-12
    assert np.max(np.abs(grads[("head", "b")] - lin.bias.grad.numpy())) < 1e-12


# ----------------------------------------------------------------------------
# central finite differences (metric of SURVEY.md §8(c))
# ----------------------------------------------------------------------------

def _fd_metric(fd, an):
    return np.max(np.abs(fd - an) / np.maximum(1e-7, np.abs(fd) + np.abs(an)))


@pytest.mark.parametrize("seed", range(20))
def test_layer_gradients_central_fd(seed):
    g = synth.rng(100 + seed)
    T, B, D, H = (int(v) for v in g.integers(1, 7, size=4))
    B = min(B, 3)
    direction = 1 if seed % 2 == 0 else -1
    case = synth.random_small_case(seed, T, B, D, H)
    c = {k: (v.astype(np.float64) if isinstance(v, np.ndarray) and v.dtype == np.float32 else v)
         for k, v in case.items()}

    def loss(x=c["x"], W=c["W"], R=c["R"], b=c["b"], h0=c["h0"], c0=c["c0"]):
        f = oracle.lstm_fwd(x, c["mask"], W, R, b, h0, c0, direction)
        return (np.sum(f["y"] * c["dy"] * c["mask"][..., None]) + np.sum(f["hT"] * c["dhT"])
                + np.sum(f["cT"] * c["dcT"]))

    f = oracle.lstm_fwd(c["x"], c["mask"], c["W"], c["R"], c["b"], c["h0"], c["c0"], direction)
    an = oracle.lstm_bwd(c["x"], c["mask"], c["W"], c["R"], f, c["dy"], c["dhT"], c["dcT"], direction)
    eps = 1e-4
    worst = 0.0
    for name, grad in (("x", "dx"), ("W", "dW"), ("R", "dR"), ("b", "db"), ("h0", "dh0"), ("c0", "dc0")):
        base = c[name]
        fd = np.zeros_like(base)
        it = np.nditer(base, flags=["multi_index"])
        for _ in it:
            i = it.multi_index
            p = base.copy(); p[i] += eps
            m = base.copy(); m[i] -= eps
            fd[i] = (loss(**{name: p}) - loss(**{name: m})) / (2 * eps)
        worst = max(worst, _fd_metric(fd, an[grad]))
    assert worst <= 1e-5, worst


def test_stack_gradients_central_fd():
    """FD on the whole step's loss (stack + CE head), a sample of theta entries."""
    L, T, B, D, H, K = 2, 4, 3, 3, 3, 5
    params = synth.stack_params(L, D, H, K)
    batch = synth.speech_batch(T, B, D, K, np.array([4, 3, 2]), seed=9)
    theta = oracle.pack_params(params, L, D, H, K)
    g = synth.rng(4)
    theta = theta + 0.3 * g.standard_normal(theta.size)  # move biases / head off init
    res = oracle.blstm_step(theta, batch.x, batch.mask, L, H, K, labels=batch.labels)
    idx = g.choice(theta.size, size=60, replace=False)
    eps = 1e-4
    fd = np.zeros(len(idx))
    for q, i in enumerate(idx):
        tp = theta.copy(); tp[i] += eps
        tm = theta.copy(); tm[i] -= eps
        fd[q] = (oracle.blstm_step(tp, batch.x, batch.mask, L, H, K, labels=batch.labels)["loss"]
                 - oracle.blstm_step(tm, batch.x, batch.mask, L, H, K, labels=batch.labels)["loss"]) / (2 * eps)
    assert _fd_metric(fd, res["grad"][idx]) <= 1e-5


# ----------------------------------------------------------------------------
# invariants
# ----------------------------------------------------------------------------

def _rev(a, lengths):
    out = np.array(a, copy=True)
    for b, n in enumerate(lengths):
        out[:n, b] = a[:n, b][::-1]
    return out


def test_direction_duality():
    """reverse layer == per-sequence reverse o forward layer o reverse."""
    c = synth.random_small_case(7, T=6, B=3, D=4, H=5, lengths=np.array([6, 4, 2]))
    c = {k: (v.astype(np.float64) if isinstance(v, np.ndarray) and v.dtype == np.float32 else v)
         for k, v in c.items()}
    lens = c["lengths"]
    r = oracle.lstm_fwd(c["x"], c["mask"], c["W"], c["R"], c["b"], c["h0"], c["c0"], -1)
    f = oracle.lstm_fwd(_rev(c["x"], lens), c["mask"], c["W"], c["R"], c["b"], c["h0"], c["c0"], 1)
    assert np.max(np.abs(r["y"] - _rev(f["y"], lens))) <= 1e-12
    assert np.max(np.abs(r["hT"] - f["hT"])) <= 1e-12
    gr = oracle.lstm_bwd(c["x"], c["mask"], c["W"], c["R"], r, c["dy"], c["dhT"], c["dcT"], -1)
    gf = oracle.lstm_bwd(_rev(c["x"], lens), c["mask"], c["W"], c["R"], f, _rev(c["dy"], lens),
                         c["dhT"], c["dcT"], 1)
    for k in ("dW", "dR", "db", "dh0", "dc0"):
        assert np.max(np.abs(gr[k] - gf[k])) <= 1e-12, k
    assert np.max(np.abs(gr["dx"] - _rev(gf["dx"], lens))) <= 1e-12


def test_masked_frames_carry_state_and_emit_zero_gradient():
    """Reading R2/R4: appending masked frames with garbage x changes nothing;
    perturbing x at masked frames changes nothing."""
    L, T, B, D, H, K = 2, 5, 3, 3, 4, 6
    params = synth.stack_params(L, D, H, K)
    batch = synth.speech_batch(T, B, D, K, np.array([5, 3, 2]), seed=13)
    theta = oracle.pack_params(params, L, D, H, K)
    base = oracle.blstm_step(theta, batch.x, batch.mask, L, H, K, labels=batch.labels,
                             want_states=True, want_dx=True)
    p = 3
    g = synth.rng(5)
    x2 = np.concatenate([batch.x, 10 * g.standard_normal((p, B, D))], 0)
    m2 = np.concatenate([batch.mask, np.zeros((p, B), np.uint8)], 0)
    lab2 = np.concatenate([batch.labels, g.integers(0, K, (p, B)).astype(np.int32)], 0)
    ext = oracle.blstm_step(theta, x2, m2, L, H, K, labels=lab2, want_states=True, want_dx=True)
    assert abs(ext["loss"] - base["loss"]) <= 1e-12 * abs(base["loss"])
    assert np.max(np.abs(ext["grad"] - base["grad"])) <= 1e-12
    assert np.all(ext["Ys"][:, T:] == 0)
    assert np.max(np.abs(ext["Ys"][:, :T] - base["Ys"])) <= 1e-12
    assert np.all(ext["dX1"][T:] == 0)
    # perturb x at masked-out frames inside the original window
    x3 = batch.x.copy()
    x3[batch.mask == 0] = 7.0
    pert = oracle.blstm_step(theta, x3, batch.mask, L, H, K, labels=batch.labels)
    assert np.max(np.abs(pert["grad"] - base["grad"])) <= 1e-12


def test_masked_frame_gate_gradient_is_zero_and_state_passes():
    c = synth.random_small_case(11, T=5, B=2, D=3, H=4, lengths=np.array([5, 3]))
    c = {k: (v.astype(np.float64) if isinstance(v, np.ndarray) and v.dtype == np.float32 else v)
         for k, v in c.items()}
    f = oracle.lstm_fwd(c["x"], c["mask"], c["W"], c["R"], c["b"], c["h0"], c["c0"], 1)
    # state after the last valid frame is carried to the end of the scan
    assert np.array_equal(f["hT"][1], f["y"][2, 1])
    assert np.array_equal(f["cT"][1], f["C"][2, 1])
    assert np.all(f["y"][3:, 1] == 0)
    g = oracle.lstm_bwd(c["x"], c["mask"], c["W"], c["R"], f, c["dy"], c["dhT"], c["dcT"], 1)
    assert np.all(g["dA"][3:, 1] == 0)
    assert np.all(g["dx"][3:, 1] == 0)


def test_sum_semantics_duplicate_batch_doubles_gradients():
    """PAPER.md §4.3 P:253-254 (unscaled batch gradients)."""
    L, T, B, D, H, K = 2, 4, 2, 3, 4, 5
    params = synth.stack_params(L, D, H, K)
    batch = synth.speech_batch(T, B, D, K, np.array([4, 2]), seed=21)
    theta = oracle.pack_params(params, L, D, H, K)
    one = oracle.blstm_step(theta, batch.x, batch.mask, L, H, K, labels=batch.labels)
    two = oracle.blstm_step(theta, np.concatenate([batch.x] * 2, 1), np.concatenate([batch.mask] * 2, 1),
                            L, H, K, labels=np.concatenate([batch.labels] * 2, 1))
    assert abs(two["loss"] - 2 * one["loss"]) <= 1e-12 * abs(one["loss"])
    assert np.max(np.abs(two["grad"] - 2 * one["grad"])) <= 1e-12 * max(1.0, np.max(np.abs(one["grad"])))


def test_ce_uniform_logits():
    """uniform logits -> loss = n ln K; argmax ties -> lowest index."""
    L, T, B, D, H, K = 1, 5, 3, 3, 4, 4
    params = synth.stack_params(L, D, H, K)
    params.W_out[:] = 0.0
    params.b_out[:] = 0.0
    batch = synth.speech_batch(T, B, D, K, np.array([5, 4, 1]), seed=2)
    theta = oracle.pack_params(params, L, D, H, K)
    res = oracle.blstm_step(theta, batch.x, batch.mask, L, H, K, labels=batch.labels)
    n = int(batch.mask.sum())
    assert abs(res["loss"] - n * np.log(K)) <= 1e-12 * n
    assert res["frame_errors"] == int(((batch.labels != 0) & (batch.mask == 1)).sum())


def test_no_head_dy_top_matches_layer_backward():
    """K=0: the stack's gradient equals the per-layer oracle driven by dy_top."""
    L, T, B, D, H = 1, 5, 2, 3, 4
    params = synth.stack_params(L, D, H, 0)
    batch = synth.speech_batch(T, B, D, 0, np.array([5, 3]), seed=4)
    dy = synth.rng(8).standard_normal((T, B, 2 * H)) * batch.mask[..., None]
    theta = oracle.pack_params(params, L, D, H, 0)
    res = oracle.blstm_step(theta, batch.x, batch.mask, L, H, 0, dy_top=dy, want_dx=True)
    gr = oracle.unpack(res["grad"], L, D, H, 0)
    dx = 0
    for d, p in enumerate(params.layers[0]):
        f = oracle.lstm_fwd(batch.x, batch.mask, p.W, p.R, p.b, direction=1 - 2 * d)
        g = oracle.lstm_bwd(batch.x, batch.mask, p.W, p.R, f, dy[..., d * H:(d + 1) * H], direction=1 - 2 * d)
        assert np.max(np.abs(gr[(0, d, "W")] - g["dW"])) <= 1e-13
        assert np.max(np.abs(gr[(0, d, "R")] - g["dR"])) <= 1e-13
        dx = dx + g["dx"]
    assert np.max(np.abs(res["dX1"] - dx)) <= 1e-13


# ----------------------------------------------------------------------------
# data-parallel algebra (§4.1)
# ----------------------------------------------------------------------------

def test_dp_average_identity_and_symmetric_perturbation():
    g = synth.rng(6)
    th = g.standard_normal(1000)
    assert np.array_equal(oracle.dp_average([th]), th)
    d = g.standard_normal(1000) * 1e-3
    avg = oracle.dp_average([th + d, th - d])
    assert np.max(np.abs(avg - th)) <= 4 * np.finfo(float).eps * np.max(np.abs(th))


def test_dp_avg_k1_equals_mean_gradient_step():
    g = synth.rng(7)
    th = g.standard_normal(500)
    grads = [g.standard_normal(500) for _ in range(4)]
    lr = 0.1
    avg = oracle.dp_average([oracle.sgd(th, gr, lr) for gr in grads])
    expect = th - (lr / 4) * np.sum(grads, 0)
    assert np.max(np.abs(avg - expect)) <= 1e-14


def test_dp_sync_sum_equals_concatenated_batch():
    """Sync mode: sum of rank gradients == one step on the concatenated batch."""
    L, T, D, H, K = 2, 5, 3, 4, 6
    params = synth.stack_params(L, D, H, K)
    b1 = synth.speech_batch(T, 2, D, K, np.array([5, 3]), seed=31)
    b2 = synth.speech_batch(T, 3, D, K, np.array([4, 5, 1]), seed=32)
    theta = oracle.pack_params(params, L, D, H, K)
    r1 = oracle.blstm_step(theta, b1.x, b1.mask, L, H, K, labels=b1.labels)
    r2 = oracle.blstm_step(theta, b2.x, b2.mask, L, H, K, labels=b2.labels)
    rc = oracle.blstm_step(theta, np.concatenate([b1.x, b2.x], 1), np.concatenate([b1.mask, b2.mask], 1),
                           L, H, K, labels=np.concatenate([b1.labels, b2.labels], 1))
    assert abs(rc["loss"] - r1["loss"] - r2["loss"]) <= 1e-12 * abs(rc["loss"])
    assert np.max(np.abs(rc["grad"] - r1["grad"] - r2["grad"])) <= 1e-12 * np.max(np.abs(rc["grad"]))


def test_param_layout_counts():
    n, offs = oracle.param_offsets(5, 40, 500, 1501)
    per_dir_l0 = 40 * 2000 + 500 * 2000 + 2000
    per_dir = 1000 * 2000 + 500 * 2000 + 2000
    assert n == 2 * per_dir_l0 + 8 * per_dir + 1000 * 1501 + 1501
    assert offs[3] == per_dir_l0 and offs[6] == 2 * per_dir_l0
