"""Parity of blstm_opt_update (optim.cu) with the oracle's update rules (oracle.c ref_opt_update,
PAPER.md §4.3, R19) on seeded inputs, through the C-ABI.

Tolerance: the kernel computes in fp32 from the same fp32 theta / grad / state the oracle reads
in fp64.  Each rule is a handful of roundings per element and step, so the update agrees to
rel-L2 1e-5 (TOL, ~100x the fp32 unit roundoff u = 2^-24) of the oracle's change of theta, plus
the rounding of theta's fp32 storage itself, half an ulp per step: ||theta - theta_ref|| <=
TOL*||theta_ref - theta0|| + steps*u*||theta_ref||.  (The second term matters where the step is
tiny against theta, e.g. Adadelta's first steps ~ lr*sqrt(eps).)  State agrees to rel-L2 TOL;
the clip scale and the bias/weight split are exact decisions on both sides.
"""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from paper_1608_00895_b200 import blstm  # noqa: E402

RULES = ["sgd", "momentum", "nesterov", "adagrad", "adadelta", "adam"]
HYPER = dict(lr=0.02, mu=0.9, rho=0.95, beta1=0.9, beta2=0.999, eps=1e-6)
TOL = 1e-5


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _bias_mask(desc, n):
    _, offs = blstm.blstm_param_offsets(desc)
    m = np.zeros(n, np.uint8)
    for l in range(desc.L):
        for d in range(2):
            b0 = offs[6 * l + 3 * d + 2]
            m[b0:b0 + 4 * desc.H] = 1
    if desc.K > 0:
        m[offs[6 * desc.L + 1]:offs[6 * desc.L + 1] + desc.K] = 1
    return m


def _run(rule, n, steps, layout=None, l2=0.0, max_norm=0.0, seed=0, zero_grad=False):
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(seed)
    th0 = rng.normal(size=n).astype(np.float32)
    grads = [rng.normal(size=n).astype(np.float32) * np.float32(0.5) for _ in range(steps)]
    ns = blstm.blstm_opt_state_floats(rule, n)
    n4 = (n + 3) // 4 * 4
    theta = torch.tensor(th0, device=dev)
    state = torch.zeros(max(ns, 4), dtype=torch.float32, device=dev)
    ws = torch.empty(blstm.blstm_opt_workspace_bytes(n), dtype=torch.uint8, device=dev)
    # oracle, fp64, from the same fp32 values
    is_bias = _bias_mask(layout, n) if layout is not None else None
    th_r, s0, s1 = th0.astype(np.float64), None, None
    for k, g in enumerate(grads, start=1):
        grad = torch.tensor(g, device=dev)
        P = blstm.opt_params(rule, step=k, l2=l2, max_norm=max_norm, **HYPER)
        blstm.blstm_opt_update(P, layout, theta, grad, state if ns else None, zero_grad, ws)
        th_r, _, s0, s1 = oracle.opt_update(rule, th_r, g.astype(np.float64), s0, s1, step=k, l2=l2,
                                            max_norm=max_norm, is_bias=is_bias, **HYPER)
        if zero_grad:
            assert torch.count_nonzero(grad).item() == 0
        else:
            assert np.array_equal(grad.cpu().numpy(), g)
    torch.cuda.synchronize()
    th = theta.cpu().numpy().astype(np.float64)
    st = state.cpu().numpy().astype(np.float64)
    err = np.linalg.norm(th - th_r)
    bound = TOL * np.linalg.norm(th_r - th0) + steps * 2.0 ** -24 * np.linalg.norm(th_r)
    assert err <= bound, (rule, err, bound)
    if ns:
        assert _rel(st[:n], s0) <= TOL
        if ns > n4:
            assert _rel(st[n4:n4 + n], s1) <= TOL
    return theta


@pytest.mark.parametrize("rule", RULES)
@pytest.mark.parametrize("n", [1, 7, 4099, 300_001])
def test_rules_match_oracle(rule, n):
    _run(rule, n, steps=3, zero_grad=(n % 2 == 1))


@pytest.mark.parametrize("rule", RULES)
def test_l2_on_stack_layout_weights_only(rule):
    layout = blstm.stack_desc(2, 3, 5, 7, 4, 2)  # bias ranges of odd lengths, ragged tail
    n = blstm.blstm_param_count(layout)
    _run(rule, n, steps=3, layout=layout, l2=0.05)


@pytest.mark.parametrize("rule", ["sgd", "momentum", "adam"])
@pytest.mark.parametrize("max_norm", [1.0, 1e6])  # active / inactive constraint
def test_norm_constraint(rule, max_norm):
    layout = blstm.stack_desc(3, 40, 64, 31, 4, 2)
    n = blstm.blstm_param_count(layout)
    _run(rule, n, steps=2, layout=layout, l2=0.01, max_norm=max_norm)


def test_clipped_update_is_bitwise_reproducible():
    a = _run("adam", 1_000_003, steps=2, max_norm=5.0, seed=3).cpu()
    b = _run("adam", 1_000_003, steps=2, max_norm=5.0, seed=3).cpu()
    assert torch.equal(a, b)


def test_lr_zero_identity_on_device():
    dev = torch.device("cuda:0")
    th0 = torch.randn(1003, device=dev)
    for rule in RULES:
        theta = th0.clone()
        state = torch.zeros(max(blstm.blstm_opt_state_floats(rule, 1003), 4), device=dev)
        P = blstm.opt_params(rule, 0.0)
        blstm.blstm_opt_update(P, None, theta, torch.randn(1003, device=dev), state, True, None)
        assert torch.equal(theta, th0), rule


def test_trainer_sgd_rule_equals_sgd_update():
    """StackTrainer with opt={"rule": "sgd"} takes the same steps, bit for bit, as the default
    sgd_update path (both theta -= lr*g in fp32)."""
    from paper_1608_00895_b200 import synth
    from paper_1608_00895_b200.train import StackTrainer
    cfg, params, batch = synth.make_workload(synth.CONFIGS["C2"])
    dev = torch.device("cuda:0")
    a = StackTrainer(cfg, params, batch, dev, lr=1e-3)
    b = StackTrainer(cfg, params, batch, dev, lr=1e-3, opt={"rule": "sgd", "lr": 1e-3})
    for _ in range(2):
        a.step()
        b.step()
    torch.cuda.synchronize()
    assert torch.equal(a.theta, b.theta)
    assert torch.count_nonzero(b.grad).item() == 0


def test_trainer_adam_with_l2_and_clip_runs():
    from paper_1608_00895_b200 import synth
    from paper_1608_00895_b200.train import StackTrainer
    cfg, params, batch = synth.make_workload(synth.CONFIGS["C3"], B=16)  # softmax-CE head: a loss
    dev = torch.device("cuda:0")
    tr = StackTrainer(cfg, params, batch, dev, opt={"rule": "adam", "lr": 1e-3, "l2": 1e-4, "max_norm": 1.0})
    th0 = tr.theta.clone()
    losses = []
    for k in range(5):
        tr.step()
        torch.cuda.synchronize()
        losses.append(float(tr.loss.item()))
        if k == 0:  # the first bias-corrected Adam step moves each entry by at most lr (+ theta's ulp)
            ulp = 2.0 ** -23 * float(th0.abs().max())
            assert float((tr.theta - th0).abs().max()) <= 1e-3 * (1 + 1e-5) + ulp
    assert all(np.isfinite(losses))
    assert losses[-1] < losses[0]  # the same batch: the loss goes down


@pytest.mark.parametrize("opt", [None, {"rule": "adam", "lr": 1e-3, "l2": 1e-4},
                                 {"rule": "momentum", "lr": 1e-5, "max_norm": 5.0}])
def test_fused_train_step_equals_separate_update(opt):
    """blstm_stack_train_step (update per gradient bucket on the side stream; with the norm
    constraint one update at the end) gives bit for bit the step of blstm_stack_fwd_bwd followed
    by blstm_opt_update / sgd_update."""
    from paper_1608_00895_b200 import synth
    from paper_1608_00895_b200.train import StackTrainer
    cfg, params, batch = synth.make_workload(synth.CONFIGS["C3"], B=16)
    dev = torch.device("cuda:0")
    a = StackTrainer(cfg, params, batch, dev, lr=1e-5, opt=opt, fused=True, dropout=0.1, dropout_seed=3)
    b = StackTrainer(cfg, params, batch, dev, lr=1e-5, opt=opt, fused=False, dropout=0.1, dropout_seed=3)
    for _ in range(3):
        a.step()
        b.step()
    torch.cuda.synchronize()
    assert torch.equal(a.theta, b.theta)
    assert torch.count_nonzero(a.grad).item() == 0
    if opt is not None and a.opt_state is not None:
        assert torch.equal(a.opt_state, b.opt_state)
