"""Pins of the oracle's update rules (oracle.c ref_opt_update; §4.3, DESIGN.md
reading R19).  Each check is a closed form or a hand-derived value, never the oracle's own code:

* lr = 0 leaves theta unchanged for every rule;
* Adam's first bias-corrected step is -lr*sign(g) as eps -> 0;
* Adadelta, rho = 0.95, eps = 1e-6, g = 1, first step: -sqrt(1e-6)/sqrt(0.05 + 1e-6);
* classical momentum / simplified Nesterov with a constant gradient: geometric sums of mu;
* Adagrad with a constant gradient: the t-th step is -lr*g/(sqrt(t)*|g| + eps);
* Adam with a constant gradient: every bias-corrected step is -lr*g/(|g| + eps);
* the L2 term 2*l2*theta reaches weight entries only, and the global-norm constraint rescales
  the (conditioned) gradient to norm max_norm only when it is exceeded;
* zero_grad clears the gradient buffer.
"""
import math
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402

RULES = ["sgd", "momentum", "nesterov", "adagrad", "adadelta", "adam"]


@pytest.mark.parametrize("rule", RULES)
def test_lr_zero_is_identity(rule):
    rng = np.random.default_rng(0)
    th0 = rng.normal(size=7)
    th, s0, s1 = th0, None, None
    for step in range(1, 4):
        th, _, s0, s1 = oracle.opt_update(rule, th, rng.normal(size=7), s0, s1, lr=0.0, step=step)
    assert np.array_equal(th, th0)


def test_adam_first_step_is_sign():
    g = np.array([3.0, -0.5, 1e-3, -7.0])
    th, _, _, _ = oracle.opt_update("adam", np.zeros(4), g, lr=0.01, eps=1e-14, step=1)
    np.testing.assert_allclose(th, -0.01 * np.sign(g), rtol=1e-9)


def test_adadelta_first_step_spec_value():
    th, _, _, _ = oracle.opt_update("adadelta", [0.0], [1.0], lr=1.0, rho=0.95, eps=1e-6)
    assert abs(th[0] - (-4.4721e-3)) <= 1e-7
    assert abs(th[0] - (-math.sqrt(1e-6) / math.sqrt(0.05 + 1e-6))) < 1e-15


@pytest.mark.parametrize("rule", ["momentum", "nesterov"])
def test_momentum_constant_gradient(rule):
    lr, mu, g = 0.1, 0.8, 2.0
    th, s0 = np.array([1.0]), None
    for step in range(1, 4):
        th, _, s0, _ = oracle.opt_update(rule, th, [g], s0, lr=lr, mu=mu, step=step)
    # v_t = -lr*g*(1 + mu + ... + mu^(t-1))
    v = [-lr * g * sum(mu ** k for k in range(t)) for t in (1, 2, 3)]
    if rule == "momentum":
        expect = 1.0 + sum(v)
    else:  # theta += mu*v_t - lr*g
        expect = 1.0 + sum(mu * vt - lr * g for vt in v)
    assert abs(th[0] - expect) < 1e-14
    assert abs(s0[0] - v[-1]) < 1e-14


def test_adagrad_constant_gradient():
    lr, g, eps = 0.5, -1.5, 1e-8
    th, s0 = np.array([0.0]), None
    expect = 0.0
    for t in range(1, 6):
        th, _, s0, _ = oracle.opt_update("adagrad", th, [g], s0, lr=lr, eps=eps, step=t)
        expect -= lr * g / (math.sqrt(t) * abs(g) + eps)
        assert abs(th[0] - expect) < 1e-14
    assert abs(s0[0] - 5 * g * g) < 1e-13


def test_adam_constant_gradient():
    lr, g, eps = 0.01, 0.25, 1e-8
    th, s0, s1 = np.array([0.0]), None, None
    for t in range(1, 6):
        th, _, s0, s1 = oracle.opt_update("adam", th, [g], s0, s1, lr=lr, beta1=0.9, beta2=0.999, eps=eps, step=t)
        assert abs(th[0] - (-t * lr * g / (abs(g) + eps))) < 1e-13  # m_hat = g, v_hat = g^2 exactly


def test_l2_reaches_weights_only():
    th0 = np.array([1.0, -2.0, 3.0, 0.5])
    g = np.array([0.1, 0.2, 0.3, 0.4])
    is_bias = np.array([0, 1, 0, 1])
    lr, l2 = 0.1, 0.05
    th, _, _, _ = oracle.opt_update("sgd", th0, g, lr=lr, l2=l2, is_bias=is_bias)
    expect = th0 - lr * (g + 2 * l2 * th0 * (1 - is_bias))
    np.testing.assert_allclose(th, expect, rtol=0, atol=1e-15)


def test_norm_constraint():
    g = np.array([3.0, 4.0])  # norm 5
    th, _, _, _ = oracle.opt_update("sgd", np.zeros(2), g, lr=1.0, max_norm=2.5)
    np.testing.assert_allclose(-th, g * 0.5, rtol=1e-15)  # rescaled to norm 2.5
    th, _, _, _ = oracle.opt_update("sgd", np.zeros(2), g, lr=1.0, max_norm=10.0)
    np.testing.assert_allclose(-th, g, rtol=0)            # not exceeded: unchanged


def test_zero_grad():
    _, grad, _, _ = oracle.opt_update("adam", np.ones(3), np.ones(3), lr=0.1, zero_grad=True)
    assert np.all(grad == 0.0)
    _, grad, _, _ = oracle.opt_update("adam", np.ones(3), np.ones(3), lr=0.1, zero_grad=False)
    assert np.all(grad == 1.0)


def test_sgd_rule_equals_ref_sgd():
    rng = np.random.default_rng(1)
    th0, g = rng.normal(size=9), rng.normal(size=9)
    th, _, _, _ = oracle.opt_update("sgd", th0, g, lr=0.3)
    np.testing.assert_array_equal(th, th0 - 0.3 * g)
