"""NEXT-1 building blocks on the GPU: blstm_reduce_replicas (N workers' buffers on one device)
against the oracle's parameter average (oracle.c ref_dp_average), and the
SimulatedDP schedule against the DP algebra of SPEC S:517-531 (R8).
"""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from paper_1608_00895_b200 import blstm, synth  # noqa: E402
from paper_1608_00895_b200.train import DPSchedule, SimulatedDP  # noqa: E402


@pytest.mark.parametrize("n", [1, 2, 3, 8, 16])
@pytest.mark.parametrize("length", [1, 6, 4099, 1_000_003])
def test_average_matches_oracle(n, length):
    dev = torch.device("cuda:0")
    g = np.random.default_rng(n * 7 + length)
    xs = [g.normal(size=length).astype(np.float32) for _ in range(n)]
    ts = [torch.tensor(x, device=dev) for x in xs]
    blstm.blstm_reduce_replicas(ts, 1.0 / n)
    ref = oracle.dp_average(xs)
    out = [t.cpu().numpy() for t in ts]
    for o in out[1:]:
        assert np.array_equal(o, out[0])  # every replica gets the same bits
    # fp32 sum of n terms in fixed order, then one scaling: |err| <= (n + 1) u sum|x_q| / n
    bound = (n + 1) * 2.0 ** -24 * np.sum(np.abs(np.stack(xs)), axis=0) / n + 1e-30
    assert np.all(np.abs(out[0] - ref) <= bound)


def test_sum_scale_one():
    dev = torch.device("cuda:0")
    ts = [torch.full((1003,), float(r + 1), device=dev) for r in range(4)]
    blstm.blstm_reduce_replicas(ts, 1.0)
    assert torch.all(ts[2] == 10.0)


def test_rejects_aliases_and_too_many():
    dev = torch.device("cuda:0")
    t = torch.zeros(8, device=dev)
    with pytest.raises(blstm.BlstmError):
        blstm.blstm_reduce_replicas([t, t], 0.5)
    with pytest.raises(blstm.BlstmError):
        blstm.blstm_reduce_replicas([torch.zeros(8, device=dev) for _ in range(17)], 1.0)


def _echo_setup(N):
    cfg = synth.Config("ECHO", L=2, D=40, H=64, K=synth.ECHO_SYMBOLS + 1, T=40, B=16)
    params = synth.stack_params(cfg.L, cfg.D, cfg.H, cfg.K)
    batches = [[synth.echo_batch(cfg.T, cfg.B, cfg.D, 5000 + 100 * r)] for r in range(N)]
    return cfg, params, batches


def test_avg1_sgd_equals_mean_gradient_step():
    """one local SGD step per worker, then averaging (avg(K=1)), equals one SGD step with
    the mean of the workers' gradients: theta - lr (g_1 + g_2) / 2."""
    dev = torch.device("cuda:0")
    cfg, params, batches = _echo_setup(2)
    lr = 1e-3
    sim = SimulatedDP(cfg, params, batches, dev, DPSchedule("avg", 1), lr=lr)
    th0 = sim.workers[0].theta.clone()
    grads = []
    for w in sim.workers:  # the gradients each worker computes at theta_0
        gw = torch.zeros_like(w.grad)
        w._grad(w.theta, gw)
        grads.append(gw)
    sim.step()
    torch.cuda.synchronize()
    expect = th0 - lr * (grads[0] + grads[1]) / 2
    got = sim.workers[1].theta
    assert torch.equal(sim.workers[0].theta, got)
    err = (got - expect).abs().max().item()
    assert err <= 4 * 2.0 ** -24 * th0.abs().max().item() + 1e-7, err


def test_sync_equals_one_big_batch_sum():
    """R8: sync mode sums the N gradients every step (one big batch, unscaled): after one step
    every replica equals theta - lr (g_1 + g_2)."""
    dev = torch.device("cuda:0")
    cfg, params, batches = _echo_setup(2)
    lr = 1e-3
    sim = SimulatedDP(cfg, params, batches, dev, DPSchedule("sync"), lr=lr)
    th0 = sim.workers[0].theta.clone()
    grads = []
    for w in sim.workers:
        gw = torch.zeros_like(w.grad)
        w._grad(w.theta, gw)
        grads.append(gw)
    sim.step()
    torch.cuda.synchronize()
    expect = th0 - lr * (grads[0] + grads[1])
    for w in sim.workers:
        assert (w.theta - expect).abs().max().item() <= 4 * 2.0 ** -24 * th0.abs().max().item() + 1e-7
    assert torch.equal(sim.workers[0].theta, sim.workers[1].theta)


def test_avg_k_replicas_diverge_then_agree():
    dev = torch.device("cuda:0")
    cfg, params, batches = _echo_setup(3)
    sim = SimulatedDP(cfg, params, batches, dev, DPSchedule("avg", 3), lr=1e-3)
    sim.step()
    sim.step()
    torch.cuda.synchronize()
    assert not torch.equal(sim.workers[0].theta, sim.workers[1].theta)  # local steps on own data
    sim.step()  # third step: averaged
    torch.cuda.synchronize()
    assert torch.equal(sim.workers[0].theta, sim.workers[1].theta)
    assert torch.equal(sim.workers[0].theta, sim.workers[2].theta)
