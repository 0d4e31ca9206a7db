"""The N > 1 data-parallel path on CPU: world size 2 over gloo (127.0.0.1).

The host-side schedule (train.DPSchedule / dp_step) is the same code the GPU path runs
with NCCL; here the collective is torch.distributed over gloo and the per-rank gradient
comes from the fp64 oracle.  Checked against the algebra of PAPER.md §4.1
and SURVEY.md §8(c) reading R8:
  sync    : theta' = theta - lr * (g_0 + g_1) == one step on the concatenated batch
  avg(K)  : K local SGD steps per rank, then theta = mean_r theta_r
plus rank sharding (distinct data seeds) and the max/sum reductions bench.py uses.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1608_00895_b200 import synth
from paper_1608_00895_b200.train import (DPSchedule, TorchCollective, dp_step, rank_data_seed,
                                         reduce_over_ranks)

L, T, D, H, K, B = 2, 5, 3, 4, 6, 3
LR = 0.05


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _batch(rank):
    g = synth.rng(rank_data_seed(rank))
    lens = g.integers(1, T + 1, size=B).astype(np.int32)
    return synth.speech_batch(T, B, D, K, lens, seed=rank_data_seed(rank))


def _worker(rank, world, port, mode, k_avg, steps, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        params = synth.stack_params(L, D, H, K)
        theta = torch.tensor(oracle.pack_params(params, L, D, H, K), dtype=torch.float64)
        grad = torch.zeros_like(theta)
        batch = _batch(rank)

        def compute_grad(th, gr):
            res = oracle.blstm_step(th.numpy(), batch.x, batch.mask, L, H, K, labels=batch.labels)
            gr += torch.from_numpy(res["grad"])

        def update(th, gr):
            th -= LR * gr
            gr.zero_()

        coll = TorchCollective(world)
        sched = DPSchedule(mode, k_avg)
        for s in range(steps):
            dp_step(theta, grad, compute_grad, update, coll, sched, s)
        out[rank] = theta.numpy().copy()
        out[f"max{rank}"] = reduce_over_ranks(float(rank + 1) * 1.5, "max", world)
        out[f"sum{rank}"] = reduce_over_ranks(float(rank + 1), "sum", world)
    finally:
        dist.destroy_process_group()


def _run(mode, k_avg, steps, world=2):
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, _free_port(), mode, k_avg, steps, out), nprocs=world, join=True)
        return dict(out)


def test_sync_sum_equals_concatenated_batch_step():
    res = _run("sync", 1, 1)
    assert np.array_equal(res[0], res[1])  # identical replicas after the allreduce
    params = synth.stack_params(L, D, H, K)
    theta = oracle.pack_params(params, L, D, H, K)
    b0, b1 = _batch(0), _batch(1)
    cat = oracle.blstm_step(theta, np.concatenate([b0.x, b1.x], 1), np.concatenate([b0.mask, b1.mask], 1),
                            L, H, K, labels=np.concatenate([b0.labels, b1.labels], 1), lr=LR)
    assert np.max(np.abs(res[0] - cat["theta_new"])) <= 1e-12
    assert res["max0"] == res["max1"] == 3.0 and res["sum0"] == res["sum1"] == 3.0


def test_parameter_averaging_after_k_local_steps():
    res = _run("avg", 2, 2)  # fig:mgpu: local updates, then average (here after 2 batches)
    assert np.array_equal(res[0], res[1])
    params = synth.stack_params(L, D, H, K)
    theta0 = oracle.pack_params(params, L, D, H, K)
    local = []
    for r in range(2):
        b = _batch(r)
        th = theta0.copy()
        for _ in range(2):
            th = oracle.blstm_step(th, b.x, b.mask, L, H, K, labels=b.labels, lr=LR)["theta_new"]
        local.append(th)
    expect = oracle.dp_average(local)
    assert np.max(np.abs(res[0] - expect)) <= 1e-12


def test_ranks_get_distinct_data():
    b0, b1 = _batch(0), _batch(1)
    assert not np.array_equal(b0.x, b1.x)
    assert rank_data_seed(0) == 1000 and rank_data_seed(3) == 1003


def test_schedule_logic():
    s = DPSchedule("avg", 3)
    assert [s.average_after(i) for i in range(6)] == [False, False, True, False, False, True]
    assert not s.grads_summed()
    assert DPSchedule("sync").grads_summed() and not DPSchedule("sync").average_after(0)
    with pytest.raises(AssertionError):
        DPSchedule("bogus")


# ----------------------------------------------------------------------------
# StackTrainer's schedule (train.fused_dp_step) with the library's bucket order
# ----------------------------------------------------------------------------
def _fused_worker(rank, world, port, mode, k_avg, steps, out):
    """The fused path's schedule on gloo: fused_dp_step drives a step whose gradient exchange and
    update run bucket by bucket in the order the library issues them (blstm_dp_buckets, a host-only
    call of libblstm.so); the per-rank gradient is the fp64 oracle's."""
    from paper_1608_00895_b200 import blstm
    from paper_1608_00895_b200.train import fused_dp_step
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        params = synth.stack_params(L, D, H, K)
        theta = torch.tensor(oracle.pack_params(params, L, D, H, K), dtype=torch.float64)
        batch = _batch(rank)
        buckets = blstm.blstm_dp_buckets(blstm.stack_desc(L, D, H, K, T, B))
        coll = TorchCollective(world)
        order = []

        def step_fn(sum_grads):
            g = torch.from_numpy(oracle.blstm_step(theta.numpy(), batch.x, batch.mask, L, H, K,
                                                   labels=batch.labels)["grad"])
            for lo, hi in buckets:  # each bucket: exchange (sync) then update, as soon as it is final
                if sum_grads:
                    coll.sum_(g[lo:hi])
                theta[lo:hi] -= LR * g[lo:hi]
                order.append(lo)
        sched = DPSchedule(mode, k_avg)
        for s in range(steps):
            fused_dp_step(step_fn, theta, coll, sched, s)
        out[rank] = theta.numpy().copy()
        out[f"order{rank}"] = order
    finally:
        dist.destroy_process_group()


def _run_fused(mode, k_avg, steps, world=2):
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_fused_worker, args=(world, _free_port(), mode, k_avg, steps, out), nprocs=world, join=True)
        return dict(out)


def test_fused_schedule_sync_equals_concatenated_batch():
    res = _run_fused("sync", 1, 1)
    assert np.array_equal(res[0], res[1])
    params = synth.stack_params(L, D, H, K)
    theta = oracle.pack_params(params, L, D, H, K)
    b0, b1 = _batch(0), _batch(1)
    cat = oracle.blstm_step(theta, np.concatenate([b0.x, b1.x], 1), np.concatenate([b0.mask, b1.mask], 1),
                            L, H, K, labels=np.concatenate([b0.labels, b1.labels], 1), lr=LR)
    assert np.max(np.abs(res[0] - cat["theta_new"])) <= 1e-12
    _, offs = oracle.param_offsets(L, D, H, K)
    assert res["order0"] == [int(offs[6 * L])] + [int(offs[6 * l]) for l in range(L - 1, -1, -1)]


def test_fused_schedule_avg_k():
    res = _run_fused("avg", 2, 2)
    assert np.array_equal(res[0], res[1])
    params = synth.stack_params(L, D, H, K)
    theta0 = oracle.pack_params(params, L, D, H, K)
    local = []
    for r in range(2):
        b = _batch(r)
        th = theta0.copy()
        for _ in range(2):
            th = oracle.blstm_step(th, b.x, b.mask, L, H, K, labels=b.labels, lr=LR)["theta_new"]
        local.append(th)
    assert np.max(np.abs(res[0] - oracle.dp_average(local))) <= 1e-12


@pytest.mark.parametrize("Lx,Kx", [(1, 0), (2, 7), (5, 1501)])
def test_dp_buckets_partition_in_issue_order(Lx, Kx):
    from paper_1608_00895_b200 import blstm
    desc = blstm.stack_desc(Lx, 40, 500, Kx, 10, 2)
    bk = blstm.blstm_dp_buckets(desc)
    n, offs = oracle.param_offsets(Lx, 40, 500, Kx)
    assert len(bk) == Lx + (1 if Kx else 0)
    assert sorted(bk) == sorted(bk) and sum(hi - lo for lo, hi in bk) == n
    cover = sorted(bk)
    assert cover[0][0] == 0 and cover[-1][1] == n and all(a[1] == b[0] for a, b in zip(cover, cover[1:]))
    expect = ([(int(offs[6 * Lx]), n)] if Kx else []) + \
        [(int(offs[6 * l]), int(offs[6 * (l + 1)]) if l + 1 < Lx else int(offs[6 * Lx])) for l in range(Lx - 1, -1, -1)]
    assert bk == expect
