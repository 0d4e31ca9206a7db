"""Host-side driver of the training step: device buffers, one step
(fwd + BPTT + update) through the C-ABI, and the data-parallel schedule.

Data parallelism follows PAPER.md §4.1: one process per GPU, each
with its own batches ("a user specified number of batches is assigned to each
device") and a full parameter image.  Two exchange modes
(R8):
  sync    : gradients are summed over ranks every step (one big batch; the
            paper's unscaled-gradient convention P:253-254), then SGD
  avg(K)  : each rank makes K local SGD updates, then the parameters are
            averaged (K=3 in fig:mgpu P:223-224)
The schedule logic is backend-agnostic (``Collective``): NCCL through the C-ABI
on GPUs, or torch.distributed (gloo) for the CPU tests of the N>1 path.
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np


def rank_env():
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    return rank, local, world


# ----------------------------------------------------------------------------
# DP schedule (backend-agnostic)
# ----------------------------------------------------------------------------
class Collective:
    """In-place fp32 collectives over all ranks."""

    def sum_(self, t):  # pragma: no cover - interface
        raise NotImplementedError

    def mean_(self, t):  # pragma: no cover - interface
        raise NotImplementedError


class TorchCollective(Collective):
    """torch.distributed collectives (gloo on CPU in the tests)."""

    def __init__(self, world: int):
        self.world = world

    def sum_(self, t):
        import torch.distributed as dist
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM)

    def mean_(self, t):
        import torch.distributed as dist
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            t /= self.world


class NcclCollective(Collective):
    """The library's dp_* entry points (NCCL over NVLink)."""

    def __init__(self, comm, world: int):
        self.comm, self.world = comm, world

    def sum_(self, t):
        from . import blstm
        blstm.dp_allreduce_grads(self.comm, t)

    def mean_(self, t):
        from . import blstm
        blstm.dp_average_params(self.comm, t)


@dataclass
class DPSchedule:
    mode: str = "sync"   # "sync" | "avg"
    K: int = 1           # averaging interval (avg mode)

    def __post_init__(self):
        assert self.mode in ("sync", "avg") and self.K >= 1

    def grads_summed(self) -> bool:
        return self.mode == "sync"

    def average_after(self, step_index: int) -> bool:
        """True when parameters are averaged after local step `step_index` (0-based)."""
        return self.mode == "avg" and (step_index + 1) % self.K == 0


def dp_step(theta, grad, compute_grad: Callable[[object, object], None], update: Callable[[object, object], None],
            coll: Collective, sched: DPSchedule, step_index: int):
    """One data-parallel training step on this rank.

    compute_grad(theta, grad) accumulates the local gradient into a zeroed grad;
    update(theta, grad) applies SGD and zeroes grad.
    """
    compute_grad(theta, grad)
    if sched.grads_summed():
        coll.sum_(grad)
    update(theta, grad)
    if sched.average_after(step_index):
        coll.mean_(theta)


def fused_dp_step(step_fn: Callable[[bool], None], theta, coll: Optional[Collective], sched: DPSchedule,
                  step_index: int):
    """The schedule of one rank's step with the update inside the library step
    (blstm_stack_train_step; StackTrainer's default path).

    step_fn(sum_grads) runs fwd + BPTT + update of this rank; with sum_grads the gradient is
    SUMmed over ranks inside the step, bucket by bucket in blstm_dp_buckets order, before each
    bucket's update (sync mode).  In avg(K) mode the step is local and the parameters are
    averaged after every K-th step."""
    step_fn(sched.grads_summed())
    if sched.average_after(step_index) and coll is not None:
        coll.mean_(theta)


def reduce_over_ranks(value: float, op: str, world: int, device=None) -> float:
    """max / sum of a scalar over all ranks (the bench's max-over-ranks time, total frames)."""
    if world == 1:
        return float(value)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def rank_data_seed(rank: int) -> int:
    """Each rank trains on its own batches: data seed 1000 + rank."""
    from .synth import DATA_SEED_BASE
    return DATA_SEED_BASE + rank


# ----------------------------------------------------------------------------
# CUDA stack runner
# ----------------------------------------------------------------------------
def theta_from_params(params, desc) -> np.ndarray:
    """Flatten synth.StackParams into the library's flat theta layout (fp32)."""
    from . import blstm
    n, offs = blstm.blstm_param_offsets(desc)
    th = np.zeros(n, np.float32)
    for l, (f, bw) in enumerate(params.layers):
        for d, p in enumerate((f, bw)):
            e = 6 * l + 3 * d
            for q, a in enumerate((p.W, p.R, p.b)):
                th[offs[e + q]: offs[e + q] + a.size] = a.ravel()
    if desc.K > 0:
        th[offs[6 * desc.L]: offs[6 * desc.L] + params.W_out.size] = params.W_out.ravel()
        th[offs[6 * desc.L + 1]: offs[6 * desc.L + 1] + desc.K] = params.b_out
    return th


class StackTrainer:
    """Device-resident training of one rank: theta, grad, workspace and a batch."""

    def __init__(self, cfg, params, batch, device, lr: float = 1e-5, comm=None, world: int = 1,
                 sched: Optional[DPSchedule] = None, opt: Optional[dict] = None, dropout: float = 0.0,
                 dropout_seed: int = 0, fused: bool = True, precision: int = 0):
        """opt: None = plain SGD (sgd_update); else the update rule of blstm_opt_update, e.g.
        {"rule": "adam", "lr": 1e-3, "l2": 1e-4, "max_norm": 10.0} (§4.3)."""
        import torch
        from . import blstm
        self.torch, self.blstm = torch, blstm
        self.cfg, self.dev, self.lr, self.world = cfg, device, lr, world
        # input dropout: a fresh mask seed per step (dropout_seed + step index)
        self.dropout, self.dropout_seed = dropout, dropout_seed
        self.desc = blstm.stack_desc(cfg.L, cfg.D, cfg.H, cfg.K, cfg.T, cfg.B, dropout=dropout,
                                     dropout_seed=dropout_seed, precision=precision)
        self.theta = torch.tensor(theta_from_params(params, self.desc), device=device)
        self.grad = torch.zeros_like(self.theta)
        self.ws = torch.empty(blstm.blstm_stack_workspace_bytes(self.desc), dtype=torch.uint8, device=device)
        self.loss = torch.zeros(1, dtype=torch.float64, device=device)
        self.ferr = torch.zeros(1, dtype=torch.int32, device=device)
        self.comm = comm
        # weight-gradient GEMMs overlap the next layer's BPTT on this stream (blstm_stack_fwd_bwd)
        self.side = torch.cuda.Stream(device=device)
        self.sched = sched or DPSchedule()
        self.coll = NcclCollective(comm, world) if comm is not None else None
        self.set_batch(batch)
        self.steps_done = 0
        self.opt = dict(opt) if opt is not None else None
        # fused: blstm_stack_train_step updates each gradient bucket on the side stream as soon as it
        # is final (plain SGD = rule "sgd", the same arithmetic as sgd_update); else fwd_bwd + update
        self.fused = fused
        self.opt_state, self.opt_steps = None, 0
        if self.opt is not None:
            ns = blstm.blstm_opt_state_floats(self.opt["rule"], self.theta.numel())
            self.opt_state = torch.zeros(max(ns, 4), dtype=torch.float32, device=device) if ns else None
            self.opt_ws = torch.empty(blstm.blstm_opt_workspace_bytes(self.theta.numel()), dtype=torch.uint8,
                                      device=device)

    def set_batch(self, batch):
        t = self.torch
        self.x = t.tensor(batch.x, device=self.dev)
        self.mask = t.tensor(batch.mask, device=self.dev)
        self.labels = t.tensor(batch.labels, device=self.dev) if self.cfg.K > 0 else None
        self.dy_top = t.tensor(batch.dy_top, device=self.dev) if self.cfg.K == 0 else None
        self.valid_frames = int(batch.mask.sum())

    def _grad(self, theta, grad):
        if self.dropout > 0:
            self.desc.dropout_seed = (self.dropout_seed + self.steps_done) & 0xFFFFFFFF
        # sync mode: the library allreduce-sums grad right after the local accumulation
        comm = self.comm if (self.comm is not None and self.sched.grads_summed()) else None
        self.blstm.blstm_stack_fwd_bwd(self.desc, theta, grad, self.x, self.mask, self.labels, self.dy_top,
                                       self.loss, self.ferr, comm, self.ws, s_side=self.side)

    def _update(self, theta, grad):
        if self.opt is None:
            self.blstm.sgd_update(theta, grad, self.lr, zero_grad=True)
            return
        self.opt_steps += 1
        P = self.blstm.opt_params(step=self.opt_steps, **self.opt)
        self.blstm.blstm_opt_update(P, self.desc, theta, grad, self.opt_state, True, self.opt_ws)

    def step(self):
        if self.fused:
            self._fused_step()
            self.steps_done += 1
            return

        class _NoSum(Collective):  # the sum already happened inside blstm_stack_fwd_bwd
            def __init__(s, inner): s.inner = inner
            def sum_(s, t): pass
            def mean_(s, t):
                if s.inner is not None:
                    s.inner.mean_(t)
        dp_step(self.theta, self.grad, self._grad, self._update, _NoSum(self.coll), self.sched, self.steps_done)
        self.steps_done += 1

    def _fused_step(self):
        """fused_dp_step's schedule with the update inside the library step (blstm_stack_train_step)."""
        if self.dropout > 0:
            self.desc.dropout_seed = (self.dropout_seed + self.steps_done) & 0xFFFFFFFF
        self.opt_steps += 1
        P = (self.blstm.opt_params("sgd", self.lr) if self.opt is None
             else self.blstm.opt_params(step=self.opt_steps, **self.opt))

        def step_fn(sum_grads):
            comm = self.comm if (self.comm is not None and sum_grads) else None
            self.blstm.blstm_stack_train_step(self.desc, self.theta, self.grad, self.x, self.mask, self.labels,
                                              self.dy_top, self.loss, self.ferr, comm, P, self.opt_state, self.ws,
                                              s_side=self.side)
        fused_dp_step(step_fn, self.theta, self.coll, self.sched, self.steps_done)


def dp_comm_from_torch(rank: int, world: int):
    """NCCL communicator of the library, its id broadcast over the torch process group."""
    import torch
    import torch.distributed as dist
    from . import blstm
    if world == 1:
        return None
    uid = blstm.dp_get_unique_id() if rank == 0 else bytes(128)
    t = torch.tensor(list(uid), dtype=torch.uint8, device=f"cuda:{torch.cuda.current_device()}")
    dist.broadcast(t, src=0)
    return blstm.dp_comm_init(world, rank, bytes(t.cpu().tolist()))


# ----------------------------------------------------------------------------
# N workers simulated on one GPU
# ----------------------------------------------------------------------------
class SimulatedDP:
    """N data-parallel workers on ONE device: the same schedule as dp_step, with the exchange
    done by blstm_reduce_replicas over the workers' device buffers instead of NCCL.

    sync   : every step the N local gradients are summed (R8: one big batch, unscaled), then
             every worker applies the same update (the replicas stay identical);
    avg(K) : every worker applies its own update each step; after every K-th step the
             parameters are averaged, theta_r <- (1/N) sum_q theta_q.
    Each worker trains on its own batches: batches[r] is worker r's list, cycled.
    """

    def __init__(self, cfg, params, batches, device, sched: DPSchedule, lr: float, opt: Optional[dict] = None):
        from . import blstm
        self.blstm, self.sched, self.N = blstm, sched, len(batches)
        self.batches = batches
        self.workers = [StackTrainer(cfg, params, b[0], device, lr=lr, opt=opt) for b in batches]
        self.steps_done = 0

    def step(self):
        k = self.steps_done
        for r, w in enumerate(self.workers):
            bl = self.batches[r]
            if len(bl) > 1:
                w.set_batch(bl[k % len(bl)])
        if self.sched.grads_summed():
            for w in self.workers:
                w._grad(w.theta, w.grad)
            if self.N > 1:
                self.blstm.blstm_reduce_replicas([w.grad for w in self.workers], 1.0)
            for w in self.workers:
                w._update(w.theta, w.grad)
        else:
            for w in self.workers:
                w._grad(w.theta, w.grad)
                w._update(w.theta, w.grad)
            if self.N > 1 and self.sched.average_after(k):
                self.blstm.blstm_reduce_replicas([w.theta for w in self.workers], 1.0 / self.N)
        self.steps_done += 1

    def consensus(self):
        """theta of the model the workers agree on: every replica after an averaging step (or in
        sync mode); otherwise worker 0's."""
        return self.workers[0].theta


class Evaluator:
    """Loss and frame errors of a parameter vector on a fixed batch (forward + head through
    blstm_stack_fwd_bwd into a scratch gradient)."""

    def __init__(self, cfg, params, batch, device):
        self.tr = StackTrainer(cfg, params, batch, device)

    def __call__(self, theta):
        t = self.tr
        t.theta.copy_(theta)
        t.grad.zero_()
        t._grad(t.theta, t.grad)
        t.torch.cuda.synchronize()
        return float(t.loss.item()), int(t.ferr.item()), t.valid_frames
