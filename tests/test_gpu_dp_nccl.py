"""The NCCL data plane on one GPU ("every dp_* entry point is executed by a green
test").  A 1-rank communicator runs the same calls as N ranks (§4.1 P:204-211;
DESIGN.md §8): dp_get_unique_id, dp_comm_init, the per-bucket allreduce inside
blstm_stack_train_step, dp_allreduce_grads, dp_average_params and dp_comm_destroy.  The sum over
one rank and the mean over one rank are the identity, so every result must equal the comm = NULL
run bit for bit."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from paper_1608_00895_b200 import blstm, synth  # noqa: E402
from paper_1608_00895_b200.train import DPSchedule, StackTrainer  # noqa: E402


@pytest.fixture(scope="module")
def comm():
    torch.cuda.set_device(0)
    c = blstm.dp_comm_init(1, 0, blstm.dp_get_unique_id())
    yield c
    torch.cuda.synchronize()
    blstm.dp_comm_destroy(c)


def test_collectives_identity(comm):
    g = torch.Generator(device="cuda").manual_seed(3)
    for n in (1, 5, 4099, 1 << 20):
        t = torch.randn(n, device="cuda", generator=g)
        ref = t.clone()
        blstm.dp_allreduce_grads(comm, t)
        blstm.dp_average_params(comm, t)
        torch.cuda.synchronize()
        assert torch.equal(t, ref)


@pytest.mark.parametrize("H,opt", [(200, None), (500, {"rule": "adam", "lr": 1e-3, "l2": 1e-4})])
def test_train_step_with_comm_equals_without(comm, H, opt):
    L, D, K, T, B = 3, 40, 31, 30, 20
    c = synth.Config("t", L=L, D=D, H=H, K=K, T=T, B=B)
    params = synth.stack_params(L, D, H, K)
    lengths = np.array([30 - (i * 5) % 27 for i in range(B)], np.int32)
    batch = synth.speech_batch(T, B, D, K, lengths, seed=1000)
    dev = torch.device("cuda:0")
    runs = []
    for use_comm in (False, True):
        tr = StackTrainer(c, params, batch, dev, lr=1e-3, comm=comm if use_comm else None, world=1,
                          sched=DPSchedule("sync"), opt=opt)
        for _ in range(2):
            tr.step()
        torch.cuda.synchronize()
        runs.append((tr.theta.clone(), tr.grad.clone(), tr.loss.clone()))
    assert torch.equal(runs[0][0], runs[1][0])
    assert torch.equal(runs[0][1], runs[1][1])
    assert torch.equal(runs[0][2], runs[1][2])


def test_avg_mode_averages_through_nccl(comm):
    L, D, H, K, T, B = 2, 40, 200, 17, 20, 9
    params = synth.stack_params(L, D, H, K)
    batch = synth.speech_batch(T, B, D, K, np.full(B, T, np.int32), seed=1001)
    c = synth.Config("t", L=L, D=D, H=H, K=K, T=T, B=B)
    dev = torch.device("cuda:0")
    a = StackTrainer(c, params, batch, dev, lr=1e-3, comm=comm, world=1, sched=DPSchedule("avg", 2))
    b = StackTrainer(c, params, batch, dev, lr=1e-3, comm=None, world=1, sched=DPSchedule("avg", 2))
    for _ in range(4):  # two averaging points on the comm run
        a.step()
        b.step()
    torch.cuda.synchronize()
    assert torch.equal(a.theta, b.theta)
