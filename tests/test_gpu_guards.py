"""Out-of-bounds write checks of our own (compute-sanitizer is not available on the GPU pool):
every buffer the library writes -- workspace, reserve, theta / grad / optimizer state, outputs --
is allocated with a guard band of GUARD bytes after its end, filled with a fixed pattern; after the
call the guard bands must be untouched.  Covers the persistent stack step (with dropout and the
fused update rule), the step-launched recurrence, the MDLSTM layer and the update rules."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from paper_1608_00895_b200 import blstm, synth  # noqa: E402

GUARD = 1 << 20
PAT = 0x5A


class Guarded:
    """A device buffer of n elements followed by a guard band of GUARD bytes."""

    def __init__(self, n, dtype, init=None):
        dev = torch.device("cuda:0")
        esz = torch.tensor([], dtype=dtype).element_size()
        self.raw = torch.full((n * esz + GUARD,), PAT, dtype=torch.uint8, device=dev)
        self.t = self.raw[:n * esz].view(dtype)
        if init is not None:
            self.t.copy_(torch.as_tensor(init, dtype=dtype).reshape(-1))
        else:
            self.t.zero_()

    def intact(self):
        return bool(torch.all(self.raw[-GUARD:] == PAT).item())


def _check(bufs):
    torch.cuda.synchronize()
    bad = [k for k, b in bufs.items() if not b.intact()]
    assert not bad, f"guard band overwritten after: {bad}"


def _stack_case(force_step):
    if force_step:
        os.environ["BLSTM_FORCE_STEP"] = "1"
    try:
        L, D, H, K, T, B = 2, 40, 130, 17, 9, 7
        params = synth.stack_params(L, D, H, K)
        batch = synth.speech_batch(T, B, D, K, np.array([9, 8, 6, 9, 3, 2, 1]), seed=1000)
        theta = oracle.pack_params(params, L, D, H, K).astype(np.float32)
        desc = blstm.stack_desc(L, D, H, K, T, B, dropout=0.25, dropout_seed=4)
        n = blstm.blstm_param_count(desc)
        P = blstm.opt_params("adam", 1e-3, l2=1e-4)
        ns = blstm.blstm_opt_state_floats("adam", n)
        bufs = dict(theta=Guarded(n, torch.float32, theta), grad=Guarded(n, torch.float32),
                    state=Guarded(ns, torch.float32),
                    ws=Guarded(blstm.blstm_stack_workspace_bytes(desc), torch.uint8),
                    loss=Guarded(1, torch.float64), ferr=Guarded(1, torch.int32))
        dev = torch.device("cuda:0")
        x = torch.tensor(batch.x, device=dev)
        m = torch.tensor(batch.mask, device=dev)
        lab = torch.tensor(batch.labels, device=dev)
        side = torch.cuda.Stream()
        for _ in range(2):
            blstm.blstm_stack_train_step(desc, bufs["theta"].t, bufs["grad"].t, x, m, lab, None, bufs["loss"].t,
                                         bufs["ferr"].t, None, P, bufs["state"].t, bufs["ws"].t, s_side=side)
        _check(bufs)
        # forward-only view: Y, C outputs
        Y = Guarded(L * T * B * 2 * H, torch.float32)
        C = Guarded(L * 2 * T * B * H, torch.float32)
        blstm.blstm_stack_fwd(desc, bufs["theta"].t, x, m, Y.t, C.t, bufs["ws"].t)
        _check(dict(Y=Y, C=C, ws=bufs["ws"]))
    finally:
        os.environ.pop("BLSTM_FORCE_STEP", None)


def test_stack_persistent_guards():
    _stack_case(False)


def test_stack_step_mode_guards():
    _stack_case(True)


@pytest.mark.parametrize("stable", [False, True])
def test_mdlstm_guards(stable):
    U, V, B, D, H = 5, 7, 3, 6, 21
    desc = blstm.mdlstm_desc(U, V, B, D, H, stable)
    n, wsb, rsb = blstm.mdlstm_sizes(desc)
    g = np.random.default_rng(1)
    bufs = dict(ws=Guarded(wsb, torch.uint8), res=Guarded(rsb, torch.uint8),
                y=Guarded(U * V * B * 4 * H, torch.float32), dx=Guarded(U * V * B * D, torch.float32),
                grad=Guarded(n, torch.float32))
    dev = torch.device("cuda:0")
    th = torch.tensor(0.3 * g.standard_normal(n), dtype=torch.float32, device=dev)
    x = torch.tensor(g.standard_normal((U, V, B, D)), dtype=torch.float32, device=dev)
    mask = torch.ones((U, V, B), dtype=torch.uint8, device=dev)
    mask[3:, :, 1] = 0
    dy = torch.tensor(g.standard_normal((U, V, B, 4 * H)), dtype=torch.float32, device=dev)
    blstm.mdlstm_fwd(desc, th, x, mask, bufs["y"].t, bufs["res"].t, bufs["ws"].t)
    blstm.mdlstm_bwd(desc, th, x, mask, bufs["res"].t, dy, bufs["dx"].t, bufs["grad"].t, bufs["ws"].t)
    _check(bufs)


@pytest.mark.parametrize("n", [1, 7, 4099])
def test_opt_update_guards(n):
    bufs = dict(theta=Guarded(n, torch.float32, np.ones(n)), grad=Guarded(n, torch.float32, np.ones(n)),
                state=Guarded(blstm.blstm_opt_state_floats("adadelta", n), torch.float32),
                ws=Guarded(blstm.blstm_opt_workspace_bytes(n), torch.uint8))
    P = blstm.opt_params("adadelta", 1.0, max_norm=0.5)
    blstm.blstm_opt_update(P, None, bufs["theta"].t, bufs["grad"].t, bufs["state"].t, True, bufs["ws"].t)
    _check(bufs)


def _stack_grad(fill, force_step):
    if force_step:
        os.environ["BLSTM_FORCE_STEP"] = "1"
    try:
        L, D, H, K, T, B = 2, 40, 130, 17, 9, 7
        params = synth.stack_params(L, D, H, K)
        batch = synth.speech_batch(T, B, D, K, np.array([9, 8, 6, 9, 3, 2, 1]), seed=1000)
        theta = oracle.pack_params(params, L, D, H, K).astype(np.float32)
        desc = blstm.stack_desc(L, D, H, K, T, B)
        dev = torch.device("cuda:0")
        ws = torch.full((blstm.blstm_stack_workspace_bytes(desc),), fill, dtype=torch.uint8, device=dev)
        th = torch.tensor(theta, device=dev)
        grad = torch.zeros_like(th)
        loss = torch.zeros(1, dtype=torch.float64, device=dev)
        ferr = torch.zeros(1, dtype=torch.int32, device=dev)
        blstm.blstm_stack_fwd_bwd(desc, th, grad, torch.tensor(batch.x, device=dev), torch.tensor(batch.mask, device=dev),
                                  torch.tensor(batch.labels, device=dev), None, loss, ferr, None, ws,
                                  s_side=torch.cuda.Stream())
        torch.cuda.synchronize()
        return grad.cpu().numpy(), loss.item()
    finally:
        os.environ.pop("BLSTM_FORCE_STEP", None)


@pytest.mark.parametrize("force_step", [False, True])
def test_stack_reads_no_stale_workspace(force_step):
    """A workspace pre-filled with 0x00 or 0xFF (NaN in fp16 / fp32) gives the same step bit for bit:
    no kernel reads workspace bytes this call did not write."""
    g0, l0 = _stack_grad(0x00, force_step)
    g1, l1 = _stack_grad(0xFF, force_step)
    assert np.all(np.isfinite(g1)) and l0 == l1 and np.array_equal(g0, g1)


def test_mdlstm_reads_no_stale_workspace():
    U, V, B, D, H = 5, 7, 3, 6, 21
    desc = blstm.mdlstm_desc(U, V, B, D, H)
    n, wsb, rsb = blstm.mdlstm_sizes(desc)
    g = np.random.default_rng(2)
    dev = torch.device("cuda:0")
    th = torch.tensor(0.3 * g.standard_normal(n), dtype=torch.float32, device=dev)
    x = torch.tensor(g.standard_normal((U, V, B, D)), dtype=torch.float32, device=dev)
    mask = torch.ones((U, V, B), dtype=torch.uint8, device=dev)
    mask[3:, :, 1] = 0
    dy = torch.tensor(g.standard_normal((U, V, B, 4 * H)), dtype=torch.float32, device=dev)
    out = []
    for fill in (0x00, 0xFF):
        ws = torch.full((wsb,), fill, dtype=torch.uint8, device=dev)
        res = torch.full((rsb,), fill, dtype=torch.uint8, device=dev)
        y = torch.zeros((U, V, B, 4 * H), device=dev)
        dx = torch.zeros_like(x)
        grad = torch.zeros_like(th)
        blstm.mdlstm_fwd(desc, th, x, mask, y, res, ws)
        blstm.mdlstm_bwd(desc, th, x, mask, res, dy, dx, grad, ws)
        torch.cuda.synchronize()
        out.append((y.cpu(), dx.cpu(), grad.cpu()))
    for a, b in zip(*out):
        assert torch.all(torch.isfinite(b)) and torch.equal(a, b)


@pytest.mark.parametrize("force_step", [False, True])
def test_mask_entry_outside_01_is_reported(force_step):
    """blstm.h / SURVEY §8(b): a mask entry outside {0,1} -> BLSTM_ERR_ARG, detected on device and
    reported by the next call (or blstm_check_errors) once the kernel that saw it has completed."""
    if force_step:
        os.environ["BLSTM_FORCE_STEP"] = "1"
    try:
        L, D, H, K, T, B = 1, 8, 32, 5, 6, 3
        params = synth.stack_params(L, D, H, K)
        batch = synth.speech_batch(T, B, D, K, np.array([6, 4, 2]), seed=1000)
        theta = torch.tensor(oracle.pack_params(params, L, D, H, K), dtype=torch.float32, device="cuda:0")
        desc = blstm.stack_desc(L, D, H, K, T, B)
        ws = torch.empty(blstm.blstm_stack_workspace_bytes(desc), dtype=torch.uint8, device="cuda:0")
        x = torch.tensor(batch.x, device="cuda:0")
        Y = torch.zeros((L, T, B, 2 * H), device="cuda:0")
        C = torch.zeros((L, 2, T, B, H), device="cuda:0")
        good = torch.tensor(batch.mask, device="cuda:0")
        blstm.blstm_stack_fwd(desc, theta, x, good, Y, C, ws)
        torch.cuda.synchronize()
        blstm.blstm_check_errors()  # clean so far
        bad = good.clone()
        bad[1, 0] = 2
        blstm.blstm_stack_fwd(desc, theta, x, bad, Y, C, ws)  # the error is found on device ...
        torch.cuda.synchronize()
        with pytest.raises(blstm.BlstmError) as e:  # ... and reported by the next call
            blstm.blstm_stack_fwd(desc, theta, x, good, Y, C, ws)
        assert e.value.code == -1 and "outside {0,1}" in str(e.value)
        blstm.blstm_stack_fwd(desc, theta, x, good, Y, C, ws)  # reported once, then clear
        torch.cuda.synchronize()
        blstm.blstm_check_errors()
        blstm.blstm_stack_fwd(desc, theta, x, bad, Y, C, ws)
        torch.cuda.synchronize()
        with pytest.raises(blstm.BlstmError):
            blstm.blstm_check_errors()
    finally:
        os.environ.pop("BLSTM_FORCE_STEP", None)
