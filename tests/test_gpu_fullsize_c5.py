"""Parity at BASELINE configs[4]'s full size (C5: 4 x 1024-unit BLSTM, B = 128, T = 1000; the
step-launched recurrence of DESIGN.md §5.7), in the launch configuration bench.py --config C5 times.

The oracle cannot afford a C5 step in fp64, so (as for C3, tests/test_gpu_fullsize.py) it runs
the batch's shortest sequence alone, truncated to its 50 valid frames -- a sequence's outputs
depend only on its own valid frames (R2), and masked frames contribute nothing (R4):
  * forward: the GPU runs the full C5 batch; that sequence's outputs of every layer and
    direction are compared;
  * training step: the GPU runs the full C5 shapes with every other sequence masked out; loss and
    every gradient tensor must equal the oracle's step on the one sequence.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a GPU", allow_module_level=True)

import oracle  # noqa: E402
from paper_1608_00895_b200 import synth  # noqa: E402
from tests.gpu_util import GRAD_TOL, OUT_TOL, Stack, grad_errors, norm_rel  # noqa: E402


@pytest.fixture(scope="module")
def c5():
    cfg, params, batch = synth.make_workload(synth.CONFIGS["C5"])
    theta = oracle.pack_params(params, cfg.L, cfg.D, cfg.H, cfg.K)
    lens = batch.mask.sum(0)
    col = int(np.argmin(lens))
    n = int(lens[col])
    sub = synth.Batch(x=np.ascontiguousarray(batch.x[:n, [col]]), mask=np.ascontiguousarray(batch.mask[:n, [col]]),
                      labels=np.ascontiguousarray(batch.labels[:n, [col]]))
    ref = oracle.blstm_step(theta, sub.x, sub.mask, cfg.L, cfg.H, cfg.K, labels=sub.labels, want_states=True)
    return cfg, theta, batch, col, n, ref


def test_c5_forward_sampled_sequence(c5):
    cfg, theta, batch, col, n, ref = c5
    Y, C = Stack(cfg.L, cfg.D, cfg.H, cfg.K, cfg.T, cfg.B).forward(theta, batch)
    worst = 0.0
    for l in range(cfg.L):
        for d in range(2):
            y = Y[l][:n, [col], d * cfg.H:(d + 1) * cfg.H]
            e = max(norm_rel(y, ref["Ys"][l][..., d * cfg.H:(d + 1) * cfg.H]), norm_rel(C[l, d][:n, [col]], ref["Cs"][l, d]))
            worst = max(worst, e)
            assert e <= OUT_TOL, (l, d, e)
        assert np.all(Y[l][n:, col] == 0)  # masked frames output 0
    print(f"C5 forward, worst normwise error: {worst:.2e}")


def test_c5_training_step_masked_to_sample(c5):
    cfg, theta, batch, col, n, ref = c5
    keep = np.zeros(cfg.B, bool)
    keep[col] = True
    masked = synth.Batch(x=batch.x.copy(), mask=(batch.mask * keep[None, :]).astype(np.uint8), labels=batch.labels.copy())
    got = Stack(cfg.L, cfg.D, cfg.H, cfg.K, cfg.T, cfg.B).step(theta, masked, side_stream=True)
    assert abs(got["loss"] - ref["loss"]) / abs(ref["loss"]) <= OUT_TOL
    errs = grad_errors(got["grad"], ref["grad"], cfg.L, cfg.D, cfg.H, cfg.K)
    print("C5 masked-sample step, worst gradient rel-L2:", max(errs.values()))
    assert max(errs.values()) <= GRAD_TOL, errs
