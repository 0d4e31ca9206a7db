"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

The oracle cannot afford a whole C3 step (81 chunks x 250 frames x 5 BLSTM layers in
fp64), so (SURVEY.md §8(d) parity plan):
  * forward: the GPU runs the full C3 batch; the forward pass is independent per
    sequence, so 2 sampled chunks are compared with the oracle run on those 2 alone;
  * training step: the GPU runs the C3 shapes (B = 81, T = 250, same kernels and
    launch configuration) with all but 2 chunks masked out -- masked chunks carry
    zero state and contribute nothing (R2/R4) -- so loss and every
    gradient must equal the oracle's step on the 2 chunks.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a GPU", allow_module_level=True)

import oracle  # noqa: E402
from paper_1608_00895_b200 import synth  # noqa: E402
from tests.gpu_util import GRAD_TOL, OUT_TOL, Stack, grad_errors, norm_rel, record  # noqa: E402

SAMPLE = [5, 60]  # two chunks of the C3 batch (one full-length, one partial)


@pytest.fixture(scope="module")
def c3():
    cfg, params, batch = synth.make_workload(synth.CONFIGS["C3"])
    theta = oracle.pack_params(params, cfg.L, cfg.D, cfg.H, cfg.K)
    return cfg, theta, batch


def _sub(batch, idx):
    return synth.Batch(x=np.ascontiguousarray(batch.x[:, idx]), mask=np.ascontiguousarray(batch.mask[:, idx]),
                       labels=np.ascontiguousarray(batch.labels[:, idx]))


@pytest.mark.parametrize("precision", [0, 1], ids=["fp16", "fp16x2w"])
def test_c3_forward_sampled_chunks(c3, precision):
    cfg, theta, batch = c3
    st = Stack(cfg.L, cfg.D, cfg.H, cfg.K, cfg.T, cfg.B, precision=precision)
    Y, C = st.forward(theta, batch)
    sub = _sub(batch, SAMPLE)
    ref = oracle.blstm_step(theta, sub.x, sub.mask, cfg.L, cfg.H, cfg.K, labels=sub.labels, want_states=True)
    errs = {}
    for l in range(cfg.L):
        for d in range(2):
            y = Y[l][:, SAMPLE, d * cfg.H:(d + 1) * cfg.H]
            yr = ref["Ys"][l][..., d * cfg.H:(d + 1) * cfg.H]
            errs[f"y[{l}][{d}]"] = norm_rel(y, yr)
            errs[f"c[{l}][{d}]"] = norm_rel(C[l, d][:, SAMPLE], ref["Cs"][l, d])
    record("C3 forward, full batch, chunks %s, precision %d" % (SAMPLE, precision), errs, metric="normwise")
    worst = max(errs.values())
    print(f"C3 forward, worst normwise error over layers/directions: {worst:.2e}")
    assert worst <= OUT_TOL, errs


@pytest.mark.parametrize("precision", [0, 1], ids=["fp16", "fp16x2w"])
def test_c3_training_step_masked_to_sample(c3, precision):
    cfg, theta, batch = c3
    keep = np.zeros(cfg.B, bool)
    keep[SAMPLE] = True
    masked = synth.Batch(x=batch.x.copy(), mask=(batch.mask * keep[None, :]).astype(np.uint8),
                         labels=batch.labels.copy())
    got = Stack(cfg.L, cfg.D, cfg.H, cfg.K, cfg.T, cfg.B, precision=precision).step(theta, masked, side_stream=True)
    sub = _sub(batch, SAMPLE)
    ref = oracle.blstm_step(theta, sub.x, sub.mask, cfg.L, cfg.H, cfg.K, labels=sub.labels)
    assert abs(got["loss"] - ref["loss"]) / abs(ref["loss"]) <= OUT_TOL
    assert got["frame_errors"] == ref["frame_errors"] or abs(got["frame_errors"] - ref["frame_errors"]) <= 2
    errs = grad_errors(got["grad"], ref["grad"], cfg.L, cfg.D, cfg.H, cfg.K)
    record("C3 step masked to chunks %s, precision %d" % (SAMPLE, precision), errs, metric="rel-L2",
           loss_rel=abs(got["loss"] - ref["loss"]) / abs(ref["loss"]),
           frame_errors=[got["frame_errors"], ref["frame_errors"]])
    print("C3 masked-sample step, worst gradient rel-L2:", max(errs.values()))
    assert max(errs.values()) <= GRAD_TOL, errs
