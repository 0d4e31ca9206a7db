"""Parity at BASELINE configs[4]'s full size (C5: 4 x 1024-unit BLSTM, B = 128, T = 1000; the
step-launched recurrence of DESIGN.md §5.7), in the launch configuration bench.py --config C5 times.

north_star: outputs and cell states within 1e-3 "over T<=1000".  The oracle cannot afford a C5
step in fp64 (128 sequences), so it runs two sequences of the batch: the LONGEST one (forced to the
full T = 1000 frames by the recipe) and the shortest one (50 frames) -- a sequence's
outputs depend only on its own valid frames (R2), and masked frames contribute nothing (R4):
  * forward: the GPU runs the full C5 batch; both sequences' y and c of every layer and direction
    are compared over all their frames (the long one over all 1000 steps of the scan);
  * training step: the GPU runs the full C5 shapes with every other sequence masked out; loss and
    every gradient tensor must equal the oracle's step on the two sequences (BPTT over 1000 steps).
Every magnitude goes to $BLSTM_PARITY_LOG (profiles/r02_parity_*.jsonl).
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


@pytest.fixture(scope="module")
def c5():
    cfg, params, batch = synth.make_workload(synth.CONFIGS["C5"])
    theta = oracle.pack_params(params, cfg.L, cfg.D, cfg.H, cfg.K)
    lens = batch.mask.sum(0)
    cols = [int(np.argmax(lens)), int(np.argmin(lens))]
    assert lens[cols[0]] == cfg.T == 1000  # the recipe forces one full-length sequence
    sub = synth.Batch(x=np.ascontiguousarray(batch.x[:, cols]), mask=np.ascontiguousarray(batch.mask[:, cols]),
                      labels=np.ascontiguousarray(batch.labels[:, cols]))
    ref = oracle.blstm_step(theta, sub.x, sub.mask, cfg.L, cfg.H, cfg.K, labels=sub.labels, want_states=True)
    return cfg, theta, batch, cols, [int(lens[c]) for c in cols], ref


@pytest.mark.parametrize("precision", [0, 1], ids=["fp16", "fp16x2w"])
def test_c5_forward_longest_and_shortest_sequence(c5, precision):
    cfg, theta, batch, cols, lens, ref = c5
    Y, C = Stack(cfg.L, cfg.D, cfg.H, cfg.K, cfg.T, cfg.B, precision=precision).forward(theta, batch)
    errs = {}
    for l in range(cfg.L):
        for d in range(2):
            for j, (col, n) in enumerate(zip(cols, lens)):
                y = Y[l][:n, [col], d * cfg.H:(d + 1) * cfg.H]
                yr = ref["Ys"][l][:n, [j], d * cfg.H:(d + 1) * cfg.H]
                errs[f"y[{l}][{d}] T={n}"] = norm_rel(y, yr)
                errs[f"c[{l}][{d}] T={n}"] = norm_rel(C[l, d][:n, [col]], ref["Cs"][l, d][:n, [j]])
            assert np.all(Y[l][lens[1]:, cols[1]] == 0)  # masked frames output 0
    record("C5 forward, full batch, sequences T=%s, precision %d" % (lens, precision), errs, metric="normwise")
    worst = max(errs.values())
    print(f"C5 forward, worst normwise error: {worst:.2e} (margin {OUT_TOL / worst:.2f}x)")
    assert worst <= OUT_TOL, errs


@pytest.mark.parametrize("precision", [0, 1], ids=["fp16", "fp16x2w"])
def test_c5_training_step_masked_to_sample(c5, precision):
    cfg, theta, batch, cols, lens, ref = c5
    keep = np.zeros(cfg.B, bool)
    keep[cols] = True
    masked = synth.Batch(x=batch.x.copy(), mask=(batch.mask * keep[None, :]).astype(np.uint8), labels=batch.labels.copy())
    got = Stack(cfg.L, cfg.D, cfg.H, cfg.K, cfg.T, cfg.B, precision=precision).step(theta, masked, side_stream=True)
    loss_rel = abs(got["loss"] - ref["loss"]) / abs(ref["loss"])
    errs = grad_errors(got["grad"], ref["grad"], cfg.L, cfg.D, cfg.H, cfg.K)
    record("C5 step masked to sequences T=%s, precision %d" % (lens, precision), errs, metric="rel-L2", loss_rel=loss_rel,
           frame_errors=[got["frame_errors"], ref["frame_errors"]])
    print("C5 masked-sample step, worst gradient rel-L2:", max(errs.values()), "loss rel", loss_rel)
    assert loss_rel <= OUT_TOL
    assert max(errs.values()) <= GRAD_TOL, errs
