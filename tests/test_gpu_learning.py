"""Multi-step learning (the parity tests check one step at a time): a small BLSTM trained on the
delayed-echo task (synth.echo_batch; label of frame t = input symbol of frame t-3, so a correct
model reaches 0 frame errors) must drive the held-out frame error well below its start, through
the fused training step on the persistent path, the step-launched path (forced) and with input
dropout, and through the separate update call.  Full-size run: scripts/train_echo_c3.py."""
import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from paper_1608_00895_b200 import synth  # noqa: E402
from paper_1608_00895_b200.train import Evaluator, StackTrainer  # noqa: E402

STEPS = 200


@pytest.mark.parametrize("force_step,dropout,fused", [(False, 0.0, True), (True, 0.0, True),
                                                      (False, 0.1, True), (False, 0.0, False)])
def test_echo_task_learns(force_step, dropout, fused):
    if force_step:
        os.environ["BLSTM_FORCE_STEP"] = "1"
    try:
        cfg = synth.Config("ECHO", L=2, D=40, H=128, K=synth.ECHO_SYMBOLS + 1, T=60, B=32)
        params = synth.stack_params(cfg.L, cfg.D, cfg.H, cfg.K)
        batches = [synth.echo_batch(cfg.T, cfg.B, cfg.D, 6000 + i) for i in range(8)]
        val = synth.echo_batch(cfg.T, cfg.B, cfg.D, 999)
        dev = torch.device("cuda:0")
        tr = StackTrainer(cfg, params, batches[0], dev, opt={"rule": "adam", "lr": 1e-3, "max_norm": 0.0},
                          dropout=dropout, dropout_seed=11, fused=fused)
        ev = Evaluator(cfg, params, val, dev)
        loss0, ferr0, nv = ev(tr.theta)
        for k in range(STEPS):
            tr.set_batch(batches[k % len(batches)])
            tr.step()
        loss1, ferr1, _ = ev(tr.theta)
        fer0, fer1 = ferr0 / nv, ferr1 / nv
        assert torch.all(torch.isfinite(tr.theta))
        assert fer0 > 0.6 and fer1 < 0.25 and loss1 < 0.5 * loss0, (fer0, fer1, loss0, loss1)
    finally:
        os.environ.pop("BLSTM_FORCE_STEP", None)
