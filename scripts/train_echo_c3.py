"""End-to-end training at the benchmark's scale: the C3 network shape (5 x 500 BLSTM, 40-dim
input, 81 chunks x 250 frames) trained on the learnable delayed-echo task (synth.echo_batch,
label = input symbol 3 frames earlier, V = 10 symbols + blank) with the fused training step
(blstm_stack_train_step: fwd + BPTT + update per gradient bucket), Adam.  Reports the frame error
rate and the loss per frame on a held-out batch every few steps, and the device time per step.
Evidence that the whole path trains at full size, beyond the single-step parity tests."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1608_00895_b200 import synth  # noqa: E402
from paper_1608_00895_b200.train import Evaluator, StackTrainer  # noqa: E402


def main(steps=150, every=15, lr=3e-4):
    cfg = synth.Config("C3-echo", L=5, D=40, H=500, K=synth.ECHO_SYMBOLS + 1, T=250, B=81)
    params = synth.stack_params(cfg.L, cfg.D, cfg.H, cfg.K)
    batches = [synth.echo_batch(cfg.T, cfg.B, cfg.D, 7000 + i, min_len=50) for i in range(16)]
    val = synth.echo_batch(cfg.T, cfg.B, cfg.D, 999, min_len=50)
    dev = torch.device("cuda:0")
    tr = StackTrainer(cfg, params, batches[0], dev, opt={"rule": "adam", "lr": lr, "max_norm": 0.0})
    ev = Evaluator(cfg, params, val, dev)
    out = []
    loss, ferr, nv = ev(tr.theta)
    out.append(dict(step=0, fer=ferr / nv, loss_per_frame=loss / nv))
    st = torch.cuda.current_stream()
    dev_ms = 0.0
    t0 = time.time()
    for k in range(1, steps + 1):
        tr.set_batch(batches[k % len(batches)])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        tr.step()
        e1.record(st)
        e1.synchronize()
        dev_ms += e0.elapsed_time(e1)
        if k % every == 0:
            loss, ferr, nv = ev(tr.theta)
            out.append(dict(step=k, fer=round(ferr / nv, 4), loss_per_frame=round(loss / nv, 4)))
            print(json.dumps(out[-1]), flush=True)
    print(json.dumps(dict(task="delayed echo k=3 on the C3 network shape", rule="adam", lr=lr, steps=steps,
                          valid_frames_per_step=tr.valid_frames, ms_per_step=round(dev_ms / steps, 3),
                          wall_s=round(time.time() - t0, 1), final_fer=out[-1]["fer"])))


if __name__ == "__main__":
    main()
