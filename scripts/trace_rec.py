"""Per-step phase timing of the persistent recurrence kernels (debug trace hook).

Runs training steps of a config (default C3) with the library's trace hook on and
prints the median duration of each phase of one time step (CTA 0, thread 0).
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1608_00895_b200 import blstm, synth  # noqa: E402
from paper_1608_00895_b200.train import StackTrainer  # noqa: E402

FWD = ["wait h (DSMEM)", "MMA issue", "MMA wait", "epilogue+sync", "send h", "stores+prefetch"]
BWD = ["loads", "wait P + gather", "dA+smem+sync", "MMA (+dA stores)", "send P"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    args = ap.parse_args()
    cfg, params, batch = synth.make_workload(synth.CONFIGS[args.config])
    dev = torch.device("cuda:0")
    tr = StackTrainer(cfg, params, batch, dev)
    tr.step()
    tf = torch.zeros((cfg.T, 8), dtype=torch.int64, device=dev)
    tb = torch.zeros((cfg.T, 8), dtype=torch.int64, device=dev)
    blstm.blstm_debug_set_trace(tf, tb)
    tr.step()
    torch.cuda.synchronize()
    blstm.blstm_debug_set_trace(None, None)
    f = tf.cpu().numpy().astype(np.float64)
    b = tb.cpu().numpy().astype(np.float64)
    step_f = np.diff(f[:, 0])
    print(f"forward: median step {np.median(step_f):.0f} ns")
    for k, name in enumerate(FWD):
        d = f[:, k + 1] - f[:, k]
        print(f"  {name:16s} {np.median(d[1:]):8.0f} ns")
    # backward rows are indexed by s descending; use processing order
    bb = b[::-1]
    step_b = np.diff(bb[:, 0])
    print(f"backward: median step {np.median(step_b):.0f} ns")
    for k, name in enumerate(BWD):
        d = bb[:, k + 1] - bb[:, k]
        print(f"  {name:16s} {np.median(d[1:]):8.0f} ns")
    print("  backward send split: staging", np.median((bb[:, 6] - bb[:, 4])[1:]),
          "sync", np.median((bb[:, 7] - bb[:, 6])[1:]), "copies+loads", np.median((bb[:, 5] - bb[:, 7])[1:]))


if __name__ == "__main__":
    main()
