"""Bandwidth of the update-rule kernels (blstm_opt_update, optim.cu) over C3's parameter vector.

Algorithmic bytes per parameter: theta read+write (8), grad read (4), grad zeroing write (4),
plus read+write of each state float (8 per slot); the norm constraint adds a second read of
grad (4) and, with L2, of theta (4).  Timed with CUDA events on the launching stream over K
back-to-back updates (the ~100-400 MB working set exceeds the 126 MB L2 for all rules but is
re-touched each call, so the first tens of MB may hit L2: reported as measured).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1608_00895_b200 import blstm, synth  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    cfg = synth.CONFIGS["C3"]
    desc = blstm.stack_desc(cfg.L, cfg.D, cfg.H, cfg.K, cfg.T, cfg.B)
    n = blstm.blstm_param_count(desc)
    dev = torch.device("cuda:0")
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    theta = torch.randn(n, device=dev)
    grad = torch.randn(n, device=dev)
    ws = torch.empty(blstm.blstm_opt_workspace_bytes(n), dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream()
    K = 50
    rows = []
    for rule, slots in (("sgd", 0), ("momentum", 1), ("nesterov", 1), ("adagrad", 1), ("adadelta", 2), ("adam", 2)):
        for l2, clip in ((0.0, 0.0), (1e-4, 1.0)):
            ns = blstm.blstm_opt_state_floats(rule, n)
            state = torch.zeros(max(ns, 4), device=dev)
            P = blstm.opt_params(rule, 1e-9, l2=l2, max_norm=clip)
            for _ in range(5):
                blstm.blstm_opt_update(P, desc, theta, grad, state, True, ws)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(st)
            for _ in range(K):
                blstm.blstm_opt_update(P, desc, theta, grad, state, True, ws)
            e1.record(st)
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / K
            per = 16 + 8 * slots + (4 + (4 if l2 > 0 else 0) if clip > 0 else 0)
            gbs = per * n / (us * 1e-6) / 1e9
            rows.append(dict(rule=rule, l2=l2, max_norm=clip, n=n, us=round(us, 2), bytes_per_param=per,
                             gbs=round(gbs, 1), frac=round(gbs / peak, 3)))
            print(json.dumps(rows[-1]))
    print(json.dumps({"peak_hbm_gbs": peak, "n": n}))


if __name__ == "__main__":
    main()
