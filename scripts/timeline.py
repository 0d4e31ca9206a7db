"""Launch timeline of one overlapped training step (blstm_profile_timeline).

Runs a few warm-up steps of a config (default C3), then one step with the library's per-launch
CUDA events on, and prints every launch (stream, start, end, duration, GEMM shape) in start
order, followed by per-stream busy time and the gaps of the main stream.  Events recorded
between launches perturb the schedule slightly: read shares and ordering, not absolutes.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1608_00895_b200 import blstm, synth  # noqa: E402
from paper_1608_00895_b200.train import StackTrainer  # noqa: E402

CAT = {0: "rec_fwd(+Z)", 1: "rec_bwd", 2: "gemm", 3: "helper"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--dropout", type=float, default=0.0)
    args = ap.parse_args()
    cfg, params, batch = synth.make_workload(synth.CONFIGS[args.config])
    dev = torch.device("cuda:0")
    tr = StackTrainer(cfg, params, batch, dev, dropout=args.dropout)
    for _ in range(args.warmup):
        tr.step()
    torch.cuda.synchronize()
    blstm.blstm_profile_enable(2)
    tr.step()
    torch.cuda.synchronize()
    recs = blstm.blstm_profile_timeline()
    blstm.blstm_profile_enable(False)
    recs.sort(key=lambda r: r[2])
    print(f"{'stream':>6} {'start':>8} {'end':>8} {'dur':>7}  kind          shape")
    for cat, si, t0, t1, a, b, c in recs:
        shape = f"M={int(a)} N={int(b)} K={int(c)}" if cat == 2 else ""
        print(f"{int(si):>6} {t0:8.3f} {t1:8.3f} {t1 - t0:7.3f}  {CAT[int(cat)]:12s}  {shape}")
    end = max(r[3] for r in recs)
    print(f"\nstep span {end:.3f} ms")
    for s in sorted(set(int(r[1]) for r in recs)):
        rs = [r for r in recs if int(r[1]) == s]
        busy = sum(r[3] - r[2] for r in rs)
        bycat = {}
        for r in rs:
            bycat[CAT[int(r[0])]] = bycat.get(CAT[int(r[0])], 0.0) + r[3] - r[2]
        print(f"stream {s}: {len(rs)} launches, busy {busy:.3f} ms: " +
              ", ".join(f"{k} {v:.3f}" for k, v in sorted(bycat.items())))
    main = sorted((r for r in recs if int(r[1]) == 0), key=lambda r: r[2])
    gaps = [(b[2] - a[3], a[3]) for a, b in zip(main, main[1:]) if b[2] - a[3] > 0.005]
    print(f"main-stream gaps > 5 us: {len(gaps)}, total {sum(g for g, _ in gaps):.3f} ms")
    for g, t in sorted(gaps, reverse=True)[:10]:
        print(f"  {g:.3f} ms at {t:.3f}")


if __name__ == "__main__":
    main()
