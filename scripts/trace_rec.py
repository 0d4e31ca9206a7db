"""Per-step phase timing of the persistent recurrence kernels (debug trace hook).

Runs training steps of a config (default C3) with the library's trace hook on (library built
with `python paper_1608_00895_b200/csrc/build.py --trace --force`) and prints the median
duration of each phase of one time step of CTA 0 / thread 0, from the SM cycle counter
(clock64), converted to ns at the SM clock given by --mhz.  Trace slot k of step s is written
at the point marked TRACE(k) in lstm_rec.cu.
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1608_00895_b200 import blstm, synth  # noqa: E402
from paper_1608_00895_b200.train import StackTrainer  # noqa: E402

SLOTS = 16
# (slot sequence in program order, label of the phase ending at that slot)
FWD = [(0, None), (11, "wait own half of h"), (1, "wait partner relay"), (2, "MMA issue"), (12, "prev-step HBM stores"),
       (13, "Z wait + mask ballot"), (3, "MMA wait"),
       (8, "TMEM ld"), (9, "gate activations"), (10, "cell update + staging"), (7, "proxy fence"),
       (4, "bulk_wait + __syncthreads"), (5, "send h + arm"), (6, "Z prefetch")]
BWD = [(0, None), (1, "issue next-step loads"), (2, "wait P + gather"), (8, "wait inputs + smem reads"), (9, "dA math + smem"),
       (3, "fences + __syncthreads"), (12, "wait partner's dA half"), (13, "wait partner's B complete"),
       (10, "MMA issue + dA stores"), (4, "MMA wait"),
       (11, "TMEM ld"), (6, "P staging"), (7, "bulk_wait + __syncthreads"), (5, "send P + loads")]
# the persistent forward of the step-launched path (rec_step.cu, BLSTM_STEP_PERSIST=1)
PFWD = [(0, None), (1, "Z loads issued"), (2, "grid barrier wait"), (3, "TMA issue"), (4, "MMA wait"),
        (5, "TMEM ld + send"), (6, "cluster sync"), (7, "gate math + stores"), (8, "__syncthreads"), (9, "arrive")]
# the persistent BPTT of the step path (rec_step.cu step_bwd_persist_kernel), CTA 0 thread 0 (the TMA lane)
PBWD = [(0, None), (1, "state loads issued"), (2, "counter wait"), (3, "TMA issue"), (4, "MMA wait"),
        (5, "TMEM ld + sends"), (6, "recv wait"), (7, "dh sum + arrive"), (8, "gate math + dA stores"),
        (9, "__syncthreads")]


def report(name, tr, seq):
    step = np.diff(tr[:, 0])
    print(f"{name}: median step {np.median(step):.0f} ns, mean {np.mean(step):.0f}, p90 {np.percentile(step, 90):.0f}, "
          f"max {np.max(step):.0f}, total {np.sum(step) / 1e3:.1f} us")
    for (a, _), (b, label) in zip(seq[:-1], seq[1:]):
        d = tr[1:, b] - tr[1:, a]
        print(f"  {label:28s} {np.median(d):8.0f} ns  (mean {np.mean(d):6.0f})")
    last = seq[-1][0]
    d = tr[1:, 0] - tr[:-1, last]
    print(f"  {'(to next step)':28s} {np.median(d):8.0f} ns")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--mhz", type=float, default=1965.0)
    ap.add_argument("--B", type=int, default=None, help="batch override (e.g. C3 at B=40: N=16 per cluster)")
    args = ap.parse_args()
    cfg, params, batch = synth.make_workload(synth.CONFIGS[args.config], B=args.B)
    dev = torch.device("cuda:0")
    tr = StackTrainer(cfg, params, batch, dev)
    tr.step()
    tf = torch.zeros((cfg.T, SLOTS), dtype=torch.int64, device=dev)
    tb = torch.zeros((cfg.T, SLOTS), dtype=torch.int64, device=dev)
    blstm.blstm_debug_set_trace(tf, tb)
    tr.step()
    torch.cuda.synchronize()
    blstm.blstm_debug_set_trace(None, None)
    f = tf.cpu().numpy().astype(np.float64) * 1e3 / args.mhz
    b = tb.cpu().numpy().astype(np.float64) * 1e3 / args.mhz
    if cfg.H > 512 and os.environ.get("BLSTM_STEP_PERSIST") != "0":  # the step path (H beyond the cluster kernels)
        print(f"forward kernel entry -> exit (globaltimer): {(tf.cpu().numpy()[-1, 14] - tf.cpu().numpy()[0, 14]) / 1e3:.1f} us")
        print(f"forward kernel prologue (entry -> step 0): {f[0, 0] - f[0, 15]:.0f} ns; "
              f"scan (step 0 -> end of the last step): {(f[-1, 9] - f[0, 0]) / 1e3:.1f} us")
        report("forward (persistent step path)", f, PFWD)
        if os.environ.get("BLSTM_STEP_PERSIST_BWD") != "0":
            report("backward (persistent step path)", b, PBWD)  # rows in processing order (s)
        return
    report("forward", f, FWD)
    # backward rows are indexed by s descending; use processing order
    report("backward", b[::-1], BWD)


if __name__ == "__main__":
    main()
