"""NEXT-1: convergence of the paper's data-parallel modes on a learnable
synthetic task, with N workers simulated on one B200 (train.SimulatedDP).

Task: delayed echo (synth.echo_batch, k=3): the label of frame t is the input symbol of frame
t-3, so a correct model reaches 0 frame errors.  Network: L-layer BLSTM + softmax-CE head
(the benchmark's network, smaller).  Each worker trains on its own batches (seed 5000 + 100 r
+ i); validation is a fixed held-out batch (seed 999).

Modes (R8): sync (gradients summed over the N workers every step, one big batch,
unscaled as in PAPER.md P:253-254) and avg(K) (K local updates per worker, then the parameters
are averaged; the paper's fig:mgpu uses K=3).  Reported: validation frame error
rate vs update steps; updates and worker-steps to reach a target error; device time per step.

Usage: python scripts/dp_convergence.py [--steps S] [--lr LR] [--out profiles/r01_dp_convergence]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1608_00895_b200 import synth  # noqa: E402
from paper_1608_00895_b200.train import DPSchedule, Evaluator, SimulatedDP  # noqa: E402


def run(cfg, params, val, dev, mode, N, K, steps, lr, eval_every, n_batches, opt):
    batches = [[synth.echo_batch(cfg.T, cfg.B, cfg.D, 5000 + 100 * r + i) for i in range(n_batches)]
               for r in range(N)]
    if mode == "syncmean":  # sync with lr/N: the mean-gradient step (not the paper's unscaled sum)
        lr = lr / N
        opt = None if opt is None else dict(opt, lr=opt["lr"] / N)
    sched = DPSchedule("avg", K) if mode == "avg" else DPSchedule("sync")
    sim = SimulatedDP(cfg, params, batches, dev, sched, lr=lr, opt=opt)
    ev = Evaluator(cfg, params, val, dev)
    curve = []
    loss, ferr, nv = ev(sim.consensus())
    curve.append((0, ferr / nv, loss / nv))
    st = torch.cuda.current_stream()
    dev_ms = 0.0
    for k in range(1, steps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        sim.step()
        e1.record(st)
        e1.synchronize()
        dev_ms += e0.elapsed_time(e1)
        if k % eval_every == 0:
            loss, ferr, nv = ev(sim.consensus())
            curve.append((k, ferr / nv, loss / nv))
    return curve, dev_ms / steps


def first_below(curve, thr):
    for k, fer, _ in curve:
        if fer <= thr:
            return k
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=240)
    ap.add_argument("--lr", type=float, default=2e-4)
    ap.add_argument("--rule", default="sgd")
    ap.add_argument("--mu", type=float, default=0.9)
    ap.add_argument("--max-norm", type=float, default=0.0)
    ap.add_argument("--eval-every", type=int, default=6)
    ap.add_argument("--K", type=int, default=3)
    ap.add_argument("--workers", default="1,2,4,8")
    ap.add_argument("--modes", default="sync,syncmean,avg")
    ap.add_argument("--target", type=float, default=0.05)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    cfg = synth.Config("ECHO", L=2, D=40, H=128, K=synth.ECHO_SYMBOLS + 1, T=100, B=32)
    params = synth.stack_params(cfg.L, cfg.D, cfg.H, cfg.K)
    val = synth.echo_batch(cfg.T, cfg.B, cfg.D, 999)
    dev = torch.device("cuda:0")
    opt = None if (args.rule == "sgd" and args.max_norm == 0) else \
        {"rule": args.rule, "lr": args.lr, "mu": args.mu, "max_norm": args.max_norm}
    results = []
    for mode in args.modes.split(","):
        for N in [int(n) for n in args.workers.split(",")]:
            if mode in ("avg", "syncmean") and N == 1:
                continue
            t0 = time.time()
            curve, ms = run(cfg, params, val, dev, mode, N, args.K, args.steps, args.lr, args.eval_every, 8, opt)
            hit = first_below(curve, args.target)
            name = {"sync": "sync (sum, lr)", "syncmean": "sync (sum, lr/N)"}.get(mode, f"avg(K={args.K})")
            res = dict(mode=name, N=N, curve=curve,
                       ms_per_update=ms, updates_to_target=hit,
                       worker_steps_to_target=None if hit is None else hit * N,
                       final_fer=curve[-1][1], final_loss_per_frame=curve[-1][2])
            results.append(res)
            print(json.dumps({k: v for k, v in res.items() if k != "curve"}), f"({time.time() - t0:.1f}s)", flush=True)
    meta = dict(task=f"delayed echo k={synth.ECHO_DELAY}, V={synth.ECHO_SYMBOLS}", cfg=cfg.__dict__, lr=args.lr,
                rule=args.rule, mu=args.mu, max_norm=args.max_norm, steps=args.steps, target_fer=args.target,
                note="N workers simulated on one GPU; ms_per_update is the device time of all N worker steps "
                     "run one after another plus the exchange, not a multi-GPU wall clock")
    if args.out:
        with open(args.out + ".json", "w") as f:
            json.dump(dict(meta=meta, results=results), f, indent=1)
        with open(args.out + ".md", "w") as f:
            f.write(f"# K-step parameter averaging vs sync (NEXT-1), {meta['task']}\n\n")
            f.write(f"Network L={cfg.L} H={cfg.H} K={cfg.K}, T={cfg.T}, B={cfg.B} per worker; rule {args.rule}, "
                    f"lr {args.lr}, mu {args.mu}, max_norm {args.max_norm} (gradients unscaled); validation: held-out batch, frame error rate.\n\n")
            cols = [k for k, _, _ in results[0]["curve"] if k % (args.eval_every * 5) == 0 or k == args.steps]
            f.write("| mode | N | " + " | ".join(f"FER@{k}" for k in cols) +
                    f" | updates to FER<={args.target} | worker-steps | ms/update (sim) |\n")
            f.write("|---|---|" + "---|" * len(cols) + "---|---|---|\n")
            for r in results:
                d = {k: fer for k, fer, _ in r["curve"]}
                f.write(f"| {r['mode']} | {r['N']} | " + " | ".join(f"{d[k]:.3f}" for k in cols) +
                        f" | {r['updates_to_target']} | {r['worker_steps_to_target']} | {r['ms_per_update']:.2f} |\n")
            f.write("\n" + meta["note"] + ".\n")


if __name__ == "__main__":
    main()
