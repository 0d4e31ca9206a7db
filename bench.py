"""Benchmark: BLSTM training frames/sec (fwd + BPTT + SGD) on N B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl cuda|reference]

One step = one full pass of the hot path over one
batch: the 5-layer 500-unit BLSTM + 1501-class CE head training step of
BASELINE.json configs[2] (81 chunks x 250 frames per GPU, §6 shape),
synthetic speech-shaped data (paper_1608_00895_b200/synth.py).  For N > 1 the
driver launches one process per GPU with torchrun; each rank trains on its own
batch (data seed 1000 + rank) and gradients are summed over NVLink with NCCL
every step (sync mode; --dp-mode avg --avg-k K for the paper's averaging).

Prints ONE JSON line (rank 0).  value = valid frames processed by all ranks /
max-over-ranks device time of exactly K steps (CUDA events, barrier + sync on
both sides).  The per-step working set (~2.3 GB) exceeds the 126 MB L2, so no
extra L2 flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_1608_00895_b200 import synth  # noqa: E402
from paper_1608_00895_b200.train import DPSchedule, rank_env  # noqa: E402

METRIC = "BLSTM train frames/sec (fwd+BPTT) at 1/2/4/8 B200; % of roofline"
UNIT = "frames/s"


def workload_desc(cfg, world):
    return {
        "workload": (f"{cfg.name}: {cfg.L}-layer BLSTM {cfg.H} units/direction, {cfg.D}-dim input, "
                     f"{cfg.K}-class softmax-CE, {cfg.B} chunks x {cfg.T} frames per GPU, fwd+BPTT+SGD"),
        "L": cfg.L, "H": cfg.H, "D": cfg.D, "K": cfg.K, "T": cfg.T, "B_per_gpu": cfg.B,
        "global_batch": cfg.B * world, "parallelism": f"dp{world}",
        "l2": "no flush: per-step working set ~2.3 GB > 126 MB L2",
    }


# ----------------------------------------------------------------------------
# algorithmic work
# ----------------------------------------------------------------------------
def alg_flops_per_frame(cfg):
    H, K = cfg.H, cfg.K
    f = 0
    for l in range(cfg.L):
        Dl = cfg.D if l == 0 else 2 * H
        f += 2 * (8 * Dl * H + 8 * Dl * H + 8 * H * H)   # Z, dW, dR per direction
        f += 2 * (8 * H * H + 8 * H * H)                 # recurrent fwd + bwd MMAs
        if l > 0:
            f += 2 * 8 * Dl * H                          # dX
    f += 12 * H * K                                      # logits, dY, dW_out
    return f


def z_flops_per_frame(cfg):
    """the input projections (a1): 2 directions x 8*D_l*H per layer"""
    return sum(2 * 8 * (cfg.D if l == 0 else 2 * cfg.H) * cfg.H for l in range(cfg.L))


def kernel_roofline(cat, total_ms, launches, cfg, V, peaks, steps):
    """achieved / peak of the dominant kernel category, in algorithmic units per launch.

    Recurrence (cat 0/1): one launch per layer (both directions): 2*V*8H^2 FLOPs and 2*V*40H
    bytes.  GEMMs (cat 2): all dense contractions of a step over all GEMM
    launches of the step; with the Z GEMM overlapped beside the forward recurrence (DESIGN.md
    5.4) its time is inside the lstm_rec_fwd scope, so its FLOPs are excluded here."""
    H = cfg.H
    per_launch_s = total_ms / max(launches, 1) / 1e3
    if cat == 2:
        fl = alg_flops_per_frame(cfg) - cfg.L * 2 * 16 * H * H
        if os.environ.get("BLSTM_OVERLAP", "1") != "0":
            fl -= z_flops_per_frame(cfg)
        a = V * fl * steps / (total_ms / 1e3) / 1e12
        return {"bound": "tensor", "achieved": a, "peak": peaks["tf"], "unit": "TFLOP/s", "frac": a / peaks["tf"],
                "note": "aggregate over the step's GEMM launches (several shapes); the weight-gradient GEMMs "
                        "run on a side stream capped at the SMs the recurrence clusters leave free (52 of 148 at "
                        "C3) and the Z GEMMs beside the forward recurrence (inside its timed scope), so this "
                        "understates the kernel: alone on the GPU the big GEMMs run at 1.2-1.25 PFLOP/s "
                        "(DESIGN.md 5.1)"}
    flops = 2 * V * 8 * H * H
    bytes_ = 2 * V * 40 * H
    a_tf = flops / per_launch_s / 1e12
    a_gb = bytes_ / per_launch_s / 1e9
    f_tf, f_gb = a_tf / peaks["tf"], a_gb / peaks["gbs"]
    if f_gb >= f_tf:
        return {"bound": "hbm", "achieved": a_gb, "peak": peaks["gbs"], "unit": "GB/s", "frac": f_gb,
                "alt": {"bound": "tensor", "achieved": a_tf, "peak": peaks["tf"], "unit": "TFLOP/s", "frac": f_tf}}
    return {"bound": "tensor", "achieved": a_tf, "peak": peaks["tf"], "unit": "TFLOP/s", "frac": f_tf,
            "alt": {"bound": "hbm", "achieved": a_gb, "peak": peaks["gbs"], "unit": "GB/s", "frac": f_gb}}


def ncu_traffic(kernel_prefix, config):
    """DRAM bytes (read + write) per launch of a kernel category, averaged over the launches of one
    `ncu --set full` capture of ONE training step of this config (scripts/ncu_step.py, summarised by
    scripts/ncu_summarize.py --config into profiles/r*_ncu_*.json), newest round first; None when no
    capture of this config exists."""
    import glob
    import re
    files = glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_*.json"))
    rnd = lambda f: int(re.findall(r"r(\d+)_", os.path.basename(f))[0])  # noqa: E731
    for f in sorted(files, key=lambda f: (rnd(f), os.path.getmtime(f)), reverse=True):
        try:
            with open(f) as fh:
                j = json.load(fh)
        except Exception:
            continue
        if j.get("config") != config:
            continue
        for rep, ks in j.get("full_captures", {}).items():
            sel = [k for k in ks if k["kernel"].startswith(kernel_prefix) and "dram_read" in k]
            if not sel:
                continue
            scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            tot = sum(k["dram_read"] * scale.get(k.get("dram_read_unit"), 1e6) +
                      k["dram_write"] * scale.get(k.get("dram_write_unit"), 1e6) for k in sel)
            return {"bytes": tot / len(sel), "launches": len(sel),
                    "source": f"{os.path.relpath(f, ROOT)} ({os.path.basename(rep)}: {len(sel)} x {kernel_prefix})"}
    return None


def gemm_shapes(cfg):
    """(M, N, K) of every dense contraction of one training step as stack_step_impl launches them,
    in the kernels' padded layouts (Hq = H rounded up to 256; Dn = D rounded up to 64
    for layer 0, 2Hq above; Kp = K rounded up to 64)."""
    rup = lambda a, b: (a + b - 1) // b * b  # noqa: E731
    Hq = rup(cfg.H, 256)
    TB = cfg.T * cfg.B
    Kp = rup(cfg.K, 64) if cfg.K else 0
    sh = []
    for l in range(cfg.L):
        Dn = rup(cfg.D, 64) if l == 0 else 2 * Hq
        sh += [(TB, 8 * Hq, Dn), (8 * Hq, Dn, TB), (4 * Hq, Hq, TB), (4 * Hq, Hq, TB)]  # Z, dW^T, dR^T x 2
        if l > 0:
            sh.append((TB, Dn, 8 * Hq))  # dX
    if cfg.K:
        sh += [(TB, cfg.K, 2 * Hq), (TB, 2 * Hq, Kp), (cfg.K, 2 * Hq, TB)]  # logits, dY_top, dW_out^T
    return sh


def gemm_alg_bytes(cfg):
    """algorithmic bytes of the step's GEMMs: fp16 A and B read once, fp32 C written once"""
    return sum(2 * (M * K + N * K) + 4 * M * N for M, N, K in gemm_shapes(cfg))


def step_floor(config):
    """the per-timestep floor terms measured by scripts/step_floor.cu + scripts/dsmem_bench.cu
    (profiles/r02_step_floor.json), or None"""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_step_floor.json")) as f:
            j = json.load(f)
        return j.get(config)
    except Exception:
        return None


def alg_bytes_per_frame(cfg):
    """sum_l 2*4*(3 D_l + 13 H) + head 4*(4H + 2K)"""
    b = sum(2 * 4 * (3 * (cfg.D if l == 0 else 2 * cfg.H) + 13 * cfg.H) for l in range(cfg.L))
    if cfg.K:
        b += 4 * (4 * cfg.H + 2 * cfg.K)
    return b


def crit_flops_per_frame(cfg):
    """dense contractions on the dependency chain: Z of every layer, dX of layers
    >= 1, and the head's logits and dY"""
    f = z_flops_per_frame(cfg) + sum(2 * 8 * 2 * cfg.H * cfg.H for l in range(1, cfg.L))
    if cfg.K:
        f += 2 * 2 * (2 * cfg.H) * cfg.K
    return f


def step_roofline(cfg, V, peaks, t_measured_ms):
    """T_roof = max(T_tc, T_hbm, T_crit), T_crit = F_crit / P_tc + N_steps * t_floor,
    t_floor = max(t_mma + t_epi + t_xchg, bytes_step / BW) per direction pair and step; roofline
    fraction = T_roof / T_measured."""
    P, BW = peaks["tf"] * 1e12, peaks["gbs"] * 1e9
    t_tc = V * alg_flops_per_frame(cfg) / P * 1e3
    t_hbm = V * alg_bytes_per_frame(cfg) / BW * 1e3
    t_gemm_crit = V * crit_flops_per_frame(cfg) / P * 1e3
    fl = step_floor(cfg.name)
    out = {"T_tc_ms": t_tc, "T_hbm_ms": t_hbm, "F_crit_over_P_tc_ms": t_gemm_crit, "T_measured_ms": t_measured_ms}
    if fl:
        bytes_step = 2 * (V / cfg.T) * 40 * cfg.H  # both directions' recurrence bytes per step
        t_hbm_step = bytes_step / BW * 1e9
        tf_ = max(fl["t_mma_ns"] + fl["t_epi_fwd_ns"] + fl["t_xchg_ns"], t_hbm_step)
        tb_ = max(fl["t_mma_ns"] + fl["t_epi_bwd_ns"] + fl["t_xchg_ns"], t_hbm_step)
        n_steps = cfg.L * cfg.T
        t_crit = t_gemm_crit + n_steps * (tf_ + tb_) / 1e6
        t_roof = max(t_tc, t_hbm, t_crit)
        out.update({"t_floor_fwd_ns": tf_, "t_floor_bwd_ns": tb_, "hbm_ns_per_step": t_hbm_step,
                    "serial_steps": 2 * n_steps, "T_crit_ms": t_crit, "T_roof_ms": t_roof,
                    "frac": t_roof / t_measured_ms, "floor_terms": fl,
                    "bound": "latency (T_crit)" if t_roof == t_crit else ("tensor" if t_roof == t_tc else "hbm")})
    else:
        t_roof = max(t_tc, t_hbm, t_gemm_crit)
        out.update({"T_roof_ms": t_roof, "frac": t_roof / t_measured_ms, "T_crit_ms": None,
                    "note": f"no measured step floor for {cfg.name}: T_roof without the serial-step term"})
    return out


def measured_peaks():
    p = {"gbs": 6549.8, "tf": 1378.5, "source": "MEASURED_PEAKS.json (hbm_gbs, bf16_tflops_sustained)"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            j = json.load(f)
        p["gbs"] = float(j["hbm_gbs"])
        p["tf"] = float(j.get("bf16_tflops_sustained", j["bf16_tflops"]))
    except Exception:
        p = {"gbs": 6650.0, "tf": 1590.0, "source": "fallback (B200_PROFILING.md)"}
    p["note"] = "fp16 dense peak taken = bf16 measured peak (nominal ratio 1)"
    return p


# ----------------------------------------------------------------------------
# clocks during the timed region
# ----------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi sampled every 50 ms from before the warm-up; stop(t0, t1) keeps the samples taken
    inside the timed region's wall-clock window [t0, t1] (a C3 region is ~70 ms), widened by 0.25 s
    on each side only if none fell inside (then "window": "widened")."""
    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self, t0=None, t1=None):
        if self.proc is None:
            return None
        time.sleep(0.1)  # the sample after the region's end
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        import datetime
        stamped = []
        for line in open(self.path):
            parts = [s.strip() for s in line.split(",")]
            if len(parts) >= 10:
                try:
                    ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                except ValueError:
                    ts = None
                stamped.append((ts, parts[1:]))
        os.unlink(self.path)
        window = "timed region"
        rows = [r for ts, r in stamped if t0 is None or (ts is not None and t0 <= ts <= t1)]
        if not rows and t0 is not None:
            window = "widened"
            rows = [r for ts, r in stamped if ts is not None and t0 - 0.25 <= ts <= t1 + 0.25]
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = max((float(r[2]) for r in rows if r[2].replace(".", "").isdigit()), default=None)
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for n, v in zip(names, r[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        loaded = [s for s in sm if mx and s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(rows), "window": window}


# ----------------------------------------------------------------------------
# the oracle, timed on the host cores (cpu_baseline / --impl reference)
# ----------------------------------------------------------------------------
def time_oracle(cfg, budget_s: float, rank: int = 0, single_thread: bool = False):
    """frames/s of the fp64 oracle on a bounded sample (b chunks) of the same workload."""
    import oracle
    _, params, batch = synth.make_workload(cfg, rank)
    theta = oracle.pack_params(params, cfg.L, cfg.D, cfg.H, cfg.K)

    def run(b, T):
        x = np.ascontiguousarray(batch.x[:T, :b])
        m = np.ascontiguousarray(batch.mask[:T, :b])
        lab = np.ascontiguousarray(batch.labels[:T, :b]) if cfg.K > 0 else None
        dy = np.ascontiguousarray(batch.dy_top[:T, :b]) if cfg.K == 0 else None
        t0 = time.perf_counter()
        oracle.blstm_step(theta, x, m, cfg.L, cfg.H, cfg.K, labels=lab, dy_top=dy, lr=1e-5)
        return time.perf_counter() - t0, int(m.sum())

    cores = oracle.num_threads()
    b = min(cfg.B, cores)                      # one chunk per host thread
    dt, _ = run(b, 8)                          # calibration: cost per frame-step
    T = int(np.clip(budget_s / max(dt / 8, 1e-6), 8, cfg.T))
    dt, fr = run(b, T)
    res = {"value": fr / dt, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
           "sample": f"one training step (fwd+BPTT+SGD, fp64) of {cfg.name} restricted to {b} of its "
                     f"{cfg.B} chunks and their first {T} of {cfg.T} frames ({fr} valid frames) in "
                     f"{dt:.1f} s; OpenMP over batch rows / output rows"}
    if single_thread and cores > 1:  # the same oracle on one host thread (OMP_NUM_THREADS=1 equivalent)
        lib = oracle.lib()
        lib.omp_set_num_threads(1)
        try:
            d1, _ = run(1, 8)
            T1 = int(np.clip(0.35 * budget_s / max(d1 / 8, 1e-6), 8, cfg.T))
            d1, f1 = run(1, T1)
        finally:
            lib.omp_set_num_threads(cores)
        res["single_thread"] = {"value": f1 / d1, "unit": UNIT, "cores": 1,
                                "sample": f"1 chunk, its first {T1} frames ({f1} valid frames) in {d1:.1f} s"}
    return res


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(args, cfg):
    rank, _, world = rank_env()
    if rank != 0:
        return
    budget = max(2.0, min(10.0, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        time_oracle(cfg, budget)
    vals = [time_oracle(cfg, budget) for _ in range(args.steps)]
    v = statistics.median(r["value"] for r in vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": workload_desc(cfg, world),
            "cpu_baseline": dict(vals[-1], value=v),
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------
# the CUDA path
# ----------------------------------------------------------------------------
def spawn_ranks(args):
    """`bench.py --gpus N` without a launcher: re-run this script under torchrun with N ranks on
    this node (127.0.0.1), the launch the driver uses.  Fails loudly when the node has fewer than N
    GPUs rather than timing fewer."""
    import socket
    if args.impl == "cuda":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} requested but this node has {have} GPU(s)")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3", choices=sorted(synth.CONFIGS))
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--dp-mode", default="sync", choices=["sync", "avg"])
    ap.add_argument("--avg-k", type=int, default=3)
    ap.add_argument("--lr", type=float, default=1e-5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dropout", type=float, default=0.0, help="input dropout of every layer (NEXT-4); 0 = off")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--precision", default="fp16", choices=["fp16", "fp16x2w"],
                    help="tensor-core operand precision (blstm.h BLSTM_PREC_*)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = synth.CONFIGS[args.config]
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn_ranks(args)  # one process per GPU (the driver's torchrun launch, done here)
    _, _, world = rank_env()
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} ranks were launched")
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist
    from paper_1608_00895_b200 import blstm
    from paper_1608_00895_b200.train import StackTrainer, dp_comm_from_torch

    rank, local, world = rank_env()
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    comm = dp_comm_from_torch(rank, world)
    cfg, params, batch = synth.make_workload(cfg, rank)
    tr = StackTrainer(cfg, params, batch, dev, lr=args.lr, comm=comm, world=world,
                      sched=DPSchedule(args.dp_mode, args.avg_k if args.dp_mode == "avg" else 1),
                      dropout=args.dropout, dropout_seed=7 + 1000 * rank,
                      precision={"fp16": 0, "fp16x2w": 1}[args.precision])

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    def max_over_ranks(v):
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    def sum_over_ranks(v):
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return t.item()

    clocks = ClockSampler(local)  # sampling from before the warm-up: running by the timed region
    clocks.start()
    for _ in range(args.warmup):
        tr.step()
    barrier()

    # ---------------- untimed profiled pass: every launch category ----------------
    # Each profiled launch is bracketed by two event records between the stream's kernels (~1.7 us
    # per launch, ~1 % of a C3 step), so the timed region below brackets only the dominant
    # category (the roofline's kernel); the others' per-step times come from this pass.
    n_prof = max(1, min(args.steps, 5))
    blstm.blstm_profile_select(-1)
    blstm.blstm_profile_enable(True)
    for _ in range(n_prof):
        tr.step()
    prof_all = {c: blstm.blstm_profile_read(c) for c in (blstm.PROF_REC_FWD, blstm.PROF_REC_BWD, blstm.PROF_GEMM)}
    blstm.blstm_profile_enable(False)
    dom = max(prof_all, key=lambda c: prof_all[c][0])
    barrier()

    # ---------------- device-resident timed region ----------------
    n0 = blstm.blstm_launch_count()
    blstm.blstm_profile_select(1 << dom)
    blstm.blstm_profile_enable(True)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    w0 = time.time()
    e0.record(st)
    for _ in range(args.steps):
        tr.step()
    e1.record(st)
    barrier()
    w1 = time.time()
    t_local = e0.elapsed_time(e1) / 1e3
    launches = blstm.blstm_launch_count() - n0
    # the dominant category live from the timed region; the others scaled from the untimed pass
    prof = {c: (prof_all[c][0] * args.steps / n_prof, prof_all[c][1] * args.steps // n_prof) for c in prof_all}
    prof[dom] = blstm.blstm_profile_read(dom)
    blstm.blstm_profile_enable(False)
    blstm.blstm_profile_select(-1)
    clk = clocks.stop(w0, w1)
    t_max = max_over_ranks(t_local)
    frames = sum_over_ranks(tr.valid_frames * args.steps)
    value = frames / t_max

    # ---------------- end to end: host buffers, H2D + D2H inside the timed region ----------------
    ek = args.e2e_steps or args.steps
    hx = torch.tensor(batch.x).pin_memory()
    hm = torch.tensor(batch.mask).pin_memory()
    hl = torch.tensor(batch.labels).pin_memory() if cfg.K > 0 else None
    hloss = torch.zeros(1, dtype=torch.float64).pin_memory()
    h2d = hx.numel() * 4 + hm.numel() + (hl.numel() * 4 if hl is not None else 0)
    # double-buffered inputs: step i+1's H2D copies run on a copy stream while step i computes (each
    # step's inputs are still copied from pinned host memory inside the timed region)
    bufs = [(tr.x, tr.mask, tr.labels),
            (torch.empty_like(tr.x), torch.empty_like(tr.mask), torch.empty_like(tr.labels) if hl is not None else None)]
    cs = torch.cuda.Stream(device=dev)
    copied = [torch.cuda.Event(), torch.cuda.Event()]
    used = [torch.cuda.Event(), torch.cuda.Event()]

    def h2d_into(k):
        xb, mb, lb = bufs[k]
        xb.copy_(hx, non_blocking=True)
        mb.copy_(hm, non_blocking=True)
        if hl is not None:
            lb.copy_(hl, non_blocking=True)
        copied[k].record(cs)

    barrier()
    e0.record(st)
    cs.wait_stream(st)
    with torch.cuda.stream(cs):
        h2d_into(0)
    for i in range(ek):
        k = i & 1
        st.wait_event(copied[k])
        tr.x, tr.mask, tr.labels = bufs[k]
        tr.step()
        used[k].record(st)
        if i + 1 < ek:  # the next step's inputs, into the other buffer once its last reader is done
            with torch.cuda.stream(cs):
                if i >= 1:
                    cs.wait_event(used[1 - k])
                h2d_into(1 - k)
        hloss.copy_(tr.loss, non_blocking=True)
    e1.record(st)
    barrier()
    tr.x, tr.mask, tr.labels = bufs[0]
    t_e2e = max_over_ranks(e0.elapsed_time(e1) / 1e3)
    e2e_value = sum_over_ranks(tr.valid_frames * ek) / t_e2e

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peaks = measured_peaks()
    cats = {0: "lstm_rec_fwd", 1: "lstm_rec_bwd", 2: "gemm_f16 (all GEMMs)"}
    roof = kernel_roofline(dom, prof[dom][0], prof[dom][1], cfg, tr.valid_frames, peaks, args.steps)
    kprefix = {0: "step_fwd" if cfg.H > 512 else "lstm_rec_fwd_kernel",
               1: "step_bwd" if cfg.H > 512 else "lstm_rec_bwd_kernel", 2: "gemm_f16_kernel"}[dom]
    tr_ncu = ncu_traffic(kprefix, cfg.name)
    n_gemm = len(gemm_shapes(cfg))
    alg_launch = (roof["achieved"] * 1e9 * prof[dom][0] / max(prof[dom][1], 1) / 1e3 if roof["unit"] == "GB/s"
                  else gemm_alg_bytes(cfg) / n_gemm if dom == 2 else 2 * tr.valid_frames * 40 * cfg.H)
    roof.update({"kernel": cats[dom], "traffic": tr_ncu["bytes"] if tr_ncu else None,
                 "traffic_unit": "bytes/launch (dram read + write)",
                 "traffic_source": tr_ncu["source"] if tr_ncu else None,
                 "algorithmic_bytes_per_launch": alg_launch,
                 "launch_ms": prof[dom][0] / max(prof[dom][1], 1),
                 "share_of_step": prof[dom][0] / (t_local * 1e3),
                 "peak_source": peaks["source"], "peak_note": peaks["note"]})
    step_ms = t_max / args.steps * 1e3
    V = tr.valid_frames
    roof["step"] = step_roofline(cfg, V, peaks, step_ms)
    t_tc = V * alg_flops_per_frame(cfg) / (peaks["tf"] * 1e12) * 1e3
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f16 MMA operands / f32 accumulate+state", "data": "synthetic",
        "config": dict(workload_desc(cfg, world), valid_frames_per_gpu=V, dp_mode=args.dp_mode,
                       **({"avg_k": args.avg_k} if args.dp_mode == "avg" else {}),
                       **({"input_dropout": args.dropout} if args.dropout > 0 else {}),
                       precision=args.precision),
        "roofline": roof,
        "kernel_ms_per_step": {cats[c]: prof[c][0] / args.steps for c in prof},
        "kernel_ms_source": {"timed_region": cats[dom], "untimed_pass_steps": n_prof},
        "roofline_by_kernel": {cats[c]: kernel_roofline(c, prof[c][0], prof[c][1], cfg, tr.valid_frames, peaks, args.steps)
                               for c in prof},
        "step_tensor_bound_ms": t_tc,
        "gpu_launches": launches,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 8},
        "clocks": clk,
        "tflops_achieved": V * world * alg_flops_per_frame(cfg) * args.steps / t_max / 1e12,
    }
    if world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = time_oracle(cfg, 15.0, single_thread=True)
        except Exception as e:  # the oracle is a reported baseline, never the product path
            line["cpu_baseline"] = {"error": str(e)}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
