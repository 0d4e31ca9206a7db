"""Per-launch table of one training step's `ncu --set full` capture (scripts/ncu_step.py, summarised
by scripts/ncu_summarize.py --config): each GEMM launch labelled with its shape (the launch order of
stack_step_impl with BLSTM_OVERLAP=0), its algorithmic bytes (fp16 operands read once, fp32 output
written once) and FLOPs next to ncu's DRAM bytes, tensor-pipe % and duration.

usage: python scripts/ncu_step_table.py profiles/r02_ncu_full_C3.json > profiles/r02_ncu_full_C3_table.md
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1608_00895_b200 import synth  # noqa: E402


def labels(cfg):
    """kernel labels in launch order (host order; ncu serialises in that order)"""
    rup = lambda a, b: (a + b - 1) // b * b  # noqa: E731
    Hq, TB = rup(cfg.H, 256), cfg.T * cfg.B
    Kp = rup(cfg.K, 64)
    Dn = lambda l: rup(cfg.D, 64) if l == 0 else 2 * Hq  # noqa: E731
    out = []
    for l in range(cfg.L):
        out += [("gemm", f"Z{l}", TB, 8 * Hq, Dn(l)), ("rec", f"fwd{l}")]
    out += [("gemm", "logits", TB, cfg.K, 2 * Hq), ("gemm", "dY_top", TB, 2 * Hq, Kp)]
    for l in range(cfg.L - 1, -1, -1):
        out.append(("rec", f"bwd{l}"))
        if l == cfg.L - 1:
            out.append(("gemm", "dW_out^T", cfg.K, 2 * Hq, TB))
        else:
            out += [("gemm", f"dW{l + 1}^T", 8 * Hq, Dn(l + 1), TB), ("gemm", f"dR{l + 1}^T d0", 4 * Hq, Hq, TB),
                    ("gemm", f"dR{l + 1}^T d1", 4 * Hq, Hq, TB)]
        if l > 0:
            out.append(("gemm", f"dX{l}", TB, Dn(l), 8 * Hq))
    out += [("gemm", "dW0^T", 8 * Hq, Dn(0), TB), ("gemm", "dR0^T d0", 4 * Hq, Hq, TB), ("gemm", "dR0^T d1", 4 * Hq, Hq, TB)]
    return out


def main():
    j = json.load(open(sys.argv[1]))
    cfg = synth.CONFIGS[j["config"]]
    ks = next(iter(j["full_captures"].values()))
    lab = labels(cfg)
    # the launch order of the capture: forward GEMMs/recurrences, head, then per layer the BPTT
    # followed (host order) by the side work it overlaps and the dX GEMM
    gem = [x for x in lab if x[0] == "gemm"]
    rec = [x for x in lab if x[0] == "rec"]
    gi = ri = 0
    print(f"# One {cfg.name} training step under `ncu --set full` (BLSTM_OVERLAP=0, serialised, cold cache)\n")
    print(f"Source: `{sys.argv[1]}` ({len(ks)} launches).  alg MB = fp16 A and B read once + fp32 C written once;")
    print("DRAM MB = dram__bytes_read.sum + dram__bytes_write.sum.  The weight-gradient GEMMs ran capped to the")
    print("SMs the recurrence leaves (grid 32-52) as in the live step.\n")
    print("| # | kernel | shape (M x N x K) | grid | us | TFLOP/s | tensor pipe % | alg MB | DRAM MB | DRAM / alg |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    tot = {"gemm_us": 0, "gemm_alg": 0, "gemm_dram": 0, "gemm_flop": 0}
    for n, k in enumerate(ks):
        dram = (k["dram_read"] + k["dram_write"])  # Mbyte
        if k["kernel"].startswith("gemm"):
            _, name, M, N, K = gem[gi] if gi < len(gem) else ("gemm", "?", 0, 0, 0)
            gi += 1
            alg = (2 * (M * K + N * K) + 4 * M * N) / 1e6
            fl = 2 * M * N * K
            tf = fl / (k["duration"] * 1e-6) / 1e12 if k["duration"] else 0
            tot["gemm_us"] += k["duration"]; tot["gemm_alg"] += alg; tot["gemm_dram"] += dram; tot["gemm_flop"] += fl
            print(f"| {n} | {name} | {M} x {N} x {K} | {k['grid']:.0f} | {k['duration']:.1f} | {tf:.0f} | "
                  f"{k['tensor_pipe_pct']:.1f} | {alg:.1f} | {dram:.1f} | {dram / alg:.2f} |")
        else:
            name = rec[ri][1] if ri < len(rec) else "?"
            ri += 1
            print(f"| {n} | {k['kernel']} ({name}) | - | {k['grid']:.0f} | {k['duration']:.1f} | - | "
                  f"{k['tensor_pipe_pct']:.1f} | - | {dram:.1f} | - |")
    print(f"\nGEMMs: {tot['gemm_us']:.0f} us, {tot['gemm_flop'] / 1e12:.2f} TFLOP "
          f"({tot['gemm_flop'] / (tot['gemm_us'] * 1e-6) / 1e12:.0f} TFLOP/s serialised), "
          f"DRAM {tot['gemm_dram']:.0f} MB vs algorithmic {tot['gemm_alg']:.0f} MB "
          f"({tot['gemm_dram'] / tot['gemm_alg']:.2f}x)")


if __name__ == "__main__":
    main()
