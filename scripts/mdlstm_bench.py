"""Throughput of the MDLSTM layer (NEXT-2, mdlstm.cu) on a handwriting-line-shaped workload:
U x V = 32 x 256 grid (text-line height x width after patching), B = 16 images, D = 16 input
channels, H units per direction (32 and 64), four directions, two-forget cell, full masks.

Reported per forward+backward call: device time (CUDA events), grid cells per second, and the
wavefront kernels' time (library launch events, categories rec_fwd / rec_bwd).  The recurrent
contraction is 2 x 5H x H multiply-adds per (cell, direction) in the forward and the same in the
backward's dh.  Two paths (BLSTM_MD_WAVE=1 default / 0): the tensor-core wavefront (one CTA per
(direction, image), 3-term split fp16 products on tcgen05; latency-bound: the per-diagonal chain of
MMA -> TMEM -> gates -> next B operand inside one SM) and the CUDA-core per-diagonal kernels (fp32
FMA; FP32 peak = 148 SMs x 128 lanes x 2 x 1.965 GHz = 74.4 TFLOP/s)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1608_00895_b200 import blstm  # noqa: E402

PEAK_FP32 = 148 * 128 * 2 * 1.965e9 / 1e12


PEAK_TC = 1378.5  # dense fp16/bf16 tensor TFLOP/s, sustained (MEASURED_PEAKS.json bf16_tflops_sustained)


def roof(path, rec_flop, fw_ms, bw_ms, ndiag):
    """The recurrent contraction against the roof of the path that ran it.  CUDA cores: fp32 FMA peak.
    tcgen05: the MMAs issue 3x the algorithmic FLOPs (hi/lo split products) and the wavefront is a
    chain of ndiag dependent steps, so the tensor fraction is tiny by construction; the latency view
    (us per diagonal, 2 passes) is the one that bounds it."""
    a_f, a_b = rec_flop / (fw_ms * 1e-3) / 1e12, rec_flop / (bw_ms * 1e-3) / 1e12
    if path.startswith("per-diagonal"):
        return {"bound": "alu (fp32 FMA)", "achieved_tflops_fwd": round(a_f, 2), "achieved_tflops_bwd": round(a_b, 2),
                "peak_tflops": round(PEAK_FP32, 1), "frac_fwd": round(a_f / PEAK_FP32, 4)}
    return {"bound": "latency (dependent anti-diagonals)", "achieved_tflops_fwd": round(a_f, 2),
            "achieved_tflops_bwd": round(a_b, 2), "mma_issued_tflops_fwd": round(3 * a_f, 2),
            "peak_tflops": PEAK_TC, "tensor_frac_fwd": round(3 * a_f / PEAK_TC, 4),
            "us_per_diagonal_fwd_bwd": round(1e3 * (fw_ms + bw_ms) / ndiag, 2)}


def run(U, V, B, D, H, K=20):
    dev = torch.device("cuda:0")
    desc = blstm.mdlstm_desc(U, V, B, D, H)
    n, wsb, rsb = blstm.mdlstm_sizes(desc)
    g = torch.Generator(device=dev).manual_seed(0)
    th = 0.2 * torch.randn(n, device=dev, generator=g)
    P1 = n // 4  # per direction: W [D,5H], Ru, Rv [H,5H], b [5H]; forget-gate biases -1.5 (fu + fv < 1:
    for k in range(4):  # the two-forget cell stays finite over 287 diagonals)
        o = k * P1 + D * 5 * H + 2 * H * 5 * H
        th[o + H:o + 3 * H] -= 1.5
    x = torch.randn((U, V, B, D), device=dev, generator=g)
    m = torch.ones((U, V, B), dtype=torch.uint8, device=dev)
    dy = torch.randn((U, V, B, 4 * H), device=dev, generator=g)
    y = torch.empty((U, V, B, 4 * H), device=dev)
    dx = torch.empty_like(x)
    grad = torch.zeros_like(th)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    res = torch.empty(rsb, dtype=torch.uint8, device=dev)
    for _ in range(3):
        blstm.mdlstm_fwd(desc, th, x, m, y, res, ws)
        blstm.mdlstm_bwd(desc, th, x, m, res, dy, dx, grad, ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(K):
        blstm.mdlstm_fwd(desc, th, x, m, y, res, ws)
        blstm.mdlstm_bwd(desc, th, x, m, res, dy, dx, grad, ws)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    blstm.blstm_profile_enable(1)
    blstm.mdlstm_fwd(desc, th, x, m, y, res, ws)
    blstm.mdlstm_bwd(desc, th, x, m, res, dy, dx, grad, ws)
    torch.cuda.synchronize()
    fw = blstm.blstm_profile_read(blstm.PROF_REC_FWD)
    bw = blstm.blstm_profile_read(blstm.PROF_REC_BWD)
    gm = blstm.blstm_profile_read(blstm.PROF_GEMM)
    blstm.blstm_profile_enable(0)
    cells = U * V * B
    rec_flop = cells * 4 * 2 * 5 * H * H * 2  # per pass: 2 predecessors x 5H x H FMAs = 2 flop each
    path = "per-diagonal (CUDA cores)" if os.environ.get("BLSTM_MD_WAVE", "1") == "0" else (
        "wavefront (tcgen05, one CTA per direction x image)" if os.environ.get("BLSTM_MD_PAIR", "1") == "0"
        else "wavefront (tcgen05, CTA pair per direction x image)")
    out = dict(path=path,
               U=U, V=V, B=B, D=D, H=H, diagonals=U + V - 1, ms_fwd_bwd=round(ms, 3),
               cells_per_s=round(cells / (ms * 1e-3)), wavefront_fwd_ms=round(fw[0], 3), wavefront_bwd_ms=round(bw[0], 3),
               gemm_ms=round(gm[0], 3), us_per_diagonal_fwd=round(1e3 * fw[0] / (U + V - 1), 2),
               us_per_diagonal_bwd=round(1e3 * bw[0] / (U + V - 1), 2),
               roofline=roof(path, rec_flop, fw[0], bw[0], U + V - 1))
    print(json.dumps(out), flush=True)
    return out


if __name__ == "__main__":
    for wave, pair in (("1", "1"), ("1", "0"), ("0", "0")):
        os.environ["BLSTM_MD_WAVE"] = wave
        os.environ["BLSTM_MD_PAIR"] = pair
        for H in (32, 64):
            run(32, 256, 16, 16, H)
