"""Times every GEMM shape of one C3 training step on the library's tcgen05 GEMM (C-ABI test hook
blstm_gemm_f16, plain row-major fp32 output) and, beside it, cuBLAS through torch.matmul on the
same fp16 operands (fp16 output), as a yardstick.  Prints ms and TFLOP/s per shape.

Shapes (C3: T*B = 20250 frames, Hq = 512, D padded 64, K = 1501 padded 1536), with the operand
majors the stack uses (api.cu): a_mn / b_mn = 1 means MN-major.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1608_00895_b200 import blstm  # noqa: E402

TB, Hq, Dp0, Kp = 20250, 512, 64, 1536
SHAPES = [  # name, M, N, K, a_mn, b_mn, per-step count
    ("Z layer0", TB, 8 * Hq, Dp0, 0, 1, 1),
    ("Z layer1-4", TB, 8 * Hq, 2 * Hq, 0, 1, 4),
    ("logits", TB, Kp, 2 * Hq, 0, 1, 1),
    ("dY_top", TB, 2 * Hq, Kp, 0, 0, 1),
    ("dW_out", 1501, 2 * Hq, TB, 1, 1, 1),
    ("dX layer1-4", TB, 2 * Hq, 8 * Hq, 0, 0, 4),
    ("dW layer0", 8 * Hq, Dp0, TB, 1, 1, 1),
    ("dW layer1-4", 8 * Hq, 2 * Hq, TB, 1, 1, 4),
    ("dR (x2/layer)", 4 * Hq, Hq, TB, 1, 1, 10),
    # not in the C3 total (count 0): C5 (T*B = 128000, Hq = 1024) and the MDLSTM bench (32x256x16
    # cells, 20Hp = 1280 at H = 64, K = 3 Dp for the split projection)
    ("C5 Z layer0", 128000, 8192, 64, 0, 1, 0),
    ("C5 dX layer1-3", 128000, 2048, 8192, 0, 0, 0),
    ("MD Z (K=3Dp)", 131072, 1280, 192, 0, 0, 0),
]


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(0)
    tot_ours = tot_cublas = 0.0
    print(f"{'gemm':16s} {'M':>6} {'N':>6} {'K':>6}  {'ours ms':>8} {'TF/s':>6}  {'cuBLAS ms':>9} {'TF/s':>6}")
    for name, M, N, K, amn, bmn, cnt in SHAPES:
        r8 = lambda v: (v + 7) // 8 * 8  # noqa: E731  (ld must be a multiple of 8)
        A = (torch.randn((K, r8(M)) if amn else (M, r8(K)), device=dev, generator=g) * 0.1).half()
        A = A[:, :M] if amn else A[:, :K]
        B = (torch.randn((K, r8(N)) if bmn else (N, r8(K)), device=dev, generator=g) * 0.1).half()
        B = B[:, :N] if bmn else B[:, :K]
        C = torch.empty((M, r8(N)), device=dev, dtype=torch.float32)[:, :N]
        ours = timeit(lambda: blstm.blstm_gemm_f16(A, amn, B, bmn, C, M, N, K))
        Am = A.t() if amn else A            # [M, K] view
        Bm = B if bmn else B.t()            # [K, N] view
        cub = timeit(lambda: torch.matmul(Am, Bm))
        fl = 2.0 * M * N * K
        tot_ours += cnt * ours
        tot_cublas += cnt * cub
        print(f"{name:16s} {M:6d} {N:6d} {K:6d}  {ours:8.3f} {fl / ours / 1e9:6.0f}  {cub:9.3f} {fl / cub / 1e9:6.0f}")
    print(f"per-step total (x count): ours {tot_ours:.3f} ms, cuBLAS {tot_cublas:.3f} ms")


if __name__ == "__main__":
    main()
