"""One GEMM shape through the C-ABI hook, launched `reps` times (an ncu capture target):
python scripts/gemm_one.py M N K a_mn b_mn [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1608_00895_b200 import blstm  # noqa: E402

M, N, K, amn, bmn = (int(v) for v in sys.argv[1:6])
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 3
dev = torch.device("cuda:0")
r8 = lambda v: (v + 7) // 8 * 8  # noqa: E731
A = (torch.randn((K, r8(M)) if amn else (M, r8(K)), device=dev) * 0.1).half()
A = A[:, :M] if amn else A[:, :K]
B = (torch.randn((K, r8(N)) if bmn else (N, r8(K)), device=dev) * 0.1).half()
B = B[:, :N] if bmn else B[:, :K]
C = torch.empty((M, r8(N)), device=dev, dtype=torch.float32)[:, :N]
for _ in range(reps):
    blstm.blstm_gemm_f16(A, amn, B, bmn, C, M, N, K)
torch.cuda.synchronize()
print("ok", M, N, K)
