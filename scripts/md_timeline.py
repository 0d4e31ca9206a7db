"""Launch timeline of one MDLSTM fwd + bwd call at the bench grid (32 x 256 x 16, H = 64)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1608_00895_b200 import blstm
U, V, B, D, H = 32, 256, 16, 16, 64
dev = torch.device("cuda:0")
desc = blstm.mdlstm_desc(U, V, B, D, H)
n, wsb, rsb = blstm.mdlstm_sizes(desc)
th = 0.2 * torch.randn(n, device=dev); x = torch.randn((U, V, B, D), device=dev); m = torch.ones((U, V, B), dtype=torch.uint8, device=dev)
dy = torch.randn((U, V, B, 4 * H), device=dev); y = torch.empty((U, V, B, 4 * H), device=dev); dx = torch.empty_like(x); grad = torch.zeros_like(th)
ws = torch.empty(wsb, dtype=torch.uint8, device=dev); res = torch.empty(rsb, dtype=torch.uint8, device=dev)
for _ in range(3):
    blstm.mdlstm_fwd(desc, th, x, m, y, res, ws); blstm.mdlstm_bwd(desc, th, x, m, res, dy, dx, grad, ws)
torch.cuda.synchronize()
blstm.blstm_profile_enable(2)
blstm.mdlstm_fwd(desc, th, x, m, y, res, ws); blstm.mdlstm_bwd(desc, th, x, m, res, dy, dx, grad, ws)
torch.cuda.synchronize()
import numpy as np
recs = sorted(blstm.blstm_profile_timeline(), key=lambda r: r[2])
for cat, si, t0, t1, a, b, c in recs:
    print(f"{int(cat)} {t0:8.3f} {t1 - t0:7.3f}  M={int(a)} N={int(b)} K={int(c)}")
