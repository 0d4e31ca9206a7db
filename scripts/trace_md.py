"""Per-diagonal phase timing of the tensor-core MDLSTM wavefront (mdlstm.cu md_wave_*_kernel; CTA 0
thread 0, clock64 -> ns at --mhz).  Needs a trace build (build.py --trace)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1608_00895_b200 import blstm
from scripts.trace_rec import report

FWD = [(0, None), (1, "MMA issue"), (2, "Z prefetch + mask loads"), (3, "(waiting warp: Z + MMA)"), (4, "__syncthreads"),
       (5, "TMEM ld -> staging"), (6, "__syncthreads"), (7, "gates + cell + stores"), (8, "fence + __syncthreads")]
BWD = [(0, None), (1, "MMA issue"), (2, "input prefetch + dy loads"), (3, "(waiting warp: inputs + MMA)"), (4, "__syncthreads"),
       (5, "TMEM ld -> staging"), (6, "__syncthreads"), (7, "gate gradients + stores"), (8, "fence + __syncthreads")]
# the CTA-pair backward (BLSTM_MD_PAIR=1, Hp in {32, 64}): slot 9 = after the partner's partial landed
BWD2 = [(0, None), (1, "MMA issue"), (2, "input prefetch"), (3, "wait inputs + MMA"), (4, "__syncthreads"),
        (5, "TMEM ld -> own stg / partner st.async"), (9, "wait partner's partial"), (6, "__syncthreads"),
        (7, "gate gradients + stores"), (8, "fence + __syncthreads")]

ap = argparse.ArgumentParser()
ap.add_argument("--H", type=int, default=64)
ap.add_argument("--mhz", type=float, default=1965.0)
args = ap.parse_args()
U, V, B, D, H = 32, 256, 16, 16, args.H
dev = torch.device("cuda:0")
desc = blstm.mdlstm_desc(U, V, B, D, H)
n, wsb, rsb = blstm.mdlstm_sizes(desc)
g = torch.Generator(device=dev).manual_seed(0)
th = 0.2 * torch.randn(n, device=dev, generator=g)
x = torch.randn((U, V, B, D), device=dev, generator=g)
m = torch.ones((U, V, B), dtype=torch.uint8, device=dev)
dy = torch.randn((U, V, B, 4 * H), device=dev, generator=g)
y = torch.empty((U, V, B, 4 * H), device=dev)
dx = torch.empty_like(x)
grad = torch.zeros_like(th)
ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
res = torch.empty(rsb, dtype=torch.uint8, device=dev)
ND = U + V - 1
tf = torch.zeros((ND, 16), dtype=torch.int64, device=dev)
tb = torch.zeros((ND, 16), dtype=torch.int64, device=dev)
blstm.mdlstm_fwd(desc, th, x, m, y, res, ws)
blstm.mdlstm_bwd(desc, th, x, m, res, dy, dx, grad, ws)
blstm.blstm_debug_set_trace(tf, tb)
blstm.mdlstm_fwd(desc, th, x, m, y, res, ws)
blstm.mdlstm_bwd(desc, th, x, m, res, dy, dx, grad, ws)
torch.cuda.synchronize()
blstm.blstm_debug_set_trace(None, None)
f = tf.cpu().numpy().astype(np.float64) * 1e3 / args.mhz
b = tb.cpu().numpy().astype(np.float64) * 1e3 / args.mhz
print(f"U={U} V={V} B={B} H={H}")
report("wavefront forward (per diagonal)", f, FWD)
report("wavefront backward (per diagonal)", b, BWD2 if os.environ.get("BLSTM_MD_PAIR", "1") != "0" and H in (32, 64) else BWD)
