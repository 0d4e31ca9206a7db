"""Debug: the tensor-core MDLSTM wavefront vs the CUDA-core kernels, per grid size (y and grads)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1608_00895_b200 import blstm

def run(U, V, B, D, H, wave, stable=False, irregular=True, seed=1):
    os.environ["BLSTM_MD_WAVE"] = wave
    dev = torch.device("cuda:0")
    g = np.random.default_rng(seed)
    desc = blstm.mdlstm_desc(U, V, B, D, H, stable)
    n, wsb, rsb = blstm.mdlstm_sizes(desc)
    th = torch.tensor((float(os.environ.get("MD_SCALE", "0.4")) * g.standard_normal(n)).astype(np.float32), device=dev)
    x = torch.tensor(g.standard_normal((U, V, B, D)).astype(np.float32), device=dev)
    m = np.ones((U, V, B), np.uint8)
    if irregular:
        m[g.random((U, V, B)) < 0.15] = 0
    mt = torch.tensor(m, device=dev)
    dy = torch.tensor(g.standard_normal((U, V, B, 4 * H)).astype(np.float32), device=dev) * mt[..., None]
    y = torch.zeros((U, V, B, 4 * H), device=dev)
    ws = torch.zeros(wsb, dtype=torch.uint8, device=dev)
    res = torch.zeros(rsb, dtype=torch.uint8, device=dev)
    blstm.mdlstm_fwd(desc, th, x, mt, y, res, ws)
    dx = torch.zeros_like(x); grad = torch.zeros_like(th)
    blstm.mdlstm_bwd(desc, th, x, mt, res, dy, dx, grad, ws)
    torch.cuda.synchronize()
    return y.cpu().numpy(), dx.cpu().numpy(), grad.cpu().numpy()

if __name__ == '__main__':
  for (U, V, B, H, irr) in [(12, 12, 1, 16, False), (17, 17, 1, 16, False), (24, 24, 1, 16, False), (32, 32, 1, 16, False),
                          (32, 64, 1, 16, False), (32, 256, 1, 16, False), (32, 256, 2, 64, True), (20, 40, 2, 32, True)]:
    a = run(U, V, B, 8, H, "1", irregular=irr)
    b = run(U, V, B, 8, H, "0", irregular=irr)
    ey = np.abs(a[0] - b[0]).max() / max(np.abs(b[0]).max(), 1e-30)
    # first diagonal (per direction 0 frame) with a mismatch
    dif = np.abs(a[0] - b[0]).max(axis=(2, 3))
    bad = np.argwhere(dif > 1e-4)
    first = None
    if len(bad):
        dd = bad.sum(axis=1)
        first = (int(dd.min()), bad[dd.argmin()].tolist())
    print(f"U={U} V={V} B={B} H={H} irr={irr}: y {ey:.2e} nan(wave) {np.isnan(a[0]).sum()} first bad (u+v, cell) {first} "
          f"dx nan {np.isnan(a[1]).sum()} grad nan {np.isnan(a[2]).sum()} "
          f"dx rel {np.abs(a[1]-b[1]).max()/max(np.abs(b[1]).max(),1e-30):.2e} g rel {np.nanmax(np.abs(a[2]-b[2]))/max(np.abs(b[2]).max(),1e-30):.2e}", flush=True)
