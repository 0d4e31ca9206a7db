"""Shared helpers of the GPU parity tests: run the C-ABI on torch device tensors
and compare with the fp64 oracle.  Tolerances (BASELINE.json north_star, DESIGN.md
R10): outputs and cell states normwise max|g-r|/max|r| <= 1e-3; gradients
relative L2 <= 1e-2."""
import json
import os

import numpy as np
import torch

import oracle
from paper_1608_00895_b200 import blstm

OUT_TOL = 1e-3
GRAD_TOL = 1e-2


def record(case, errs, **extra):
    """Append one parity record (per-tensor error magnitudes) as a JSON line to $BLSTM_PARITY_LOG,
    when set.  The committed summaries under profiles/ (r02_parity_*.jsonl) come from this."""
    path = os.environ.get("BLSTM_PARITY_LOG")
    if not path:
        return
    rec = {"case": case, "errors": {(k if isinstance(k, str) else "/".join(map(str, k))): float(v)
                                    for k, v in errs.items()}}
    rec.update(extra)
    with open(path, "a") as f:
        f.write(json.dumps(rec) + "\n")


def dev():
    return torch.device("cuda:0")


def T_(a, dtype=None):
    t = torch.as_tensor(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(dev())


def np_(t):
    return t.detach().double().cpu().numpy()


def norm_rel(g, r):
    den = np.max(np.abs(r))
    return float(np.max(np.abs(g - r)) / den) if den > 0 else float(np.max(np.abs(g)))


def l2_rel(g, r):
    den = np.linalg.norm(r)
    return float(np.linalg.norm(g - r) / den) if den > 0 else float(np.linalg.norm(g))


def run_layer(case, direction=1, with_state=True, ldx_pad=0, ldy_pad=0, precision=0):
    """lstm_fwd + lstm_bwd through the ABI; returns numpy fp64 results."""
    x = case["x"].astype(np.float32)
    T, B, D = x.shape
    H = case["R"].shape[0]
    ldx, ldy = D + ldx_pad, H + ldy_pad
    xp = np.zeros((T, B, ldx), np.float32)
    xp[..., :D] = x
    desc = blstm.lstm_desc(T, B, D, H, direction, ldx=ldx, ldy=ldy, precision=precision)
    ws = torch.zeros(blstm.lstm_workspace_bytes(desc), dtype=torch.uint8, device=dev())
    res = torch.zeros(blstm.lstm_reserve_bytes(desc), dtype=torch.uint8, device=dev())
    gx = T_(xp)
    gm = T_(case["mask"].astype(np.uint8))
    W, R, b = T_(case["W"], torch.float32), T_(case["R"], torch.float32), T_(case["b"], torch.float32)
    h0 = T_(case["h0"], torch.float32) if with_state else None
    c0 = T_(case["c0"], torch.float32) if with_state else None
    y = torch.full((T, B, ldy), 7.0, device=dev())
    c = torch.zeros((T, B, H), device=dev())
    hT = torch.zeros((B, H), device=dev())
    cT = torch.zeros((B, H), device=dev())
    blstm.lstm_fwd(desc, gx, gm, W, R, b, h0, c0, y, c, hT, cT, res, ws)
    dyp = np.zeros((T, B, ldy), np.float32)
    dyp[..., :H] = case["dy"]
    dy = T_(dyp)
    dhT = T_(case["dhT"], torch.float32) if with_state else None
    dcT = T_(case["dcT"], torch.float32) if with_state else None
    dx = torch.full((T, B, ldx), 3.0, device=dev())
    dW = torch.zeros_like(W); dR = torch.zeros_like(R); db = torch.zeros_like(b)
    dh0 = torch.zeros((B, H), device=dev()); dc0 = torch.zeros((B, H), device=dev())
    blstm.lstm_bwd(desc, gx, gm, W, R, h0, c0, c, res, dy, dhT, dcT, dx, dW, dR, db, dh0, dc0, ws)
    torch.cuda.synchronize()
    return dict(y=np_(y)[..., :H], y_pad=np_(y)[..., H:], c=np_(c), hT=np_(hT), cT=np_(cT),
                dx=np_(dx)[..., :D], dx_pad=np_(dx)[..., D:], dW=np_(dW), dR=np_(dR), db=np_(db),
                dh0=np_(dh0), dc0=np_(dc0))


def oracle_layer(case, direction=1, with_state=True):
    f = oracle.lstm_fwd(case["x"], case["mask"], case["W"], case["R"], case["b"],
                        case["h0"] if with_state else None, case["c0"] if with_state else None, direction)
    g = oracle.lstm_bwd(case["x"], case["mask"], case["W"], case["R"], f, case["dy"],
                        case["dhT"] if with_state else None, case["dcT"] if with_state else None, direction)
    return dict(y=f["y"], c=f["C"], hT=f["hT"], cT=f["cT"], dx=g["dx"], dW=g["dW"], dR=g["dR"],
                db=g["db"], dh0=g["dh0"], dc0=g["dc0"])


def compare_layer(got, ref, label=""):
    errs = {k: norm_rel(got[k], ref[k]) for k in ("y", "c", "hT", "cT")}
    errs.update({k: l2_rel(got[k], ref[k]) for k in ("dx", "dW", "dR", "db", "dh0", "dc0")})
    record(label, errs, metric={"y,c,hT,cT": "normwise", "rest": "rel-L2"})
    for k in ("y", "c", "hT", "cT"):
        assert errs[k] <= OUT_TOL, (label, k, errs)
    for k in ("dx", "dW", "dR", "db", "dh0", "dc0"):
        assert errs[k] <= GRAD_TOL, (label, k, errs)
    return errs


class Stack:
    """Device buffers + one call of blstm_stack_fwd_bwd / blstm_stack_fwd."""

    def __init__(self, L, D, H, K, T, B, dropout=0.0, seed=0, precision=0):
        self.L, self.D, self.H, self.K, self.T, self.B = L, D, H, K, T, B
        self.desc = blstm.stack_desc(L, D, H, K, T, B, dropout=dropout, dropout_seed=seed, precision=precision)
        self.n, self.offs = blstm.blstm_param_offsets(self.desc)
        self.ws = torch.empty(blstm.blstm_stack_workspace_bytes(self.desc), dtype=torch.uint8, device=dev())

    def step(self, theta_np, batch, dy_top=None, side_stream=False):
        theta = T_(theta_np, torch.float32)
        grad = torch.zeros(self.n, dtype=torch.float32, device=dev())
        loss = torch.zeros(1, dtype=torch.float64, device=dev())
        ferr = torch.zeros(1, dtype=torch.int32, device=dev())
        labels = T_(batch.labels) if self.K > 0 else None
        dyt = T_(dy_top, torch.float32) if dy_top is not None else None
        side = torch.cuda.Stream() if side_stream else None
        blstm.blstm_stack_fwd_bwd(self.desc, theta, grad, T_(batch.x), T_(batch.mask), labels, dyt, loss, ferr,
                                  None, self.ws, s_side=side)
        torch.cuda.synchronize()
        return dict(grad=np_(grad), loss=loss.item(), frame_errors=int(ferr.item()))

    def forward(self, theta_np, batch):
        theta = T_(theta_np, torch.float32)
        L, T, B, H = self.L, self.T, self.B, self.H
        Y = torch.zeros((L, T, B, 2 * H), device=dev())
        C = torch.zeros((L, 2, T, B, H), device=dev())
        blstm.blstm_stack_fwd(self.desc, theta, T_(batch.x), T_(batch.mask), Y, C, self.ws)
        torch.cuda.synchronize()
        return np_(Y), np_(C)


def grad_errors(g, ref_grad, L, D, H, K):
    """rel-L2 per parameter tensor of the flat gradient."""
    gv = oracle.unpack(g, L, D, H, K)
    rv = oracle.unpack(ref_grad, L, D, H, K)
    return {k: l2_rel(gv[k], rv[k]) for k in rv}
