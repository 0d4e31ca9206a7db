"""fp64 CPU oracle — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The CUDA product path
(paper_1608_00895_b200) never imports it and shares no code with it.

The arithmetic lives in oracle/oracle.c (plain C, fp64); this module builds it
with gcc, loads it with ctypes and converts numpy arrays.  See oracle.c's header
for the passages each routine follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_i32p = ctypes.POINTER(ctypes.c_int32)
_lp = ctypes.POINTER(ctypes.c_long)


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.ref_param_layout.restype = ctypes.c_long
        _lib.oracle_num_threads.restype = ctypes.c_int
    return _lib


def _d(a: Optional[np.ndarray]):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def lstm_fwd(x, mask, W, R, b, h0=None, c0=None, direction: int = 1):
    """One layer, one direction.  Returns dict y, C, hT, cT, G, Hprev, Cprev (fp64)."""
    x = _f64(x); W = _f64(W); R = _f64(R); b = _f64(b); h0 = _f64(h0); c0 = _f64(c0)
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    T, B, D = x.shape
    H = R.shape[0]
    out = {k: np.zeros((T, B, H)) for k in ("y", "C", "Hprev", "Cprev")}
    out["G"] = np.zeros((T, B, 4 * H))
    out["hT"] = np.zeros((B, H))
    out["cT"] = np.zeros((B, H))
    rc = lib().ref_lstm_fwd(T, B, D, H, int(direction), _d(x), mask.ctypes.data_as(_u8p),
                            _d(W), _d(R), _d(b), _d(h0), _d(c0),
                            _d(out["y"]), _d(out["C"]), _d(out["hT"]), _d(out["cT"]),
                            _d(out["G"]), _d(out["Hprev"]), _d(out["Cprev"]))
    assert rc == 0, rc
    return out


def lstm_bwd(x, mask, W, R, fwd, dy, dhT=None, dcT=None, direction: int = 1):
    """Backward of lstm_fwd.  Returns dict dx, dW, dR, db, dh0, dc0, dA (fp64)."""
    x = _f64(x); W = _f64(W); R = _f64(R); dy = _f64(dy); dhT = _f64(dhT); dcT = _f64(dcT)
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    T, B, D = x.shape
    H = R.shape[0]
    out = dict(dx=np.zeros((T, B, D)), dW=np.zeros((D, 4 * H)), dR=np.zeros((H, 4 * H)),
               db=np.zeros(4 * H), dh0=np.zeros((B, H)), dc0=np.zeros((B, H)),
               dA=np.zeros((T, B, 4 * H)))
    rc = lib().ref_lstm_bwd(T, B, D, H, int(direction), _d(x), mask.ctypes.data_as(_u8p),
                            _d(W), _d(R), _d(fwd["C"]), _d(fwd["G"]), _d(fwd["Hprev"]),
                            _d(fwd["Cprev"]), _d(dy), _d(dhT), _d(dcT),
                            _d(out["dx"]), _d(out["dW"]), _d(out["dR"]), _d(out["db"]),
                            _d(out["dh0"]), _d(out["dc0"]), _d(out["dA"]))
    assert rc == 0, rc
    return out


def param_offsets(L: int, D: int, H: int, K: int):
    offs = np.zeros(6 * L + 2, dtype=np.int64)
    n = lib().ref_param_layout(L, D, H, K, offs.ctypes.data_as(_lp))
    return int(n), offs


def pack_params(params, L: int, D: int, H: int, K: int) -> np.ndarray:
    """Flatten synth.StackParams into the oracle's own flat fp64 theta."""
    n, offs = param_offsets(L, D, H, K)
    th = np.zeros(n)
    for l, (f, bw) in enumerate(params.layers):
        for d, p in enumerate((f, bw)):
            e = 6 * l + 3 * d
            for q, a in enumerate((p.W, p.R, p.b)):
                th[offs[e + q]: offs[e + q] + a.size] = a.ravel()
    if K > 0:
        th[offs[6 * L]: offs[6 * L] + params.W_out.size] = params.W_out.ravel()
        th[offs[6 * L + 1]: offs[6 * L + 1] + K] = params.b_out
    return th


def unpack(theta: np.ndarray, L: int, D: int, H: int, K: int):
    """Views of a flat theta/grad: dict[(l, d, name)] -> array; ('head','W'/'b')."""
    n, offs = param_offsets(L, D, H, K)
    out = {}
    for l in range(L):
        Dl = D if l == 0 else 2 * H
        for d in range(2):
            e = 6 * l + 3 * d
            out[(l, d, "W")] = theta[offs[e]: offs[e] + Dl * 4 * H].reshape(Dl, 4 * H)
            out[(l, d, "R")] = theta[offs[e + 1]: offs[e + 1] + 4 * H * H].reshape(H, 4 * H)
            out[(l, d, "b")] = theta[offs[e + 2]: offs[e + 2] + 4 * H]
    if K > 0:
        out[("head", "W")] = theta[offs[6 * L]: offs[6 * L] + 2 * H * K].reshape(2 * H, K)
        out[("head", "b")] = theta[offs[6 * L + 1]: offs[6 * L + 1] + K]
    return out


def dropout_keep(seed: int, site: int, i: int, p: float) -> bool:
    """oracle.c ref_dropout_keep: the counter-based keep decision of input dropout (R20)."""
    return bool(lib().ref_dropout_keep(ctypes.c_uint32(seed), site, ctypes.c_uint64(i), ctypes.c_double(p)))


def blstm_step(theta, x, mask, L: int, H: int, K: int, labels=None, dy_top=None,
               lr: float = 0.0, want_states: bool = False, want_dx: bool = False,
               dropout: float = 0.0, seed: int = 0):
    """One training step of the L-layer BLSTM (+ CE head when K > 0).

    Returns dict loss, frame_errors, grad (flat), theta_new, and optionally
    Ys [L,T,B,2H], Cs [L,2,T,B,H], dX1 [T,B,D].
    """
    theta = _f64(theta); x = _f64(x); dy_top = _f64(dy_top)
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    T, B, D = x.shape
    n, _ = param_offsets(L, D, H, K)
    assert theta.size == n
    grad = np.zeros(n)
    theta_new = np.zeros(n)
    Ys = np.zeros((L, T, B, 2 * H)) if want_states else None
    Cs = np.zeros((L, 2, T, B, H)) if want_states else None
    dX1 = np.zeros((T, B, D)) if want_dx else None
    loss = ctypes.c_double(0.0)
    ferr = ctypes.c_long(0)
    lab = None
    if K > 0:
        labels = np.ascontiguousarray(labels, dtype=np.int32)
        lab = labels.ctypes.data_as(_i32p)
    rc = lib().ref_blstm_step_ex(L, D, H, K, T, B, _d(theta), _d(x), mask.ctypes.data_as(_u8p),
                                 lab, _d(dy_top), ctypes.c_double(lr), ctypes.byref(loss),
                                 ctypes.byref(ferr), _d(grad), _d(Ys), _d(Cs), _d(dX1),
                                 _d(theta_new), ctypes.c_double(dropout), ctypes.c_uint32(seed))
    assert rc == 0, rc
    return dict(loss=loss.value, frame_errors=ferr.value, grad=grad, theta_new=theta_new,
                Ys=Ys, Cs=Cs, dX1=dX1)


def sgd(theta, grad, lr: float):
    theta = np.array(theta, dtype=np.float64, copy=True)
    grad = _f64(grad)
    lib().ref_sgd(_d(theta), _d(grad), ctypes.c_long(theta.size), ctypes.c_double(lr))
    return theta


OPT_RULES = {"sgd": 0, "momentum": 1, "nesterov": 2, "adagrad": 3, "adadelta": 4, "adam": 5}


def opt_update(rule, theta, grad, s0=None, s1=None, *, lr, mu=0.9, rho=0.95, beta1=0.9, beta2=0.999, eps=1e-8,
               l2=0.0, max_norm=0.0, step=1, is_bias=None, zero_grad=False):
    """One update of oracle.c ref_opt_update (fp64); returns (theta, grad, s0, s1) as new arrays."""
    theta = np.array(theta, dtype=np.float64, copy=True)
    grad = np.array(grad, dtype=np.float64, copy=True)
    n = theta.size
    s0 = np.zeros(n) if s0 is None else np.array(s0, dtype=np.float64, copy=True)
    s1 = np.zeros(n) if s1 is None else np.array(s1, dtype=np.float64, copy=True)
    ib = None if is_bias is None else np.ascontiguousarray(is_bias, dtype=np.uint8)
    lib().ref_opt_update(ctypes.c_int(OPT_RULES[rule] if isinstance(rule, str) else rule), ctypes.c_double(lr),
                         ctypes.c_double(mu), ctypes.c_double(rho), ctypes.c_double(beta1), ctypes.c_double(beta2),
                         ctypes.c_double(eps), ctypes.c_double(l2), ctypes.c_double(max_norm), ctypes.c_long(step),
                         ctypes.c_long(n), _d(theta), _d(grad), _d(s0), _d(s1),
                         None if ib is None else ib.ctypes.data_as(_u8p), ctypes.c_int(int(zero_grad)))
    return theta, grad, s0, s1


def dp_average(thetas):
    th = np.ascontiguousarray(np.stack([np.asarray(t, np.float64) for t in thetas]))
    out = np.zeros(th.shape[1])
    lib().ref_dp_average(th.shape[0], ctypes.c_long(th.shape[1]), _d(th), _d(out))
    return out


# ----------------------------------------------------------------------------
# MDLSTM (§4.2; R21)
# ----------------------------------------------------------------------------
MD_FLIPS = ((False, False), (True, False), (False, True), (True, True))  # identity, flip-u, flip-v, both


def mdlstm_fwd(x, mask, W, Ru, Rv, b, stable: bool):
    """One direction in raster order (oracle.c ref_mdlstm_fwd): x [U,V,B,D], mask [U,V,B]."""
    x = _f64(x)
    U, V, B, D = x.shape
    H = Ru.shape[0]
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    h = np.zeros((U, V, B, H)); c = np.zeros((U, V, B, H)); act = np.zeros((U, V, B, 5 * H))
    rc = lib().ref_mdlstm_fwd(U, V, B, D, H, int(stable), _d(x), mask.ctypes.data_as(_u8p), _d(_f64(W)),
                              _d(_f64(Ru)), _d(_f64(Rv)), _d(_f64(b)), _d(h), _d(c), _d(act))
    assert rc == 0
    return dict(h=h, c=c, act=act)


def mdlstm_bwd(x, mask, W, Ru, Rv, fwd, dh, stable: bool):
    x = _f64(x)
    U, V, B, D = x.shape
    H = Ru.shape[0]
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    dx = np.zeros_like(x)
    dW = np.zeros((D, 5 * H)); dRu = np.zeros((H, 5 * H)); dRv = np.zeros((H, 5 * H)); db = np.zeros(5 * H)
    rc = lib().ref_mdlstm_bwd(U, V, B, D, H, int(stable), _d(x), mask.ctypes.data_as(_u8p), _d(_f64(W)),
                              _d(_f64(Ru)), _d(_f64(Rv)), _d(fwd["h"]), _d(fwd["c"]), _d(fwd["act"]),
                              _d(_f64(dh)), _d(dx), _d(dW), _d(dRu), _d(dRv), _d(db))
    assert rc == 0
    return dict(dx=dx, dW=dW, dRu=dRu, dRv=dRv, db=db)


def _flip(a, fu, fv):
    if fu:
        a = a[::-1]
    if fv:
        a = a[:, ::-1]
    return np.ascontiguousarray(a)


def mdlstm_multidir(x, mask, params, stable: bool):
    """Four directions: direction k runs on the grid flipped by MD_FLIPS[k], its
    output is flipped back; y [U,V,B,4H] = [y_0 | y_1 | y_2 | y_3].  params: 4 x (W, Ru, Rv, b)."""
    outs, fwds = [], []
    for (fu, fv), (W, Ru, Rv, b) in zip(MD_FLIPS, params):
        f = mdlstm_fwd(_flip(_f64(x), fu, fv), _flip(mask, fu, fv), W, Ru, Rv, b, stable)
        fwds.append(f)
        outs.append(_flip(f["h"], fu, fv))
    return np.concatenate(outs, axis=3), fwds


def mdlstm_multidir_bwd(x, mask, params, fwds, dy, stable: bool):
    """Gradients of sum(y * dy): dx (summed over the directions) and per-direction (dW, dRu, dRv, db)."""
    H = params[0][1].shape[0]
    dx = np.zeros(np.shape(x))
    grads = []
    for k, ((fu, fv), (W, Ru, Rv, b)) in enumerate(zip(MD_FLIPS, params)):
        g = mdlstm_bwd(_flip(_f64(x), fu, fv), _flip(mask, fu, fv), W, Ru, Rv, fwds[k],
                       _flip(_f64(dy)[..., k * H:(k + 1) * H], fu, fv), stable)
        dx += _flip(g["dx"], fu, fv)
        grads.append((g["dW"], g["dRu"], g["dRv"], g["db"]))
    return dx, grads
