"""Thin ctypes binding of libblstm.so (include/blstm.h): same names, argument
marshalling only.  Every step of the path runs in the library's CUDA kernels;
there is no Python or CPU fallback — a missing library raises.

Tensors are torch tensors (device memory is torch's); streams default to torch's
current stream.  Errors raise BlstmError with the library's error text.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libblstm.so")

BLSTM_NO_DX = 4
BLSTM_ACCUM_DX = 2
BLSTM_PREC_FP16 = 0
BLSTM_PREC_FP16X2W = 1  # the input projection with W split hi + lo (blstm.h)

_lib = None


class BlstmError(RuntimeError):
    def __init__(self, fn: str, code: int, msg: str):
        super().__init__(f"{fn} returned {code}: {msg}")
        self.code = code


class LstmDesc(ctypes.Structure):
    _fields_ = [("T", ctypes.c_int), ("B", ctypes.c_int), ("D", ctypes.c_int), ("H", ctypes.c_int),
                ("direction", ctypes.c_int), ("ldx", ctypes.c_int), ("ldy", ctypes.c_int),
                ("flags", ctypes.c_int), ("precision", ctypes.c_int)]


class StackDesc(ctypes.Structure):
    _fields_ = [("L", ctypes.c_int), ("D", ctypes.c_int), ("H", ctypes.c_int), ("K", ctypes.c_int),
                ("T", ctypes.c_int), ("B", ctypes.c_int), ("flags", ctypes.c_int),
                ("precision", ctypes.c_int), ("dropout", ctypes.c_float), ("dropout_seed", ctypes.c_uint32)]


class OptParams(ctypes.Structure):
    _fields_ = [("rule", ctypes.c_int), ("lr", ctypes.c_double), ("mu", ctypes.c_double), ("rho", ctypes.c_double),
                ("beta1", ctypes.c_double), ("beta2", ctypes.c_double), ("eps", ctypes.c_double),
                ("l2", ctypes.c_double), ("max_norm", ctypes.c_double), ("step", ctypes.c_long)]


# update rules (include/blstm.h BLSTM_OPT_*)
OPT_RULES = {"sgd": 0, "momentum": 1, "nesterov": 2, "adagrad": 3, "adadelta": 4, "adam": 5}

class MdDesc(ctypes.Structure):
    _fields_ = [("U", ctypes.c_int), ("V", ctypes.c_int), ("B", ctypes.c_int), ("D", ctypes.c_int),
                ("H", ctypes.c_int), ("stable", ctypes.c_int)]


_vp = ctypes.c_void_p
_sz = ctypes.c_size_t
_i = ctypes.c_int

_SIGS = {
    "blstm_last_error": (ctypes.c_char_p, []),
    "blstm_version": (_i, []),
    "blstm_check_errors": (_i, []),
    "lstm_workspace_bytes": (_sz, [ctypes.POINTER(LstmDesc)]),
    "lstm_reserve_bytes": (_sz, [ctypes.POINTER(LstmDesc)]),
    "lstm_fwd": (_i, [ctypes.POINTER(LstmDesc)] + [_vp] * 13 + [_sz, _vp]),
    "lstm_bwd": (_i, [ctypes.POINTER(LstmDesc)] + [_vp] * 18 + [_sz, _vp]),
    "blstm_param_count": (_sz, [ctypes.POINTER(StackDesc)]),
    "blstm_param_offsets": (_sz, [ctypes.POINTER(StackDesc), ctypes.POINTER(ctypes.c_size_t)]),
    "blstm_stack_workspace_bytes": (_sz, [ctypes.POINTER(StackDesc)]),
    "blstm_stack_fwd_bwd": (_i, [ctypes.POINTER(StackDesc)] + [_vp] * 10 + [_sz, _vp, _vp]),
    "blstm_stack_train_step": (_i, [ctypes.POINTER(StackDesc)] + [_vp] * 9 + [ctypes.POINTER(OptParams), _vp, _vp,
                                                                             _sz, _vp, _vp]),
    "blstm_stack_fwd": (_i, [ctypes.POINTER(StackDesc)] + [_vp] * 6 + [_sz, _vp]),
    "sgd_update": (_i, [_vp, _vp, _sz, ctypes.c_float, _i, _vp]),
    "blstm_opt_state_floats": (_sz, [_i, _sz]),
    "blstm_opt_workspace_bytes": (_sz, [_sz]),
    "blstm_opt_update": (_i, [ctypes.POINTER(OptParams), ctypes.POINTER(StackDesc), _vp, _vp, _vp, _sz, _i, _vp,
                              _sz, _vp]),
    "dp_get_unique_id": (_i, [ctypes.c_char_p]),
    "dp_comm_init": (_i, [_i, _i, ctypes.c_char_p, ctypes.POINTER(_vp)]),
    "dp_allreduce_grads": (_i, [_vp, _vp, _sz, _vp]),
    "dp_average_params": (_i, [_vp, _vp, _sz, _vp]),
    "dp_comm_destroy": (_i, [_vp]),
    "blstm_dp_buckets": (_i, [ctypes.POINTER(StackDesc), ctypes.POINTER(ctypes.c_size_t),
                              ctypes.POINTER(ctypes.c_size_t), _i]),
    "mdlstm_param_count": (_sz, [ctypes.POINTER(MdDesc)]),
    "mdlstm_workspace_bytes": (_sz, [ctypes.POINTER(MdDesc)]),
    "mdlstm_reserve_bytes": (_sz, [ctypes.POINTER(MdDesc)]),
    "mdlstm_fwd": (_i, [ctypes.POINTER(MdDesc)] + [_vp] * 6 + [_sz, _vp]),
    "mdlstm_bwd": (_i, [ctypes.POINTER(MdDesc)] + [_vp] * 8 + [_sz, _vp]),
    "blstm_gather_chunks": (_i, [_vp, _vp, _i, _vp, _vp, _i, _i, _vp, _vp, _vp, _vp]),
    "blstm_reduce_replicas": (_i, [ctypes.POINTER(ctypes.c_void_p), _i, _sz, ctypes.c_float, _vp]),
    "blstm_gemm_f16": (_i, [_i, _i, _i, _vp, ctypes.c_long, _i, _vp, ctypes.c_long, _i, _vp, ctypes.c_long,
                            ctypes.c_float, _i, _vp, _vp]),
    "blstm_launch_count": (ctypes.c_long, []),
    "blstm_profile_enable": (_i, [_i]),
    "blstm_profile_select": (_i, [_i]),
    "blstm_profile_read": (_i, [_i, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_long)]),
    "blstm_profile_timeline": (_i, [ctypes.POINTER(ctypes.c_double), _i]),
    "blstm_debug_set_trace": (_i, [_vp, _vp]),
}

PROF_REC_FWD, PROF_REC_BWD, PROF_GEMM = 0, 1, 2


def blstm_launch_count() -> int:
    return int(lib().blstm_launch_count())


def blstm_profile_enable(on):
    """on: False/0 off, True/1 recurrence + GEMM launches, 2 also helper kernels (timeline)."""
    _check("blstm_profile_enable", lib().blstm_profile_enable(int(on)))


def blstm_profile_select(cat_mask: int = -1):
    """Record only the launch categories whose bit is set (-1: all)."""
    _check("blstm_profile_select", lib().blstm_profile_select(int(cat_mask)))


def blstm_profile_read(cat: int):
    """(total device ms, launches) of one launch category since profiling was enabled."""
    ms = ctypes.c_double(0.0)
    n = ctypes.c_long(0)
    _check("blstm_profile_read", lib().blstm_profile_read(cat, ctypes.byref(ms), ctypes.byref(n)))
    return ms.value, n.value


def blstm_profile_timeline(max_recs: int = 4096):
    """[(cat, stream, t0_ms, t1_ms, a, b, c)] of the launches recorded since profiling was enabled."""
    buf = (ctypes.c_double * (7 * max_recs))()
    n = lib().blstm_profile_timeline(buf, max_recs)
    if n < 0:
        raise BlstmError("blstm_profile_timeline", n, last_error())
    return [tuple(buf[7 * i + k] for k in range(7)) for i in range(n)]


EXPORTS = tuple(_SIGS)


def lib():
    """Load libblstm.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                               "(the CUDA path has no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def blstm_check_errors():
    """Raises BlstmError if a kernel of a completed earlier call saw a mask entry outside {0,1}."""
    _check("blstm_check_errors", lib().blstm_check_errors())


def last_error() -> str:
    return lib().blstm_last_error().decode(errors="replace")


def _check(fn: str, rc: int):
    if rc != 0:
        raise BlstmError(fn, rc, last_error())


def _p(t) -> Optional[int]:
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _stream(s) -> Optional[int]:
    if s is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(s, int):
        return s
    return s.cuda_stream


def lstm_desc(T, B, D, H, direction=1, ldx=None, ldy=None, flags=0, precision=BLSTM_PREC_FP16) -> LstmDesc:
    return LstmDesc(T, B, D, H, direction, ldx or D, ldy or H, flags, precision)


def stack_desc(L, D, H, K, T, B, flags=0, precision=BLSTM_PREC_FP16, dropout=0.0, dropout_seed=0) -> StackDesc:
    return StackDesc(L, D, H, K, T, B, flags, precision, dropout, dropout_seed)


def lstm_workspace_bytes(desc: LstmDesc) -> int:
    n = lib().lstm_workspace_bytes(ctypes.byref(desc))
    if n == 0:
        raise BlstmError("lstm_workspace_bytes", -1, last_error())
    return n


def lstm_reserve_bytes(desc: LstmDesc) -> int:
    n = lib().lstm_reserve_bytes(ctypes.byref(desc))
    if n == 0:
        raise BlstmError("lstm_reserve_bytes", -1, last_error())
    return n


def lstm_fwd(desc, x, mask, W, R, b, h0, c0, y, c, hT, cT, reserve, workspace, stream=None):
    _check("lstm_fwd", lib().lstm_fwd(ctypes.byref(desc), _p(x), _p(mask), _p(W), _p(R), _p(b), _p(h0),
                                      _p(c0), _p(y), _p(c), _p(hT), _p(cT), _p(reserve), _p(workspace),
                                      workspace.numel() * workspace.element_size(), _stream(stream)))


def lstm_bwd(desc, x, mask, W, R, h0, c0, c, reserve, dy, dhT, dcT, dx, dW, dR, db, dh0, dc0, workspace,
             stream=None):
    _check("lstm_bwd", lib().lstm_bwd(ctypes.byref(desc), _p(x), _p(mask), _p(W), _p(R), _p(h0), _p(c0),
                                      _p(c), _p(reserve), _p(dy), _p(dhT), _p(dcT), _p(dx), _p(dW), _p(dR),
                                      _p(db), _p(dh0), _p(dc0), _p(workspace),
                                      workspace.numel() * workspace.element_size(), _stream(stream)))


def blstm_param_count(desc: StackDesc) -> int:
    return int(lib().blstm_param_count(ctypes.byref(desc)))


def blstm_param_offsets(desc: StackDesc):
    offs = (ctypes.c_size_t * (6 * desc.L + 2))()
    n = lib().blstm_param_offsets(ctypes.byref(desc), offs)
    return int(n), [int(v) for v in offs]


def blstm_stack_workspace_bytes(desc: StackDesc) -> int:
    n = lib().blstm_stack_workspace_bytes(ctypes.byref(desc))
    if n == 0:
        raise BlstmError("blstm_stack_workspace_bytes", -1, last_error())
    return n


def blstm_stack_fwd_bwd(desc, theta, grad, x, mask, labels, dy_top, loss_sum, frame_errors, comm, workspace,
                        s_main=None, s_side=None):
    sm = _stream(s_main)
    _check("blstm_stack_fwd_bwd", lib().blstm_stack_fwd_bwd(
        ctypes.byref(desc), _p(theta), _p(grad), _p(x), _p(mask), _p(labels), _p(dy_top), _p(loss_sum),
        _p(frame_errors), comm, _p(workspace), workspace.numel() * workspace.element_size(), sm,
        _stream(s_side) if s_side is not None else sm))


def blstm_stack_train_step(desc, theta, grad, x, mask, labels, dy_top, loss_sum, frame_errors, comm, opt: "OptParams",
                           opt_state, workspace, s_main=None, s_side=None):
    sm = _stream(s_main)
    _check("blstm_stack_train_step", lib().blstm_stack_train_step(
        ctypes.byref(desc), _p(theta), _p(grad), _p(x), _p(mask), _p(labels), _p(dy_top), _p(loss_sum),
        _p(frame_errors), comm, ctypes.byref(opt), _p(opt_state), _p(workspace),
        workspace.numel() * workspace.element_size(), sm, _stream(s_side) if s_side is not None else sm))


def blstm_stack_fwd(desc, theta, x, mask, Y, C, workspace, stream=None):
    _check("blstm_stack_fwd", lib().blstm_stack_fwd(
        ctypes.byref(desc), _p(theta), _p(x), _p(mask), _p(Y), _p(C), _p(workspace),
        workspace.numel() * workspace.element_size(), _stream(stream)))


def sgd_update(theta, grad, lr: float, zero_grad: bool = False, stream=None):
    _check("sgd_update", lib().sgd_update(_p(theta), _p(grad), theta.numel(), float(lr), int(zero_grad),
                                          _stream(stream)))


def opt_params(rule, lr, mu=0.9, rho=0.95, beta1=0.9, beta2=0.999, eps=1e-8, l2=0.0, max_norm=0.0,
               step=1) -> OptParams:
    r = OPT_RULES[rule] if isinstance(rule, str) else int(rule)
    return OptParams(r, lr, mu, rho, beta1, beta2, eps, l2, max_norm, step)


def blstm_opt_state_floats(rule, n: int) -> int:
    return int(lib().blstm_opt_state_floats(OPT_RULES[rule] if isinstance(rule, str) else int(rule), n))


def blstm_opt_workspace_bytes(n: int) -> int:
    return int(lib().blstm_opt_workspace_bytes(n))


def blstm_opt_update(params: OptParams, layout, theta, grad, state, zero_grad: bool, workspace, stream=None):
    """One update-rule step in place (theta, grad, state: fp32 DEVICE; layout: StackDesc or None)."""
    _check("blstm_opt_update", lib().blstm_opt_update(
        ctypes.byref(params), ctypes.byref(layout) if layout is not None else None, _p(theta), _p(grad),
        _p(state), theta.numel(), int(zero_grad), _p(workspace),
        workspace.numel() * workspace.element_size() if workspace is not None else 0, _stream(stream)))


def dp_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check("dp_get_unique_id", lib().dp_get_unique_id(buf))
    return buf.raw


def dp_comm_init(nranks: int, rank: int, uid: bytes):
    h = ctypes.c_void_p()
    _check("dp_comm_init", lib().dp_comm_init(nranks, rank, uid, ctypes.byref(h)))
    return h


def dp_allreduce_grads(comm, grad, stream=None):
    _check("dp_allreduce_grads", lib().dp_allreduce_grads(comm, _p(grad), grad.numel(), _stream(stream)))


def blstm_dp_buckets(desc: StackDesc):
    """[(lo, hi)] of the step's exchange buckets, in issue order (host-only)."""
    n = desc.L + 1
    lo, hi = (ctypes.c_size_t * n)(), (ctypes.c_size_t * n)()
    k = lib().blstm_dp_buckets(ctypes.byref(desc), lo, hi, n)
    if k < 0:
        raise BlstmError("blstm_dp_buckets", k, last_error())
    return [(int(lo[i]), int(hi[i])) for i in range(k)]


def dp_average_params(comm, theta, stream=None):
    _check("dp_average_params", lib().dp_average_params(comm, _p(theta), theta.numel(), _stream(stream)))


def mdlstm_desc(U, V, B, D, H, stable=False) -> MdDesc:
    return MdDesc(U, V, B, D, H, int(stable))


def mdlstm_sizes(desc: MdDesc):
    """(parameter count, workspace bytes, reserve bytes)."""
    L = lib()
    n, w, r = L.mdlstm_param_count(ctypes.byref(desc)), L.mdlstm_workspace_bytes(ctypes.byref(desc)), \
        L.mdlstm_reserve_bytes(ctypes.byref(desc))
    if n == 0:
        raise BlstmError("mdlstm_param_count", -1, last_error())
    return int(n), int(w), int(r)


def mdlstm_fwd(desc, theta, x, mask, y, reserve, workspace, stream=None):
    _check("mdlstm_fwd", lib().mdlstm_fwd(ctypes.byref(desc), _p(theta), _p(x), _p(mask), _p(y), _p(reserve),
                                          _p(workspace), workspace.numel() * workspace.element_size(),
                                          _stream(stream)))


def mdlstm_bwd(desc, theta, x, mask, reserve, dy, dx, grad, workspace, stream=None):
    _check("mdlstm_bwd", lib().mdlstm_bwd(ctypes.byref(desc), _p(theta), _p(x), _p(mask), _p(reserve), _p(dy), _p(dx),
                                          _p(grad), _p(workspace), workspace.numel() * workspace.element_size(),
                                          _stream(stream)))


def blstm_gather_chunks(frames, frame_labels, D: int, cstart, clen, B: int, T: int, x, mask, labels=None,
                        stream=None):
    _check("blstm_gather_chunks", lib().blstm_gather_chunks(_p(frames), _p(frame_labels), D, _p(cstart), _p(clen), B,
                                                            T, _p(x), _p(mask), _p(labels), _stream(stream)))


def blstm_reduce_replicas(tensors, scale: float, stream=None):
    """x_r <- scale * sum_q x_q for every tensor (all the same length, one device)."""
    arr = (ctypes.c_void_p * len(tensors))(*[t.data_ptr() for t in tensors])
    _check("blstm_reduce_replicas", lib().blstm_reduce_replicas(arr, len(tensors), tensors[0].numel(), float(scale),
                                                                  _stream(stream)))


def dp_comm_destroy(comm):
    _check("dp_comm_destroy", lib().dp_comm_destroy(comm))


def blstm_gemm_f16(A, a_mn: int, B, b_mn: int, C, M: int, N: int, K: int, alpha: float = 1.0,
                   beta: int = 0, bias=None, stream=None):
    """Test hook: C = alpha op(A) op(B)^T (+C) (+bias) on the tcgen05 GEMM."""
    _check("blstm_gemm_f16", lib().blstm_gemm_f16(M, N, K, _p(A), A.stride(0), a_mn, _p(B), B.stride(0), b_mn,
                                                  _p(C), C.stride(0), float(alpha), int(beta), _p(bias),
                                                  _stream(stream)))


def blstm_debug_set_trace(fwd=None, bwd=None):
    """Debug: per-step phase timestamps of the next recurrence launches (uint64 [T, 16] tensors)."""
    _check("blstm_debug_set_trace", lib().blstm_debug_set_trace(_p(fwd), _p(bwd)))
