"""CPU-side checks of the C-ABI library: it loads without a GPU, exports every
function include/blstm.h declares, and its flat-theta layout agrees with the
oracle's independently computed layout (the layout is an interface contract,
stated in the header; each side implements it on its own)."""
import os
import re

import numpy as np
import pytest

import oracle
from paper_1608_00895_b200 import blstm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "blstm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b([a-z_][a-z0-9_]*)\s*\(", src, flags=re.M)
    return sorted(set(n for n in names if n not in ("if", "sizeof")))


def test_header_declares_expected_boundary():
    names = _declared_functions()
    for n in ("lstm_fwd", "lstm_bwd", "blstm_stack_fwd_bwd", "dp_average_params", "dp_allreduce_grads",
              "sgd_update", "blstm_param_offsets", "lstm_workspace_bytes", "lstm_reserve_bytes",
              "blstm_opt_update", "blstm_opt_state_floats", "blstm_opt_workspace_bytes"):
        assert n in names, n


def test_library_loads_and_exports_every_declared_symbol():
    L = blstm.lib()
    for n in _declared_functions():
        assert hasattr(L, n), f"libblstm.so does not export {n}"
    assert set(_declared_functions()) == set(blstm.EXPORTS)
    assert L.blstm_version() >= 100


@pytest.mark.parametrize("L,D,H,K", [(5, 40, 500, 1501), (1, 4, 8, 0), (3, 3, 5, 7), (4, 40, 1024, 1501)])
def test_param_layout_matches_oracle(L, D, H, K):
    desc = blstm.stack_desc(L, D, H, K, 10, 2)
    n, offs = blstm.blstm_param_offsets(desc)
    n_o, offs_o = oracle.param_offsets(L, D, H, K)
    assert n == n_o == blstm.blstm_param_count(desc)
    assert list(offs) == [int(v) for v in offs_o]


def test_invalid_arguments_fail_before_any_launch():
    # argument checks run on the host; no GPU is touched
    bad = blstm.lstm_desc(T=4, B=2, D=3, H=5, direction=0)
    with pytest.raises(blstm.BlstmError):
        blstm.lstm_workspace_bytes(bad)
    assert "direction" in blstm.last_error()
    bad = blstm.lstm_desc(T=4, B=0, D=3, H=5)
    with pytest.raises(blstm.BlstmError):
        blstm.lstm_reserve_bytes(bad)


def test_no_cpu_fallback_when_library_missing(monkeypatch, tmp_path):
    monkeypatch.setattr(blstm, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(blstm, "_lib", None)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        blstm.lib()


def test_opt_state_sizes():
    for n in (0, 1, 4, 5, 1001):
        n4 = (n + 3) // 4 * 4
        assert blstm.blstm_opt_state_floats("sgd", n) == 0
        for r in ("momentum", "nesterov", "adagrad"):
            assert blstm.blstm_opt_state_floats(r, n) == n4
        for r in ("adadelta", "adam"):
            assert blstm.blstm_opt_state_floats(r, n) == 2 * n4
    assert blstm.blstm_opt_workspace_bytes(10) >= 8


def test_opt_update_rejects_bad_arguments():
    """Host-side validation of blstm_opt_update returns an error code before any launch."""
    import ctypes
    L = blstm.lib()
    fake = ctypes.c_void_p(1 << 20)  # aligned, never dereferenced (validation fails first)
    P = blstm.opt_params("adam", 0.1, step=0)
    assert L.blstm_opt_update(ctypes.byref(P), None, fake, fake, fake, 16, 0, None, 0, None) != 0
    assert "step" in blstm.last_error()
    P = blstm.opt_params(9, 0.1)
    assert L.blstm_opt_update(ctypes.byref(P), None, fake, fake, fake, 16, 0, None, 0, None) != 0
    P = blstm.opt_params("momentum", 0.1)
    assert L.blstm_opt_update(ctypes.byref(P), None, fake, fake, None, 16, 0, None, 0, None) != 0  # no state
    assert L.blstm_opt_update(ctypes.byref(P), None, ctypes.c_void_p((1 << 20) + 4), fake, fake, 16, 0, None, 0,
                              None) != 0  # misaligned theta
    P = blstm.opt_params("sgd", 0.1, max_norm=1.0)
    assert L.blstm_opt_update(ctypes.byref(P), None, fake, fake, None, 16, 0, None, 0, None) != 0  # no workspace
    d = blstm.stack_desc(2, 3, 5, 7, 4, 2)
    P = blstm.opt_params("sgd", 0.1)
    n = blstm.blstm_param_count(d)
    assert L.blstm_opt_update(ctypes.byref(P), ctypes.byref(d), fake, fake, None, n + 1, 0, None, 0, None) != 0
    assert L.blstm_opt_update(ctypes.byref(P), None, fake, fake, None, 0, 0, None, 0, None) == 0  # n = 0: no-op
