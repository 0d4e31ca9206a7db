"""Build libblstm.so (all CUDA sources, sm_100a) in-tree.  Used by __graft_entry__.build()."""
import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.dirname(HERE)
ROOT = os.path.dirname(PKG)
SOURCES = ["api.cu", "gemm.cu", "lstm_rec.cu", "rec_step.cu", "mdlstm.cu", "graph.cu", "ops.cu", "optim.cu", "dp.cu", "prof.cu"]
OUT = os.path.join(PKG, "libblstm.so")


def nccl_dir():
    for base in sys.path + [sysconfig.get_paths()["purelib"]]:
        d = os.path.join(base, "nvidia", "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("nccl headers not found (expected site-packages/nvidia/nccl)")


def build(force: bool = False, verbose: bool = False, trace: bool = False) -> str:
    """trace=True adds -DBLSTM_TRACE (per-step phase timestamps, scripts/trace_rec.py)."""
    srcs = [os.path.join(HERE, s) for s in SOURCES]
    deps = srcs + [os.path.join(HERE, h) for h in os.listdir(HERE) if h.endswith((".h", ".cuh"))]
    deps.append(os.path.join(ROOT, "include", "blstm.h"))
    if not force and os.path.exists(OUT) and os.path.getmtime(OUT) >= max(os.path.getmtime(p) for p in deps):
        return OUT
    nd = nccl_dir()
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    tmp = OUT + f".tmp{os.getpid()}"
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
           "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nd, "include"),
           "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2",
           "-Xlinker", "-rpath=" + os.path.join(nd, "lib"),
           "-o", tmp] + srcs
    for f in os.environ.get("BLSTM_NVCC_EXTRA", "").split():  # experiment builds (e.g. -DBLSTM_WAIT_HINT_NS=0)
        cmd.insert(1, f)
    if trace:
        cmd.insert(1, "-DBLSTM_TRACE")
        if os.environ.get("BLSTM_TRACE_CTA"):  # trace another CTA than 0 (e.g. 1: an odd pair CTA)
            cmd.insert(1, "-DBLSTM_TRACE_CTA=" + str(int(os.environ["BLSTM_TRACE_CTA"])))
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd)
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, trace="--trace" in sys.argv))
