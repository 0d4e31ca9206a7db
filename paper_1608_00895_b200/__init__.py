"""B200-native (sm_100a) fused BLSTM training hot path of RETURNN (arXiv:1608.00895).

The compute lives in the C-ABI library ``libblstm.so`` (csrc/, declared in
include/blstm.h); ``paper_1608_00895_b200.blstm`` is the thin ctypes binding.
Importing this package does not load CUDA; the binding loads the library on
first use and raises if it is missing (there is no CPU fallback).
"""
__all__ = ["blstm", "synth"]
