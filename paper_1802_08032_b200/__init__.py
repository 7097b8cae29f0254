"""B200-native QuEST-style backend for the state-vector / density-matrix gate
path of arxiv/paper_1802_08032 (the QuEST paper; reference: a C++20 CPU
re-implementation under /root/reference/proj).

The product is the C-ABI shared library ``_lib/libqgpu.so`` (include/QuEST.h,
include/qgpu.h): hand-written sm_100a kernels over complex-double amplitudes in
HBM, a C++ runtime that fuses queued gates into HBM passes, and an NCCL
exchange engine. ``quest`` binds it with ctypes; ``qsim`` mirrors the
reference's C++ operation names on top; ``circuits`` holds the workloads.
"""
from . import circuits  # noqa: F401  (pure Python)

__all__ = ["circuits", "quest", "qsim", "build"]
