"""B200-native PaReprop training engine (arxiv 2306.09342).

Host C++ + hand-written sm_100a CUDA kernels behind the C ABI in include/revprop_b200.h.
The Python modules are thin ctypes front ends used by the tests and the benchmark.
"""
__all__ = ["build", "_capi"]
