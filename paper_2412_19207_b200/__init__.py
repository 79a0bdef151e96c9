"""B200-native (sm_100a, FP64) solve pipeline for the RaNN + overlapping-Schwarz method of
arXiv 2412.19207: a drop-in for the reference `rannddm` hot path (runner.hpp:202-275).

The product is the in-tree C-ABI library `librdd.so` (CUDA kernels in csrc/); `rdd.Solver` is
its Python binding, `configs` the named workloads, `abi` the struct mirrors.
"""
from . import abi, configs  # noqa: F401

__all__ = ["abi", "configs", "rdd"]
