"""TEST INFRASTRUCTURE ONLY — ctypes wrapper for the reference itself (oracle/_ref/libref.so).

oracle/_ref/libref.so is the UNMODIFIED reference (header-only C++, /root/reference/proj/include)
compiled here against the Eigen-subset shim (oracle/eigen_shim/) by oracle/ref/Makefile. It runs
the reference's own run_single and phase functions for configurations its RunConfig expresses
(example1/2/3, reference decomposition, absolute or no PCA threshold). Only tests/ and bench.py's
CPU legs load it; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)
from paper_2412_19207_b200 import abi as A  # noqa: E402
from oracle import lapack_path  # noqa: E402

LIB_PATH = os.path.join(HERE, "_ref", "libref.so")
_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        os.environ.setdefault("RDD_LAPACK_PATH", lapack_path())
        L = C.CDLL(LIB_PATH)
        vp, dp = C.c_void_p, C.POINTER(C.c_double)
        L.ref_create.restype = vp
        L.ref_destroy.argtypes = [vp]
        L.ref_last_error.restype = C.c_char_p
        L.ref_last_error.argtypes = [vp]
        L.ref_run_single.argtypes = [vp, C.POINTER(A.Config), C.c_uint64, C.POINTER(A.Summary)]
        L.ref_build.argtypes = [vp, C.POINTER(A.Config), C.c_uint64, C.c_int]
        L.ref_run_baseline.argtypes = [vp, C.POINTER(A.Config), C.c_uint64, C.POINTER(A.Summary)]
        L.ref_matvec.argtypes = [vp, dp, dp]
        L.ref_matvec_transpose.argtypes = [vp, dp, dp]
        L.ref_precond_apply.argtypes = [vp, dp, dp, C.c_int]
        L.ref_get_i.restype = C.c_int64
        L.ref_get_i.argtypes = [vp, C.c_char_p, C.c_int, C.POINTER(C.c_int32), C.c_int64]
        L.ref_get_d.restype = C.c_int64
        L.ref_get_d.argtypes = [vp, C.c_char_p, C.c_int, dp, C.c_int64]
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class Reference:
    """The reference's run_single and phases (runner.hpp:40-275) on the reference's own code."""

    def __init__(self):
        self.L = lib()
        self.h = self.L.ref_create()

    def close(self):
        if self.h:
            self.L.ref_destroy(self.h)
            self.h = None

    __del__ = close

    def _check(self, st):
        if st != 0:
            msg = self.L.ref_last_error(self.h).decode()
            raise {1: ValueError, 2: RuntimeError, 3: ArithmeticError}.get(st, RuntimeError)(msg)

    def run_single(self, cfg, seed=None) -> dict:
        s = A.Summary()
        self._check(self.L.ref_run_single(self.h, C.byref(cfg), cfg.seed if seed is None else seed, C.byref(s)))
        return s.as_dict()

    def run_baseline(self, cfg, seed=None) -> dict:
        """run_single for a BASELINE configuration (C1-C5 problems, cell decomposition, relative
        τ, edge points) on the reference's own functions and types (oracle/ref/ref_capi.cpp)."""
        s = A.Summary()
        self._check(self.L.ref_run_baseline(self.h, C.byref(cfg), cfg.seed if seed is None else seed, C.byref(s)))
        return s.as_dict()

    def build(self, cfg, precond=A.PRECOND_AS, seed=None):
        self._check(self.L.ref_build(self.h, C.byref(cfg), cfg.seed if seed is None else seed, precond))
        return self

    def geti(self, what, index=0):
        n = self.L.ref_get_i(self.h, what.encode(), index, None, 0)
        if n < 0:
            raise ValueError(self.L.ref_last_error(self.h).decode())
        out = np.zeros(n, dtype=np.int32)
        self.L.ref_get_i(self.h, what.encode(), index, out.ctypes.data_as(C.POINTER(C.c_int32)), n)
        return out

    def getd(self, what, index=0):
        n = self.L.ref_get_d(self.h, what.encode(), index, None, 0)
        if n < 0:
            raise ValueError(self.L.ref_last_error(self.h).decode())
        out = np.zeros(n)
        self.L.ref_get_d(self.h, what.encode(), index, _dp(out), n)
        return out

    def matvec(self, w):
        w = np.ascontiguousarray(w, dtype=np.float64)
        N = len(self.getd("F"))
        y = np.zeros(N)
        self._check(self.L.ref_matvec(self.h, _dp(w), _dp(y)))
        return y

    def matvec_transpose(self, r):
        r = np.ascontiguousarray(r, dtype=np.float64)
        y = np.zeros(int(self.geti("p")[0]))
        self._check(self.L.ref_matvec_transpose(self.h, _dp(r), _dp(y)))
        return y

    def precond_apply(self, v, transpose=False):
        v = np.ascontiguousarray(v, dtype=np.float64)
        z = np.zeros_like(v)
        self._check(self.L.ref_precond_apply(self.h, _dp(v), _dp(z), int(transpose)))
        return z
