"""TEST INFRASTRUCTURE ONLY — ctypes wrapper for the CPU oracle (oracle/liboracle.so).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import glob
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from paper_2412_19207_b200 import abi as A  # noqa: E402

LIB_PATH = os.path.join(HERE, "liboracle.so")


def lapack_path() -> str:
    """Locate scipy's bundled OpenBLAS (LP64, `scipy_` symbol prefix)."""
    import importlib.util
    spec = importlib.util.find_spec("scipy")
    roots = [os.path.dirname(os.path.dirname(spec.origin))] if spec and spec.origin else []
    for r in roots:
        hits = sorted(glob.glob(os.path.join(r, "scipy.libs", "libscipy_openblas-*.so")))
        if hits:
            return hits[0]
    raise RuntimeError("scipy's bundled OpenBLAS not found")


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-C", HERE, "-s"], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB_PATH)
        L.orc_create.restype = C.c_void_p
        L.orc_create.argtypes = [C.c_char_p, C.c_int]
        L.orc_destroy.argtypes = [C.c_void_p]
        L.orc_last_error.restype = C.c_char_p
        L.orc_last_error.argtypes = [C.c_void_p]
        for n in ("orc_build_instance", "orc_run_single"):
            getattr(L, n).restype = C.c_int
        L.orc_build_instance.argtypes = [C.c_void_p, C.POINTER(A.Config), C.c_uint64]
        L.orc_run_single.argtypes = [C.c_void_p, C.POINTER(A.Config), C.c_uint64, C.POINTER(A.Summary)]
        L.orc_assemble.argtypes = [C.c_void_p, C.c_int]
        L.orc_build_preconditioner.argtypes = [C.c_void_p, C.c_int]
        L.orc_normal_blocks.argtypes = [C.c_void_p]
        L.orc_solve.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int]
        L.orc_evaluate.argtypes = [C.c_void_p, C.POINTER(C.c_int)]
        L.orc_get_summary.argtypes = [C.c_void_p, C.POINTER(A.Summary)]
        dp = C.POINTER(C.c_double)
        L.orc_matvec.argtypes = [C.c_void_p, dp, dp]
        L.orc_matvec_transpose.argtypes = [C.c_void_p, dp, dp]
        L.orc_precond_apply.argtypes = [C.c_void_p, dp, dp, C.c_int]
        L.orc_spectra.argtypes = [C.c_void_p, dp, dp, dp, dp]
        L.orc_get_i.restype = C.c_int64
        L.orc_get_i.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.POINTER(C.c_int32), C.c_int64]
        L.orc_get_d.restype = C.c_int64
        L.orc_get_d.argtypes = [C.c_void_p, C.c_char_p, C.c_int, dp, C.c_int64]
        L.orc_max_threads.restype = C.c_int
        L.orc_set_option.restype = C.c_int
        L.orc_set_option.argtypes = [C.c_char_p, C.c_int]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class Oracle:
    """Pipeline handle mirroring the reference's run_single phases (runner.hpp:202-275)."""

    def __init__(self, threads: int = 0):
        self.L = lib()
        self.h = self.L.orc_create(lapack_path().encode(), threads)
        if not self.h:
            raise OracleError("orc_create failed")

    @staticmethod
    def set_option(name: str, value: int):
        """Fixture-generation switches: 'parallel_pca' (independent per-subdomain PCAs run
        concurrently), 'keep_samples' (keep the unreduced sample matrices)."""
        if lib().orc_set_option(name.encode(), int(value)) != 0:
            raise OracleError(f"unknown oracle option {name}")

    def close(self):
        if self.h:
            self.L.orc_destroy(self.h)
            self.h = None

    __del__ = close

    def _check(self, st: int):
        if st != 0:
            msg = self.L.orc_last_error(self.h).decode()
            exc = {1: ValueError, 2: RuntimeError, 3: ArithmeticError}.get(st, OracleError)
            raise exc(msg)

    # ---- pipeline
    def build_instance(self, cfg: A.Config, seed: int | None = None):
        self._check(self.L.orc_build_instance(self.h, C.byref(cfg), cfg.seed if seed is None else seed))
        return self

    def assemble(self, equilibrate: bool = True):
        self._check(self.L.orc_assemble(self.h, int(equilibrate)))
        return self

    def build_preconditioner(self, kind: int):
        self._check(self.L.orc_build_preconditioner(self.h, kind))
        return self

    def normal_blocks(self):
        self._check(self.L.orc_normal_blocks(self.h))
        return self

    def solve(self, solver: int, rel_tol: float, max_iter: int = 0, restart: int = 0, true_residual: bool = True):
        self._check(self.L.orc_solve(self.h, solver, rel_tol, max_iter, restart, int(true_residual)))
        return self

    def evaluate(self, test_res):
        arr = (C.c_int * len(test_res))(*test_res)
        self._check(self.L.orc_evaluate(self.h, arr))
        return self

    def run_single(self, cfg: A.Config, seed: int | None = None) -> dict:
        s = A.Summary()
        self._check(self.L.orc_run_single(self.h, C.byref(cfg), cfg.seed if seed is None else seed, C.byref(s)))
        return s.as_dict()

    def summary(self) -> dict:
        s = A.Summary()
        self.L.orc_get_summary(self.h, C.byref(s))
        return s.as_dict()

    # ---- operators
    def matvec(self, w):
        w = np.ascontiguousarray(w, dtype=np.float64)
        y = np.zeros(self.geti("N")[0])
        self._check(self.L.orc_matvec(self.h, _dp(w), _dp(y)))
        return y

    def matvec_transpose(self, r):
        r = np.ascontiguousarray(r, dtype=np.float64)
        y = np.zeros(self.geti("p")[0])
        self._check(self.L.orc_matvec_transpose(self.h, _dp(r), _dp(y)))
        return y

    def precond_apply(self, v, transpose: bool = False):
        v = np.ascontiguousarray(v, dtype=np.float64)
        z = np.zeros_like(v)
        self._check(self.L.orc_precond_apply(self.h, _dp(v), _dp(z), int(transpose)))
        return z

    def spectra(self, with_precond: bool = True):
        p = self.geti("p")[0]
        normal = np.zeros(p)
        pre = np.zeros(p)
        cn = np.zeros(1)
        cp = np.zeros(1)
        self._check(self.L.orc_spectra(self.h, _dp(normal), _dp(pre) if with_precond else None, _dp(cn),
                                       _dp(cp) if with_precond else None))
        return normal, pre, float(cn[0]), float(cp[0])

    # ---- exports
    def geti(self, what: str, index: int = 0) -> np.ndarray:
        n = self.L.orc_get_i(self.h, what.encode(), index, None, 0)
        if n < 0:
            raise OracleError(self.L.orc_last_error(self.h).decode())
        out = np.zeros(n, dtype=np.int32)
        self.L.orc_get_i(self.h, what.encode(), index, out.ctypes.data_as(C.POINTER(C.c_int32)), n)
        return out

    def getd(self, what: str, index: int = 0) -> np.ndarray:
        n = self.L.orc_get_d(self.h, what.encode(), index, None, 0)
        if n < 0:
            raise OracleError(self.L.orc_last_error(self.h).decode())
        out = np.zeros(n, dtype=np.float64)
        self.L.orc_get_d(self.h, what.encode(), index, _dp(out), n)
        return out

    def block(self, j: int) -> np.ndarray:
        """H_j as a (rows_j, p_j) array (column-major storage)."""
        rows = len(self.geti("rows", j))
        return self.getd("H", j).reshape(-1, rows).T

    def V(self, j: int) -> np.ndarray:
        m = self.geti("J") and None
        v = self.getd("V", j)
        pj = int(self.geti("p_j")[j])
        return v.reshape(pj, -1).T
