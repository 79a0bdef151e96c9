"""ctypes binding of the C ABI (include/rdd.h) — the product's Python host layer.

Mirrors the reference's pipeline functions (runner.hpp:40-275, assembly.hpp, schwarz.hpp,
krylov.hpp) with the same names and argument meaning; errors are raised with the reference's
exception classes (ValueError for std::invalid_argument, RuntimeError for std::runtime_error,
ArithmeticError for std::domain_error). There is no CPU fallback: without the in-tree
librdd.so or without a CUDA device the constructor raises.
"""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np

from . import abi as A

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "librdd.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "rdd.h")

_lib = None


class DeviceError(RuntimeError):
    """CUDA failure or missing device (no reference analogue)."""


def exported_symbols() -> list[str]:
    """Function names declared in include/rdd.h."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(rdd_[a-z_]+)\s*\(", txt)))


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(f"{LIB_PATH} is missing: build it with __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        dp = C.POINTER(C.c_double)
        L.rdd_create.argtypes = [C.POINTER(vp), C.c_int]
        L.rdd_destroy.argtypes = [vp]
        L.rdd_last_error.restype = C.c_char_p
        L.rdd_last_error.argtypes = [vp]
        L.rdd_version.restype = C.c_char_p
        L.rdd_build_instance.argtypes = [vp, C.POINTER(A.Config), C.c_uint64]
        L.rdd_assemble.argtypes = [vp, C.c_int]
        L.rdd_build_preconditioner.argtypes = [vp, C.c_int]
        L.rdd_solve.argtypes = [vp, C.c_int, C.c_double, C.c_int, C.c_int]
        L.rdd_evaluate.argtypes = [vp, C.POINTER(C.c_int)]
        L.rdd_run_single.argtypes = [vp, C.POINTER(A.Config), C.c_uint64, C.POINTER(A.Summary)]
        L.rdd_get_summary.argtypes = [vp, C.POINTER(A.Summary)]
        L.rdd_rerun_resident.argtypes = [vp, C.POINTER(A.Summary)]
        L.rdd_launch_count.restype = C.c_int64
        L.rdd_launch_count.argtypes = []
        L.rdd_io_bytes.argtypes = [C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.rdd_event_record.argtypes = [vp, C.c_int]
        L.rdd_event_elapsed.argtypes = [vp, C.c_int, C.c_int, dp]
        i64 = C.c_int64
        L.rdd_matvec.argtypes = [vp, dp, i64, dp, i64]
        L.rdd_matvec_transpose.argtypes = [vp, dp, i64, dp, i64]
        L.rdd_normal_apply.argtypes = [vp, dp, i64, dp, i64]
        L.rdd_precond_apply.argtypes = [vp, dp, i64, dp, i64, C.c_int]
        L.rdd_get_i.restype = C.c_int64
        L.rdd_get_i.argtypes = [vp, C.c_char_p, C.c_int, C.POINTER(C.c_int32), C.c_int64]
        L.rdd_get_d.restype = C.c_int64
        L.rdd_get_d.argtypes = [vp, C.c_char_p, C.c_int, dp, C.c_int64]
        L.rdd_kernel_stats.argtypes = [vp, C.c_char_p, dp, C.POINTER(C.c_int64)]
        L.rdd_reset_stats.argtypes = [vp]
        L.rdd_set_timing.argtypes = [vp, C.c_int]
        L.rdd_set_verbose.argtypes = [vp, C.c_int]
        L.rdd_set_param.argtypes = [vp, C.c_char_p, C.c_double]
        L.rdd_bench_operator.argtypes = [vp, C.c_int, C.c_int, dp, dp]
        L.rdd_bench_precond.argtypes = [vp, C.c_int, C.c_int, dp, dp]
        L.rdd_bench_gemm.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, dp]
        L.rdd_bench_jacobi.argtypes = [vp, C.c_int, C.c_int, C.c_int, dp]
        L.rdd_spectra.argtypes = [vp, C.c_int, dp, dp, dp, dp, dp, dp]
        L.rdd_dense_spectrum.argtypes = [vp, i64, i64, dp, C.c_int, dp, dp]
        L.rdd_dense_singular_values.argtypes = [vp, i64, i64, dp, C.c_int, dp]
        L.rdd_dense_condition_number.argtypes = [vp, i64, i64, dp, C.c_int, dp]
        _lib = L
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


_EXC = {A.INVALID_ARGUMENT: ValueError, A.RUNTIME_ERROR: RuntimeError, A.DOMAIN_ERROR: ArithmeticError,
        A.CUDA_ERROR: DeviceError}


class Solver:
    """One device context: the reference's run_single pipeline, phase by phase."""

    def __init__(self, device: int = 0):
        self.L = lib()
        h = C.c_void_p()
        st = self.L.rdd_create(C.byref(h), device)
        if st != 0:
            raise DeviceError(f"rdd_create failed (status {st}): no usable CUDA device {device}")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.L.rdd_destroy(self.h)
            self.h = None

    __del__ = close

    def _check(self, st: int):
        if st != 0:
            raise _EXC.get(st, RuntimeError)(self.L.rdd_last_error(self.h).decode())

    # ---- pipeline (runner.hpp)
    def build_instance(self, cfg: A.Config, seed: int | None = None):
        self._check(self.L.rdd_build_instance(self.h, C.byref(cfg), cfg.seed if seed is None else seed))
        return self

    def assemble(self, equilibrate: bool = True):
        self._check(self.L.rdd_assemble(self.h, int(equilibrate)))
        return self

    def build_preconditioner(self, kind: int):
        self._check(self.L.rdd_build_preconditioner(self.h, kind))
        return self

    normal_blocks = None  # built inside build_preconditioner (assembly.hpp:148 + schwarz.hpp:93)

    def solve(self, solver: int, rel_tol: float, max_iter: int = 0, restart: int = 0):
        self._check(self.L.rdd_solve(self.h, solver, rel_tol, max_iter, restart))
        return self

    def evaluate(self, test_res):
        arr = (C.c_int * len(test_res))(*test_res)
        self._check(self.L.rdd_evaluate(self.h, arr))
        return self

    def run_single(self, cfg: A.Config, seed: int | None = None) -> dict:
        s = A.Summary()
        self._check(self.L.rdd_run_single(self.h, C.byref(cfg), cfg.seed if seed is None else seed, C.byref(s)))
        return s.as_dict()

    def rerun_resident(self) -> dict:
        """run_single again on the inputs already resident in HBM."""
        s = A.Summary()
        self._check(self.L.rdd_rerun_resident(self.h, C.byref(s)))
        return s.as_dict()

    def launch_count(self) -> int:
        return int(self.L.rdd_launch_count())

    def summary(self) -> dict:
        s = A.Summary()
        self.L.rdd_get_summary(self.h, C.byref(s))
        return s.as_dict()

    # ---- operators (LinearMap plug-ins)
    def matvec(self, w):
        w = np.ascontiguousarray(w, dtype=np.float64)
        y = np.zeros(self.geti("N")[0])
        self._check(self.L.rdd_matvec(self.h, _dp(w), w.size, _dp(y), y.size))
        return y

    def matvec_transpose(self, r):
        r = np.ascontiguousarray(r, dtype=np.float64)
        y = np.zeros(self.geti("p")[0])
        self._check(self.L.rdd_matvec_transpose(self.h, _dp(r), r.size, _dp(y), y.size))
        return y

    def normal_apply(self, w):
        w = np.ascontiguousarray(w, dtype=np.float64)
        y = np.zeros(self.geti("p")[0])
        self._check(self.L.rdd_normal_apply(self.h, _dp(w), w.size, _dp(y), y.size))
        return y

    def precond_apply(self, v, transpose: bool = False):
        v = np.ascontiguousarray(v, dtype=np.float64)
        z = np.zeros(self.geti("p")[0])
        self._check(self.L.rdd_precond_apply(self.h, _dp(v), v.size, _dp(z), z.size, int(transpose)))
        return z

    # ---- exports
    def geti(self, what: str, index: int = 0) -> np.ndarray:
        n = self.L.rdd_get_i(self.h, what.encode(), index, None, 0)
        if n < 0:
            raise ValueError(self.L.rdd_last_error(self.h).decode())
        out = np.zeros(n, dtype=np.int32)
        self.L.rdd_get_i(self.h, what.encode(), index, out.ctypes.data_as(C.POINTER(C.c_int32)), n)
        return out

    def getd(self, what: str, index: int = 0) -> np.ndarray:
        n = self.L.rdd_get_d(self.h, what.encode(), index, None, 0)
        if n < 0:
            raise ValueError(self.L.rdd_last_error(self.h).decode())
        out = np.zeros(n, dtype=np.float64)
        self.L.rdd_get_d(self.h, what.encode(), index, _dp(out), n)
        return out

    def block(self, j: int) -> np.ndarray:
        rows = len(self.geti("rows", j))
        return self.getd("H", j).reshape(-1, rows).T

    # ---- instrumentation
    def set_timing(self, on: bool):
        self.L.rdd_set_timing(self.h, int(on))

    def set_verbose(self, on: bool):
        self.L.rdd_set_verbose(self.h, int(on))

    def set_param(self, name: str, value: float):
        self._check(self.L.rdd_set_param(self.h, name.encode(), float(value)))

    def reset_stats(self):
        self.L.rdd_reset_stats(self.h)

    def kernel_stats(self, family: str):
        ms = C.c_double()
        n = C.c_int64()
        self.L.rdd_kernel_stats(self.h, family.encode(), C.byref(ms), C.byref(n))
        return ms.value, n.value

    def bench_jacobi(self, n: int, batch: int, sweeps: int) -> float:
        ms = C.c_double()
        self._check(self.L.rdd_bench_jacobi(self.h, n, batch, sweeps, C.byref(ms)))
        return ms.value

    # ---- dense diagnostics (krylov.hpp:403-440; runner.hpp:344-400)
    K_DENSE_SPECTRUM_CAP = 4000  # krylov.hpp:404

    def spectra(self, with_precond: bool = True, cap: int = 0):
        """spectrum_cmd's two spectra and sweep_tau's two condition numbers (runner.hpp:344-393)
        on the assembled system: (eig(HᵀH) ascending, eig(M⁻¹HᵀH) complex sorted by real part,
        cond(HᵀH), cond(M⁻¹HᵀH)). The preconditioned parts need build_preconditioner first."""
        p = int(self.geti("p")[0])
        nre, nim = np.zeros(p), np.zeros(p)
        pre, pim = np.zeros(p), np.zeros(p)
        cn, cp = np.zeros(1), np.zeros(1)
        wp = with_precond
        self._check(self.L.rdd_spectra(self.h, cap, _dp(nre), _dp(nim), _dp(pre) if wp else None,
                                       _dp(pim) if wp else None, _dp(cn), _dp(cp) if wp else None))
        return (nre + 1j * nim, (pre + 1j * pim) if wp else None, float(cn[0]), float(cp[0]) if wp else None)

    @staticmethod
    def _fortran(a):
        a = np.asarray(a, dtype=np.float64)
        if a.ndim != 2:
            raise ValueError("dense diagnostics: matrix must be 2-D")
        return np.asfortranarray(a)

    def spectrum(self, a, cap: int = 0) -> np.ndarray:
        """krylov.hpp:413 spectrum: all eigenvalues, sorted by (real, imag)."""
        a = self._fortran(a)
        n = a.shape[0]
        wr, wi = np.zeros(n), np.zeros(n)
        self._check(self.L.rdd_dense_spectrum(self.h, a.shape[0], a.shape[1], _dp(a), cap, _dp(wr), _dp(wi)))
        return wr + 1j * wi

    def singular_values(self, a, cap: int = 0) -> np.ndarray:
        """krylov.hpp:423 singular_values: non-increasing."""
        a = self._fortran(a)
        s = np.zeros(min(a.shape))
        self._check(self.L.rdd_dense_singular_values(self.h, a.shape[0], a.shape[1], _dp(a), cap, _dp(s)))
        return s

    def condition_number(self, a, cap: int = 0) -> float:
        """krylov.hpp:430 condition_number: σmax / smallest positive σ."""
        a = self._fortran(a)
        k = C.c_double()
        self._check(self.L.rdd_dense_condition_number(self.h, a.shape[0], a.shape[1], _dp(a), cap, C.byref(k)))
        return k.value

    def bench_operator(self, op_form: int, reps: int = 20):
        ms = C.c_double()
        by = C.c_double()
        self._check(self.L.rdd_bench_operator(self.h, op_form, reps, C.byref(ms), C.byref(by)))
        return ms.value, by.value

    def bench_gemm(self, mode: int, M: int, N: int, K: int, batch: int = 1, reps: int = 5) -> float:
        ms = C.c_double()
        self._check(self.L.rdd_bench_gemm(self.h, mode, M, N, K, batch, reps, C.byref(ms)))
        return ms.value

    def bench_precond(self, transpose: bool = False, reps: int = 20):
        ms = C.c_double()
        by = C.c_double()
        self._check(self.L.rdd_bench_precond(self.h, int(transpose), reps, C.byref(ms), C.byref(by)))
        return ms.value, by.value
