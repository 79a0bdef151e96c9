"""ctypes mirror of include/rdd.h (config/summary structs and constants).

The structs mirror rannddm::RunConfig (config.hpp:23-68) and RunSummary (runner.hpp:147-156);
`configs.py` holds the named workloads (BASELINE.json C1..C5 and the reference's golden cases).
"""
from __future__ import annotations

import ctypes as C

OK, INVALID_ARGUMENT, RUNTIME_ERROR, DOMAIN_ERROR, CUDA_ERROR = 0, 1, 2, 3, 4

PROBLEM_EXAMPLE1, PROBLEM_EXAMPLE2, PROBLEM_EXAMPLE3 = 1, 2, 3
PROBLEM_POISSON, PROBLEM_MULTISCALE, PROBLEM_HEAT, PROBLEM_ADVECTION = 10, 11, 12, 13
PROBLEM_DIM = {1: 2, 2: 2, 3: 3, 11: 2, 12: 3, 13: 2}

DECOMP_REFERENCE, DECOMP_CELL = 0, 1
TAU_OFF, TAU_ABSOLUTE, TAU_RELATIVE = 0, 1, 2
PCA_PSI, PCA_OP_APPLIED = 0, 1
SOLVER_QR, SOLVER_CG, SOLVER_CGS, SOLVER_BICG, SOLVER_GMRES = 0, 1, 2, 3, 4
PRECOND_NONE, PRECOND_AS, PRECOND_SAS, PRECOND_RAS = -1, 0, 1, 2
OPERATOR_TWO_PASS, OPERATOR_NORMAL = 0, 1

SOLVER_NAMES = {0: "qr_direct", 1: "cg", 2: "cgs", 3: "bicg", 4: "gmres"}
PRECOND_NAMES = {-1: "none", 0: "AS", 1: "SAS", 2: "RAS"}


class Config(C.Structure):
    _fields_ = [
        ("problem", C.c_int),
        ("n", C.c_int),
        ("dim", C.c_int),
        ("counts", C.c_int * 4),
        ("decomposition", C.c_int),
        ("delta", C.c_double),
        ("m", C.c_int),
        ("activation", C.c_int),
        ("seed", C.c_uint64),
        ("colloc", C.c_int * 4),
        ("boundary_per_edge", C.c_int),
        ("test", C.c_int * 4),
        ("tau_mode", C.c_int),
        ("tau", C.c_double),
        ("pca_matrix", C.c_int),
        ("solver", C.c_int),
        ("precond", C.c_int),
        ("rel_tol", C.c_double),
        ("max_iter", C.c_int),
        ("gmres_restart", C.c_int),
        ("op_form", C.c_int),
        ("true_residual", C.c_int),
        ("ref_resolution", C.c_int),
    ]

    @property
    def d(self) -> int:
        return self.dim or PROBLEM_DIM.get(self.problem, 2)

    def as_dict(self) -> dict:
        d = self.d
        return {
            "problem": self.problem, "n": self.n, "dim": d,
            "counts": list(self.counts)[:d], "decomposition": self.decomposition,
            "delta": self.delta, "m": self.m, "activation": self.activation, "seed": self.seed,
            "colloc": list(self.colloc)[:d], "boundary_per_edge": self.boundary_per_edge,
            "test": list(self.test)[:d], "tau_mode": self.tau_mode, "tau": self.tau,
            "pca_matrix": self.pca_matrix, "solver": SOLVER_NAMES[self.solver],
            "precond": PRECOND_NAMES[self.precond], "rel_tol": self.rel_tol,
            "max_iter": self.max_iter, "gmres_restart": self.gmres_restart,
            "op_form": self.op_form, "true_residual": self.true_residual, "ref_resolution": self.ref_resolution,
        }


class Summary(C.Structure):
    _fields_ = [
        ("seed", C.c_uint64),
        ("J", C.c_int), ("DoF", C.c_int), ("N", C.c_int), ("p", C.c_int),
        ("iterations", C.c_int), ("converged", C.c_int), ("breakdown", C.c_int),
        ("e_l2", C.c_double), ("e_l1n", C.c_double),
        ("t_assemble", C.c_double), ("t_precond", C.c_double), ("t_solve", C.c_double),
        ("t_evaluate", C.c_double), ("t_pca", C.c_double), ("final_residual", C.c_double),
    ]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


def make_config(problem: int, counts, m: int, colloc, *, n: int = 2, dim: int = 0,
                decomposition: int = DECOMP_REFERENCE, delta: float = 2.0, activation: int = 0,
                seed: int = 1000, boundary_per_edge: int = 0, test=None, tau_mode: int = TAU_OFF,
                tau: float = 0.0, pca_matrix: int = PCA_OP_APPLIED, solver: int = SOLVER_GMRES,
                precond: int = PRECOND_AS, rel_tol: float = 1e-5, max_iter: int = 0,
                gmres_restart: int = 0, op_form: int = OPERATOR_TWO_PASS,
                true_residual: int = 1, ref_resolution: int = 0) -> Config:
    """Build a Config; defaults follow RunConfig (config.hpp:23-68)."""
    c = Config()
    c.problem = problem
    c.n = n
    c.dim = dim or PROBLEM_DIM.get(problem, len(counts))
    for i, v in enumerate(counts):
        c.counts[i] = v
    c.decomposition = decomposition
    c.delta = delta
    c.m = m
    c.activation = activation
    c.seed = seed
    for i, v in enumerate(colloc):
        c.colloc[i] = v
    c.boundary_per_edge = boundary_per_edge
    for i, v in enumerate(test if test is not None else [350] * len(counts)):
        c.test[i] = v
    c.tau_mode = tau_mode
    c.tau = tau
    c.pca_matrix = pca_matrix
    c.solver = solver
    c.precond = precond
    c.rel_tol = rel_tol
    c.max_iter = max_iter
    c.gmres_restart = gmres_restart
    c.op_form = op_form
    c.true_residual = true_residual
    c.ref_resolution = ref_resolution
    return c
