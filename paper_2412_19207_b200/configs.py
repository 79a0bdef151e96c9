"""Named workloads.

BASELINE.json configs C1..C5 mapped onto reference-compatible inputs as SURVEY §8d specifies
(cell-centred boxes extended by 10% of their width per side; global cell-centred grid with
P points per subdomain per axis; relative PCA threshold 1e-6 on the operator-applied sample
matrix; column equilibration on). The golden cases reproduce the configurations that produced
the reference's committed artefacts (proj/h_export.txt, runner_out*/, schwarz_diag.csv).
"""
from __future__ import annotations

from . import abi as A


def c1(**kw) -> A.Config:
    """2-D Poisson, 4x4 subdomains, m=200, 40x40 per subdomain + 4x160 boundary points."""
    args = dict(decomposition=A.DECOMP_CELL, delta=0.1, boundary_per_edge=160, test=[350, 350],
                tau_mode=A.TAU_RELATIVE, tau=1e-6, pca_matrix=A.PCA_OP_APPLIED,
                solver=A.SOLVER_CG, precond=A.PRECOND_AS, rel_tol=1e-10, seed=1000, op_form=A.OPERATOR_TWO_PASS)
    args.update(kw)
    return A.make_config(A.PROBLEM_POISSON, [4, 4], 200, [160, 160], dim=2, **args)


def c2(**kw) -> A.Config:
    """2-D multiscale Poisson, 16x16 subdomains, m=300, 60x60 per subdomain (0.92M rows)."""
    args = dict(decomposition=A.DECOMP_CELL, delta=0.1, test=[350, 350], tau_mode=A.TAU_RELATIVE,
                tau=1e-6, pca_matrix=A.PCA_OP_APPLIED, solver=A.SOLVER_CG, precond=A.PRECOND_AS,
                rel_tol=1e-10, seed=1000, op_form=A.OPERATOR_TWO_PASS)
    args.update(kw)
    return A.make_config(A.PROBLEM_MULTISCALE, [16, 16], 300, [960, 960], **args)


def c3(**kw) -> A.Config:
    """2-D heat equation in space-time, 8x8x8 subdomains, m=300, 16^3 per subdomain; RAS-GMRES(50)."""
    args = dict(decomposition=A.DECOMP_CELL, delta=0.1, test=[50, 50, 50], tau_mode=A.TAU_RELATIVE,
                tau=1e-6, pca_matrix=A.PCA_OP_APPLIED, solver=A.SOLVER_GMRES, precond=A.PRECOND_RAS,
                gmres_restart=50, rel_tol=1e-10, seed=1000, op_form=A.OPERATOR_TWO_PASS)
    args.update(kw)
    return A.make_config(A.PROBLEM_HEAT, [8, 8, 8], 300, [128, 128, 128], **args)


def c4(**kw) -> A.Config:
    """1-D advection in space-time on [0,2]x[0,1], 64x16 subdomains, m=250; RAS-GMRES(50)."""
    args = dict(decomposition=A.DECOMP_CELL, delta=0.1, test=[350, 350], tau_mode=A.TAU_RELATIVE,
                tau=1e-6, pca_matrix=A.PCA_OP_APPLIED, solver=A.SOLVER_GMRES, precond=A.PRECOND_RAS,
                gmres_restart=50, rel_tol=1e-10, seed=1000, op_form=A.OPERATOR_TWO_PASS)
    args.update(kw)
    return A.make_config(A.PROBLEM_ADVECTION, [64, 16], 250, [2560, 640], **args)


def c5(counts=(8, 8, 8), per=20, **kw) -> A.Config:
    """3-D Poisson, 8x8x8 subdomains (or the 2x2x2 C5s slice), m=400, 20^3 per subdomain."""
    args = dict(decomposition=A.DECOMP_CELL, delta=0.1, test=[50, 50, 50], tau_mode=A.TAU_RELATIVE,
                tau=1e-6, pca_matrix=A.PCA_OP_APPLIED, solver=A.SOLVER_CG, precond=A.PRECOND_AS,
                rel_tol=1e-10, seed=1000, op_form=A.OPERATOR_TWO_PASS)
    args.update(kw)
    return A.make_config(A.PROBLEM_POISSON, list(counts), 400, [c * per for c in counts], dim=3, **args)


def scaled(cfg: A.Config, counts, per_axis_points, m=None) -> A.Config:
    """A slice of a config keeping d, the operator, P and (by default) m."""
    out = A.Config.from_buffer_copy(cfg)
    for i, c in enumerate(counts):
        out.counts[i] = c
        out.colloc[i] = c * per_axis_points
    if m is not None:
        out.m = m
    if out.boundary_per_edge:
        out.boundary_per_edge = out.colloc[0]
    return out


BASELINE = {"C1": c1, "C2": c2, "C3": c3, "C4": c4, "C5": c5}


def aspcg(name: str) -> A.Config:
    """The metric's solver on any config: AS-preconditioned CG (C3/C4 name RAS-GMRES(50) as their
    own solver; the BASELINE metric reports AS-PCG for every config)."""
    cfg = BASELINE[name]()
    cfg.solver, cfg.precond = A.SOLVER_CG, A.PRECOND_AS
    return cfg


# ---- golden cases (reference test artefacts) -------------------------------------------
def golden_h_export() -> A.Config:
    """test_assembly.cpp:188-210 build_pipeline(2,3,6,21): example1 n=2, 2x2, delta 2, m=3, 6x6."""
    return A.make_config(A.PROBLEM_EXAMPLE1, [2, 2], 3, [6, 6], n=2, seed=21, test=[40, 40])


def golden_runner(seed=77) -> A.Config:
    """test_runner.cpp:13-42 small_config: example1 n=1, 2x2, m=8, 12x12, GMRES+AS, tol 1e-5."""
    return A.make_config(A.PROBLEM_EXAMPLE1, [2, 2], 8, [12, 12], n=1, seed=seed, test=[40, 40],
                         solver=A.SOLVER_GMRES, precond=A.PRECOND_AS, rel_tol=1e-5)


def golden_scaling(precond=A.PRECOND_AS) -> A.Config:
    """runner.hpp:434-492 scaling_cmd at n=2 (test_runner.cpp:173-184): 2x2, (5*4)^2, m=32, tau 1e-3."""
    restart = 30 if precond == A.PRECOND_NONE else 0
    return A.make_config(A.PROBLEM_EXAMPLE1, [2, 2], 32, [20, 20], n=2, seed=77, test=[40, 40],
                         tau_mode=A.TAU_ABSOLUTE, tau=1e-3, pca_matrix=A.PCA_OP_APPLIED,
                         solver=A.SOLVER_GMRES, precond=precond, rel_tol=1e-5, gmres_restart=restart)


def golden_sweep(tau: float, seed: int) -> A.Config:
    """runner.hpp:375-417 sweep_tau (test_runner.cpp:162-171): small_config with m=12."""
    return A.make_config(A.PROBLEM_EXAMPLE1, [2, 2], 12, [12, 12], n=1, seed=seed, test=[40, 40],
                         tau_mode=A.TAU_ABSOLUTE, tau=tau, pca_matrix=A.PCA_OP_APPLIED,
                         solver=A.SOLVER_GMRES, precond=A.PRECOND_AS, rel_tol=1e-5)


def golden_schwarz_diag() -> A.Config:
    """test_schwarz.cpp:190-203 build_setup({2,2},6,12,61): example1 n=2, identity reduction."""
    return A.make_config(A.PROBLEM_EXAMPLE1, [2, 2], 6, [12, 12], n=2, seed=61, test=[40, 40],
                         solver=A.SOLVER_GMRES, precond=A.PRECOND_AS)
