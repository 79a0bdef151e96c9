"""Error behaviour of the device path, mirroring the reference's exceptions: the C ABI
returns RDD_INVALID_ARGUMENT / RDD_RUNTIME_ERROR / RDD_DOMAIN_ERROR with the reference's message,
the Python binding raises ValueError / RuntimeError / ArithmeticError like the reference's
std::invalid_argument / std::runtime_error / std::domain_error."""
import numpy as np
import pytest

from paper_2412_19207_b200 import abi as A
from paper_2412_19207_b200 import configs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    from paper_2412_19207_b200 import rdd
    return rdd.Solver(0)


def _small(**kw):
    cfg = configs.golden_runner(77)
    for k, v in kw.items():
        setattr(cfg, k, v)
    return cfg


def test_decomposition_arguments(dev):
    with pytest.raises(ValueError, match="delta must exceed 1"):  # geometry.hpp:113
        dev.build_instance(_small(delta=1.0))
    bad = _small()
    bad.counts[0] = 0
    with pytest.raises(ValueError, match=">= 1"):  # geometry.hpp:115
        dev.build_instance(bad)
    with pytest.raises(ValueError, match="dimension"):  # runner.hpp:45 (test_runner.cpp:189)
        dev.build_instance(_small(dim=3))
    bad = _small()
    bad.colloc[1] = 0
    with pytest.raises(ValueError, match="resolutions"):  # geometry.hpp:204
        dev.build_instance(bad)


def test_truncation_and_solver_arguments(dev):
    with pytest.raises(ValueError, match="tau must be >= 0"):  # reduction.hpp:90
        dev.build_instance(_small(tau_mode=A.TAU_ABSOLUTE, tau=-1.0))
    with pytest.raises(ValueError, match="max_iter"):  # krylov.hpp:79
        dev.run_single(_small(max_iter=-1))


def test_empty_subdomain(dev):
    # 4x4 boxes over a 2x2 collocation grid: most boxes hold no point (reduction.hpp:38/62)
    cfg = A.make_config(A.PROBLEM_EXAMPLE1, [4, 4], 8, [2, 2], n=1, seed=3, test=[10, 10], delta=1.05,
                        tau_mode=A.TAU_ABSOLUTE, tau=1e-3)
    with pytest.raises(RuntimeError, match="contains no collocation points"):
        dev.build_instance(cfg)


def test_operator_lengths(dev):
    cfg = _small()
    dev.build_instance(cfg).assemble(True).build_preconditioner(A.PRECOND_AS)
    p, N = int(dev.geti("p")[0]), int(dev.geti("N")[0])
    with pytest.raises(ValueError, match="wrong length"):  # assembly.hpp:111 (test_assembly.cpp:132)
        dev.matvec(np.zeros(p + 1))
    with pytest.raises(ValueError, match="wrong length"):  # assembly.hpp:124 (test_assembly.cpp:133)
        dev.matvec_transpose(np.zeros(N - 1))
    with pytest.raises(ValueError, match="wrong vector length"):  # schwarz.hpp:154 (test_schwarz.cpp:164)
        dev.precond_apply(np.zeros(3))
    # valid lengths still work afterwards (the context survives an error)
    assert dev.matvec(np.ones(p)).shape == (N,)


def test_full_gmres_cap(dev):
    # krylov.hpp:294 / test_krylov.cpp:214: a full (unrestarted) basis beyond 4096 vectors is refused
    cfg = configs.scaled(configs.c2(), [8, 8], 12, m=80)  # τ off: p = 64·80 = 5120 > 4096
    cfg.tau_mode = A.TAU_OFF
    cfg.solver, cfg.precond, cfg.gmres_restart, cfg.max_iter = A.SOLVER_GMRES, A.PRECOND_NONE, 0, 5000
    with pytest.raises(RuntimeError, match="full GMRES basis"):
        dev.run_single(cfg)


def test_bit_identical_reruns(dev):
    # test_runner.cpp:109-117: the same seed twice gives identical results (fixed-order reductions)
    cfg = _small(solver=A.SOLVER_CG, precond=A.PRECOND_AS, rel_tol=1e-10)
    a, b = dev.run_single(cfg), dev.run_single(cfg)
    assert a["iterations"] == b["iterations"] and a["e_l2"] == b["e_l2"]  # bit-identical reruns
