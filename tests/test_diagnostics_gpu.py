"""GPU dense diagnostics (§8f row 4): spectrum / singular_values / condition_number
(krylov.hpp:403-440) and the spectrum_cmd / sweep_tau quantities (runner.hpp:344-393), through
the C ABI, against the reference's golden artefacts (runner_out_spec, runner_out_sweep), the
CPU oracle (LAPACK dsyevd/dgeev/dgesvd on the same systems) and numpy on random matrices.

Tolerances: eigenvalues and singular values are backward-stable results, so they are compared
with an absolute bound relative to the matrix norm (|Δλ| <= 1e-11·‖A‖ for symmetric matrices and
normal-ish random ones; the nonsymmetric preconditioned operators use 1e-9·‖M⁻¹A‖); condition
numbers relative 1e-8 where cond·ε stays below that.
"""
import numpy as np
import pytest
from scipy.optimize import linear_sum_assignment

from paper_2412_19207_b200 import abi as A
from paper_2412_19207_b200 import configs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    from paper_2412_19207_b200 import rdd
    return rdd.Solver(0)


@pytest.fixture(scope="module")
def orc(oracle_cls):
    return oracle_cls()


def _match(a, b):
    """max |a_i - b_π(i)| over the best one-to-one matching (order-free spectrum comparison)."""
    D = np.abs(a[:, None] - b[None, :])
    r, c = linear_sum_assignment(D)
    return D[r, c].max()


@pytest.mark.parametrize("n", [1, 2, 3, 5, 40, 257])
def test_spectrum_random_nonsymmetric(dev, n):
    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, n))
    got = dev.spectrum(a)
    ref = np.linalg.eigvals(a)
    assert got.shape == (n,)
    assert _match(got, ref) <= 1e-9 * max(1.0, np.linalg.norm(a, 2))
    # sorted by real part, then imaginary part (write_spectrum_csv order)
    assert np.all(np.diff(got.real) >= 0)
    # real input: eigenvalues come in conjugate pairs
    assert _match(got, np.conj(got)) <= 1e-9 * max(1.0, np.linalg.norm(a, 2))


def test_spectrum_known_structures(dev):
    # symmetric with a prescribed spectrum spanning 12 orders of magnitude
    rng = np.random.default_rng(3)
    q, _ = np.linalg.qr(rng.standard_normal((120, 120)))
    lam = np.logspace(-6, 6, 120)
    s = (q * lam) @ q.T
    s = 0.5 * (s + s.T)
    got = dev.spectrum(s)
    assert np.max(np.abs(got.imag)) <= 1e-9 * lam.max()
    assert np.max(np.abs(np.sort(got.real) - lam)) <= 1e-11 * lam.max() * 10
    # rotation blocks: exact complex pairs ±i·k
    b = np.zeros((6, 6))
    for k in range(3):
        b[2 * k, 2 * k + 1] = k + 1.0
        b[2 * k + 1, 2 * k] = -(k + 1.0)
    got = dev.spectrum(b)
    want = np.array([1j * (k + 1) * sgn for k in range(3) for sgn in (1, -1)])
    assert _match(got, want) <= 1e-12
    # upper triangular (already reduced): the diagonal
    t = np.triu(rng.standard_normal((30, 30)))
    assert _match(dev.spectrum(t), np.diag(t).astype(complex)) <= 1e-10


@pytest.mark.parametrize("shape", [(1, 1), (7, 3), (3, 7), (64, 64), (300, 120), (90, 250)])
def test_singular_values_random(dev, shape):
    rng = np.random.default_rng(shape[0] * 1000 + shape[1])
    a = rng.standard_normal(shape)
    got = dev.singular_values(a)
    ref = np.linalg.svd(a, compute_uv=False)
    assert got.shape == ref.shape
    assert np.all(np.diff(got) <= 0)
    assert np.max(np.abs(got - ref)) <= 1e-12 * ref[0] * max(shape)
    assert dev.condition_number(a) == pytest.approx(ref[0] / ref[-1], rel=1e-9)


def test_condition_number_rank_deficient_and_zero(dev):
    rng = np.random.default_rng(11)
    u = rng.standard_normal((50, 4))
    a = u @ rng.standard_normal((4, 50))  # rank 4: cond is over the positive σ, huge from noise
    sv = dev.singular_values(a)
    ref = np.linalg.svd(a, compute_uv=False)
    assert np.max(np.abs(sv - ref)) <= 1e-12 * ref[0] * 50
    graded = np.diag([1.0, 1e-3, 1e-6, 1e-9])
    assert dev.condition_number(graded) == pytest.approx(1e9, rel=1e-9)
    with pytest.raises(ArithmeticError, match="all singular values are zero"):
        dev.condition_number(np.zeros((5, 5)))


def test_diagnostics_errors(dev):
    with pytest.raises(ValueError, match="matrix must be square"):
        dev.spectrum(np.ones((3, 4)))
    with pytest.raises(ValueError, match=r"matrix of size 10 exceeds the dense diagnostics cap \(8\)"):
        dev.spectrum(np.eye(10), cap=8)
    with pytest.raises(ValueError, match="exceeds the dense diagnostics cap"):
        dev.singular_values(np.eye(9), cap=8)


def test_spectra_golden_runner_out_spec(dev, golden):
    # test_runner.cpp:139-160 spectrum command on the runner config, AS preconditioner
    dev.build_instance(configs.golden_runner(77))
    dev.assemble(True)
    dev.build_preconditioner(A.PRECOND_AS)
    normal, pre, cn, cp = dev.spectra(True)
    ref_n = np.array(golden["spectrum_normal"])
    ref_p = np.array(golden["spectrum_preconditioned"])
    assert len(normal) == len(ref_n) == 32
    assert np.all(normal.imag == 0)
    assert np.max(np.abs(normal.real - ref_n)) <= 1e-11 * ref_n.max()
    assert np.all(np.diff(pre.real) >= 0)
    # M⁻¹HᵀH is similar to a symmetric matrix but far from normal (cond(HᵀH) ~ 1e8 here), so the
    # 32-fold cluster at 4 is resolved only to ~1e-8 by any backward-stable solver: the oracle's
    # LAPACK dgeev sits at the same distance from the golden (test_oracle_golden.py)
    assert np.max(np.abs(pre.real - ref_p)) <= 5e-8
    assert np.max(np.abs(pre.imag)) <= 5e-8


def test_spectra_golden_sweep_tau(dev, golden):
    # test_runner.cpp:162-171: median over seeds 77/78 of cond(HᵀH), cond(M⁻¹HᵀH) = 1 (AS exact)
    for ref in golden["sweep_tau"]:
        tau = float(ref["tau"])
        cn = []
        for seed in (77, 78):
            dev.build_instance(configs.golden_sweep(tau, seed))
            dev.assemble(True)
            dev.build_preconditioner(A.PRECOND_AS)
            _, _, c1, c2 = dev.spectra(True)
            cn.append(c1)
            assert c2 == pytest.approx(1.0, rel=1e-6)
        # golden printed with 10 significant digits; cond·ε bounds the agreement
        assert np.median(cn) == pytest.approx(float(ref["cond_HtH"]), rel=1e-8)


@pytest.mark.parametrize("kind", [A.PRECOND_AS, A.PRECOND_SAS, A.PRECOND_RAS])
def test_spectra_vs_oracle(dev, orc, kind):
    cfg = configs.scaled(configs.c1(), [2, 2], 12, m=40)
    dev.build_instance(cfg)
    dev.assemble(True)
    dev.build_preconditioner(kind)
    normal, pre, cn, cp = dev.spectra(True)
    orc.build_instance(cfg).assemble(True).build_preconditioner(kind)
    o_n, o_pre_re, o_cn, o_cp = orc.spectra(True)
    p = len(o_n)
    assert len(normal) == p
    lmax = o_n.max()
    # Weyl: |λ_i(A_dev) − λ_i(A_ref)| ≤ ‖A_dev − A_ref‖₂ (A = HᵀH, the two PCAs differ by ~1e-11)
    dA = np.linalg.norm(dev.getd("nb_dense").reshape(p, p) - orc.getd("nb_dense").reshape(p, p), 2)
    assert np.max(np.abs(np.sort(normal.real) - o_n)) <= dA + 1e-13 * lmax
    # full complex spectrum of the oracle's own M⁻¹HᵀH (dense, numpy) and the sorted real parts
    AtA = orc.getd("nb_dense").reshape(p, p)
    MA = np.stack([orc.precond_apply(AtA[:, c]) for c in range(p)], axis=1)
    scale = np.linalg.norm(MA, 2)
    assert _match(pre, np.linalg.eigvals(MA)) <= 1e-9 * scale
    assert np.max(np.abs(np.sort(pre.real) - o_pre_re)) <= 1e-9 * scale
    # condition numbers (LAPACK dgesvd in the oracle); agreement bounded by cond·ε
    assert cn == pytest.approx(o_cn, rel=max(1e-8, 50 * o_cn * np.finfo(float).eps))
    assert cp == pytest.approx(o_cp, rel=max(1e-8, 50 * o_cp * np.finfo(float).eps))


def test_spectra_needs_preconditioner_and_cap(dev):
    dev.build_instance(configs.golden_runner(78))
    dev.assemble(True)
    normal, pre, cn, cp = dev.spectra(False)
    assert pre is None and cp is None and len(normal) == 32 and cn > 1
    with pytest.raises(ValueError, match="no preconditioner built"):
        dev.spectra(True)
    with pytest.raises(ValueError, match=r"matrix of size 32 exceeds the dense diagnostics cap \(31\)"):
        dev.spectra(False, cap=31)


@pytest.mark.parametrize("case", ["repeated", "rotations", "triangular_perturbed", "graded", "zero", "scaled_identity"])
def test_spectrum_multibulge_structures(dev, case):
    # active blocks above 112 take the windowed multi-bulge sweeps; structures that stress the
    # shifts and deflation (repeated, complex-pair, nonnormal, graded, degenerate spectra)
    rng = np.random.default_rng(hash(case) % 2**32)
    n = 240
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    if case == "repeated":
        lam = np.repeat([1.0, 2.0, 5.0, -3.0], n // 4)
        a = (q * lam) @ q.T
        want = lam.astype(complex)
    elif case == "rotations":
        b = np.zeros((n, n))
        want = []
        for k in range(n // 2):
            re, im = rng.uniform(-2, 2), rng.uniform(0.1, 3)
            b[2 * k:2 * k + 2, 2 * k:2 * k + 2] = [[re, im], [-im, re]]
            want += [re + 1j * im, re - 1j * im]
        a = q @ b @ q.T
        want = np.array(want)
    elif case == "triangular_perturbed":
        # strongly nonnormal: eigenvalues are ill-conditioned, so check the backward error of each
        # computed eigenvalue (σ_min(A − λI) small) rather than distances to another solver's values
        t = np.triu(rng.standard_normal((n, n)))
        a = q @ t @ q.T
        got = dev.spectrum(a)
        na = np.linalg.norm(a, 2)
        worst = max(np.linalg.svd(a - z * np.eye(n), compute_uv=False)[-1] for z in got[::8])
        assert worst <= 1e-12 * n * na
        assert abs(got.sum() - np.trace(a)) <= 1e-9 * n * na  # trace = Σλ
        return
    elif case == "graded":
        lam = np.logspace(-8, 4, n)
        a = (q * lam) @ q.T
        want = lam.astype(complex)
    elif case == "zero":
        a = np.zeros((n, n))
        want = np.zeros(n, dtype=complex)
    else:
        a = 3.5 * np.eye(n)
        want = np.full(n, 3.5, dtype=complex)
    got = dev.spectrum(a)
    scale = max(1.0, np.linalg.norm(a, 2))
    tol = 1e-9
    if case == "repeated":
        tol = 1e-7  # a multiple eigenvalue of a symmetric matrix rounded through a nonsymmetric solver
    assert _match(got, want) <= tol * scale, case
