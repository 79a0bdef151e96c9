"""Pins the CPU oracle against the reference's own committed artefacts.

The oracle is the parity checker for the GPU path, so it is validated first: assembly and
normal blocks against proj/h_export.txt / ata_export.txt (no LAPACK involved, bit-level),
the full run_single pipeline against runner_out/, PCA ranks against the tau sweep and the
weak-scaling row, local Schwarz ranks/conditions against schwarz_diag.csv.
"""
import numpy as np
import pytest

from paper_2412_19207_b200 import abi as A
from paper_2412_19207_b200 import configs


@pytest.fixture(scope="module")
def orc(oracle_cls):
    return oracle_cls()


def test_h_export_bitlevel(orc, golden):
    # test_assembly.cpp:188-210 build_pipeline(2,3,6,21), no equilibration
    orc.build_instance(configs.golden_h_export()).assemble(equilibrate=False)
    g = golden["h_export"]
    p = int(orc.geti("p")[0])
    H = orc.getd("H_dense").reshape(p, -1).T
    assert H.shape == (g["rows"], g["cols"]) == (36, 12)
    G = np.zeros_like(H)
    for r, c, v in g["triples"]:
        G[r, c] = v
    assert len(g["triples"]) == 432
    # the golden was printed with 17 significant digits; one entry differs by 2 ulp (libm tanh/cos)
    ulp = np.spacing(np.abs(G))
    assert np.all(np.abs(H - G) <= 2 * ulp)
    assert (H == G).sum() >= 431


def test_ata_export_bitlevel(orc, golden):
    orc.build_instance(configs.golden_h_export()).assemble(equilibrate=False).normal_blocks()
    A_ = orc.getd("nb_dense").reshape(12, 12)
    B = np.array(golden["ata_export"])
    assert np.max(np.abs(A_ - B)) <= 4 * np.spacing(np.abs(B).max())


@pytest.mark.parametrize("row", [0, 1])
def test_runner_summary(orc, golden, row):
    ref = golden["runner_summary"][row]
    seed = int(ref["seed"])
    s = orc.run_single(configs.golden_runner(seed))
    assert s["DoF"] == int(ref["DoF"]) == 32
    assert s["N"] == int(ref["N"]) == 144
    assert s["J"] == 4
    assert s["iterations"] == int(ref["iter"])
    assert s["converged"] == 1
    # GMRES stops at a preconditioned residual ~1e-8 (tol 1e-5); e_l2 agrees to that level
    assert s["e_l2"] == pytest.approx(float(ref["e_l2"]), rel=5e-7)
    assert s["e_l1n"] == pytest.approx(float(ref["e_l1n"]), rel=5e-7)
    hist = orc.getd("hist")
    assert len(hist) == 2 and hist[0] == 1.0 and hist[1] < 1e-7


def test_scaling_row(orc, golden):
    ref_as, ref_none = golden["scaling"]
    s = orc.run_single(configs.golden_scaling(A.PRECOND_AS))
    assert s["DoF"] == int(float(ref_as["DoF"])) == 87   # PCA ranks (op_applied, tau 1e-3)
    assert s["N"] == 400
    assert s["iterations"] == int(float(ref_as["iter"]))
    assert s["e_l1n"] == pytest.approx(float(ref_as["e_l1n"]), rel=1e-6)
    s = orc.run_single(configs.golden_scaling(A.PRECOND_NONE))
    assert s["DoF"] == 87
    # unpreconditioned GMRES(30) on cond ~1e10 is rounding-sensitive; with the PCA in Eigen's
    # QR-preconditioned Jacobi form the oracle reproduces the reference's 86 iterations exactly
    assert s["iterations"] == int(float(ref_none["iter"])) == 86
    assert s["e_l1n"] == pytest.approx(float(ref_none["e_l1n"]), rel=1e-3)


def test_sweep_tau(orc, golden):
    for ref in golden["sweep_tau"]:
        tau = float(ref["tau"])
        dofs, cn, el2 = [], [], []
        for seed in (77, 78):
            s = orc.run_single(configs.golden_sweep(tau, seed))
            dofs.append(s["DoF"])
            el2.append(s["e_l2"])
            orc.build_instance(configs.golden_sweep(tau, seed)).assemble(True).build_preconditioner(A.PRECOND_AS)
            _, _, c1, c2 = orc.spectra(True)
            cn.append(c1)
            assert c2 == pytest.approx(1.0, rel=1e-6)
        assert np.median(dofs) == float(ref["DoF"])
        assert np.median(cn) == pytest.approx(float(ref["cond_HtH"]), rel=1e-8)
        assert np.median(el2) == pytest.approx(float(ref["e_l2"]), rel=1e-8)


def test_schwarz_diag(orc, golden):
    orc.build_instance(configs.golden_schwarz_diag()).assemble(False).build_preconditioner(A.PRECOND_AS)
    ranks = orc.geti("local_rank")
    conds = orc.getd("local_cond")
    for i, ref in enumerate(golden["schwarz_diag"]):
        assert ranks[i] == int(ref["rank"])
        assert len(orc.geti("set", i)) == int(ref["size"])
        assert conds[i] == pytest.approx(float(ref["cond_estimate"]), rel=1e-5)


def test_spectra(orc, golden):
    orc.build_instance(configs.golden_runner(77)).assemble(True).build_preconditioner(A.PRECOND_AS)
    normal, pre, _, _ = orc.spectra(True)
    ref_n = np.array(golden["spectrum_normal"])
    ref_p = np.array(golden["spectrum_preconditioned"])
    assert len(normal) == len(ref_n) == 32
    # golden printed with 12 significant digits; eigenvalues resolved to ~eps * lambda_max
    assert np.max(np.abs(normal - ref_n)) <= 1e-11 * ref_n.max()
    assert np.max(np.abs(pre - ref_p)) <= 5e-8


def test_truncation_known_answer(orc):
    # test_reduction.cpp:57-79: diag(3, 1, 1e-5) with tau 1e-3 keeps 2 (exercised via the tau sweep
    # ranks above; here the relative mode's floor rule p >= 1 on a tiny config)
    cfg = configs.golden_sweep(10.0, 77)
    cfg.tau_mode = A.TAU_ABSOLUTE
    cfg.tau = 1e300
    orc.build_instance(cfg)
    assert list(orc.geti("p_j")) == [1, 1, 1, 1]


def test_errors_mirror_reference(orc):
    cfg = configs.golden_runner(77)
    with pytest.raises(ValueError):
        bad = configs.golden_runner(77)
        bad.n = 9
        orc.build_instance(bad)
    # an empty subdomain under PCA raises runtime_error naming the subdomain (reduction.hpp:37-38)
    cfg = A.make_config(A.PROBLEM_EXAMPLE1, [4, 4], 3, [1, 1], n=2, tau_mode=A.TAU_ABSOLUTE, tau=1e-3,
                        pca_matrix=A.PCA_PSI)
    with pytest.raises(RuntimeError, match="subdomain 0"):
        orc.build_instance(cfg)
