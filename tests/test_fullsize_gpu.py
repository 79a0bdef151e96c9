"""BASELINE.json's configurations at full size, against the CPU oracle.

* C1 and C5s (the 2x2x2 run of C5) are run on the oracle inside the test.
* C2, C3, C4 and C5 are compared with committed full-size oracle fixtures
  (tests/golden/fullsize/*.npz, written by tests/golden/make_fullsize.py; the oracle needs
  minutes to hours for these, so it is not run on the GPU box):
    - PCA of every subdomain (reduction.hpp:89-109): ranks p_j bit-exact; σ_i within 1e-9
      relative above 20% of the threshold; one seeded probe per subdomain through the kept
      projector, ‖(P_dev − P_ref)x‖ ≤ 1e-8‖x‖; the exact projector 2-norm ‖P_dev − P_ref‖₂ ≤ 1e-8 on
      four subdomains per config (from the stored basis or its complement). Where the kept
      subspace is ill-conditioned (relative gap σ_{p-1}−σ_p ~ 1e-8 at the threshold) the bar is
      20·ε·σ_0/gap instead (Wedin; projector_bar), on at most 1% of the subdomains.
    - full run_single with AS-PCG to 1e-10 on C2 and C4 (runner.hpp:202-275): iterations within
      5%, e_L2 and e_L1n within 1e-8 relative, the final relative residual within 1e-8 relative,
      the approximation at the test points ‖u_dev − u_ref‖ ≤ 1e-8‖u_exact‖.
* C2 and C4 are also checked through size-independent properties of the domain: covering and
  ordering of the point-to-subdomain index, the PCA threshold rule on the exported spectra,
  orthonormal kept bases, the operator's adjoint identity and linearity, symmetry and positivity
  of the AS preconditioner, a converged solve with bit-identical reruns, and the true
  normal-equation residual of the returned coefficients.
"""
import os

import numpy as np
import pytest

from paper_2412_19207_b200 import abi as A
from paper_2412_19207_b200 import configs

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def dev():
    from paper_2412_19207_b200 import rdd
    return rdd.Solver(0)


@pytest.fixture(scope="module")
def orc(oracle_cls):
    return oracle_cls()


@pytest.mark.parametrize("name", ["C1", "C5s"])
def test_full_size_vs_oracle(dev, orc, name):
    cfg = configs.c1() if name == "C1" else configs.c5(counts=(2, 2, 2))
    sd = dev.run_single(cfg)
    pd = dev.geti("p_j")
    so = orc.run_single(cfg)
    assert np.array_equal(pd, orc.geti("p_j"))  # PCA ranks bit-exact
    assert sd["DoF"] == so["DoF"] and sd["N"] == so["N"] and sd["J"] == so["J"]
    assert sd["converged"] == so["converged"] == 1
    assert abs(sd["iterations"] - so["iterations"]) <= int(0.05 * so["iterations"]), (sd, so)
    # relative L2 / normalised L1 errors within 1e-8 of each other, and the solutions themselves
    assert abs(sd["e_l2"] - so["e_l2"]) <= 1e-8, (sd["e_l2"], so["e_l2"])
    assert abs(sd["e_l1n"] - so["e_l1n"]) <= 1e-8
    ua, ue = dev.getd("approx"), dev.getd("exact")
    assert np.linalg.norm(ua - orc.getd("approx")) <= 1e-8 * np.linalg.norm(ue)


def _properties(dev, cfg, precond_symmetric):
    s = dev.run_single(cfg)
    assert s["converged"] == 1
    J, N, p = s["J"], s["N"], s["DoF"]
    # index: ascending rows, every point covered by 1..2^d boxes, Σ|rows_j| consistent
    cover = np.zeros(N, dtype=np.int64)
    total = 0
    for j in range(J):
        rows = dev.geti("rows", j)
        assert rows.size > 0 and np.all(np.diff(rows) > 0)
        cover[rows] += 1
        total += rows.size
    d = cfg.d
    assert cover.min() >= 1 and cover.max() <= 2 ** d and cover.sum() == total
    # PCA: p_j = #{σ > τ·σmax} (strict, floor 1), σ non-increasing, kept V orthonormal
    pj = dev.geti("p_j")
    assert pj.sum() == p
    for j in range(0, J, max(1, J // 16)):
        sig = dev.getd("sigma", j)
        assert np.all(np.diff(sig) <= 0)
        assert pj[j] == max(1, int(np.sum(sig > cfg.tau * sig[0])))
        V = dev.getd("V", j).reshape(pj[j], cfg.m).T
        assert np.linalg.norm(V.T @ V - np.eye(pj[j])) <= 1e-11
    # operator: adjoint identity and linearity of H·w / Hᵀ·r
    rng = np.random.default_rng(7)
    w1, w2, r = rng.standard_normal(p), rng.standard_normal(p), rng.standard_normal(N)
    y1, y2 = dev.matvec(w1), dev.matvec(w2)
    t = dev.matvec_transpose(r)
    assert abs(y1 @ r - w1 @ t) <= 1e-11 * np.linalg.norm(y1) * np.linalg.norm(r)
    y12 = dev.matvec(2.0 * w1 - 3.0 * w2)
    assert np.linalg.norm(y12 - (2.0 * y1 - 3.0 * y2)) <= 1e-12 * np.linalg.norm(y12)
    n1, n2 = dev.normal_apply(w1), dev.normal_apply(w2)
    assert abs(n1 @ w2 - n2 @ w1) <= 1e-11 * abs(n1 @ w2) + 1e-12 * np.linalg.norm(n1) * np.linalg.norm(w2)
    assert n1 @ w1 > 0
    # preconditioner: AS is symmetric positive semi-definite (a sum of local pseudo-inverses)
    z1, z2 = dev.precond_apply(w1), dev.precond_apply(w2)
    if precond_symmetric:
        assert abs(z1 @ w2 - z2 @ w1) <= 1e-10 * np.linalg.norm(z1) * np.linalg.norm(w2)
        assert z1 @ w1 > 0
    zt = dev.precond_apply(w2, transpose=True)
    assert abs(z1 @ w2 - w1 @ zt) <= 1e-10 * np.linalg.norm(z1) * np.linalg.norm(w2)  # Mᵀ is the adjoint
    # the returned coefficients (equilibrated) solve the normal equations: ‖HᵀHW − HᵀF‖ small
    W = dev.getd("W", 0) * dev.getd("scales")
    F = dev.getd("F")[:N]
    res = dev.normal_apply(W) - dev.matvec_transpose(F)
    assert np.linalg.norm(res) <= 1e-5 * np.linalg.norm(dev.matvec_transpose(F))
    # bit-identical rerun of the whole pipeline on the resident inputs
    s2 = dev.rerun_resident()
    assert s2["iterations"] == s["iterations"] and s2["e_l2"] == s["e_l2"] and s2["DoF"] == s["DoF"]
    return s


def test_c2_full_size_properties(dev):
    s = _properties(dev, configs.c2(), True)
    assert s["N"] == 921_600 and s["J"] == 256
    assert s["e_l2"] < 1e-2


def test_c4_full_size_properties(dev):
    cfg = configs.aspcg("C4")
    s = _properties(dev, cfg, True)
    assert s["N"] == 1_638_400 and s["J"] == 1024
    ras = configs.c4(max_iter=50)
    dev.run_single(ras)  # RAS-GMRES(50) path: the transpose apply is the adjoint of the apply
    rng = np.random.default_rng(9)
    p = int(dev.geti("p")[0])
    v, w = rng.standard_normal(p), rng.standard_normal(p)
    z, zt = dev.precond_apply(v), dev.precond_apply(w, transpose=True)
    assert abs(z @ w - v @ zt) <= 1e-10 * np.linalg.norm(z) * np.linalg.norm(w)


# ---------------------------------------------------------------- committed full-size oracle fixtures
FIX = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "fullsize")
PROBE_SEED = 20250  # tests/golden/make_fullsize.py


def _fixture(kind, name):
    path = os.path.join(FIX, f"{kind}_{name}.npz")
    if not os.path.exists(path):
        pytest.fail(f"missing fixture {path} (tests/golden/make_fullsize.py)")
    return np.load(path)


EPS = np.finfo(float).eps


def projector_bar(so, p):
    """The projector bar of subdomain j: 1e-8 (north_star), except where the kept subspace is
    itself ill-conditioned. By Wedin's theorem a backward error ‖E‖ ~ ε‖S‖ moves the projector
    onto the leading p right singular vectors by ‖E‖/(σ_{p-1} − σ_p); the oracle and the device
    both carry such an error, so where ε·σ_0/gap approaches 1e-8 (relative gaps of ~1e-8 at the
    1e-6 threshold, a few subdomains of C3/C5) they can only agree to a small multiple of it."""
    gap = so[p - 1] - (so[p] if p < len(so) else 0.0)
    return max(1e-8, 20.0 * EPS * so[0] / gap)


def _check_pca(dev, cfg, fx):
    m = cfg.m
    pd = dev.geti("p_j")
    assert np.array_equal(pd, fx["p_j"]), np.flatnonzero(pd != fx["p_j"])[:10]  # bit-exact ranks
    off, sig_ref = fx["sigma_off"], fx["sigma"]
    worst, over_1e8 = 0.0, 0
    for j in range(len(pd)):
        so = sig_ref[off[j]:off[j + 1]]
        sd = dev.getd("sigma", j)[:len(so)]
        big = so > 0.2 * cfg.tau * so[0]
        np.testing.assert_allclose(sd[big], so[big], rtol=1e-9, atol=0, err_msg=f"sigma j={j}")
        V = dev.getd("V", j).reshape(int(pd[j]), m).T
        x = np.random.default_rng(PROBE_SEED + j).standard_normal(m)
        d = np.linalg.norm(V @ (V.T @ x) - fx["probe_px"][j]) / np.linalg.norm(x)
        assert d <= projector_bar(so, int(pd[j])), (j, d, projector_bar(so, int(pd[j])))
        worst = max(worst, d)
        over_1e8 += d > 1e-8
    assert over_1e8 <= max(1, len(pd) // 100), over_1e8  # the ill-conditioned ones are rare
    for j in fx["subset"]:
        B = fx[f"basis_{j}"]
        Pr = B @ B.T
        if int(fx[f"basis_kind_{j}"]) == 1:
            Pr = np.eye(m) - Pr
        V = dev.getd("V", int(j)).reshape(int(pd[j]), m).T
        so = sig_ref[off[j]:off[j + 1]]
        assert np.linalg.norm(V @ V.T - Pr, 2) <= projector_bar(so, int(pd[j])), int(j)


@pytest.mark.parametrize("name", ["C3", "C5"])
def test_full_size_pca_vs_oracle_fixture(dev, name):
    cfg = configs.BASELINE[name]()
    dev.build_instance(cfg)
    _check_pca(dev, cfg, _fixture("pca", name))


@pytest.mark.parametrize("name", ["C2", "C4"])
def test_full_size_run_vs_oracle_fixture(dev, name):
    cfg = configs.aspcg(name)
    fx = _fixture("run", name)
    sd = dev.run_single(cfg)
    _check_pca(dev, cfg, fx)
    assert sd["DoF"] == int(fx["DoF"]) and sd["N"] == int(fx["N"])
    assert sd["converged"] == int(fx["converged"]) == 1
    its = int(fx["iterations"])
    assert abs(sd["iterations"] - its) <= int(0.05 * its), (sd["iterations"], its)
    # here e_L2 (2e-3 on C2, 1.4e-5 on C4) is resolved: relative agreement 1e-8 holds
    assert sd["e_l2"] == pytest.approx(float(fx["e_l2"]), rel=1e-8), (sd["e_l2"], float(fx["e_l2"]))
    assert sd["e_l1n"] == pytest.approx(float(fx["e_l1n"]), rel=1e-8)
    assert sd["final_residual"] == pytest.approx(float(fx["final_residual"]), rel=1e-8)
    ue = dev.getd("exact")
    assert np.linalg.norm(dev.getd("approx") - fx["approx"]) <= 1e-8 * np.linalg.norm(ue)
    # the residual histories follow each other while they are far above rounding
    hd, ho = dev.getd("hist", 0), fx["hist"]
    k = min(len(hd), len(ho))
    np.testing.assert_allclose(hd[:k][ho[:k] > 1e-6], ho[:k][ho[:k] > 1e-6], rtol=1e-6)


# RAS-GMRES(50) (krylov.hpp:275-389) with the full m and points per subdomain on slices of C3 and
# C4: the CPU oracle's histories (tests/golden/ras_gmres_slices_oracle.jsonl, written by
# tools/ras_stagnation.py) — the C3 slice stagnates at 1.03e-2 on the oracle as on the device,
# the C4 slices converge; the device reproduces every 50th residual
@pytest.mark.parametrize("case", ["C4_16x4", "C4_8x8", "C3_3x3x2"])
def test_ras_gmres_slices_vs_oracle(dev, case):
    import json
    recs = [json.loads(l) for l in open(os.path.join(os.path.dirname(FIX), "ras_gmres_slices_oracle.jsonl"))]
    ref = next(r for r in recs if r["case"] == case)
    base = {"C4": configs.c4(), "C3": configs.c3()}[case[:2]]
    counts = [int(x) for x in case[3:].split("x")]
    cfg = configs.scaled(base, counts, 40 if case.startswith("C4") else 16)
    cfg.solver, cfg.precond, cfg.gmres_restart, cfg.max_iter = A.SOLVER_GMRES, A.PRECOND_RAS, 50, 1500
    s = dev.run_single(cfg)
    assert s["DoF"] == ref["DoF"] and s["converged"] == ref["converged"]
    assert abs(s["iterations"] - ref["iterations"]) <= int(0.05 * ref["iterations"])
    h = dev.getd("hist", 0)[::50]
    np.testing.assert_allclose(h[:len(ref["hist_every_50"])], ref["hist_every_50"], rtol=1e-6)


@pytest.mark.parametrize("name", ["C1", "C5s"])
def test_full_size_vs_compiled_reference(dev, name):
    # C1 at full size and C5s (the 2x2x2 run BASELINE names for C5) on the reference itself
    # (oracle/_ref: the unmodified headers on the Eigen-subset shim, the BASELINE objects built from
    # its own types): ranks bit-exact, iterations within 5%, errors and solutions within 1e-8
    import ref as refmod
    if not refmod.available():
        pytest.fail("oracle/_ref/libref.so missing (built by __graft_entry__.build() next to /root/reference)")
    cfg = configs.c1() if name == "C1" else configs.c5(counts=(2, 2, 2))
    rf = refmod.Reference()
    sr = rf.run_baseline(cfg)
    pr = rf.geti("p_j")
    sd = dev.run_single(cfg)
    assert np.array_equal(dev.geti("p_j"), pr)
    assert sd["DoF"] == sr["DoF"] and sd["N"] == sr["N"] and sd["converged"] == sr["converged"] == 1
    assert abs(sd["iterations"] - sr["iterations"]) <= int(0.05 * sr["iterations"]), (sd, sr)
    assert abs(sd["e_l2"] - sr["e_l2"]) <= 1e-8, (sd["e_l2"], sr["e_l2"])
    assert abs(sd["e_l1n"] - sr["e_l1n"]) <= 1e-8


@pytest.mark.parametrize("name", ["C2", "C4"])
def test_full_size_run_vs_reference_fixture(dev, name):
    # the full-size AS-PCG solves of C2 and C4 on the reference itself (tests/golden/make_fullsize.py
    # refrun: oracle/_ref with the BASELINE objects built from the reference's own types)
    fx = _fixture("ref_run", name)
    sd = dev.run_single(configs.aspcg(name))
    assert np.array_equal(dev.geti("p_j"), fx["p_j"])
    assert sd["DoF"] == int(fx["DoF"]) and sd["N"] == int(fx["N"]) and sd["converged"] == int(fx["converged"]) == 1
    its = int(fx["iterations"])
    assert abs(sd["iterations"] - its) <= int(0.05 * its), (sd["iterations"], its)
    assert sd["e_l2"] == pytest.approx(float(fx["e_l2"]), rel=1e-8), (sd["e_l2"], float(fx["e_l2"]))
    assert sd["e_l1n"] == pytest.approx(float(fx["e_l1n"]), rel=1e-8)
    hd, ho = dev.getd("hist", 0), fx["hist"]
    k = min(len(hd), len(ho))
    np.testing.assert_allclose(hd[:k][ho[:k] > 1e-6], ho[:k][ho[:k] > 1e-6], rtol=1e-6)
