"""Wall time of the dense diagnostics (spectrum_cmd quantities) on the device vs the CPU oracle
(LAPACK dsyevd/dgeev/dgesvd, single-threaded OpenBLAS like Eigen), C1 full size, and of the
standalone dense routines at n = 1000/2000/4000 (random matrices)."""
import json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_2412_19207_b200 import abi as A, configs, rdd

s = rdd.Solver(0)
out = []
cfg = configs.aspcg("C1")
s.build_instance(cfg); s.assemble(True); s.build_preconditioner(A.PRECOND_AS)
s.spectra(True)  # warm
t = time.perf_counter(); n_, pre, cn, cp = s.spectra(True); tg = time.perf_counter() - t
rec = {"case": "C1 spectra (AtA + M^-1 AtA spectra, both cond)", "p": len(n_), "gpu_s": tg, "cond_normal": cn, "cond_precond": cp}
if "--no-oracle" not in sys.argv:
    from oracle import Oracle
    o = Oracle()
    o.build_instance(cfg).assemble(True).build_preconditioner(A.PRECOND_AS)
    t = time.perf_counter(); on, opre, ocn, ocp = o.spectra(True); rec["oracle_s"] = time.perf_counter() - t
    rec["max_abs_dnormal_over_lmax"] = float(np.max(np.abs(n_.real - on)) / on.max())
    rec["max_abs_dpre_re"] = float(np.max(np.abs(np.sort(pre.real) - opre)))
    rec["cond_rel"] = [abs(cn - ocn) / ocn, abs(cp - ocp) / ocp]
out.append(rec)
for n in (1000, 2000, 4000):
    a = np.random.default_rng(n).standard_normal((n, n))
    for name, f in (("spectrum", s.spectrum), ("singular_values", s.singular_values)):
        f(a[:64, :64])
        t = time.perf_counter(); got = f(a); dt = time.perf_counter() - t
        rec = {"case": f"{name} n={n}", "gpu_s": dt}
        if n <= 2000:
            t = time.perf_counter()
            ref = np.linalg.eigvals(a) if name == "spectrum" else np.linalg.svd(a, compute_uv=False)
            rec["numpy_s"] = time.perf_counter() - t
            if name == "spectrum":
                from scipy.optimize import linear_sum_assignment
                D = np.abs(got[:, None] - ref[None, :]); r, cc = linear_sum_assignment(D)
                rec["max_err_over_norm"] = float(D[r, cc].max() / np.linalg.norm(a, 2))
            else:
                rec["max_err_over_norm"] = float(np.max(np.abs(got - ref)) / ref[0])
        out.append(rec)
for r in out:
    print(json.dumps(r))
