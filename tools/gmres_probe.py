"""RAS-GMRES(50) per-iteration time on C4 (capped at 400 iterations) and C2 AS-GMRES(50)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_19207_b200 import rdd, configs, abi as A
for name, mi in (("C4", 400), ("C2", 400)):
    cfg = configs.BASELINE[name](max_iter=mi) if name == "C4" else configs.c2(solver=A.SOLVER_GMRES, gmres_restart=50, max_iter=mi)
    s = rdd.Solver(0)
    s.run_single(cfg)
    r = s.rerun_resident()
    print(name, {k: r[k] for k in ("iterations", "converged", "t_solve", "final_residual", "e_l2")}, "ms/iter", 1e3 * r["t_solve"] / max(1, r["iterations"]))
