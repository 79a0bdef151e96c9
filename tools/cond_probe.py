"""Local-block conditioning and the Cholesky/eigen routing.

  python tools/cond_probe.py full        local_cond max / n_fallback of C1..C5 at full size
  python tools/cond_probe.py cluster     the two cluster-Jacobi parity cases at several
                                         full_rank_cond thresholds against the oracle
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_2412_19207_b200 import abi as A  # noqa: E402
from paper_2412_19207_b200 import configs, rdd  # noqa: E402


def full():
    s = rdd.Solver(0)
    for name in ("C1", "C2", "C3", "C4", "C5"):
        r = s.run_single(configs.aspcg(name))
        lc = s.getd("local_cond")
        print(json.dumps({"config": name, "local_cond_max": float(lc.max()), "local_cond_median": float(np.median(lc)),
                          "n_fallback": int(s.geti("n_fallback")[0]), "iterations": r["iterations"],
                          "t_precond": r["t_precond"]}), flush=True)


def cluster():
    from oracle import Oracle
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from test_parity_gpu import CASES
    o = Oracle()
    s = rdd.Solver(0)
    names = sys.argv[2:] or ["cluster2_jacobi", "cluster4_jacobi", "runner77", "scaling_as", "example3", "example2"]
    for name in names:
        cfg = CASES[name]
        so = o.run_single(cfg)
        oa, oe = o.getd("approx"), o.getd("exact")
        o.build_instance(cfg).assemble(True).build_preconditioner(A.PRECOND_AS)
        p = int(o.geti("p")[0])
        v = np.random.default_rng(7).standard_normal(p)
        zo = o.precond_apply(v)
        for frc in (1e11, 1e9, 1e7, 0.0):
            s.set_param("full_rank_cond", frc)
            sd = s.run_single(cfg)
            zd = s.precond_apply(v)
            print(json.dumps({"case": name, "full_rank_cond": frc, "n_fallback": int(s.geti("n_fallback")[0]),
                              "its_dev": sd["iterations"], "its_orc": so["iterations"],
                              "apply_rel": float(np.linalg.norm(zd - zo) / np.linalg.norm(zo)),
                              "e_dev": sd["e_l2"], "e_orc": so["e_l2"],
                              "u_rel": float(np.linalg.norm(s.getd("approx") - oa) / np.linalg.norm(oe)),
                              "res_dev": sd["final_residual"], "res_orc": so["final_residual"],
                              "t_precond": sd["t_precond"]}), flush=True)


if __name__ == "__main__":
    {"full": full, "cluster": cluster}[sys.argv[1]]()
