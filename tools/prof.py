"""Profiling driver (one process, one GPU) for ncu launch lists and captures.

  python tools/prof.py step C5      one setup run + one resident rerun of run_single (launch lists)
  python tools/prof.py kernels C5   instance + preconditioner (no solve), then one normal operator and one Schwarz apply
                                    (ncu --set full with -k on the operator/apply kernels)
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_19207_b200 import configs, rdd  # noqa: E402


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "step"
    name = sys.argv[2] if len(sys.argv) > 2 else "C5"
    cfg = configs.aspcg(name) if name in configs.BASELINE else configs.c5(counts=(2, 2, 2))
    s = rdd.Solver(0)
    if mode == "step":
        r = s.run_single(cfg)
        r = s.rerun_resident()
        print({k: r[k] for k in ("J", "DoF", "iterations", "e_l2", "t_pca", "t_assemble", "t_precond", "t_solve")})
    else:  # no solve: the only operator / apply launches are the two below (one ncu capture each)
        s.build_instance(cfg).assemble(True).build_preconditioner(cfg.precond)
        p = int(s.geti("p")[0])
        v = np.random.default_rng(1).standard_normal(p)
        s.normal_apply(v)
        s.precond_apply(v)
        print({"p": p, "inv_mode": int(s.geti("inv_mode")[0])})


if __name__ == "__main__":
    main()
