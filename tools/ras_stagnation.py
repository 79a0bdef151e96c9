"""RAS-GMRES(50) on slices of C4 / C3 with the full m and points per subdomain: does the method
stagnate on the CPU oracle (the reference restated) as it does on the device?

  python tools/ras_stagnation.py oracle   -> profiles/ras_gmres_slices_oracle_r02.jsonl
  python tools/ras_stagnation.py device   -> stdout (run on the GPU box)
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_2412_19207_b200 import abi as A  # noqa: E402
from paper_2412_19207_b200 import configs  # noqa: E402

CAP = 1500


def cases():
    c4 = configs.c4()  # 64x16, m=250, 40x40 points per subdomain
    yield "C4_16x4", configs.scaled(c4, [16, 4], 40)
    yield "C4_8x8", configs.scaled(c4, [8, 8], 40)
    c3 = configs.c3()  # 8x8x8, m=300, 16^3 per subdomain
    yield "C3_3x3x2", configs.scaled(c3, [3, 3, 2], 16)


def main():
    side = sys.argv[1]
    if side == "oracle":
        from oracle import Oracle
        runner = Oracle(threads=os.cpu_count() or 1)
    else:
        from paper_2412_19207_b200 import rdd
        runner = rdd.Solver(0)
    out = []
    for name, cfg in cases():
        cfg.solver, cfg.precond, cfg.gmres_restart, cfg.max_iter = A.SOLVER_GMRES, A.PRECOND_RAS, 50, CAP
        t = time.perf_counter()
        s = runner.run_single(cfg)
        h = runner.getd("hist", 0)
        rec = {"case": name, "side": side, "J": s["J"], "DoF": s["DoF"], "iterations": s["iterations"],
               "converged": s["converged"], "final_residual": float(h[-1]), "e_l2": s["e_l2"],
               "hist_every_50": [float(x) for x in h[::50]], "wall_s": time.perf_counter() - t}
        print(json.dumps(rec), flush=True)
        out.append(rec)
    if side == "oracle":
        with open(os.path.join(ROOT, "profiles", "ras_gmres_slices_oracle_r02.jsonl"), "w") as f:
            for r in out:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
