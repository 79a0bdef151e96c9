"""RAS apply with owner-row panels: bytes, time and the RAS-GMRES(50) step time on C4 (and C2)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_19207_b200 import abi as A  # noqa: E402
from paper_2412_19207_b200 import configs, rdd  # noqa: E402

s = rdd.Solver(0)
for name in sys.argv[1:] or ["C4", "C2"]:
    cfg = configs.BASELINE[name](max_iter=300)
    cfg.solver, cfg.precond, cfg.gmres_restart = A.SOLVER_GMRES, A.PRECOND_RAS, 50
    s.run_single(cfg)
    r = s.rerun_resident()
    ms, by = s.bench_precond(False, reps=20)
    mst, byt = s.bench_precond(True, reps=20)
    print(json.dumps({"config": name, "ras_apply_ms": ms, "ras_apply_bytes": by, "ras_apply_gbs": by / ms / 1e6,
                      "ras_transpose_ms": mst, "gmres_its": r["iterations"], "t_solve": r["t_solve"],
                      "ms_per_gmres_step": 1e3 * r["t_solve"] / max(1, r["iterations"])}), flush=True)
