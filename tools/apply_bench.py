"""Schwarz AS apply and operator bandwidth on BASELINE configs (tuning aid)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_19207_b200 import configs, rdd  # noqa: E402

s = rdd.Solver(0)
for name in sys.argv[1:] or ["C1", "C2", "C4"]:
    cfg = configs.aspcg(name)
    r = s.run_single(cfg)
    ms, by = s.bench_precond(False, reps=20)
    print(json.dumps({"config": name, "apply_ms": ms, "apply_GB": by / 1e9, "apply_GBs": by / ms / 1e6,
                      "its": r["iterations"], "t_solve": r["t_solve"], "e_l2": r["e_l2"]}), flush=True)
