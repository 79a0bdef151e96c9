"""Schwarz apply (AS) and normal operator: time, algorithmic bytes and bandwidth per BASELINE config."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_19207_b200 import abi as A  # noqa: E402
from paper_2412_19207_b200 import configs, rdd  # noqa: E402

s = rdd.Solver(0)
for name in sys.argv[1:] or ["C2", "C4", "C3", "C5"]:
    cfg = configs.aspcg(name)
    s.build_instance(cfg).assemble(True).build_preconditioner(cfg.precond)
    ms, by = s.bench_precond(False, reps=20)
    oms, oby = s.bench_operator(A.OPERATOR_TWO_PASS, reps=20)
    print(json.dumps({"config": name, "inv_mode": int(s.geti("inv_mode")[0]), "apply_ms": ms, "apply_bytes": by,
                      "apply_gbs": by / ms / 1e6, "operator_ms": oms, "operator_bytes": oby,
                      "operator_gbs": oby / oms / 1e6}), flush=True)
