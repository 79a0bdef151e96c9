"""Normal-operator time and achieved GB/s for a config (resident system, CUDA events)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_19207_b200 import rdd, configs, abi as A
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
s = rdd.Solver(0)
cfg = configs.BASELINE[name]()
cfg.solver, cfg.precond = A.SOLVER_CG, A.PRECOND_AS  # the operator does not depend on the solver
s.run_single(cfg)
ms, by = s.bench_operator(A.OPERATOR_TWO_PASS, reps=50)
print(json.dumps({"config": name, "op_ms": ms, "GBps": by / ms / 1e6, "frac": by / ms / 1e6 / 6458.7}))
