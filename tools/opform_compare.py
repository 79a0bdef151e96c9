"""C2 (or argv[1]) with the two-pass operator (the reference's Hᵀ(H·w)) vs the assembled normal
blocks (HᵀH block-sparse): iterations, e_L2, solve time, operator time."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_19207_b200 import rdd, configs, abi as A
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
for of in (A.OPERATOR_TWO_PASS, A.OPERATOR_NORMAL):
    cfg = configs.aspcg(name)
    cfg.op_form = of
    s = rdd.Solver(0)
    s.run_single(cfg)
    r = s.rerun_resident()
    ms, by = s.bench_operator(of, reps=50)
    print(json.dumps({"op_form": of, "iterations": r["iterations"], "e_l2": r["e_l2"], "t_solve": r["t_solve"],
                      "op_ms": ms, "op_GBps": by / ms / 1e6, "final_residual": r["final_residual"]}))
