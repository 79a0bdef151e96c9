"""One C2 solve on resident inputs after a setup run (for ncu launch lists / captures)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_19207_b200 import rdd, configs
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = configs.aspcg(name)
s = rdd.Solver(0)
s.run_single(cfg)
r = s.rerun_resident()
print({k: r[k] for k in ("iterations", "e_l2", "t_pca", "t_precond", "t_solve")})
