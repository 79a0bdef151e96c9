"""Stage-2 Jacobi time on C5 (syevj family) for cluster-shape experiments (RDD_JACOBI_K / _NT)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_19207_b200 import configs, rdd  # noqa: E402

s = rdd.Solver(0)
cfg = configs.aspcg(sys.argv[1] if len(sys.argv) > 1 else "C5")
s.run_single(cfg)
s.set_timing(True)
s.reset_stats()
r = s.rerun_resident()
print(os.environ.get("RDD_JACOBI_K"), os.environ.get("RDD_JACOBI_NT"), "syevj", s.kernel_stats("syevj"), "t_pca", r["t_pca"],
      "DoF", r["DoF"], "its", r["iterations"], "e_l2", r["e_l2"])
