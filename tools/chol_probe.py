"""One C3 4x4x4 slice (large-block Cholesky path) setup + rerun, for ncu captures of the Schwarz build."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_19207_b200 import rdd, configs, abi as A
cfg = configs.scaled(configs.c3(), [4, 4, 4], 16)
cfg.solver, cfg.precond = A.SOLVER_CG, A.PRECOND_AS
s = rdd.Solver(0)
s.run_single(cfg)
s.set_timing(True)
s.reset_stats()
r = s.rerun_resident()
n = s.geti("local_n")
print({k: r[k] for k in ("iterations", "t_pca", "t_precond", "t_solve")}, "n_max", n.max(), "sum n3/3", float((n.astype(float)**3/3).sum()),
      {f: s.kernel_stats(f) for f in ("cholesky", "gemm_nt", "inv_power", "schwarz_gather", "potrf")})
