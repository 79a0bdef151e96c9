import sys; sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/oracle')
import numpy as np
from oracle import Oracle
from paper_2412_19207_b200 import abi as A, configs, rdd
cfg = configs.scaled(configs.c4(), [4, 2], 8, m=40)
cfg.solver, cfg.precond, cfg.rel_tol = A.SOLVER_GMRES, A.PRECOND_RAS, 1e-14
cfg.gmres_restart, cfg.max_iter = 3, 10
d = rdd.Solver(0); o = Oracle()
sd, so = d.run_single(cfg), o.run_single(cfg)
print("dev", sd["iterations"], sd["converged"], sd["breakdown"], d.getd("hist"))
print("orc", so["iterations"], so["converged"], o.getd("hist"))
