import sys; sys.path.insert(0,'/root/repo')
from paper_2412_19207_b200 import rdd, configs, abi as A
for name in ("C2","C4"):
    cfg = configs.aspcg(name); s = rdd.Solver(0); s.run_single(cfg)
    s.build_instance(cfg); s.assemble(True); s.set_verbose(True); s.build_preconditioner(A.PRECOND_AS); s.set_verbose(False)
