import sys; sys.path.insert(0,'/root/repo')
from paper_2412_19207_b200 import rdd, configs, abi as A
for name in ("C3", "C5"):
    cfg = configs.aspcg(name); s = rdd.Solver(0); s.run_single(cfg); s.set_verbose(True); s.rerun_resident(); s.set_verbose(False)
