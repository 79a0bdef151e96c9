import sys; sys.path.insert(0,'/root/repo')
import numpy as np
from paper_2412_19207_b200 import rdd, configs
for name in ("C3","C5"):
    cfg = configs.aspcg(name); s = rdd.Solver(0); r = s.run_single(cfg)
    n = s.geti("local_n").astype(np.int64); T = (n + 63)//64
    pb = (T*(T+1)//2*64*64*8).sum()
    print(name, "P GB", pb/1e9, "apply bytes (2 passes) GB", 2*pb/1e9, "iters", r["iterations"], "t_solve", r["t_solve"])
