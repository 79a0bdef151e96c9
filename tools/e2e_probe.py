import sys, time; sys.path.insert(0,'/root/repo')
from paper_2412_19207_b200 import rdd, configs
cfg = configs.aspcg("C2"); s = rdd.Solver(0); s.run_single(cfg)
for i in range(3):
    t = time.perf_counter(); r = s.run_single(cfg); w = time.perf_counter() - t
    r2 = s.rerun_resident()
    print("e2e wall", round(w*1e3,2), "ms; phases e2e", round(1e3*(r["t_assemble"]+r["t_precond"]+r["t_solve"]+r["t_evaluate"]),2), "resident", round(1e3*(r2["t_assemble"]+r2["t_precond"]+r2["t_solve"]+r2["t_evaluate"]),2), "pca e2e", round(1e3*r["t_pca"],2), "pca res", round(1e3*r2["t_pca"],2))
s.set_verbose(True); s.run_single(cfg); s.set_verbose(False)
