"""Run one named workload through the device pipeline with per-kernel-family timing."""
import argparse, json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
from paper_2412_19207_b200 import rdd, configs, abi as A

FAMS = ["index", "problem", "assemble", "assemble_psi", "gemm_tn", "gemm_nn", "gemm_nt", "syevj", "pca_total",
        "project", "equilibrate", "normal_blocks", "schwarz_build", "spd_inverse", "power", "solve", "matvec",
        "matvec_t", "normal_apply", "precond_apply", "evaluate"]

ap = argparse.ArgumentParser()
ap.add_argument("name")
ap.add_argument("--counts", type=int, nargs="*")
ap.add_argument("--per", type=int, default=0)
ap.add_argument("--m", type=int, default=0)
ap.add_argument("--timing", type=int, default=1)
ap.add_argument("--op", type=int, default=0)
ap.add_argument("--oracle", type=int, default=0)
a = ap.parse_args()
cfg = configs.BASELINE[a.name]()
if a.counts:
    cfg = configs.scaled(cfg, a.counts, a.per, m=a.m or None)
elif a.m:
    cfg.m = a.m
cfg.op_form = a.op
s = rdd.Solver(0)
s.set_timing(bool(a.timing))
s.set_verbose(True)
t = time.time()
r = s.run_single(cfg)
wall = time.time() - t
out = {"config": cfg.as_dict(), "summary": r, "wall": wall, "p_j_min": int(s.geti("p_j").min()),
       "p_j_max": int(s.geti("p_j").max()), "n_fallback": int(s.geti("n_fallback")[0])}
if cfg.precond >= 0:
    lr = s.geti("local_rank")
    out["local_rank_min"] = int(lr.min())
    import numpy as np
    lc = s.getd("local_cond")
    out["local_cond_max"] = float(lc.max())
out["families"] = {f: s.kernel_stats(f) for f in FAMS if s.kernel_stats(f)[1]}
print(json.dumps(out, indent=1))
if a.oracle:
    from oracle import Oracle
    t = time.time()
    ro = Oracle().run_single(cfg)
    print(json.dumps({"oracle": ro, "wall": time.time() - t}, indent=1))
