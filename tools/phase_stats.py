"""Per-family device time (CUDA events around each host-side phase) for one resident rerun."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_19207_b200 import rdd, configs
FAMILIES = ["index", "problem", "assemble", "assemble_psi", "pca_total", "syevj", "project", "gemm_tn", "gemm_nn",
            "gemm_nt", "equilibrate", "matvec", "matvec_t", "normal_blocks", "normal_apply",
            "schwarz_build", "schwarz_alloc", "schwarz_gather", "cholesky", "inv_power", "power", "gram", "precond_apply", "solve", "evaluate"]
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = configs.aspcg(name)
for kv in sys.argv[2:]:
    k, v = kv.split("=")
    setattr(cfg, k, type(getattr(cfg, k))(float(v)) if isinstance(getattr(cfg, k), float) else int(v))
s = rdd.Solver(0)
s.run_single(cfg)
s.set_timing(True)
s.reset_stats()
r = s.rerun_resident()
out = {f: s.kernel_stats(f) for f in FAMILIES}
print(json.dumps({"config": name, "summary": {k: r[k] for k in ("iterations", "t_pca", "t_assemble", "t_precond",
                                                                "t_solve")},
                  "families_ms": {f: round(v[0], 3) for f, v in out.items() if v[1]},
                  "calls": {f: v[1] for f, v in out.items() if v[1]}}))
