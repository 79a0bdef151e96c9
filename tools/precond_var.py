"""Per-step Schwarz-build family times (CUDA events) over several resident reruns (variance hunt)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_19207_b200 import rdd, configs
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
s = rdd.Solver(0)
s.run_single(configs.aspcg(name))
fams = ["schwarz_build", "schwarz_alloc", "schwarz_gather", "cholesky", "inv_power", "normal_blocks", "gemm_nn",
        "gemm_tn", "gemm_nt"]
s.set_timing(True)
for i in range(12):
    s.reset_stats()
    r = s.rerun_resident()
    print(i, "pre %.4f" % r["t_precond"], " ".join(f"{f}={s.kernel_stats(f)[0]:.2f}" for f in fams))
