"""Per-family device time of the Schwarz build (cholesky = whole factor [+ inverse] family; potrf =
its diagonal steps; gemm_* = every DMMA GEMM launched meanwhile) for BASELINE configs."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_19207_b200 import configs, rdd  # noqa: E402

s = rdd.Solver(0)
for name in sys.argv[1:] or ["C1", "C2", "C4"]:
    cfg = configs.aspcg(name)
    s.run_single(cfg)
    s.build_instance(cfg).assemble(True)
    s.set_timing(True)
    s.reset_stats()
    s.build_preconditioner(cfg.precond)
    st = {f: s.kernel_stats(f) for f in ("cholesky", "potrf", "gemm_nt", "gemm_nn", "gemm_tn", "inv_power", "power",
                                          "normal_blocks", "schwarz_build", "schwarz_gather", "schwarz_alloc")}
    s.set_timing(False)
    n = s.geti("local_n").astype(np.float64)
    print(json.dumps({"config": name, "sum_n3_3": float((n ** 3 / 3).sum()), "n_mean": float(n.mean()),
                      "stats": {k: v for k, v in st.items() if v[1]}}), flush=True)
