"""Per-family device time of the PCA phase (run_pca) for BASELINE configs."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_19207_b200 import configs, rdd  # noqa: E402

FAM = ("pca_total", "assemble", "gram", "syevj", "pca_refine", "pca_house", "pca_stage2_gemm", "project", "index",
       "problem")
s = rdd.Solver(0)
for name in sys.argv[1:] or ["C2", "C5"]:
    cfg = configs.aspcg(name)
    s.run_single(cfg)
    s.set_timing(True)
    s.reset_stats()
    r = s.rerun_resident()
    st = {f: s.kernel_stats(f) for f in FAM}
    s.set_timing(False)
    print(json.dumps({"config": name, "t_pca": r["t_pca"], "stats": {k: v for k, v in st.items() if v[1]}}), flush=True)
