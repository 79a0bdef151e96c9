"""Per-subdomain PCA agreement with the full-size oracle fixtures (and live oracle on C5s):
rank, probe projector difference, and the relative spectral gap at the threshold."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_19207_b200 import configs, rdd  # noqa: E402

PROBE_SEED = 20250


def main():
    s = rdd.Solver(0)
    args = sys.argv[1:]
    if args and args[0].startswith("refine="):
        s.set_param("pca_refine", float(args[0].split("=")[1]))
        args = args[1:]
    while args and args[0].startswith("stop="):
        s.set_param("pca_stop", float(args[0].split("=")[1]))
        args = args[1:]
    for name in args or ["C3", "C5", "C2", "C4"]:
        kind = "pca" if name in ("C3", "C5") else "run"
        fx = np.load(os.path.join(ROOT, "tests", "golden", "fullsize", f"{kind}_{name}.npz"))
        cfg = configs.BASELINE[name]()
        s.build_instance(cfg)
        s.set_timing(True)
        s.reset_stats()
        s.build_instance(cfg)
        tm = {f: s.kernel_stats(f)[0] for f in ("pca_total", "syevj", "pca_refine", "pca_house", "pca_stage2_gemm")}
        s.set_timing(False)
        pd = s.geti("p_j")
        rows = []
        for j in range(len(pd)):
            so = fx["sigma"][fx["sigma_off"][j]:fx["sigma_off"][j + 1]]
            sd = s.getd("sigma", j)
            V = s.getd("V", j).reshape(int(pd[j]), cfg.m).T
            x = np.random.default_rng(PROBE_SEED + j).standard_normal(cfg.m)
            pr = np.linalg.norm(V @ (V.T @ x) - fx["probe_px"][j]) / np.linalg.norm(x)
            p = int(fx["p_j"][j])
            gap = (so[p - 1] - (so[p] if p < len(so) else 0.0)) / so[0]
            rows.append((pr, j, int(pd[j]), p, so[p - 1] / so[0], so[p] / so[0] if p < len(so) else 0.0, gap,
                         float(np.max(np.abs(sd[:len(so)] - so) / so[0]))))
        rows.sort(reverse=True)
        print(json.dumps({"config": name, "ms": tm, "rank_mismatch": int(np.sum(pd != fx["p_j"])),
                          "worst": [dict(zip(("probe", "j", "p_dev", "p_ref", "s_p", "s_p1", "gap", "sig_abs_rel"), r))
                                    for r in rows[:6]],
                          "probe_quantiles": [float(np.quantile([r[0] for r in rows], q)) for q in (0.5, 0.9, 0.99)]}),
              flush=True)


if __name__ == "__main__":
    main()
