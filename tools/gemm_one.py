"""One GEMM batch for ncu captures: python tools/gemm_one.py [nt|nn|tn|tn80]
(nt: the Schwarz Cholesky trailing-update shape; nn: S·Q of C5; tn / tn80: Sᵀ·Z of C5 with the
64- and 80-wide CTA tiles)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_19207_b200 import rdd  # noqa: E402

SHAPES = {"nt": (2, 5184, 5184, 512, 8), "nn": (0, 13824, 386, 400, 32), "tn": (1, 400, 386, 13824, 64),
          "tn80": (11, 400, 386, 13824, 64)}
s = rdd.Solver(0)
for which in sys.argv[1:] or ["nt"]:
    mode, M, N, K, b = SHAPES[which]
    ms = s.bench_gemm(mode, M, N, K, b, reps=1)
    print(which, "ms", ms, "TF/s", 2.0 * M * N * K * b / ms / 1e9)
