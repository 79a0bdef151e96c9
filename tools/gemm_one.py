"""One large NT GEMM batch (the Schwarz Cholesky trailing-update shape) for ncu captures."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_19207_b200 import rdd  # noqa: E402

s = rdd.Solver(0)
ms = s.bench_gemm(2, 5184, 5184, 512, 8, reps=1)
print("ms", ms, "TF/s", 2.0 * 5184 * 5184 * 512 * 8 / ms / 1e9)
