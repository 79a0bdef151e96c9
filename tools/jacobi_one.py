"""One batched Jacobi eigensolve (the PCA stage-2 shape of C5: order 386) for ncu captures and timing:
python tools/jacobi_one.py [n] [batch] [sweeps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_19207_b200 import rdd  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 386
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 37
sweeps = int(sys.argv[3]) if len(sys.argv) > 3 else 7
s = rdd.Solver(0)
ms = s.bench_jacobi(n, batch, sweeps)
print({"n": n, "batch": batch, "sweeps": sweeps, "ms": ms, "us_per_step": 1e3 * ms / (sweeps * (n + (n & 1)))})
