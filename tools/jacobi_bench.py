"""Batched Jacobi throughput probe: ms for B random n x n matrices at a fixed sweep count."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_19207_b200 import rdd
s = rdd.Solver(0)
for n, B, sw in [(300, 256, 5), (112, 256, 7), (400, 512, 5), (64, 1024, 6)]:
    ms = s.bench_jacobi(n, B, sw)
    steps = sw * (n + (n & 1))
    print(json.dumps({"n": n, "B": B, "sweeps": sw, "ms": round(ms, 3), "us_per_step_per_matrix_slot": None,
                      "ms_per_sweep": round(ms / sw, 3)}))
