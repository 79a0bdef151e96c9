"""One batched Jacobi probe call (n, B, sweeps from argv) for ncu captures."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_19207_b200 import rdd
n, B, sw = (int(x) for x in sys.argv[1:4])
print(rdd.Solver(0).bench_jacobi(n, B, sw))
