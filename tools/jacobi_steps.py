import json, os, sys
sys.path.insert(0, '/root/repo')
from paper_2412_19207_b200 import rdd
s = rdd.Solver(0)
for n, B, sw in [(386, 512, 7), (386, 148, 7), (113, 256, 7), (200, 512, 7)]:
    ms = s.bench_jacobi(n, B, sw)
    print(json.dumps({"K_env": os.environ.get("RDD_JACOBI_K"), "n": n, "B": B, "sweeps": sw, "ms": round(ms, 3), "us_per_step": round(1e3 * ms / (sw * (n + (n & 1))), 2)}))
