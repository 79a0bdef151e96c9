import sys, time, numpy as np
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_19207_b200 import rdd
s = rdd.Solver(0)
for n in (1000, 2000):
    a = np.random.default_rng(n).standard_normal((n, n))
    s.spectrum(a[:100,:100])
    s.set_timing(True); s.reset_stats()
    t = time.perf_counter(); s.spectrum(a); dt = time.perf_counter() - t
    print(n, dt, {f: s.kernel_stats(f) for f in ("diag_eig", "diag_hessenberg", "diag_qr", "diag_shifts", "diag_sweep", "diag_block", "diag_windows")})
    s.set_timing(False)
