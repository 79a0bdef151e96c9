"""Wall vs device time of build_preconditioner (normal blocks + Schwarz build) on a resident config."""
import ctypes as C, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_19207_b200 import rdd, configs, abi as A
cfg = configs.aspcg(sys.argv[1] if len(sys.argv) > 1 else "C2")
s = rdd.Solver(0)
s.run_single(cfg)
for rep in range(4):
    s.build_instance(cfg)
    s.assemble(True)
    s.L.rdd_event_record(s.h, 0)
    t = time.perf_counter()
    s.build_preconditioner(A.PRECOND_AS)
    w = time.perf_counter() - t
    s.L.rdd_event_record(s.h, 1)
    ms = C.c_double()
    s.L.rdd_event_elapsed(s.h, 0, 1, C.byref(ms))
    print(f"build_preconditioner: wall {w*1e3:.2f} ms, events {ms.value:.2f} ms")
s.set_timing(True)
s.reset_stats()
s.build_preconditioner(A.PRECOND_AS)
print({f: s.kernel_stats(f) for f in ("normal_blocks", "schwarz_build", "schwarz_gather", "cholesky", "gemm_nt", "gemm_nn", "gemm_tn", "inv_power", "power", "potrf")})
