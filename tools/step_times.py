"""Per-step device-event time vs wall time vs summed phases for resident reruns."""
import ctypes as C, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_19207_b200 import rdd, configs
cfg = configs.aspcg(sys.argv[1] if len(sys.argv) > 1 else "C2")
s = rdd.Solver(0)
s.run_single(cfg)
for i in range(6):
    s.L.rdd_event_record(s.h, 0)
    t = time.perf_counter()
    r = s.rerun_resident()
    w = time.perf_counter() - t
    s.L.rdd_event_record(s.h, 1)
    ms = C.c_double()
    s.L.rdd_event_elapsed(s.h, 0, 1, C.byref(ms))
    ph = r["t_assemble"] + r["t_precond"] + r["t_solve"] + r["t_evaluate"]
    print(f"step {i}: event {ms.value/1e3:.4f}s wall {w:.4f}s phases {ph:.4f}s (pca {r['t_pca']:.4f} asm {r['t_assemble']-r['t_pca']:.4f} pre {r['t_precond']:.4f} sol {r['t_solve']:.4f})")
