"""Run a BASELINE config (optionally sliced) once with setup + one resident rerun; print summary + timing."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_19207_b200 import rdd, configs, abi as A
name = sys.argv[1]
cfg = configs.BASELINE[name]()
if len(sys.argv) > 3 and sys.argv[2]:
    counts = [int(x) for x in sys.argv[2].split(",")]
    cfg = configs.scaled(cfg, counts, int(sys.argv[3]))
for kv in sys.argv[4:]:
    k, v = kv.split("=")
    setattr(cfg, k, type(getattr(cfg, k))(float(v)) if isinstance(getattr(cfg, k), float) else int(v))
s = rdd.Solver(0)
s.set_verbose(True)
t = time.time()
r = s.run_single(cfg)
t1 = time.time() - t
s.rerun_resident()  # first rerun may still grow workspaces; report the steady state
t = time.time()
r2 = s.rerun_resident()
t2 = time.time() - t
print(json.dumps({"config": name, "counts": list(cfg.counts)[:cfg.d], "m": cfg.m, "first_s": t1, "rerun_s": t2,
                  "p_j_min": int(s.geti("p_j").min()), "p_j_max": int(s.geti("p_j").max()),
                  "n_fallback": int(s.geti("n_fallback")[0]), **{k: r2[k] for k in r2}}))
