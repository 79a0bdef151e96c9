"""Setup + one resident solve of a named config (for ncu launch lists)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_19207_b200 import rdd, configs
cfg = configs.BASELINE[sys.argv[1]]()
s = rdd.Solver(0)
s.run_single(cfg)
print(s.rerun_resident())
