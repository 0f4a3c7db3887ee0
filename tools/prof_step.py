"""Run a few steps of a bench workload (for ncu captures): python tools/prof_step.py CONFIG STEPS"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2507_05643_b200 import crm  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "bed256x256x64"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
sc = bench.scenario(cfg)
g = crm.load_scenario(sc)
g.step(sc.dt, steps)
print("done", cfg, steps, g.launch_count())
