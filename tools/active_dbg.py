"""Small active-domain wheel run for compute-sanitizer: python tools/active_dbg.py [nx]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads  # noqa: E402
from paper_2507_05643_b200 import crm  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 120
prof = len(sys.argv) > 2
sc = workloads.mgru3_wheel(n=(nx, 40, 25), active=True)
g = crm.load_scenario(sc)
if prof:
    g.profile(True)
for k in range(6):
    g.step(sc.dt, 1)
    print(k, g.active_stats(), flush=True)
print("ok")
