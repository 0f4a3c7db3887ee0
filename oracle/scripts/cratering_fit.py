"""TEST INFRASTRUCTURE: run the sphere-cratering sweep (6 cases) on the fp64 oracle, the
sphere's depth measured at rest (reading A23, workloads/crater.py `penetration`), and store D and
the fit in tests/golden/cratering_oracle_d<d0 in 0.1 mm>_E<E>.json.  Calls only oracle/ and
workloads/ (no CUDA path).  Usage: python oracle/scripts/cratering_fit.py [d0] [E]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from workloads import crater as cr  # noqa: E402

d0 = float(sys.argv[1]) if len(sys.argv) > 1 else 5e-3
E = float(sys.argv[2]) if len(sys.argv) > 2 else 1e6
rows = []
for rho_s, H in cr.CASES:
    sc = cr.scenario(rho_s, H, d0=d0, E=E)
    s = oracle.load_scenario(sc)
    t0 = time.time()
    res = cr.penetration(s, sc)
    res.update(rho_s=rho_s, H=H, x=cr.law_abscissa(rho_s, H), D_law=0.14 * cr.law_abscissa(rho_s, H),
               wall_s=time.time() - t0)
    print(res, flush=True)
    rows.append(res)
f = cr.fit([r["x"] for r in rows], [r["D"] for r in rows])
f_first = cr.fit([r["x"] for r in rows], [r["D_first_stop"] for r in rows])
out = {"_cite": "P:5-12 (setup, Eq. ballDropEquation), P:60 (paper fit: slope 0.1336, R2 0.9714, MSE 1e-7 m^2); "
                "depth at rest (reading A23); written by oracle/scripts/cratering_fit.py (oracle only)",
       "d0": d0, "E": E, "cases": rows, "fit": f, "fit_first_stop": f_first, "threads": oracle.num_threads()}
path = os.path.join(ROOT, "tests", "golden", f"cratering_oracle_d{int(round(d0 * 1e4))}_E{E:.0e}.json")
json.dump(out, open(path, "w"), indent=1)
print(json.dumps(f), "->", path)
