"""GPU sweep of the six sphere drops with the depth measured at rest (reading A23):
python tools/crater_sweep_gpu.py [d0] -> one JSON line per (E, ps_freq) variant with the depths and
the fits (slope through the origin, OLS slope, R^2, MSE against D = 0.14 x)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from workloads import crater as cr  # noqa: E402
from paper_2507_05643_b200 import crm  # noqa: E402

d0 = float(sys.argv[1]) if len(sys.argv) > 1 else 2.5e-3
for E in (1e6, 2e5):
    for ps in (1, 10):
        rows = []
        for rho_s, H in cr.CASES:
            sc = cr.scenario(rho_s, H, d0=d0, E=E)
            sc.params["ps_freq"] = ps
            g = crm.load_scenario(sc)
            res = cr.penetration(g, sc)
            res.update(rho_s=rho_s, H=H, x=cr.law_abscissa(rho_s, H))
            rows.append(res)
            g.close()
        f = cr.fit([r["x"] for r in rows], [r["D"] for r in rows])
        f1 = cr.fit([r["x"] for r in rows], [r["D_first_stop"] for r in rows])
        print(json.dumps(dict(d0=d0, E=E, ps_freq=ps, fit=f, fit_first_stop=f1,
                              D_mm=[round(r["D"] * 1e3, 3) for r in rows],
                              D_first_mm=[round(r["D_first_stop"] * 1e3, 3) for r in rows],
                              at_rest=[r["at_rest"] for r in rows], t=[r["t"] for r in rows],
                              law_mm=[round(0.14 * r["x"] * 1e3, 3) for r in rows])), flush=True)
