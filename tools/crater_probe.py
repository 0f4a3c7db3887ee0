import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from workloads import crater as cr
from paper_2507_05643_b200 import crm
for d0 in (5e-3, 2.5e-3):
    for rho_s, H in [(700.0, 0.05), (2200.0, 0.2)]:
        sc = cr.scenario(rho_s, H, d0=d0)
        g = crm.load_scenario(sc)
        z0 = sc.meta["z0"]
        out = []
        for k in range(60):
            g.step(sc.dt, 40)
            b = g.get_body(1)
            out.append((round((k + 1) * 40 * sc.dt * 1e3, 1), round((z0 - b["pos"][2]) * 1e3, 2), round(b["vel"][2], 3), round(b["force"][2], 3)))
        print("d0", d0, "rho_s", rho_s, "H", H, "D_law mm", round(0.14 * cr.law_abscissa(rho_s, H) * 1e3, 2))
        print(out[:30])
        print(out[30:])
