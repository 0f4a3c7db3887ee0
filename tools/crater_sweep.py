import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads
from workloads import crater as cr
from paper_2507_05643_b200 import crm
d0 = float(sys.argv[1]) if len(sys.argv) > 1 else 2.5e-3
variants = [("E1e6", {}), ("E2e5", {"E": 2e5}), ("E5e4", {"E": 5e4}), ("E1e6_noAV", {"gamma_a": 0.0})]
for name, var in variants:
    xs, Ds, Dfin = [], [], []
    for rho_s, H in cr.CASES:
        sc = cr.scenario(rho_s, H, d0=d0)
        if "E" in var:
            K, G = workloads.elastic_moduli(var["E"], 0.3)
            sc.params["K"], sc.params["G"] = K, G
        if "gamma_a" in var:
            sc.params["gamma_a"] = var["gamma_a"]
        g = crm.load_scenario(sc)
        res = cr.penetration(g, sc)
        g.step(sc.dt, 1000)
        xs.append(cr.law_abscissa(rho_s, H)); Ds.append(res["D"]); Dfin.append(sc.meta["z0"] - g.get_body(1)["pos"][2])
    f = cr.fit(xs, Ds)
    print(name, "D mm", [round(d * 1e3, 2) for d in Ds], "D+50ms", [round(d * 1e3, 2) for d in Dfin], "law", [round(0.14 * x * 1e3, 2) for x in xs], json.dumps(f), flush=True)
