import os, sys
import numpy as np
sys.path.insert(0, "/root/repo")
import workloads
from paper_2507_05643_b200 import crm
sc = workloads.mgru3_wheel(n=(160, 60, 25), active=False)
g = crm.load_scenario(sc)
prev = None
for t in range(400):
    try:
        g.step(sc.dt, 10)
    except Exception as e:
        print("fail at block", t, e)
        x, u, r, s = prev
        bad = int(str(e).split("id ")[1].split()[0])
        print("pos", x[bad], "vel", u[bad], "rho", r[bad], "sig", s[bad])
        sp = np.linalg.norm(u[:sc.n_fluid], axis=1)
        print("max speed", sp.max(), "argmax", sp.argmax(), x[sp.argmax()])
        print("wheel", g.get_body(1)["pos"] if hasattr(g, "get_body") else None)
        break
    prev = [a.copy() for a in g.get_state()]
    if t % 20 == 0:
        sp = np.linalg.norm(prev[1][:sc.n_fluid], axis=1)
        print(t, "max speed", sp.max(), "zmax", prev[0][:sc.n_fluid, 2].max(), "F", g.get_body(1)["force"])
