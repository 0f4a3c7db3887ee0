"""Single-wheel rig with and without active domains (diagnostic for tests/test_active_gpu.py):
python tools/wheel_loads.py [steps_per_sample] [samples] [free]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads  # noqa: E402
from paper_2507_05643_b200 import crm  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 5
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 80
free = len(sys.argv) > 3 and sys.argv[3] == "free"
series = {}
for on in (False, True):
    sc = workloads.mgru3_wheel(n=(160, 60, 25), active=on, free=free)
    g = crm.load_scenario(sc)
    fs = []
    for _ in range(ns):
        g.step(sc.dt, k)
        b = g.get_body(1)
        fs.append(np.concatenate([b["force"], b["pos"], b["vel"]]))
    series[on] = np.array(fs)
    g.close()
off, on = series[False], series[True]
for t in range(0, ns, max(1, ns // 40)):
    print(f"{(t + 1) * k:5d}  off F {off[t, 0]:8.2f} {off[t, 2]:8.2f} x {off[t, 3]:.4f} z {off[t, 5]:.4f} vx {off[t, 6]:.4f}"
          f"   on F {on[t, 0]:8.2f} {on[t, 2]:8.2f} x {on[t, 3]:.4f} z {on[t, 5]:.4f} vx {on[t, 6]:.4f}")
h = ns // 2
for a, nm in ((0, "Fx"), (2, "Fz"), (5, "z"), (6, "vx")):
    print(nm, "mean of 2nd half off/on", off[h:, a].mean(), on[h:, a].mean())
