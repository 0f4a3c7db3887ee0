"""Per-kernel device time of the MGRU3 wheel bin with active domains on/off:
python tools/active_prof.py [steps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2507_05643_b200 import crm  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for on in (False, True):
    sc = workloads.mgru3_wheel(active=on)
    g = crm.load_scenario(sc)
    g.step(sc.dt, 3)
    g.profile(True)
    g.profile_reset()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g.step(sc.dt, steps)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / steps * 1e3
    prof = g.profile_read()
    dev = sum(v[0] for v in prof.values()) / steps
    print(f"active={on}: wall {wall:.3f} ms/step, kernels {dev:.3f} ms/step", g.active_stats() if on else "")
    for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0]):
        print(f"   {k:18s} {v[0] / steps:8.4f} ms  x{v[1] // steps}")
    g.close()
