import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads
from paper_2507_05643_b200 import crm, dist
sc = workloads.bed(n=(64, 24, 12))
world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
ref = crm.load_scenario(sc)
c0 = crm.load_scenario(sc, rank=0, world=world)
ctxs = [c0] + [crm.load_scenario(sc, rank=r, world=world, stream=c0.stream()) for r in range(1, world)]
for s in range(steps):
    try:
        crm.group_step(ctxs, sc.dt, 1)
    except crm.CrmError as e:
        print("step", s, "error", e); break
    ref.step(sc.dt, 1)
    got = dist.merge_owned([c.get_state() for c in ctxs])
    r = ref.get_state()
    nan = int(np.isnan(got[2]).sum())
    diff = [float(np.nanmax(np.abs(a - b))) for a, b in zip(got, r)]
    print("step", s, "owned", [c.count(crm.CRM_OWNED) for c in ctxs], "nan rows", nan, "maxdiff", diff, flush=True)
