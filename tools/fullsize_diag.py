import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle, workloads
from paper_2507_05643_b200 import crm
sc = workloads.cone_bed()
sc.fluid_sig = np.zeros((sc.n_fluid, 6))
nf = sc.n_fluid
allpos = np.concatenate([sc.fluid_pos, sc.wall_pos])
s = np.float32(2.0 * sc.params["h"]); lo = np.asarray(sc.params["lo"], np.float32)
cells = np.floor((allpos.astype(np.float32) - lo) / s).astype(np.int64)
c = np.array([1, 20, 20])
g = crm.load_scenario(sc); g.debug_arm(True); g.step(sc.dt, 1)
rg = [g.last_rates(0), g.last_rates(1)]
ug = [g.last_bce(0), g.last_bce(1)]
d = np.abs(cells - c).max(axis=1); sub = np.nonzero(d <= 5)[0]
subf = sub[sub < nf]; subw = sub[sub >= nf]
o = oracle.OracleSim(sc.params); o.add_fluid(sc.fluid_pos[subf], None, sc.fluid_sig[subf]); o.add_bce(0, sc.wall_pos[subw - nf])
local = np.concatenate([subf, subw])
rows = np.nonzero((np.abs(cells[local] - c).max(axis=1) <= 1) & (local < nf))[0]
ids = local[rows]
o.step(sc.dt, 1)
for st in (0, 1):
    ro = o.last_rates(st)
    for nm, a, b in zip(("drho", "acc", "dsig"), rg[st], ro):
        ga, oa = a[ids], b[rows]
        k = np.unravel_index(np.argmax(np.abs(ga - oa)), ga.shape)
        print("stage", st, nm, "maxabs", np.abs(oa).max(), "err", np.abs(ga - oa).max(), "at", k, ga[k], oa[k])
    # markers near patch
mrows = np.nonzero((np.abs(cells[local] - c).max(axis=1) <= 2) & (local >= nf))[0]
mids = local[mrows]
for st in (0, 1):
    uo, so_ = o.last_bce(st)
    print("bce stage", st, "u err", np.abs(ug[st][0][mids] - uo[mrows]).max(), "u max", np.abs(uo[mrows]).max(),
          "sig err", np.abs(ug[st][1][mids] - so_[mrows]).max(), "sig max", np.abs(so_[mrows]).max())
