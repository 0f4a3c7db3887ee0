"""Per-rank device time of the slab step and its halo bytes: the C5 bed split into W
x-slabs as in-process contexts on one GPU (crm_group_step, loopback halos), every kernel timed per
rank with the library's event pairs; the halo bytes per exchange from the plane counts of the input
(rule B1) and the slab partition the library uses.  The NVLink transfer time is then modelled from
the bytes (it cannot be measured on one GPU).
python tools/slab_phases.py [W ...]   -> JSON on stdout"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads  # noqa: E402
from paper_2507_05643_b200 import crm, dist  # noqa: E402

STATE_B = 16 + 16 + 16 + 16 + 8      # P, L, U, S1, S2 per particle
STEPS = 4


def main():
    worlds = [int(a) for a in sys.argv[1:]] or [8]
    sc = workloads.bed(n=tuple(int(v) for v in os.environ.get("SLAB_BED", "1024x512x64").split("x")))
    lo_x, cell, nplanes = dist.grid_planes(sc.params)
    allpos = np.concatenate([sc.fluid_pos, sc.wall_pos])
    counts = dist.plane_counts(allpos, lo_x, cell, nplanes)
    out = {"workload": "bed32M", "n": int(len(allpos)), "planes": nplanes, "steps": STEPS}
    one = crm.load_scenario(sc)
    one.step(sc.dt, 3)
    one.profile(True)
    one.profile_reset()
    one.step(sc.dt, STEPS)
    p1 = one.profile_read()
    out["one_gpu_kernels_ms"] = {k: v[0] / STEPS for k, v in p1.items()}
    out["one_gpu_ms"] = sum(v[0] for v in p1.values()) / STEPS
    one.close()
    for W in worlds:
        bounds = crm.slab_partition(counts, W, 2)
        c0 = crm.load_scenario(sc, rank=0, world=W)
        ctxs = [c0] + [crm.load_scenario(sc, rank=r, world=W, stream=c0.stream()) for r in range(1, W)]
        crm.group_step(ctxs, sc.dt, 3)
        for c in ctxs:
            c.profile(True)
            c.profile_reset()
        crm.group_step(ctxs, sc.dt, STEPS)
        ranks = []
        for r, c in enumerate(ctxs):
            pr = c.profile_read()
            ks = {k: v[0] / STEPS for k, v in pr.items()}
            # halo bytes of this rank per step (both faces, send side): ghost planes of y_n with ids at
            # the rebuild (E3), y_n after BCE (E4), y_mid after stage A (E5) and after BCE (E6)
            faces = ([int(bounds[r])] if r > 0 else []) + ([int(bounds[r + 1]) - 1] if r < W - 1 else [])
            plane = [int(counts[b]) for b in faces]
            byts = {"E3": sum(plane) * (STATE_B + 4), "E4": sum(plane) * STATE_B, "E5": sum(plane) * STATE_B,
                    "E6": sum(plane) * STATE_B}
            ranks.append({"rank": r, "planes": [int(bounds[r]), int(bounds[r + 1])],
                          "owned": int(c.count(crm.CRM_OWNED)), "kernels_ms": ks,
                          "device_ms": sum(ks.values()), "halo_bytes": byts, "boundary_plane_particles": plane})
        for c in reversed(ctxs):   # rank 0 owns the shared stream: close it last
            c.close()
        dev = max(r["device_ms"] for r in ranks)
        out[f"W{W}"] = {"ranks": ranks, "max_rank_device_ms": dev,
                        "sum_rank_device_ms": sum(r["device_ms"] for r in ranks)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
