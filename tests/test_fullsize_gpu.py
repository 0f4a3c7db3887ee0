"""Parity at BASELINE.json's full size (C5, the 32M-particle bed that bench.py times), on sampled
outputs the oracle can compute: eight patches of fluid particles (interior, next to a side wall, in a
floor corner, at the free surface).  For each patch the oracle runs on the sub-problem of every
particle within 5 cells (10 h) of the patch centre cell — enough for the samples' stage-A and stage-B
rates to be exact (their neighbours within 2h, those neighbours' neighbours and the markers'
extrapolation sources).  Bars: neighbour counts bit-exact, rates 1e-4 relative L-inf per field."""
import numpy as np
import pytest

import oracle
import workloads

pytestmark = pytest.mark.gpu


def cell_coords(pos, params):
    s = np.float32(2.0 * params["h"])
    lo = np.asarray(params["lo"], np.float32)
    return np.floor((pos.astype(np.float32) - lo) / s).astype(np.int64)


CONFIGS = {"bed32M": workloads.bed, "cone1M": workloads.cone_bed, "mgru3": workloads.mgru3_bin}


@pytest.mark.parametrize("name", list(CONFIGS))
def test_full_size_sampled_parity(name):
    from paper_2507_05643_b200 import build
    build.build_library()
    from paper_2507_05643_b200 import crm
    # the rate-parity state recipe S0 on the full-size geometry: jitter 0.1 d0,
    # u = A x + noise, lithostatic + noisy stress.  A state at rest would make the stage-B rates a
    # near-total cancellation (every u_mid = dt/2 g), where the fp32 vs fp64 mid states alone
    # exceed 1e-4 of the (tiny) field.
    sc = workloads.rate_state_S0(CONFIGS[name](), A_scale=0.5)
    nf = sc.n_fluid
    allpos = np.concatenate([sc.fluid_pos, sc.wall_pos])
    cells = cell_coords(allpos, sc.params)
    fcells = cells[:nf]
    mn, mx = fcells.min(0), fcells.max(0)
    rng = np.random.default_rng(2024)
    margin = np.minimum(6, (mx - mn) // 2 - 1)       # the C4 bin is ~10 cells deep
    centres = [rng.integers(mn + margin, mx - margin + 1) for _ in range(4)]
    mid = (mn + mx) // 2
    centres += [np.array([mn[0], mid[1], mid[2]]),                    # next to the x = 0 wall
                mn.copy(),                                            # floor corner
                np.array([(mn[0] + mx[0]) // 3, mid[1], mx[2]]),      # free surface
                np.array([mid[0], mn[1], mx[2]])]                     # surface at the y = 0 wall

    g = crm.load_scenario(sc)
    st = g.structure()
    g.debug_arm(True)
    g.step(sc.dt, 1)
    rates_g = [g.last_rates(0), g.last_rates(1)]
    g.close()

    worst = 0.0
    for c in centres:
        d = np.abs(cells - c).max(axis=1)
        sub = np.nonzero(d <= 5)[0]
        samp_mask = (d[sub] <= 1) & (sub < nf)
        assert samp_mask.sum() > 20
        subf = sub[sub < nf]
        subw = sub[sub >= nf]
        o = oracle.OracleSim(sc.params)
        o.add_fluid(sc.fluid_pos[subf], sc.fluid_vel[subf], sc.fluid_sig[subf])
        if len(subw):
            o.add_bce(0, sc.wall_pos[subw - nf])
        local = np.concatenate([subf, subw])            # oracle row -> global id
        samp_rows = np.nonzero((np.abs(cells[local] - c).max(axis=1) <= 1) & (local < nf))[0]
        samp_ids = local[samp_rows]
        so = o.structure()
        assert np.array_equal(so["counts"][samp_rows], st["counts"][samp_ids])
        o.step(sc.dt, 1)
        for stage in (0, 1):
            for a_g, a_o in zip(rates_g[stage], o.last_rates(stage)):
                ga, oa = a_g[samp_ids], a_o[samp_rows]
                err = np.abs(ga - oa).max() / max(np.abs(oa).max(), 1e-30)
                worst = max(worst, err)
                assert err <= 1e-4, (c, stage, err)
        o.close()
    print("worst relative L-inf over the sampled patches", worst)
