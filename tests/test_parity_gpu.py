"""GPU parity: the CUDA path (libcrm.so, through the C-ABI) against the fp64 oracle on the same
seeded inputs.  Bars (BASELINE.json north_star):
  * cell hashes, sorted order, cellStart and neighbour counts/sets: bit-exact;
  * per-step fp32 rates: relative L-inf <= 1e-4 per field (drho, acc, dsigma);
  * 100-step macroscopic outputs: within 2 %.
"""
import numpy as np
import pytest

import oracle
import workloads

pytestmark = pytest.mark.gpu

RATE_TOL = 1e-4


@pytest.fixture(scope="module")
def crm():
    from paper_2507_05643_b200 import build
    build.build_library()
    from paper_2507_05643_b200 import crm as m
    m.load_library()
    return m


def rel_linf(a, b):
    den = np.abs(b).max()
    return np.abs(a - b).max() / (den if den > 0 else 1.0)


def both(crm, sc, **kw):
    g = crm.load_scenario(sc, **kw)
    o = oracle.load_scenario(sc)
    return g, o


def assert_structure_equal(g, o):
    sg, so = g.structure(), o.structure()
    assert np.array_equal(sg["cell"], so["cell"])
    assert np.array_equal(sg["sorted_ids"], so["sorted_ids"])
    assert np.array_equal(sg["cell_start"], so["cell_start"])
    assert np.array_equal(sg["counts"], so["counts"])
    og, lg = g.neighbors()
    oo, lo = o.neighbors()
    assert np.array_equal(og, oo) and np.array_equal(lg, lo)


# ---------------------------------------------------------------- structure (bit-exact)
@pytest.mark.parametrize("jitter", [0.0, 0.05])
def test_structure_block8k(crm, jitter):
    sc = workloads.block_settle(jitter=jitter, seed=0)
    g, o = both(crm, sc)
    assert_structure_equal(g, o)
    fluid_counts = g.structure()["counts"][: sc.n_fluid]
    if jitter == 0.0:
        assert fluid_counts.max() == 80          # interior lattice count at h = 1.3 d0


def test_structure_rate_state_S0(crm):
    sc = workloads.rate_state_S0(workloads.block_settle())
    g, o = both(crm, sc)
    assert_structure_equal(g, o)


def test_structure_random_clouds(crm):
    rng = np.random.default_rng(77)
    for k in range(12):
        n = int(rng.integers(1, 5000))
        h = float(rng.uniform(0.01, 0.08))
        x = workloads.random_cloud(n, seed=500 + k)
        p = workloads.base_params(rho0=1000.0, mu_s=0.5, mu_2=0.5, I0=0.08, cohesion=0.0, grain_d=1e-3,
                                  d0=h / 1.3, h=h, visc_mode=0, gamma_a=0.0, lo=(-0.05,) * 3, hi=(1.05,) * 3)
        sc = workloads.Scenario("cloud", p, x, None, None, np.zeros((0, 3)), [], 1e-5, 1)
        g, o = both(crm, sc, max_neighbors=1024)
        assert_structure_equal(g, o)


def test_structure_h12_tie_margin(crm):
    # h = 1.2 d0: the first outside shell is only 2 % beyond 2h; jitter flips pairs
    sc = workloads.block_settle(jitter=0.02, seed=3)
    p = dict(sc.params, h=1.2 * sc.params["d0"])
    sc = workloads.Scenario("b12", p, sc.fluid_pos, None, None, sc.wall_pos, [], sc.dt, 1)
    g, o = both(crm, sc)
    assert_structure_equal(g, o)


# ---------------------------------------------------------------- rates (1e-4)
def run_one_armed(crm, sc, dt):
    g, o = both(crm, sc)
    g.debug_arm(True)
    g.step(dt, 1)
    o.step(dt, 1)
    return g, o


@pytest.mark.parametrize("visc", [workloads.VISC_BILATERAL, workloads.VISC_UNILATERAL])
def test_rates_stage_A_and_B_S0(crm, visc):
    sc = workloads.rate_state_S0(workloads.block_settle())
    sc.params["visc_mode"] = visc
    sc.params["gamma_a"] = 0.2
    g, o = run_one_armed(crm, sc, sc.dt)
    nf = sc.n_fluid
    for stage in (0, 1):
        dg, ag, sg = g.last_rates(stage)
        do, ao, so = o.last_rates(stage)
        assert rel_linf(dg[:nf], do[:nf]) <= RATE_TOL, ("drho", stage)
        assert rel_linf(ag[:nf], ao[:nf]) <= RATE_TOL, ("acc", stage)
        assert rel_linf(sg[:nf], so[:nf]) <= RATE_TOL, ("dsig", stage)
        ug, tg = g.last_bce(stage)
        uo, to = o.last_bce(stage)
        assert rel_linf(ug[nf:], uo[nf:]) <= RATE_TOL, ("bce u", stage)
        assert rel_linf(tg[nf:], to[nf:]) <= RATE_TOL, ("bce sigma", stage)


def test_rates_state_S100(crm):
    """rate parity at S100 — the GPU's own state after 100 steps of the jittered
    settling block, loaded into the oracle with set_state (identical fp32 inputs, so identical
    neighbour sets): one more armed step, stage-A and stage-B rates and BCE values within 1e-4."""
    sc = workloads.block_settle(jitter=0.05, seed=0)
    g = crm.load_scenario(sc)
    g.step(sc.dt, 100)
    o = oracle.load_scenario(sc)
    o.set_state(0, *g.get_state())
    assert_structure_equal(g, o)
    g.debug_arm(True)
    g.step(sc.dt, 1)
    o.step(sc.dt, 1)
    nf = sc.n_fluid
    for stage in (0, 1):
        for a_g, a_o in zip(g.last_rates(stage), o.last_rates(stage)):
            assert rel_linf(a_g[:nf], a_o[:nf]) <= RATE_TOL, stage
        for a_g, a_o in zip(g.last_bce(stage), o.last_bce(stage)):
            assert rel_linf(a_g[nf:], a_o[nf:]) <= RATE_TOL, stage


@pytest.mark.parametrize("visc", [workloads.VISC_BILATERAL, workloads.VISC_UNILATERAL])
def test_rates_wendland_S0(crm, visc):
    """Quintic Wendland kernel (A28): same bars as the cubic spline."""
    sc = workloads.rate_state_S0(workloads.block_settle())
    sc.params.update(kernel=1, visc_mode=visc, gamma_a=0.2)
    g, o = run_one_armed(crm, sc, sc.dt)
    nf = sc.n_fluid
    for stage in (0, 1):
        for a_g, a_o in zip(g.last_rates(stage), o.last_rates(stage)):
            assert rel_linf(a_g[:nf], a_o[:nf]) <= RATE_TOL, stage
        for a_g, a_o in zip(g.last_bce(stage), o.last_bce(stage)):
            assert rel_linf(a_g[nf:], a_o[nf:]) <= RATE_TOL, stage
    # the kernel choice matters: the cubic-spline rates differ at this state by far more than the bar
    sc.params["kernel"] = 0
    oc = oracle.load_scenario(sc)
    oc.step(sc.dt, 1)
    assert rel_linf(oc.last_rates(0)[1][:nf], o.last_rates(0)[1][:nf]) > 100 * RATE_TOL


def test_wendland_100_steps_macroscopic(crm):
    sc = workloads.block_settle()
    sc.params["kernel"] = 1
    g, o = both(crm, sc)
    g.step(sc.dt, 100)
    o.step(sc.dt, 100)
    nf = sc.n_fluid
    top = np.argsort(sc.fluid_pos[:, 2])[-400:]
    xg, xo = g.get_state()[0][:nf], o.get_state()[0][:nf]
    hg, ho = settled_height(xg, top, sc.params["d0"]), settled_height(xo, top, sc.params["d0"])
    assert abs(hg - ho) <= 0.02 * ho
    assert np.abs(xg - xo).max() < 0.02 * sc.params["d0"]


def test_one_step_state_S0_confined(crm):
    sc = workloads.rate_state_S0(workloads.block_settle())
    sc.fluid_sig = workloads.f32(sc.fluid_sig + np.array([-2000.0, -2000.0, -2000.0, 0, 0, 0]))
    g, o = run_one_armed(crm, sc, sc.dt)
    nf = sc.n_fluid
    x0, u0, r0, s0 = sc.fluid_pos, sc.fluid_vel, np.full(nf, sc.params["rho0"]), sc.fluid_sig
    xg, ug, rg, sg = [a[:nf] for a in g.get_state()]
    xo, uo, ro, so = [a[:nf] for a in o.get_state()]
    assert np.abs(xg - xo).max() <= 1e-6 * sc.params["d0"] + 2e-9
    assert rel_linf(ug - u0, uo - u0) <= 1e-3
    assert rel_linf(rg - r0, ro - r0) <= 1e-3
    assert rel_linf(sg - s0, so - s0) <= 1e-3


def test_rates_settling_block_bilateral(crm):
    sc = workloads.block_settle(jitter=0.05)
    g, o = both(crm, sc)
    g.step(sc.dt, 3)
    o.step(sc.dt, 3)
    # continue from each side's own state; compare the 4th step's rates
    g.debug_arm(True)
    g.step(sc.dt, 1)
    o.step(sc.dt, 1)
    nf = sc.n_fluid
    da, aa, sa = g.last_rates(0)
    db, ab, sb = o.last_rates(0)
    assert rel_linf(aa[:nf], ab[:nf]) <= 1e-3
    assert rel_linf(da[:nf], db[:nf]) <= 1e-3


def test_slope_rotated_gravity(crm):
    """Slopes as in the MGRU3 runs ('we modified the direction of the gravitational
    acceleration vector ... instead of tilting all the elements'): a 20 deg ramp, gravity
    g (sin 20, 0, -cos 20).  Rates at S0 within the bar, and the block creeps downhill (+x) on both
    sides by the same amount over 60 steps."""
    th = np.radians(20.0)
    sc = workloads.rate_state_S0(workloads.block_settle())
    sc.params["gravity"] = (9.81 * np.sin(th), 0.0, -9.81 * np.cos(th))
    g, o = run_one_armed(crm, sc, sc.dt)
    nf = sc.n_fluid
    for stage in (0, 1):
        for a_g, a_o in zip(g.last_rates(stage), o.last_rates(stage)):
            assert rel_linf(a_g[:nf], a_o[:nf]) <= RATE_TOL, stage
        for a_g, a_o in zip(g.last_bce(stage), o.last_bce(stage)):
            assert rel_linf(a_g[nf:], a_o[nf:]) <= RATE_TOL, stage
    sc = workloads.block_settle()
    sc.params["gravity"] = (9.81 * np.sin(th), 0.0, -9.81 * np.cos(th))
    g, o = both(crm, sc)
    g.step(sc.dt, 60)
    o.step(sc.dt, 60)
    ug, uo = g.get_state()[1][:nf], o.get_state()[1][:nf]
    assert ug[:, 0].mean() > 0 and uo[:, 0].mean() > 0            # downhill
    assert abs(ug[:, 0].mean() - uo[:, 0].mean()) <= 0.02 * abs(uo[:, 0].mean())
    assert np.abs(g.get_state()[0][:nf] - o.get_state()[0][:nf]).max() < 0.02 * sc.params["d0"]


# ---------------------------------------------------------------- macroscopic (2 %)
def settled_height(pos, ids_top, d0):
    return pos[ids_top, 2].mean() + 0.5 * d0


def test_block_100_steps_macroscopic(crm):
    sc = workloads.block_settle()
    g, o = both(crm, sc)
    g.step(sc.dt, 100)
    o.step(sc.dt, 100)
    nf = sc.n_fluid
    top = np.argsort(sc.fluid_pos[:, 2])[-400:]
    xg = g.get_state()[0][:nf]
    xo = o.get_state()[0][:nf]
    hg, ho = settled_height(xg, top, sc.params["d0"]), settled_height(xo, top, sc.params["d0"])
    assert abs(hg - ho) <= 0.02 * ho
    # the two trajectories stay close particle by particle too
    assert np.abs(xg - xo).max() < 0.02 * sc.params["d0"]


def test_determinism_bit_identical(crm):
    sc = workloads.block_settle(jitter=0.05)
    a = crm.load_scenario(sc)
    b = crm.load_scenario(sc)
    a.step(sc.dt, 20)
    b.step(sc.dt, 20)
    for x, y in zip(a.get_state(), b.get_state()):
        assert np.array_equal(x, y)


# ---------------------------------------------------------------- edge cases
def test_single_particle_ballistic(crm):
    p = workloads.base_params(rho0=1500.0, mu_s=0.5, mu_2=0.5, I0=0.08, cohesion=0.0, grain_d=1e-3, d0=0.01,
                              h=0.013, visc_mode=0, gamma_a=0.1, lo=(-1, -1, -1), hi=(1, 1, 1),
                              gravity=(0.1, -0.2, -9.81))
    g = crm.Crm(p)
    g.add_fluid(np.array([[0.1, 0.2, 0.3]]), np.array([[0.5, -0.3, 1.0]]))
    dt = 1e-3
    g.step(dt, 1)
    x, u, rho, s = g.get_state()
    gg = np.array(p["gravity"])
    assert np.allclose(x[0], [0.1, 0.2, 0.3] + dt * np.array([0.5, -0.3, 1.0]) + 0.5 * dt * dt * gg, atol=1e-6)
    assert np.allclose(u[0], [0.5, -0.3, 1.0] + dt * gg, atol=1e-6)


def test_domain_error_names_particle(crm):
    sc = workloads.block_settle(n=(6, 6, 6))
    sc.fluid_pos[7] = [10.0, 0.0, 0.0]
    g = crm.load_scenario(sc)
    with pytest.raises(crm.CrmError) as e:
        g.step(sc.dt, 1)
    assert e.value.code == crm.CRM_E_DOMAIN and "id 7" in str(e.value)


def test_capacity_error(crm):
    sc = workloads.block_settle(n=(6, 6, 6))
    g = crm.load_scenario(sc, max_neighbors=16)
    with pytest.raises(crm.CrmError) as e:
        g.step(sc.dt, 1)
    assert e.value.code == crm.CRM_E_CAPACITY


def test_nonfinite_error(crm):
    sc = workloads.block_settle(n=(6, 6, 6))
    sc.fluid_vel = np.zeros_like(sc.fluid_pos)
    sc.fluid_vel[11] = [np.inf, 0, 0]
    g = crm.load_scenario(sc)
    with pytest.raises(crm.CrmError) as e:
        g.step(sc.dt, 1)
    assert e.value.code in (crm.CRM_E_NONFINITE, crm.CRM_E_DOMAIN)


def test_add_after_step_rejected(crm):
    sc = workloads.block_settle(n=(4, 4, 4))
    g = crm.load_scenario(sc)
    g.step(sc.dt, 1)
    with pytest.raises(crm.CrmError) as e:
        g.add_fluid(np.zeros((1, 3)))
    assert e.value.code == crm.CRM_E_STATE


def test_get_set_state_roundtrip(crm):
    sc = workloads.rate_state_S0(workloads.block_settle(n=(8, 8, 8)))
    g = crm.load_scenario(sc)
    g.step(sc.dt, 2)
    st = g.get_state()
    g2 = crm.load_scenario(sc)
    g2.set_state(0, *st)
    for x, y in zip(g2.get_state(), st):
        assert np.array_equal(x, y)


def test_dense_windows_global_mode(crm):
    # h = 2 d0: ~64 particles per cell, tile windows exceed the shared-memory capacity, so the
    # kernels read the window from global memory ("global mode"); results must not change
    sc = workloads.rate_state_S0(workloads.block_settle(n=(12, 12, 12)))
    sc.params["h"] = 2.0 * sc.params["d0"]
    L = workloads.bce_layers(sc.params["h"], sc.params["d0"])
    sc.wall_pos = workloads.f32(workloads.box_walls(12, 12, 12, sc.params["d0"], L, 2))
    m = (L + 1) * sc.params["d0"]
    sc.params["lo"] = (-m, -m, -m)
    sc.params["hi"] = (12 * sc.params["d0"] + m, 12 * sc.params["d0"] + m, 24 * sc.params["d0"])
    g, o = both(crm, sc)
    assert_structure_equal(g, o)
    g.debug_arm(True)
    g.step(sc.dt, 1)
    o.step(sc.dt, 1)
    nf = sc.n_fluid
    for stage in (0, 1):
        for a, b in zip(g.last_rates(stage), o.last_rates(stage)):
            assert rel_linf(a[:nf], b[:nf]) <= RATE_TOL


# ---------------------------------------------------------------- rigid bodies (A9, C2 shape)
def test_crater_body_loads_and_penetration(crm):
    # desk-scale cratering (d0 = 5 mm): 28 x 20 x 30 soil, R = 12.5 mm sphere (rho_s = 2200)
    # entering at sqrt(2 g H), H = 0.1 m.  Stage-B marker accelerations (A13) and the body force at
    # 1e-4; 100-step penetration within 2 %.
    sc = workloads.cratering(rho_s=2200.0, H_drop=0.1, d0=5e-3)
    g, o = both(crm, sc)
    g.debug_arm(True)
    g.step(sc.dt, 1)
    o.step(sc.dt, 1)
    nf, nw = sc.n_fluid, sc.wall_pos.shape[0]
    ag = g.last_rates(1)[1][nf + nw:]
    ao = o.last_rates(1)[1][nf + nw:]
    assert np.abs(ao).max() > 0
    assert rel_linf(ag, ao) <= RATE_TOL
    bg, bo = g.get_body(1), o.get_body(1)
    assert rel_linf(bg["force"], bo["force"]) <= RATE_TOL
    g.step(sc.dt, 99)
    o.step(sc.dt, 99)
    z0 = sc.bodies[0].pos[2]
    dg = z0 - g.get_body(1)["pos"][2]
    do = z0 - o.get_body(1)["pos"][2]
    assert do > 0.002
    assert abs(dg - do) <= 0.02 * do


# ---------------------------------------------------------------- Alg. 2 persistent lists (NEXT #1)
def test_alg2_stale_pairs_like_oracle(crm):
    h = 0.01
    p = workloads.base_params(rho0=1000.0, mu_s=0.5, mu_2=0.5, I0=0.08, cohesion=0.0, grain_d=1e-3, d0=h, h=h,
                              visc_mode=0, gamma_a=0.5, lo=(-0.1,) * 3, hi=(0.1,) * 3, gravity=(0.0, 0.0, 0.0))
    p["ps_freq"] = 10
    x = np.array([[0.0, 0.0, 0.0], [2.02 * h, 0.0, 0.0]])
    v = np.array([[1.0, 0.0, 0.0], [-1.0, 0.0, 0.0]])
    g = crm.Crm(p)
    g.add_fluid(x, v)
    g.debug_arm(True)
    for _ in range(10):
        g.step(1e-4, 1)
        assert np.abs(g.last_rates(0)[1]).max() == 0      # the step-0 list is empty and reused
    g.step(1e-4, 1)                                        # t = 10: rebuild
    assert np.abs(g.last_rates(0)[1]).max() > 0


def test_alg2_ps10_trajectory_and_rates(crm):
    sc = workloads.rate_state_S0(workloads.block_settle())
    sc.params["ps_freq"] = 10
    g, o = both(crm, sc)
    g.step(sc.dt, 13)
    o.step(sc.dt, 13)
    g.debug_arm(True)
    g.step(sc.dt, 1)          # t = 13: a reuse step
    o.step(sc.dt, 1)
    nf = sc.n_fluid
    for a, b in zip(g.last_rates(0), o.last_rates(0)):
        assert rel_linf(a[:nf], b[:nf]) <= 1e-3
    xg = g.get_state()[0][:nf]
    xo = o.get_state()[0][:nf]
    assert np.abs(xg - xo).max() < 1e-3 * sc.params["d0"]


def test_alg2_reuse_step_rates_match_oracle_at_1e4(crm):
    """Alg. 2 at the 1e-4 rate bar: both sides rebuild at t = 10 from the GPU's state y_10
    (identical lists), then at t = 11 — a reuse step on the stale t = 10 lists — the oracle gets the
    GPU's u, rho, sigma of y_11 (positions kept: setting them would rebuild its lists), so both evaluate
    the same stale pair set on the same fields."""
    sc = workloads.rate_state_S0(workloads.block_settle())
    sc.params["ps_freq"] = 10
    g, o = both(crm, sc)
    g.step(sc.dt, 10)
    o.step(sc.dt, 10)                       # (its own trajectory; only the step counter matters)
    o.set_state(0, *g.get_state())          # y_10 of the GPU; the oracle's lists are dropped
    nf = sc.n_fluid
    g.debug_arm(True)
    for t in (10, 11):
        if t == 11:
            _, vel, rho, sig = g.get_state()
            o.set_state(0, None, vel, rho, sig)
        g.step(sc.dt, 1)                    # t = 10: rebuild, t = 11: reuse
        o.step(sc.dt, 1)
        for stage in (0, 1):
            for a, b in zip(g.last_rates(stage), o.last_rates(stage)):
                assert rel_linf(a[:nf], b[:nf]) <= 1e-4, (t, stage, rel_linf(a[:nf], b[:nf]))


def test_cuda_graph_replay_bit_identical(crm):
    # the captured step (default) equals the kernel-by-kernel step, also across Alg. 2 rebuilds
    for ps in (1, 3):
        sc = workloads.block_settle(jitter=0.05)
        sc.params["ps_freq"] = ps
        a = crm.load_scenario(sc)
        b = crm.load_scenario(sc)
        b.set_graphs(False)
        a.step(sc.dt, 7)
        b.step(sc.dt, 7)
        for x, y in zip(a.get_state(), b.get_state()):
            assert np.array_equal(x, y)


def test_work_counters_match_the_structure(crm):
    """bench.py's roofline counts (directed fluid pairs, Alg. 1 candidates) against the oracle's
    structure: pairs = sum of fluid neighbour counts; candidates = particles of the 27 cells around
    each particle's cell minus itself."""
    sc = workloads.block_settle(jitter=0.05)
    g, o = both(crm, sc)
    g.step(sc.dt, 1)
    o2 = oracle.load_scenario(sc)       # the structure the GPU step built: from the initial state
    so = o2.structure()
    nf = sc.n_fluid
    assert g.pair_count() == int(so["counts"][:nf].sum())
    cs = so["cell_start"].astype(np.int64)
    occ = np.diff(cs)
    p = sc.params
    dims = [int(np.ceil((p["hi"][a] - p["lo"][a]) / (2 * p["h"]))) for a in range(3)]
    occ3 = occ.reshape(dims)
    pad = np.pad(occ3, 1)
    s27 = sum(pad[1 + a:1 + a + dims[0], 1 + b:1 + b + dims[1], 1 + c:1 + c + dims[2]]
              for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1)).ravel()
    cand = s27[so["cell"]] - 1
    f, m = g.candidate_count()
    assert f == int(cand[:nf].sum()) and m == int(cand[nf:].sum())


# ---------------------------------------------------------------- return map, every branch
def _branches(sig_n, dsig_B, sig_new, dt, p):
    """Branch of each particle from the step's own numbers (output-based, no return-map arithmetic):
    0 cut-off (sigma_{n+1} = 0), 1 admissible (sigma_{n+1} = sigma*), 2 radial return with mu = mu_s,
    3 radial return with mu(I) > mu_s; and whether the particle is clear of every branch boundary
    (p* not within 1 Pa of p_cri; admissible only below (mu_s p* + c)(1 - 1e-3), where no mu(I) can
    make it yield; radial with tau_bar scaled by < 1 - 1e-3; mu_eff = mu_s to 1e-4 or above it by > 1 %)."""
    s_star = sig_n + dt * dsig_B
    p_star = -s_star[:, :3].mean(1)
    tau = s_star.copy(); tau[:, :3] += p_star[:, None]
    tb_star = np.sqrt(0.5 * (tau[:, :3] ** 2).sum(1) + (tau[:, 3:] ** 2).sum(1))
    tn = sig_new.copy(); pn = -sig_new[:, :3].mean(1); tn[:, :3] += pn[:, None]
    tb_new = np.sqrt(0.5 * (tn[:, :3] ** 2).sum(1) + (tn[:, 3:] ** 2).sum(1))
    scale = tb_new / np.maximum(tb_star, 1e-30)
    cut = np.all(sig_new == 0.0, axis=1)
    c, mu_s = p["cohesion"], p["mu_s"]
    mu_rel = (tb_new - c) / np.maximum(p_star, 1e-30) / mu_s - 1.0
    adm = ~cut & (np.abs(scale - 1.0) < 1e-5)
    br = np.where(cut, 0, np.where(adm, 1, np.where(mu_rel > 1e-2, 3, 2)))
    p_cri = -c / mu_s
    clear = np.abs(p_star - p_cri) > 1.0
    clear &= np.where(br == 1, tb_star < (mu_s * p_star + c) * (1 - 1e-3), True)
    clear &= np.where(br >= 2, (scale < 1 - 1e-3) & ((np.abs(mu_rel) < 1e-4) | (mu_rel > 1e-2)), True)
    return br, clear


def test_return_map_every_branch_elementwise(crm):
    """One step from a state that puts >= 100 particles in each branch of the return map (tension
    cut-off, admissible, radial return at mu_s, radial return with mu(I) > mu_s): the branch of every
    particle away from a branch boundary is the same on both sides, and sigma_{n+1} agrees element by
    element within 1e-4 of max |sigma|."""
    sc = workloads.return_map_state()
    g, o = both(crm, sc)
    g.debug_arm(True)
    g.step(sc.dt, 1)
    o.step(sc.dt, 1)
    nf = sc.n_fluid
    sig_n = sc.fluid_sig
    sg = g.get_state()[3][:nf]
    so = o.get_state()[3][:nf]
    bg, cg = _branches(sig_n, g.last_rates(1)[2][:nf], sg, sc.dt, sc.params)
    bo, co = _branches(sig_n, o.last_rates(1)[2][:nf], so, sc.dt, sc.params)
    clear = cg & co
    counts = np.bincount(bo[clear], minlength=4)
    assert np.all(counts >= 100), counts
    assert np.array_equal(bg[clear], bo[clear])
    assert np.abs(sg[clear] - so[clear]).max() <= 1e-4 * np.abs(so).max()


def test_structure_random_clouds_50(crm):
    """bit-exact structure on 50 random clouds (N <= 5000, random h)."""
    rng = np.random.default_rng(78)
    for k in range(50):
        n = int(rng.integers(1, 5000))
        h = float(rng.uniform(0.01, 0.08))
        x = workloads.random_cloud(n, seed=1000 + k)
        p = workloads.base_params(rho0=1000.0, mu_s=0.5, mu_2=0.5, I0=0.08, cohesion=0.0, grain_d=1e-3,
                                  d0=h / 1.3, h=h, visc_mode=0, gamma_a=0.0, lo=(-0.05,) * 3, hi=(1.05,) * 3)
        sc = workloads.Scenario("cloud", p, x, None, None, np.zeros((0, 3)), [], 1e-5, 1)
        g, o = both(crm, sc, max_neighbors=1024)
        assert_structure_equal(g, o)
        g.close()
