"""Pins of the oracle's BCE extrapolation (readings A11, A12), return map
(A15, A16, A27) and RK2 explicit midpoint integrator."""
import json
import math
import os

import numpy as np
import pytest

import workloads

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def slab_with_floor(d0=0.01, h_over=1.3, n=(8, 8, 6), gravity=(0.0, 0.0, -9.81)):
    nx, ny, nz = n
    h = h_over * d0
    L = workloads.bce_layers(h, d0)
    walls = workloads.box_walls(nx, ny, nz, d0, L, 2)
    pos = workloads.lattice_block(nx, ny, nz, d0)
    m = (L + 1) * d0
    p = workloads.base_params(rho0=1600.0, mu_s=0.5, mu_2=0.5, I0=0.08, cohesion=0.0,
                              grain_d=1e-3, d0=d0, h=h, visc_mode=0, gamma_a=0.0,
                              lo=(-m, -m, -m), hi=(nx * d0 + m, ny * d0 + m, (nz + 6) * d0),
                              gravity=gravity)
    return p, pos, walls


def run_stage_a(oracle_mod, p, pos, vel, sig, walls, bodies=()):
    s = oracle_mod.OracleSim(p)
    s.add_fluid(pos, vel, sig)
    wid = s.add_bce(0, walls)
    ids = []
    for b, mk in bodies:
        bid = s.add_body(b)
        ids.append(s.add_bce(bid, mk))
    s.step(1e-7, 1)
    u, sg = s.last_bce(0)
    return s, wid, u, sg, ids


def has_fluid_neighbour(oracle_mod, pos, walls, h):
    # markers within 2h of some fluid particle (brute force on the union)
    allp = np.concatenate([pos, walls])
    off, lst = oracle_mod.brute_neighbors(allp, 2 * h)
    nf = len(pos)
    return np.array([np.any(lst[off[nf + k]:off[nf + k + 1]] < nf) for k in range(len(walls))])


def test_bce_reproduces_linear_hydrostatic_field(oracle_mod):
    # sigma_f = -rho g (H - z_f) I  =>  sigma_a = -rho g (H - z_a) I exactly (reading A12)
    p, pos, walls = slab_with_floor()
    g = 9.81
    H = pos[:, 2].max() + 0.005
    sig = np.zeros((len(pos), 6)); sig[:, :3] = (-p["rho0"] * g * (H - pos[:, 2]))[:, None]
    s, wid, u, sg, _ = run_stage_a(oracle_mod, p, pos, None, sig, walls)
    near = has_fluid_neighbour(oracle_mod, pos, walls, p["h"])
    mk = slice(wid, wid + len(walls))
    expect = -p["rho0"] * g * (H - walls[:, 2])
    got = sg[mk]
    assert near.sum() > 100
    for c in range(3):
        assert np.allclose(got[near, c], expect[near], rtol=1e-9, atol=1e-9 * np.abs(expect).max())
    assert np.allclose(got[near, 3:], 0, atol=1e-9)
    # no fluid neighbour -> sigma = 0, u = u_body (A11)
    assert np.all(got[~near] == 0) and np.all(u[mk][~near] == 0)


def test_bce_velocity_no_slip_and_constant_stress(oracle_mod):
    p, pos, walls = slab_with_floor(gravity=(0.0, 0.0, 0.0))
    v = np.array([0.3, -0.1, 0.05])
    s0 = np.array([-100.0, -200.0, -300.0, 10.0, 20.0, -30.0])
    vel = np.tile(v, (len(pos), 1)); sig = np.tile(s0, (len(pos), 1))
    s, wid, u, sg, _ = run_stage_a(oracle_mod, p, pos, vel, sig, walls)
    near = has_fluid_neighbour(oracle_mod, pos, walls, p["h"])
    mk = slice(wid, wid + len(walls))
    assert np.allclose(u[mk][near], -v, atol=1e-12)                 # static body: u_a = -v
    assert np.allclose(sg[mk][near], s0, rtol=1e-12, atol=1e-9)     # constant field


def test_bce_moving_body_no_slip_consistency(oracle_mod):
    # body moving at v, fluid moving at v -> u_a = 2v - v = v
    p, pos, walls = slab_with_floor(gravity=(0.0, 0.0, 0.0))
    d0 = p["d0"]
    v = np.array([0.0, 0.0, -0.4])
    blk = workloads.lattice_block(3, 3, 2, d0, origin=(3 * d0, 3 * d0, 6 * d0))
    body = workloads.Body(mass=1.0, inertia=(1, 1, 1), pos=tuple(blk.mean(0)), vel=tuple(v),
                          motion=workloads.BODY_PRESCRIBED, markers=blk)
    vel = np.tile(v, (len(pos), 1))
    s, wid, u, sg, ids = run_stage_a(oracle_mod, p, pos, vel, None, walls, [(body, blk)])
    mk = slice(ids[0], ids[0] + len(blk))
    assert np.allclose(u[mk], v, atol=1e-12)


def test_return_map_paper_examples(oracle_mod):
    ex = GOLD["return_map_examples"]
    base = dict(rho0=1500.0, G=3e5, mu_2=0.7, I0=0.08, grain_d=1e-3)
    t = ex["tension_cutoff"]
    P = dict(base, mu_s=t["mu_s"], mu_2=max(t["mu_s"], 0.7), cohesion=t["c"])
    s = np.array([300.0, 300.0, 300.0, 50.0, 0, 0])              # p* = -300
    assert np.all(oracle_mod.return_map(s, s, P, 1e-4) == 0)
    a = ex["admissible"]
    P = dict(base, mu_s=a["mu_s"], cohesion=a["c"])
    tau = a["tau_bar_star"]                                      # sigma* = -p I + tau e_xy
    s = np.array([-a["p_star"]] * 3 + [tau, 0, 0])
    assert np.array_equal(oracle_mod.return_map(s, s, P, 1e-4), s)
    r = ex["radial_return"]
    P = dict(base, mu_s=r["mu_s"], cohesion=r["c"])
    s = np.array([-r["p_star"]] * 3 + [r["tau_bar_star"], 0, 0])
    out = oracle_mod.return_map(s, s, P, 1e-4)
    p_out = -out[:3].mean()
    tau_out = out.copy(); tau_out[:3] += p_out
    tb = math.sqrt(0.5 * (np.sum(tau_out[:3] ** 2) + 2 * np.sum(tau_out[3:] ** 2)))
    assert p_out == pytest.approx(r["expect_p"], rel=1e-12)
    assert tb == pytest.approx(r["expect_tau_bar"], rel=1e-12)


def _decomp(s):
    p = -(s[0] + s[1] + s[2]) / 3
    t = s.copy(); t[:3] += p
    tb = math.sqrt(0.5 * (np.sum(t[:3] ** 2) + 2 * np.sum(t[3:] ** 2)))
    return p, t, tb


def test_return_map_random_admissibility_idempotence(oracle_mod):
    # 1e5 random trial stresses -> admissible or zero; step 4 keeps p and direction
    rng = np.random.default_rng(11)
    P = dict(rho0=1500.0, G=3e5, mu_s=0.4, mu_2=0.9, I0=0.1, grain_d=2e-3, cohesion=150.0)
    dt = 1e-4
    n = 100_000
    S = rng.normal(0, 2000, (n, 6)) + np.array([-1500, -1500, -1500, 0, 0, 0])
    Sn = S + rng.normal(0, 300, (n, 6))
    for k in range(n):
        out = oracle_mod.return_map(S[k], Sn[k], P, dt)
        if np.all(out == 0):
            continue
        ps, ts, tbs = _decomp(S[k])
        po, to, tbo = _decomp(out)
        _, _, tbn = _decomp(Sn[k])
        gd = max(0.0, (tbs - tbn) / (P["G"] * dt))
        I = gd * P["grain_d"] * math.sqrt(P["rho0"] / max(ps, 1.0))
        mu = P["mu_s"] + (P["mu_2"] - P["mu_s"]) / (1 + P["I0"] / I) if I > 0 else P["mu_s"]
        assert tbo <= max(mu * po + P["cohesion"], 0) + 1e-9 * (abs(po) + P["cohesion"])
        assert po == pytest.approx(ps, rel=1e-12, abs=1e-9)     # pressure preserved
        if tbo < tbs:                                            # radial: same direction
            assert np.allclose(to * tbs, ts * tbo, rtol=1e-9, atol=1e-9 * tbs * tbo)
    # idempotence holds for the rate-independent law (mu_2 = mu_s): with mu_2 > mu_s a
    # second application sees a smaller gamma_dot, hence a smaller mu(I), by construction
    P1 = dict(P, mu_2=P["mu_s"])
    for k in range(0, n, 50):
        out = oracle_mod.return_map(S[k], Sn[k], P1, dt)
        out2 = oracle_mod.return_map(out, Sn[k], P1, dt)
        assert np.allclose(out2, out, rtol=1e-12, atol=1e-9)


def test_mu_of_I_monotone(oracle_mod):
    # mu(I) increasing from mu_s (I -> 0) to mu_2 (I -> inf): the returned tau_bar grows with the
    # plastic rate and stays within [mu_s p, mu_2 p]
    P = dict(rho0=1500.0, G=3e5, mu_s=0.4, mu_2=0.9, I0=0.1, grain_d=2e-3, cohesion=0.0)
    p = 1000.0
    tbn = 100.0
    sn = np.array([-p] * 3 + [tbn, 0, 0])
    prev = 0.0
    for tb in [450, 1e3, 1e4, 1e5, 1e6, 1e7]:
        s = np.array([-p] * 3 + [tb, 0, 0])
        out = oracle_mod.return_map(s, sn, P, 1e-4)
        _, _, tbo = _decomp(out)
        assert P["mu_s"] * p - 1e-9 <= tbo <= P["mu_2"] * p + 1e-9
        assert tbo >= prev
        prev = tbo


def test_rk2_ballistic_is_exact(oracle_mod):
    # x'' = g: the explicit midpoint method is exact (S:339 with lambda = 0 on u)
    p = workloads.base_params(rho0=1500.0, mu_s=0.5, mu_2=0.5, I0=0.08, cohesion=0.0, grain_d=1e-3,
                              d0=0.01, h=0.013, visc_mode=0, gamma_a=0.1, lo=(-1, -1, -1), hi=(1, 1, 1),
                              gravity=(0.1, -0.2, -9.81))
    s = oracle_mod.OracleSim(p)
    x0 = np.array([[0.1, 0.2, 0.3]]); u0 = np.array([[0.5, -0.3, 1.0]])
    s.add_fluid(x0, u0)
    dt = 1e-3
    s.step(dt, 1)
    x, u, rho, sg = s.get_state()
    g = np.array(p["gravity"])
    assert np.allclose(x[0], x0[0] + dt * u0[0] + 0.5 * dt * dt * g, rtol=0, atol=1e-15)
    assert np.allclose(u[0], u0[0] + dt * g, rtol=0, atol=1e-15)
    assert rho[0] == p["rho0"] and np.all(sg == 0)


def _blob_run(oracle_mod, dt, T):
    rng = np.random.default_rng(12)
    d0 = 0.01
    pos = workloads.lattice_block(4, 4, 4, d0) + rng.uniform(-0.1, 0.1, (64, 3)) * d0
    vel = rng.normal(0, 0.05, pos.shape)
    sig = rng.normal(0, 300, (64, 6)) + np.array([-2000, -2000, -2000, 0, 0, 0])
    p = workloads.base_params(rho0=1500.0, mu_s=10.0, mu_2=10.0, I0=0.08, cohesion=1e6, grain_d=1e-3,
                              d0=d0, h=1.3 * d0, visc_mode=0, gamma_a=0.1, lo=(-0.1,) * 3, hi=(0.2,) * 3,
                              gravity=(0.0, 0.0, 0.0))
    s = oracle_mod.OracleSim(p)
    s.add_fluid(pos, vel, sig)
    s.step(dt, int(round(T / dt)))
    x, u, rho, sg = s.get_state()
    return np.concatenate([x.ravel() / d0, u.ravel(), sg.ravel() / 2000.0, rho / 1500.0])


def test_rk2_self_convergence_order(oracle_mod):
    # observed order within [1.7, 2.3] (an Euler or a lost midpoint would give ~1)
    dt0 = 2e-5
    T = 40 * dt0
    ref = _blob_run(oracle_mod, dt0 / 8, T)
    e = [np.abs(_blob_run(oracle_mod, dt0 / k, T) - ref).max() for k in (1, 2)]
    order = math.log2(e[0] / e[1])
    assert 1.7 <= order <= 2.3, (e, order)


def test_body_loads_newton_third_law(oracle_mod):
    # A13 / S:439: the force on a body equals minus the force its markers exert on the fluid, so with
    # no gravity and no walls sum_f m a_f (stage B) + F_body = 0
    rng = np.random.default_rng(21)
    d0 = 0.01
    pos = workloads.lattice_block(10, 10, 6, d0) + rng.uniform(-0.1, 0.1, (600, 3)) * d0
    vel = rng.normal(0, 0.1, pos.shape)
    sig = rng.normal(0, 300, (600, 6)) + np.array([-1500, -1500, -1500, 0, 0, 0])
    blk = workloads.lattice_block(4, 4, 3, d0, origin=(3 * d0, 3 * d0, 6 * d0))
    p = workloads.base_params(rho0=1500.0, mu_s=0.5, mu_2=0.5, I0=0.08, cohesion=0.0, grain_d=1e-3, d0=d0,
                              h=1.3 * d0, visc_mode=0, gamma_a=0.2, lo=(-0.05,) * 3, hi=(0.2,) * 3,
                              gravity=(0.0, 0.0, 0.0))
    s = oracle_mod.OracleSim(p)
    s.add_fluid(pos, vel, sig)
    body = workloads.Body(mass=1.0, inertia=(1, 1, 1), pos=tuple(blk.mean(0)), vel=(0.0, 0.0, -0.2),
                          motion=workloads.BODY_PRESCRIBED, markers=blk)
    bid = s.add_body(body)
    s.add_bce(bid, blk)
    s.step(1e-5, 1)
    _, acc, _ = s.last_rates(1)
    m = p["rho0"] * d0 ** 3
    F_fluid = m * acc[:600].sum(0)
    F_body = s.get_body(bid)["force"]
    assert np.abs(F_body).max() > 0
    assert np.allclose(F_fluid + F_body, 0, atol=1e-10 * (np.abs(m * acc[:600]).sum()))
