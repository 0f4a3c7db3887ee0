"""Pins of the oracle's SPH rates: Eq. continuity_dis, momentum_dis,
stress_rate_dis (readings A4–A6), artificial viscosity (A9)."""
import json
import math
import os

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import workloads

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))
C13 = GOLD["lattice_h13"]["M_diag"]


def make_sim(oracle_mod, pos, vel=None, sig=None, *, h_over_d0=1.3, d0=0.01, gamma_a=0.0,
             visc=0, gravity=(0.0, 0.0, 0.0), rho0=1500.0, box=None, E=1e6, nu=0.3, **kw):
    lo = pos.min(0) - 4 * d0 if box is None else box[0]
    hi = pos.max(0) + 4 * d0 if box is None else box[1]
    p = workloads.base_params(rho0=rho0, mu_s=kw.get("mu_s", 0.5), mu_2=kw.get("mu_2", 0.5),
                              I0=0.08, cohesion=kw.get("cohesion", 0.0), grain_d=1e-3, d0=d0,
                              h=h_over_d0 * d0, visc_mode=visc, gamma_a=gamma_a, lo=lo, hi=hi,
                              gravity=gravity, E=E, nu=nu)
    s = oracle_mod.OracleSim(p)
    s.add_fluid(pos, vel, sig)
    return s, p


def stage_a_rates(s, dt=1e-6):
    s.step(dt, 1)
    return s.last_rates(0)


def center_index(pos):
    c = pos.mean(0)
    return int(np.argmin(np.linalg.norm(pos - c, axis=1)))


def test_linear_velocity_field_gives_lattice_gradient(oracle_mod):
    # u = A x on a perfect lattice: L = sum V (A x_ji) (x) grad W = A M = 0.9934837 A (h = 1.3 d0)
    d0 = 0.01
    pos = workloads.lattice_block(9, 9, 9, d0)
    A = np.random.default_rng(1).normal(0, 1.0, (3, 3))
    sig0 = np.array([-300.0, -200.0, -500.0, 40.0, -25.0, 10.0])   # uniform, anisotropic
    vel = pos @ A.T
    sig = np.tile(sig0, (len(pos), 1))
    s, p = make_sim(oracle_mod, pos, vel, sig)
    drho, acc, ds = stage_a_rates(s)
    i = center_index(pos)
    L = C13 * A
    assert drho[i] == pytest.approx(-p["rho0"] * np.trace(L), rel=1e-9, abs=1e-9)
    expect = oracle_mod.stress_rate(L, sig0, p["K"], p["G"])
    assert np.allclose(ds[i], expect, rtol=1e-9, atol=1e-9 * np.abs(expect).max())
    # uniform stress: sum V grad W = 0 on the lattice -> no stress force at the centre
    assert np.allclose(acc[i], 0.0, atol=1e-9)


def test_rigid_translation_has_no_rates(oracle_mod):
    d0 = 0.01
    pos = workloads.lattice_block(6, 6, 6, d0)
    pos = pos + np.random.default_rng(3).uniform(-0.1, 0.1, pos.shape) * d0
    vel = np.tile([0.3, -0.2, 0.1], (len(pos), 1))
    s, _ = make_sim(oracle_mod, pos, vel)
    drho, acc, ds = stage_a_rates(s)
    assert np.abs(drho).max() < 1e-9
    assert np.abs(ds).max() < 1e-6


def test_linear_pressure_gradient(oracle_mod):
    # sigma = -(P0 + k z) I: F3 sum gives a = -(c k / rho) e_z at an interior lattice particle
    d0 = 0.01
    pos = workloads.lattice_block(9, 9, 9, d0)
    P0, k = 2000.0, 5.0e4
    p_ = P0 + k * pos[:, 2]
    sig = np.zeros((len(pos), 6)); sig[:, 0] = sig[:, 1] = sig[:, 2] = -p_
    s, p = make_sim(oracle_mod, pos, None, sig)
    _, acc, _ = stage_a_rates(s)
    i = center_index(pos)
    assert acc[i] == pytest.approx([0.0, 0.0, -C13 * k / p["rho0"]], rel=1e-9, abs=1e-9)


def test_zero_stress_gives_gravity(oracle_mod):
    d0 = 0.01
    pos = workloads.lattice_block(5, 5, 5, d0)
    pos = pos + np.random.default_rng(4).uniform(-0.2, 0.2, pos.shape) * d0
    g = (0.3, -1.0, -9.81)
    s, _ = make_sim(oracle_mod, pos, None, None, gravity=g)
    _, acc, _ = stage_a_rates(s)
    assert np.allclose(acc, g, rtol=0, atol=1e-12)


def test_two_particle_antisymmetry(oracle_mod):
    rng = np.random.default_rng(5)
    d0 = 0.01
    for _ in range(10):
        pos = np.array([[0.0, 0.0, 0.0], rng.uniform(-1.2, 1.2, 3) * d0]) + 0.05
        if np.linalg.norm(pos[1] - pos[0]) >= 2.6 * d0:
            continue
        vel = rng.normal(0, 0.5, (2, 3))
        sig = rng.normal(0, 500, (2, 6))
        s, p = make_sim(oracle_mod, pos, vel, sig, gamma_a=0.3, visc=0)
        _, acc, _ = stage_a_rates(s)
        # equal masses: m a_i + m a_j = 0 (F3 symmetry + AV antisymmetry)
        assert np.allclose(acc[0] + acc[1], 0, atol=1e-12 * np.abs(acc).max())
        assert np.abs(acc).max() > 0


def test_blob_momentum_conservation(oracle_mod):
    # S:343 / S:627: no walls, no gravity, bilateral AV: sum m a = 0 to round-off
    rng = np.random.default_rng(6)
    d0 = 0.01
    pos = workloads.lattice_block(15, 15, 14, d0)          # 3150 particles
    pos = pos + rng.uniform(-0.15, 0.15, pos.shape) * d0
    vel = rng.normal(0, 0.2, pos.shape)
    sig = rng.normal(0, 800, (len(pos), 6))
    s, p = make_sim(oracle_mod, pos, vel, sig, gamma_a=0.5, visc=0)
    _, acc, _ = stage_a_rates(s)
    assert np.abs(acc.sum(0)).max() <= 1e-10 * np.abs(acc).sum()


def _pair(oracle_mod, vi, vj, visc, gamma=0.5):
    d0 = 0.01
    pos = np.array([[0.05, 0.05, 0.05], [0.05 + 1.5 * d0 * 1.3 / 1.3, 0.05, 0.05]])
    vel = np.array([vi, vj], float)
    s, p = make_sim(oracle_mod, pos, vel, None, gamma_a=gamma, visc=visc)
    _, acc, _ = stage_a_rates(s)
    return pos, vel, acc


def test_artificial_viscosity_sign_dissipation_and_modes(oracle_mod):
    # approaching along x: particle 0 must be pushed away from particle 1 (-x) (A9)
    pos, vel, acc = _pair(oracle_mod, [1.0, 0, 0], [-1.0, 0, 0], visc=0)
    assert acc[0, 0] < 0 and acc[1, 0] > 0
    assert np.dot(vel[0], acc[0]) + np.dot(vel[1], acc[1]) < 0          # dissipative
    # separating: unilateral gives zero, bilateral gives a nonzero damping
    _, _, acc_u = _pair(oracle_mod, [-1.0, 0, 0], [1.0, 0, 0], visc=1)
    assert np.all(acc_u == 0)
    pos, vel, acc_b = _pair(oracle_mod, [-1.0, 0, 0], [1.0, 0, 0], visc=0)
    assert acc_b[0, 0] > 0                                                # slows separation
    assert np.dot(vel[0], acc_b[0]) + np.dot(vel[1], acc_b[1]) < 0
    # gamma_a = 0 -> no contribution
    _, _, acc0 = _pair(oracle_mod, [1.0, 0, 0], [-1.0, 0, 0], visc=0, gamma=0.0)
    assert np.all(acc0 == 0)


def test_artificial_viscosity_random_pairs_dissipate(oracle_mod):
    rng = np.random.default_rng(8)
    d0 = 0.01
    for _ in range(20):
        pos = np.array([[0.05, 0.05, 0.05], [0.05, 0.05, 0.05] + rng.uniform(-1.4, 1.4, 3) * d0])
        if np.linalg.norm(pos[1] - pos[0]) >= 2.6 * d0:
            continue
        vel = rng.normal(0, 1, (2, 3))
        s, p = make_sim(oracle_mod, pos, vel, None, gamma_a=0.4, visc=0)
        _, acc, _ = stage_a_rates(s)
        assert np.dot(vel[0], acc[0]) + np.dot(vel[1], acc[1]) <= 1e-15


# ---- the Jaumann stress rate as a pure function ----
def test_stress_rate_rigid_rotation_matches_rotated_stress(oracle_mod):
    rng = np.random.default_rng(9)
    for _ in range(10):
        w = rng.normal(0, 1, 3)
        Lw = np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]])   # u = w x x
        S = rng.normal(0, 100, (3, 3)); S = S + S.T
        s6 = np.array([S[0, 0], S[1, 1], S[2, 2], S[0, 1], S[0, 2], S[1, 2]])
        out = oracle_mod.stress_rate(Lw, s6, 1e6, 4e5)        # rotation: no strain rate
        dt = 1e-6
        R = Rotation.from_rotvec(w * dt).as_matrix()
        Sd = (R @ S @ R.T - S) / dt                           # d/dt (R S R^T)
        expect = np.array([Sd[0, 0], Sd[1, 1], Sd[2, 2], Sd[0, 1], Sd[0, 2], Sd[1, 2]])
        assert np.allclose(out, expect, rtol=1e-4, atol=1e-4 * np.abs(expect).max())


def test_stress_rate_hydrostatic_rotation_shear_compression(oracle_mod):
    K, G = 8.0e5, 3.0e5
    w = np.array([0.2, -0.5, 0.7])
    Lw = np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]])
    assert np.allclose(oracle_mod.stress_rate(Lw, [-500, -500, -500, 0, 0, 0], K, G), 0, atol=1e-12)
    gd = 0.3
    Ls = np.array([[0, gd, 0], [0, 0, 0], [0, 0, 0]])        # simple shear, eps_12 = gd/2
    out = oracle_mod.stress_rate(Ls, np.zeros(6), K, G)
    assert out[3] == pytest.approx(2 * G * gd / 2) and np.allclose(out[[0, 1, 2, 4, 5]], 0)
    a = 0.4
    Lc = -a * np.eye(3)                                      # uniform compression tr eps = -3a
    out = oracle_mod.stress_rate(Lc, np.zeros(6), K, G)
    assert np.allclose(out, [-3 * a * K] * 3 + [0] * 3)


# ---- artificial viscosity magnitude, worked two-particle example (Eq. 13; A9, A10) ----
def _av_pair(oracle_mod, *, rho_i, rho_j, vi, cs, xi2, gamma, h_over_d0=1.3, visc=0, r_over_h=1.5):
    d0 = 0.01
    h = h_over_d0 * d0
    pos = np.array([[0.05 + r_over_h * h, 0.05, 0.05], [0.05, 0.05, 0.05]])   # x_ij = +r e_x
    vel = np.array([[vi, 0.0, 0.0], [0.0, 0.0, 0.0]])
    lo, hi = pos.min(0) - 4 * d0, pos.max(0) + 4 * d0
    p = workloads.base_params(rho0=1500.0, mu_s=0.5, mu_2=0.5, I0=0.08, cohesion=0.0, grain_d=1e-3, d0=d0,
                              h=h, visc_mode=visc, gamma_a=gamma, lo=lo, hi=hi, gravity=(0.0, 0.0, 0.0))
    p["cs"] = cs
    p["xi2"] = xi2
    s = oracle_mod.OracleSim(p)
    s.add_fluid(pos, vel, None)
    s.set_state(0, rho=np.array([rho_i, rho_j]))
    _, acc, _ = stage_a_rates(s)
    return acc[0], p


def test_artificial_viscosity_magnitude_two_particles(oracle_mod):
    """Pi_i = gamma_a h c_s (m_j / rho_bar_ij) (v_ij . r_ij)/(r_ij^2 + xi^2) grad_i W_ij (Eq. 13 with the
    sign of reading A9, rho_bar = (rho_i + rho_j)/2 and xi^2, c_s as given, A10), written out for a pair
    on the x axis at r = 1.5 h, where the cubic spline's derivative is W'(r) = -(3/4)(2 - q)^2/(pi h^4)
    = -0.1875/(pi h^4) (A1): grad_i W_ij = W'(r) e_x.  sigma = 0 and g = 0, so a_i = Pi_i exactly.
    Several (rho_i, rho_j, c_s, xi^2, gamma, v) so that m_j/rho_j, m_j/rho_i, a dropped h or c_s, xi in
    place of xi^2 or a transposed v_ij . r_ij would each change the value."""
    d0 = 0.01
    cases = [dict(rho_i=1500.0, rho_j=1500.0, vi=-0.8, cs=20.0, xi2=1e-6, gamma=0.5),
             dict(rho_i=1400.0, rho_j=1700.0, vi=-0.8, cs=20.0, xi2=1e-6, gamma=0.5),
             dict(rho_i=1700.0, rho_j=1300.0, vi=0.3, cs=35.0, xi2=4e-5, gamma=0.2),
             dict(rho_i=1450.0, rho_j=1600.0, vi=1.7, cs=11.0, xi2=2.5e-5, gamma=1.3, h_over_d0=1.2)]
    for c in cases:
        a, p = _av_pair(oracle_mod, **c)
        h = p["h"]
        r = 1.5 * h
        m = p["rho0"] * d0 ** 3                       # m = rho0 d0^3
        rho_bar = 0.5 * (c["rho_i"] + c["rho_j"])
        vr = c["vi"] * r                              # (u_i - u_j) . (x_i - x_j)
        dW = -0.1875 / (math.pi * h ** 4)
        expect = c["gamma"] * h * c["cs"] * (m / rho_bar) * vr / (r * r + c["xi2"]) * dW
        assert a[0] == pytest.approx(expect, rel=1e-12), c
        assert a[1] == 0.0 and a[2] == 0.0
    # unilateral (Eq. 14): the separating pair (v_ij . r_ij > 0) gets nothing, the approaching one
    # the bilateral value
    a_sep, _ = _av_pair(oracle_mod, rho_i=1500.0, rho_j=1600.0, vi=0.5, cs=20.0, xi2=1e-6, gamma=0.5, visc=1)
    assert np.all(a_sep == 0.0)
    a_app_u, _ = _av_pair(oracle_mod, rho_i=1500.0, rho_j=1600.0, vi=-0.5, cs=20.0, xi2=1e-6, gamma=0.5, visc=1)
    a_app_b, _ = _av_pair(oracle_mod, rho_i=1500.0, rho_j=1600.0, vi=-0.5, cs=20.0, xi2=1e-6, gamma=0.5, visc=0)
    assert a_app_u[0] == a_app_b[0] and a_app_u[0] > 0.0      # approaching: pushed apart (+x)
