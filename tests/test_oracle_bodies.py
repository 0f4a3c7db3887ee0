"""Pins of the oracle's rigid-body layer (§2.5.1; reading A13 and the rigid integrator of
DESIGN.md §3): marker kinematics of a prescribed rotating body, the loads (force and torque) from
the marker accelerations, and the free-body update (semi-implicit Euler; Euler's equations in the
principal frame).  Each closed form below is written from the mechanics, not from the oracle."""
import math

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import workloads
from workloads import BODY_FREE, BODY_PRESCRIBED, Body


def _params(lo, hi, *, d0=0.01, gravity=(0.0, 0.0, 0.0), gamma=0.0, rho0=1500.0):
    return workloads.base_params(rho0=rho0, mu_s=0.5, mu_2=0.5, I0=0.08, cohesion=0.0, grain_d=1e-3, d0=d0,
                                 h=1.3 * d0, visc_mode=0, gamma_a=gamma, lo=lo, hi=hi, gravity=gravity)


def _quat_mul(a, b):
    w1, x1, y1, z1 = a
    w2, x2, y2, z2 = b
    return np.array([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2, w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                     w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2, w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2])


def _R(q):
    w, x, y, z = q
    return Rotation.from_quat([x, y, z, w]).as_matrix()


def _lone_body_sim(oracle_mod, body, gravity):
    """A free body without markers (no loads) plus one far-away fluid particle."""
    p = _params((-0.1, -0.1, -0.2), (0.2, 0.2, 0.1), gravity=gravity)
    s = oracle_mod.OracleSim(p)
    s.add_fluid(np.array([[0.05, 0.05, 0.05]]))
    s.add_body(body)
    return s


def test_free_body_without_loads_follows_the_semi_implicit_euler_sequence(oracle_mod):
    # v_n = v_0 + n dt g,  x_n = x_0 + dt sum_{k=1..n} v_k = x_0 + n dt v_0 + dt^2 g n(n+1)/2
    g = np.array([0.3, -1.1, -9.81])
    v0 = np.array([0.2, 0.05, 1.5])
    x0 = np.array([0.01, -0.02, 0.03])
    b = Body(mass=2.0, inertia=(0.1, 0.2, 0.3), pos=tuple(x0), vel=tuple(v0), motion=BODY_FREE, dof_mask=0b111111)
    s = _lone_body_sim(oracle_mod, b, g)
    dt, n = 1e-3, 137
    s.step(dt, n)
    st = s.get_body(1)
    assert np.allclose(st["vel"], v0 + n * dt * g, rtol=0, atol=1e-13)
    assert np.allclose(st["pos"], x0 + n * dt * v0 + dt * dt * g * n * (n + 1) / 2, rtol=0, atol=1e-13)
    # a locked translation (dof bit clear) keeps its velocity
    b2 = Body(mass=2.0, inertia=(0.1, 0.2, 0.3), pos=tuple(x0), vel=tuple(v0), motion=BODY_FREE, dof_mask=0b111011)
    s2 = _lone_body_sim(oracle_mod, b2, g)
    s2.step(dt, n)
    assert s2.get_body(1)["vel"][2] == v0[2]


def test_torque_free_spin_about_a_principal_axis(oracle_mod):
    # omega along the body z axis of a rotated body: omega stays constant and the attitude is the
    # closed-form rotation q(t) = [cos(w t/2), sin(w t/2) n] (x) q0
    q0 = Rotation.from_rotvec([0.3, -0.7, 0.4]).as_quat()
    q0 = np.array([q0[3], q0[0], q0[1], q0[2]])
    w = 3.0
    n_hat = _R(q0) @ np.array([0.0, 0.0, 1.0])
    omega = w * n_hat
    b = Body(mass=1.0, inertia=(0.2, 0.5, 0.9), pos=(0.0, 0.0, 0.0), quat=tuple(q0), omega=tuple(omega),
             motion=BODY_FREE, dof_mask=0b111111)
    s = _lone_body_sim(oracle_mod, b, (0.0, 0.0, 0.0))
    dt, n = 2e-3, 400
    s.step(dt, n)
    st = s.get_body(1)
    assert np.allclose(st["omega"], omega, rtol=0, atol=1e-12)
    t = n * dt
    q_exp = _quat_mul(np.concatenate([[math.cos(w * t / 2)], math.sin(w * t / 2) * n_hat]), q0)
    q = st["quat"]
    assert min(np.abs(q - q_exp).max(), np.abs(q + q_exp).max()) < 1e-10


def test_torque_free_symmetric_top_precesses_in_the_body_frame(oracle_mod):
    # I1 = I2 = 1, I3 = 2, omega_b(0) = (a, 0, c): Euler's equations give omega_b(t) = (a cos ct,
    # a sin ct, c) (body frame) and a constant angular momentum R I omega_b (world frame).  A
    # world-axis-aligned update (alpha = T / I) would keep omega_b = (a, 0, c).
    a, c = 0.8, 2.0
    b = Body(mass=1.0, inertia=(1.0, 1.0, 2.0), pos=(0.0, 0.0, 0.0), quat=(1.0, 0.0, 0.0, 0.0),
             omega=(a, 0.0, c), motion=BODY_FREE, dof_mask=0b111111)
    s = _lone_body_sim(oracle_mod, b, (0.0, 0.0, 0.0))
    dt, n = 1e-4, 10000
    I = np.diag([1.0, 1.0, 2.0])
    L0 = I @ np.array([a, 0.0, c])
    s.step(dt, n)
    st = s.get_body(1)
    R = _R(st["quat"])
    wb = R.T @ st["omega"]
    t = n * dt
    assert np.allclose(wb, [a * math.cos(c * t), a * math.sin(c * t), c], atol=2e-3 * c)
    assert np.allclose(R @ I @ wb, L0, atol=2e-3 * np.linalg.norm(L0))
    # first order in dt: halving dt halves the error
    s2 = _lone_body_sim(oracle_mod, b, (0.0, 0.0, 0.0))
    s2.step(dt / 2, 2 * n)
    st2 = s2.get_body(1)
    wb2 = _R(st2["quat"]).T @ st2["omega"]
    e1 = np.abs(wb - [a * math.cos(c * t), a * math.sin(c * t), c]).max()
    e2 = np.abs(wb2 - [a * math.cos(c * t), a * math.sin(c * t), c]).max()
    assert 1.6 < e1 / e2 < 2.4


def _rotating_marker_case(oracle_mod, gravity=(0.0, 0.0, -9.81)):
    """A prescribed body turning at omega about z through c, translating at v, with one marker at
    r = (R, 0, 0) from c; four fluid particles at distance d from the marker, all on the +x side,
    uniform velocity u_f and uniform stress sigma0, density rho0."""
    d0 = 0.01
    c = np.array([0.2, 0.2, 0.2])
    Rr = 0.05
    xa = c + np.array([Rr, 0.0, 0.0])
    d = 1.6 * d0
    dirs = np.array([[0.6, 0.8, 0.0], [0.8, 0.0, 0.6], [0.8, 0.0, -0.6], [0.6, -0.8, 0.0]])   # mean 0.7 e_x
    fluid = xa + d * dirs
    u_f = np.array([0.3, -0.2, 0.1])
    sig0 = np.array([-800.0, -700.0, -900.0, 50.0, -30.0, 20.0])
    p = _params((0.0, 0.0, 0.0), (0.4, 0.4, 0.4), gravity=gravity)
    s = oracle_mod.OracleSim(p)
    s.add_fluid(fluid, np.tile(u_f, (4, 1)), np.tile(sig0, (4, 1)))
    w = 4.0
    v = np.array([0.05, 0.0, 0.0])
    bid = s.add_body(Body(mass=1.0, inertia=(1, 1, 1), pos=tuple(c), vel=tuple(v), omega=(0.0, 0.0, w),
                          motion=BODY_PRESCRIBED))
    s.add_bce(bid, xa[None, :])
    return s, dict(c=c, xa=xa, fluid=fluid, u_f=u_f, sig0=sig0, w=w, v=v, rho0=p["rho0"], g=np.array(gravity))


def test_rotating_body_marker_velocity_and_centripetal_stress_term(oracle_mod):
    """Adami extrapolation onto a marker of a prescribed body turning at omega (A12):
    u_a = 2 (v + omega x r) - mean(u_f) and sigma_a = sigma0 - rho0 ((g - a_a) . (x_a - xbar)) I with
    the body acceleration at the marker a_a = omega x (omega x r) (constant omega: centripetal only).
    The four fluid particles are equidistant from the marker, so the kernel weights are equal and
    xbar is their plain mean."""
    s, k = _rotating_marker_case(oracle_mod)
    s.step(1e-6, 1)
    u_b, sig_b = s.last_bce(0)
    r = k["xa"] - k["c"]
    om = np.array([0.0, 0.0, k["w"]])
    u_body = k["v"] + np.cross(om, r)
    assert np.allclose(u_b[4], 2 * u_body - k["u_f"], rtol=0, atol=1e-13)
    a_a = np.cross(om, np.cross(om, r))                       # = -w^2 r
    xbar = k["fluid"].mean(0)
    hyd = k["rho0"] * np.dot(k["g"] - a_a, k["xa"] - xbar)
    expect = k["sig0"] - hyd * np.array([1, 1, 1, 0, 0, 0])
    assert np.allclose(sig_b[4], expect, rtol=1e-12, atol=1e-9)
    assert abs(k["rho0"] * np.dot(a_a, k["xa"] - xbar)) > 1.0   # the centripetal part is resolved


def test_body_torque_is_the_sum_of_marker_moments(oracle_mod):
    """F = sum m a_s and T = sum (x_s - x_c) x m a_s over the stage-B marker accelerations, with the
    lever arms taken at the mid-step pose (A13).  Two markers of a translating, turning
    prescribed body, each with its own fluid neighbours."""
    d0 = 0.01
    c = np.array([0.2, 0.2, 0.2])
    xa = np.array([c + [0.05, 0.0, 0.0], c + [0.0, -0.04, 0.03]])
    rng = np.random.default_rng(4)
    fluid = np.concatenate([x + rng.uniform(-1.5, 1.5, (5, 3)) * d0 for x in xa])
    sig = rng.normal(-500.0, 150.0, (len(fluid), 6))
    vel = rng.normal(0.0, 0.1, (len(fluid), 3))
    p = _params((0.0, 0.0, 0.0), (0.4, 0.4, 0.4), gravity=(0.0, 0.0, -9.81), gamma=0.3)
    s = oracle_mod.OracleSim(p)
    s.add_fluid(fluid, vel, sig)
    v = np.array([0.4, -0.1, 0.2])
    bid = s.add_body(Body(mass=1.0, inertia=(1, 1, 1), pos=tuple(c), vel=tuple(v), omega=(0.5, -1.0, 3.0),
                          motion=BODY_PRESCRIBED))
    s.add_bce(bid, xa)
    dt = 1e-3
    s.step(dt, 1)
    _, acc, _ = s.last_rates(1)
    m = p["rho0"] * d0 ** 3
    Fk = m * acc[len(fluid):]
    assert np.abs(Fk).max() > 0
    # mid-step pose: centre c + v dt/2, markers turned by omega dt/2 about it
    cm = c + 0.5 * dt * v
    Rm = Rotation.from_rotvec(np.array([0.5, -1.0, 3.0]) * 0.5 * dt).as_matrix()
    xm = cm + (xa - c) @ Rm.T
    st = s.get_body(bid)
    assert np.allclose(st["force"], Fk.sum(0), rtol=1e-12, atol=1e-15)
    T = np.cross(xm - cm, Fk).sum(0)
    assert np.allclose(st["torque"], T, rtol=1e-10, atol=1e-14)
