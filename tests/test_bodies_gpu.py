"""GPU parity of the rigid-body layer (§2.5.1; reading A13; the rigid integrator of
DESIGN.md §3) and of the per-step error reporting: the CUDA path (libcrm.so through the C-ABI)
against the fp64 oracle and against the closed forms of tests/test_oracle_bodies.py."""
import math

import numpy as np
import pytest

import oracle
import workloads
from workloads import BODY_FREE, BODY_PRESCRIBED, Body

pytestmark = pytest.mark.gpu


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


def _params(lo, hi, *, d0=0.01, gravity=(0.0, 0.0, -9.81), gamma=0.0):
    return workloads.base_params(rho0=1500.0, mu_s=0.5, mu_2=0.5, I0=0.08, cohesion=0.0, grain_d=1e-3, d0=d0,
                                 h=1.3 * d0, visc_mode=0, gamma_a=gamma, lo=lo, hi=hi, gravity=gravity)


def _rotating_marker(sim_cls):
    d0 = 0.01
    c = np.array([0.2, 0.2, 0.2])
    xa = c + np.array([0.05, 0.0, 0.0])
    dirs = np.array([[0.6, 0.8, 0.0], [0.8, 0.0, 0.6], [0.8, 0.0, -0.6], [0.6, -0.8, 0.0]])
    fluid = xa + 1.6 * d0 * dirs
    u_f = np.array([0.3, -0.2, 0.1])
    sig0 = np.array([-800.0, -700.0, -900.0, 50.0, -30.0, 20.0])
    s = sim_cls(_params((0.0, 0.0, 0.0), (0.4, 0.4, 0.4)))
    s.add_fluid(fluid, np.tile(u_f, (4, 1)), np.tile(sig0, (4, 1)))
    bid = s.add_body(Body(mass=1.0, inertia=(1, 1, 1), pos=tuple(c), vel=(0.05, 0.0, 0.0), omega=(0.0, 0.0, 4.0),
                          motion=BODY_PRESCRIBED))
    s.add_bce(bid, xa[None, :])
    return s, dict(c=c, xa=xa, fluid=fluid, u_f=u_f, sig0=sig0)


def test_rotating_body_marker_extrapolation(crm):
    """The marker of a turning prescribed body: u_a = 2 (v + omega x r) - u_f and the centripetal
    term of the Adami stress (closed form of test_oracle_bodies.py), GPU against the closed form and
    against the oracle in both RK stages."""
    g, k = _rotating_marker(crm.Crm)
    o, _ = _rotating_marker(oracle.OracleSim)
    g.debug_arm(True)
    dt = 1e-3
    g.step(dt, 1)
    o.step(dt, 1)
    r = k["xa"] - k["c"]
    om = np.array([0.0, 0.0, 4.0])
    u_body = np.array([0.05, 0.0, 0.0]) + np.cross(om, r)
    ug, sg = g.last_bce(0)
    assert np.allclose(ug[4], 2 * u_body - k["u_f"], rtol=0, atol=2e-6)
    a_a = np.cross(om, np.cross(om, r))
    hyd = 1500.0 * np.dot(np.array([0.0, 0.0, -9.81]) - a_a, k["xa"] - k["fluid"].mean(0))
    assert np.allclose(sg[4], k["sig0"] - hyd * np.array([1, 1, 1, 0, 0, 0]), rtol=0, atol=1e-4 * 900)
    for stage in (0, 1):
        ug, sg = g.last_bce(stage)
        uo, so = o.last_bce(stage)
        assert rel_linf(ug[4], uo[4]) <= 1e-5 and rel_linf(sg[4], so[4]) <= 1e-5, stage


def test_free_symmetric_top_matches_the_oracle(crm):
    """Euler's equations in the principal frame (no loads): the GPU's fp64 body update against the
    oracle's (the closed-form precession is pinned on the oracle, test_oracle_bodies.py)."""
    b = Body(mass=1.0, inertia=(1.0, 1.0, 2.0), pos=(0.0, 0.0, 0.0), quat=(0.9, 0.1, -0.3, 0.2),
             omega=(0.8, -0.3, 2.0), motion=BODY_FREE, dof_mask=0b111111)
    out = []
    for cls in (crm.Crm, oracle.OracleSim):
        s = cls(_params((-0.1, -0.1, -0.2), (0.2, 0.2, 0.1), gravity=(0.0, 0.0, 0.0)))
        s.add_fluid(np.array([[0.05, 0.05, 0.05]]))
        s.add_body(b)
        s.step(1e-3, 500)
        out.append(s.get_body(1))
    for key in ("omega", "quat", "pos"):
        assert np.allclose(out[0][key], out[1][key], rtol=0, atol=1e-10), key


def _wheel_case():
    return workloads.mgru3_wheel(n=(40, 16, 12), R=0.06, width=0.06, vx=0.1, slip=0.3, sinkage=0.02,
                                 active=False, x0=0.2)


def test_rotating_wheel_loads_match_the_oracle(crm):
    """A prescribed wheel turning at constant omega (the paper's wheel and drum rigs, P:117, P:128,
    P:156) in a small soil bin: stage-B marker accelerations (A13) at 1e-4 of their largest value,
    force and torque within 1e-4 of the sum of the magnitudes of their per-marker terms; after 100
    steps the mean load over the last 20 steps within 2 %."""
    sc = _wheel_case()
    g = crm.load_scenario(sc)
    o = oracle.load_scenario(sc)
    g.debug_arm(True)
    g.step(sc.dt, 1)
    o.step(sc.dt, 1)
    nf, nw = sc.n_fluid, sc.wall_pos.shape[0]
    ag = g.last_rates(1)[1][nf + nw:]
    ao = o.last_rates(1)[1][nf + nw:]
    assert np.abs(ao).max() > 0
    assert rel_linf(ag, ao) <= 1e-4
    m = sc.params["rho0"] * sc.params["d0"] ** 3
    bg, bo = g.get_body(1), o.get_body(1)
    Fscale = (m * np.abs(ao)).sum(0)
    assert np.all(np.abs(bg["force"] - bo["force"]) <= 1e-4 * Fscale.max())
    xm = sc.bodies[0].markers   # lever arms ~ R
    Tscale = np.abs(np.cross(xm - np.asarray(sc.bodies[0].pos), m * ao)).sum(0)
    assert np.all(np.abs(bg["torque"] - bo["torque"]) <= 1e-4 * Tscale.max())
    assert np.abs(bo["torque"][1]) > 1e-3 * Tscale.max()     # the wheel's driving torque is resolved
    g.debug_arm(False)
    Fg, Fo, Tg, To = [], [], [], []
    for k in range(99):
        g.step(sc.dt, 1)
        o.step(sc.dt, 1)
        if k >= 79:
            bg, bo = g.get_body(1), o.get_body(1)
            Fg.append(bg["force"]); Fo.append(bo["force"]); Tg.append(bg["torque"]); To.append(bo["torque"])
    Fg, Fo, Tg, To = map(np.array, (Fg, Fo, Tg, To))
    assert np.allclose(g.get_body(1)["pos"], o.get_body(1)["pos"], rtol=0, atol=1e-9)   # prescribed travel
    for a, b in ((Fg, Fo), (Tg, To)):
        assert np.all(np.abs(a.mean(0) - b.mean(0)) <= 0.02 * np.abs(b.mean(0)).max())


def test_more_than_64_bodies_are_posed(crm):
    """every body gets its pose (the pose kernel covers all bodies, not one block of 64):
    65 prescribed bodies, one marker each, far from the fluid; after n steps marker b sits at
    x0 + n dt v_b."""
    p = _params((0.0, 0.0, 0.0), (1.0, 1.0, 0.2), gravity=(0.0, 0.0, 0.0))
    g = crm.Crm(p)
    g.add_fluid(np.array([[0.9, 0.9, 0.1]]))
    x0s, vs = [], []
    for b in range(65):
        x0 = np.array([0.05 + 0.011 * b, 0.1 + 0.005 * (b % 7), 0.1])
        v = np.array([0.0, 0.01 + 0.001 * b, 0.0])
        bid = g.add_body(Body(mass=1.0, inertia=(1, 1, 1), pos=tuple(x0), vel=tuple(v), motion=BODY_PRESCRIBED))
        g.add_bce(bid, x0[None, :] + [0.0, 0.0, 0.02])
        x0s.append(x0); vs.append(v)
    n, dt = 40, 1e-3
    g.step(dt, n)
    x = g.get_state()[0][1:]
    expect = np.array(x0s) + [0.0, 0.0, 0.02] + n * dt * np.array(vs)
    assert np.abs(x - expect).max() < 1e-6


def test_body_count_limit(crm):
    """The body index has 7 bits of the marker tag (the rest holds the flags and the quantised
    position compensation): 126 bodies besides the walls are accepted, the next one is
    refused with CRM_E_INVALID; the last body's markers follow it."""
    p = _params((0.0, 0.0, 0.0), (1.0, 1.0, 0.2), gravity=(0.0, 0.0, 0.0))
    g = crm.Crm(p)
    g.add_fluid(np.array([[0.9, 0.9, 0.1]]))
    for b in range(126):
        x0 = (0.02 + 0.006 * b, 0.05, 0.1)
        bid = g.add_body(Body(mass=1.0, inertia=(1, 1, 1), pos=x0, vel=(0.0, 0.01, 0.0), motion=BODY_PRESCRIBED))
        assert bid == b + 1
    g.add_bce(126, np.array([[0.02 + 0.006 * 125, 0.05, 0.12]]))
    with pytest.raises(crm.CrmError) as e:
        g.add_body(Body(mass=1.0, inertia=(1, 1, 1), pos=(0.5, 0.5, 0.1), motion=BODY_PRESCRIBED))
    assert e.value.code == crm.CRM_E_INVALID
    g.step(1e-3, 10)
    x = g.get_state()[0][1]
    assert np.abs(x - np.array([0.02 + 0.006 * 125, 0.05 + 10 * 1e-3 * 0.01, 0.12])).max() < 1e-6


def test_error_latch_names_the_failing_step_and_stops(crm):
    """S:147 / S:318: a particle leaving the grid box is reported with the step in which it left,
    also from a replayed CUDA graph, and the later steps of the call compute nothing."""
    p = _params((0.0, 0.0, 0.0), (0.1, 0.1, 0.1), gravity=(0.0, 0.0, 0.0))
    x0 = np.array([[0.05, 0.05, 0.05]])
    v0 = np.array([[2.1, 0.0, 0.0]])
    o = oracle.OracleSim(p)
    o.add_fluid(x0, v0)
    with pytest.raises(oracle.OracleError) as eo:
        o.step(1e-3, 200)
    for graphs in (True, False):
        g = crm.Crm(p)
        g.add_fluid(x0, v0)
        g.set_graphs(graphs)
        g.step(1e-3, 3)
        with pytest.raises(crm.CrmError) as eg:
            g.step(1e-3, 200)
        assert eg.value.code == crm.CRM_E_DOMAIN
        assert "step 26" in str(eg.value) and "step 26" in str(eo.value), (str(eg.value), str(eo.value))
        x = g.get_state()[0][0, 0]
        assert abs(x - (0.05 + 26 * 2.1e-3)) < 1e-6      # the state the failing step left (x_26)
