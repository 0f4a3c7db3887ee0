"""Pins of the oracle's persistent neighbour lists (Alg. 2): rebuilt when
t mod ps_freq = 0, otherwise reused as they are — no distance re-check, so particles that come
within 2h between rebuilds do not interact until the next rebuild."""
import numpy as np

import workloads


def pair_sim(oracle_mod, ps_freq, gap):
    h = 0.01
    p = workloads.base_params(rho0=1000.0, mu_s=0.5, mu_2=0.5, I0=0.08, cohesion=0.0, grain_d=1e-3, d0=h,
                              h=h, visc_mode=0, gamma_a=0.5, lo=(-0.1,) * 3, hi=(0.1,) * 3,
                              gravity=(0.0, 0.0, 0.0))
    p["ps_freq"] = ps_freq
    s = oracle_mod.OracleSim(p)
    x = np.array([[0.0, 0.0, 0.0], [gap * h, 0.0, 0.0]])
    v = np.array([[1.0, 0.0, 0.0], [-1.0, 0.0, 0.0]])
    s.add_fluid(x, v)
    return s


def test_stale_list_ignores_new_pairs_until_rebuild(oracle_mod):
    # two particles 2.02 h apart closing at 2 m/s: within 2h after ~1 step of 1e-4 s
    dt = 1e-4
    s1, s10 = pair_sim(oracle_mod, 1, 2.02), pair_sim(oracle_mod, 10, 2.02)
    acc1, acc10 = [], []
    for _ in range(10):
        s1.step(dt, 1)
        s10.step(dt, 1)
        acc1.append(np.abs(s1.last_rates(0)[1]).max())
        acc10.append(np.abs(s10.last_rates(0)[1]).max())
    assert max(acc1[2:]) > 0                       # ps_freq = 1: the approaching pair interacts
    assert max(acc10) == 0                         # ps_freq = 10: the step-0 list is empty and kept
    s10.step(dt, 1)                                # t = 10: rebuild
    assert np.abs(s10.last_rates(0)[1]).max() > 0


def test_static_configuration_independent_of_ps_freq(oracle_mod):
    # nothing moves and nothing changes: every rebuild reproduces the same lists
    sc = workloads.block_settle(n=(6, 6, 6))
    sc.params["gravity"] = (0.0, 0.0, 0.0)
    out = []
    for ps in (1, 4):
        p = dict(sc.params, ps_freq=ps)
        s = oracle_mod.OracleSim(p)
        s.add_fluid(sc.fluid_pos, None, None)
        s.add_bce(0, sc.wall_pos)
        s.step(sc.dt, 9)
        out.append(s.get_state())
    for a, b in zip(*out):
        assert np.array_equal(a, b)


def test_ps_freq_one_is_the_default(oracle_mod):
    sc = workloads.rate_state_S0(workloads.block_settle(n=(6, 6, 6)))
    res = []
    for extra in ({}, {"ps_freq": 1}):
        s = oracle_mod.OracleSim(dict(sc.params, **extra))
        s.add_fluid(sc.fluid_pos, sc.fluid_vel, sc.fluid_sig)
        s.add_bce(0, sc.wall_pos)
        s.step(sc.dt, 3)
        res.append(s.get_state())
    for a, b in zip(*res):
        assert np.array_equal(a, b)
