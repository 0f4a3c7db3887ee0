"""Oracle pins of active domains (Alg. 3; readings A29–A31).

* ManageArrayMemory: SPEC's scripted sequence 1000 -> 1200 -> 1200 -> 700 @ step 50 gives
  Grow -> 1440, Keep, Shrink -> 700 with the paper's constants G = 1.2, S = 0.75, S_I = 50.
* UpdateActivity: inside -> Active, face + 1.5h -> Extended-Active, face + 2.5h -> Inactive;
  the Euclidean distance to the box decides at corners (A29); the box turns with its body.
* Full coverage is bit-identical to the feature off; an Inactive or Extended-Active particle
  keeps exactly its frozen state (A31) and re-enters with it; inactive particles have no neighbours and no rates;
  the active set's structure equals brute force on that subset; t_delay gates the feature (Alg. 3)."""
import numpy as np
import pytest

import oracle
import workloads


def test_capacity_policy_paper_constants(oracle_mod):
    cap, a = oracle.manage_capacity(1000, 1200, 1)
    assert (cap, a) == (1440, 1)                      # Grow to N G
    cap, a = oracle.manage_capacity(cap, 1200, 2)
    assert (cap, a) == (1440, 0)                      # Keep
    cap, a = oracle.manage_capacity(1000, 700, 50)
    assert (cap, a) == (700, 2)                       # 0.7 < 0.75 at a multiple of S_I: Shrink
    assert oracle.manage_capacity(1000, 700, 49) == (1000, 0)     # not a shrink step
    assert oracle.manage_capacity(1000, 750, 100) == (1000, 0)    # ratio == S: keep (strict <)
    assert oracle.manage_capacity(1000, 1000, 50) == (1000, 0)    # exactly full: keep
    assert oracle.manage_capacity(1440, 1500, 50) == (1800, 1)    # growth wins on a shrink step


def test_activity_predicate(oracle_mod):
    h = 0.1
    I = np.eye(3)
    box = [((0.0, 0.0, 0.0), I, (1.0, 1.0, 1.0))]
    A = lambda x, b=box: oracle.activity(np.array(x, float), b, 2 * h)
    assert A([0.3, -0.9, 0.99]) == 0
    assert A([1.0, 0.0, 0.0]) == 0                    # on the face: inside (|x| <= half)
    assert A([1.0 + 1.5 * h, 0.0, 0.0]) == 1
    assert A([1.0 + 2.5 * h, 0.0, 0.0]) == 2
    assert A([-1.0 - 1.5 * h, 0.2, -0.3]) == 1
    assert A([1.1, 1.1, 1.1]) == 1                    # corner distance 0.173 < 2h
    assert A([1.13, 1.13, 1.13]) == 2                 # 0.225 > 2h: Euclidean, not per-axis (A29)
    c, s = np.cos(np.pi / 4), np.sin(np.pi / 4)
    Rz = np.array([[c, -s, 0], [s, c, 0], [0, 0, 1]])     # body -> world
    rot = [((0.0, 0.0, 0.0), Rz, (1.0, 1.0, 1.0))]
    assert A([1.2, 0.0, 0.0], rot) == 0               # inside the turned box
    assert A([1.2, 0.0, 0.0]) == 1
    two = box + [((5.0, 0.0, 0.0), I, (0.5, 0.5, 0.5))]
    assert A([5.2, 0.1, 0.0], two) == 0 and A([5.6, 0.0, 0.0], two) == 1 and A([3.0, 0, 0], two) == 2
    assert A([0.0, 0.0, 0.0], []) == 2                # no box at all: nothing is near one


def _bed(nx=16, ny=10, nz=8):
    sc = workloads.block_settle(n=(nx, ny, nz), jitter=0.05, seed=4)
    return sc


def test_full_coverage_is_bit_identical(oracle_mod):
    sc = _bed()
    p = sc.params
    half = [0.5 * (p["hi"][a] - p["lo"][a]) + 1.0 for a in range(3)]
    ref = oracle.load_scenario(sc)
    sc.active = {"boxes": {0: half}, "t_delay": -1.0}
    act = oracle.load_scenario(sc)
    ref.step(sc.dt, 15)
    act.step(sc.dt, 15)
    assert np.all(act.activity() == 0)
    for a, b in zip(ref.get_state(), act.get_state()):
        assert np.array_equal(a, b)


def _moving_box_bed():
    """A bed with a prescribed 'plough' body (a small marker cube) moving along +x through it;
    its active box travels with it."""
    sc = _bed(20, 8, 8)
    d0 = sc.params["d0"]
    g = np.arange(3) * d0
    cube = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3) - d0
    pos0 = np.array([4 * d0, 4 * d0, 9 * d0])
    b = workloads.Body(mass=1.0, inertia=(1, 1, 1), pos=tuple(pos0), vel=(0.5, 0.0, 0.0),
                       motion=workloads.BODY_PRESCRIBED, markers=workloads.f32(cube + pos0))
    sc.bodies = [b]
    sc.active = {"boxes": {1: (3 * d0, 3 * d0, 6 * d0)}, "t_delay": -1.0}
    return sc


def test_inactive_particles_are_frozen_and_reenter(oracle_mod):
    sc = _moving_box_bed()
    o = oracle.load_scenario(sc)
    nf = sc.n_fluid
    x0, u0, r0, s0 = [a[:nf].copy() for a in o.get_state()]
    o.step(sc.dt, 1)
    f1 = o.activity()[:nf]
    assert (f1 == 0).any() and (f1 == 1).any() and (f1 == 2).any()
    x1, u1, r1, s1 = [a[:nf] for a in o.get_state()]
    ina = f1 == 2
    fro = f1 != 0
    # frozen: Inactive and Extended-Active particles keep exactly the initial state (A31)
    assert np.array_equal(x1[fro], x0[fro]) and np.array_equal(u1[fro], u0[fro])
    assert np.array_equal(r1[fro], r0[fro]) and np.array_equal(s1[fro], s0[fro])
    # the Active set moved (gravity acts on every one of them)
    assert np.all(u1[~fro] != u0[~fro])
    # rates: zero outside the Active set (A31)
    for stage in (0, 1):
        d, acc, ds = o.last_rates(stage)
        assert np.all(acc[:nf][fro] == 0) and np.all(d[:nf][fro] == 0) and np.all(ds[:nf][fro] == 0)
        assert np.all(np.abs(acc[:nf][~fro]).sum(axis=1) > 0)
    # the box travels 0.5 m/s: after enough steps a particle ahead of it re-enters
    ahead = np.nonzero(ina & (x0[:, 0] > x0[:, 0].min() + 0.5 * (x0[:, 0].max() - x0[:, 0].min())))[0]
    steps = 0
    while steps < 400:
        o.step(sc.dt, 10)
        steps += 10
        f = o.activity()[:nf]
        newly = ahead[f[ahead] == 0]
        if len(newly):
            break
    assert len(newly), "the moving box never reached the particles ahead of it"
    # re-entry state: those particles were frozen until the rebuild that activated them, i.e. their
    # state at that step start equals the initial state; the step that activated them moved them
    xs = o.get_state()[0][:nf]
    assert np.all(xs[newly] != x0[newly])
    o.close()


def test_active_structure_equals_brute_force_on_the_active_set(oracle_mod):
    sc = _moving_box_bed()
    o = oracle.load_scenario(sc)
    o.step(sc.dt, 3)
    st = o.structure()
    f = o.activity()
    n = o.count()
    M = len(st["cell_start"]) - 1
    act = np.nonzero(f != 2)[0]
    assert np.all(st["cell"][f == 2] == M)
    assert np.all(st["counts"][f == 2] == 0)
    assert st["cell_start"][-1] == len(act)
    # sorted prefix: (cell, id) order of the non-inactive particles, inactive ones behind by id
    srt = st["sorted_ids"]
    key = np.lexsort((act, st["cell"][act]))
    assert np.array_equal(srt[: len(act)], act[key])
    assert np.array_equal(srt[len(act):], np.nonzero(f == 2)[0])
    # neighbour sets = brute force over the active subset (B2 on fp32 positions)
    x = o.get_state()[0].astype(np.float32)
    off, lst = oracle.brute_neighbors(np.ascontiguousarray(x[act]), 2 * sc.params["h"])
    oo, lo = o.neighbors()
    for k, i in enumerate(act):
        mine = np.sort(lo[oo[i]:oo[i + 1]])
        assert np.array_equal(mine, np.sort(act[lst[off[k]:off[k + 1]]]))
    o.close()


def test_t_delay_gates_the_culling(oracle_mod):
    sc = _moving_box_bed()
    sc.active["t_delay"] = 2.5 * sc.dt
    o = oracle.load_scenario(sc)
    for k in range(3):                 # t = 0, dt, 2 dt: not yet
        o.step(sc.dt, 1)
        assert np.all(o.activity() == 0), k
    o.step(sc.dt, 1)                   # t = 3 dt > t_delay
    assert (o.activity() == 2).any()
    o.close()
