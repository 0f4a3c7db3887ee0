"""Multi-GPU slab decomposition on one GPU: W slab contexts in one process step together with
in-process ("loopback") halo copies (crm_group_step).  The owned particles must follow
bit-identical trajectories to a one-context run (SURVEY.md §8(e) invariant): the neighbour
order is the global (cell, id) order restricted to each slab plus its ghost planes."""
import numpy as np
import pytest

import workloads

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def crm():
    from paper_2507_05643_b200 import build
    build.build_library()
    from paper_2507_05643_b200 import crm as m
    m.load_library()
    return m


def run_slabs(crm, sc, world, steps):
    from paper_2507_05643_b200 import dist
    c0 = crm.load_scenario(sc, rank=0, world=world)
    ctxs = [c0] + [crm.load_scenario(sc, rank=r, world=world, stream=c0.stream()) for r in range(1, world)]
    crm.group_step(ctxs, sc.dt, steps)
    owned = [c.count(crm.CRM_OWNED) for c in ctxs]
    return dist.merge_owned([c.get_state() for c in ctxs]), owned


@pytest.mark.parametrize("world", [2, 4])
def test_bed_slabs_bit_identical(crm, world):
    sc = workloads.bed(n=(64, 24, 12))
    ref = crm.load_scenario(sc)
    ref.step(sc.dt, 20)
    got, owned = run_slabs(crm, sc, world, 20)
    assert sum(owned) == sc.n_fluid + sc.n_bce
    for a, b in zip(got, ref.get_state()):
        assert not np.isnan(a).any()
        assert np.array_equal(a, b)


def test_block_with_migration_bit_identical(crm):
    # a block moving at 1 m/s along x: particles cross slab faces (migration path)
    sc = workloads.block_settle()
    sc.fluid_vel = np.zeros_like(sc.fluid_pos)
    sc.fluid_vel[:, 0] = 1.0
    ref = crm.load_scenario(sc)
    ref.step(sc.dt, 60)
    got, owned = run_slabs(crm, sc, 3, 60)
    x0 = sc.fluid_pos[:, 0]
    assert np.abs(got[0][: sc.n_fluid, 0] - x0).max() > 2e-3   # the block really moved
    for a, b in zip(got, ref.get_state()):
        assert np.array_equal(a, b)


def test_slabs_with_persistent_lists_bit_identical(crm):
    sc = workloads.block_settle()
    sc.params["ps_freq"] = 5
    sc.fluid_vel = np.zeros_like(sc.fluid_pos)
    sc.fluid_vel[:, 0] = 1.0
    ref = crm.load_scenario(sc)
    ref.step(sc.dt, 23)
    got, _ = run_slabs(crm, sc, 2, 23)
    for a, b in zip(got, ref.get_state()):
        assert np.array_equal(a, b)


def test_moving_body_across_slabs(crm):
    """A free sphere dropped into the cratering soil with its markers spread over slab
    faces: every slab sums the loads of the markers it owns, the partial sums are exchanged and
    added in rank order (SURVEY §8(e) bodies), so the body follows the one-GPU trajectory up to the
    regrouping of one fp64 sum."""
    from paper_2507_05643_b200 import dist
    from workloads import crater as cr
    sc = cr.scenario(2200.0, 0.1, d0=5e-3)
    steps = 60
    ref = crm.load_scenario(sc)
    ref.step(sc.dt, steps)
    world = 2                                        # the balanced cut runs through the centred sphere
    c0 = crm.load_scenario(sc, rank=0, world=world)
    ctxs = [c0] + [crm.load_scenario(sc, rank=r, world=world, stream=c0.stream()) for r in range(1, world)]
    # the sphere's markers really are split over more than one slab
    owned_markers = [int(np.isfinite(c.get_state()[0][sc.n_fluid + sc.wall_pos.shape[0]:, 0]).sum()) for c in ctxs]
    assert sum(v > 0 for v in owned_markers) >= 2, owned_markers
    crm.group_step(ctxs, sc.dt, steps)
    b_ref = ref.get_body(1)
    for c in ctxs:                                   # every rank integrated the same body
        b = c.get_body(1)
        assert np.allclose(b["pos"], b_ref["pos"], rtol=0, atol=1e-9)
        assert np.allclose(b["vel"], b_ref["vel"], rtol=1e-7, atol=1e-9)
    got = dist.merge_owned([c.get_state() for c in ctxs])
    x_ref = ref.get_state()[0]
    assert not np.isnan(got[0]).any()
    assert np.abs(got[0] - x_ref).max() < 1e-5 * sc.params["d0"]


def test_slab_step_graph_replay_equals_eager(crm):
    """The slab step reads no device value on the host (device-resident counts, fixed-size
    transfers: DESIGN §7), so it is captured once per (buffer parity, rebuild) and replayed; the
    replay must give the eager launches' state bit for bit, across several calls, with migration
    and Alg. 2 reuse steps."""
    from paper_2507_05643_b200 import dist
    sc = workloads.block_settle()
    sc.params["ps_freq"] = 3
    sc.fluid_vel = np.zeros_like(sc.fluid_pos)
    sc.fluid_vel[:, 0] = 1.0
    out = []
    for graphs in (False, True):
        c0 = crm.load_scenario(sc, rank=0, world=3)
        ctxs = [c0] + [crm.load_scenario(sc, rank=r, world=3, stream=c0.stream()) for r in range(1, 3)]
        for c in ctxs:
            c.set_graphs(graphs)
        for _ in range(4):
            crm.group_step(ctxs, sc.dt, 7)
        assert [c.count(crm.CRM_GRAPH_REPLAYS) for c in ctxs] == [28 if graphs else 0] * 3
        out.append(dist.merge_owned([c.get_state() for c in ctxs]))
    for a, b in zip(*out):
        assert not np.isnan(a).any()
        assert np.array_equal(a, b)


def test_slab_halo_overflow_is_latched(crm, monkeypatch):
    """A boundary plane larger than the fixed-capacity halo buffer (forced small here) is a
    CRM_E_CAPACITY error latched on the device and reported by the step, with its message."""
    monkeypatch.setenv("CRM_SLAB_CAP_G", "16")
    sc = workloads.block_settle()
    c0 = crm.load_scenario(sc, rank=0, world=2)
    ctxs = [c0, crm.load_scenario(sc, rank=1, world=2, stream=c0.stream())]
    with pytest.raises(crm.CrmError) as ei:
        crm.group_step(ctxs, sc.dt, 3)
    assert ei.value.code == -9
    assert "halo buffer" in str(ei.value) or "pack buffer" in str(ei.value)
