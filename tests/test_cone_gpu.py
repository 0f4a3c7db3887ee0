"""Cone penetration: a free 60 deg / 19.8 mm steel cone dropped
into the glass-bead bed with the speed of a fall from H = L.  GPU against the oracle on a reduced
bed (32 mm cube, d0 = 1 mm, the paper's resolution): the cone's trajectory within the 2 %
macroscopic bar, the bed particle by particle within 0.02 d0; and on the GPU alone the
penetration grows monotonically and the cone slows down (the soil carries it)."""
import numpy as np
import pytest

import oracle
import workloads

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def crm():
    from paper_2507_05643_b200 import build
    build.build_library()
    from paper_2507_05643_b200 import crm as m
    m.load_library()
    return m


def test_cone_drop_matches_oracle(crm):
    sc = workloads.cone_drop(n=(32, 32, 32), H_over_L=1.0)
    g = crm.load_scenario(sc)
    o = oracle.load_scenario(sc)
    steps = 60
    g.step(sc.dt, steps)
    o.step(sc.dt, steps)
    bg, bo = g.get_body(1), o.get_body(1)
    z0 = sc.meta["com0"][2]
    dz_g, dz_o = z0 - bg["pos"][2], z0 - bo["pos"][2]
    assert dz_o > 0.5 * sc.params["d0"]                       # it moved into the bed
    assert abs(dz_g - dz_o) <= 0.02 * dz_o
    assert abs(bg["vel"][2] - bo["vel"][2]) <= 0.02 * abs(bo["vel"][2])
    assert abs(bg["force"][2] - bo["force"][2]) <= 0.05 * abs(bo["force"][2]) + 1e-3
    nf = sc.n_fluid
    assert np.abs(g.get_state()[0][:nf] - o.get_state()[0][:nf]).max() < 0.02 * sc.params["d0"]


def test_cone_penetration_curve(crm):
    sc = workloads.cone_drop(n=(32, 32, 32), H_over_L=1.0)
    g = crm.load_scenario(sc)
    depth, vz = [], []
    surface = 32 * sc.params["d0"]
    for _ in range(10):
        g.step(sc.dt, 100)
        b = g.get_body(1)
        tip = b["pos"][2] - 0.75 * sc.meta["cone_L"]
        depth.append(surface - tip)
        vz.append(b["vel"][2])
    assert np.all(np.diff(depth) >= -1e-6)                  # monotone penetration
    v0 = np.sqrt(2 * 9.81 * sc.meta["cone_L"])
    assert abs(vz[-1]) < 0.8 * v0                              # the bed decelerated the cone
    assert 0 < depth[-1] < sc.meta["cone_L"] + 10 * sc.params["d0"]
