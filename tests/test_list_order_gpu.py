"""The bank-group-major list order (filter.cuh drain_masks_gm, reading A34) is a permutation
of each stored list: the same neighbour set, summed in another fixed order.  Against the filter's
candidate order the states may differ only by fp32 rounding; against the oracle both stay within the
parity tolerances (the ps_freq > 1 tests of test_parity_gpu.py run with it on by default)."""
import os

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


def _run(crm, sc, order, steps):
    old = os.environ.get("CRM_LIST_ORDER")
    os.environ["CRM_LIST_ORDER"] = order   # read by crm_create
    try:
        g = crm.load_scenario(sc)
    finally:
        if old is None:
            del os.environ["CRM_LIST_ORDER"]
        else:
            os.environ["CRM_LIST_ORDER"] = old
    g.step(sc.dt, steps)
    return g.get_state()


@pytest.mark.parametrize("ps_freq", [1, 4])
def test_group_major_order_is_a_permutation(crm, ps_freq):
    sc = workloads.block_settle(jitter=0.05, seed=3)
    sc.params["ps_freq"] = ps_freq
    rr = _run(crm, sc, "gmajor", 20)
    scan = _run(crm, sc, "scan", 20)
    pos_rr, vel_rr, rho_rr, sig_rr = rr[:4]
    pos_sc, vel_sc, rho_sc, sig_sc = scan[:4]
    assert not np.array_equal(sig_rr, sig_sc)   # the order really changed the summation
    assert np.abs(pos_rr - pos_sc).max() < 1e-6   # d0 / 2500
    assert np.abs(rho_rr - rho_sc).max() / np.abs(rho_sc).max() < 1e-5
    vs = np.abs(vel_sc).max()
    assert np.abs(vel_rr - vel_sc).max() < 1e-4 * max(vs, 1e-3)
    ss = np.abs(sig_sc).max()
    assert np.abs(sig_rr - sig_sc).max() < 1e-4 * ss
