"""CPU checks of the boundary: libcrm.so builds for sm_100a, loads, exports every symbol that
include/crm.h declares, and refuses to run without an sm_100 device (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2507_05643_b200 import build
    build.build_library()
    from paper_2507_05643_b200 import crm
    return crm.load_library()


def declared_functions():
    src = open(os.path.join(ROOT, "include", "crm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(crm_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for required in ["crm_create", "crm_add_fluid", "crm_add_bce", "crm_step", "crm_get_state"]:
        assert required in names


def test_library_exports_every_declared_symbol(lib):
    from paper_2507_05643_b200 import crm
    names = declared_functions()
    for nm in names:
        assert hasattr(lib, nm), nm
    assert sorted(crm.EXPORTS) == names
    out = subprocess.run(["nm", "-D", "--defined-only", crm.LIB_PATH], capture_output=True, text=True).stdout
    for nm in names:
        assert re.search(rf"\bT {nm}\b", out), nm


def test_library_is_sm100a_cubin(lib):
    from paper_2507_05643_b200 import crm
    out = subprocess.run(["cuobjdump", "--list-elf", crm.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_strerror_and_kernel_names(lib):
    from paper_2507_05643_b200 import crm
    assert lib.crm_strerror(0) == b"ok"
    assert lib.crm_strerror(-2) == b"particle outside the grid box"
    names = crm.kernel_names()
    assert "k_rates_B" in names and "k_bce_A" in names


def test_invalid_parameters_rejected_before_device(lib):
    import workloads
    from paper_2507_05643_b200 import crm
    sc = workloads.block_settle(n=(4, 4, 4))
    p = dict(sc.params, h=sc.params["d0"] * 0.5)      # h < d0
    with pytest.raises(crm.CrmError) as e:
        crm.Crm(p)
    assert e.value.code == crm.CRM_E_INVALID
    p = dict(sc.params, mu_s=0.9, mu_2=0.5)           # mu_s > mu_2
    with pytest.raises(crm.CrmError) as e:
        crm.Crm(p)
    assert e.value.code == crm.CRM_E_INVALID
    p = dict(sc.params, ps_freq=-1)                   # Alg. 2 period must be >= 1
    with pytest.raises(crm.CrmError) as e:
        crm.Crm(p)
    assert e.value.code == crm.CRM_E_INVALID
    p = dict(sc.params, kernel=2)                     # only cubic (0) and Wendland (1)
    with pytest.raises(crm.CrmError) as e:
        crm.Crm(p)
    assert e.value.code == crm.CRM_E_INVALID
    p = dict(sc.params, support=3.0)                  # both kernels have support 2h
    with pytest.raises(crm.CrmError) as e:
        crm.Crm(p)
    assert e.value.code == crm.CRM_E_UNSUPPORTED


def test_no_cpu_fallback_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    import workloads
    from paper_2507_05643_b200 import crm
    sc = workloads.block_settle(n=(4, 4, 4))
    with pytest.raises(crm.CrmError) as e:
        crm.Crm(sc.params)
    assert e.value.code == crm.CRM_E_CUDA


def test_capacity_policy_host_function(lib):
    """ManageArrayMemory of Alg. 3 in the product (host logic, no GPU): SPEC's scripted sequence
    1000 -> 1200 -> 1200 -> 700 @ step 50 gives Grow -> 1440, Keep, Shrink -> 700 (G = 1.2, S = 0.75,
    S_I = 50), and the same answers as the oracle's independent implementation."""
    import oracle
    from paper_2507_05643_b200 import crm
    assert crm.manage_capacity(1000, 1200, 1) == (1440, 1)
    assert crm.manage_capacity(1440, 1200, 2) == (1440, 0)
    assert crm.manage_capacity(1000, 700, 50) == (700, 2)
    rng = np.random.default_rng(3)
    for _ in range(500):
        cap, req, step = (int(v) for v in rng.integers(1, 5000, 3))
        assert crm.manage_capacity(cap, req, step) == oracle.manage_capacity(cap, req, step)


@pytest.mark.gpu   # crm_create needs a device
def test_active_box_validation(lib):
    import workloads
    from paper_2507_05643_b200 import crm
    sc = workloads.block_settle(n=(4, 4, 4))
    c = crm.Crm(sc.params)
    with pytest.raises(crm.CrmError) as e:
        c.set_active_box(3, (0.1, 0.1, 0.1))          # no such body
    assert e.value.code == crm.CRM_E_INVALID
    with pytest.raises(crm.CrmError) as e:
        c.set_active_box(0, (0.1, -1.0, 0.1))
    assert e.value.code == crm.CRM_E_INVALID
    with pytest.raises(crm.CrmError) as e:
        c.set_active_policy(0.0, 0.5, 0.75, 50)       # growth < 1
    assert e.value.code == crm.CRM_E_INVALID
    c.set_active_box(0, (0.1, 0.1, 0.1))
    c.set_active_policy(0.01)
    c.close()


def test_binding_constants_match_the_header():
    """The Python binding's CRM_* constants are the header's #defines (marshalling only: one source)."""
    from paper_2507_05643_b200 import crm
    src = open(os.path.join(ROOT, "include", "crm.h")).read()
    defs = {k: int(v) for k, v in re.findall(r"#define\s+(CRM_[A-Z0-9_]+)\s+(-?\d+)\b", src)}
    shared = [k for k in dir(crm) if k.startswith("CRM_") and isinstance(getattr(crm, k), int)]
    assert {"CRM_OWNED", "CRM_GRAPH_REPLAYS", "CRM_E_CAPACITY"} <= set(shared)
    for k in shared:
        assert k in defs, k
        assert getattr(crm, k) == defs[k], k
