"""Pins of the oracle's structural layer: hash, sort + cellStart,
Alg. 1 neighbour lists against the O(N^2) definition, with rules B1–B5."""
import json
import os

import numpy as np
import pytest

import workloads

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def test_paper_hash_example(oracle_mod):
    g = GOLD["hash_example"]
    X, Y, _ = g["dims_XYZ"]
    x, y, z = g["coords_xyz"]
    assert oracle_mod.paper_cell_index(x, y, z, X, Y) == g["c"]
    assert oracle_mod.paper_cell_index(0, 0, 0, X, Y) == 0


def test_cell_coords_rules(oracle_mod):
    dims = (4, 5, 6)
    rc, c = oracle_mod.cell_coords([0.0, 0.0, 0.0], [0, 0, 0], 0.5, dims)
    assert rc == 0 and c == (0, 0, 0)
    # exactly on a face -> the higher cell (half-open cells)
    rc, c = oracle_mod.cell_coords([0.5, 1.0, 2.5], [0, 0, 0], 0.5, dims)
    assert rc == 0 and c == (1, 2, 5)
    # outside -> domain error
    assert oracle_mod.cell_coords([-1e-3, 0, 0], [0, 0, 0], 0.5, dims)[0] == oracle_mod.OC_E_DOMAIN
    assert oracle_mod.cell_coords([2.0, 0, 0], [0, 0, 0], 0.5, dims)[0] == oracle_mod.OC_E_DOMAIN


@pytest.mark.parametrize("bce", [(0.012, 0.01, 3), (0.006, 0.005, 3), (0.01, 0.01, 2), (0.00325, 0.0025, 3)])
def test_bce_layer_count(bce):
    h, d0, n = bce
    assert workloads.bce_layers(h, d0) == n


def _sim_from_cloud(oracle_mod, x, h, lo=-0.1, hi=1.1):
    p = workloads.base_params(rho0=1000.0, mu_s=0.5, mu_2=0.5, I0=0.08, cohesion=0.0,
                              grain_d=1e-3, d0=h, h=h, visc_mode=0, gamma_a=0.0,
                              lo=(lo,) * 3, hi=(hi,) * 3)
    s = oracle_mod.OracleSim(p)
    s.add_fluid(x)
    return s


def test_pair_predicate_strict(oracle_mod):
    h = 0.5    # 2h = 1 exactly in fp32
    x = np.array([[0, 0, 0], [1.0, 0, 0], [0, 0.95, 0]], float)
    off, lst = oracle_mod.brute_neighbors(x, 2 * h)
    assert list(lst[off[0]:off[1]]) == [2]          # distance 2h is NOT a neighbour
    assert list(lst[off[1]:off[2]]) == []
    # equilateral triangle of side 1.5h -> 2 neighbours each
    t = np.array([[0, 0, 0], [0.75, 0, 0], [0.375, 0.75 * np.sqrt(3) / 2, 0]], np.float32).astype(float)
    off, _ = oracle_mod.brute_neighbors(t, 2 * h)
    assert list(np.diff(off)) == [2, 2, 2]


def test_alg1_equals_brute_force_random_clouds(oracle_mod):
    # 50 random configurations, random h, cell-list result == brute force, set-equal
    rng = np.random.default_rng(123)
    for k in range(50):
        n = int(rng.integers(1, 1500))
        h = float(rng.uniform(0.01, 0.12))
        x = workloads.random_cloud(n, seed=1000 + k)
        s = _sim_from_cloud(oracle_mod, x, h)
        off, lst = s.neighbors()
        boff, blst = oracle_mod.brute_neighbors(x, 2 * h)
        assert np.array_equal(off, boff)
        assert np.array_equal(lst, blst)
        # symmetry j in P(i) <=> i in P(j)
        pairs = set()
        for i in range(n):
            for j in lst[off[i]:off[i + 1]]:
                pairs.add((i, int(j)))
        assert all((j, i) in pairs for (i, j) in pairs)
        s.close()


def test_sort_and_cell_start(oracle_mod):
    x = workloads.random_cloud(3000, seed=9)
    s = _sim_from_cloud(oracle_mod, x, 0.05)
    st = s.structure()
    cell = st["cell"].astype(np.int64)
    ids = np.arange(len(cell))
    # lexicographic (cell, id) order (B4) via numpy's library sort
    assert np.array_equal(st["sorted_ids"], np.lexsort((ids, cell)))
    cs = st["cell_start"].astype(np.int64)
    assert cs[0] == 0 and cs[-1] == len(cell)
    assert np.array_equal(np.diff(cs), np.bincount(cell, minlength=len(cs) - 1))
    # B1/B3: cell id from floor((x - lo)/s) with z fastest, x slowest
    s32 = np.float32(0.1)
    lo = np.float32(-0.1)
    cx = np.floor((x.astype(np.float32) - lo) / s32).astype(np.int64)
    dims = int(np.ceil((1.1 - -0.1) / (2 * 0.05)))
    assert np.array_equal(cell, cx[:, 0] * dims * dims + cx[:, 1] * dims + cx[:, 2])
    s.close()


@pytest.mark.parametrize("hd,count", [(1.3, 80), (1.2, 56)])
def test_lattice_interior_counts(oracle_mod, hd, count):
    d0 = 0.01
    pos = workloads.f32(workloads.lattice_block(12, 12, 12, d0))
    s = _sim_from_cloud(oracle_mod, pos, hd * d0, lo=-0.05, hi=0.17)
    cnt = s.structure()["counts"]
    interior = np.all((pos > 3 * d0) & (pos < 9 * d0), axis=1)
    assert np.all(cnt[interior] == count)
    s.close()
