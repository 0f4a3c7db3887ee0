"""Pins of the oracle's kernel (P:53–55 'Cubic', P:726 support 2h; reading A1) and of
the lattice constants that follow from it (SURVEY.md §8 lattice sums, independent NumPy)."""
import json
import math
import os

import numpy as np
import pytest
from scipy import integrate

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


@pytest.mark.parametrize("h", [1.0, 3.25e-3, 0.012])
def test_kernel_normalisation(oracle_mod, h):
    # integral of W over the support ball = 1 (closed form of a normalised kernel)
    val, _ = integrate.quad(lambda r: 4 * math.pi * r * r * oracle_mod.W(r, h), 0, 2 * h,
                            points=[h], epsabs=0, epsrel=1e-12, limit=200)
    assert abs(val - 1.0) < 1e-9


def test_kernel_textbook_values(oracle_mod):
    h = 0.7
    s3 = 1.0 / (math.pi * h ** 3)          # M4 cubic spline 3-D normalisation (Monaghan 1985)
    assert oracle_mod.W(0.0, h) == pytest.approx(s3, rel=1e-15)
    assert oracle_mod.W(h, h) == pytest.approx(0.25 * s3, rel=1e-14)
    assert oracle_mod.W(2 * h, h) == 0.0
    assert oracle_mod.W(2.5 * h, h) == 0.0
    # continuity at q = 1 and at q = 2 (no jump)
    e = 1e-9
    assert oracle_mod.W(h * (1 - e), h) == pytest.approx(oracle_mod.W(h * (1 + e), h), rel=1e-7)
    assert oracle_mod.W(h * (2 - e), h) < 1e-20 * s3 + 1e-24


def test_kernel_monotone(oracle_mod):
    h = 1.3
    r = np.linspace(0, 2.2 * h, 5000)
    w = np.array([oracle_mod.W(x, h) for x in r])
    assert np.all(np.diff(w) <= 0)
    assert np.all(w >= 0)


def test_gradient_matches_finite_difference(oracle_mod):
    # central difference of W vs dW/dr at 50 random radii in (0, 2h)
    rng = np.random.default_rng(5)
    h = 3.25e-3
    for r in rng.uniform(0.01 * h, 1.99 * h, 50):
        if abs(r - h) < 1e-4 * h:
            continue
        eps = 1e-7 * h
        fd = (oracle_mod.W(r + eps, h) - oracle_mod.W(r - eps, h)) / (2 * eps)
        an = oracle_mod.dWdr(r, h)
        assert an == pytest.approx(fd, rel=1e-6, abs=1e-9 * abs(oracle_mod.dWdr(0.5 * h, h)))


def test_gradient_radial_antisymmetric_zero_at_origin(oracle_mod):
    rng = np.random.default_rng(7)
    h = 1.0
    assert np.all(oracle_mod.gradW([0, 0, 0], h) == 0)
    for _ in range(100):
        x = rng.uniform(-2, 2, 3)
        g = oracle_mod.gradW(x, h)
        gm = oracle_mod.gradW(-x, h)
        assert np.array_equal(g, -gm)                       # bit-exact antisymmetry
        r = np.linalg.norm(x)
        if r < 2 * h:
            # radial and pointing towards -x (W decreasing): grad_i W_ij = W'(r) x_ij / r
            assert np.allclose(np.cross(g, x), 0, atol=1e-14)
            assert np.dot(g, x) <= 0
        else:
            assert np.all(g == 0)


def _lattice_sums(oracle_mod, hd):
    d0 = 1.0
    h = hd * d0
    V = d0 ** 3
    rng = np.arange(-4, 5)
    sumW = 0.0
    M = np.zeros((3, 3))
    G = np.zeros(3)
    count = 0
    shells = {}
    for a in rng:
        for b in rng:
            for c in rng:
                xj = np.array([a, b, c], float) * d0
                sumW += V * oracle_mod.W(np.linalg.norm(xj), h)
                if a == b == c == 0:
                    continue
                g = oracle_mod.gradW(-xj, h)               # grad_i W_ij with x_i = 0
                M += V * np.outer(xj, g)
                G += V * g
                n2 = a * a + b * b + c * c
                if n2 * d0 * d0 < (2 * h) ** 2:
                    count += 1
                    shells[n2] = shells.get(n2, 0) + 1
    return sumW, M, G, count, shells


@pytest.mark.parametrize("key", ["lattice_h13", "lattice_h12"])
def test_lattice_constants(oracle_mod, key):
    gold = GOLD[key]
    sumW, M, G, count, shells = _lattice_sums(oracle_mod, gold["h_over_d0"])
    assert count == gold["count"]
    assert sumW == pytest.approx(gold["sum_VW"], abs=1e-6)
    assert np.allclose(np.diag(M), gold["M_diag"], atol=1e-7)
    assert np.allclose(M - np.diag(np.diag(M)), 0, atol=1e-12)
    assert np.allclose(G, 0, atol=1e-12)
    pw = GOLD["partition_window"]
    assert pw["lo"] <= sumW <= pw["hi"]
    if "shells" in gold:
        assert {str(k): v for k, v in shells.items()} == gold["shells"]
