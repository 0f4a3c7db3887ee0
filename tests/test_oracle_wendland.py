"""Pins of the oracle's quintic Wendland kernel ("Quintic Wendland [Wendland 1995] ... K = 2";
reading A28: W = a (1 - q/2)^4 (2q + 1), a = 21/(16 pi h^3), q = r/h < 2).

Each pin fixes a different part of the formula so that a plausible slip fails one of them:
  * normalisation (integral over the support ball = 1) fixes the constant a;
  * W'(0) = 0 (a smooth peak, the defining C2 property at the origin) fixes the linear factor
    (2q + 1): (c q + 1) has W'(0) = 0 only for c = 2;
  * W, W' and W'' vanish at q = 2 (C2 compact support) fixes the fourth power of (1 - q/2);
  * dW/dr against a central finite difference pins the derivative the rates use;
  * the interior-lattice sums at h = 1.3 d0 sit in the partition-of-unity window S:109 and give
    M = c I (isotropy), the properties the stress divergence relies on."""
import math

import numpy as np
import pytest
from scipy import integrate

import oracle


@pytest.mark.parametrize("h", [1.0, 3.25e-3, 0.012])
def test_wendland_normalisation(oracle_mod, h):
    val, _ = integrate.quad(lambda r: 4 * math.pi * r * r * oracle_mod.W_wendland(r, h), 0, 2 * h,
                            epsabs=0, epsrel=1e-12, limit=200)
    assert abs(val - 1.0) < 1e-10


def test_wendland_smooth_peak_and_compact_support(oracle_mod):
    h = 0.8
    W = lambda r: oracle_mod.W_wendland(r, h)
    dW = lambda r: oracle_mod.dWdr_wendland(r, h)
    e = 1e-5 * h
    assert dW(0.0) == 0.0
    assert abs((W(e) - W(0.0)) / e) < 1e-3 * W(0.0) / h          # flat top (one-sided slope -> 0)
    assert W(2 * h) == 0.0 and dW(2 * h) == 0.0 and W(3 * h) == 0.0
    # W and W' -> 0 continuously at the support edge, and W'' too (C2): second difference
    r0 = 2 * h - 3 * e
    d2 = (W(r0 + e) - 2 * W(r0) + W(r0 - e)) / (e * e)
    d2_mid = (W(h + e) - 2 * W(h) + W(h - e)) / (e * e)
    assert abs(d2) < 1e-4 * abs(d2_mid)
    assert abs(dW(2 * h - e)) < 1e-8 * abs(dW(h))


def test_wendland_monotone_positive(oracle_mod):
    h = 1.3
    r = np.linspace(0, 2.2 * h, 4000)
    w = np.array([oracle_mod.W_wendland(x, h) for x in r])
    assert np.all(np.diff(w) <= 0) and np.all(w >= 0) and w[0] > 0


def test_wendland_gradient_matches_finite_difference(oracle_mod):
    rng = np.random.default_rng(11)
    h = 6.5e-3
    for r in rng.uniform(0.01 * h, 1.99 * h, 50):
        eps = 1e-7 * h
        fd = (oracle_mod.W_wendland(r + eps, h) - oracle_mod.W_wendland(r - eps, h)) / (2 * eps)
        assert oracle_mod.dWdr_wendland(r, h) == pytest.approx(fd, rel=1e-6)


def test_wendland_lattice_sums(oracle_mod):
    h, V = 1.3, 1.0
    rng = np.arange(-4, 5)
    sumW, M = 0.0, np.zeros((3, 3))
    for a in rng:
        for b in rng:
            for c in rng:
                xj = np.array([a, b, c], float)
                r = np.linalg.norm(xj)
                sumW += V * oracle_mod.W_wendland(r, h)
                if r == 0:
                    continue
                g = oracle_mod.dWdr_wendland(r, h) * (-xj) / r      # grad_i W_ij with x_i = 0
                M += V * np.outer(xj, g)
    assert 0.95 <= sumW <= 1.05                                     # S:109 window
    assert np.allclose(M, M[0, 0] * np.eye(3), atol=1e-12)          # isotropic
    assert 0.95 <= M[0, 0] <= 1.05                                  # consistency of the gradient


def test_simulation_uses_the_selected_kernel(oracle_mod):
    """Two particles, sigma = 0, no gravity, bilateral AV: the pair force scales with W'(r);
    the ratio Wendland / cubic of the stage-A acceleration equals the ratio of the kernels' W'."""
    import workloads
    d0, h = 1e-3, 1.3e-3
    p = workloads.base_params(rho0=1000.0, mu_s=0.3, mu_2=0.3, I0=0.08, cohesion=0.0, grain_d=1e-3,
                              d0=d0, h=h, visc_mode=0, gamma_a=0.1, lo=(-0.01,) * 3, hi=(0.01,) * 3,
                              gravity=(0.0, 0.0, 0.0))
    x = np.array([[0.0, 0.0, 0.0], [1.5 * d0, 0.0, 0.0]])
    u = np.array([[1e-3, 0.0, 0.0], [-1e-3, 0.0, 0.0]])
    acc = {}
    for k in (0, 1):
        o = oracle.OracleSim(dict(p, kernel=k))
        o.add_fluid(x, u, np.zeros((2, 6)))
        o.step(1e-7, 1)
        acc[k] = o.last_rates(0)[1][0, 0]
        o.close()
    r = 1.5 * d0
    ratio = oracle_mod.dWdr_wendland(r, h) / oracle_mod.dWdr(r, h)
    assert acc[1] / acc[0] == pytest.approx(ratio, rel=1e-12)
