"""Oracle pin: a lithostatic column at rest is an equilibrium of the whole step.

Mechanics fixes the answer: a granular column of height H at rest in a rigid box under gravity g carries
sigma_zz(z) = -rho0 g (H - z) and stays at rest as long as the lateral stress K0 sigma_zz keeps the
deviatoric stress inside the mu(I) yield surface (Jaky's K0 = 1 - sin(atan mu_s) gives tau/p = 0.20 <
mu_s = 0.3, reading A20).  Every term of the step takes part: the momentum sum (Eq. momentum)
must balance gravity with the discrete stress divergence (lattice constant M = 0.9935, tests/golden
lattice_h13), the Adami wall extrapolation must carry the hydrostatic term into the markers
(else the bottom layers accelerate), the stress rate must vanish for u = 0, the return map must leave an
admissible stress alone, and RK2 must not inject motion.  A sign error, a dropped term or a wrong factor
in any of them breaks the balance within a few dozen steps (measured: |u| reaches 1e-3..1e-1 g t)."""
import numpy as np

import oracle
import workloads


def test_lithostatic_column_stays_at_rest(oracle_mod):
    sc = workloads.block_settle(n=(8, 8, 12))
    p = sc.params
    g = -p["gravity"][2]
    H = 12 * p["d0"]
    K0 = 1.0 - np.sin(np.arctan(p["mu_s"]))
    nf = sc.n_fluid
    sig = workloads.lithostatic_stress(sc.fluid_pos, p["rho0"], g, H, K0)
    o = oracle.OracleSim(p)
    o.add_fluid(sc.fluid_pos, np.zeros_like(sc.fluid_pos), sig)
    o.add_bce(0, sc.wall_pos)
    steps = 100
    o.step(sc.dt, steps)
    x, u, rho, s = o.get_state(0, nf)
    o.close()
    # at rest: the velocity stays a tiny fraction of free fall g t
    assert np.abs(u).max() < 0.01 * g * steps * sc.dt
    # no settlement: mean vertical displacement far below a lattice spacing
    assert abs((x[:, 2] - sc.fluid_pos[:, 2]).mean()) < 1e-4 * p["d0"]
    # sigma_zz per lattice layer follows -rho0 g (H - z) (1 % of the base stress per layer, measured 1.0 %
    # at the free surface, <= 0.2 % inside)
    szz = -p["rho0"] * g * (H - sc.fluid_pos[:, 2])
    layer = np.round(sc.fluid_pos[:, 2] / p["d0"] - 0.5).astype(int)
    base = p["rho0"] * g * H
    for k in range(12):
        m = layer == k
        assert abs(s[m, 2].mean() - szz[m].mean()) < 0.015 * base, k
    # lateral stress stays at K0 sigma_zz (no spurious yield)
    inner = (layer >= 2) & (layer <= 9)
    ratio = s[inner, 0].sum() / s[inner, 2].sum()
    assert abs(ratio - K0) < 0.02
