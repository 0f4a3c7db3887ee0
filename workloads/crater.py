"""Sphere-cratering measurement driver (readings A22, A23).  Holds no method
arithmetic: it drives any simulation object with the crm call shape (.step, .get_body) — the oracle
or the CUDA path — and measures the penetration depth D of the free sphere, then fits the empirical
law D = 0.14/mu_s (rho_s/rho_g)^1/2 (2R)^2/3 H^1/3 (Eq. ballDropEquation)."""
from __future__ import annotations

import math

import numpy as np

from . import (BODY_FREE, E_CRATER_SOIL, Body, Scenario, bce_layers, box_walls, f32, lattice_block,
               sphere_shell_markers)

RHO_G, MU_S, R_SPHERE = 1510.0, 0.3, 0.0125   # P:7
CASES = [(rs, H) for rs in (700.0, 2200.0) for H in (0.05, 0.1, 0.2)]


def law_abscissa(rho_s: float, H: float, mu_s: float = MU_S, rho_g: float = RHO_G, R: float = R_SPHERE) -> float:
    """x = (1/mu_s) (rho_s/rho_g)^1/2 (2R)^2/3 H^1/3, so that the law reads D = 0.14 x."""
    return (1.0 / mu_s) * math.sqrt(rho_s / rho_g) * (2 * R) ** (2.0 / 3.0) * H ** (1.0 / 3.0)


def scenario(rho_s: float, H: float, d0: float = 5e-3, dt: float = 5e-5, E: float = E_CRATER_SOIL) -> Scenario:
    """Settled-looking bed (lithostatic start, K0 = 1 - sin(atan mu_s), reading A20) in the
    0.14 x 0.10 x 0.15 m container, sphere bottom at the surface moving down at sqrt(2 g H)."""
    from . import base_params, lithostatic_stress
    h = 1.3 * d0
    nx, ny, nz = int(round(0.14 / d0)), int(round(0.10 / d0)), int(round(0.15 / d0))
    L = bce_layers(h, d0)
    fb = int(round(0.06 / d0))                      # walls 6 cm above the bed keep the ejecta inside
    walls = box_walls(nx, ny, nz, d0, L, fb)
    m = (L + 1) * d0
    head = int(round(0.15 / d0))
    p = base_params(rho0=RHO_G, mu_s=MU_S, mu_2=MU_S, I0=0.08, cohesion=0.0, grain_d=1e-3, d0=d0, h=h, E=E,
                    visc_mode=0, gamma_a=0.01, lo=(-m, -m, -m), hi=(nx * d0 + m, ny * d0 + m, (nz + 4 + head) * d0))
    pos = f32(lattice_block(nx, ny, nz, d0))
    K0 = 1.0 - math.sin(math.atan(MU_S))
    sig = f32(lithostatic_stress(pos, RHO_G, 9.81, nz * d0, K0))
    surface = nz * d0
    centre = f32(np.array([nx * d0 / 2, ny * d0 / 2, surface + R_SPHERE + 0.5 * d0]))
    mass = rho_s * 4.0 / 3.0 * math.pi * R_SPHERE ** 3
    I = 0.4 * mass * R_SPHERE ** 2
    v = math.sqrt(2 * 9.81 * H)
    local = sphere_shell_markers(R_SPHERE, d0, L)
    sphere = Body(mass=mass, inertia=(I, I, I), pos=tuple(centre), vel=(0.0, 0.0, -v), motion=BODY_FREE,
                  dof_mask=0b000111, markers=f32(local + centre))
    return Scenario(f"crater_{int(rho_s)}_{H}", p, pos, None, sig, f32(walls), [sphere], dt, 0,
                    meta=dict(rho_s=rho_s, H=H, surface=surface, z0=float(centre[2]), E=E))


def penetration(sim, sc: Scenario, chunk: int = 20, t_max: float = 0.25, window: float = 0.02,
                ke_rest: float = 1e-5, drift: float = 5e-3) -> dict:
    """Depth of the free sphere at rest (reading A23): D = initial minus resting centre height (the
    sphere bottom starts at the undisturbed surface, A22/A23).  "At rest" (S:604-605 ask for a
    sphere kinetic energy below 1e-6 of the impact energy; the SPH contact keeps a jitter of
    ~1e-6 of it, so the test is made on a window): over the last `window` seconds the mean
    KE/KE0 is below `ke_rest` and the depth moved by less than `drift` D.  Also reports the depth
    at the first upward velocity (the earlier, bounce-based measure) and the deepest point."""
    z0 = sc.meta["z0"]
    v0 = math.sqrt(2 * 9.81 * sc.meta["H"])
    nwin = max(2, int(round(window / (chunk * sc.dt))))
    hist = []        # (D, KE/KE0) per chunk
    zmin, steps, D_first = z0, 0, None
    at_rest = False
    max_steps = int(round(t_max / sc.dt))
    while steps < max_steps:
        sim.step(sc.dt, chunk)
        steps += chunk
        b = sim.get_body(1)
        z = float(b["pos"][2])
        zmin = min(zmin, z)
        v = np.asarray(b["vel"], float)
        hist.append((z0 - z, float(v @ v) / (v0 * v0)))
        if D_first is None and v[2] >= 0.0:
            D_first = z0 - zmin
        if len(hist) > nwin:
            Dw = [h[0] for h in hist[-nwin - 1:]]
            ke = float(np.mean([h[1] for h in hist[-nwin:]]))
            if ke < ke_rest and abs(Dw[-1] - Dw[0]) < drift * abs(Dw[-1]):
                at_rest = True
                break
    return dict(D=hist[-1][0], D_first_stop=D_first if D_first is not None else z0 - zmin, D_max=z0 - zmin,
                at_rest=at_rest, steps=steps, t=steps * sc.dt,
                ke_window=float(np.mean([h[1] for h in hist[-nwin:]])))


def fit(xs, Ds) -> dict:
    """Slope through the origin and OLS line with R^2 and MSE against D = 0.14 x."""
    x = np.asarray(xs, float)
    D = np.asarray(Ds, float)
    slope0 = float((x * D).sum() / (x * x).sum())
    A = np.vstack([x, np.ones_like(x)]).T
    (a, b), *_ = np.linalg.lstsq(A, D, rcond=None)
    pred = a * x + b
    ss_res = float(((D - pred) ** 2).sum())
    ss_tot = float(((D - D.mean()) ** 2).sum())
    r2 = 1.0 - ss_res / ss_tot if ss_tot > 0 else 1.0
    mse_law = float(((D - 0.14 * x) ** 2).mean())
    return dict(slope_origin=slope0, slope_ols=float(a), intercept=float(b), R2=r2, MSE_vs_law=mse_law)
