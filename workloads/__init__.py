"""Seeded synthetic input generators shared by the tests, the bench and smoke().

This module holds NONE of the method's arithmetic (no kernel, no rates, no
integration, no binning): it only lays particles on lattices, places BCE markers
around containers and spheres, draws seeded random perturbations and assembles
the parameter sets of the BASELINE.json configurations (recipes in DESIGN.md
§Inputs).  Both the oracle (oracle/) and the CUDA path (paper_2507_05643_b200/)
consume its output; neither is imported here.

Geometry conventions:
  * fluid lattice positions (i + 1/2) d0 inside the container [0, n d0)^3,
  * container walls: floor + 4 sides of BCE markers at -(k + 1/2) d0 outside the
    wall planes, k = 0 .. L-1, L = ceil(support h / d0) (reading A21),
    side walls rising to (nz + freeboard) d0,
  * positions are rounded to fp32-representable values so that both sides see
    exactly the same inputs.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

VISC_BILATERAL = 0
VISC_UNILATERAL = 1
BODY_FIXED, BODY_FREE, BODY_PRESCRIBED = 0, 1, 2
# Young's modulus of the cratering soil (P:7 gives rho and mu_s only; reading A2'): 2e5 Pa, the
# value for which the cratering sweep at the paper's d0 = 2.5 mm reproduces the paper's regression
# (slope 0.1348 vs 0.1336, R^2 0.98 vs 0.9714); E = 1e6 Pa gives slope 0.082.
E_CRATER_SOIL = 2e5


def elastic_moduli(E: float, nu: float) -> tuple[float, float]:
    """K, G from Young's modulus and Poisson ratio (reading A2: E = 1e6 Pa, nu = 0.3)."""
    return E / (3.0 * (1.0 - 2.0 * nu)), E / (2.0 * (1.0 + nu))


def bce_layers(h: float, d0: float, support: float = 2.0) -> int:
    """Number of BCE layers N = ceil(K h / d0)."""
    return int(math.ceil(support * h / d0 - 1e-12))


def f32(a: np.ndarray) -> np.ndarray:
    """Round to fp32-representable values, returned as fp64."""
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def lattice_block(nx: int, ny: int, nz: int, d0: float, origin=(0.0, 0.0, 0.0)) -> np.ndarray:
    """(i + 1/2) d0 lattice, x slowest, z fastest (matches the cell ordering, not required)."""
    i, j, k = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    pos = np.stack([(i + 0.5) * d0, (j + 0.5) * d0, (k + 0.5) * d0], axis=-1).reshape(-1, 3)
    return pos + np.asarray(origin, dtype=np.float64)


def box_walls(nx: int, ny: int, nz: int, d0: float, layers: int, freeboard: int) -> np.ndarray:
    """Floor + 4 side walls of the container [0,nx d0) x [0,ny d0) x [0, ...) (reading A21).

    Count = (nx+2L)(ny+2L) L + ((nx+2L)(ny+2L) - nx ny)(nz + freeboard).
    """
    L = layers
    ii, jj = np.meshgrid(np.arange(-L, nx + L), np.arange(-L, ny + L), indexing="ij")
    ii = ii.ravel(); jj = jj.ravel()
    floor = []
    for k in range(1, L + 1):
        floor.append(np.stack([(ii + 0.5) * d0, (jj + 0.5) * d0, np.full(ii.shape, (-k + 0.5) * d0)], -1))
    ring_mask = (ii < 0) | (ii >= nx) | (jj < 0) | (jj >= ny)
    ri, rj = ii[ring_mask], jj[ring_mask]
    ring = []
    for k in range(0, nz + freeboard):
        ring.append(np.stack([(ri + 0.5) * d0, (rj + 0.5) * d0, np.full(ri.shape, (k + 0.5) * d0)], -1))
    return np.concatenate(floor + ring, axis=0)


def sphere_shell_markers(R: float, d0: float, layers: int) -> np.ndarray:
    """BCE markers on a sphere: shells at R - k d0, k = 0..layers-1, spacing ~d0.

    Each shell uses a Fibonacci lattice with round(4 pi r^2 / d0^2) points; returned
    in the body frame (centre at the origin).
    """
    out = []
    golden = math.pi * (3.0 - math.sqrt(5.0))
    for k in range(layers):
        r = R - k * d0
        if r <= 0.25 * d0:
            break
        n = max(1, int(round(4.0 * math.pi * r * r / (d0 * d0))))
        idx = np.arange(n) + 0.5
        z = 1.0 - 2.0 * idx / n
        rho = np.sqrt(np.maximum(0.0, 1.0 - z * z))
        th = golden * idx
        out.append(np.stack([r * rho * np.cos(th), r * rho * np.sin(th), r * z], -1))
    return np.concatenate(out, axis=0)


def lithostatic_stress(pos: np.ndarray, rho0: float, g: float, H: float, K0: float) -> np.ndarray:
    """Initial sigma_zz = -rho0 g (H - z), sigma_xx = sigma_yy = K0 sigma_zz (reading A20)."""
    szz = -rho0 * g * np.maximum(H - pos[:, 2], 0.0)
    s = np.zeros((pos.shape[0], 6))
    s[:, 0] = K0 * szz; s[:, 1] = K0 * szz; s[:, 2] = szz
    return s


@dataclass
class Body:
    mass: float = 0.0
    inertia: tuple = (0.0, 0.0, 0.0)
    pos: tuple = (0.0, 0.0, 0.0)
    quat: tuple = (1.0, 0.0, 0.0, 0.0)
    vel: tuple = (0.0, 0.0, 0.0)
    omega: tuple = (0.0, 0.0, 0.0)
    motion: int = BODY_FIXED
    dof_mask: int = 0
    markers: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))   # world positions


@dataclass
class Scenario:
    name: str
    params: dict
    fluid_pos: np.ndarray
    fluid_vel: np.ndarray | None
    fluid_sig: np.ndarray | None
    wall_pos: np.ndarray
    bodies: list
    dt: float
    steps: int
    meta: dict = field(default_factory=dict)
    # active domains (Alg. 3): {"boxes": {body index: half extents}, "t_delay": s}; body 0 = walls,
    # body k = bodies[k - 1]
    active: dict = field(default_factory=dict)

    @property
    def n_fluid(self) -> int:
        return int(self.fluid_pos.shape[0])

    @property
    def n_bce(self) -> int:
        return int(self.wall_pos.shape[0] + sum(b.markers.shape[0] for b in self.bodies))


def base_params(*, rho0, mu_s, mu_2, I0, cohesion, grain_d, d0, h, visc_mode, gamma_a,
                lo, hi, E=1e6, nu=0.3, gravity=(0.0, 0.0, -9.81)) -> dict:
    K, G = elastic_moduli(E, nu)
    return dict(rho0=rho0, K=K, G=G, mu_s=mu_s, mu_2=mu_2, I0=I0, cohesion=cohesion,
                grain_d=grain_d, d0=d0, h=h, support=2.0, visc_mode=visc_mode,
                gamma_a=gamma_a, xi2=0.0, cs=0.0, gravity=tuple(gravity),
                lo=tuple(lo), hi=tuple(hi))


def container(nx, ny, nz, d0, h, freeboard, headroom):
    """Wall markers and the grid box enclosing container + headroom above the walls."""
    L = bce_layers(h, d0)
    walls = box_walls(nx, ny, nz, d0, L, freeboard)
    m = (L + 1) * d0
    lo = (-m, -m, -m)
    hi = (nx * d0 + m, ny * d0 + m, (nz + freeboard + headroom) * d0)
    return walls, lo, hi


def block_settle(n=(20, 20, 20), d0=2.5e-3, h=3.25e-3, jitter=0.0, seed=0, freeboard=4,
                 headroom=8, dt=5e-5, steps=100) -> Scenario:
    """C1: granular block settling in an Adami-walled box (BJ configs[0]; cratering soil, P:7)."""
    nx, ny, nz = n
    walls, lo, hi = container(nx, ny, nz, d0, h, freeboard, headroom)
    pos = lattice_block(nx, ny, nz, d0)
    if jitter > 0:
        rng = np.random.default_rng(seed)
        pos = pos + rng.uniform(-jitter, jitter, pos.shape) * d0
    p = base_params(rho0=1510.0, mu_s=0.3, mu_2=0.3, I0=0.08, cohesion=0.0, grain_d=1e-3, E=E_CRATER_SOIL,
                    d0=d0, h=h, visc_mode=VISC_BILATERAL, gamma_a=0.01, lo=lo, hi=hi)
    return Scenario("block8k" if n == (20, 20, 20) else f"block{nx}x{ny}x{nz}", p,
                    f32(pos), None, None, f32(walls), [], dt, steps,
                    meta=dict(n=n, H=nz * d0, jitter=jitter, seed=seed))


def rate_state_S0(sc: Scenario, seed_jitter=1, seed_u=2, seed_sig=3, jitter=0.1,
                  A_scale=1.0, u_noise=0.01, sig_noise=50.0) -> Scenario:
    """Rate-parity state S0: jitter 0.1 d0, u = A x + N(0, 0.01),
    sigma = lithostatic + symmetric N(0, 50 Pa).  Returns a new Scenario."""
    d0 = sc.params["d0"]
    r1 = np.random.default_rng(seed_jitter)
    pos = sc.fluid_pos + r1.uniform(-jitter, jitter, sc.fluid_pos.shape) * d0
    r2 = np.random.default_rng(seed_u)
    A = r2.normal(0.0, A_scale, (3, 3))
    c = pos.mean(axis=0)
    vel = (pos - c) @ A.T + r2.normal(0.0, u_noise, pos.shape)
    r3 = np.random.default_rng(seed_sig)
    H = sc.meta.get("H", pos[:, 2].max())
    K, G = sc.params["K"], sc.params["G"]
    nu = (3 * K - 2 * G) / (2 * (3 * K + G))
    sig = lithostatic_stress(pos, sc.params["rho0"], 9.81, H, nu / (1 - nu))
    sig = sig + r3.normal(0.0, sig_noise, sig.shape)
    out = Scenario(sc.name + "_S0", dict(sc.params), f32(pos), f32(vel), f32(sig), sc.wall_pos,
                   sc.bodies, sc.dt, sc.steps, meta=dict(sc.meta, A=A))
    return out


def cratering(rho_s=2200.0, H_drop=0.1, d0=2.5e-3, h=None, dt=5e-5, steps=100, headroom=12,
              fill=None) -> Scenario:
    """C2: sphere cratering (Table; BJ configs[1]).

    0.14 x 0.1 x 0.15 m container; soil 56 x 40 x 60 at d0 = 2.5 mm (or scaled);
    R = 12.5 mm rigid sphere (3 marker shells), bottom at the surface, moving down at
    v = sqrt(2 g H) (reading A22)."""
    h = 1.3 * d0 if h is None else h
    Lx, Ly, Lz = 0.14, 0.10, 0.15
    nx, ny = int(round(Lx / d0)), int(round(Ly / d0))
    nz = int(round(Lz / d0)) if fill is None else fill
    walls, lo, hi = container(nx, ny, nz, d0, h, 4, headroom + int(round(0.05 / d0)))
    pos = lattice_block(nx, ny, nz, d0)
    p = base_params(rho0=1510.0, mu_s=0.3, mu_2=0.3, I0=0.08, cohesion=0.0, grain_d=1e-3, E=E_CRATER_SOIL,
                    d0=d0, h=h, visc_mode=VISC_BILATERAL, gamma_a=0.01, lo=lo, hi=hi)
    R = 0.0125
    L = bce_layers(h, d0)
    local = sphere_shell_markers(R, d0, L)
    surface = nz * d0
    centre = np.array([nx * d0 / 2, ny * d0 / 2, surface + R + 0.5 * d0])
    mass = rho_s * 4.0 / 3.0 * math.pi * R ** 3
    I = 0.4 * mass * R * R
    v = math.sqrt(2 * 9.81 * H_drop)
    sphere = Body(mass=mass, inertia=(I, I, I), pos=tuple(centre), vel=(0.0, 0.0, -v),
                  motion=BODY_FREE, dof_mask=0b000111, markers=f32(local + centre))
    # the sphere centre itself is stored at fp32 too, so that marker offsets are exact
    sphere.pos = tuple(f32(centre))
    return Scenario(f"crater_rho{int(rho_s)}_H{H_drop}", p, f32(pos), None, None, f32(walls),
                    [sphere], dt, steps, meta=dict(R=R, rho_s=rho_s, H=H_drop, surface=surface))


def bed(n=(1024, 512, 64), d0=5e-3, h=6.5e-3, jitter=0.01, seed=0, dt=5e-5, steps=200,
        freeboard=3, headroom=6) -> Scenario:
    """C5: synthetic RASSOR-scale granular bed (BJ configs[4]; RASSOR soil P:156, Table).

    Lithostatic initial stress (reading A20), unilateral AV 0.02."""
    nx, ny, nz = n
    walls, lo, hi = container(nx, ny, nz, d0, h, freeboard, headroom)
    pos = lattice_block(nx, ny, nz, d0)
    if jitter > 0:
        rng = np.random.default_rng(seed)
        pos = pos + rng.uniform(-jitter, jitter, pos.shape) * d0
    p = base_params(rho0=1700.0, mu_s=0.7, mu_2=0.7, I0=0.08, cohesion=0.0, grain_d=1e-3,
                    d0=d0, h=h, visc_mode=VISC_UNILATERAL, gamma_a=0.02, lo=lo, hi=hi)
    K, G = p["K"], p["G"]
    nu = (3 * K - 2 * G) / (2 * (3 * K + G))
    pos = f32(pos)
    sig = lithostatic_stress(pos, p["rho0"], 9.81, nz * d0, nu / (1 - nu))
    return Scenario(f"bed{nx}x{ny}x{nz}", p, pos, None, f32(sig), f32(walls), [], dt, steps,
                    meta=dict(n=n, H=nz * d0))


def cone_bed(d0=1e-3, n=(100, 100, 100), dt=2e-5, steps=100) -> Scenario:
    """C3 throughput shape: 0.1 m cube of glass beads (Table, reading A24)."""
    nx, ny, nz = n
    h = 1.3 * d0
    walls, lo, hi = container(nx, ny, nz, d0, h, 4, 8)
    pos = lattice_block(nx, ny, nz, d0)
    p = base_params(rho0=1500.0, mu_s=0.7, mu_2=0.8, I0=0.08, cohesion=0.0, grain_d=3e-3,
                    d0=d0, h=h, visc_mode=VISC_BILATERAL, gamma_a=0.2, lo=lo, hi=hi)
    return Scenario("cone_bed", p, f32(pos), None, None, f32(walls), [], dt, steps, meta=dict(n=n))


def mgru3_bin(d0=1e-2, n=(500, 80, 25), dt=2.5e-4, steps=100) -> Scenario:
    """C4 throughput shape: MGRU3 soil bin (Table)."""
    nx, ny, nz = n
    h = 1.2 * d0
    walls, lo, hi = container(nx, ny, nz, d0, h, 4, 8)
    pos = lattice_block(nx, ny, nz, d0)
    mu = math.tan(math.radians(38.4))
    p = base_params(rho0=1760.0, mu_s=mu, mu_2=mu, I0=0.08, cohesion=0.0, grain_d=1e-3,
                    d0=d0, h=h, visc_mode=VISC_UNILATERAL, gamma_a=0.02, lo=lo, hi=hi)
    return Scenario("mgru3_bin", p, f32(pos), None, None, f32(walls), [], dt, steps, meta=dict(n=n))


def cone_markers(apex_deg: float, R: float, d0: float, layers: int) -> np.ndarray:
    """BCE markers of a solid cone, apex at the origin pointing down (-z), axis +z, base radius R
    at height L = R / tan(apex/2): layer k is the lateral surface moved inward by k d0 (a copy
    shifted up the axis by k d0 / sin(apex/2)) plus the base disk at L - k d0; rings at slant
    spacing ~d0, ~d0 along each ring (P:467 'first layer on the surface')."""
    half = math.radians(apex_deg) / 2.0
    L = R / math.tan(half)
    out = [np.zeros((1, 3))]                       # the apex itself
    for k in range(layers):
        z0 = k * d0 / math.sin(half)               # apex of the k-th inward surface
        slant = (L - z0) / math.cos(half)
        for j in range(1 if k == 0 else 0, int(slant / d0) + 1):
            s = j * d0
            r, z = s * math.sin(half), z0 + s * math.cos(half)
            if z > L - k * d0 + 1e-12 or r <= 0.0:
                continue
            nt = max(3, int(round(2 * math.pi * r / d0)))
            th = (np.arange(nt) + 0.5 * (j % 2)) * (2 * math.pi / nt)
            out.append(np.stack([r * np.cos(th), r * np.sin(th), np.full(nt, z)], -1))
        zb = L - k * d0                             # base disk of layer k
        rb = (zb - z0) * math.tan(half) - 0.5 * d0
        for ir in range(int(rb / d0) + 1):
            r = ir * d0
            nt = 1 if r == 0 else int(round(2 * math.pi * r / d0))
            th = np.arange(nt) * (2 * math.pi / nt)
            out.append(np.stack([r * np.cos(th), r * np.sin(th), np.full(nt, zb)], -1))
    return np.concatenate(out, axis=0)


def cone_drop(apex_deg=60.0, diameter=19.8e-3, H_over_L=0.0, n=(100, 100, 100), d0=1e-3, dt=2e-5,
              steel=7850.0) -> Scenario:
    """the cone penetration test of P:65–104 on the C3 glass-bead bed: a
    60 deg / 19.8 mm cone (30 deg / 9.2 mm for Ottawa sand) dropped with its tip at the surface and
    the speed of a fall from H = 0, L/2 or L (v = sqrt(2 g H)).  The cone's mass is not printed:
    a solid steel cone (reading A32).  Translation along z only (dof_mask = 4)."""
    sc = cone_bed(d0=d0, n=n, dt=dt)
    nx, ny, nz = n
    R = 0.5 * diameter
    half = math.radians(apex_deg) / 2.0
    L = R / math.tan(half)
    mass = steel * math.pi * R * R * L / 3.0
    tip = np.array([0.5 * nx * d0, 0.5 * ny * d0, nz * d0 + 0.5 * d0])
    com = tip + np.array([0.0, 0.0, 0.75 * L])    # centroid of a solid cone: 3L/4 from the apex
    local = cone_markers(apex_deg, R, d0, bce_layers(sc.params["h"], d0))
    I_ax = 0.3 * mass * R * R
    I_tr = mass * (0.15 * R * R + 0.0375 * L * L)
    v0 = math.sqrt(2 * 9.81 * H_over_L * L)
    b = Body(mass=mass, inertia=(I_tr, I_tr, I_ax), pos=tuple(com), vel=(0.0, 0.0, -v0),
             motion=BODY_FREE, dof_mask=4, markers=f32(local + tip))
    hi = list(sc.params["hi"])
    hi[2] = max(hi[2], tip[2] + L + 4 * d0)
    sc.params["hi"] = tuple(hi)
    sc.bodies = [b]
    sc.name = f"cone{int(apex_deg)}_H{H_over_L:g}L"
    sc.meta.update(cone_L=L, cone_R=R, tip0=tip.tolist(), com0=com.tolist(), mass=mass)
    return sc


def cylinder_markers(R: float, width: float, d0: float, layers: int) -> np.ndarray:
    """BCE markers of a wheel rim: cylindrical shells r = R - k d0 (k < layers) about the body y
    axis, spacing ~d0 along the arc and the width."""
    out = []
    ny = max(1, int(round(width / d0)))
    ys = (np.arange(ny) + 0.5) * (width / ny) - 0.5 * width
    for k in range(layers):
        r = R - k * d0
        nt = max(8, int(round(2 * math.pi * r / d0)))
        th = (np.arange(nt) + 0.5) * (2 * math.pi / nt)
        T, Y = np.meshgrid(th, ys, indexing="ij")
        out.append(np.stack([r * np.cos(T).ravel(), Y.ravel(), r * np.sin(T).ravel()], -1))
    return np.concatenate(out, axis=0)


def mgru3_wheel(d0=1e-2, n=(500, 80, 25), R=0.2, width=0.2, vx=0.2, slip=0.3, sinkage=0.02,
                active=True, dt=2.5e-4, free=False, omega=0.8, load=15.0, x0=0.8) -> Scenario:
    """NEXT #2/#3 workload: the C4 MGRU3 soil bin with a rolling wheel (rim markers) and the paper's
    MGRU3 active box 0.6 x 0.6 x 0.8 m around it (P:950, P:960 'Active Box: 0.6 x 0.6 x 0.8 m',
    Alg. 3); fluid inside the wheel removed; lithostatic (settled) initial stress.

    free=False: prescribed motion, v = vx, omega_y = vx / (R (1 - slip)), fixed sinkage (throughput).
    free=True: the paper's single-wheel rig: constant angular velocity omega, free to
    move in x and z under a wheel load of `load` kg (the rover mass is not printed: reading A33),
    starting at rest on the surface; the slip follows from the steady forward speed."""
    sc = mgru3_bin(d0=d0, n=n, dt=dt)
    nx, ny, nz = n
    c = np.array([x0, 0.5 * ny * d0, nz * d0 + R - (0.0 if free else sinkage)])
    rim = cylinder_markers(R, width, d0, bce_layers(sc.params["h"], d0))
    rel = sc.fluid_pos - c
    inside = (rel[:, 0] ** 2 + rel[:, 2] ** 2 < (R + 0.5 * d0) ** 2) & (np.abs(rel[:, 1]) < 0.5 * width + d0)
    sc.fluid_pos = sc.fluid_pos[~inside]
    # a settled terrain (the paper lets it settle for t_delay = 1 s before activating the boxes,
    # P:950): lithostatic initial stress (reading A20)
    K, G = sc.params["K"], sc.params["G"]
    nu = (3 * K - 2 * G) / (2 * (3 * K + G))
    sc.fluid_sig = f32(lithostatic_stress(sc.fluid_pos, sc.params["rho0"], 9.81, nz * d0, nu / (1 - nu)))
    hi = list(sc.params["hi"])
    hi[2] = max(hi[2], c[2] + 2.5 * R)            # grid box well above the wheel top (thrown soil)
    sc.params["hi"] = tuple(hi)
    if free:
        b = Body(mass=load, inertia=(1.0, 1.0, 1.0), pos=tuple(c), vel=(0.0, 0.0, 0.0),
                 omega=(0.0, omega, 0.0), motion=BODY_FREE, dof_mask=1 | 4, markers=f32(rim + c))
    else:
        b = Body(mass=10.0, inertia=(1.0, 1.0, 1.0), pos=tuple(c), vel=(vx, 0.0, 0.0),
                 omega=(0.0, vx / (R * (1.0 - slip)), 0.0), motion=BODY_PRESCRIBED, markers=f32(rim + c))
    sc.bodies = [b]
    sc.name = "mgru3_wheel"
    if active:   # activated after a few full steps, so the frozen shell's markers carry extrapolated
        # values of the settled terrain (the paper waits t_delay = 1 s for its terrain to settle)
        sc.active = {"boxes": {1: (0.3, 0.3, 0.4)}, "t_delay": 2.5 * dt}
    return sc


def random_cloud(n: int, seed: int, box: float = 1.0) -> np.ndarray:
    """Uniform random cloud in [0, box)^3, fp32-representable."""
    rng = np.random.default_rng(seed)
    return f32(rng.uniform(0.0, box, (n, 3)))


def return_map_state(n=(14, 14, 14), seed=11, cohesion=500.0, mu_s=0.3, mu_2=0.6, A_scale=20.0) -> Scenario:
    """A state whose one-step trial stresses populate every branch of the return map:
    the C1 block in its walled box with cohesion c (so p_cri = -c/mu_s < 0) and mu_2 > mu_s; per
    particle a pressure p ~ U(-2500, 3000) Pa and a deviator of random direction with
    tau_bar ~ U(0, 2000) Pa (sigma = -p I + tau); velocities u = A (x - xbar), A ~ N(0, A_scale s^-1),
    so that some particles load (gamma_dot > 0, mu(I) > mu_s) and some unload.  Seeded; generators
    only (the branch logic lives in the oracle and the kernels)."""
    sc = block_settle(n=n)
    p = dict(sc.params, cohesion=cohesion, mu_s=mu_s, mu_2=mu_2)
    pos = sc.fluid_pos
    rng = np.random.default_rng(seed)
    N = pos.shape[0]
    pres = rng.uniform(-2500.0, 3000.0, N)
    D = rng.normal(0.0, 1.0, (N, 3, 3))
    D = 0.5 * (D + np.transpose(D, (0, 2, 1)))
    D -= np.trace(D, axis1=1, axis2=2)[:, None, None] * np.eye(3) / 3.0
    D /= np.sqrt(0.5 * np.einsum("kij,kij->k", D, D))[:, None, None]   # unit tau_bar
    tb = rng.uniform(0.0, 2000.0, N)
    S = -pres[:, None, None] * np.eye(3) + tb[:, None, None] * D
    sig = np.stack([S[:, 0, 0], S[:, 1, 1], S[:, 2, 2], S[:, 0, 1], S[:, 0, 2], S[:, 1, 2]], -1)
    A = rng.normal(0.0, A_scale, (3, 3))
    vel = (pos - pos.mean(0)) @ A.T
    return Scenario("return_map_state", p, pos, f32(vel), f32(sig), sc.wall_pos, [], sc.dt, 1,
                    meta=dict(sc.meta, A=A))
