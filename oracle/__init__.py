"""oracle — TEST INFRASTRUCTURE ONLY (not part of the product).

ctypes wrapper over liboracle.so (oracle/crm_oracle.c), the plain fp64 CPU oracle
of the Chrono::CRM per-step SPH update (arXiv 2507.05643, §2, §4.1).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this package.  It imports nothing from
paper_2507_05643_b200/ and the CUDA path imports nothing from here.

Every function of crm_oracle.c cites the passage it follows; the pins that tie
each one to the paper are in tests/test_oracle_*.py.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "crm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OC_OK, OC_E_INVALID, OC_E_DOMAIN, OC_E_NONFINITE, OC_E_UNSUPPORTED, OC_E_STATE, OC_E_OOM = 0, -1, -2, -3, -4, -5, -6


def build(force: bool = False) -> str:
    """Compile liboracle.so: -O2 -fopenmp -ffp-contract=off, no fast-math."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "crm_oracle.h"))):
        cmd = ["gcc", "-std=gnu11", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
               "-fPIC", "-shared", "-o", f"{_LIB}.{os.getpid()}.tmp", _SRC, "-lm"]
        subprocess.check_call(cmd, cwd=_HERE)
        os.replace(f"{_LIB}.{os.getpid()}.tmp", _LIB)
    return _LIB


class Params(C.Structure):
    _fields_ = [("rho0", C.c_double), ("K", C.c_double), ("G", C.c_double), ("mu_s", C.c_double),
                ("mu_2", C.c_double), ("I0", C.c_double), ("cohesion", C.c_double),
                ("grain_d", C.c_double), ("d0", C.c_double), ("h", C.c_double),
                ("support", C.c_double), ("visc_mode", C.c_int), ("gamma_a", C.c_double),
                ("xi2", C.c_double), ("cs", C.c_double), ("gravity", C.c_double * 3),
                ("lo", C.c_double * 3), ("hi", C.c_double * 3), ("ps_freq", C.c_int),
                ("kernel", C.c_int)]


class BodyS(C.Structure):
    _fields_ = [("mass", C.c_double), ("inertia", C.c_double * 3), ("pos", C.c_double * 3),
                ("quat", C.c_double * 4), ("vel", C.c_double * 3), ("omega", C.c_double * 3),
                ("motion", C.c_int), ("dof_mask", C.c_int)]


_lib = None
_D = C.POINTER(C.c_double)
_F = C.POINTER(C.c_float)
_I64 = C.POINTER(C.c_int64)
_U32 = C.POINTER(C.c_uint32)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        L.oc_W.restype = C.c_double; L.oc_W.argtypes = [C.c_double, C.c_double]
        L.oc_dWdr.restype = C.c_double; L.oc_dWdr.argtypes = [C.c_double, C.c_double]
        L.oc_gradW.argtypes = [_D, C.c_double, _D]
        L.oc_W_wendland.restype = C.c_double; L.oc_W_wendland.argtypes = [C.c_double, C.c_double]
        L.oc_dWdr_wendland.restype = C.c_double; L.oc_dWdr_wendland.argtypes = [C.c_double, C.c_double]
        L.oc_paper_cell_index.restype = C.c_int64
        L.oc_paper_cell_index.argtypes = [C.c_int64] * 5
        L.oc_cell_coords.argtypes = [_F, _F, C.c_float, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.oc_pair_predicate.argtypes = [_F, _F, C.c_float]
        L.oc_brute_neighbors.argtypes = [C.c_int64, _F, C.c_double, _I64, _I64]
        L.oc_stress_rate.argtypes = [_D, _D, C.c_double, C.c_double, _D]
        L.oc_return_map.argtypes = [_D, _D, C.POINTER(Params), C.c_double, _D]
        L.oc_create.argtypes = [C.POINTER(Params), C.POINTER(C.c_void_p)]
        L.oc_destroy.argtypes = [C.c_void_p]
        L.oc_add_fluid.argtypes = [C.c_void_p, C.c_int64, _D, _D, _D, _I64]
        L.oc_add_body.argtypes = [C.c_void_p, C.POINTER(BodyS), C.POINTER(C.c_int32)]
        L.oc_add_bce.argtypes = [C.c_void_p, C.c_int32, C.c_int64, _D, _I64]
        L.oc_step.argtypes = [C.c_void_p, C.c_double, C.c_int64]
        L.oc_count.restype = C.c_int64; L.oc_count.argtypes = [C.c_void_p, C.c_int]
        L.oc_get_state.argtypes = [C.c_void_p, C.c_int64, C.c_int64, _D, _D, _D, _D]
        L.oc_set_state.argtypes = [C.c_void_p, C.c_int64, C.c_int64, _D, _D, _D, _D]
        L.oc_get_body.argtypes = [C.c_void_p, C.c_int32, C.POINTER(BodyS), _D, _D]
        L.oc_structure.argtypes = [C.c_void_p, _U32, _I64, _U32, _U32, _I64]
        L.oc_neighbors.argtypes = [C.c_void_p, _I64, _I64]
        L.oc_last_rates.argtypes = [C.c_void_p, C.c_int, _D, _D, _D]
        L.oc_last_bce.argtypes = [C.c_void_p, C.c_int, _D, _D]
        L.oc_last_error.restype = C.c_char_p; L.oc_last_error.argtypes = [C.c_void_p]
        L.oc_num_threads.restype = C.c_int
        L.oc_set_num_threads.argtypes = [C.c_int]; L.oc_set_num_threads.restype = None
        L.oc_activity.restype = C.c_int
        L.oc_activity.argtypes = [_D, C.c_int, _D, _D, _D, C.c_double]
        L.oc_manage_capacity.restype = C.c_int64
        L.oc_manage_capacity.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_int,
                                         C.POINTER(C.c_int)]
        L.oc_set_active_box.argtypes = [C.c_void_p, C.c_int32, _D]
        L.oc_set_active_delay.argtypes = [C.c_void_p, C.c_double]
        L.oc_get_activity.argtypes = [C.c_void_p, C.POINTER(C.c_uint8)]
        _lib = L
    return _lib


def _p(a, t=_D):
    return None if a is None else a.ctypes.data_as(t)


def _d(a, shape=None):
    if a is None:
        return None
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a if shape is None else a.reshape(shape)


class OracleError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


# ---------------- pure functions ----------------
def W(r: float, h: float) -> float:
    return lib().oc_W(float(r), float(h))


def dWdr(r: float, h: float) -> float:
    return lib().oc_dWdr(float(r), float(h))


def W_wendland(r: float, h: float) -> float:
    return lib().oc_W_wendland(float(r), float(h))


def dWdr_wendland(r: float, h: float) -> float:
    return lib().oc_dWdr_wendland(float(r), float(h))


def gradW(xij, h: float) -> np.ndarray:
    x = _d(xij, (3,)); out = np.zeros(3)
    lib().oc_gradW(_p(x), float(h), _p(out))
    return out


def paper_cell_index(x, y, z, X, Y) -> int:
    return lib().oc_paper_cell_index(x, y, z, X, Y)


def cell_coords(x, lo, s, dims):
    xf = np.ascontiguousarray(x, np.float32); lf = np.ascontiguousarray(lo, np.float32)
    d = (C.c_int * 3)(*dims); out = (C.c_int * 3)()
    rc = lib().oc_cell_coords(_p(xf, _F), _p(lf, _F), C.c_float(s), d, out)
    return rc, tuple(out)


def brute_neighbors(x32: np.ndarray, radius: float):
    """Per-particle sorted neighbour index arrays, O(N^2) definition."""
    x = np.ascontiguousarray(x32, np.float32).reshape(-1, 3)
    n = x.shape[0]
    off = np.zeros(n + 1, np.int64)
    lib().oc_brute_neighbors(n, _p(x, _F), float(radius), _p(off, _I64), None)
    lst = np.zeros(max(1, off[-1]), np.int64)
    lib().oc_brute_neighbors(n, _p(x, _F), float(radius), _p(off, _I64), _p(lst, _I64))
    return off, lst[: off[-1]]


def stress_rate(L, sig, K, G) -> np.ndarray:
    Lm = _d(L, (9,)); s = _d(sig, (6,)); out = np.zeros(6)
    lib().oc_stress_rate(_p(Lm), _p(s), float(K), float(G), _p(out))
    return out


def make_params(p: dict) -> Params:
    P = Params()
    for k in ("rho0", "K", "G", "mu_s", "mu_2", "I0", "cohesion", "grain_d", "d0", "h",
              "support", "gamma_a", "xi2", "cs"):
        setattr(P, k, float(p.get(k, 0.0)))
    P.visc_mode = int(p.get("visc_mode", 0))
    P.ps_freq = int(p.get("ps_freq", 1))
    P.kernel = int(p.get("kernel", 0))
    for k in ("gravity", "lo", "hi"):
        v = p.get(k, (0.0, 0.0, 0.0))
        setattr(P, k, (C.c_double * 3)(*[float(t) for t in v]))
    return P


def return_map(sig_star, sig_n, params: dict, dt: float) -> np.ndarray:
    P = make_params(params)
    a = _d(sig_star, (6,)); b = _d(sig_n, (6,)); out = np.zeros(6)
    lib().oc_return_map(_p(a), _p(b), C.byref(P), float(dt), _p(out))
    return out


def num_threads() -> int:
    return lib().oc_num_threads()


def set_num_threads(n: int) -> None:
    lib().oc_set_num_threads(int(n))


# ---------------- simulation ----------------
class OracleSim:
    """Same call shape as the product's crm_* ABI, on liboracle.so."""

    def __init__(self, params: dict):
        self._L = lib()
        self._P = make_params(params)
        h = C.c_void_p()
        rc = self._L.oc_create(C.byref(self._P), C.byref(h))
        if rc:
            raise OracleError(rc, "oc_create")
        self.h = h

    def close(self):
        if self.h:
            self._L.oc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, rc, what):
        if rc:
            raise OracleError(rc, f"{what}: {self._L.oc_last_error(self.h).decode()}")

    def add_fluid(self, pos, vel=None, sig6=None) -> int:
        pos = _d(pos, (-1, 3)); n = pos.shape[0]
        vel = _d(vel, (n, 3)); sig6 = _d(sig6, (n, 6))
        fid = C.c_int64()
        self._chk(self._L.oc_add_fluid(self.h, n, _p(pos), _p(vel), _p(sig6), C.byref(fid)), "add_fluid")
        return fid.value

    def add_body(self, body) -> int:
        b = BodyS()
        b.mass = body.mass
        b.inertia = (C.c_double * 3)(*body.inertia); b.pos = (C.c_double * 3)(*body.pos)
        b.quat = (C.c_double * 4)(*body.quat); b.vel = (C.c_double * 3)(*body.vel)
        b.omega = (C.c_double * 3)(*body.omega); b.motion = body.motion; b.dof_mask = body.dof_mask
        bid = C.c_int32()
        self._chk(self._L.oc_add_body(self.h, C.byref(b), C.byref(bid)), "add_body")
        return bid.value

    def add_bce(self, body: int, pos) -> int:
        pos = _d(pos, (-1, 3))
        fid = C.c_int64()
        self._chk(self._L.oc_add_bce(self.h, body, pos.shape[0], _p(pos), C.byref(fid)), "add_bce")
        return fid.value

    def step(self, dt: float, n: int = 1):
        self._chk(self._L.oc_step(self.h, float(dt), int(n)), "step")

    def count(self, which: int = 2) -> int:
        return self._L.oc_count(self.h, which)

    def get_state(self, first=0, count=None):
        n = self.count() - first if count is None else count
        pos = np.zeros((n, 3)); vel = np.zeros((n, 3)); rho = np.zeros(n); sig = np.zeros((n, 6))
        self._chk(self._L.oc_get_state(self.h, first, n, _p(pos), _p(vel), _p(rho), _p(sig)), "get_state")
        return pos, vel, rho, sig

    def set_state(self, first, pos=None, vel=None, rho=None, sig6=None):
        arrs = [a for a in (pos, vel, rho, sig6) if a is not None]
        n = np.asarray(arrs[0]).shape[0]
        pos = _d(pos, (n, 3)); vel = _d(vel, (n, 3)); rho = _d(rho, (n,)); sig6 = _d(sig6, (n, 6))
        self._chk(self._L.oc_set_state(self.h, first, n, _p(pos), _p(vel), _p(rho), _p(sig6)), "set_state")

    def get_body(self, body: int):
        b = BodyS(); F = np.zeros(3); T = np.zeros(3)
        self._chk(self._L.oc_get_body(self.h, body, C.byref(b), _p(F), _p(T)), "get_body")
        return dict(pos=np.array(b.pos[:]), vel=np.array(b.vel[:]), quat=np.array(b.quat[:]),
                    omega=np.array(b.omega[:]), force=F, torque=T)

    def structure(self):
        n = self.count()
        cell = np.zeros(n, np.uint32); srt = np.zeros(n, np.int64); cnt = np.zeros(n, np.uint32)
        M = C.c_int64()
        self._chk(self._L.oc_structure(self.h, None, None, None, None, C.byref(M)), "structure")
        cs = np.zeros(M.value + 1, np.uint32)
        self._chk(self._L.oc_structure(self.h, _p(cell, _U32), _p(srt, _I64), _p(cnt, _U32),
                                       _p(cs, _U32), C.byref(M)), "structure")
        return dict(cell=cell, sorted_ids=srt, counts=cnt, cell_start=cs)

    def neighbors(self):
        n = self.count()
        off = np.zeros(n + 1, np.int64)
        self._chk(self._L.oc_neighbors(self.h, _p(off, _I64), None), "neighbors")
        lst = np.zeros(max(1, off[-1]), np.int64)
        self._chk(self._L.oc_neighbors(self.h, _p(off, _I64), _p(lst, _I64)), "neighbors")
        return off, lst[: off[-1]]

    def last_rates(self, stage: int):
        n = self.count()
        drho = np.zeros(n); acc = np.zeros((n, 3)); ds = np.zeros((n, 6))
        self._chk(self._L.oc_last_rates(self.h, stage, _p(drho), _p(acc), _p(ds)), "last_rates")
        return drho, acc, ds

    def last_bce(self, stage: int):
        n = self.count()
        vel = np.zeros((n, 3)); sig = np.zeros((n, 6))
        self._chk(self._L.oc_last_bce(self.h, stage, _p(vel), _p(sig)), "last_bce")
        return vel, sig

    # ---- active domains (Alg. 3)
    def set_active_box(self, body: int, half):
        h = _d(half, (3,))
        self._chk(self._L.oc_set_active_box(self.h, int(body), _p(h)), "set_active_box")

    def set_active_delay(self, t_delay: float):
        self._chk(self._L.oc_set_active_delay(self.h, float(t_delay)), "set_active_delay")

    def activity(self) -> np.ndarray:
        f = np.zeros(self.count(), np.uint8)
        self._chk(self._L.oc_get_activity(self.h, f.ctypes.data_as(C.POINTER(C.c_uint8))), "activity")
        return f


def activity(x, boxes, radius: float) -> int:
    """UpdateActivity of one point; boxes = [(pos[3], R[3x3] body->world, half[3]), ...]."""
    nb = len(boxes)
    bp = np.zeros(3 * nb + 1); bR = np.zeros(9 * nb + 1); bh = np.zeros(3 * nb + 1)
    for k, (pos, R, half) in enumerate(boxes):
        bp[3 * k:3 * k + 3] = pos
        bR[9 * k:9 * k + 9] = np.asarray(R, float).ravel()
        bh[3 * k:3 * k + 3] = half
    xx = _d(x, (3,))
    return lib().oc_activity(_p(xx), nb, _p(bp), _p(bR), _p(bh), float(radius))


def manage_capacity(capacity: int, required: int, step: int, growth=1.2, shrink=0.75, interval=50):
    a = C.c_int(0)
    cap = lib().oc_manage_capacity(int(capacity), int(required), int(step), float(growth), float(shrink),
                                   int(interval), C.byref(a))
    return int(cap), int(a.value)


def load_scenario(sc) -> OracleSim:
    """Build an OracleSim from a workloads.Scenario (fluid first, then walls, then bodies)."""
    s = OracleSim(sc.params)
    s.add_fluid(sc.fluid_pos, sc.fluid_vel, sc.fluid_sig)
    if sc.wall_pos.shape[0]:
        s.add_bce(0, sc.wall_pos)
    for b in sc.bodies:
        bid = s.add_body(b)
        if b.markers.shape[0]:
            s.add_bce(bid, b.markers)
    act = getattr(sc, "active", None) or {}
    for body, half in act.get("boxes", {}).items():
        s.set_active_box(body, half)
    if "t_delay" in act:
        s.set_active_delay(act["t_delay"])
    return s
