"""Thin ctypes binding of include/crm.h (libcrm.so): argument marshalling only.

Every step of the particle update runs in the CUDA kernels of libcrm.so; this module
converts numpy arrays to pointers and return codes to exceptions.  There is no CPU
fallback: if libcrm.so is missing or no sm_100 device is visible the calls raise.
"""
from __future__ import annotations

import ctypes as C
import weakref
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CRM_LIB") or os.path.join(_HERE, "libcrm.so")

CRM_OK, CRM_E_INVALID, CRM_E_DOMAIN, CRM_E_NONFINITE, CRM_E_UNSUPPORTED = 0, -1, -2, -3, -4
CRM_E_STATE, CRM_E_OOM, CRM_E_CUDA, CRM_E_COMM, CRM_E_CAPACITY = -5, -6, -7, -8, -9
CRM_FLUID, CRM_BCE, CRM_ALL, CRM_OWNED, CRM_GRAPH_REPLAYS = 0, 1, 2, 3, 4

# every symbol include/crm.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "crm_create", "crm_destroy", "crm_add_fluid", "crm_add_body", "crm_add_bce", "crm_step",
    "crm_get_state", "crm_set_state", "crm_get_body", "crm_count", "crm_last_error", "crm_strerror",
    "crm_stream", "crm_launch_count", "crm_profile_enable", "crm_profile_read", "crm_profile_reset",
    "crm_kernel_name", "crm_set_graphs", "crm_debug_arm", "crm_debug_structure", "crm_debug_neighbors",
    "crm_debug_rates", "crm_debug_bce", "crm_group_step", "crm_nccl_unique_id", "crm_slab_partition",
    "crm_pair_count", "crm_candidate_count", "crm_set_active_box", "crm_set_active_policy", "crm_active_stats", "crm_manage_capacity",
    "crm_debug_activity",
]


class Material(C.Structure):
    _fields_ = [("rho0", C.c_double), ("K", C.c_double), ("G", C.c_double), ("mu_s", C.c_double),
                ("mu_2", C.c_double), ("I0", C.c_double), ("cohesion", C.c_double), ("grain_d", C.c_double)]


class Kernel(C.Structure):
    _fields_ = [("kernel", C.c_int), ("d0", C.c_double), ("h", C.c_double), ("support", C.c_double),
                ("visc_mode", C.c_int), ("gamma_a", C.c_double), ("xi2", C.c_double), ("cs", C.c_double),
                ("ps_freq", C.c_int), ("gravity", C.c_double * 3), ("max_neighbors", C.c_int)]


class Boundary(C.Structure):
    _fields_ = [("method", C.c_int), ("n_layers", C.c_int), ("lo", C.c_double * 3), ("hi", C.c_double * 3),
                ("slab_axis", C.c_int)]


class Dist(C.Structure):
    _fields_ = [("rank", C.c_int), ("world", C.c_int), ("device", C.c_int), ("nccl_id", C.c_void_p),
                ("cuda_stream", C.c_void_p)]


class ActiveT(C.Structure):
    _fields_ = [("t_delay", C.c_double), ("growth", C.c_double), ("shrink", C.c_double),
                ("shrink_interval", C.c_int)]


class BodyT(C.Structure):
    _fields_ = [("mass", C.c_double), ("inertia", C.c_double * 3), ("pos", C.c_double * 3),
                ("quat", C.c_double * 4), ("vel", C.c_double * 3), ("omega", C.c_double * 3),
                ("motion", C.c_int), ("dof_mask", C.c_int)]


_D = C.POINTER(C.c_double)
_I64 = C.POINTER(C.c_int64)
_U32 = C.POINTER(C.c_uint32)
_lib = None


def load_library(path: str = LIB_PATH):
    """Load libcrm.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"libcrm.so not found at {path}; run __graft_entry__.build()")
    L = C.CDLL(path)
    vp = C.c_void_p
    L.crm_create.argtypes = [C.POINTER(Material), C.POINTER(Kernel), C.POINTER(Boundary), C.POINTER(Dist),
                             C.POINTER(vp)]
    L.crm_destroy.argtypes = [vp]; L.crm_destroy.restype = None
    L.crm_add_fluid.argtypes = [vp, C.c_int64, _D, _D, _D, _I64]
    L.crm_add_body.argtypes = [vp, C.POINTER(BodyT), C.POINTER(C.c_int32)]
    L.crm_add_bce.argtypes = [vp, C.c_int32, C.c_int64, _D, _I64]
    L.crm_step.argtypes = [vp, C.c_double, C.c_int64]
    L.crm_get_state.argtypes = [vp, C.c_int64, C.c_int64, _D, _D, _D, _D]
    L.crm_set_state.argtypes = [vp, C.c_int64, C.c_int64, _D, _D, _D, _D]
    L.crm_get_body.argtypes = [vp, C.c_int32, C.POINTER(BodyT), _D, _D]
    L.crm_count.argtypes = [vp, C.c_int]; L.crm_count.restype = C.c_int64
    L.crm_last_error.argtypes = [vp]; L.crm_last_error.restype = C.c_char_p
    L.crm_strerror.argtypes = [C.c_int]; L.crm_strerror.restype = C.c_char_p
    L.crm_stream.argtypes = [vp]; L.crm_stream.restype = vp
    L.crm_launch_count.argtypes = [vp]; L.crm_launch_count.restype = C.c_int64
    L.crm_profile_enable.argtypes = [vp, C.c_int]
    L.crm_profile_read.argtypes = [vp, C.c_int, _D, _I64]
    L.crm_profile_reset.argtypes = [vp]
    L.crm_kernel_name.argtypes = [C.c_int]; L.crm_kernel_name.restype = C.c_char_p
    L.crm_set_graphs.argtypes = [vp, C.c_int]
    L.crm_debug_arm.argtypes = [vp, C.c_int]
    L.crm_debug_structure.argtypes = [vp, _U32, _I64, _U32, _U32, _I64]
    L.crm_debug_neighbors.argtypes = [vp, _I64, _I64]
    L.crm_debug_rates.argtypes = [vp, C.c_int, _D, _D, _D]
    L.crm_debug_bce.argtypes = [vp, C.c_int, _D, _D]
    L.crm_group_step.argtypes = [C.POINTER(vp), C.c_int, C.c_double, C.c_int64]
    L.crm_nccl_unique_id.argtypes = [C.c_void_p]
    L.crm_slab_partition.argtypes = [_I64, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int)]
    L.crm_pair_count.argtypes = [vp, _I64]
    L.crm_candidate_count.argtypes = [vp, _I64, _I64]
    L.crm_set_active_box.argtypes = [vp, C.c_int32, _D]
    L.crm_set_active_policy.argtypes = [vp, C.POINTER(ActiveT)]
    L.crm_active_stats.argtypes = [vp, _I64]
    L.crm_manage_capacity.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_int,
                                      C.POINTER(C.c_int)]
    L.crm_manage_capacity.restype = C.c_int64
    L.crm_debug_activity.argtypes = [vp, C.POINTER(C.c_uint8)]
    _lib = L
    return L


def manage_capacity(capacity: int, required: int, step: int, growth=1.2, shrink=0.75, interval=50):
    """ManageArrayMemory policy of Alg. 3 (host function of libcrm.so): (new capacity, action)."""
    a = C.c_int(0)
    cap = load_library().crm_manage_capacity(int(capacity), int(required), int(step), float(growth),
                                             float(shrink), int(interval), C.byref(a))
    return int(cap), int(a.value)


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId (rank 0 creates it, torch.distributed broadcasts it)."""
    buf = C.create_string_buffer(128)
    rc = load_library().crm_nccl_unique_id(buf)
    if rc:
        raise CrmError(rc, "crm_nccl_unique_id")
    return buf.raw


def slab_partition(plane_counts, world: int, align: int = 2) -> np.ndarray:
    """Slab boundaries (world + 1 plane indices) balancing per-plane counts (host only)."""
    pc = np.ascontiguousarray(plane_counts, dtype=np.int64)
    out = (C.c_int * (world + 1))()
    rc = load_library().crm_slab_partition(pc.ctypes.data_as(_I64), len(pc), world, align, out)
    if rc:
        raise CrmError(rc, "crm_slab_partition")
    return np.array(out[:], dtype=np.int64)


def group_step(ctxs, dt: float, n: int = 1):
    """Step in-process slab contexts (ranks 0..W-1 on one device/stream) with loopback halos."""
    arr = (C.c_void_p * len(ctxs))(*[c.h.value for c in ctxs])
    rc = load_library().crm_group_step(arr, len(ctxs), float(dt), int(n))
    if rc:
        msgs = "; ".join(c._L.crm_last_error(c.h).decode() for c in ctxs)
        raise CrmError(rc, f"crm_group_step: {msgs}")


# library stream handle -> the Crm that created it (weak: borrowers hold strong references)
_STREAM_OWNERS: "weakref.WeakValueDictionary[int, Crm]" = weakref.WeakValueDictionary()


class CrmError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"crm error {code}: {msg}")
        self.code = code


def _p(a, t=_D):
    return None if a is None else a.ctypes.data_as(t)


def _d(a, shape):
    if a is None:
        return None
    return np.ascontiguousarray(a, dtype=np.float64).reshape(shape)


def kernel_names() -> list[str]:
    L = load_library()
    out = []
    k = 0
    while True:
        nm = L.crm_kernel_name(k)
        if nm is None:
            return out
        out.append(nm.decode())
        k += 1


class Crm:
    """One simulation context on one GPU (crm_create ... crm_destroy)."""

    def __init__(self, params: dict, *, device: int = 0, stream: int | None = None, max_neighbors: int = 0,
                 rank: int = 0, world: int = 1, nccl_id: bytes | None = None):
        self._L = load_library()
        m = Material(params["rho0"], params["K"], params["G"], params["mu_s"], params["mu_2"], params["I0"],
                     params["cohesion"], params["grain_d"])
        k = Kernel()
        k.kernel = int(params.get("kernel", 0))
        k.d0 = params["d0"]; k.h = params["h"]; k.support = params.get("support", 2.0)
        k.visc_mode = int(params["visc_mode"]); k.gamma_a = params["gamma_a"]
        k.xi2 = params.get("xi2", 0.0); k.cs = params.get("cs", 0.0); k.ps_freq = int(params.get("ps_freq", 1))
        k.gravity = (C.c_double * 3)(*params["gravity"])
        k.max_neighbors = int(max_neighbors)
        b = Boundary()
        b.method = 0; b.n_layers = 0
        b.lo = (C.c_double * 3)(*params["lo"]); b.hi = (C.c_double * 3)(*params["hi"]); b.slab_axis = 0
        self._nccl_id = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        d = Dist(rank, world, device, C.cast(self._nccl_id, C.c_void_p) if self._nccl_id is not None else None, stream)
        h = C.c_void_p()
        rc = self._L.crm_create(C.byref(m), C.byref(k), C.byref(b), C.byref(d), C.byref(h))
        if rc:
            raise CrmError(rc, self._L.crm_strerror(rc).decode())
        self.h = h
        # a context on another context's stream keeps that context (and its stream) alive
        self._stream_owner = _STREAM_OWNERS.get(int(stream)) if stream else None
        if not stream:
            _STREAM_OWNERS[int(self.stream())] = self

    def close(self):
        if getattr(self, "h", None):
            sid = int(self.stream())
            if _STREAM_OWNERS.get(sid) is self:
                del _STREAM_OWNERS[sid]
            self._L.crm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, rc: int, what: str):
        if rc:
            raise CrmError(rc, f"{what}: {self._L.crm_last_error(self.h).decode()}")

    # ---- problem setup ----
    def add_fluid(self, pos, vel=None, sig6=None) -> int:
        pos = _d(pos, (-1, 3)); n = pos.shape[0]
        vel = _d(vel, (n, 3)); sig6 = _d(sig6, (n, 6))
        fid = C.c_int64()
        self._chk(self._L.crm_add_fluid(self.h, n, _p(pos), _p(vel), _p(sig6), C.byref(fid)), "crm_add_fluid")
        return fid.value

    def add_body(self, body) -> int:
        b = BodyT()
        b.mass = body.mass
        b.inertia = (C.c_double * 3)(*body.inertia); b.pos = (C.c_double * 3)(*body.pos)
        b.quat = (C.c_double * 4)(*body.quat); b.vel = (C.c_double * 3)(*body.vel)
        b.omega = (C.c_double * 3)(*body.omega); b.motion = body.motion; b.dof_mask = body.dof_mask
        bid = C.c_int32()
        self._chk(self._L.crm_add_body(self.h, C.byref(b), C.byref(bid)), "crm_add_body")
        return bid.value

    def add_bce(self, body: int, pos) -> int:
        pos = _d(pos, (-1, 3))
        fid = C.c_int64()
        self._chk(self._L.crm_add_bce(self.h, body, pos.shape[0], _p(pos), C.byref(fid)), "crm_add_bce")
        return fid.value

    # ---- stepping and state ----
    def step(self, dt: float, n: int = 1):
        self._chk(self._L.crm_step(self.h, float(dt), int(n)), "crm_step")

    def count(self, which: int = CRM_ALL) -> int:
        return self._L.crm_count(self.h, which)

    def get_state(self, first: int = 0, count: int | None = None, out=None):
        n = self.count() - first if count is None else count
        if out is None:
            out = (np.zeros((n, 3)), np.zeros((n, 3)), np.zeros(n), np.zeros((n, 6)))
        pos, vel, rho, sig = out
        self._chk(self._L.crm_get_state(self.h, first, n, _p(pos), _p(vel), _p(rho), _p(sig)), "crm_get_state")
        return pos, vel, rho, sig

    def set_state(self, first: int, pos=None, vel=None, rho=None, sig6=None):
        arrs = [a for a in (pos, vel, rho, sig6) if a is not None]
        n = np.asarray(arrs[0]).shape[0]
        pos = _d(pos, (n, 3)); vel = _d(vel, (n, 3)); rho = _d(rho, (n,)); sig6 = _d(sig6, (n, 6))
        self._chk(self._L.crm_set_state(self.h, first, n, _p(pos), _p(vel), _p(rho), _p(sig6)), "crm_set_state")

    def get_body(self, body: int) -> dict:
        b = BodyT(); F = np.zeros(3); T = np.zeros(3)
        self._chk(self._L.crm_get_body(self.h, body, C.byref(b), _p(F), _p(T)), "crm_get_body")
        return dict(pos=np.array(b.pos[:]), vel=np.array(b.vel[:]), quat=np.array(b.quat[:]),
                    omega=np.array(b.omega[:]), force=F, torque=T)

    # ---- measurement ----
    def stream(self) -> int:
        return self._L.crm_stream(self.h)

    def launch_count(self) -> int:
        return self._L.crm_launch_count(self.h)

    def profile(self, on: bool = True):
        self._chk(self._L.crm_profile_enable(self.h, 1 if on else 0), "crm_profile_enable")

    def profile_reset(self):
        self._chk(self._L.crm_profile_reset(self.h), "crm_profile_reset")

    def profile_read(self) -> dict:
        out = {}
        for k, nm in enumerate(kernel_names()):
            ms = C.c_double(); nl = C.c_int64()
            self._chk(self._L.crm_profile_read(self.h, k, C.byref(ms), C.byref(nl)), "crm_profile_read")
            if nl.value:
                out[nm] = (ms.value, nl.value)
        return out

    def pair_count(self) -> int:
        v = C.c_int64()
        self._chk(self._L.crm_pair_count(self.h, C.byref(v)), "crm_pair_count")
        return v.value

    def candidate_count(self) -> tuple[int, int]:
        """Alg. 1 candidates (fluid, markers) of the last structure."""
        f, b = C.c_int64(), C.c_int64()
        self._chk(self._L.crm_candidate_count(self.h, C.byref(f), C.byref(b)), "crm_candidate_count")
        return f.value, b.value

    def set_graphs(self, on: bool):
        self._chk(self._L.crm_set_graphs(self.h, 1 if on else 0), "crm_set_graphs")

    # ---- debug exports ----
    def debug_arm(self, on: bool = True):
        self._chk(self._L.crm_debug_arm(self.h, 1 if on else 0), "crm_debug_arm")

    def structure(self) -> dict:
        n = self.count()
        M = C.c_int64()
        self._chk(self._L.crm_debug_structure(self.h, None, None, None, None, C.byref(M)), "crm_debug_structure")
        cell = np.zeros(n, np.uint32); srt = np.zeros(n, np.int64); cnt = np.zeros(n, np.uint32)
        cs = np.zeros(M.value + 1, np.uint32)
        self._chk(self._L.crm_debug_structure(self.h, _p(cell, _U32), _p(srt, _I64), _p(cnt, _U32), _p(cs, _U32),
                                              C.byref(M)), "crm_debug_structure")
        return dict(cell=cell, sorted_ids=srt, counts=cnt, cell_start=cs)

    def neighbors(self):
        n = self.count()
        off = np.zeros(n + 1, np.int64)
        self._chk(self._L.crm_debug_neighbors(self.h, _p(off, _I64), None), "crm_debug_neighbors")
        lst = np.zeros(max(1, int(off[-1])), np.int64)
        self._chk(self._L.crm_debug_neighbors(self.h, _p(off, _I64), _p(lst, _I64)), "crm_debug_neighbors")
        return off, lst[: off[-1]]

    def last_rates(self, stage: int):
        n = self.count()
        drho = np.zeros(n); acc = np.zeros((n, 3)); ds = np.zeros((n, 6))
        self._chk(self._L.crm_debug_rates(self.h, stage, _p(drho), _p(acc), _p(ds)), "crm_debug_rates")
        return drho, acc, ds

    def last_bce(self, stage: int):
        n = self.count()
        vel = np.zeros((n, 3)); sig = np.zeros((n, 6))
        self._chk(self._L.crm_debug_bce(self.h, stage, _p(vel), _p(sig)), "crm_debug_bce")
        return vel, sig

    # ---- active domains (Alg. 3)
    def set_active_box(self, body: int, half):
        h = _d(half, (3,))
        self._chk(self._L.crm_set_active_box(self.h, int(body), _p(h)), "crm_set_active_box")

    def set_active_policy(self, t_delay: float = 0.0, growth: float = 0.0, shrink: float = 0.0,
                          interval: int = 0):
        a = ActiveT(float(t_delay), float(growth), float(shrink), int(interval))
        self._chk(self._L.crm_set_active_policy(self.h, C.byref(a)), "crm_set_active_policy")

    def active_stats(self) -> dict:
        out = np.zeros(6, np.int64)
        self._chk(self._L.crm_active_stats(self.h, _p(out, _I64)), "crm_active_stats")
        keys = ("active", "extended", "inactive", "n_ae", "capacity", "action")
        return {k: int(v) for k, v in zip(keys, out)}

    def activity(self) -> np.ndarray:
        f = np.zeros(self.count(), np.uint8)
        self._chk(self._L.crm_debug_activity(self.h, f.ctypes.data_as(C.POINTER(C.c_uint8))), "crm_debug_activity")
        return f


def load_scenario(sc, **kw) -> Crm:
    """Build a Crm from a workloads.Scenario: fluid first, then walls (body 0), then bodies."""
    s = Crm(sc.params, **kw)
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
    if "t_delay" in act or "policy" in act:
        s.set_active_policy(act.get("t_delay", 0.0), *act.get("policy", ()))
    return s
