"""Multi-GPU plumbing around the C-ABI (torch.distributed is used only for bootstrap and for
host-side gathers; every halo exchange runs inside libcrm.so over NCCL).

  * bootstrap_nccl_id(): rank 0 creates the ncclUniqueId (crm_nccl_unique_id) and broadcasts
    it through the default torch.distributed process group (gloo or NCCL);
  * plane_counts(): per-x-plane particle counts of the global input, binned with rule B1
    (fp32 sub + div + floor), i.e. exactly what the library uses to cut the slabs;
  * merge_owned(): combine per-rank crm_get_state outputs (non-owned rows are NaN).
"""
from __future__ import annotations

import numpy as np

from . import crm as _crm


def bootstrap_nccl_id(rank: int) -> bytes:
    import torch.distributed as dist
    obj = [_crm.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def plane_counts(positions: np.ndarray, lo_x: float, cell: float, nplanes: int) -> np.ndarray:
    x = np.asarray(positions, dtype=np.float64)[:, 0].astype(np.float32)
    p = np.floor((x - np.float32(lo_x)) / np.float32(cell)).astype(np.int64)
    if p.size and (p.min() < 0 or p.max() >= nplanes):
        raise ValueError("particle outside the grid box")
    return np.bincount(p, minlength=nplanes)


def grid_planes(params: dict) -> tuple[float, float, int]:
    """(lo_x, cell size, number of x planes) of the fixed grid (B1, B3)."""
    cell = 2.0 * params["h"]
    n = int(np.ceil((params["hi"][0] - params["lo"][0]) / cell))
    return float(params["lo"][0]), cell, n


def merge_owned(states):
    """Merge per-rank (pos, vel, rho, sig) tuples whose non-owned rows are NaN."""
    out = [np.full_like(a, np.nan) for a in states[0]]
    for st in states:
        own = ~np.isnan(st[2])
        for o, a in zip(out, st):
            o[own] = a[own]
    return out
