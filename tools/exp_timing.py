"""Timing experiment (CRM_EXP_TIMING build): per-CTA phase clocks of k_rates_t<1> on a bed.
CRM_LIB=build/variants/tim.so python tools/exp_timing.py [config]"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2507_05643_b200 import crm  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "bed256x256x64"
sc = bench.scenario(cfg)
g = crm.load_scenario(sc)
g.step(sc.dt, 2)
lib = crm.load_library()
lib.crm_exp_timing_reset()
g.step(sc.dt, 1)
buf = (ctypes.c_ulonglong * (8192 * 6))()
lib.crm_exp_timing(buf, 8192 * 6)
T = np.frombuffer(buf, dtype=np.uint64).reshape(8192, 6).astype(np.int64)
T = T[(T[:, 0] > 0) & (T[:, 5] > 0) & (T[:, 4] > 0)]
d = np.diff(T, axis=1)
names = ["setup", "marker/bookkeeping+or", "lo loads+stage wait", "relativize", "pair loops+epilogue"]
tot = (T[:, 5] - T[:, 0]).astype(float)
print(f"{len(T)} CTAs, mean lifetime {tot.mean():.0f} cycles (median {np.median(tot):.0f})")
for k, n in enumerate(names):
    print(f"  {n:24s} mean {d[:, k].mean():8.0f}  median {np.median(d[:, k]):8.0f}  share {d[:, k].sum() / tot.sum():6.1%}")
