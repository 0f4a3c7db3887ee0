"""In-tree build of libcrm.so for sm_100a (nvcc; no torch JIT cache involved).

Flags: -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo; never --use_fast_math
(the structural rules B1/B2 need IEEE fp32 sub/div/fma).
"""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libcrm.so")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared"]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + [os.path.join(ROOT, "include", "crm.h")])


def nccl_paths():
    """(include dir, library path) of the NCCL shipped with the environment (nvidia-nccl wheel).
    Only the header is needed to build; libnccl.so.2 is dlopen'ed at run time for world > 1."""
    try:
        import nvidia.nccl
        base = list(nvidia.nccl.__path__)[0]
        return os.path.join(base, "include"), os.path.join(base, "lib", "libnccl.so.2")
    except Exception:
        return None, None


def _fresh() -> bool:
    return os.path.exists(LIB) and os.path.getmtime(LIB) >= max(os.path.getmtime(s) for s in _sources())


def build_library(force: bool = False, verbose: bool = False) -> str:
    if not force and _fresh():
        return LIB
    # several processes (torchrun ranks) may get here at once: one builds, the others wait for it
    import fcntl
    with open(LIB + ".lock", "w") as lock:
        fcntl.flock(lock, fcntl.LOCK_EX)
        if not force and _fresh():
            return LIB
        return _build(verbose)


def _build(verbose: bool) -> str:
    nvcc = os.environ.get("NVCC", "nvcc")
    inc, lib = nccl_paths()
    if inc is None:
        raise RuntimeError("nccl.h not found (nvidia-nccl wheel)")
    tmp = f"{LIB}.{os.getpid()}.tmp"
    cmd = [nvcc, *NVCC_FLAGS, "-I", inc, f'-DCRM_NCCL_DEFAULT="{lib}"', "-o", tmp,
           os.path.join(CSRC, "crm.cu"), "-ldl"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd, cwd=ROOT)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build_library(force=True, verbose=True))
