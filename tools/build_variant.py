"""Build an experimental libcrm variant with extra -D flags: python tools/build_variant.py NAME -DX=1 ...
(load it with CRM_LIB=build/variants/NAME.so)"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_05643_b200 import build as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(b.ROOT, "build", "variants", name + ".so")
os.makedirs(os.path.dirname(out), exist_ok=True)
inc, lib = b.nccl_paths()
cmd = ["nvcc", *b.NVCC_FLAGS, *defs, "-I", inc, f'-DCRM_NCCL_DEFAULT="{lib}"', "-o", out,
       os.path.join(b.CSRC, "crm.cu"), "-ldl"]
subprocess.check_call(cmd, cwd=b.ROOT)
print(out)
