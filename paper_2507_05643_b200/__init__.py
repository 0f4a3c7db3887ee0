"""paper_2507_05643_b200 — B200-native CRM SPH particle update (arXiv 2507.05643).

The product is libcrm.so (include/crm.h): hand-written sm_100a CUDA kernels behind a
C-ABI.  `crm` is the thin ctypes binding with the same call names; `build` compiles the
library in-tree with nvcc for sm_100a.
"""
from . import build as _build
from .crm import Crm, CrmError, load_library, load_scenario  # noqa: F401

build_library = _build.build_library
