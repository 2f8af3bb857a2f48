"""paper_1905_00661_b200 — B200-native device side of Speculative HeTM.

The product is libhetm_b200.so (hand-written sm_100a CUDA behind the C-ABI in
include/hetm_b200/capi.h); this package is its Python mirror of the reference
HeTM interface.  Importing it without the built library raises ImportError.
"""
from .api import *  # noqa: F401,F403
from .api import GpuDevice, HetmError, check, device_count  # noqa: F401
from ._lib import LIB_PATH, EXPORTED  # noqa: F401

__all__ = [n for n in dir() if not n.startswith("_")]
