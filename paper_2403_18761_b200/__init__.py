"""B200-native RPD hot path of MATTopo (arXiv 2403.18761).

The product is ``librpd.so`` (CUDA for sm_100a behind the C ABI in ``include/rpd.h``); this
package holds its sources (``csrc/``), the in-tree build and the thin ctypes binding.
"""
from ._build import LIB, build  # noqa: F401
from .rpd import (EXPORTED, RPDContext, RPDError, load_library, rpd_full)  # noqa: F401

__all__ = ["build", "RPDContext", "RPDError", "load_library", "rpd_full", "EXPORTED"]
