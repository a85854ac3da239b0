"""B200-native batched NDF range query from CP factors (Deng et al., arXiv 2109.14807).

The product is libpndf.so (CUDA, sm_100a; C ABI in include/pndf.h); ``pndf``
is its thin ctypes binding.  See DESIGN.md.
"""
from . import pndf  # noqa: F401
from .pndf import Store, load_factors, make_desc  # noqa: F401

__all__ = ["pndf", "Store", "load_factors", "make_desc"]
