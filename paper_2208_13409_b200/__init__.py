"""B200-native Lagrange + DirectCF (unsplit 9-point) remap step.

The product is ``libh2d.so`` (CUDA sm_100a, built from ``csrc/``) behind the
C-ABI of ``include/h2d.h``; this package is the Python host mirror of the
reference solver interface (proj/include/hydro/*.hpp) over that ABI.
"""
import os as _os

from . import errors
from .abi import (BC_PERIODIC, BC_WALL, CORNER_LINEARDIAG, CORNER_UPWIND, EOS_PERFECT, EOS_STIFFENED,
                  REMAP_DIRECTCF, HostLagrange, HostState, Library, RemapDiag, Solver, make_config)

PKG_DIR = _os.path.dirname(_os.path.abspath(__file__))
# H2D_PRODUCT_LIB selects another build of the same sources (tools/variants.py
# builds launch-bound / tile variants for measurement); default: the in-tree build
PRODUCT_LIB = _os.environ.get("H2D_PRODUCT_LIB") or _os.path.join(PKG_DIR, "libh2d.so")

_product = None


def product_library() -> Library:
    """Load the CUDA product library. There is no CPU fallback: a missing or
    unloadable ``libh2d.so`` is an error (run ``__graft_entry__.build()``)."""
    global _product
    if _product is None:
        if not _os.path.exists(PRODUCT_LIB):
            raise ImportError(f"{PRODUCT_LIB} is missing: build it with __graft_entry__.build()")
        _product = Library(PRODUCT_LIB, "h2d_")
    return _product


def solver(cfg, device: int = 0) -> Solver:
    """A device-resident solver context on ``device`` (CUDA)."""
    return Solver(product_library(), cfg, device)
