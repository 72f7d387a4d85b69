"""B200-native parallel negative sampling trainer (GraphVite, arXiv 1903.00757).

The hot path lives in libgv.so (csrc/, C ABI include/gv.h); `gv` is its thin
ctypes binding. Importing the package loads the library and raises if it is
missing (no CPU fallback)."""
from . import gv  # noqa: F401
from .gv import GraphVite, GVError  # noqa: F401

__all__ = ["gv", "GraphVite", "GVError"]
