"""B200-native parallel negative sampling trainer (GraphVite, arXiv 1903.00757).

The hot path lives in libgv.so (csrc/, C ABI include/gv.h); `gv` is its thin
ctypes binding. Importing `gv` loads the library and raises if it is missing
(no CPU fallback). `build` compiles it and does not load it."""
import importlib

__all__ = ["gv", "GraphVite", "GVError", "build"]


def __getattr__(name):
    if name in ("gv", "GraphVite", "GVError"):
        mod = importlib.import_module(".gv", __name__)
        return mod if name == "gv" else getattr(mod, name)
    raise AttributeError(name)
