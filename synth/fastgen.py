"""ctypes wrapper of synth/gen.c (large Chung-Lu configs). Input generator."""
import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_LIB = os.path.join(_HERE, "libsynthgen.so")


def _lib():
    if not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O3", "-fopenmp", "-fPIC", "-shared", _SRC, "-o",
                               _LIB + ".tmp", "-lm"])
        os.replace(_LIB + ".tmp", _LIB)
    lib = C.CDLL(_LIB)
    lib.synth_chung_lu.restype = C.c_int
    lib.synth_chung_lu.argtypes = [C.c_uint32, C.c_uint64, C.c_double, C.c_double, C.c_uint64,
                                   C.c_uint64, C.c_int, C.c_void_p, C.c_void_p]
    return lib


def chung_lu_draws(nv, ne, gamma, wmax, seed=1, perm_seed=2, threads=0):
    """ne Chung-Lu edge draws (duplicates / self-loops kept), uint32 (src, dst)."""
    src = np.empty(ne, np.uint32)
    dst = np.empty(ne, np.uint32)
    rc = _lib().synth_chung_lu(nv, ne, gamma, wmax, seed, perm_seed, threads or os.cpu_count(),
                               src.ctypes.data, dst.ctypes.data)
    if rc:
        raise MemoryError("synth_chung_lu failed")
    return src, dst
