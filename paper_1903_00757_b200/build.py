"""Build libgv.so (the product C-ABI library) in-tree for sm_100a.

    python -m paper_1903_00757_b200.build [--force]

nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo; the CUDA
runtime is linked statically; NCCL is dlopen'ed at run time (multi-process
only). Objects are compiled in parallel and cached by mtime.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build" + os.environ.get("GV_BUILD_TAG", ""))
LIB = os.environ.get("GV_LIB_OUT", os.path.join(PKG, "libgv.so"))
EXTRA = os.environ.get("GV_EXTRA_FLAGS", "").split()  # experiments, e.g. -DGV_PREFETCH=8
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3,-Wall",
          "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]
SOURCES = ["sgd.cu", "bucket.cu", "sampler.cu", "engine.cpp", "transport_local.cpp", "transport_ipc.cpp", "outofcore.cpp",
           "host_graph.cpp", "augment.cpp", "run.cpp", "ipc.cpp", "graph_share.cpp"]
HEADERS = ["kernels.cuh", "device_common.cuh", "bucket_common.cuh", "philox.cuh", "host_graph.hpp", "augment.hpp", "ipc.hpp",
           "graph_share.hpp", "engine.hpp", "transport.hpp"]


def _newest_dep():
    paths = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "gv.h")]
    return max(os.path.getmtime(p) for p in paths)


def _compile(src, force, verbose):
    path = os.path.join(CSRC, src)
    obj = os.path.join(BUILD, src + ".o")
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(
            os.path.getmtime(path), _newest_dep()):
        return obj, ""
    cmd = [NVCC, *ARCH, *COMMON, *EXTRA, "-c", path, "-o", obj]
    if verbose and src.endswith(".cu"):
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(lambda s: _compile(s, force, verbose), SOURCES))
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            if log:
                print(log, file=sys.stderr)
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB + ".tmp", *objs, "-ldl", "-lpthread", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
