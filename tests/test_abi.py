"""CPU tests of the boundary: libgv.so loads without a GPU, exports every
symbol include/gv.h declares, host-only calls work, and the ctypes struct
layouts match the header."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gv.h")


def _declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gv_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_north_star_calls():
    names = _declared_functions()
    for f in ["gv_create", "gv_load_edges", "gv_push_sample_pool", "gv_train_episode",
              "gv_get_vertex_embeddings", "gv_get_context_embeddings", "gv_destroy"]:
        assert f in names


def test_library_exports_every_declared_symbol():
    from paper_1903_00757_b200 import gv
    lib = C.CDLL(gv.LIB_PATH)
    missing = [f for f in _declared_functions() if not hasattr(lib, f)]
    assert not missing, missing
    # the binding covers the whole header, under the same names
    assert set(_declared_functions()) <= set(gv.SIGNATURES)
    for f in _declared_functions():
        assert hasattr(gv, f), f


def test_host_only_calls():
    from paper_1903_00757_b200 import gv
    assert gv.gv_abi_version() == 4
    o = gv.gv_default_options()
    assert (o.seed, o.init_seed, o.neg_weight, o.world_size, o.virtual_ranks, o.ordered) == (5, 4, 5.0, 1, 1, 0)
    assert gv.lib.gv_status_string(3) == b"GV_ERR_OUT_OF_RANGE"


def test_struct_sizes_match_header():
    """Compile a probe against include/gv.h and compare sizeof/offsetof."""
    import subprocess
    import tempfile
    from paper_1903_00757_b200 import gv
    src = r'''
#include <stdio.h>
#include <stddef.h>
#include "gv.h"
int main(void){
 printf("%zu %zu %zu %zu %zu\n", sizeof(gv_options), sizeof(gv_episode_stats),
        sizeof(gv_lr_schedule), sizeof(gv_augment_cfg), sizeof(gv_run_report));
 printf("%zu %zu %zu %zu %zu\n", offsetof(gv_options, max_pool_samples), offsetof(gv_episode_stats, ms_total),
        offsetof(gv_episode_stats, kernel_launches), offsetof(gv_episode_stats, ms_device_max),
        offsetof(gv_episode_stats, ms_rotate_rank));
 return 0;}
'''
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "p.c")
        open(c, "w").write(src)
        exe = os.path.join(d, "p")
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe])
        out = subprocess.check_output([exe]).decode().split()
    sizes = [C.sizeof(gv.gv_options), C.sizeof(gv.gv_episode_stats), C.sizeof(gv.gv_lr_schedule),
             C.sizeof(gv.gv_augment_cfg), C.sizeof(gv.gv_run_report)]
    assert [int(x) for x in out[:5]] == sizes
    assert int(out[5]) == gv.gv_options.max_pool_samples.offset
    assert int(out[6]) == gv.gv_episode_stats.ms_total.offset
    assert int(out[7]) == gv.gv_episode_stats.kernel_launches.offset
    assert int(out[8]) == gv.gv_episode_stats.ms_device_max.offset
    assert int(out[9]) == gv.gv_episode_stats.ms_rotate_rank.offset


def test_no_cuda_device_fails_loudly():
    """Without a GPU the product refuses (no CPU fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1903_00757_b200 import gv
    with pytest.raises(gv.GVError) as e:
        gv.gv_create(100, 8, 1)
    assert e.value.status == gv.GV_ERR_CUDA


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_1903_00757_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".cuh", ".hpp", ".h")):
                text = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "oracle" not in re.sub(r"(#|//).*", "", text).lower() or f == "__init__.py", f


@pytest.mark.parametrize("args,kw", [
    ((0, 128, 1), {}),                     # num_nodes = 0
    ((100, 0, 1), {}),                     # dim = 0
    ((100, 6, 1), {}),                     # dim % 4 != 0
    ((100, 516, 1), {}),                   # dim > 512
    ((100, 128, 0), {}),                   # n_partitions = 0
    ((100, 128, 101), {}),                 # n_partitions > num_nodes
    ((1000, 128, 65), {}),                 # n_partitions > 64
    ((100, 128, 4, 0), {}),                # K = 0
    ((100, 128, 4, 9), {}),                # K > 8
    ((100, 128, 3), {"world_size": 2}),    # n % ranks != 0
    ((100, 128, 4), {"virtual_ranks": 3}),
    ((100, 128, 4), {"world_size": 2, "virtual_ranks": 2}),
    ((100, 128, 4), {"rank": 2, "world_size": 2}),
    ((100, 128, 1), {"host_partitions": 1}),            # out-of-core needs n >= 2
    ((100, 128, 4), {"host_partitions": 1, "virtual_ranks": 2}),
])
def test_create_rejects_bad_arguments_without_a_gpu(args, kw):
    """gv_create validates every argument before touching the device
    (include/gv.h: GV_ERR_INVALID_ARG)."""
    from paper_1903_00757_b200 import gv
    opt = gv.gv_default_options(**kw)
    with pytest.raises(gv.GVError) as e:
        gv.gv_create(*args, opt=opt)
    assert e.value.status == gv.GV_ERR_INVALID_ARG


def test_plan_step_is_host_only():
    """gv_plan_step runs without a GPU (the gloo multi-rank test relies on it)."""
    from paper_1903_00757_b200 import gv
    p = gv.gv_plan_step(8, 4, 3, 5)
    assert p["blocks"] == [(6, 3), (7, 4)] and p["send_to"] == 2 and p["recv_from"] == 0


def build_c_smoke(out_dir):
    """Compile tests/c/abi_smoke.c (plain C99, gcc) against include/gv.h and
    link it to libgv.so: the boundary is usable without Python."""
    import subprocess
    from paper_1903_00757_b200 import gv
    exe = os.path.join(out_dir, "abi_smoke")
    libdir = os.path.dirname(gv.LIB_PATH)
    subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "c", "abi_smoke.c"), "-o", exe, "-L", libdir,
                           "-lgv", "-Wl,-rpath," + libdir, "-lm"])
    return exe


def test_plain_c_program_compiles_and_links(tmp_path):
    assert os.path.exists(build_c_smoke(str(tmp_path)))
