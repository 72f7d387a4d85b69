"""Thin ctypes binding of libgv.so (include/gv.h). Argument marshalling only:
every step of the hot path runs in the library's CUDA kernels.

The functions keep the C names (gv_create, gv_load_edges, ...). Arrays are
numpy (host) arrays; device pointers are plain integers. Errors raise
GVError carrying the gv_status and gv_last_error(). There is no fallback:
if libgv.so is missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GV_LIB_PATH", os.path.join(_HERE, "libgv.so"))  # override: A/B builds

STATUS = ["GV_OK", "GV_ERR_INVALID_ARG", "GV_ERR_STATE", "GV_ERR_OUT_OF_RANGE", "GV_ERR_EMPTY",
          "GV_ERR_CAPACITY", "GV_ERR_NOMEM", "GV_ERR_CUDA", "GV_ERR_COMM"]
GV_OK, GV_ERR_INVALID_ARG, GV_ERR_STATE, GV_ERR_OUT_OF_RANGE, GV_ERR_EMPTY, GV_ERR_CAPACITY, \
    GV_ERR_NOMEM, GV_ERR_CUDA, GV_ERR_COMM = range(9)
GV_LR_CONSTANT, GV_LR_LINEAR = 0, 1
GV_SHUFFLE_PSEUDO, GV_SHUFFLE_NONE, GV_SHUFFLE_RANDOM = 0, 1, 2
GV_IDS_ORIGINAL, GV_IDS_RELABELED = 0, 1


class GVError(RuntimeError):
    def __init__(self, status, msg):
        self.status = status
        name = STATUS[status] if 0 <= status < len(STATUS) else str(status)
        super().__init__(f"{name}: {msg}")


class gv_lr_schedule(C.Structure):
    _fields_ = [("kind", C.c_int), ("floor_ratio", C.c_double), ("total_samples", C.c_uint64)]


class gv_options(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("init_seed", C.c_uint64), ("neg_weight", C.c_float),
                ("device", C.c_int), ("rank", C.c_int), ("world_size", C.c_int),
                ("virtual_ranks", C.c_int), ("ordered", C.c_int), ("compute_loss", C.c_int),
                ("host_threads", C.c_int), ("max_pool_samples", C.c_uint64),
                ("host_partitions", C.c_int), ("host_pool", C.c_int), ("pool_ids", C.c_int),
                ("vertex_tile", C.c_int)]


class gv_episode_stats(C.Structure):
    _fields_ = [("pool_index", C.c_uint64), ("samples", C.c_uint64), ("samples_global", C.c_uint64),
                ("n_steps", C.c_uint32), ("lr_first", C.c_float), ("lr_last", C.c_float),
                ("loss_sum", C.c_double), ("ms_bucket", C.c_double), ("ms_exchange", C.c_double),
                ("ms_sgd", C.c_double), ("ms_rotate", C.c_double), ("ms_total", C.c_double),
                ("sgd_launches", C.c_uint32), ("kernel_launches", C.c_uint32),
                ("n_ranks", C.c_uint32), ("ms_device_max", C.c_double),
                ("ms_total_rank", C.c_double * 64), ("ms_bucket_rank", C.c_double * 64),
                ("ms_exchange_rank", C.c_double * 64), ("ms_sgd_rank", C.c_double * 64),
                ("ms_rotate_rank", C.c_double * 64)]

    def as_dict(self):
        d = {}
        for k, _ in self._fields_:
            v = getattr(self, k)
            d[k] = list(v)[:self.n_ranks] if k.endswith("_rank") else v
        return d


class gv_step_plan(C.Structure):
    _fields_ = [("n_blocks", C.c_uint32), ("vpart", C.c_uint32 * 64), ("cpart", C.c_uint32 * 64),
                ("send_part", C.c_uint32), ("send_to", C.c_uint32), ("recv_part", C.c_uint32),
                ("recv_from", C.c_uint32), ("wait_block", C.c_uint32)]


class gv_augment_cfg(C.Structure):
    _fields_ = [("walk_len", C.c_uint32), ("s", C.c_uint32), ("threads", C.c_uint32),
                ("pool_samples", C.c_uint64), ("seed", C.c_uint64), ("collaborate", C.c_int),
                ("device", C.c_int)]


class gv_run_report(C.Structure):
    _fields_ = [("pools", C.c_uint64), ("samples", C.c_uint64), ("wall_ms", C.c_double),
                ("produce_ms", C.c_double), ("train_wait_ms", C.c_double),
                ("producer_wait_ms", C.c_double), ("loss_sum", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


ctx_p = C.c_void_p
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
f32p = C.POINTER(C.c_float)
u8p = C.POINTER(C.c_uint8)
st = C.c_int

# name -> (restype, argtypes); every symbol of include/gv.h
SIGNATURES = {
    "gv_default_options": (None, [C.POINTER(gv_options)]),
    "gv_create": (st, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_float,
                       C.POINTER(gv_lr_schedule), C.POINTER(gv_options), C.POINTER(ctx_p)]),
    "gv_comm_unique_id": (st, [u8p]),
    "gv_comm_init": (st, [ctx_p, u8p]),
    "gv_load_edges": (st, [ctx_p, u32p, u32p, f32p, C.c_uint64]),
    "gv_push_sample_pool": (st, [ctx_p, u32p, C.c_uint64]),
    "gv_push_sample_pool_device": (st, [ctx_p, C.c_void_p, C.c_uint64]),
    "gv_replay_pool": (st, [ctx_p]),
    "gv_train_episode": (st, [ctx_p, C.POINTER(gv_episode_stats)]),
    "gv_synchronize": (st, [ctx_p]),
    "gv_read_stats": (st, [ctx_p, C.POINTER(gv_episode_stats)]),
    "gv_get_vertex_embeddings": (st, [ctx_p, f32p, C.c_uint64]),
    "gv_get_context_embeddings": (st, [ctx_p, f32p, C.c_uint64]),
    "gv_set_vertex_embeddings": (st, [ctx_p, f32p, C.c_uint64]),
    "gv_set_context_embeddings": (st, [ctx_p, f32p, C.c_uint64]),
    "gv_get_stream": (st, [ctx_p, C.c_int, C.POINTER(C.c_size_t)]),
    "gv_get_progress": (st, [ctx_p, u64p, u64p]),
    "gv_set_progress": (st, [ctx_p, C.c_uint64, C.c_uint64]),
    "gv_augment": (st, [ctx_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64, u32p]),
    "gv_run": (st, [ctx_p, C.POINTER(gv_augment_cfg), C.c_uint64, C.POINTER(gv_run_report)]),
    "gv_augment_device": (st, [ctx_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64]),
    "gv_augment_device_ex": (st, [ctx_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64,
                                  C.c_int]),
    "gv_augment_device_blocks": (st, [ctx_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                      C.c_uint64, C.c_int]),
    "gv_debug_get_pending": (st, [ctx_p, u32p, C.c_uint64, u64p]),
    "gv_get_partition": (st, [ctx_p, u32p, u64p]),
    "gv_get_alias": (st, [ctx_p, C.c_uint32, u32p, u32p, C.c_uint64]),
    "gv_prepare_episode": (st, [ctx_p]),
    "gv_debug_get_buckets": (st, [ctx_p, u32p, C.c_uint64, u64p]),
    "gv_debug_get_negatives": (st, [ctx_p, C.c_uint32, C.c_uint32, u32p, C.c_uint64]),
    "gv_train_explicit": (st, [ctx_p, u32p, u32p, u32p, C.c_uint64, C.c_float]),
    "gv_device_bytes": (st, [ctx_p, u64p]),
    "gv_plan_step": (st, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(gv_step_plan)]),
    "gv_last_error": (C.c_char_p, [ctx_p]),
    "gv_status_string": (C.c_char_p, [C.c_int]),
    "gv_abi_version": (C.c_int, []),
    "gv_destroy": (None, [ctx_p]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1903_00757_b200.build`"
                          " (there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def _ck(status, ctx=None):
    if status != GV_OK:
        msg = lib.gv_last_error(ctx)
        raise GVError(status, msg.decode() if msg else "")


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _ptr(a, t):
    return None if a is None else a.ctypes.data_as(t)


# ------------------------------------------------------------------ functions

def gv_default_options(**kw) -> gv_options:
    o = gv_options()
    lib.gv_default_options(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def gv_create(num_nodes, dim, n_partitions, num_negatives=1, lr0=0.025, alpha=None, opt=None):
    """Returns an opaque context handle (int)."""
    h = ctx_p()
    a = C.byref(alpha) if alpha is not None else None
    o = C.byref(opt) if opt is not None else None
    _ck(lib.gv_create(num_nodes, dim, n_partitions, num_negatives, lr0, a, o, C.byref(h)))
    return h


def gv_comm_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _ck(lib.gv_comm_unique_id(buf))
    return bytes(buf)


def gv_comm_init(ctx, uid: bytes):
    buf = (C.c_uint8 * 128).from_buffer_copy(uid)
    _ck(lib.gv_comm_init(ctx, buf), ctx)


def gv_load_edges(ctx, src, dst, weight=None):
    src = _u32(src).reshape(-1)
    dst = _u32(dst).reshape(-1)
    w = None if weight is None else np.ascontiguousarray(weight, dtype=np.float32).reshape(-1)
    if len(dst) != len(src) or (w is not None and len(w) != len(src)):
        raise ValueError("gv_load_edges: src, dst (and weight) must have the same length")
    _ck(lib.gv_load_edges(ctx, _ptr(src, u32p), _ptr(dst, u32p), _ptr(w, f32p), len(src)), ctx)


def gv_push_sample_pool(ctx, pairs):
    """pairs: (count, 2) uint32 ORIGINAL ids, host memory (pinned is faster)."""
    if hasattr(pairs, "data_ptr"):  # a CPU torch tensor (e.g. pinned) — marshal its pointer
        assert not pairs.is_cuda and pairs.is_contiguous()
        count = pairs.numel() // 2
        _ck(lib.gv_push_sample_pool(ctx, C.cast(pairs.data_ptr(), u32p), count), ctx)
        return
    p = _u32(pairs).reshape(-1)
    _ck(lib.gv_push_sample_pool(ctx, _ptr(p, u32p), len(p) // 2), ctx)


def gv_push_sample_pool_device(ctx, dev_ptr: int, count: int):
    _ck(lib.gv_push_sample_pool_device(ctx, C.c_void_p(dev_ptr), count), ctx)


def gv_replay_pool(ctx):
    _ck(lib.gv_replay_pool(ctx), ctx)


def gv_train_episode(ctx, stats=True):
    s = gv_episode_stats() if stats else None
    _ck(lib.gv_train_episode(ctx, C.byref(s) if s is not None else None), ctx)
    return s.as_dict() if s is not None else None


def gv_read_stats(ctx):
    s = gv_episode_stats()
    _ck(lib.gv_read_stats(ctx, C.byref(s)), ctx)
    return s.as_dict()


def gv_synchronize(ctx):
    _ck(lib.gv_synchronize(ctx), ctx)


def _emb_get(fn, ctx, nv, dim):
    out = np.empty((nv, dim), np.float32)
    _ck(fn(ctx, _ptr(out, f32p), out.size), ctx)
    return out


def gv_get_vertex_embeddings(ctx, nv, dim):
    return _emb_get(lib.gv_get_vertex_embeddings, ctx, nv, dim)


def gv_get_context_embeddings(ctx, nv, dim):
    return _emb_get(lib.gv_get_context_embeddings, ctx, nv, dim)


def gv_set_vertex_embeddings(ctx, arr):
    a = np.ascontiguousarray(arr, dtype=np.float32)
    _ck(lib.gv_set_vertex_embeddings(ctx, _ptr(a, f32p), a.size), ctx)


def gv_set_context_embeddings(ctx, arr):
    a = np.ascontiguousarray(arr, dtype=np.float32)
    _ck(lib.gv_set_context_embeddings(ctx, _ptr(a, f32p), a.size), ctx)


def gv_get_progress(ctx):
    e = C.c_uint64(0)
    sd = C.c_uint64(0)
    _ck(lib.gv_get_progress(ctx, C.byref(e), C.byref(sd)), ctx)
    return e.value, sd.value


def gv_set_progress(ctx, pool_index, samples_done):
    _ck(lib.gv_set_progress(ctx, pool_index, samples_done), ctx)


def gv_get_stream(ctx, vrank=0) -> int:
    s = C.c_size_t(0)
    _ck(lib.gv_get_stream(ctx, vrank, C.byref(s)), ctx)
    return s.value


def gv_augment(ctx, walk_len, s, threads, count, seed, out=None):
    if out is None:
        out = np.empty((count, 2), np.uint32)
    ptr = C.cast(out.data_ptr(), u32p) if hasattr(out, "data_ptr") else _ptr(out, u32p)
    _ck(lib.gv_augment(ctx, walk_len, s, threads, count, seed, ptr), ctx)
    return out


def gv_augment_device(ctx, walk_len, s, segments, count, seed):
    """Generate a pool on the GPU and append it to the pending pool (NEXT-1)."""
    _ck(lib.gv_augment_device(ctx, walk_len, s, segments, count, seed), ctx)


def gv_augment_device_ex(ctx, walk_len, s, segments, count, seed, shuffle):
    """gv_augment_device with a shuffle mode (tab:shuffle ablation)."""
    _ck(lib.gv_augment_device_ex(ctx, walk_len, s, segments, count, seed, shuffle), ctx)


def gv_augment_device_blocks(ctx, walk_len, s, segments, count, seed, shuffle=GV_SHUFFLE_PSEUDO):
    _ck(lib.gv_augment_device_blocks(ctx, walk_len, s, segments, count, seed, shuffle), ctx)


def gv_debug_get_pending(ctx):
    n = C.c_uint64(0)
    _ck(lib.gv_debug_get_pending(ctx, None, 0, C.byref(n)), ctx)
    out = np.empty((max(n.value, 1), 2), np.uint32)
    _ck(lib.gv_debug_get_pending(ctx, _ptr(out, u32p), n.value, C.byref(n)), ctx)
    return out[:n.value]


def gv_run(ctx, walk_len, s, threads, pool_samples, seed, total_samples, collaborate=True,
           device=False):
    cfg = gv_augment_cfg(walk_len, s, threads, pool_samples, seed, 1 if collaborate else 0,
                         1 if device else 0)
    rep = gv_run_report()
    _ck(lib.gv_run(ctx, C.byref(cfg), total_samples, C.byref(rep)), ctx)
    return rep.as_dict()


def gv_get_partition(ctx, nv, n):
    perm = np.empty(nv, np.uint32)
    off = np.empty(n + 1, np.uint64)
    _ck(lib.gv_get_partition(ctx, _ptr(perm, u32p), _ptr(off, u64p)), ctx)
    return perm, off


def gv_get_alias(ctx, p, size):
    prob = np.empty(max(size, 1), np.uint32)
    alias = np.empty(max(size, 1), np.uint32)
    _ck(lib.gv_get_alias(ctx, p, _ptr(prob, u32p), _ptr(alias, u32p), size), ctx)
    return prob[:size], alias[:size]


def gv_prepare_episode(ctx):
    _ck(lib.gv_prepare_episode(ctx), ctx)


def gv_debug_get_buckets(ctx, n, count):
    pairs = np.empty(max(2 * count, 2), np.uint32)
    off = np.empty(n * n + 1, np.uint64)
    _ck(lib.gv_debug_get_buckets(ctx, _ptr(pairs, u32p), count, _ptr(off, u64p)), ctx)
    return pairs[:2 * count].reshape(-1, 2), off


def gv_debug_get_negatives(ctx, i, j, count, K):
    out = np.empty(max(count * K, 1), np.uint32)
    _ck(lib.gv_debug_get_negatives(ctx, i, j, _ptr(out, u32p), count * K), ctx)
    return out[:count * K].reshape(count, K)


def gv_train_explicit(ctx, u, v, negs, lr):
    u = _u32(u)
    v = _u32(v)
    negs = _u32(negs).reshape(-1)
    _ck(lib.gv_train_explicit(ctx, _ptr(u, u32p), _ptr(v, u32p), _ptr(negs, u32p), len(u), lr), ctx)


def gv_plan_step(n, D, d, t):
    """Host-only schedule of rank d at offset step t (no GPU needed)."""
    p = gv_step_plan()
    _ck(lib.gv_plan_step(n, D, d, t, C.byref(p)))
    m = p.n_blocks
    none = 0xFFFFFFFF
    return {"blocks": [(p.vpart[g], p.cpart[g]) for g in range(m)],
            "send_part": None if p.send_part == none else p.send_part, "send_to": p.send_to,
            "recv_part": None if p.recv_part == none else p.recv_part, "recv_from": p.recv_from,
            "wait_block": None if p.wait_block == none else p.wait_block}


def gv_device_bytes(ctx):
    b = C.c_uint64(0)
    _ck(lib.gv_device_bytes(ctx, C.byref(b)), ctx)
    return b.value


def gv_last_error(ctx=None):
    m = lib.gv_last_error(ctx)
    return m.decode() if m else ""


def gv_abi_version():
    return lib.gv_abi_version()


def gv_destroy(ctx):
    lib.gv_destroy(ctx)


class GraphVite:
    """Convenience owner of a gv_ctx (marshalling only)."""

    def __init__(self, num_nodes, dim=128, n_partitions=1, num_negatives=1, lr0=0.025,
                 total_samples=0, lr_kind=GV_LR_LINEAR, floor_ratio=1e-4, **opts):
        self.nv, self.dim, self.n, self.K = num_nodes, dim, n_partitions, num_negatives
        alpha = gv_lr_schedule(lr_kind, floor_ratio, total_samples)
        self.opt = gv_default_options(**opts)
        self.ctx = gv_create(num_nodes, dim, n_partitions, num_negatives, lr0, alpha, self.opt)

    def close(self):
        if getattr(self, "ctx", None):
            gv_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def load_edges(self, src, dst, weight=None):
        gv_load_edges(self.ctx, src, dst, weight)

    def push(self, pairs):
        gv_push_sample_pool(self.ctx, pairs)

    def train_episode(self, stats=True):
        return gv_train_episode(self.ctx, stats)

    def synchronize(self):
        gv_synchronize(self.ctx)

    def read_stats(self):
        return gv_read_stats(self.ctx)

    def replay(self):
        gv_replay_pool(self.ctx)

    def vertex(self):
        return gv_get_vertex_embeddings(self.ctx, self.nv, self.dim)

    def context(self):
        return gv_get_context_embeddings(self.ctx, self.nv, self.dim)

    def set_vertex(self, a):
        gv_set_vertex_embeddings(self.ctx, a)

    def set_context(self, a):
        gv_set_context_embeddings(self.ctx, a)

    def augment(self, walk_len, s, threads, count, seed, out=None):
        return gv_augment(self.ctx, walk_len, s, threads, count, seed, out)

    def augment_device(self, walk_len, s, segments, count, seed, shuffle=GV_SHUFFLE_PSEUDO):
        gv_augment_device_ex(self.ctx, walk_len, s, segments, count, seed, shuffle)

    def augment_device_blocks(self, walk_len, s, segments, count, seed, shuffle=GV_SHUFFLE_PSEUDO):
        gv_augment_device_blocks(self.ctx, walk_len, s, segments, count, seed, shuffle)

    def partition(self):
        return gv_get_partition(self.ctx, self.nv, self.n)

    def checkpoint(self):
        """(vertex, context, pool_index, samples_done) — everything a resume needs."""
        e, sd = gv_get_progress(self.ctx)
        return self.vertex(), self.context(), e, sd

    def restore(self, vertex, context, pool_index, samples_done):
        self.set_vertex(vertex)
        self.set_context(context)
        gv_set_progress(self.ctx, pool_index, samples_done)

    def stream(self, vrank=0):
        return gv_get_stream(self.ctx, vrank)


def gv_status_string(status: int) -> str:
    return lib.gv_status_string(status).decode()
