"""TEST INFRASTRUCTURE ONLY — ctypes wrapper of the serial C oracle.

The oracle (oracle/gv_oracle.c) is a plain, slow, serial implementation of
the GraphVite hot path written from PAPER.md (see its header for citations).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this module. The product package
(paper_1903_00757_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gv_oracle.c")
_HDR = os.path.join(_HERE, "gv_oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")

OK = 0


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (IEEE float, no contraction)."""
    newest = max(os.path.getmtime(_SRC), os.path.getmtime(_HDR))
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < newest:
        # -fopenmp only affects or_trainer_train_pool_hogwild (the CPU
        # baseline class); every other function is serial
        cmd = ["gcc", "-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-fPIC", "-shared", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _declare(_lib)
    return _lib


u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)
vp = C.c_void_p


def _declare(L):
    sig = {
        "or_philox4x32_10": (None, [u32p, u32p, u32p]),
        "or_graph_build": (C.c_int, [C.c_uint32, u32p, u32p, f32p, C.c_uint64, C.POINTER(vp)]),
        "or_graph_free": (None, [vp]),
        "or_graph_entries": (C.c_uint64, [vp]),
        "or_graph_csr": (None, [vp, u64p, u32p, f64p]),
        "or_graph_degree": (None, [vp, f64p]),
        "or_zigzag": (C.c_int, [C.c_uint32, f64p, C.c_uint32, u32p, u32p, u64p]),
        "or_alias_build": (C.c_int, [f64p, C.c_uint32, u32p, u32p]),
        "or_alias_draw": (C.c_uint32, [u32p, u32p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32]),
        "or_lr": (C.c_float, [C.c_int, C.c_double, C.c_double, C.c_uint64, C.c_uint64]),
        "or_sgd_sample": (C.c_double, [f32p, C.POINTER(f32p), C.c_uint32, C.c_uint32, C.c_float, C.c_float]),
        "or_bucket": (C.c_int, [u32p, C.c_uint64, C.c_uint32, u32p, u64p, C.c_uint32, u32p, u64p]),
        "or_bucket_tiled": (C.c_int, [u32p, C.c_uint64, C.c_uint32, u32p, u64p, C.c_uint32,
                                      C.c_uint32, u32p, u64p]),
        "or_schedule_cid": (C.c_uint32, [C.c_uint32, C.c_uint32, C.c_uint32]),
        "or_trainer_set_vertex_tile": (C.c_int, [vp, C.c_uint32]),
        "or_trainer_create": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_float,
                                        C.c_int, C.c_double, C.c_uint64, C.c_uint64, C.c_uint64,
                                        C.c_float, C.POINTER(vp)]),
        "or_trainer_load_edges": (C.c_int, [vp, u32p, u32p, f32p, C.c_uint64]),
        "or_trainer_train_pool": (C.c_int, [vp, u32p, C.c_uint64, f64p]),
        "or_trainer_train_pool_hogwild": (C.c_int, [vp, u32p, C.c_uint64, C.c_int, f64p]),
        "or_trainer_train_block": (C.c_int, [vp, u32p, C.c_uint64, C.c_uint32, C.c_uint32,
                                             C.c_uint32, C.c_float, f64p]),
        "or_trainer_negatives": (C.c_int, [vp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, u32p]),
        "or_trainer_negative_at": (C.c_uint32, [vp, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32]),
        "or_trainer_explicit": (C.c_int, [vp, u32p, u32p, u32p, C.c_uint64, C.c_float]),
        "or_trainer_get": (None, [vp, C.c_int, f32p]),
        "or_trainer_set": (None, [vp, C.c_int, f32p]),
        "or_trainer_partition": (None, [vp, u32p, u64p]),
        "or_trainer_alias": (C.c_int, [vp, C.c_uint32, u32p, u32p]),
        "or_trainer_samples_done": (C.c_uint64, [vp]),
        "or_trainer_graph": (vp, [vp]),
        "or_trainer_free": (None, [vp]),
        "or_init_vertex": (None, [C.c_uint32, C.c_uint32, C.c_uint64, f32p]),
        "or_sampler_create": (C.c_int, [vp, C.POINTER(vp)]),
        "or_sampler_free": (None, [vp]),
        "or_sampler_walk": (C.c_int, [vp, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, u32p]),
        "or_pairs_within": (C.c_uint64, [u32p, C.c_uint32, C.c_uint32, u32p]),
        "or_pseudo_shuffle": (None, [u32p, C.c_uint64, C.c_uint32, u32p]),
        "or_augment": (C.c_int, [vp, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64, u32p]),
        "or_cosine": (C.c_double, [f32p, f32p, C.c_uint32]),
        "or_auc": (C.c_double, [f64p, C.c_uint64, f64p, C.c_uint64]),
        "or_linkpred_auc": (C.c_double, [f32p, C.c_uint32, u32p, C.c_uint64, u32p, C.c_uint64]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args


def _p(a, t):
    return a.ctypes.data_as(t) if a is not None else None


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


class OracleError(RuntimeError):
    pass


def _check(rc, what):
    if rc != OK:
        raise OracleError(f"{what} failed with code {rc}")


# ---------------------------------------------------------------- primitives

def philox(ctr, key):
    c = _u32(ctr)
    k = _u32(key)
    out = np.zeros(4, np.uint32)
    lib().or_philox4x32_10(_p(c, u32p), _p(k, u32p), _p(out, u32p))
    return out


def alias_build(weights):
    w = np.ascontiguousarray(weights, dtype=np.float64)
    m = len(w)
    prob = np.zeros(max(m, 1), np.uint32)
    alias = np.zeros(max(m, 1), np.uint32)
    _check(lib().or_alias_build(_p(w, f64p), m, _p(prob, u32p), _p(alias, u32p)), "alias_build")
    return prob[:m], alias[:m]


def alias_draw(prob, alias, r0, r1, r2):
    prob = _u32(prob)
    alias = _u32(alias)
    return int(lib().or_alias_draw(_p(prob, u32p), _p(alias, u32p), len(prob), r0, r1, r2))


def lr(kind, lr0, floor_ratio, s_before, s_total):
    return float(lib().or_lr(kind, lr0, floor_ratio, s_before, s_total))


def sgd_sample(U, Cs, lr_, neg_weight):
    """In-place update of float32 arrays U (d,) and each C in Cs (list of (d,)).
    Rows that are the same object alias (sequential semantics)."""
    d = len(U)
    arr = (f32p * len(Cs))(*[c.ctypes.data_as(f32p) for c in Cs])
    return lib().or_sgd_sample(U.ctypes.data_as(f32p), arr, len(Cs), d, lr_, neg_weight)


def zigzag(deg, n):
    deg = np.ascontiguousarray(deg, dtype=np.float64)
    nv = len(deg)
    perm = np.zeros(nv, np.uint32)
    inv = np.zeros(nv, np.uint32)
    off = np.zeros(n + 1, np.uint64)
    _check(lib().or_zigzag(nv, _p(deg, f64p), n, _p(perm, u32p), _p(inv, u32p), _p(off, u64p)), "zigzag")
    return perm, inv, off


def bucket(pairs, nv, perm, part_off, n):
    pairs = _u32(pairs).reshape(-1)
    cnt = len(pairs) // 2
    out = np.zeros(max(2 * cnt, 2), np.uint32)
    boff = np.zeros(n * n + 1, np.uint64)
    perm = _u32(perm)
    part_off = np.ascontiguousarray(part_off, dtype=np.uint64)
    _check(lib().or_bucket(_p(pairs, u32p), cnt, nv, _p(perm, u32p), _p(part_off, u64p), n,
                           _p(out, u32p), _p(boff, u64p)), "bucket")
    return out[:2 * cnt].reshape(-1, 2), boff


def bucket_tiled(pairs, nv, perm, part_off, n, tile_bits):
    """or_bucket_tiled: bucketing, then each block in vertex-tile order (R-VTILE)."""
    pairs = _u32(pairs).reshape(-1)
    cnt = len(pairs) // 2
    out = np.zeros(max(2 * cnt, 2), np.uint32)
    boff = np.zeros(n * n + 1, np.uint64)
    perm = _u32(perm)
    part_off = np.ascontiguousarray(part_off, dtype=np.uint64)
    _check(lib().or_bucket_tiled(_p(pairs, u32p), cnt, nv, _p(perm, u32p), _p(part_off, u64p), n,
                                 tile_bits, _p(out, u32p), _p(boff, u64p)), "bucket_tiled")
    return out[:2 * cnt].reshape(-1, 2), boff


def schedule_cid(n, t, i):
    return int(lib().or_schedule_cid(n, t, i))


def init_vertex(nv, d, seed):
    out = np.zeros((nv, d), np.float32)
    lib().or_init_vertex(nv, d, seed, _p(out, f32p))
    return out


def pairs_within(walk, s):
    walk = _u32(walk)
    out = np.zeros(max(2 * len(walk) * s, 2), np.uint32)
    c = lib().or_pairs_within(_p(walk, u32p), len(walk), s, _p(out, u32p))
    return out[:2 * c].reshape(-1, 2)


def pseudo_shuffle(pairs, s):
    pairs = _u32(pairs).reshape(-1)
    cnt = len(pairs) // 2
    out = np.zeros(max(2 * cnt, 2), np.uint32)
    lib().or_pseudo_shuffle(_p(pairs, u32p), cnt, s, _p(out, u32p))
    return out[:2 * cnt].reshape(-1, 2)


def auc(pos_scores, neg_scores):
    p = np.ascontiguousarray(pos_scores, dtype=np.float64)
    q = np.ascontiguousarray(neg_scores, dtype=np.float64)
    return float(lib().or_auc(_p(p, f64p), len(p), _p(q, f64p), len(q)))


def linkpred_auc(emb, pos_pairs, neg_pairs):
    emb = np.ascontiguousarray(emb, dtype=np.float32)
    pp = _u32(pos_pairs).reshape(-1)
    npr = _u32(neg_pairs).reshape(-1)
    return float(lib().or_linkpred_auc(_p(emb, f32p), emb.shape[1], _p(pp, u32p), len(pp) // 2,
                                       _p(npr, u32p), len(npr) // 2))


# ---------------------------------------------------------------- graph

class Graph:
    def __init__(self, nv, src, dst, w=None):
        self.nv = nv
        src = _u32(src)
        dst = _u32(dst)
        wa = None if w is None else np.ascontiguousarray(w, dtype=np.float32)
        h = vp()
        _check(lib().or_graph_build(nv, _p(src, u32p), _p(dst, u32p), _p(wa, f32p), len(src),
                                    C.byref(h)), "graph_build")
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.or_graph_free(self.h)
            self.h = None

    def csr(self):
        m = lib().or_graph_entries(self.h)
        off = np.zeros(self.nv + 1, np.uint64)
        nbr = np.zeros(max(m, 1), np.uint32)
        w = np.zeros(max(m, 1), np.float64)
        lib().or_graph_csr(self.h, _p(off, u64p), _p(nbr, u32p), _p(w, f64p))
        return off, nbr[:m], w[:m]

    def degree(self):
        deg = np.zeros(self.nv, np.float64)
        lib().or_graph_degree(self.h, _p(deg, f64p))
        return deg


class _TrainerGraph:
    """Borrowed view of a Trainer's ingested graph (kept alive by the trainer)."""

    def __init__(self, trainer):
        self.trainer = trainer
        self.h = lib().or_trainer_graph(trainer.h)


class Sampler:
    def __init__(self, graph):
        self.graph = graph
        h = vp()
        _check(lib().or_sampler_create(graph.h, C.byref(h)), "sampler_create")
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.or_sampler_free(self.h)
            self.h = None

    def walk(self, thread, walk, walk_len, seed):
        out = np.zeros(walk_len + 1, np.uint32)
        _check(lib().or_sampler_walk(self.h, thread, walk, walk_len, seed, _p(out, u32p)), "walk")
        return out

    def augment(self, walk_len, s, threads, count, seed):
        out = np.zeros(max(2 * count, 2), np.uint32)
        _check(lib().or_augment(self.h, walk_len, s, threads, count, seed, _p(out, u32p)), "augment")
        return out[:2 * count].reshape(-1, 2)


class Trainer:
    """Serial oracle trainer."""

    def __init__(self, nv, d, n, K=1, lr0=0.025, lr_kind=1, floor_ratio=1e-4, total_samples=0,
                 seed=5, init_seed=4, neg_weight=5.0, vertex_tile=0):
        self.nv, self.d, self.n, self.K = nv, d, n, K
        h = vp()
        _check(lib().or_trainer_create(nv, d, n, K, lr0, lr_kind, floor_ratio, total_samples, seed,
                                       init_seed, neg_weight, C.byref(h)), "trainer_create")
        self.h = h
        if vertex_tile:  # R-VTILE: blocks in vertex-tile order (or_bucket_tiled)
            _check(lib().or_trainer_set_vertex_tile(h, vertex_tile), "set_vertex_tile")

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.or_trainer_free(self.h)
            self.h = None

    def sampler(self):
        """Online-augmentation sampler over the graph this trainer ingested
        (no second ingest: the Friendster-shaped graph is 43 GB as CSR)."""
        return Sampler(_TrainerGraph(self))

    def load_edges(self, src, dst, w=None):
        src = _u32(src)
        dst = _u32(dst)
        wa = None if w is None else np.ascontiguousarray(w, dtype=np.float32)
        _check(lib().or_trainer_load_edges(self.h, _p(src, u32p), _p(dst, u32p), _p(wa, f32p),
                                           len(src)), "load_edges")

    def train_pool(self, pairs):
        pairs = _u32(pairs).reshape(-1)
        loss = C.c_double(0)
        _check(lib().or_trainer_train_pool(self.h, _p(pairs, u32p), len(pairs) // 2,
                                           C.byref(loss)), "train_pool")
        return loss.value

    def train_pool_hogwild(self, pairs, threads):
        """CPU baseline class (bench only): OpenMP Hogwild over each block."""
        pairs = _u32(pairs).reshape(-1)
        loss = C.c_double(0)
        _check(lib().or_trainer_train_pool_hogwild(self.h, _p(pairs, u32p), len(pairs) // 2,
                                                   threads, C.byref(loss)), "train_pool_hogwild")
        return loss.value

    def train_block(self, local_pairs, i, j, e, lr_):
        lp = _u32(local_pairs).reshape(-1)
        loss = C.c_double(0)
        _check(lib().or_trainer_train_block(self.h, _p(lp, u32p), len(lp) // 2, i, j, e, lr_,
                                            C.byref(loss)), "train_block")
        return loss.value

    def negatives(self, count, i, j, e):
        out = np.zeros(max(count * self.K, 1), np.uint32)
        _check(lib().or_trainer_negatives(self.h, count, i, j, e, _p(out, u32p)), "negatives")
        return out[:count * self.K].reshape(count, self.K)

    def negative_at(self, q, i, j, e, k=0):
        return int(lib().or_trainer_negative_at(self.h, q, i, j, e, k))

    def explicit(self, u, v, negs, lr_):
        u = _u32(u)
        v = _u32(v)
        negs = _u32(negs).reshape(-1)
        _check(lib().or_trainer_explicit(self.h, _p(u, u32p), _p(v, u32p), _p(negs, u32p), len(u),
                                         lr_), "explicit")

    def get(self, which):
        out = np.zeros((self.nv, self.d), np.float32)
        lib().or_trainer_get(self.h, 1 if which == "context" else 0, _p(out, f32p))
        return out

    def set(self, which, arr):
        arr = np.ascontiguousarray(arr, dtype=np.float32)
        assert arr.shape == (self.nv, self.d)
        lib().or_trainer_set(self.h, 1 if which == "context" else 0, _p(arr, f32p))

    def partition(self):
        perm = np.zeros(self.nv, np.uint32)
        off = np.zeros(self.n + 1, np.uint64)
        lib().or_trainer_partition(self.h, _p(perm, u32p), _p(off, u64p))
        return perm, off

    def alias(self, p):
        _, off = self.partition()
        m = int(off[p + 1] - off[p])
        prob = np.zeros(max(m, 1), np.uint32)
        al = np.zeros(max(m, 1), np.uint32)
        _check(lib().or_trainer_alias(self.h, p, _p(prob, u32p), _p(al, u32p)), "alias")
        return prob[:m], al[:m]

    @property
    def samples_done(self):
        return int(lib().or_trainer_samples_done(self.h))
