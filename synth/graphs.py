"""Seeded synthetic graph and pool generators (input recipe).

The paper gives only |V| and |E| of its datasets (tab:datasets);
degree shape is a proposal: Chung-Lu expected degrees
w_i ∝ (i+10)^(-1/(gamma-1)), capped at w_max, rescaled to sum 2|E|; edges
u ~ w, v ~ w; self-loops and duplicates are discarded until |E| unique
undirected edges exist; node ids are randomly permuted. The DC-SBM variant
draws v inside u's community with probability 1-mu (quality tests).

Nothing here computes any part of the method (no alias tables, no
partitioning, no training); both the oracle and the CUDA path consume these
arrays unchanged.
"""
from __future__ import annotations

import numpy as np

# BASELINE.json configs -> generator parameters.
CONFIGS = {
    "C1": dict(nv=10_000, ne=50_000, gamma=2.1, wmax=300.0, kind="dcsbm", c=50, mu=0.2,
               d=128, K=1, s=1, n=1, pool=2_000_000),
    "C2": dict(nv=1_138_499, ne=4_945_382, gamma=2.1, wmax=3e4, kind="chung_lu",
               d=128, K=1, s=5, n=1, pool=200_000_000),
    "C4": dict(nv=7_944_949, ne=447_219_610, gamma=2.5, wmax=1e4, kind="chung_lu",
               d=128, K=1, s=2, n=8, pool=1_600_000_000),
    "C5": dict(nv=65_608_376, ne=1_806_067_142, gamma=2.5, wmax=5e3, kind="chung_lu",
               d=128, K=1, s=2, n=8, pool=4_000_000_000),
}


def _weights(nv, ne, gamma, wmax):
    i = np.arange(nv, dtype=np.float64)
    w = (i + 10.0) ** (-1.0 / (gamma - 1.0))
    w *= 2.0 * ne / w.sum()
    w = np.minimum(w, wmax)
    w *= 2.0 * ne / w.sum()
    return w


def _unique_edges(us, vs, nv):
    """Keep the first occurrence of each undirected non-self-loop edge."""
    keep = us != vs
    us, vs = us[keep], vs[keep]
    lo = np.minimum(us, vs).astype(np.uint64)
    hi = np.maximum(us, vs).astype(np.uint64)
    key = lo * np.uint64(nv) + hi
    _, first = np.unique(key, return_index=True)
    first.sort()
    return us[first], vs[first]


def _draw_until(nv, ne, draw, rng):
    src = np.zeros(0, np.int64)
    dst = np.zeros(0, np.int64)
    need = ne
    while True:
        batch = int(need * 1.15) + 1024
        u, v = draw(batch)
        src = np.concatenate([src, u])
        dst = np.concatenate([dst, v])
        src, dst = _unique_edges(src, dst, nv)
        if len(src) >= ne:
            return src[:ne], dst[:ne]
        need = ne - len(src)


def chung_lu(nv, ne, gamma=2.1, wmax=None, seed=1, perm_seed=2):
    """Power-law Chung-Lu graph: returns (src, dst) uint32 arrays of ne unique
    undirected edges over nv nodes (ids randomly permuted)."""
    rng = np.random.default_rng(seed)
    w = _weights(nv, ne, gamma, wmax if wmax is not None else float(nv))
    cdf = np.cumsum(w)
    cdf /= cdf[-1]

    def draw(k):
        u = np.searchsorted(cdf, rng.random(k), side="right")
        v = np.searchsorted(cdf, rng.random(k), side="right")
        return np.minimum(u, nv - 1), np.minimum(v, nv - 1)

    src, dst = _draw_until(nv, ne, draw, rng)
    perm = np.random.default_rng(perm_seed).permutation(nv)
    return perm[src].astype(np.uint32), perm[dst].astype(np.uint32)


def dcsbm(nv, ne, gamma=2.1, wmax=None, c=50, mu=0.2, seed=1, perm_seed=2):
    """Degree-corrected SBM: c communities; with probability 1-mu the second
    endpoint is drawn (∝ w) inside the first endpoint's community.
    Returns (src, dst, community) with community indexed by the permuted id."""
    rng = np.random.default_rng(seed)
    w = _weights(nv, ne, gamma, wmax if wmax is not None else float(nv))
    comm = rng.integers(0, c, nv)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    members = [np.flatnonzero(comm == k) for k in range(c)]
    ccdf = []
    for mem in members:
        cw = np.cumsum(w[mem])
        ccdf.append(cw / cw[-1] if len(mem) else cw)

    def draw(k):
        u = np.minimum(np.searchsorted(cdf, rng.random(k), side="right"), nv - 1)
        v = np.minimum(np.searchsorted(cdf, rng.random(k), side="right"), nv - 1)
        inside = rng.random(k) >= mu
        cu = comm[u]
        for q in range(c):
            sel = np.flatnonzero(inside & (cu == q))
            if len(sel) == 0 or len(members[q]) == 0:
                continue
            idx = np.searchsorted(ccdf[q], rng.random(len(sel)), side="right")
            v[sel] = members[q][np.minimum(idx, len(members[q]) - 1)]
        return u, v

    src, dst = _draw_until(nv, ne, draw, rng)
    perm = np.random.default_rng(perm_seed).permutation(nv)
    comm_new = np.empty(nv, np.int64)
    comm_new[perm] = comm
    return perm[src].astype(np.uint32), perm[dst].astype(np.uint32), comm_new


def edge_pool(src, dst, count, seed=3):
    """LINE-style edge samples (s = 1 pools): directed edges drawn uniformly
    from the symmetrised edge list, interleaved (u, v) uint32 [count, 2]."""
    rng = np.random.default_rng(seed)
    k = rng.integers(0, len(src), count)
    flip = rng.random(count) < 0.5
    u = np.where(flip, dst[k], src[k])
    v = np.where(flip, src[k], dst[k])
    return np.stack([u, v], axis=1).astype(np.uint32)


def uniform_pool(nv, count, seed=3):
    """Uniform random (u, v) pairs — bucketing/parity edge cases."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, nv, (count, 2), dtype=np.uint32)


def linkpred_split(src, dst, nv, holdout=0.01, seed=6):
    """Link-prediction protocol: hold out a fraction of the
    edges as positives and draw as many uniform node pairs as negatives,
    rejecting self-pairs and edges of the FULL graph. Returns
    (train_src, train_dst, pos_pairs[h,2], neg_pairs[h,2])."""
    rng = np.random.default_rng(seed)
    ne = len(src)
    h = int(round(ne * holdout))
    idx = rng.permutation(ne)
    hold, keep = idx[:h], np.sort(idx[h:])
    pos = np.stack([src[hold], dst[hold]], axis=1).astype(np.uint32)
    lo = np.minimum(src, dst).astype(np.uint64)
    hi = np.maximum(src, dst).astype(np.uint64)
    edge_keys = np.unique(lo * np.uint64(nv) + hi)
    neg = np.zeros((0, 2), np.uint32)
    while len(neg) < h:
        k = 2 * (h - len(neg)) + 16
        a = rng.integers(0, nv, k, dtype=np.int64)
        b = rng.integers(0, nv, k, dtype=np.int64)
        ok = a != b
        key = np.minimum(a, b).astype(np.uint64) * np.uint64(nv) + np.maximum(a, b).astype(np.uint64)
        pos_idx = np.searchsorted(edge_keys, key)
        pos_idx = np.minimum(pos_idx, len(edge_keys) - 1)
        ok &= edge_keys[pos_idx] != key
        cand = np.stack([a[ok], b[ok]], axis=1).astype(np.uint32)
        neg = np.concatenate([neg, cand])[:h]
    return src[keep], dst[keep], pos, neg
