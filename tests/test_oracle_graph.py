"""Oracle pins, part 2: ingest, zig-zag partition, bucketing (SURVEY §8(c)
steps 1, 2, 6). CPU only."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import oracle as O
import synth


def test_ingest_triangle_and_duplicates():
    """triangle -> 3 edges, all degrees 2; 'a b 2.0' + 'b a 3.0' ->
    one undirected edge of weight 5; self-loops dropped."""
    g = O.Graph(3, [0, 1, 2], [1, 2, 0])
    off, nbr, w = g.csr()
    assert len(nbr) == 6 and list(g.degree()) == [2, 2, 2]
    g = O.Graph(3, [0, 1, 2], [1, 0, 2], np.array([2.0, 3.0, 9.0], np.float32))
    off, nbr, w = g.csr()
    assert list(off) == [0, 1, 2, 2] and list(nbr) == [1, 0] and list(w) == [5.0, 5.0]
    assert list(g.degree()) == [5.0, 5.0, 0.0]


def test_ingest_errors():
    with pytest.raises(O.OracleError):
        O.Graph(3, [0, 1], [1, 3])            # out of range
    with pytest.raises(O.OracleError):
        O.Graph(3, [0], [1], np.array([-1.0], np.float32))
    with pytest.raises(O.OracleError):
        O.Graph(3, [1, 2], [1, 2])            # only self-loops -> empty


def test_ingest_matches_scipy_symmetrisation():
    """Library routine special case: CSR of A + A^T with duplicates summed and
    the diagonal removed (scipy.sparse) equals the oracle's CSR; degree
    conservation sum(deg) = 2 sum(w)."""
    rng = np.random.default_rng(0)
    nv, ne = 300, 2000
    src = rng.integers(0, nv, ne).astype(np.uint32)
    dst = rng.integers(0, nv, ne).astype(np.uint32)
    w = rng.integers(1, 5, ne).astype(np.float32)  # dyadic: exact sums in any order
    g = O.Graph(nv, src, dst, w)
    off, nbr, ww = g.csr()
    keep = src != dst
    A = sp.coo_matrix((w[keep].astype(np.float64), (src[keep], dst[keep])), shape=(nv, nv))
    S = (A + A.T).tocsr()
    S.sum_duplicates()
    S.sort_indices()
    assert np.array_equal(off, S.indptr.astype(np.uint64))
    assert np.array_equal(nbr, S.indices.astype(np.uint32))
    assert np.array_equal(ww, S.data)
    deg = g.degree()
    assert np.array_equal(deg, np.asarray(S.sum(axis=1)).ravel())
    assert deg.sum() == 2 * w[keep].astype(np.float64).sum()


def test_zigzag_worked_example(golden):
    """S:196 [PAPER] fig:zig-zag_partition."""
    ex = golden("zigzag_8.json")
    perm, inv, off = O.zigzag(ex["degrees"], ex["n"])
    for p, members in enumerate(ex["parts"]):
        got = sorted(int(inv[q]) for q in range(int(off[p]), int(off[p + 1])))
        assert got == members


@pytest.mark.parametrize("seed", range(10))
def test_zigzag_invariants(seed):
    """S:210 balance |size_i - size_j| <= 1; perm is a bijection; within a
    partition local order is degree-descending (ties by id); the boustrophedon
    rule holds against an independent brute-force assignment."""
    rng = np.random.default_rng(seed)
    nv = int(rng.integers(5, 400))
    n = int(rng.integers(1, min(nv, 17) + 1))
    deg = rng.integers(0, 20, nv).astype(np.float64)
    perm, inv, off = O.zigzag(deg, n)
    sizes = np.diff(off.astype(np.int64))
    assert sizes.max() - sizes.min() <= 1
    assert np.array_equal(np.sort(perm), np.arange(nv))
    assert np.array_equal(perm[inv], np.arange(nv))
    order = sorted(range(nv), key=lambda v: (-deg[v], v))
    pattern = list(range(n)) + list(range(n - 1, -1, -1))
    expect_part = {v: pattern[r % (2 * n)] for r, v in enumerate(order)}
    for p in range(n):
        members = [int(inv[q]) for q in range(int(off[p]), int(off[p + 1]))]
        assert all(expect_part[v] == p for v in members)
        assert members == sorted(members, key=lambda v: (-deg[v], v))


def test_zigzag_degree_mass_balance():
    """S:190 (DERIVED): per-part total degree within 25% on a 10^4-node power-law graph."""
    src, dst = synth.chung_lu(10_000, 50_000, gamma=2.1, wmax=300.0, seed=1)
    deg = O.Graph(10_000, src, dst).degree()
    for n in (2, 4, 8):
        perm, inv, off = O.zigzag(deg, n)
        mass = [deg[inv[int(off[p]):int(off[p + 1])]].sum() for p in range(n)]
        assert max(mass) / min(mass) < 1.25


@pytest.mark.parametrize("n,count", [(1, 0), (1, 1000), (2, 999), (4, 4097), (8, 20000), (3, 12345)])
def test_bucket_is_stable_counting_sort(n, count):
    """Library routine special case: bucketing == numpy stable argsort by
    bin = part(u) n + part(v); conservation; membership."""
    rng = np.random.default_rng(n * 1000 + count)
    nv = 1000
    deg = rng.integers(1, 50, nv).astype(np.float64)
    perm, inv, off = O.zigzag(deg, n)
    pool = synth.uniform_pool(nv, count, seed=count)
    out, boff = O.bucket(pool, nv, perm, off, n)
    assert boff[-1] == count
    new = perm[pool] if count else np.zeros((0, 2), np.uint32)
    part = np.searchsorted(off[1:], new, side="right")
    bins = part[:, 0] * n + part[:, 1]
    order = np.argsort(bins, kind="stable")
    local = new - off[part].astype(np.uint32)
    assert np.array_equal(out, local[order])
    assert np.array_equal(boff, np.concatenate([[0], np.cumsum(np.bincount(bins, minlength=n * n))]))


def test_bucket_spec_example():
    """2 nodes in different parts, pool [(0,1),(1,0),(0,1)] ->
    block(0,1)=[(0,1),(0,1)], block(1,0)=[(1,0)]."""
    perm, inv, off = O.zigzag([2.0, 1.0], 2)
    out, boff = O.bucket([[0, 1], [1, 0], [0, 1]], 2, perm, off, 2)
    assert list(boff) == [0, 0, 2, 3, 3]
    assert out.tolist() == [[0, 0], [0, 0], [0, 0]]  # local ids: each part has one node


def test_bucket_range_error():
    perm, inv, off = O.zigzag([1.0, 1.0], 1)
    with pytest.raises(O.OracleError):
        O.bucket([[0, 2]], 2, perm, off, 1)
