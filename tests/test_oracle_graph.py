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


def test_ingest_sums_duplicates_in_input_order():
    """R-INGEST: duplicate weights are summed in INPUT order (double). With a
    weight of 2^24 and 1024 weights of 2^-30 on the same undirected edge the
    order is visible in double: small ones first gives 2^24 + 2^-20 exactly,
    the big one first absorbs every small one. The edge appears in both
    directions with the same sum, and degree = that sum."""
    big, small = np.float32(2.0 ** 24), np.float32(2.0 ** -30)
    for first_big in (False, True):
        ws = [small] * 1024 + [big]
        if first_big:
            ws = [big] + [small] * 1024
        src = np.array([0, 1] * 512 + [0], np.uint32)  # both orientations of 0-1
        dst = np.array([1, 0] * 512 + [1], np.uint32)
        if first_big:
            src, dst = np.r_[src[-1:], src[:-1]], np.r_[dst[-1:], dst[:-1]]
        src = np.r_[src, [2]].astype(np.uint32)        # a second edge 1-2 so node 2 exists
        dst = np.r_[dst, [1]].astype(np.uint32)
        w = np.r_[np.array(ws, np.float32), [np.float32(1.0)]]
        off, nbr, wt = O.Graph(3, src, dst, w).csr()
        want = 2.0 ** 24 if first_big else 2.0 ** 24 + 2.0 ** -20
        assert list(nbr[off[0]:off[1]]) == [1] and wt[off[0]] == want
        assert wt[off[1]] == want and O.Graph(3, src, dst, w).degree()[0] == want


def test_sampler_over_trainer_graph_equals_fresh_graph():
    """Trainer.sampler() walks the trainer's own ingested graph: the pool is
    the one a Sampler over a separately ingested Graph produces."""
    src, dst = synth.chung_lu(2000, 10_000, gamma=2.1, wmax=200.0, seed=3)
    t = O.Trainer(2000, 8, 2)
    t.load_edges(src, dst)
    a = t.sampler().augment(40, 3, 5, 20_000, 11)
    b = O.Sampler(O.Graph(2000, src, dst)).augment(40, 3, 5, 20_000, 11)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("n,count,bits", [(1, 0, 3), (1, 5000, 1), (1, 5000, 4), (2, 4999, 2),
                                          (3, 12345, 5), (4, 20000, 3), (8, 20000, 9)])
def test_bucket_tiled_is_stable_sort_by_block_then_tile(n, count, bits):
    """R-VTILE pinned to a library routine: or_bucket_tiled == numpy's stable
    lexsort of the relabelled pool by (block = part(u) n + part(v), vertex
    tile = local(u) >> bits) — pool order inside a (block, tile) — with the
    block offsets of plain bucketing; each block's multiset is unchanged."""
    rng = np.random.default_rng(n * 7919 + count + bits)
    nv = 1000
    deg = rng.integers(1, 50, nv).astype(np.float64)
    perm, inv, off = O.zigzag(deg, n)
    pool = synth.uniform_pool(nv, count, seed=count + 1)
    out, boff = O.bucket_tiled(pool, nv, perm, off, n, bits)
    plain, boff0 = O.bucket(pool, nv, perm, off, n)
    assert np.array_equal(boff, boff0)
    new = perm[pool] if count else np.zeros((0, 2), np.uint32)
    part = np.searchsorted(off[1:], new, side="right")
    local = new - off[part].astype(np.uint32)
    bins = part[:, 0] * n + part[:, 1]
    order = np.lexsort((local[:, 0] >> bits, bins))  # last key primary; stable
    assert np.array_equal(out, local[order])
    for b in range(n * n):
        blk, ref = out[boff[b]:boff[b + 1]], plain[boff0[b]:boff0[b + 1]]
        assert np.all(np.diff(blk[:, 0] >> bits) >= 0)  # tiles ascending inside a block
        assert sorted(map(tuple, blk)) == sorted(map(tuple, ref))


def test_bucket_tiled_special_cases():
    """tile_bits = 0 is plain bucketing; tiles at least as large as every
    partition leave each block in pool order (again plain bucketing); one-row
    tiles sort each block by local vertex id, stably; bits > 31 is rejected."""
    nv, n = 700, 3
    rng = np.random.default_rng(5)
    perm, inv, off = O.zigzag(rng.integers(1, 30, nv).astype(np.float64), n)
    pool = synth.uniform_pool(nv, 9000, seed=11)
    plain, b0 = O.bucket(pool, nv, perm, off, n)
    for bits in (0, 9, 31):  # 2^9 = 512 >= every partition (~234 rows)
        out, b = O.bucket_tiled(pool, nv, perm, off, n, bits)
        assert np.array_equal(out, plain) and np.array_equal(b, b0)
    out, b = O.bucket_tiled(pool, nv, perm, off, n, 1)
    for q in range(n * n):
        blk = out[b[q]:b[q + 1]]
        assert np.all(np.diff(blk[:, 0] >> 1) >= 0)
    # worked example: one partition, tiles of 2 rows, pool (3,0) (0,1) (2,2) (1,3) (0,0)
    perm1, _, off1 = O.zigzag([4.0, 3.0, 2.0, 1.0], 1)  # degree-descending: identity order
    assert list(perm1) == [0, 1, 2, 3]
    out, b = O.bucket_tiled([[3, 0], [0, 1], [2, 2], [1, 3], [0, 0]], 4, perm1, off1, 1, 1)
    assert out.tolist() == [[0, 1], [1, 3], [0, 0], [3, 0], [2, 2]]
    with pytest.raises(O.OracleError):
        O.bucket_tiled(pool, nv, perm, off, n, 32)
