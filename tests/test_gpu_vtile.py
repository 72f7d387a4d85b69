"""GPU parity of the vertex-tile order (reading R-VTILE, gv_options.vertex_tile):
the blocks after bucketing, the exchange and the tile sort equal the oracle's
or_bucket_tiled byte for byte (one, two and three radix passes, original and
relabelled ids, the fused multi-rank exchange, ragged and empty blocks), and
ordered-mode training over tiled blocks equals the oracle trainer with the
same vertex_tile within R-TOL. Hogwild quality with tiles is checked against
the UNTILED oracle in test_gpu_parity.test_hogwild_auc_matches_oracle."""
import numpy as np
import pytest

import synth
from _parity import assert_matrix_parity
from oracle import oracle as O

pytestmark = pytest.mark.gpu

from paper_1903_00757_b200 import gv as G  # noqa: E402  (fails loudly if libgv.so is missing)

C1 = synth.CONFIGS["C1"]


def _tiled_case(nv, ne, n, vr, bits, ids, count, seed):
    src, dst = synth.chung_lu(nv, ne, gamma=2.1, wmax=nv / 10, seed=seed)
    pool = synth.edge_pool(src, dst, count, seed=seed + 7)
    g = G.GraphVite(nv, 8, n, 1, 0.025, virtual_ranks=vr, vertex_tile=bits,
                    pool_ids=G.GV_IDS_RELABELED if ids == "relabeled" else G.GV_IDS_ORIGINAL)
    g.load_edges(src, dst)
    perm, _ = g.partition()
    g.push(perm[pool] if ids == "relabeled" else pool)
    G.gv_prepare_episode(g.ctx)
    got, boff = G.gv_debug_get_buckets(g.ctx, n, count)
    o = O.Trainer(nv, 8, n)
    o.load_edges(src, dst)
    operm, off = o.partition()
    exp, eoff = O.bucket_tiled(pool, nv, operm, off, n, bits)
    return g, got, boff, exp, eoff, off


@pytest.mark.parametrize("n,vr,bits,ids,count", [
    (1, 1, 3, "relabeled", 100_003),   # n = 1 swap mode, 250 tiles: one pass + copy back
    (1, 1, 1, "original", 77_777),     # 1000 tiles: two passes
    (1, 1, 12, "relabeled", 5000),     # one tile per partition: the sort is skipped
    (2, 1, 2, "original", 4096 * 3 + 5),
    (4, 1, 4, "relabeled", 123_457),
    (4, 4, 2, "relabeled", 100_001),   # fused exchange, then each owner sorts its blocks
    (8, 8, 1, "original", 64_000),     # empty and tiny blocks
    (16, 4, 3, "relabeled", 200_003),
    (24, 8, 2, "original", 99_999),    # two-pass grid (n >= 17) then tiles
])
def test_vertex_tile_blocks_bitexact(n, vr, bits, ids, count):
    g, got, boff, exp, eoff, _ = _tiled_case(2000, 10_000, n, vr, bits, ids, count, seed=n + vr)
    assert np.array_equal(boff, eoff)
    assert np.array_equal(got, exp)
    g.train_episode(stats=False)
    g.close()


def test_vertex_tile_three_passes_bitexact():
    """More than 65,536 tiles in a partition: three radix passes (an odd
    count, ending in the ping-pong buffer and copied back)."""
    g, got, boff, exp, eoff, off = _tiled_case(300_000, 900_000, 1, 1, 1, "relabeled", 400_001,
                                               seed=3)
    assert (int(off[1]) - 1) >> 1 >= 1 << 16
    assert np.array_equal(boff, eoff)
    assert np.array_equal(got, exp)
    g.close()


def test_vertex_tile_replay_and_range_check():
    """A replayed pool (n = 1 swap mode: the pool lies in the block buffer,
    already in tile order) is sorted again to the same blocks; an
    out-of-range id is still rejected before any update."""
    g, got, boff, exp, eoff, _ = _tiled_case(2000, 10_000, 1, 1, 2, "relabeled", 50_000, seed=9)
    g.train_episode(stats=False)
    g.replay()
    G.gv_prepare_episode(g.ctx)
    again, boff2 = G.gv_debug_get_buckets(g.ctx, 1, 50_000)
    assert np.array_equal(again, exp) and np.array_equal(boff2, eoff)
    g.train_episode(stats=False)
    bad = np.array([[0, 1], [2000, 3]], np.uint32)
    g.push(bad)
    with pytest.raises(G.GVError):
        g.train_episode()
    g.close()


def test_vertex_tile_option_checked():
    with pytest.raises(G.GVError):
        G.GraphVite(100, 8, 1, 1, 0.025, vertex_tile=32)
    with pytest.raises(G.GVError):
        G.GraphVite(100, 8, 1, 1, 0.025, vertex_tile=-1)


@pytest.fixture(scope="module")
def c1_graph():
    src, dst, _ = synth.dcsbm(C1["nv"], C1["ne"], gamma=C1["gamma"], wmax=C1["wmax"], c=C1["c"],
                              mu=C1["mu"], seed=1)
    return src, dst


@pytest.mark.parametrize("n,vr,bits,lr_kind", [(1, 1, 5, 1), (1, 1, 9, 0), (4, 1, 4, 1),
                                               (4, 2, 3, 1), (8, 4, 6, 0)])
def test_vertex_tile_ordered_matches_oracle(c1_graph, n, vr, bits, lr_kind):
    """Ordered mode over tiled blocks = the oracle trainer with the same
    vertex_tile (R-VTILE), two pools, R-TOL per matrix (constant lr in two
    cases, so late samples' updates are as large as early ones)."""
    src, dst = c1_graph
    count, pools = 200_000, 2
    p = G.GraphVite(C1["nv"], 32, n, 1, 0.025, total_samples=pools * count, lr_kind=lr_kind,
                    virtual_ranks=vr, ordered=1, vertex_tile=bits)
    p.load_edges(src, dst)
    o = O.Trainer(C1["nv"], 32, n, K=1, lr0=0.025, lr_kind=lr_kind, total_samples=pools * count,
                  vertex_tile=bits)
    o.load_edges(src, dst)
    for k in range(pools):
        pool = synth.edge_pool(src, dst, count, seed=300 + k)
        p.push(pool)
        st = p.train_episode()
        lo = o.train_pool(pool)
        assert st["samples_global"] == count
        assert abs(st["loss_sum"] - lo) <= 1e-4 * abs(lo)
    assert_matrix_parity(p.vertex(), o.get("vertex"), "vertex")
    assert_matrix_parity(p.context(), o.get("context"), "context")
    p.close()


@pytest.mark.parametrize("n,bits", [(2, 5), (4, 3)])
def test_vertex_tile_out_of_core_matches_oracle(c1_graph, n, bits):
    """Host-resident partitions (NEXT-3) train the same tiled blocks: ordered
    mode equals the oracle trainer with the same vertex_tile."""
    src, dst = c1_graph
    count = 150_000
    p = G.GraphVite(C1["nv"], 32, n, 1, 0.025, total_samples=2 * count, ordered=1,
                    host_partitions=1, vertex_tile=bits)
    p.load_edges(src, dst)
    o = O.Trainer(C1["nv"], 32, n, K=1, lr0=0.025, lr_kind=1, total_samples=2 * count,
                  vertex_tile=bits)
    o.load_edges(src, dst)
    for k in range(2):
        pool = synth.edge_pool(src, dst, count, seed=700 + k)
        p.push(pool)
        p.train_episode()
        o.train_pool(pool)
    assert_matrix_parity(p.vertex(), o.get("vertex"), "vertex")
    assert_matrix_parity(p.context(), o.get("context"), "context")
    p.close()


@pytest.mark.parametrize("n,K,d,host_pool", [(1, 3, 64, 1), (4, 2, 128, 0), (2, 5, 256, 1)])
def test_vertex_tile_shapes_and_host_pool(c1_graph, n, K, d, host_pool):
    """Tiled blocks with K > 1 negatives, d up to 256 (the full-warp kernel
    above 128) and the raw pool in pinned host memory: ordered mode
    equals the oracle trainer with the same vertex_tile."""
    src, dst = c1_graph
    count = 120_000
    p = G.GraphVite(C1["nv"], d, n, K, 0.025, total_samples=count, ordered=1,
                    neg_weight=5.0 / K, host_pool=host_pool, vertex_tile=4)
    p.load_edges(src, dst)
    o = O.Trainer(C1["nv"], d, n, K=K, lr0=0.025, lr_kind=1, total_samples=count,
                  neg_weight=5.0 / K, vertex_tile=4)
    o.load_edges(src, dst)
    pool = synth.edge_pool(src, dst, count, seed=900 + n)
    p.push(pool)
    st = p.train_episode()
    lo = o.train_pool(pool)
    assert abs(st["loss_sum"] - lo) <= 1e-4 * abs(lo)
    assert_matrix_parity(p.vertex(), o.get("vertex"), "vertex")
    assert_matrix_parity(p.context(), o.get("context"), "context")
    p.close()
