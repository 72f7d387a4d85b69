"""Small workload touching every kernel once, for compute-sanitizer
(memcheck / racecheck / synccheck). Not a test by itself: the sanitizer's
exit code is the verdict."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synth  # noqa: E402
from paper_1903_00757_b200 import gv as G  # noqa: E402

src, dst = synth.chung_lu(3000, 15_000, gamma=2.1, wmax=300.0, seed=1)
pool = synth.edge_pool(src, dst, 50_003, seed=3)
# (16, 4, 0): two-pass bucketing into the virtual ranks' buffers
for n, vr, ordered in [(1, 1, 0), (4, 1, 0), (4, 2, 0), (4, 2, 1), (2, 1, 1), (16, 4, 0), (16, 1, 1)]:
    g = G.GraphVite(3000, 128, n, 1, 0.025, total_samples=200_000, virtual_ranks=vr,
                    ordered=ordered)
    g.load_edges(src, dst)
    g.push(pool)
    G.gv_prepare_episode(g.ctx)
    G.gv_debug_get_negatives(g.ctx, 0, 0, 1, 1) if False else None
    g.train_episode()
    g.replay()
    g.train_episode()
    assert np.isfinite(g.vertex()).all()
    g.close()
for n in (3, 5):  # out-of-core: three slots, load / write-back streams, paired-step order
    g = G.GraphVite(3000, 128, n, 1, 0.025, host_partitions=1)
    g.load_edges(src, dst)
    for _ in range(2):
        g.push(pool)
        g.train_episode()
    assert np.isfinite(g.vertex()).all()
    g.close()
g = G.GraphVite(3000, 64, 1, 3, 0.025)
g.load_edges(src, dst)
g.augment_device(10, 3, 37, 20_011, 5)
g.train_episode()
for mode in (G.GV_SHUFFLE_NONE, G.GV_SHUFFLE_RANDOM):
    g.augment_device(10, 3, 37, 20_011, 6, shuffle=mode)
    g.train_episode()
G.gv_train_explicit(g.ctx, [0, 1], [2, 3], [[4, 5, 6], [7, 7, 2]], 0.1)
g.close()
# round 2: relabelled pools (n = 1: range check only, raw and block buffers
# swap; n = 4 / 16: partition from the offsets), and the sampler writing
# blocks directly (count pass, tile scans, placement)
for n, vr in [(1, 1), (4, 1), (16, 4)]:
    g = G.GraphVite(3000, 128, n, 1, 0.025, total_samples=200_000, virtual_ranks=vr,
                    pool_ids=G.GV_IDS_RELABELED)
    g.load_edges(src, dst)
    perm, _ = g.partition()
    g.push(perm[pool])
    g.train_episode()
    g.push(perm[pool])  # overlaps the first pool's training
    g.train_episode()
    g.replay()
    g.train_episode()
    assert np.isfinite(g.vertex()).all()
    g.close()
for n, ids in [(1, G.GV_IDS_ORIGINAL), (4, G.GV_IDS_RELABELED), (16, G.GV_IDS_ORIGINAL)]:
    g = G.GraphVite(3000, 64, n, 1, 0.025, pool_ids=ids)
    g.load_edges(src, dst)
    g.augment_device_blocks(10, 3, 37, 20_011, 7)
    g.train_episode()
    g.augment_device_blocks(10, 3, 37, 20_011, 8, shuffle=G.GV_SHUFFLE_NONE)
    g.train_episode()
    assert np.isfinite(g.vertex()).all()
    g.close()
# round 2: vertex-tile order (R-VTILE): one pass + copy back (n = 1 swap
# mode, 2^4-row tiles of 3000 rows: 188 tiles), two passes (2^1 rows), after
# the fused exchange (n = 4 on 2 virtual ranks); the dynamic chunk schedule
# of the ring kernel runs in every Hogwild episode above
for n, vr, bits, ids in [(1, 1, 4, G.GV_IDS_RELABELED), (1, 1, 1, G.GV_IDS_ORIGINAL),
                         (4, 2, 2, G.GV_IDS_RELABELED)]:
    g = G.GraphVite(3000, 128, n, 1, 0.025, total_samples=200_000, virtual_ranks=vr,
                    vertex_tile=bits, pool_ids=ids)
    g.load_edges(src, dst)
    perm, _ = g.partition()
    g.push(perm[pool] if ids == G.GV_IDS_RELABELED else pool)
    g.train_episode()
    g.replay()
    g.train_episode()
    assert np.isfinite(g.vertex()).all()
    g.close()
print("sanitize drive ok")
