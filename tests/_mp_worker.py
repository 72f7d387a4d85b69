"""Worker of tests/test_gpu_multiprocess.py: rank `rank` of `world` PROCESSES
sharing cuda:0, multi-process path of libgv.so (CUDA-IPC transport). Pushes
its segment of each pool, trains, writes the rows it owns."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def graph(kind, nv, ne):
    """kind 0: the Chung-Lu test graph; kind 1: the training edges of the
    link-prediction split of the AUC-parity DC-SBM graph (the graph of
    test_gpu_parity.test_hogwild_auc_matches_oracle)."""
    import synth
    if kind == 0:
        return synth.chung_lu(nv, ne, gamma=2.1, wmax=400.0, seed=11)
    src, dst, _ = synth.dcsbm(nv, ne, gamma=2.1, wmax=1000.0, c=50, mu=0.1, seed=1)
    tr_s, tr_d, _, _ = synth.linkpred_split(src, dst, nv, holdout=0.01, seed=6)
    return tr_s, tr_d


def main(rank, world, uid_hex, n, pools, count, ordered, out, nv=4000, ne=20_000, grow=0, aug=0,
         kind=0, relabeled=0, vtile=0):
    import synth
    from paper_1903_00757_b200 import gv as G
    d = 32 if kind == 0 else 128
    src, dst = graph(kind, nv, ne)
    sizes = [count * (4 ** e if grow else 1) for e in range(pools)]  # grow: receive buffers realloc
    g = G.GraphVite(nv, d, n, 1, 0.025, total_samples=sum(sizes), rank=rank, world_size=world,
                    ordered=ordered,
                    pool_ids=G.GV_IDS_RELABELED if relabeled else G.GV_IDS_ORIGINAL,
                    vertex_tile=vtile)
    G.gv_comm_init(g.ctx, bytes.fromhex(uid_hex))
    g.load_edges(src, dst)
    perm, _ = g.partition()
    losses = []
    for e in range(pools):
        cnt = sizes[e]
        if aug:  # this rank's pool segment, augmented on its own GPU (NEXT-1)
            seg = cnt * (rank + 1) // world - cnt * rank // world
            g.augment_device(40, 2, 16, seg, 500 + 1000 * e + rank)
        else:
            pool = synth.edge_pool(src, dst, cnt, seed=(900 if kind == 0 else 200) + e)
            seg = pool[cnt * rank // world: cnt * (rank + 1) // world]
            g.push(perm[seg] if relabeled else seg)
        st = g.train_episode()
        losses.append(st["loss_sum"])
        assert st["samples_global"] == cnt, st
    V, C = g.vertex(), g.context()
    perm, off = g.partition()
    m = n // world
    owned = np.flatnonzero((perm >= off[rank * m]) & (perm < off[(rank + 1) * m]))
    np.savez(out, ids=owned, vertex=V[owned], context=C[owned], loss=np.array(losses))
    g.close()


if __name__ == "__main__":
    a = sys.argv[1:]
    main(int(a[0]), int(a[1]), a[2], int(a[3]), int(a[4]), int(a[5]), int(a[6]), a[7],
         *(int(x) for x in a[8:15]))
