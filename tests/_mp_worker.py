"""Worker of tests/test_gpu_multiprocess.py: rank `rank` of `world` PROCESSES
sharing cuda:0, multi-process path of libgv.so (CUDA-IPC transport). Pushes
its segment of each pool, trains, writes the rows it owns."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(rank, world, uid_hex, n, pools, count, ordered, out, nv=4000, ne=20_000, grow=0, aug=0):
    import synth
    from paper_1903_00757_b200 import gv as G
    d = 32
    src, dst = synth.chung_lu(nv, ne, gamma=2.1, wmax=400.0, seed=11)
    sizes = [count * (4 ** e if grow else 1) for e in range(pools)]  # grow: receive buffers realloc
    g = G.GraphVite(nv, d, n, 1, 0.025, total_samples=sum(sizes), rank=rank, world_size=world,
                    ordered=ordered, transport=0)
    G.gv_comm_init(g.ctx, bytes.fromhex(uid_hex))
    g.load_edges(src, dst)
    losses = []
    for e in range(pools):
        cnt = sizes[e]
        if aug:  # this rank's pool segment, augmented on its own GPU (NEXT-1)
            seg = cnt * (rank + 1) // world - cnt * rank // world
            g.augment_device(40, 2, 16, seg, 500 + 1000 * e + rank)
        else:
            pool = synth.edge_pool(src, dst, cnt, seed=900 + e)
            g.push(pool[cnt * rank // world: cnt * (rank + 1) // world])
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
         *(int(x) for x in a[8:12]))
