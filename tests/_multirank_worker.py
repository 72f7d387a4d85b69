"""Worker of tests/test_multirank_gloo.py: one rank of the multi-rank path on
CPU, world_size ranks over torch.distributed (gloo, 127.0.0.1).

Block math comes from the oracle (test infrastructure); the SCHEDULE comes
from the product's host code, gv_plan_step in libgv.so (no GPU needed): which
blocks a rank trains at each offset step, which context partition it sends
after its first block and to whom, which one it receives and which block
waits for it. The communication is real (gloo point-to-point), in the order
the engine uses: block-row exchange of the bucketed pool, then per step
"train block 0 -> send; receive before block wait_block of the next step".
Rank 0 gathers the result and compares it with the serial oracle bit for bit.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(rank, world, port, n, pools, count, out_path, vtile=0):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    import synth
    from oracle import oracle as O
    from paper_1903_00757_b200 import gv as G

    dist.init_process_group("gloo", rank=rank, world_size=world)
    nv, ne, d = 1500, 7000, 16
    src, dst = synth.chung_lu(nv, ne, gamma=2.1, wmax=150.0, seed=1)
    total = pools * count
    mine = O.Trainer(nv, d, n, K=2, lr0=0.05, lr_kind=1, total_samples=total)
    mine.load_edges(src, dst)
    perm, off = mine.partition()
    inv = np.argsort(perm)
    m = n // world
    rows = lambda p: inv[int(off[p]):int(off[p + 1])]  # noqa: E731  original ids of partition p
    s_before = 0

    def send_rows(arr, p, to):
        dist.send(torch.from_numpy(np.ascontiguousarray(arr[rows(p)])), dst=to)

    def recv_rows(p, frm):
        buf = torch.empty((len(rows(p)), d), dtype=torch.float32)
        dist.recv(buf, src=frm)
        return buf.numpy()

    for e in range(pools):
        pool = synth.edge_pool(src, dst, count, seed=500 + e)
        seg = pool[count * rank // world: count * (rank + 1) // world]
        # a3-a5 on the rank's segment, then counts all-gather (n^2 per rank)
        lp, boff = O.bucket(seg, nv, perm, off, n)
        cnt = torch.from_numpy(np.diff(boff.astype(np.int64)))
        allc = [torch.zeros_like(cnt) for _ in range(world)]
        dist.all_gather(allc, cnt)
        allc = np.stack([c.numpy() for c in allc])  # [rank, bin]
        # a6: rank s sends its sub-blocks of rows [d m, (d+1) m) to rank d
        # (pairwise, the lower rank sends first)
        chunks = {}
        for q in range(world):
            b0, b1 = int(boff[q * m * n]), int(boff[(q + 1) * m * n])
            out = np.ascontiguousarray(lp[b0:b1]).astype(np.int64)
            if q == rank:
                chunks[q] = out
                continue
            size = int(allc[q, rank * m * n:(rank + 1) * m * n].sum())
            buf = torch.empty((size, 2), dtype=torch.int64)
            if rank < q:
                dist.send(torch.from_numpy(out), dst=q)
                dist.recv(buf, src=q)
            else:
                dist.recv(buf, src=q)
                dist.send(torch.from_numpy(out), dst=q)
            chunks[q] = buf.numpy()
        # block (i, j) of my rows = concatenation over source ranks
        blocks = {}
        for gi in range(m):
            i = rank * m + gi
            for j in range(n):
                parts = []
                for s_ in range(world):
                    c_s = allc[s_]
                    base = int(c_s[rank * m * n:i * n + j].sum())
                    parts.append(chunks[s_][base:base + int(c_s[i * n + j])])
                blk = np.concatenate(parts).astype(np.uint32)
                if vtile:  # R-VTILE: the owner orders its block by vertex tile after the exchange
                    blk = blk[np.argsort(blk[:, 0] >> vtile, kind="stable")]
                blocks[(i, j)] = blk
        glob = allc.sum(0)
        # a7/a8 with the product's plan
        pending = None  # (partition, source) received for the next step
        for t in range(n):
            lr = O.lr(1, float(np.float32(0.05)), 1e-4, s_before, total)  # lr0 is a float (gv_create)
            plan = G.gv_plan_step(n, world, rank, t)
            assert [b[0] for b in plan["blocks"]] == list(range(rank * m, rank * m + m))
            for g, (i, j) in enumerate(plan["blocks"]):
                if g == plan["wait_block"] and pending is not None:
                    p, frm, arr = pending
                    C = mine.get("context")
                    C[rows(p)] = arr
                    mine.set("context", C)
                    pending = None
                mine.train_block(blocks[(i, j)], i, j, e, lr)
                if g == 0 and plan["send_part"] is not None:
                    # exchange with neighbours: even ranks send first
                    C = mine.get("context")
                    if rank % 2 == 0:
                        send_rows(C, plan["send_part"], plan["send_to"])
                        arr = recv_rows(plan["recv_part"], plan["recv_from"])
                    else:
                        arr = recv_rows(plan["recv_part"], plan["recv_from"])
                        send_rows(C, plan["send_part"], plan["send_to"])
                    pending = (plan["recv_part"], plan["recv_from"], arr)
            s_before += int(sum(glob[i * n + (i + t) % n] for i in range(n)))
        if pending is not None:  # the last rotation of the pool restores the window
            p, frm, arr = pending
            C = mine.get("context")
            C[rows(p)] = arr
            mine.set("context", C)
    # gather owned rows on rank 0
    V, C = mine.get("vertex"), mine.get("context")
    owned = np.concatenate([rows(p) for p in range(rank * m, rank * m + m)])
    if rank == 0:
        for q in range(1, world):
            ids = torch.empty(0, dtype=torch.int64)
            sz = torch.zeros(1, dtype=torch.int64)
            dist.recv(sz, src=q)
            ids = torch.empty(int(sz), dtype=torch.int64)
            dist.recv(ids, src=q)
            vb = torch.empty((int(sz), d), dtype=torch.float32)
            cb = torch.empty((int(sz), d), dtype=torch.float32)
            dist.recv(vb, src=q)
            dist.recv(cb, src=q)
            V[ids.numpy()] = vb.numpy()
            C[ids.numpy()] = cb.numpy()
        np.savez(out_path, vertex=V, context=C)
    else:
        dist.send(torch.tensor([len(owned)], dtype=torch.int64), dst=0)
        dist.send(torch.from_numpy(owned.astype(np.int64)), dst=0)
        dist.send(torch.from_numpy(np.ascontiguousarray(V[owned])), dst=0)
        dist.send(torch.from_numpy(np.ascontiguousarray(C[owned])), dst=0)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    r, w, port, n, pools, count, out = sys.argv[1:8]
    vt = int(sys.argv[8]) if len(sys.argv) > 8 else 0
    main(int(r), int(w), int(port), int(n), int(pools), int(count), out, vt)
