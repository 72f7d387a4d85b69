"""Multi-rank path on CPU: world_size 2 over torch.distributed (gloo).

Two processes execute the product's schedule (gv_plan_step, host code of
libgv.so) with real point-to-point messages for the block-row exchange and
the context rotation; the block math is the oracle's. Because every row sees
the same update sequence as in the serial Alg. 3 loop (blocks of one offset
step are orthogonal), the gathered embeddings must equal the
serial oracle's BIT FOR BIT."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import synth
from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("n,pools,count,vt", [(2, 2, 30_000, 0), (4, 2, 40_001, 0),
                                              (8, 1, 50_000, 0), (4, 2, 40_001, 3), (2, 1, 30_000, 6)])
def test_two_ranks_match_serial_oracle_bitwise(tmp_path, n, pools, count, vt):
    """vt > 0 (R-VTILE): each owner orders its blocks by vertex tile after the
    block-row exchange — as the engine does — and the result must equal the
    serial oracle trainer with the same vertex_tile, bit for bit."""
    world = 2
    port = _free_port()
    out = str(tmp_path / "res.npz")
    worker = os.path.join(ROOT, "tests", "_multirank_worker.py")
    procs = [subprocess.Popen([sys.executable, worker, str(r), str(world), str(port), str(n),
                               str(pools), str(count), out, str(vt)]) for r in range(world)]
    for p in procs:
        assert p.wait(timeout=300) == 0
    res = np.load(out)
    # serial oracle, same graph, pools and hyper-parameters
    nv, ne, d = 1500, 7000, 16
    src, dst = synth.chung_lu(nv, ne, gamma=2.1, wmax=150.0, seed=1)
    o = O.Trainer(nv, d, n, K=2, lr0=0.05, lr_kind=1, total_samples=pools * count, vertex_tile=vt)
    o.load_edges(src, dst)
    for e in range(pools):
        o.train_pool(synth.edge_pool(src, dst, count, seed=500 + e))
    assert np.array_equal(res["vertex"], o.get("vertex"))
    assert np.array_equal(res["context"], o.get("context"))
    assert np.abs(res["vertex"]).sum() > 0 and np.abs(res["context"]).sum() > 0


@pytest.mark.parametrize("n,D", [(1, 1), (4, 1), (4, 2), (4, 4), (8, 2), (6, 3), (64, 8)])
def test_plan_covers_grid_and_ring_is_consistent(n, D):
    """gv_plan_step: every offset step is orthogonal across ranks, n steps
    cover all n^2 blocks once (Alg. 3), the partition a rank receives
    is the one its successor sends, and it is the context of the waiting
    block of the next step."""
    from paper_1903_00757_b200 import gv as G
    m = n // D
    seen = set()
    for t in range(n):
        plans = [G.gv_plan_step(n, D, d, t) for d in range(D)]
        blocks = [b for p in plans for b in p["blocks"]]
        assert sorted(i for i, _ in blocks) == list(range(n))
        assert sorted(j for _, j in blocks) == list(range(n))
        assert all(j == (i + t) % n for i, j in blocks)
        seen |= set(blocks)
        if D == 1:
            assert plans[0]["send_part"] is None
            continue
        for d, p in enumerate(plans):
            assert p["send_part"] == p["blocks"][0][1]
            succ = plans[p["recv_from"]]
            assert succ["send_to"] == d and succ["send_part"] == p["recv_part"]
            nxt = G.gv_plan_step(n, D, d, (t + 1) % n)
            assert nxt["blocks"][p["wait_block"]][1] == p["recv_part"]
            # the window after the rotation = contexts of the next step
            window = {j for _, j in p["blocks"]} - {p["send_part"]} | {p["recv_part"]}
            assert window == {j for _, j in nxt["blocks"]}
    assert len(seen) == n * n
    with pytest.raises(G.GVError):
        G.gv_plan_step(n, D, D, 0)
