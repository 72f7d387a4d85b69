"""Experiment (measurement only): L2 blocking along the vertex dimension.

Sorts the bench's C5 pool stably by u >> shift (vertex-row tiles of 2^shift
relabelled rows) before pushing it, and measures the SGD kernel on it. At
n = 1 with relabelled ids the pool is trained in push order, so this shows
what ordering the samples of a block by vertex tile buys on the Friendster-
shaped graph (each tile's vertex rows stay in L2 while its samples run).

  python tools/exp_vtile.py [--config C5] [--shifts none,14,16,18]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--shifts", default="none,14,15,16,17,18")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--pool", type=int, default=0)
    a = ap.parse_args()
    import torch

    from paper_1903_00757_b200 import gv as G
    bench.set_config(a.config)
    if a.pool:
        bench.CFG["pool"] = a.pool
    CFG = bench.CFG
    t0 = time.perf_counter()
    src, dst = bench.make_graph()
    P = CFG["pool"]
    g = G.GraphVite(CFG["nv"], CFG["d"], 1, CFG["K"], CFG["lr"], total_samples=P * 100,
                    neg_weight=CFG["neg_weight"], seed=CFG["seed"], device=0,
                    pool_ids=G.GV_IDS_RELABELED)
    g.load_edges(src, dst)
    del src, dst
    host = torch.empty((P, 2), dtype=torch.int32, pin_memory=True)
    g.augment(CFG["walk"], CFG["s"], os.cpu_count() or 16, P, 1000, out=host)
    orig = host.clone()
    print(f"setup {time.perf_counter() - t0:.0f} s", file=sys.stderr, flush=True)
    out = {"config": a.config, "pool": P, "runs": []}
    for sh in a.shifts.split(","):
        if sh == "none":
            host.copy_(orig)
        else:
            dev = orig.cuda()
            key = (dev[:, 0] >> int(sh)).to(torch.int64)
            idx = torch.sort(key, stable=True).indices
            host.copy_(dev[idx].cpu())
            del dev, key, idx
            torch.cuda.empty_cache()
        g.push(host)
        g.train_episode()
        ms, loss = [], []
        for _ in range(a.steps):
            g.replay()
            st = g.train_episode()
            ms.append(st["ms_sgd"])
            loss.append(st["loss_sum"] / max(st["samples_global"], 1))
        r = {"shift": sh, "ms_sgd": ms, "samples_per_s": P / (min(ms) / 1e3),
             "alg_gbs": P * 3072 / (min(ms) / 1e3) / 1e9, "loss_per_sample": loss}
        out["runs"].append(r)
        print(json.dumps(r), file=sys.stderr, flush=True)
    g.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
