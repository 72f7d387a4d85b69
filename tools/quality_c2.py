"""Link-prediction quality at the bench scale (C2, Youtube-shaped, 1.14 M
nodes): the Hogwild GPU path with n = 1, 4 and 8 partitions on one GPU, on
the same held-out edges, pools augmented on the GPU (walk 40, s = 5). GPU
against GPU (the oracle is too slow at this size): embeddings stay finite
over the whole run and the partition grid keeps the quality of the n = 1
run at full size (fig:episode_size). Writes one JSON line to stdout.
(It is also the run that exposed the divergence of the withdrawn hot-row
combining, profiles/README.md.)

    python tools/quality_c2.py [pools] [dcsbm|chung_lu] [vertex_tile]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from sklearn.metrics import roc_auc_score  # noqa: E402

import synth  # noqa: E402
from paper_1903_00757_b200 import gv as G  # noqa: E402

NV, NE = 1_138_499, 4_945_382
POOL = 200_000_000


def auc(V, pos, neg):
    """cosine of the vertex rows of each pair (R-AUC), ROC AUC positives vs negatives"""
    Vn = V / np.maximum(np.linalg.norm(V, axis=1, keepdims=True), 1e-12)

    def score(p):
        return np.einsum("ij,ij->i", Vn[p[:, 0]], Vn[p[:, 1]])
    y = np.r_[np.ones(len(pos)), np.zeros(len(neg))]
    return float(roc_auc_score(y, np.r_[score(pos), score(neg)]))


def main():
    pools = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    kind = sys.argv[2] if len(sys.argv) > 2 else "dcsbm"
    vt = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # R-VTILE: blocks in vertex-tile order
    if kind == "dcsbm":  # C2's size and degree shape with 200 communities (mu = 0.1)
        src, dst, _ = synth.dcsbm(NV, NE, gamma=2.1, wmax=3e4, c=200, mu=0.1, seed=1)
    else:  # the bench graph: no community structure, so link prediction is near chance
        src, dst = synth.chung_lu(NV, NE, gamma=2.1, wmax=3e4, seed=1)
    tr_s, tr_d, pos, neg = synth.linkpred_split(src, dst, NV, holdout=0.01, seed=6)
    out = {"workload": f"C2-sized {kind} graph, 1% held out, walk 40, s=5, GPU augmentation",
           "pools": pools, "samples": pools * POOL, "vertex_tile": vt, "runs": {}}
    for name, n in [("n1", 1), ("n4", 4), ("n8", 8)]:
        g = G.GraphVite(NV, 128, n, 1, 0.025, total_samples=pools * POOL, ordered=0, vertex_tile=vt)
        g.load_edges(tr_s, tr_d)
        t0 = time.time()
        st = None
        for k in range(pools):
            g.augment_device(40, 5, 1184, POOL, 1000 + k)
            st = g.train_episode()
            print(name, k, st["loss_sum"] / POOL, file=sys.stderr, flush=True)
        V = g.vertex()
        if not np.isfinite(V).all():
            raise SystemExit(f"{name}: non-finite embeddings ({int((~np.isfinite(V)).sum())} values)")
        out["runs"][name] = {"auc": auc(V, pos, neg),
                             "loss_last_pool": st["loss_sum"] / POOL, "wall_s": time.time() - t0}
        g.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
