"""Link-prediction quality of the vertex-tile order (reading R-VTILE) on a
larger DC-SBM than the C2-sized one of tools/quality_c2.py: GPU against GPU,
n = 1, pools augmented on the GPU, the same held-out edges for every b
(0 = the paper's pool order). One JSON line to stdout.

    python tools/quality_vtile.py [nv] [ne] [pools] [pool] [b,b,...]
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


def auc(V, pos, neg):
    """cosine of the vertex rows of each pair (R-AUC), ROC AUC positives vs negatives"""
    Vn = V / np.maximum(np.linalg.norm(V, axis=1, keepdims=True), 1e-12)

    def score(p):
        return np.einsum("ij,ij->i", Vn[p[:, 0]], Vn[p[:, 1]])
    y = np.r_[np.ones(len(pos)), np.zeros(len(neg))]
    return float(roc_auc_score(y, np.r_[score(pos), score(neg)]))


def main():
    a = sys.argv[1:]
    nv = int(a[0]) if len(a) > 0 else 7_944_949
    ne = int(a[1]) if len(a) > 1 else 80_000_000
    pools = int(a[2]) if len(a) > 2 else 20
    pool = int(a[3]) if len(a) > 3 else 200_000_000
    bs = [int(x) for x in a[4].split(",")] if len(a) > 4 else [0, 14, 12]
    t0 = time.time()
    src, dst, _ = synth.dcsbm(nv, ne, gamma=2.5, wmax=1e4, c=200, mu=0.1, seed=1)
    tr_s, tr_d, pos, neg = synth.linkpred_split(src, dst, nv, holdout=0.001, seed=6)
    del src, dst
    out = {"workload": f"DC-SBM {nv:,} nodes / {ne:,} edge draws (gamma 2.5, wmax 1e4, 200 "
                       f"communities, mu 0.1), 0.1% held out, walk 40, s=2, GPU augmentation, n=1",
           "pools": pools, "pool": pool, "prepare_s": time.time() - t0, "runs": {}}
    for b in bs:
        g = G.GraphVite(nv, 128, 1, 1, 0.025, total_samples=pools * pool, vertex_tile=b)
        g.load_edges(tr_s, tr_d)
        t1 = time.time()
        for k in range(pools):
            g.augment_device(40, 2, 1184, pool, 1000 + k)
            st = g.train_episode()
        V = g.vertex()
        if not np.isfinite(V).all():
            raise SystemExit(f"b={b}: non-finite embeddings")
        out["runs"][f"b{b}"] = {"auc": auc(V, pos, neg), "loss_last_pool": st["loss_sum"] / pool,
                                "wall_s": time.time() - t1}
        print(b, out["runs"][f"b{b}"], file=sys.stderr, flush=True)
        g.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
