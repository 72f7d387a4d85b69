import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import synth
from paper_1903_00757_b200 import gv as G
NV, NE, POOL = 1_138_499, 4_945_382, 200_000_000
src, dst = synth.chung_lu(NV, NE, gamma=2.1, wmax=3e4, seed=1)
tr_s, tr_d, pos, neg = synth.linkpred_split(src, dst, NV, holdout=0.01, seed=6)
for mode in ["device_aug"]:
    g = G.GraphVite(NV, 128, 1, 1, 0.025, total_samples=10 * POOL, ordered=0)
    g.load_edges(tr_s, tr_d)
    for k in range(10):
        if mode == "device_aug":
            g.augment_device(40, 5, 1184, POOL, 1000 + k)
        else:
            g.push(synth.edge_pool(tr_s, tr_d, POOL // 4, seed=k))
        st = g.train_episode()
        V = g.vertex(); C = g.context()
        print(mode, k, "loss/sample", st["loss_sum"] / st["samples_global"], "finite V", np.isfinite(V).mean(), "C", np.isfinite(C).mean(),
              "max|V|", np.nanmax(np.abs(V)), "max|C|", np.nanmax(np.abs(C)), "lr", st["lr_first"], flush=True)
    Vn = V / np.maximum(np.linalg.norm(V, axis=1, keepdims=True), 1e-12)
    print("norm zero rows", int((np.linalg.norm(V, axis=1) == 0).sum()), "nan after norm", int(np.isnan(Vn).sum()), "pos max", int(pos.max()), "neg max", int(neg.max()), pos.dtype, flush=True)
    g.close()
