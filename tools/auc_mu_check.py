"""Oracle AUC on the AUC-parity graph for a given community mixing mu.

    python tools/auc_mu_check.py <mu> <pools> <samples_per_pool>

Evidence for reading R-AUCGRAPH: the serial oracle (n = 1)
trained on SURVEY §8(c)'s AUC-parity graph (DC-SBM, 1e5 nodes / 1e6 edges,
gamma 2.1, w_max 1000, 50 communities, 1% of edges held out, d = 128, K = 1,
lr0 0.025 with linear decay over the run) prints the link-prediction AUC
 after every pool. Output: profiles/r02_auc_mu_oracle.log.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import synth  # noqa: E402
from oracle import oracle as O  # noqa: E402


def main(mu, pools, count):
    nv, ne = 100_000, 1_000_000
    src, dst, _ = synth.dcsbm(nv, ne, gamma=2.1, wmax=1000.0, c=50, mu=mu, seed=1)
    tr_s, tr_d, pos, neg = synth.linkpred_split(src, dst, nv, holdout=0.01, seed=6)
    o = O.Trainer(nv, 128, 1, K=1, lr0=0.025, lr_kind=1, total_samples=pools * count)
    o.load_edges(tr_s, tr_d)
    t0 = time.time()
    for k in range(pools):
        o.train_pool(synth.edge_pool(tr_s, tr_d, count, seed=200 + k))
        print(k, O.linkpred_auc(o.get("vertex"), pos, neg), time.time() - t0, flush=True)


if __name__ == "__main__":
    main(float(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]))
