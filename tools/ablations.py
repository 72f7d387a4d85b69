"""NEXT-2: the paper's system ablations re-measured on B200
with synthetic graphs.

  shuffle   tab:shuffle: pool shuffle none / pseudo / random —
            device augmentation time and training speed on C2, and quality
            (link-prediction AUC, node-classification Micro/Macro-F1) on a
            DC-SBM graph trained from walk pools of each kind.
  episode   fig:episode_size: training speed on C2 with n = 4
            (four virtual ranks on one GPU) against the episode size, and
            quality on DC-SBM (n = 4) against the episode size.
  threads   fig:scalability sampler axis: host augmentation
            samples/s against sampler threads.

Collaboration on/off (tab:main_components) is the bench's `pipeline` detail.

    python tools/ablations.py [--parts shuffle,episode,threads] [--out FILE]
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_1903_00757_b200 import gv as G  # noqa: E402

C2 = dict(nv=1_138_499, ne=4_945_382, gamma=2.1, wmax=3e4)
MODES = {"pseudo": G.GV_SHUFFLE_PSEUDO, "none": G.GV_SHUFFLE_NONE, "random": G.GV_SHUFFLE_RANDOM}


def _sync():
    import torch
    torch.cuda.synchronize()


def _quality(V, pos, neg, comm):
    """Link-prediction AUC of cosine scores (ties count 1/2) and
    one-vs-rest logistic-regression Micro/Macro-F1 on 10% labelled nodes
    (P:407). Evaluation only — written here, independent of oracle/."""
    from scipy.stats import rankdata
    from sklearn.linear_model import LogisticRegression
    from sklearn.metrics import f1_score
    from sklearn.multiclass import OneVsRestClassifier
    X = V / np.maximum(np.linalg.norm(V, axis=1, keepdims=True), 1e-12)
    sp = np.sum(X[pos[:, 0]] * X[pos[:, 1]], axis=1)
    sn = np.sum(X[neg[:, 0]] * X[neg[:, 1]], axis=1)
    r = rankdata(np.concatenate([sp, sn]))
    auc = (r[: len(sp)].sum() - len(sp) * (len(sp) + 1) / 2) / (len(sp) * len(sn))
    idx = np.random.default_rng(0).permutation(len(X))
    ntr = len(X) // 10
    tr, te = idx[:ntr], idx[ntr:]
    clf = OneVsRestClassifier(LogisticRegression(max_iter=300)).fit(X[tr], comm[tr])
    pred = clf.predict(X[te])
    return {"auc": round(float(auc), 5),
            "micro_f1": round(float(f1_score(comm[te], pred, average="micro")), 5),
            "macro_f1": round(float(f1_score(comm[te], pred, average="macro")), 5)}


def _dcsbm():
    nv, ne = 100_000, 1_000_000
    src, dst, comm = synth.dcsbm(nv, ne, gamma=2.1, wmax=1000.0, c=50, mu=0.1, seed=1)
    tr_s, tr_d, pos, neg = synth.linkpred_split(src, dst, nv, holdout=0.01, seed=6)
    return nv, tr_s, tr_d, pos, neg, comm


def part_shuffle(res):
    src, dst = synth.chung_lu(C2["nv"], C2["ne"], gamma=C2["gamma"], wmax=C2["wmax"], seed=1)
    P, segs, reps = 200_000_000, 1184, 3
    speed = {}
    for name, mode in MODES.items():
        g = G.GraphVite(C2["nv"], 128, 1, 1, 0.025, total_samples=P * (reps + 1))
        g.load_edges(src, dst)
        g.augment_device(40, 5, segs, P, 1, shuffle=mode)  # warm-up (uploads the CSR)
        g.train_episode(stats=False)
        aug, train = [], []
        for k in range(reps):
            _sync()
            t0 = time.perf_counter()
            g.augment_device(40, 5, segs, P, 2 + k, shuffle=mode)
            _sync()
            aug.append((time.perf_counter() - t0) * 1e3)
            train.append(g.train_episode()["ms_total"])
        a, t = statistics.median(aug), statistics.median(train)
        speed[name] = {"augment_ms": round(a, 2), "train_ms": round(t, 2),
                       "augment_samples_per_s": P / a * 1e3, "train_samples_per_s": P / t * 1e3,
                       "serial_samples_per_s": P / (a + t) * 1e3}
        g.close()
        print("shuffle speed", name, speed[name], flush=True)
    nv, tr_s, tr_d, pos, neg, comm = _dcsbm()
    quality = {}
    pools, count = 10, 4_000_000
    for name, mode in MODES.items():
        g = G.GraphVite(nv, 128, 1, 1, 0.025, total_samples=pools * count)
        g.load_edges(tr_s, tr_d)
        for k in range(pools):
            g.augment_device(40, 5, segs, count, 300 + k, shuffle=mode)
            g.train_episode(stats=False)
        quality[name] = _quality(g.vertex(), pos, neg, comm)
        g.close()
        print("shuffle quality", name, quality[name], flush=True)
    res["shuffle"] = {"speed_C2": speed, "quality_dcsbm_walk40_s5_4e7": quality,
                      "note": "augmentation on the GPU (1184 segments), Hogwild ring kernel; "
                              "random = keyed Feistel permutation of the walk-order pool"}


def part_episode(res):
    rows = []
    for ep in (1_000_000, 4_000_000, 16_000_000, 64_000_000, 200_000_000):
        cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--vranks", "4", "--pool", str(ep),
               "--steps", "5", "--warmup", "3", "--no-cpu-baseline", "--no-e2e"]
        out = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT)
        line = [l for l in out.stdout.splitlines() if l.startswith("{")]
        if not line:
            rows.append({"episode": ep, "error": out.stderr[-500:]})
            continue
        d = json.loads(line[-1])
        rows.append({"episode": ep, "samples_per_s": d["value"], "ms_per_pool": d["ms_per_step"],
                     "bucket_ms": d["detail"]["bucket_ms"], "exchange_ms": d["detail"]["exchange_ms"],
                     "rotate_exposed_ms": d["detail"]["rotate_exposed_ms"]})
        print("episode speed", rows[-1], flush=True)
    nv, tr_s, tr_d, pos, neg, comm = _dcsbm()
    total = 40_000_000
    qual = []
    for ep in (100_000, 1_000_000, 10_000_000):
        pool = 4 * ep  # n = 4: a pool is n episodes (one per offset step)
        g = G.GraphVite(nv, 128, 4, 1, 0.025, total_samples=total, virtual_ranks=4)
        g.load_edges(tr_s, tr_d)
        buf = np.empty((pool, 2), np.uint32)
        for k in range(total // pool):
            g.augment(40, 5, 16, pool, 500 + k, out=buf)
            g.push(buf)
            g.train_episode(stats=False)
        q = _quality(g.vertex(), pos, neg, comm)
        q["episode"] = ep
        qual.append(q)
        g.close()
        print("episode quality", q, flush=True)
    res["episode_size"] = {"speed_C2_n4_vranks": rows, "quality_dcsbm_n4_4e7": qual,
                           "note": "episode = one offset step = pool / n samples (DESIGN R-EPISODE); "
                                   "n = 4 virtual ranks on one GPU"}


def part_threads(res):
    src, dst = synth.chung_lu(C2["nv"], C2["ne"], gamma=C2["gamma"], wmax=C2["wmax"], seed=1)
    g = G.GraphVite(C2["nv"], 128, 1)
    g.load_edges(src, dst)
    count = 20_000_000
    buf = np.empty((count, 2), np.uint32)
    rows = []
    ncpu = os.cpu_count() or 1
    t = 1
    while t <= ncpu:
        g.augment(40, 5, t, count // 10, 1, out=buf[: count // 10])  # warm-up
        t0 = time.perf_counter()
        g.augment(40, 5, t, count, 2, out=buf)
        dt = time.perf_counter() - t0
        rows.append({"threads": t, "samples_per_s": count / dt})
        print("threads", rows[-1], flush=True)
        t *= 2
    g.close()
    res["sampler_threads"] = {"C2_walk40_s5": rows, "host_cpus": ncpu}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--parts", default="shuffle,episode,threads")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    res = {}
    for p in a.parts.split(","):
        {"shuffle": part_shuffle, "episode": part_episode, "threads": part_threads}[p](res)
    s = json.dumps(res, indent=1)
    print(s)
    if a.out:
        open(a.out, "w").write(s + "\n")


if __name__ == "__main__":
    main()
