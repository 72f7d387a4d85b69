#!/usr/bin/env python
"""Benchmark of the GraphVite hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C5|C4|C2]

A step is one pass of the whole hot path over one pool of edge samples:
bucketing (a3-a5), block-row exchange (a6, N > 1), the n offset steps of
block-SGD (a7) and the context rotations (a8) — gv_train_episode on a pool
already resident in HBM (gv_replay_pool), so `value` is device throughput.
`e2e` runs the same steps through the C ABI from pinned HOST memory
(gv_push_sample_pool every step, the step's statistics read back every step).

Default workload (north_star: ">= 60% of HBM roofline per GPU on the
Friendster-shaped workload"): configs[4], C5 — a seeded Chung-Lu graph of
65,608,376 nodes / 1,806,067,142 edge draws (tab:datasets P:272-273), d = 128,
K = 1, walks of 40 edges, augmentation distance s = 2, 5e8 samples
per rank per pool (weak scaling: 4e9 per pool at 8 GPUs),
n = 1 partition on one GPU. The Youtube-shaped C2 (configs[1], whose hot
head is L2-resident) is measured in the same run as `extra.C2`.
Under torchrun (N > 1) every rank runs the same config on an N x (m N) grid
(m = --parts-per-rank, chosen automatically when 0).
Inputs (pool 4 GB per rank + 2 x 33.6 GB of embeddings) are far larger than
the 126 MB L2, so no flush is needed between steps.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "edge samples/sec (device-timed, max over ranks) at 1/2/4/8 B200; HBM GB/s vs peak"
# BASELINE.json configs (shapes: SURVEY §8(d)); pool = samples per rank per
# pool; cpu_sample / ref_sample = bounded oracle samples (cpu_baseline line,
# reference arm per step), sized for ~10-30 s of serial CPU work.
CONFIGS = {
    "C2": dict(name="youtube-shaped", nv=1_138_499, ne=4_945_382, gamma=2.1, wmax=3e4, d=128, K=1,
               s=5, walk=40, pool=200_000_000, gen="unique", cpu_sample=20_000_000,
               ref_sample=2_000_000),
    "C4": dict(name="friendster-small-shaped", nv=7_944_949, ne=447_219_610, gamma=2.5, wmax=1e4,
               d=128, K=1, s=2, walk=40, pool=200_000_000, gen="draws", cpu_sample=10_000_000,
               ref_sample=1_000_000),
    "C5": dict(name="friendster-shaped", nv=65_608_376, ne=1_806_067_142, gamma=2.5, wmax=5e3,
               d=128, K=1, s=2, walk=40, pool=500_000_000, gen="draws", cpu_sample=10_000_000,
               ref_sample=1_000_000),
}
DEFAULT_CONFIG = "C5"
CFG = {}
BYTES_PER_SAMPLE = lambda d, K: 2 * (2 + K) * d * 4  # noqa: E731  (BASELINE.json north_star)


def distinct_vertex_rows(u, nv):
    """Number of distinct vertex ids in a pool's u column."""
    seen = np.zeros(nv, dtype=np.bool_)
    seen[u] = True
    return int(seen.sum())


def compulsory_bytes_per_sample(d, K, samples, distinct_u=None):
    """Row bytes a schedule must move per sample (DESIGN.md §6 / §11).
    Pool order: every row of a sample read and written once, 2(2+K)d4.
    Vertex-tile order (R-VTILE, n = 1): the context rows (positive and K
    negatives) still once per sample, a vertex row once per pool — its tile
    stays in L2 while the tile's samples run: 2(1+K)d4 + 2d4 distinct/samples."""
    if distinct_u is None:
        return BYTES_PER_SAMPLE(d, K)
    row = d * 4
    return 2 * (1 + K) * row + 2 * row * distinct_u / samples


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS),
                    help="C5 (default, Friendster-shaped), C4, C2 (Youtube-shaped)")
    ap.add_argument("--pool", "--episode-size", dest="pool", type=int, default=0,
                    help="samples per rank per pool (0 = config; SPEC's --episode-size)")
    ap.add_argument("--threads", type=int, default=0, help="sampler threads (0 = all cores)")
    ap.add_argument("--cpu-sample", type=int, default=0,
                    help="samples of the bounded oracle run (cpu_baseline; 0 = config)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-pipeline", action="store_true", help="skip the gv_run pipeline detail")
    ap.add_argument("--no-extra", action="store_true", help="skip the C2 line in `extra`")
    ap.add_argument("--ordered", action="store_true", help="ordered verification kernel (slow)")
    ap.add_argument("--host-partitions", type=int, default=0,
                    help="out-of-core (NEXT-3): n host-resident partitions on one GPU")
    ap.add_argument("--pool-ids", default="relabeled", choices=["relabeled", "original"],
                    help="id space of the pools the samplers write (gv_options.pool_ids): "
                         "relabeled (default; a3 needs no relabel gather, and at n = 1 the "
                         "pool is trained where it lies) or the caller's original ids")
    ap.add_argument("--host-pool", action="store_true",
                    help="raw pool in pinned host memory (P:284), read over PCIe by bucketing")
    ap.add_argument("--vertex-tile", type=int, default=14,
                    help="gv_options.vertex_tile b (reading R-VTILE): blocks in vertex-tile order, "
                         "tiles of 2^b rows reused from L2 (0 = pool order)")
    ap.add_argument("--partitions", type=int, default=0,
                    help="n, the grid size (SPEC's --partitions): parts_per_rank = n / ranks")
    ap.add_argument("--parts-per-rank", type=int, default=0,
                    help="m = n / ranks partitions per rank (0 = automatic: 1 on one GPU; with "
                         "N > 1 the smallest m whose rotation hides behind m - 1 blocks)")
    # SPEC's run flags (SURVEY §5 "Config / flags"): overrides of the config's
    # shape and method parameters, recorded in `config`
    ap.add_argument("--dim", type=int, default=0, help="embedding dimension d")
    ap.add_argument("--negatives", type=int, default=0, help="negatives per sample K")
    ap.add_argument("--neg-scale", type=float, default=0.0,
                    help="negative weight (default 5 / K, R-NEGW)")
    ap.add_argument("--lr", type=float, default=0.0, help="initial learning rate (default 0.025)")
    ap.add_argument("--walk-length", type=int, default=0, help="random-walk edges (default 40)")
    ap.add_argument("--aug-distance", type=int, default=0, help="augmentation distance s")
    ap.add_argument("--gamma", type=float, default=0.0,
                    help="power-law exponent of the synthetic graph (SURVEY 8(d) proposal)")
    ap.add_argument("--wmax", type=float, default=0.0, help="expected-degree cap of the graph")
    ap.add_argument("--seed", type=int, default=-1, help="negative-sampling Philox seed (default 5)")
    ap.add_argument("--vranks", type=int, default=1,
                    help="run the N-rank schedule (n = vranks) as virtual ranks on one GPU: "
                         "measures bucketing / exchange / rotation overheads, not scaling")
    return ap.parse_args()


def set_config(name, args=None):
    CFG.clear()
    CFG.update(CONFIGS[name])
    CFG.update(key=name, lr=0.025, neg_weight=None, seed=5)
    if args is not None:
        for flag, key in [("dim", "d"), ("negatives", "K"), ("walk_length", "walk"),
                          ("aug_distance", "s"), ("lr", "lr"), ("neg_scale", "neg_weight"),
                          ("gamma", "gamma"), ("wmax", "wmax")]:
            if getattr(args, flag):
                CFG[key] = getattr(args, flag)
        if args.seed >= 0:
            CFG["seed"] = args.seed
        if args.pool:
            CFG["pool"] = args.pool
        if args.cpu_sample:
            CFG["cpu_sample"] = args.cpu_sample
        CFG["vertex_tile"] = args.vertex_tile
    if CFG["neg_weight"] is None:
        CFG["neg_weight"] = 5.0 / CFG["K"]


def workload_name(world=1, n=1):
    return (f"{CFG['key']} {CFG['name']} synthetic power-law graph {CFG['nv']:,} nodes / "
            f"{CFG['ne']:,} edges (chung-lu gamma {CFG['gamma']}, wmax {CFG['wmax']:g}"
            f"{', edge draws, duplicates merged by ingest' if CFG['gen'] == 'draws' else ''}), "
            f"d={CFG['d']}, K={CFG['K']}, walk {CFG['walk']}, s={CFG['s']}, "
            f"pool {CFG['pool']:,} samples per rank, n={n}, {world} rank(s)"
            + (f", blocks in vertex-tile order (2^{CFG['vertex_tile']} rows, R-VTILE)"
               if CFG.get("vertex_tile") else ""))


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[5 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def make_graph():
    if CFG["gen"] == "draws":  # large configs: C generator, duplicates merged by ingest
        from synth import fastgen
        return fastgen.chung_lu_draws(CFG["nv"], CFG["ne"], CFG["gamma"], CFG["wmax"], seed=1)
    import synth
    return synth.chung_lu(CFG["nv"], CFG["ne"], gamma=CFG["gamma"], wmax=CFG["wmax"], seed=1)


# ------------------------------------------------------------------- oracle

class OracleArm:
    """The oracle as it stands (serial C, 1 core) on the same workload: a
    Trainer over the same graph (its own linear ingest, partition, alias
    tables and init), fed bounded pools from its own sampler over that graph
    (walk 40, the config's s, the same sampler-thread segmentation). Graph
    preparation and augmentation are outside the timed region."""

    def __init__(self, src, dst, sample, threads):
        from oracle import oracle as O
        self.O = O
        self.sample, self.threads = sample, threads
        t0 = time.perf_counter()
        self.t = O.Trainer(CFG["nv"], CFG["d"], 1, K=CFG["K"], lr0=CFG["lr"], lr_kind=1,
                           neg_weight=CFG["neg_weight"], seed=CFG["seed"],
                           total_samples=64 * sample,
                           vertex_tile=CFG.get("vertex_tile", 0))  # the arm's sample order
        self.t.load_edges(src, dst)
        self.sampler = self.t.sampler()
        self.setup_s = time.perf_counter() - t0

    def pool(self, seed, count=None):
        return self.sampler.augment(CFG["walk"], CFG["s"], self.threads, count or self.sample, seed)

    def step(self, seed):
        pool = self.pool(seed)
        t0 = time.perf_counter()
        self.t.train_pool(pool)
        return time.perf_counter() - t0

    def describe(self, dt):
        return (f"{self.sample:,} samples per step (a pool of the {CFG['key']} {CFG['name']} graph "
                f"augmented by the oracle's sampler: walk {CFG['walk']}, s={CFG['s']}, "
                f"{self.threads} segments), d={CFG['d']}, n=1, vertex_tile={CFG.get('vertex_tile', 0)}, "
                f"serial C oracle, {dt:.2f} s per "
                f"step; oracle setup (ingest, partition, alias, init, walk tables) "
                f"{self.setup_s:.0f} s, untimed")


def cpu_baselines(src, dst, threads):
    """cpu_baseline (the serial oracle) and cpu_hogwild (the paper's CPU
    baseline class: the oracle trainer over all host cores, lock-free
    OpenMP threads) on bounded samples of the workload."""
    arm = OracleArm(src, dst, CFG["cpu_sample"], threads)
    dt = arm.step(1000)
    cpu = {"value": arm.sample / dt, "unit": "samples/s", "cores": 1, "kind": "oracle",
           "sample": arm.describe(dt)}
    cores = os.cpu_count() or 1
    hog_n = max(4 * arm.sample, 100_000_000)  # >= 1e8 samples
    pool = arm.pool(1001, hog_n)
    t0 = time.perf_counter()
    arm.t.train_pool_hogwild(pool, cores)
    dth = time.perf_counter() - t0
    hog = {"value": hog_n / dth, "unit": "samples/s", "cores": cores,
           "kind": "oracle-hogwild-openmp",
           "sample": f"{hog_n:,} samples (one pool, same augmentation as cpu_baseline), "
                     f"d={CFG['d']}, n=1, {cores} OpenMP threads, {dth:.2f} s"}
    return cpu, hog


def run_reference(args):
    """--impl reference: the oracle, as it stands, on this arm's workload and
    metric; each step a bounded sample (ref_sample) of it. Rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    src, dst = make_graph()
    arm = OracleArm(src, dst, CFG["ref_sample"], 16)
    times = []
    for k in range(args.warmup + args.steps):
        dt = arm.step(1000 + k)
        if k >= args.warmup:
            times.append(dt)
    total = sum(times)
    value = arm.sample * len(times) / total
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * total / len(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_name() + "; serial oracle on a bounded sample per step",
                       "sample_per_step": arm.sample},
            "cpu_baseline": {"value": value, "unit": "samples/s", "cores": 1, "kind": "oracle",
                             "sample": arm.describe(total / len(times))},
            "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- our arm

def auto_parts_per_rank(world, nv, d, rate=1.7e9, pool=None, nvlink_gbs=700.0):
    """m = partitions per rank ("partitions > GPUs ... in subgroups").
    With m = 1 every context rotation (NV/n rows of d floats over NVLink,
    Alg. 3) sits between two offset steps; with m >= 2 it overlaps
    the rank's other m - 1 blocks. Smallest m whose exposed
    rotation would be <= 5% of a block's SGD time; 1 on one GPU."""
    if world <= 1:
        return 1
    pool = pool or CFG["pool"]
    for m in (1, 2, 4, 8):
        n = m * world
        if n > 64:
            break
        rot_ms = nv / n * d * 4 / (nvlink_gbs * 1e9) * 1e3
        block_ms = pool * world / (n * n) / rate * 1e3  # one block (i, j) of the global pool
        if m == 1 and rot_ms <= 0.05 * block_ms:
            return 1
        if m >= 2:
            return m
    return 1


def measure(args, world, rank, dev, n, *, steps, warmup, e2e=True, pipeline=True,
            stream_name=""):
    """One config end to end on this rank: graph, load, augmentation, the
    timed replay loop, roofline, e2e and the gv_run pipelines. Returns
    (line fields, graph arrays) and closes the context."""
    import torch
    import torch.distributed as dist

    from paper_1903_00757_b200 import gv as G

    threads = args.threads or max(1, (os.cpu_count() or 16) // max(1, world))
    t0 = time.perf_counter()
    if world > 1 and rank != 0:
        # multi-process: rank 0 prepares the graph once for the node and the
        # other ranks map it (gv_load_edges, node-shared graph): they need no
        # edge list (C5's is 14 GB per copy)
        src = dst = np.empty(0, dtype=np.uint32)
    else:
        src, dst = make_graph()
    t_gen = time.perf_counter() - t0
    P = CFG["pool"]
    total_samples = P * world * args.vranks * (warmup + steps + (steps if e2e else 0) + 1)
    g = G.GraphVite(CFG["nv"], CFG["d"], n, CFG["K"], CFG["lr"], total_samples=total_samples,
                    neg_weight=CFG["neg_weight"], seed=CFG["seed"],
                    device=dev, rank=rank, world_size=world, ordered=1 if args.ordered else 0,
                    virtual_ranks=args.vranks, host_partitions=1 if args.host_partitions else 0,
                    host_pool=1 if args.host_pool else 0,
                    pool_ids=G.GV_IDS_RELABELED if args.pool_ids == "relabeled" else G.GV_IDS_ORIGINAL,
                    vertex_tile=args.vertex_tile)
    if world > 1:
        uid = [G.gv_comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        G.gv_comm_init(g.ctx, uid[0])
    t0 = time.perf_counter()
    g.load_edges(src, dst)
    t_load = time.perf_counter() - t0
    # the rank's pool segment: host augmentation (Alg. 2), pinned host buffer
    host_pool = torch.empty((P * args.vranks, 2), dtype=torch.int32, pin_memory=True)
    t0 = time.perf_counter()
    g.augment(CFG["walk"], CFG["s"], threads, P * args.vranks, 1000 + rank, out=host_pool)
    t_aug = time.perf_counter() - t0
    # compulsory row traffic of the schedule: with blocks in
    # vertex-tile order (R-VTILE) at n = 1 a vertex row is read and written
    # once per pool (its tile's rows stay in L2 while the tile's samples run);
    # context rows (positive and negatives) are random, once per sample
    distinct_u = None
    if args.vertex_tile > 0 and n == 1 and args.pool_ids == "relabeled":
        distinct_u = distinct_vertex_rows(host_pool[:, 0].numpy(), CFG["nv"])
    g.push(host_pool)
    stream = torch.cuda.ExternalStream(g.stream())

    def allmax(x):
        dev_t = "cpu" if dist.get_backend() == "gloo" else "cuda"
        t = torch.tensor([x], dtype=torch.float64, device=dev_t)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    stats = g.train_episode()  # first pool (also warm-up)
    for _ in range(max(0, warmup - 1)):
        g.replay()
        stats = g.train_episode()
    barrier()
    clocks = Clocks(dev)
    clocks.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    sgd_ms, sgd_launches, launches, samples = 0.0, 0, 0, 0
    per_pool, per_rank = [], []
    for _ in range(steps):
        g.replay()
        st = g.train_episode()
        sgd_ms += st["ms_sgd"]
        sgd_launches += st["sgd_launches"]
        launches += st["kernel_launches"]
        samples += st["samples_global"]
        per_pool.append(st["ms_device_max"])
        per_rank.append(st)
    ev1.record(stream)
    barrier()
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        ms = allmax(ms)
    value = samples / (ms / 1e3)
    # roofline of the dominant kernel (block-SGD): algorithmic bytes per launch / launch time
    bps_untiled = BYTES_PER_SAMPLE(CFG["d"], CFG["K"])
    bps = compulsory_bytes_per_sample(CFG["d"], CFG["K"], P * args.vranks, distinct_u)
    local_samples = samples // world  # all virtual ranks of this process
    avg_launch_ms = sgd_ms / max(sgd_launches / args.vranks, 1)  # ms_sgd: max over v-ranks
    per_launch_samples = local_samples / max(sgd_launches, 1)
    achieved = per_launch_samples * bps / (avg_launch_ms / 1e3) / 1e9
    peak, peak_kind = peaks()
    traffic = tr = None
    try:  # DRAM bytes of the same kernel from the committed ncu --set full capture
        with open(os.path.join(ROOT, "profiles", "sgd_traffic.json")) as f:
            tr = json.load(f)[CFG["key"]]  # captured for this config (n = 1)
        default_shape = CFG["d"] == CONFIGS[CFG["key"]]["d"] and CFG["K"] == CONFIGS[CFG["key"]]["K"]
        same_order = tr.get("vertex_tile", 0) == args.vertex_tile  # captured on this order
        if n == 1 and world == 1 and default_shape and same_order:
            traffic = tr["dram_bytes_per_sample"] * per_launch_samples
    except Exception:
        tr = None
    kernel = (f"sgd_ring_kernel<{CFG['K']}> (d<=128 Hogwild)" if CFG["d"] <= 128
              else f"sgd_hogwild_kernel<{CFG['K']}> (d>128 Hogwild)")
    tot_ms = sum(per_pool)
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic,
            "traffic_source": "profiles/sgd_traffic.json (ncu dram__bytes_read+write of one launch "
                              "of the shipped kernel, per sample x samples per launch)",
            "kernel": kernel, "peak_source": peak_kind, "sgd_share_of_step": sgd_ms / tot_ms,
            "bytes_per_sample": bps, "launch_ms": avg_launch_ms,
            "bytes_per_sample_model": ("compulsory rows of the vertex-tile schedule: 2(1+K)d4 "
                                       "(context rows) + 2d4 x distinct vertex rows / samples "
                                       f"({distinct_u:,} / {P * args.vranks:,})"
                                       if distinct_u is not None else
                                       "2(2+K)d4: every row of a sample read and written once"),
            "alg_untiled_gbs": per_launch_samples * bps_untiled / (avg_launch_ms / 1e3) / 1e9,
            "samples_per_launch": per_launch_samples}
    if traffic is not None:
        roof["ncu_dram_bytes_per_sample"] = tr["dram_bytes_per_sample"]
        roof["ncu_l2_hit_pct"] = tr.get("l2_hit_rate_pct")
        roof["dram_frac"] = traffic / (avg_launch_ms / 1e3) / 1e9 / peak
    # end to end through the C ABI from pinned host memory
    e2e_line = None
    if e2e:
        barrier()
        t0 = time.perf_counter()
        e2e_samples = 0
        g.push(host_pool)                   # H2D of step 0's pool
        for k in range(steps):
            g.train_episode(stats=False)    # enqueue step k
            if k + 1 < steps:
                g.push(host_pool)           # H2D of step k+1 overlaps step k's training
            st = g.read_stats()             # step k's result (loss, counts) read back (D2H)
            e2e_samples += st["samples_global"]
        barrier()
        dt = time.perf_counter() - t0
        if world > 1:
            dt = allmax(dt)
        e2e_line = {"value": e2e_samples / dt, "unit": "samples/s",
                    "h2d_bytes_per_step": P * args.vranks * 8,
                    "d2h_bytes_per_step": 8 * (n * n + 2) + 8}
    # collaboration pipelines (NEXT-1/NEXT-2): wall clock of
    # gv_run over a few pools produced by the host sampler threads
    # (collaborate on / off, tab:main_components) or on the GPU (NEXT-1)
    pipe = None
    if pipeline and world == 1 and args.vranks == 1 and not args.host_partitions:
        pipe_pool, pipe_pools = min(P, 200_000_000), 3
        total = pipe_pool * pipe_pools
        pipe = {"pools": pipe_pools, "pool": pipe_pool}
        g.augment_device(CFG["walk"], CFG["s"], 1184, 1184 * 200, 4999)  # uploads the walk tables
        g.train_episode(stats=False)
        g.synchronize()
        t0 = time.perf_counter()
        g.augment_device(CFG["walk"], CFG["s"], 1184, pipe_pool, 5000)
        g.synchronize()
        pipe["gpu_augment_ms_per_pool"] = 1e3 * (time.perf_counter() - t0)
        g.train_episode(stats=False)  # consume it
        g.synchronize()
        for name, kw in [("gpu_augment", dict(threads=1184, device=True)),
                         ("host_collaborate", dict(threads=threads, collaborate=True)),
                         ("host_sequential", dict(threads=threads, collaborate=False))]:
            rep = G.gv_run(g.ctx, CFG["walk"], CFG["s"], kw.pop("threads"), pipe_pool, 6000, total,
                           **kw)
            pipe[name + "_samples_per_s"] = total / (rep["wall_ms"] / 1e3)
            if not name.startswith("gpu"):
                pipe[name + "_produce_ms"] = rep["produce_ms"]
                pipe[name + "_train_wait_ms"] = rep["train_wait_ms"]
    device_bytes = G.gv_device_bytes(g.ctx)
    g.close()
    del host_pool
    ranks = {k: [max(st[k][d] for st in per_rank) for d in range(per_rank[0]["n_ranks"])]
             for k in ("ms_sgd_rank", "ms_bucket_rank", "ms_exchange_rank", "ms_rotate_rank",
                       "ms_total_rank")}
    out = {
        "value": value, "ms_per_step": ms / steps, "gpu_launches": launches, "clocks": clk,
        "roofline": roof, "e2e": e2e_line, "pipeline": pipe,
        "per_pool_ms_device_max": {"median": statistics.median(per_pool), "min": min(per_pool),
                                   "max": max(per_pool)},
        "per_pool_samples_per_s": {"median": samples / steps / statistics.median(per_pool) * 1e3,
                                   "min": samples / steps / max(per_pool) * 1e3,
                                   "max": samples / steps / min(per_pool) * 1e3},
        "detail": {"ms_device_max_per_pool": per_pool, "sgd_ms_per_pool": sgd_ms / steps,
                   "bucket_ms": stats["ms_bucket"], "exchange_ms": stats["ms_exchange"],
                   "rotate_exposed_ms": stats["ms_rotate"],
                   "per_rank_max_over_pools": ranks,
                   "generate_s": t_gen, "load_edges_s": t_load,
                   "augment_s": t_aug, "augment_threads": threads,
                   "device_bytes": device_bytes,
                   "alg_gbs_step": value / world * bps / 1e9,
                   "kb2_samples_per_s": local_samples / max(sgd_ms / 1e3, 1e-9),
                   "seeds": {"graph": 1, "id_permutation": 2, "augmentation": 1000 + rank,
                             "init": 4, "negatives": CFG["seed"]}},
    }
    return out, (src, dst), threads


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # GV_BENCH_DEVICE=<k> puts every rank on device k: a code-path check of the
    # multi-process path on a one-GPU box (not a scaling measurement)
    dev = int(os.environ.get("GV_BENCH_DEVICE", local))
    torch.cuda.set_device(dev)
    if world > 1:
        dist.init_process_group("gloo" if "GV_BENCH_DEVICE" in os.environ else "nccl")
    main_key = CFG["key"]
    # the Youtube-shaped configs[1] beside the default (one GPU only)
    extra = {}
    if world == 1 and args.vranks == 1 and main_key != "C2" and not args.no_extra and \
            not args.host_partitions:
        saved = dict(CFG)
        set_config("C2")
        r, _, _ = measure(args, 1, 0, dev, 1, steps=min(args.steps, 10), warmup=3, e2e=False,
                          pipeline=False)
        extra["C2"] = {"workload": workload_name(), "value": r["value"], "unit": "samples/s",
                       "ms_per_step": r["ms_per_step"], "roofline": r["roofline"],
                       "kb2_samples_per_s": r["detail"]["kb2_samples_per_s"],
                       "per_pool_samples_per_s": r["per_pool_samples_per_s"],
                       "clocks": r["clocks"], "gpu_launches": r["gpu_launches"]}
        CFG.clear()
        CFG.update(saved)
        gc.collect()
    if args.partitions:
        if args.partitions % (world * args.vranks):
            raise SystemExit(f"--partitions {args.partitions} is not a multiple of the "
                             f"{world * args.vranks} ranks")
        args.parts_per_rank = args.partitions // (world * args.vranks)
    m = args.parts_per_rank or auto_parts_per_rank(world, CFG["nv"], CFG["d"])
    n = world * args.vranks * m
    if args.host_partitions:
        n = args.host_partitions
    r, (src, dst), threads = measure(args, world, rank, dev, n, steps=args.steps,
                                     warmup=args.warmup, e2e=not args.no_e2e,
                                     pipeline=not args.no_pipeline)
    gc.collect()
    cpu = cpu_hog = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu, cpu_hog = cpu_baselines(src, dst, threads)
    if rank == 0:
        line = {
            "metric": METRIC, "value": r["value"], "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": workload_name(world, n), "partitions": n,
                       "pool_per_rank": CFG["pool"], "l2": "inputs > L2 (no flush)",
                       "virtual_ranks": args.vranks, "parts_per_rank": m,
                       "method": {"d": CFG["d"], "K": CFG["K"], "walk": CFG["walk"], "s": CFG["s"],
                                  "lr0": CFG["lr"], "neg_weight": CFG["neg_weight"],
                                  "seed": CFG["seed"], "lr_schedule": "linear, floor 1e-4"},
                       "host_partitions": bool(args.host_partitions),
                       "host_pool": bool(args.host_pool), "pool_ids": args.pool_ids,
                       "vertex_tile": args.vertex_tile,
                       "mode": "ordered" if args.ordered else "hogwild"},
            "roofline": r["roofline"], "cpu_baseline": cpu, "cpu_hogwild": cpu_hog,
            "e2e": r["e2e"], "gpu_launches": r["gpu_launches"], "clocks": r["clocks"],
            "per_pool_ms_device_max": r["per_pool_ms_device_max"],
            "per_pool_samples_per_s": r["per_pool_samples_per_s"],
            "pipeline": r["pipeline"], "extra": extra or None, "detail": r["detail"],
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    set_config(args.config, args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
