#!/usr/bin/env python
"""Benchmark of the GraphVite hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one pass of the whole hot path over one pool of edge samples:
bucketing (a3-a5), block-row exchange (a6, N > 1), the n offset steps of
block-SGD (a7) and the context rotations (a8) — gv_train_episode on a pool
already resident in HBM (gv_replay_pool), so `value` is device throughput.
`e2e` runs the same steps through the C ABI from pinned HOST memory
(gv_push_sample_pool every step, stats read back every step).

N = 1: configs[1] — Youtube-shaped synthetic graph, 1,138,499 nodes /
4,945,382 edges (tab:datasets P:272), d = 128, K = 1, walks of 40 edges,
augmentation distance s = 5, pool = episode size 2e8, n = 1.
N > 1 (torchrun): configs[2] — the same graph on an N x N grid, one rank per
GPU, 2e8 samples per rank per pool (weak scaling), NCCL between ranks.
Inputs (pool 1.6 GB per rank + 2 x 583 MB of embeddings) are larger than the
126 MB L2, so no flush is needed between steps.
"""
from __future__ import annotations

import argparse
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
# BASELINE.json configs: C2/C3 Youtube-shaped (the default bench), C4
# Friendster-small-shaped, C5 Friendster-shaped (tab:datasets P:272; s = 2
# for the larger graphs). Graph shapes: SURVEY §8(d).
CONFIGS = {
    "C2": dict(name="youtube-shaped", nv=1_138_499, ne=4_945_382, gamma=2.1, wmax=3e4, d=128, K=1,
               s=5, walk=40, pool=200_000_000, gen="unique"),
    "C4": dict(name="friendster-small-shaped", nv=7_944_949, ne=447_219_610, gamma=2.5, wmax=1e4,
               d=128, K=1, s=2, walk=40, pool=200_000_000, gen="draws"),
    "C5": dict(name="friendster-shaped", nv=65_608_376, ne=1_806_067_142, gamma=2.5, wmax=5e3,
               d=128, K=1, s=2, walk=40, pool=200_000_000, gen="draws"),
}
CFG = dict(CONFIGS["C2"])
BYTES_PER_SAMPLE = lambda d, K: 2 * (2 + K) * d * 4  # noqa: E731  (BASELINE.json north_star)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS),
                    help="C2 (default, configs[1]); C4 / C5: the Friendster-shaped graphs")
    ap.add_argument("--pool", type=int, default=0, help="samples per rank per pool (0 = config)")
    ap.add_argument("--threads", type=int, default=0, help="sampler threads (0 = all cores)")
    ap.add_argument("--cpu-sample", type=int, default=4_000_000,
                    help="samples of the bounded oracle run (cpu_baseline)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-pipeline", action="store_true", help="skip the gv_run pipeline detail")
    ap.add_argument("--ordered", action="store_true", help="ordered verification kernel (slow)")
    ap.add_argument("--host-partitions", type=int, default=0,
                    help="out-of-core (NEXT-3): n host-resident partitions on one GPU")
    ap.add_argument("--parts-per-rank", type=int, default=1,
                    help="m = n / ranks partitions per rank: m >= 2 overlaps each context "
                         "rotation with the rank's remaining m - 1 blocks of the step (large "
                         "partitions, e.g. C5 over 8 GPUs)")
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


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


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


class OracleArm:
    """The oracle as it stands (serial C, 1 core) on the same workload: a
    Trainer over the same graph, fed bounded pools augmented like the GPU
    pool (walk 40, s = 5, the same sampler-thread segmentation). Graph
    preparation and augmentation are outside the timed region."""

    def __init__(self, src, dst, sample, threads):
        from oracle import oracle as O
        self.O = O
        self.sample, self.threads = sample, threads
        self.t = O.Trainer(CFG["nv"], CFG["d"], 1, K=CFG["K"], lr0=CFG["lr"], lr_kind=1,
                           neg_weight=CFG["neg_weight"], seed=CFG["seed"],
                           total_samples=64 * sample)
        self.t.load_edges(src, dst)
        self.sampler = O.Sampler(O.Graph(CFG["nv"], src, dst))

    def step(self, seed):
        pool = self.sampler.augment(CFG["walk"], CFG["s"], self.threads, self.sample, seed)
        t0 = time.perf_counter()
        self.t.train_pool(pool)
        return time.perf_counter() - t0

    def describe(self, dt):
        return (f"{self.sample} samples per step (a pool of the Youtube-shaped graph augmented with "
                f"walk {CFG['walk']}, s={CFG['s']}, {self.threads} sampler segments), d={CFG['d']}, "
                f"n=1, serial C oracle, {dt:.2f} s per step")


def cpu_baseline(src, dst, sample, threads, seed):
    arm = OracleArm(src, dst, sample, threads)
    dt = arm.step(seed)
    return {"value": sample / dt, "unit": "samples/s", "cores": 1, "kind": "oracle",
            "sample": arm.describe(dt)}


def cpu_hogwild(src, dst, sample, threads, seed):
    """The paper's CPU-baseline class (LINE-style asynchronous SGD on
    all cores): the oracle trainer with each block's samples over OpenMP
    threads, lock-free. Context only, like cpu_baseline."""
    arm = OracleArm(src, dst, sample, threads)
    cores = os.cpu_count() or 1
    pool = arm.sampler.augment(CFG["walk"], CFG["s"], threads, sample, seed)
    t0 = time.perf_counter()
    arm.t.train_pool_hogwild(pool, cores)
    dt = time.perf_counter() - t0
    return {"value": sample / dt, "unit": "samples/s", "cores": cores, "kind": "oracle-hogwild-openmp",
            "sample": f"{sample} samples (one pool, same augmentation as cpu_baseline), d={CFG['d']}, "
                      f"n=1, {cores} OpenMP threads, {dt:.2f} s"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    src, dst = make_graph()
    arm = OracleArm(src, dst, args.cpu_sample, 16)
    times = []
    for k in range(args.warmup + args.steps):
        dt = arm.step(1000 + k)
        if k >= args.warmup:
            times.append(dt)
    total = sum(times)
    value = args.cpu_sample * len(times) / total
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * total / len(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "C2 youtube-shaped 1,138,499 nodes / 4,945,382 edges, d=128, K=1, "
                                   "s=5, walk 40, n=1; serial oracle on a bounded sample per step",
                       "sample_per_step": args.cpu_sample},
            "cpu_baseline": {"value": value, "unit": "samples/s", "cores": 1, "kind": "oracle",
                             "sample": arm.describe(total / len(times))},
            "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1903_00757_b200 import gv as G

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
    # one partition per rank by default (configs[2]); n = 1 on one GPU (configs[1])
    n = world * args.vranks * args.parts_per_rank
    if args.host_partitions:
        n = args.host_partitions
    threads = args.threads or max(1, (os.cpu_count() or 16) // max(1, world))
    src, dst = make_graph()
    P = args.pool
    steps_total = args.warmup + args.steps
    total_samples = P * n * (steps_total + (0 if args.no_e2e else args.steps))
    g = G.GraphVite(CFG["nv"], CFG["d"], n, CFG["K"], CFG["lr"], total_samples=total_samples,
                    neg_weight=CFG["neg_weight"], seed=CFG["seed"],
                    device=dev, rank=rank, world_size=world, ordered=1 if args.ordered else 0,
                    virtual_ranks=args.vranks, host_partitions=1 if args.host_partitions else 0)
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
    for _ in range(max(0, args.warmup - 1)):
        g.replay()
        stats = g.train_episode()
    barrier()
    clocks = Clocks(dev)
    clocks.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    sgd_ms, sgd_launches, launches, samples, tot_ms = 0.0, 0, 0, 0, []
    for _ in range(args.steps):
        g.replay()
        st = g.train_episode()
        sgd_ms += st["ms_sgd"]
        sgd_launches += st["sgd_launches"]
        launches += st["kernel_launches"]
        samples += st["samples_global"]
        tot_ms.append(st["ms_total"])
    ev1.record(stream)
    barrier()
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        ms = allmax(ms)
    value = samples / (ms / 1e3)
    # roofline of the dominant kernel (block-SGD): algorithmic bytes per launch / launch time
    bps = BYTES_PER_SAMPLE(CFG["d"], CFG["K"])
    local_samples = samples // world  # all virtual ranks of this process
    # ms_sgd is per rank (max over virtual ranks); launches are summed over them
    avg_launch_ms = sgd_ms / max(sgd_launches / args.vranks, 1)
    per_launch_samples = local_samples / max(sgd_launches, 1)
    achieved = per_launch_samples * bps / (avg_launch_ms / 1e3) / 1e9
    peak, peak_kind = peaks()
    traffic = None
    try:  # DRAM bytes of the same kernel from the committed ncu --set full capture
        with open(os.path.join(ROOT, "profiles", "sgd_traffic.json")) as f:
            tr = json.load(f)[args.config]  # captured for this config (n = 1)
        default_shape = CFG["d"] == CONFIGS[args.config]["d"] and CFG["K"] == CONFIGS[args.config]["K"]
        if n == 1 and world == 1 and default_shape:
            traffic = tr["dram_bytes_per_sample"] * per_launch_samples
    except Exception:
        pass
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic,
            "traffic_source": "profiles/sgd_traffic.json (ncu dram__bytes_read+write per sample x "
                              "samples per launch)", "kernel": (f"sgd_ring_kernel<{CFG['K']}> (d<=128 Hogwild)" if CFG["d"] <= 128
                       else f"sgd_hogwild_kernel<{CFG['K']}> (d>128 Hogwild)"),
            "peak_source": peak_kind, "sgd_share_of_step": sgd_ms / sum(tot_ms),
            "bytes_per_sample": bps}
    if traffic is not None:
        roof["ncu_dram_bytes_per_sample"] = tr["dram_bytes_per_sample"]
        roof["ncu_l2_hit_pct"] = tr["l2_hit_rate_pct"]
    # end to end through the C ABI from pinned host memory
    e2e = None
    if not args.no_e2e:
        barrier()
        t0 = time.perf_counter()
        e2e_samples = 0
        g.push(host_pool)                   # H2D of step 0's pool
        for k in range(args.steps):
            g.train_episode(stats=False)    # enqueue step k
            if k + 1 < args.steps:
                g.push(host_pool)           # H2D of step k+1 overlaps step k's training
            st = g.read_stats()             # step k's result (loss, counts) read back (D2H)
            e2e_samples += st["samples_global"]
        barrier()
        dt = time.perf_counter() - t0
        if world > 1:
            dt = allmax(dt)
        e2e = {"value": e2e_samples / dt, "unit": "samples/s",
               "h2d_bytes_per_step": P * args.vranks * 8,
               "d2h_bytes_per_step": 8 * (n * n + 2) + 8}
    # collaboration pipelines (NEXT-1/NEXT-2): wall clock of
    # gv_run over `pipe_pools` pools, pools produced by the host sampler threads
    # (collaborate on / off, tab:main_components) or on the GPU (NEXT-1)
    pipeline = None
    if world == 1 and args.vranks == 1 and not args.host_partitions and not args.no_pipeline:
        pipe_pools = 4
        total = P * pipe_pools
        pipeline = {"pools": pipe_pools, "pool": P}
        g.augment_device(CFG["walk"], CFG["s"], 1184, 1184 * 200, 4999)  # uploads the walk tables
        g.train_episode(stats=False)
        g.synchronize()
        t0 = time.perf_counter()
        g.augment_device(CFG["walk"], CFG["s"], 1184, P, 5000)
        g.synchronize()
        pipeline["gpu_augment_ms_per_pool"] = 1e3 * (time.perf_counter() - t0)
        g.train_episode(stats=False)  # consume it
        g.synchronize()
        for name, kw in [("gpu_augment", dict(threads=1184, device=True)),
                         ("host_collaborate", dict(threads=threads, collaborate=True)),
                         ("host_sequential", dict(threads=threads, collaborate=False))]:
            rep = G.gv_run(g.ctx, CFG["walk"], CFG["s"], kw.pop("threads"), P, 6000, total, **kw)
            pipeline[name + "_samples_per_s"] = total / (rep["wall_ms"] / 1e3)
            if not name.startswith("gpu"):
                pipeline[name + "_produce_ms"] = rep["produce_ms"]
                pipeline[name + "_train_wait_ms"] = rep["train_wait_ms"]
    cpu = cpu_hog = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(src, dst, args.cpu_sample, threads, 1000)
        cpu_hog = cpu_hogwild(src, dst, args.cpu_sample * 4, threads, 1001)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": (f"{args.config} {CFG['name']}" if world == 1 or args.config != "C2"
                                    else "C3 youtube-shaped grid")
                       + f" synthetic power-law graph {CFG['nv']:,} nodes / {CFG['ne']:,} edges "
                       f"(chung-lu gamma {CFG['gamma']}, wmax {CFG['wmax']:g}), d={CFG['d']}, K={CFG['K']}, walk 40, "
                       f"s={CFG['s']}, pool {P:,} samples per rank, n={n}",
                       "partitions": n, "pool_per_rank": P, "l2": "inputs > L2 (no flush)",
                       "virtual_ranks": args.vranks, "parts_per_rank": args.parts_per_rank,
                       "method": {"d": CFG["d"], "K": CFG["K"], "walk": CFG["walk"], "s": CFG["s"],
                                  "lr0": CFG["lr"], "neg_weight": CFG["neg_weight"],
                                  "seed": CFG["seed"], "lr_schedule": "linear, floor 1e-4"},
                       "host_partitions": bool(args.host_partitions),
                       "mode": "ordered" if args.ordered else "hogwild"},
            "roofline": roof, "cpu_baseline": cpu, "cpu_hogwild": cpu_hog, "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk, "pipeline": pipeline,
            "detail": {"ms_total_per_pool": tot_ms, "sgd_ms_per_pool": sgd_ms / args.steps,
                       "bucket_ms": stats["ms_bucket"], "exchange_ms": stats["ms_exchange"],
                       "rotate_exposed_ms": stats["ms_rotate"], "load_edges_s": t_load,
                       "augment_s": t_aug, "augment_threads": threads,
                       "alg_gbs_step": value / world * bps / 1e9,
                       "kb2_samples_per_s": local_samples / max(sgd_ms / 1e3, 1e-9),
                       "seeds": {"graph": 1, "id_permutation": 2, "augmentation": 1000 + rank,
                                 "init": 4, "negatives": 5}},
        }
        print(json.dumps(line))
    g.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    CFG.clear()
    CFG.update(CONFIGS[args.config])
    CFG.update(lr=0.025, neg_weight=None, seed=5)
    for flag, key in [("dim", "d"), ("negatives", "K"), ("walk_length", "walk"),
                      ("aug_distance", "s"), ("lr", "lr"), ("neg_scale", "neg_weight"),
                      ("gamma", "gamma"), ("wmax", "wmax")]:
        if getattr(args, flag):
            CFG[key] = getattr(args, flag)
    if args.seed >= 0:
        CFG["seed"] = args.seed
    if CFG["neg_weight"] is None:
        CFG["neg_weight"] = 5.0 / CFG["K"]
    if args.pool == 0:
        args.pool = CFG["pool"]
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
