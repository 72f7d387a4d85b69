"""Time the phases of gv_load_edges on a large config (GV_INGEST_TIMING=1
prints the host ingest laps to stderr).

    GV_INGEST_TIMING=1 python tools/ingest_timing.py C5
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
from paper_1903_00757_b200 import gv as G  # noqa: E402


def main(name):
    bench.set_config(name)
    cfg = bench.CFG
    t0 = time.perf_counter()
    src, dst = bench.make_graph()
    print(f"generate {time.perf_counter() - t0:.1f} s", flush=True)
    g = G.GraphVite(cfg["nv"], cfg["d"], 1, 1, 0.025)
    t0 = time.perf_counter()
    g.load_edges(src, dst)
    print(f"load_edges {time.perf_counter() - t0:.1f} s", flush=True)
    t0 = time.perf_counter()
    g.augment_device(40, cfg["s"], 1184, 1184 * 200, 1)
    g.synchronize()
    print(f"device walk tables + first augment {time.perf_counter() - t0:.1f} s", flush=True)
    g.close()


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C5")
