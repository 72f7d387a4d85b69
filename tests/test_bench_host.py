"""CPU tests of bench.py's host logic: the partitions-per-rank rule of the
multi-GPU schedule (Alg. 3 P:233 subgroups) and the reference
arm's JSON line (the serial oracle on a bounded sample, no GPU needed)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_parts_per_rank_rule():
    bench.set_config("C5")
    assert bench.auto_parts_per_rank(1, bench.CFG["nv"], 128) == 1
    # C5 at 8 ranks: a 4.2 GB partition rotation (~6 ms) would sit between
    # ~37 ms blocks -> m = 2 hides it behind the rank's other block
    assert bench.auto_parts_per_rank(8, bench.CFG["nv"], 128) == 2
    bench.set_config("C2")
    # C2: a 73 MB partition moves in ~0.1 ms, far below 5% of a block
    assert bench.auto_parts_per_rank(8, bench.CFG["nv"], 128) == 1


def test_workload_names_the_paper_sizes():
    bench.set_config("C5")
    w = bench.workload_name(8, 16)
    assert "65,608,376 nodes / 1,806,067,142 edges" in w and "n=16" in w and "8 rank(s)" in w


@pytest.mark.timeout(600)
def test_reference_arm_json_line():
    """--impl reference: the oracle as it stands on the arm's workload; the
    line carries impl, metric/unit, cpu_baseline and a zero-copy e2e."""
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--config", "C2", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "samples/s" and line["value"] > 0
    assert line["metric"] == bench.METRIC and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] == 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert "1,138,499 nodes" in line["config"]["workload"]


def test_compulsory_bytes_model():
    """The roofline's bytes per sample: pool order is the
    per-sample model 2(2+K)d4 (3072 B at d = 128, K = 1, BASELINE.json); in
    vertex-tile order a pool whose vertex ids are all distinct needs the
    same bytes (no repeat to serve from L2), one repeated vertex needs only
    the context rows plus one vertex row per pool."""
    import numpy as np
    assert bench.compulsory_bytes_per_sample(128, 1, 1000) == 3072
    assert bench.compulsory_bytes_per_sample(128, 1, 1000, distinct_u=1000) == 3072
    assert bench.compulsory_bytes_per_sample(128, 1, 1000, distinct_u=1) == 2048 + 1024 / 1000
    assert bench.compulsory_bytes_per_sample(96, 3, 10, distinct_u=5) == 2 * 4 * 384 + 768 / 2
    u = np.array([3, 1, 3, 3, 0, 1], np.int64)
    assert bench.distinct_vertex_rows(u, 5) == 3
