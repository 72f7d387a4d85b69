"""Extract DRAM traffic of the block-SGD kernel from an `ncu --set full` report
into profiles/sgd_traffic.json (read by bench.py for roofline.traffic).

    python tools/ncu_traffic.py <report.ncu-rep> <samples_per_launch> <kernel> <config>
"""
import csv
import io
import json
import os
import subprocess
import sys

rep, samples, kernel, config = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4]
raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True)
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
get = {h: (u, v) for h, u, v in zip(hdr, units, vals)}


def gbytes(name):
    u, v = get[name]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[u]
    return float(v) * scale


rd, wr = gbytes("dram__bytes_read.sum"), gbytes("dram__bytes_write.sum")
out = {"kernel": kernel, "report": os.path.basename(rep), "samples_per_launch": samples,
       "dram_read_bytes": rd, "dram_write_bytes": wr, "dram_bytes_per_sample": (rd + wr) / samples,
       "l2_hit_rate_pct": float(get["lts__t_sector_hit_rate.pct"][1]),
       "ncu_duration_ms": float(get["gpu__time_duration.sum"][1]),
       "note": f"one launch of the {config} bench configuration (n=1), ncu --set full "
               "--clock-control none; bench.py scales bytes/sample to its launch size"}
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path = os.path.join(root, "profiles", "sgd_traffic.json")
allc = {}
if os.path.exists(path):
    with open(path) as f:
        allc = json.load(f)
    if "kernel" in allc:  # old single-config layout
        allc = {}
allc[config] = out
with open(path, "w") as f:
    json.dump(allc, f, indent=1)
print(json.dumps(out))
