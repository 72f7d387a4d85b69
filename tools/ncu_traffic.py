"""Extract DRAM traffic of the block-SGD kernel from an `ncu --set full` report
into profiles/sgd_traffic.json (read by bench.py for roofline.traffic).

    python tools/ncu_traffic.py gpurun_out/prof7.ncu-rep <samples_per_launch> <kernel>
"""
import csv
import io
import json
import os
import subprocess
import sys

rep, samples, kernel = sys.argv[1], int(sys.argv[2]), sys.argv[3]
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
       "note": "one launch of the C2 bench configuration (2e8 samples, n=1), ncu --set full "
               "--clock-control none; bench.py scales bytes/sample to its launch size"}
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
with open(os.path.join(root, "profiles", "sgd_traffic.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out))
