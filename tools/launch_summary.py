"""Per-kernel totals of an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, agg = None, collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        h = r
        continue
    if h is None or len(r) != len(h):
        continue
    d = dict(zip(h, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(d["Metric Value"].replace(",", ""))
    v *= {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(d["Metric Unit"], 1.0)
    k = d["Kernel Name"][:70]
    agg.setdefault(k, [0, 0.0])
    agg[k][0] += 1
    agg[k][1] += v
for k, (c, t) in agg.items():
    print(f"{k:70s} {c:5d} {t:9.3f} ms")
