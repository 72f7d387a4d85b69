"""Key metrics of an `ncu --page details --csv` export, one block per kernel launch.

    python tools/ncu_details_summary.py details.csv
"""
import csv
import sys

KEEP = {"Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Compute (SM) Throughput", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Warp Cycles Per Issued Instruction", "Issue Slots Busy", "Eligible Warps Per Scheduler",
        "No Eligible", "Executed Ipc Active", "Block Limit Shared Mem", "Block Limit Registers",
        "Dynamic Shared Memory Per Block", "Grid Size", "Block Size", "Mem Busy", "Max Bandwidth",
        "Mem Pipes Busy"}
rows = list(csv.reader(open(sys.argv[1])))
h, cur = None, None
for r in rows:
    if "Kernel Name" in r:
        h = r
        continue
    if h is None or len(r) < len(h) - 5:
        continue
    d = dict(zip(h, r))
    key = (d["ID"], d["Kernel Name"])
    if key != cur:
        cur = key
        print(f"\n== launch {d['ID']}: {d['Kernel Name'][:90]}  grid {d['Grid Size']} block {d['Block Size']}")
    if d["Metric Name"] in KEEP:
        print(f"  {d['Section Name'][:28]:28s} {d['Metric Name']:36s} {d['Metric Value']:>14s} {d['Metric Unit']}")
