"""Summarise an ncu report (details page): one line per (kernel, metric) for the
metrics that decide HBM-bound kernels.  Usage: python tools/ncu_summary.py REP [regex]"""
import csv
import io
import re
import subprocess
import sys

KEEP = ("Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "L1/TEX Hit Rate", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Issue Slots Busy", "Executed Ipc Active", "Grid Size",
        "Block Limit Shared Mem", "Block Limit Registers", "Dynamic Shared Memory Per Block", "Warp Cycles Per Issued Instruction",
        "Compute (SM) Throughput", "Max Bandwidth", "L2 Compression", "Mem Busy", "Mem Pipes Busy")
rep = sys.argv[1]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
for r in rows[1:]:
    if len(r) <= ix["Metric Value"] or not r[ix["Metric Name"]]:
        continue
    name = r[ix["Kernel Name"]]
    if pat and not pat.search(name):
        continue
    m = r[ix["Metric Name"]]
    if m in KEEP:
        print(f'{r[ix["ID"]]:>3} {name.split("(")[0][:60]:60s} {m:36s} {r[ix["Metric Value"]]:>14s} {r[ix["Metric Unit"]]}')
