"""Per-kernel summary of an ncu raw-page CSV: duration, DRAM bytes/throughput,
issue activity and the warp-stall sample breakdown (top reasons).
Usage: python tools/ncu_stalls.py RAW.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], newline="")))
hdr = next(r for r in rows if "Kernel Name" in r)
units = rows[rows.index(hdr) + 1]
ix = {h: i for i, h in enumerate(hdr)}
KEY = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed.sum",
       "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
       "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__occupancy_limit_shared_mem"]
for r in rows[rows.index(hdr) + 2:]:
    if len(r) < len(hdr):
        continue
    print("==", r[ix["Kernel Name"]][:150])
    for k in KEY:
        if k in ix:
            print(f"   {k:60s} {r[ix[k]]:>16s} {units[ix[k]]}")
    st = []
    for h, i in ix.items():
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
            try:
                st.append((float(r[i].replace(",", "")), h[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1.0
    for v, name in sorted(st, reverse=True)[:10]:
        print(f"   stall {name:40s} {100 * v / tot:6.1f} %")
