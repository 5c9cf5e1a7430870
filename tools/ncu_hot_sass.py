"""Top SASS lines by warp-stall samples from an ncu source-page CSV
(--page source --csv --print-source sass), per kernel block.
Usage: python tools/ncu_hot_sass.py SRC.csv [top]"""
import csv
import sys

top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
lines = open(sys.argv[1], newline="").read().splitlines()
blocks, cur = [], None
for row in csv.reader(lines):
    if any("Source" == c for c in row) and any("Sampling" in c for c in row):
        cur = {"hdr": row, "rows": []}
        blocks.append(cur)
    elif cur is not None and len(row) == len(cur["hdr"]):
        cur["rows"].append(row)
    elif row and cur is None:
        print(",".join(row)[:200])
for b in blocks:
    h = b["hdr"]
    src = h.index("Source")
    cols = [i for i, c in enumerate(h) if "Warp Stall Sampling (All" in c] or [i for i, c in enumerate(h) if "Sampling" in c]
    sc = cols[0]
    def val(r):
        try:
            return float(r[sc].replace(",", ""))
        except ValueError:
            return 0.0
    tot = sum(val(r) for r in b["rows"]) or 1.0
    print(f"== block: {len(b['rows'])} SASS lines, {tot:.0f} samples ({h[sc]})")
    for r in sorted(b["rows"], key=val, reverse=True)[:top]:
        print(f"   {100 * val(r) / tot:5.1f} %  {r[src][:110]}")
