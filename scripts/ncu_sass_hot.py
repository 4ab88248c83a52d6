"""Top SASS instructions by warp-stall samples from an `ncu --page source --print-source=sass --csv` dump."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hi = [i for i, r in enumerate(rows) if "Source" in r][0]
hdr = rows[hi]
idx = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[hi + 1:] if len(r) == len(hdr) and r[0].startswith("0x")]
key = "Warp Stall Sampling (All Samples)"
tot = sum(float(r[idx[key]] or 0) for r in data) or 1.0
exe = "Instructions Executed"
print(f"total samples {tot:.0f}, instructions {sum(float(r[idx[exe]] or 0) for r in data):.0f}")
order = sorted(range(len(data)), key=lambda i: -float(data[i][idx[key]] or 0))
for i in order[:n]:
    r = data[i]
    print(f"{float(r[idx[key]] or 0)/tot:6.3f} #{i:5d} exe={r[idx[exe]]:>8s} {r[idx['Source']].strip()[:100]}")
