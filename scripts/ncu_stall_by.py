"""Top SASS instructions for one stall reason (e.g. stall_long_sb) from an
`ncu --page source --print-source sass --csv` dump, with 3 instructions of context before."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
reason = sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 8
hi = [i for i, r in enumerate(rows) if "Source" in r][0]
hdr = rows[hi]
idx = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[hi + 1:] if len(r) == len(hdr) and r[0].startswith("0x")]
tot = sum(float(r[idx[reason]] or 0) for r in data) or 1.0
print(f"{reason}: {tot:.0f} samples")
order = sorted(range(len(data)), key=lambda i: -float(data[i][idx[reason]] or 0))
for i in order[:n]:
    print(f"-- {float(data[i][idx[reason]] or 0) / tot:.3f}")
    for j in range(max(0, i - 3), i + 1):
        r = data[j]
        print(f"   #{j:5d} exe={r[idx['Instructions Executed']]:>8s} {r[idx['Source']].strip()[:100]}")
