"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
data = []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data:
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"]
    m = re.search(r"GemmCfg<\(int\)(\d+), \(bool\)(\d), \(bool\)(\d), \(int\)(\d+)>", name) or \
        re.search(r"GemmCfg<(\d+), (\w+), (\w+), (\d+)>", name)
    fn = re.search(r"(prism_\w+_kernel)", name)
    k = ("%s kind=%s split=%s" % (fn.group(1) if fn else "gemm", m.group(1), m.group(2))) if m else name.split("(")[0][:60]
    v = float(d["Metric Value"].replace(",", ""))
    scale = 1e-3 if d.get("Metric Unit", "ns") == "ns" else (1.0 if d.get("Metric Unit") == "us" else 1e3)
    agg[k][0] += 1
    agg[k][1] += v * scale
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':58s} {'n':>5s} {'total_us':>10s} {'share':>6s} {'avg_us':>8s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:58s} {v[0]:5d} {v[1]:10.1f} {v[1]/tot:6.3f} {v[1]/v[0]:8.1f}")
print(f"total {tot:.1f} us")
