"""Per-launch table from `ncu --metrics ... --csv` output."""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = [r for r in rows if "Kernel Name" in r][0]
idx = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows if len(r) == len(hdr) and r != hdr]
out = {}
order = []
for r in data:
    key = r[idx["ID"]]
    if key not in out:
        out[key] = {"name": r[idx["Kernel Name"]]}
        order.append(key)
    out[key][r[idx["Metric Name"]]] = r[idx["Metric Value"]]
lim = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for k in order[:lim]:
    m = out[k]
    name = m.pop("name")
    g = re.search(r"GemmCfg<\(int\)(\d+), \(bool\)(\d), \(int\)(\d+), \(bool\)(\d)>", name)
    short = ("gemm" + str(g.groups())) if g else name.split("(")[0].replace("void ", "")[-30:]
    print(f"{short:34s} " + " ".join(f"{kk.split('.')[0][-22:]}={v}" for kk, v in m.items()))
