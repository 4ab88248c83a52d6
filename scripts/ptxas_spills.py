"""List kernels with spills / their register counts from paper_2601_22137_b200/_lib/ptxas.log."""
import re
import sys

log = open(sys.argv[1] if len(sys.argv) > 1 else "paper_2601_22137_b200/_lib/ptxas.log").read().splitlines()
cur = None
for ln in log:
    m = re.search(r"Compiling entry function '(\S+)'", ln)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", ln)
    if m and cur and (int(m.group(1)) or int(m.group(2))):
        print(f"SPILL {m.group(1)}/{m.group(2)}  {cur[:110]}")
