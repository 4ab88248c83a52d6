"""First-contact GPU probe: each kernel case in its own subprocess (with a
timeout) so a faulting case cannot take the others down.  Prints one JSON
line per case."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = [
    # prec, b_mn, mode, sym, M, N, K
    (0, 0, 3, 0, 128, 256, 64),
    (0, 0, 3, 0, 256, 512, 512),
    (0, 1, 3, 0, 128, 256, 64),
    (0, 1, 3, 0, 300, 520, 200),
    (0, 0, 3, 0, 300, 520, 200),
    (0, 0, 0, 1, 384, 384, 1000),
    (0, 1, 1, 0, 256, 256, 256),
    (0, 1, 2, 0, 200, 700, 192),
    (2, 0, 3, 0, 128, 128, 32),
    (2, 1, 3, 0, 300, 260, 200),
    (1, 0, 3, 0, 256, 256, 256),
    (1, 1, 3, 0, 300, 260, 200),
    (1, 0, 0, 1, 384, 384, 512),
    (1, 1, 2, 0, 200, 300, 160),
]

if len(sys.argv) > 1 and sys.argv[1] == "one":
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from gpu_cases import gemm_case
    args = [int(x) for x in sys.argv[2:]]
    print(json.dumps({"case": args, **gemm_case(*args)}))
    sys.exit(0)

for c in CASES:
    try:
        r = subprocess.run([sys.executable, __file__, "one"] + [str(x) for x in c], capture_output=True,
                           text=True, timeout=90)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else ""
        if r.returncode != 0:
            line = json.dumps({"case": list(c), "rc": r.returncode, "err": r.stderr.strip()[-400:]})
    except subprocess.TimeoutExpired:
        line = json.dumps({"case": list(c), "timeout": True})
    print(line, flush=True)
