"""End-to-end probe: library polar / sqrt vs the fp64 oracle on small inputs."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = [
    ("polar", "fp32", 5, 256, 128), ("polar", "fp32", 3, 128, 256), ("polar", "bf16", 5, 768, 768),
    ("polar", "bf16", 5, 3072, 768), ("polar", "bf16", 3, 768, 2304), ("polar", "tf32", 5, 300, 200),
    ("sqrt", "fp32", 5, 256, 256), ("sqrt", "fp32", 3, 200, 200),
]
if len(sys.argv) > 1 and sys.argv[1] == "one":
    sys.path.insert(0, ROOT)
    import numpy as np, torch
    from oracle import prism
    from paper_2601_22137_b200 import workloads as W
    import paper_2601_22137_b200 as P
    kind, prec, deg, m, n = sys.argv[2], sys.argv[3], int(sys.argv[4]), int(sys.argv[5]), int(sys.argv[6])
    d = 1 if deg == 3 else 2
    dt = torch.bfloat16 if prec == "bf16" else torch.float32
    tol = {"bf16": 3e-2, "fp32": 1e-5, "tf32": 1e-2}[prec]
    if kind == "polar":
        A = W.gaussian(m, n, seed=11)
        At = torch.tensor(A).to(dt).cuda()
        Aq = At.double().cpu().numpy()
        Q, rep = P.polar([At], degree=deg, max_iters=30, tol=tol, seed=42, precision=prec)
        torch.cuda.synchronize()
        Qo, ro = prism.polar(Aq, d=d, p=8, tol=tol, max_iters=30, seed=42)
        got = Q[0].double().cpu().numpy()
        res = {"rel": float(np.linalg.norm(got - Qo) / np.linalg.norm(Qo)), "iters": int(rep["iters"][0]),
               "oracle_iters": ro.iters, "status": int(rep["status"][0]),
               "alphas": [round(float(x), 5) for x in rep["alphas"][0][: int(rep["iters"][0])].tolist()],
               "oracle_alphas": [round(a, 5) for a in ro.alphas],
               "resid": [float(x) for x in rep["resid_hist"][0][: int(rep["iters"][0]) + 1].tolist()],
               "oracle_resid": ro.resid}
    else:
        A = W.spd_logspaced(m, 1e2, seed=5)
        At = torch.tensor(A).to(dt).cuda()
        Aq = At.double().cpu().numpy()
        X, Y, rep = P.sqrt_invsqrt([At], degree=deg, max_iters=30, tol=tol, seed=42, precision=prec)
        torch.cuda.synchronize()
        Xo, Yo, ro = prism.sqrt_invsqrt(Aq, d=d, p=8, tol=tol, max_iters=30, seed=42)
        res = {"rel_sqrt": float(np.linalg.norm(X[0].double().cpu().numpy() - Xo) / np.linalg.norm(Xo)),
               "rel_isqrt": float(np.linalg.norm(Y[0].double().cpu().numpy() - Yo) / np.linalg.norm(Yo)),
               "iters": int(rep["iters"][0]), "oracle_iters": ro.iters, "status": int(rep["status"][0]),
               "alphas": [round(float(x), 5) for x in rep["alphas"][0][: int(rep["iters"][0])].tolist()],
               "oracle_alphas": [round(a, 5) for a in ro.alphas]}
    print(json.dumps({"case": sys.argv[2:], **res}))
    sys.exit(0)
for c in CASES:
    try:
        r = subprocess.run([sys.executable, __file__, "one"] + [str(x) for x in c], capture_output=True, text=True, timeout=120)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else ""
        if r.returncode != 0:
            line = json.dumps({"case": list(c), "rc": r.returncode, "err": r.stderr.strip()[-600:]})
    except subprocess.TimeoutExpired:
        line = json.dumps({"case": list(c), "timeout": True})
    print(line, flush=True)
