"""bench.py — PRISM Newton–Schulz on B200 (BASELINE.json metric/configs).

A "step" is one call of the whole hot path over one batch: normalise, then
per iteration residual GEMM -> sketch chain -> alpha solve -> square GEMM ->
apply GEMM, until every matrix converged, then write-back.  Default workload
(N=1) is BASELINE.json configs[1]: the Muon step of GPT-2 small, 48 BF16
layer gradients 768x{768,2304,3072} / 3072x768, PRISM-5 polar.

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl prism|reference]
                        [--workload gpt2|square4096|gpt1b|shampoo]
Multi-GPU: launched by torch.distributed.run, one rank per GPU; each rank
solves its own batch (independent matrices, no data-path collective), so the
scaling is weak.  Prints one JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PRISM solves/sec and TFLOP/s vs B200 BF16 peak; iterations to tolerance"


# ---------------------------------------------------------------- workloads
def workload(name: str, rank: int):
    from paper_2601_22137_b200 import workloads as W
    if name == "gpt2":
        shapes = W.gpt2_small_shapes()
        mats = W.muon_batch(shapes, seed=1 + rank, kind="mixed")
        opts = dict(degree=5, max_iters=20, tol=3e-2, sketch_size=8, seed=42, precision="bf16")
        desc = ("GPT-2 small Muon step (BASELINE.json configs[1]): 48 BF16 gradient matrices, 12 x "
                "{768x2304, 768x768, 768x3072, 3072x768}; half Gaussian (MP), half HTMP-like kappa=0.5; "
                "PRISM-5 polar, p=8, tol 3e-2, max_iters 20")
        return "gpt2-small-muon-step", shapes, mats, opts, desc, "polar"
    if name == "square4096":
        shapes = [(4096, 4096)]
        mats = [W.gaussian(4096, 4096, seed=4096 + rank)]
        opts = dict(degree=5, max_iters=25, tol=3e-2, sketch_size=8, seed=42, precision="bf16")
        desc = "single 4096x4096 Gaussian BF16 polar (north_star 60%-of-peak target shape), PRISM-5, p=8, tol 3e-2"
        return "polar-4096-square", shapes, mats, opts, desc, "polar"
    if name == "gpt1b":
        shapes = W.gpt_1b_shapes()
        mats = W.muon_batch(shapes, seed=1 + rank, kind="gaussian")
        opts = dict(degree=5, max_iters=20, tol=3e-2, sketch_size=8, seed=42, precision="bf16")
        desc = ("1.2B-param GPT Muon step (configs[4] batch, one GPU): 96 BF16 matrices 24 x "
                "{2048x6144, 2048^2, 2048x8192, 8192x2048}, Gaussian, PRISM-5, tol 3e-2")
        return "gpt-1b-muon-step", shapes, mats, opts, desc, "polar"
    if name == "shampoo":
        shapes = [(1024, 1024)] * 8 + [(2048, 2048)] * 4 + [(4096, 4096)] * 2
        mats = [W.spd_logspaced(m, 1e2, seed=100 * rank + i) for i, (m, _) in enumerate(shapes)]
        opts = dict(degree=5, max_iters=30, tol=1e-5, sketch_size=8, seed=42, precision="fp32")
        desc = ("Shampoo step (configs[2]): 8x1024 + 4x2048 + 2x4096 SPD blocks, lambda log-spaced, kappa=1e2, "
                "FP32 (3xTF32) coupled sqrt/inv-sqrt, PRISM-5, tol 1e-5")
        return "shampoo-sqrt-step", shapes, mats, opts, desc, "sqrt"
    if name == "sign4096":
        shapes = [(4096, 4096)]
        mats = [W.sym_indefinite(4096, 1e-2, seed=4096 + rank)]
        opts = dict(degree=5, max_iters=25, tol=3e-2, sketch_size=8, seed=42, precision="bf16")
        desc = ("single 4096x4096 symmetric indefinite BF16 matrix sign (case study P:145-199; |lambda| "
                "log-spaced in [1e-2, 1], alternating signs), PRISM-5, p=8, tol 3e-2")
        return "sign-4096", shapes, mats, opts, desc, "sign"
    if name == "invroot":
        shapes = [(1024, 1024)] * 8 + [(2048, 2048)] * 4 + [(4096, 4096)] * 2
        mats = [W.spd_logspaced(m, 1e2, seed=100 * rank + i) for i, (m, _) in enumerate(shapes)]
        opts = dict(q=4, max_iters=30, tol=1e-5, sketch_size=8, seed=42, precision="fp32")
        desc = ("Shampoo step with the classic inverse 4th root (configs[2] blocks: 8x1024 + 4x2048 + 2x4096 SPD, "
                "kappa=1e2, FP32 3xTF32): PRISM coupled inverse Newton A^{-1/4} (P:549-566), tol 1e-5")
        return "shampoo-invroot4-step", shapes, mats, opts, desc, "inv_root"
    if name == "cheb4096":
        shapes = [(4096, 4096)]
        mats = [W.logspaced(4096, 4096, 0.1, seed=4096 + rank)]
        opts = dict(max_iters=30, tol=3e-2, sketch_size=8, seed=42, precision="bf16")
        desc = ("single 4096x4096 general (non-symmetric) BF16 matrix, sigma log-spaced in [0.1, 1]: PRISM "
                "Chebyshev inverse (P:596-629), p=8, tol 3e-2")
        return "chebyshev-inverse-4096", shapes, mats, opts, desc, "chebyshev"
    if name == "dbnewton":
        shapes = [(1024, 1024)] * 8 + [(2048, 2048)] * 4 + [(4096, 4096)] * 2
        mats = [W.spd_logspaced(m, 1e2, seed=100 * rank + i) for i, (m, _) in enumerate(shapes)]
        opts = dict(max_iters=30, tol=1e-5, sketch_size=8, precision="fp32")
        desc = ("Shampoo step (configs[2] blocks: 8x1024 + 4x2048 + 2x4096 SPD, kappa=1e2, FP32 3xTF32): PRISM "
                "DB Newton product form A^{1/2}, A^{-1/2} (P:499-523; exact unsketched fit), tol 1e-5")
        return "shampoo-dbnewton-step", shapes, mats, opts, desc, "db_newton"
    raise SystemExit(f"unknown workload {name}")


# ---------------------------------------------------------------- helpers
def read_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return d, "measured (MEASURED_PEAKS.json)"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
            "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region (B200_PROFILING.md
    clocks line).  NVML polled every 10 ms from a thread (the timed region of a short run
    lasts only tens of ms, too short for nvidia-smi's 200 ms loop); nvidia-smi fallback."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []          # (time, sm_mhz, set(reasons))
        self.max_mhz = None
        self.t0 = 0.0
        self.stop_ev = threading.Event()
        self.proc = None
        self.source = None

    def start(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
            masks = [(nm, getattr(N, attr)) for nm, attr in self.REASONS if hasattr(N, attr)]

            def poll():
                while not self.stop_ev.is_set():
                    try:
                        mhz = float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM))
                        r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((time.time(), mhz, {nm for nm, m in masks if r & m}))
                    except Exception:
                        pass
                    self.stop_ev.wait(0.01)
            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            self.source = "nvml 10 ms"
            return
        except Exception:
            pass
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read_smi, daemon=True)
            self.t.start()
            self.source = "nvidia-smi 100 ms"
        except Exception:
            self.proc = None

    def _read_smi(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.proc.stdout:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                mhz = float(f[0])
                self.max_mhz = float(f[1])
            except ValueError:
                continue
            self.samples.append((time.time(), mhz, {nm for nm, v in zip(names, f[4:8]) if v.lower() == "active"}))

    def mark(self):
        """Start of the timed region: samples from here on are reported."""
        self.t0 = time.time()

    def stop(self):
        self.stop_ev.set()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.source is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        time.sleep(0.02)
        sm, reasons = [], set()
        for ts, mhz, rs in list(self.samples):
            if ts < self.t0:
                continue
            sm.append(mhz)
            reasons |= rs
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(sm), "source": self.source}


def flush_l2(buf):
    buf.add_(1)   # 256 MiB write > 126 MB L2


def cpu_oracle_solve(A, kind, opts, b):
    from oracle import prism
    d = 1 if opts.get("degree", 5) == 3 else 2
    if kind == "polar":
        return prism.polar(A, d=d, p=opts["sketch_size"], tol=opts["tol"], max_iters=opts["max_iters"],
                           seed=opts["seed"], b=b)[1]
    if kind == "sign":
        return prism.sign(A, d=d, p=opts["sketch_size"], tol=opts["tol"], max_iters=opts["max_iters"],
                          seed=opts["seed"], b=b)[1]
    if kind == "chebyshev":
        return prism.chebyshev_inverse(A, p=opts["sketch_size"], tol=opts["tol"], max_iters=opts["max_iters"],
                                       seed=opts["seed"], b=b)[1]
    if kind == "db_newton":
        return prism.db_newton(A, tol=opts["tol"], max_iters=opts["max_iters"])[2]
    if kind == "inv_root":
        return prism.inv_root(A, q=opts["q"], p=opts["sketch_size"], tol=opts["tol"], max_iters=opts["max_iters"],
                              seed=opts["seed"], b=b)[1]
    return prism.sqrt_invsqrt(A, d=d, p=opts["sketch_size"], tol=opts["tol"], max_iters=opts["max_iters"],
                              seed=opts["seed"], b=b)[2]


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([int(i.get("num_threads", 1)) for i in threadpool_info()] + [1])
    except Exception:
        return os.cpu_count() or 1


def stored_inputs(mats, dtype_name):
    """Inputs rounded to the device dtype, as fp64 numpy (what the oracle reads)."""
    import torch
    dt = torch.bfloat16 if dtype_name == "bf16" else torch.float32
    return [torch.tensor(a).to(dt).double().numpy() for a in mats]


# ---------------------------------------------------------------- reference arm (the oracle)
def run_reference(args, rank, world):
    if rank != 0:
        return 0
    name, shapes, mats, opts, desc, kind = workload(args.workload, 0)
    A = stored_inputs(mats, opts["precision"])
    # bounded, representative sample: every step solves one matrix of each distinct shape
    # (the workloads hold equal numbers of each shape, so this is the batch's mix)
    seen, sample = set(), []
    for i, shp in enumerate(shapes):
        if shp not in seen:
            seen.add(shp)
            sample.append(i)
    smallest = min(range(len(A)), key=lambda i: A[i].size)
    for w in range(args.warmup):   # warm-up: BLAS threads / caches, one small solve
        cpu_oracle_solve(A[smallest], kind, opts, smallest)
    times = []
    for s in range(args.steps):
        t0 = time.perf_counter()
        for i in sample:
            cpu_oracle_solve(A[i], kind, opts, i)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = args.steps * len(sample) / total
    cores = blas_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded), inputs rounded to the device dtype",
        "config": {"workload": name, "description": desc,
                   "reference": "fp64 numpy oracle (oracle/prism.py) on host cores; one matrix of each "
                                "distinct shape per step"},
        "cpu_baseline": {"value": value, "unit": "solves/s", "cores": cores, "kind": "oracle",
                         "sample": f"{args.steps} steps x {len(sample)} matrices (one per distinct shape)"},
        "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="prism", choices=["prism", "reference"])
    ap.add_argument("--workload", default="gpt2", choices=["gpt2", "square4096", "gpt1b", "shampoo", "sign4096", "invroot", "cheb4096",
                                                             "dbnewton"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)   # timing rule: >= 3 warm-up steps

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    import paper_2601_22137_b200 as P

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    name, shapes, mats_np, opts, desc, kind = workload(args.workload, rank)
    dt = torch.bfloat16 if opts["precision"] == "bf16" else torch.float32
    host = [torch.tensor(a).to(dt).pin_memory() for a in mats_np]
    mats = [h.to(dev) for h in host]
    B = len(mats)
    h = P.Handle()
    ids = list(range(B))
    stream = torch.cuda.current_stream(dev)

    def solve(inputs, out=None):
        if kind == "polar":
            return P.polar(inputs, out=out, matrix_ids=ids, handle=h, **opts)
        if kind == "sign":
            return P.sign(inputs, out=out, matrix_ids=ids, handle=h, **opts)
        if kind == "inv_root":
            return P.inv_root(inputs, out=out, matrix_ids=ids, handle=h, **opts)
        if kind == "chebyshev":
            return P.chebyshev_inverse(inputs, out=out, matrix_ids=ids, handle=h, **opts)
        # sqrt kinds: both outputs into preallocated buffers (reused every step, as a
        # training loop would; fresh buffers would rebuild the handle's pointer-keyed plan)
        if kind == "db_newton":
            return P.db_newton(inputs, matrix_ids=ids, handle=h, out_sqrt=outs2[0], out_invsqrt=outs2[1], **dbo)
        return P.sqrt_invsqrt(inputs, matrix_ids=ids, handle=h, out_sqrt=outs2[0], out_invsqrt=outs2[1], **opts)

    dbo = {k: v for k, v in opts.items() if k != "sketch_size"}
    outs = [torch.empty_like(m) for m in mats] if kind in ("polar", "sign", "inv_root", "chebyshev") else None
    outs2 = ([torch.empty_like(m) for m in mats], [torch.empty_like(m) for m in mats]) \
        if kind in ("sqrt", "db_newton") else (None, None)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    clocks = ClockSampler(local)
    clocks.start()                      # sampled from the timed region to the end of the GPU passes
    for _ in range(args.warmup):
        solve(mats, outs)
    torch.cuda.synchronize()

    # ---- timed region: K steps, L2 flushed before each (outside the events)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark()
    rep = None
    for s in range(args.steps):
        flush_l2(flush)
        ev[s][0].record(stream)
        res = solve(mats, outs)
        ev[s][1].record(stream)
        rep = res[-1]
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev)
    launches_per_step = h.launch_count()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.barrier()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_step = ms_max / args.steps
    value = world * B * args.steps / (ms_max / 1e3)

    iters = rep["iters"].cpu().tolist()
    status = rep["status"].cpu().tolist()
    if kind == "polar":
        f_iter = [P.polar_flops_per_iter(m, n, opts["degree"], opts["sketch_size"]) for (m, n) in shapes]
    elif kind == "chebyshev":
        # A'X (residual), R.R, X.P (general products) + 3 chain passes
        f_iter = [6.0 * m ** 3 + 6.0 * m * m * opts["sketch_size"] for (m, _) in shapes]
    elif kind == "inv_root":
        # X + aX.R, M + P_q.M, the POLY products of P_q (1 for q = 2, 2 for q = 3, 4), chain
        npoly = {1: 0, 2: 1, 3: 2, 4: 2}[opts["q"]]
        f_iter = [(4.0 + 2.0 * npoly) * m ** 3 + 2.0 * (opts["q"] + 1) * m * m * opts["sketch_size"]
                  for (m, _) in shapes]
    elif kind == "db_newton":
        # Gauss-Jordan sweep M -> -M^{-1} (2 n^3), X.W and Y.W (4 n^3)
        f_iter = [6.0 * m ** 3 for (m, _) in shapes]
    elif kind == "sign":
        # general (non-symmetric-kernel) products: X.X, R.R (d = 2), X.P, plus the sketch
        f_iter = [4.0 * m ** 3 + ((2.0 * m ** 3 + 14.0 * m * m * opts["sketch_size"]) if opts["degree"] == 5
                                  else 6.0 * m * m * opts["sketch_size"]) for (m, _) in shapes]
    else:
        f_iter = [P.sqrt_flops_per_iter(m, opts["degree"], opts["sketch_size"]) for (m, _) in shapes]
    flops_step = sum(f * k for f, k in zip(f_iter, iters))
    tflops = world * flops_step * args.steps / (ms_max / 1e3) / 1e12

    # ---- e2e: pinned host inputs -> device -> solve -> host through the host-buffer C-ABI
    # entry points (prism_polar_host / prism_sqrt_invsqrt_host): every step uploads its
    # inputs and downloads its result inside the timed region; successive steps pipeline
    # (upload of step s+1 and download of step s overlap the solves).  The events bracket
    # the whole K-step sequence on the caller's stream, which waits for each download.
    host_out = [torch.empty_like(x).pin_memory() for x in host]

    def solve_host():
        if kind == "polar":
            return P.polar_host(host, out=host_out, matrix_ids=ids, handle=h, **opts)
        if kind == "sign":
            return P.sign_host(host, out=host_out, matrix_ids=ids, handle=h, **opts)
        if kind == "chebyshev":
            return P.chebyshev_inverse_host(host, out=host_out, matrix_ids=ids, handle=h, **opts)
        if kind == "inv_root":
            return P.inv_root_host(host, out=host_out, matrix_ids=ids, handle=h, **opts)
        if kind == "db_newton":
            return P.db_newton_host(host, matrix_ids=ids, handle=h, want_sqrt=False, **dbo)[1:]
        return P.sqrt_invsqrt_host(host, matrix_ids=ids, handle=h, want_sqrt=False, **opts)[1:]

    for _ in range(4):   # warm: every staging slot's buffers and plan
        solve_host()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for s in range(args.steps):
        solve_host()
    e1.record(stream)
    torch.cuda.synchronize()
    e_ms = e0.elapsed_time(e1)
    te = torch.tensor([e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e_value = world * B * args.steps / (float(te.item()) / 1e3)
    nbytes = sum(x.numel() * x.element_size() for x in host)

    # ---- per-kernel device timing (separate pass; CUDA events on the launching stream)
    h.profile(True)
    h.profile_read(reset=True)
    for s in range(args.steps):
        flush_l2(flush)
        solve(mats, outs)
    torch.cuda.synchronize()
    prof = h.profile_read(reset=True)
    h.profile(False)
    clk = clocks.stop()
    clk["window"] = "timed + e2e + profiling passes (GPU busy throughout)"
    peaks, peak_src = read_peaks()
    peak = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 1400.0)))
    if opts["precision"] != "bf16":
        peak = peak / 2.0 / 3.0   # tf32 = bf16 / 2 (nominal ratio), 3 MMAs per product in 3xTF32
    if kind == "polar":
        apply_flops = sum(2.0 * max(m, n) * min(m, n) ** 2 * k for (m, n), k in zip(shapes, iters)) * args.steps
        gram_flops = sum(max(m, n) * min(m, n) * (min(m, n) + 1) * (k + 1) for (m, n), k in zip(shapes, iters)) * args.steps
        sq_flops = sum(min(m, n) ** 2 * (min(m, n) + 1) * k for (m, n), k in zip(shapes, iters)) * args.steps
    elif kind == "chebyshev":
        apply_flops = sum(2.0 * m ** 3 * k for (m, _), k in zip(shapes, iters)) * args.steps
        gram_flops = sum(2.0 * m ** 3 * (k + 1) for (m, _), k in zip(shapes, iters)) * args.steps
        sq_flops = sum(2.0 * m ** 3 * k for (m, _), k in zip(shapes, iters)) * args.steps
    elif kind == "inv_root":
        npoly = {1: 0, 2: 1, 3: 2, 4: 2}[opts["q"]]
        apply_flops = sum(4.0 * m ** 3 * k for (m, _), k in zip(shapes, iters)) * args.steps
        gram_flops = 0.0   # R = I - M is elementwise (k_resid_inv)
        sq_flops = sum(2.0 * npoly * m ** 3 * k for (m, _), k in zip(shapes, iters)) * args.steps
    elif kind == "db_newton":
        apply_flops = sum(4.0 * m ** 3 * k for (m, _), k in zip(shapes, iters)) * args.steps
        gram_flops = 0.0   # M_k copied / residual formed elementwise (k_db_begin)
        sq_flops = sum(2.0 * m ** 3 * k for (m, _), k in zip(shapes, iters)) * args.steps   # GJ sweep
    elif kind == "sign":
        apply_flops = sum(2.0 * m ** 3 * k for (m, _), k in zip(shapes, iters)) * args.steps
        gram_flops = sum(2.0 * m ** 3 * (k + 1) for (m, _), k in zip(shapes, iters)) * args.steps
        sq_flops = sum(2.0 * m ** 3 * k for (m, _), k in zip(shapes, iters)) * args.steps
    else:
        apply_flops = sum(4.0 * m ** 3 * k for (m, _), k in zip(shapes, iters)) * args.steps
        gram_flops = sum(2.0 * m ** 3 * (k + 1) for (m, _), k in zip(shapes, iters)) * args.steps
        sq_flops = sum(2.0 * m ** 3 * k for (m, _), k in zip(shapes, iters)) * args.steps
    apply_ms = prof["apply"]["ms"]
    achieved = apply_flops / (apply_ms / 1e3) / 1e12 if apply_ms > 0 else None
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"traffic_{name}.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("apply_dram_bytes_per_launch")
        except Exception:
            traffic = None
    kernel_tflops = {k: (f / (prof[k]["ms"] / 1e3) / 1e12 if prof[k]["ms"] > 0 else None)
                     for k, f in (("gram", gram_flops), ("square", sq_flops), ("apply", apply_flops))}
    prof_total = sum(v["ms"] for v in prof.values())
    shares = {k: (v["ms"] / prof_total if prof_total > 0 else None) for k, v in prof.items()}

    # ---- CPU baseline: the oracle on a bounded sample (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        A = stored_inputs(mats_np, opts["precision"])
        seen, sample = set(), []
        for i, shp in enumerate(shapes):
            if shp not in seen:
                seen.add(shp)
                sample.append(i)
        t0 = time.perf_counter()
        done = 0
        oracle_iters = {}
        while True:          # whole passes over the one-per-shape sample, ~10 s of CPU work
            for i in sample:
                oracle_iters[i] = int(cpu_oracle_solve(A[i], kind, opts, i).iters)
            done += 1
            if time.perf_counter() - t0 >= 10.0:
                break
        sec = time.perf_counter() - t0
        cpu = {"value": done * len(sample) / sec, "unit": "solves/s", "cores": blas_threads(), "kind": "oracle",
               "sample": f"{done} pass(es) x {len(sample)} of {B} matrices (one per distinct shape), "
                         f"fp64 numpy oracle, {sec:.2f} s",
               # iterations to tolerance, device vs the fp64 oracle on the same stored inputs
               "iters_vs_oracle": {"matrix": sample, "device": [int(iters[i]) for i in sample],
                                   "oracle": [oracle_iters[i] for i in sample]}}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": opts["precision"],
            "data": "synthetic: seeded matrices shaped like the paper's workloads (no datasets)",
            "config": {"workload": name, "description": desc, "matrices_per_gpu": B, "solver": kind,
                       "degree": opts.get("degree"), "q": opts.get("q"), "sketch_size": opts["sketch_size"], "tol": opts["tol"],
                       "max_iters": opts["max_iters"], "precision": opts["precision"],
                       "l2": "flushed (256 MiB write) before every timed step, outside the events",
                       "parallelism": f"independent batch per GPU x{world}",
                       "e2e_path": "prism_*_host (the kind's host-buffer entry point): pinned host inputs uploaded and "
                                   "results downloaded every step; steps pipelined (copies overlap solves)"},
            "tflops": tflops, "tflops_unit": "F_min (symmetric products once) per second",
            "frac_of_peak_sustained": tflops / peak if peak else None,
            "iterations": {"mean": sum(iters) / B, "max": max(iters), "min": min(iters),
                           "histogram": {str(k): iters.count(k) for k in sorted(set(iters))}},
            "status_converged": sum(1 for x in status if x == 0),
            "clocks": clk,
            "e2e": {"value": e_value, "unit": "solves/s", "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes},
            "gpu_launches": launches_per_step * args.steps,
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                         "kernel": "prism_gemm_kernel apply (X + X.P), tcgen05",
                         "peak_source": peak_src + (" bf16 sustained" if opts["precision"] == "bf16"
                                                    else " bf16 sustained / 2 (tf32) / 3 (3xTF32)")},
            "kernels": {"tflops": kernel_tflops, "time_share": shares,
                        "ms_per_step": {k: v["ms"] / args.steps for k, v in prof.items()}},
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
