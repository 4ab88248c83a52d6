"""Write the judged profile summaries under profiles/ from a round's gpurun_out/ captures
(scripts/profile_round.sh): the launch list of the bench command with per-kernel shares,
one full-set capture per hot kernel (role-named tcgen05 GEMMs, a chain pass, k_alpha) with
its key metrics and top stall reasons, the DRAM traffic per apply launch that bench.py
reports as roofline.traffic, and the SASS evidence of tcgen05 / TMA in the built library.

usage: python scripts/summarize_profiles.py r2 gpt2 square4096
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "launch__grid_size", "launch__block_size", "launch__cluster_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active"]
CAPTURES = [("prism_gram_kernel", "Gram / residual GEMM (RESID epilogue)"),
            ("prism_square_kernel", "square GEMM (POLY epilogue: P = R/2 + a R^2)"),
            ("prism_apply_kernel", "apply GEMM (X + X.P)"),
            ("chain", "sketch-chain pass (prism_chaint_kernel, 8th chain launch)"),
            ("alpha", "k_alpha (fp64 quartic fit)")]
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def ncu_csv(rep, page, extra=()):
    r = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True)
    return list(csv.reader(io.StringIO(r.stdout)))


def full_capture(rep):
    rows = ncu_csv(rep, "raw")
    h, u, v = rows[0], rows[1], rows[2]
    got = {k: (x, un) for k, un, x in zip(h, u, v) if k in KEYS}
    name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
    sass = ncu_csv(rep, "source", ["--print-source", "sass"])
    stalls, n_all = [], 1.0
    hi = [i for i, r in enumerate(sass) if "Source" in r]
    if hi:
        hdr = sass[hi[0]]
        idx = {k: i for i, k in enumerate(hdr)}
        data = [r for r in sass[hi[0] + 1:] if len(r) == len(hdr) and r[0].startswith("0x")]
        reasons = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
        tot = {k: sum(float(r[idx[k]] or 0) for r in data) for k in reasons}
        n_all = sum(tot.values()) or 1.0
        stalls = sorted(tot.items(), key=lambda x: -x[1])[:8]
    return name, got, stalls, n_all


def launches(tag, w):
    path = os.path.join(OUT, f"{tag}_{w}_launches.csv")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_launches.py"), path],
                       capture_output=True, text=True)
    return r.stdout


def main():
    tag = sys.argv[1]
    for w in sys.argv[2:]:
        name = bench.workload(w, 0)[0]
        with open(os.path.join(PROF, f"{tag}_{w}_kernels_ncu.txt"), "w") as f:
            f.write(f"# {tag}: ncu --set full --clock-control none, one launch per kernel of a direct-launch\n"
                    f"# solve (scripts/profile_step.py --direct), workload {name}; scripts/profile_round.sh.\n"
                    "# Cold caches and a serialised launch: compare shares and ratios, not absolute times.\n")
            for key, what in CAPTURES:
                rep = os.path.join(OUT, f"{tag}_{w}_{key}.ncu-rep")
                if not os.path.exists(rep):
                    continue
                kname, got, stalls, n_all = full_capture(rep)
                f.write(f"\n## {what}\n# kernel: {kname}\n")
                for k in KEYS:
                    if k in got:
                        f.write(f"{k:70s} {got[k][0]:>16s} {got[k][1]}\n")
                f.write("warp-stall samples (all warps, whole kernel):\n")
                for k, v in stalls:
                    f.write(f"  {k:28s} {v:8.0f}  {v / n_all:6.3f}\n")
                if key == "prism_apply_kernel" and "dram__bytes_read.sum" in got:
                    rd = float(got["dram__bytes_read.sum"][0].replace(",", "")) * SCALE[got["dram__bytes_read.sum"][1]]
                    wr = float(got["dram__bytes_write.sum"][0].replace(",", "")) * SCALE[got["dram__bytes_write.sum"][1]]
                    with open(os.path.join(PROF, f"traffic_{name}.json"), "w") as g:
                        json.dump({"workload": name, "kernel": kname,
                                   "source": f"ncu --set full capture {tag}_{w}_prism_apply_kernel (cold caches)",
                                   "apply_dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd,
                                   "dram_write_bytes": wr}, g, indent=1)
        with open(os.path.join(PROF, f"{tag}_{w}_launches.txt"), "w") as f:
            f.write(f"# {tag}: ncu --metrics gpu__time_duration.sum --clock-control none over\n"
                    f"#   python bench.py --workload {w} --steps 2 --warmup 3 --no-cpu-baseline --no-extra\n"
                    f"# (workload {name}): every launch of the command (warm-up, timed, e2e and profiling\n"
                    "# passes), cold-cache and serialised: compare per-kernel shares, not absolute times.\n\n")
            f.write(launches(tag, w))
        print(name, "done")
    so = os.path.join(ROOT, "paper_2601_22137_b200", "_lib", "libprism.so")
    r = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True)
    import collections
    import re
    cnt = collections.Counter(m.group(0) for m in re.finditer(
        r"\b(UTC[A-Z]*MMA[A-Z0-9.]*|UTMALDG[A-Z0-9.]*|UTMASTG|UBLKCP[A-Z.]*|UTCBAR[A-Z0-9.]*|LDTM[A-Z0-9.]*|HMMA[A-Z0-9.]*)",
        r.stdout))
    with open(os.path.join(PROF, f"{tag}_sass_evidence.txt"), "w") as f:
        f.write("# cuobjdump -sass paper_2601_22137_b200/_lib/libprism.so: tcgen05 / TMA instruction counts\n")
        f.write("# (UTC*MMA = tcgen05.mma, LDTM = tcgen05.ld, UTMALDG = TMA load, UTCBAR = tcgen05.commit;\n")
        f.write("#  no HMMA: no legacy mma.sync path)\n")
        for k, v in sorted(cnt.items()):
            f.write(f"{k:32s} {v}\n")


if __name__ == "__main__":
    main()
