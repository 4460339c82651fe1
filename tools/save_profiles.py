"""Copy a round's bench lines and ncu summaries into profiles/ (tracked)."""
import csv, io, json, os, subprocess, sys
from collections import defaultdict
tag = sys.argv[1]
src = "gpurun_out"
dst = "profiles"
os.makedirs(dst, exist_ok=True)
for f in (f"bench_{tag}.json", f"bench_ref_{tag}.json"):
    p = os.path.join(src, f)
    if os.path.exists(p):
        open(os.path.join(dst, f), "w").write(open(p).read())
p = os.path.join(src, f"launches_{tag}.csv")
if os.path.exists(p):
    rows = list(csv.reader(open(p)))
    k = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[k], rows[k + 1:]
    ki, mi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) > mi:
            name = r[ki].split("(")[0]
            agg[name][0] += 1
            agg[name][1] += float(r[mi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    with open(os.path.join(dst, f"launches_{tag}.txt"), "w") as fh:
        fh.write("ncu --metrics gpu__time_duration.sum --clock-control none "
                 "(python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1); "
                 "cold-cache serialised launches, compare shares\n")
        for name, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            fh.write(f"{name:24s} launches={n:4d} total_ns={t:14.0f} share={100 * t / tot:6.2f}%\n")
rep = os.path.join(src, f"step_{tag}.ncu-rep")
kskip = int(os.environ.get("KSKIP", "4"))
kp = os.path.join(src, f"kskip_{tag}.txt")
if os.path.exists(kp):
    kskip = int(open(kp).read().strip().split("=")[1])
if os.path.exists(rep):
    out = subprocess.run([sys.executable, "tools/ncu_summary.py", rep], capture_output=True, text=True).stdout
    r = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(r.stdout)))
    hdr = rows[0]
    si, mi, ui, vi = (hdr.index(x) for x in ("Section Name", "Metric Name", "Metric Unit", "Metric Value"))
    det = [f"{r[si][:30]:30s} {r[mi]:48s} {r[vi]:>16s} {r[ui]}" for r in rows[1:]
           if r[si] in ("GPU Speed Of Light Throughput", "Memory Workload Analysis", "Occupancy",
                        "Launch Statistics", "Warp State Statistics", "Compute Workload Analysis")]
    # Krylov iterations of the captured launch (EIK_SWEEP_LOG lines of the ncu run)
    iters = None
    # the plain (non-ncu) run of the same command: identical sweep sequence
    logp = os.path.join(src, f"plain_{tag}.log")
    if os.path.exists(logp):
        for line in open(logp):
            if line.startswith(f"[eik] sweep {kskip} iters "):
                iters = int(line.split()[4])
                break
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True)
    rr = list(csv.reader(io.StringIO(raw.stdout)))
    h, u, v = rr[0], rr[1], rr[2]

    def metric(name):
        x = float(v[h.index(name)].replace(",", ""))
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}
        return x * scale.get(u[h.index(name)], 1.0)
    dram = metric("dram__bytes_read.sum") + metric("dram__bytes_write.sum")
    with open(os.path.join(dst, f"ncu_full_k_swe_sweep_{tag}.txt"), "w") as fh:
        fh.write(f"ncu --set full --clock-control none -k regex:k_swe_sweep -s {kskip} -c 1 "
                 f"(one Krylov sweep launch of a C3 L8 exprb42 step, host-loop mode; "
                 f"{iters} Krylov iterations in the launch; DRAM bytes per iteration "
                 f"{dram / iters / 1e6 if iters else float('nan'):.1f} MB)\n\n{out}\n\n"
                 + "\n".join(det) + "\n")
    if iters:
        json.dump({"source": f"profiles/ncu_full_k_swe_sweep_{tag}.txt", "kernel": "k_swe_sweep",
                   "cells": 655362, "dram_bytes_per_launch": dram, "krylov_iters_in_launch": iters,
                   "dram_bytes_per_iter": dram / iters},
                  open(os.path.join(dst, "traffic.json"), "w"), indent=1)
# the continuation and dense kernels (one launch each)
for kern, stem in (("k_swe_cont", "cont"), ("k_swe_dense", "dense")):
    rep = os.path.join(src, f"{stem}_{tag}.ncu-rep")
    if not os.path.exists(rep):
        continue
    out = subprocess.run([sys.executable, "tools/ncu_summary.py", rep], capture_output=True, text=True).stdout
    r = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(r.stdout)))
    hdr = rows[0]
    si, mi, ui, vi = (hdr.index(x) for x in ("Section Name", "Metric Name", "Metric Unit", "Metric Value"))
    det = [f"{r[si][:30]:30s} {r[mi]:48s} {r[vi]:>16s} {r[ui]}" for r in rows[1:]
           if r[si] in ("GPU Speed Of Light Throughput", "Memory Workload Analysis", "Occupancy",
                        "Launch Statistics", "Warp State Statistics", "Compute Workload Analysis")]
    with open(os.path.join(dst, f"ncu_full_{kern}_{tag}.txt"), "w") as fh:
        fh.write(f"ncu --set full --clock-control none -k regex:{kern} -s 3 -c 1 (host-loop "
                 f"mode, C3 L8 exprb42 bench steps)\n\n{out}\n\n" + "\n".join(det) + "\n")
print(sorted(os.listdir(dst)))
