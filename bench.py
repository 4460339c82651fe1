"""Benchmark: EXPRB4 steps/s at 655k cells (fp64) on B200, plus the
J*v+IOM2 roofline -- BASELINE.json's metric on config C3.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config C3] [--scheme exprb42] [--no-cpu-baseline]

One process per GPU (torchrun for N > 1).  The path does not shard (SURVEY.md
§8e: replicas only): every rank integrates its own trajectory of the same
workload on its own GPU, with no data-path collective; ``value`` is the sum of
steps over ranks divided by the max-over-ranks device time ("weak" scaling).

A step is one EXPRB4 step of the resident state: F(u_n), eta, n_A, two
phipm/IOM2 engine calls, the stage perturbation.  Both arms time the same
steps: trajectory steps 1-2 of the config from its seeded initial state with
cold engine seeds (the reference arm's bounded CPU sample); the GPU arm
replays that episode K times, restoring the initial state and seeds from a
device-side snapshot at the start of each episode.  ``full_run`` adds the
device time of the config's whole stated run (C3: 144 steps, one day).
Each step is one CUDA graph
(libeik's split step: a continuation kernel and, under a device-driven while
node, one cooperative Krylov-sweep kernel ``k_swe_sweep`` per IOM2 sweep plus
its dense phi kernel).  Timing: CUDA events recorded by libeik around every
step graph on its stream, barrier + device synchronise before and after the
timed loop.  The roofline is that of ``k_swe_sweep``, timed with CUDA events
around each sweep launch in a second pass of the same steps launched kernel by
kernel (host-loop mode: conditional graph nodes hide their kernels).  Each Krylov iteration
streams ~0.5 GB, far more than the 126 MB L2, so no explicit flush is done.

``--impl reference`` times the reference algorithm's CPU implementation (the
numpy/scipy oracle port in oracle/, the reference itself being Python that
cannot travel to the GPU box) on the host cores, rank 0 only.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "EXPRB4 steps/s at 655k cells fp64; J*v+IOM2 achieved HBM GB/s vs peak"
FALLBACK_HBM = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--scheme", default="exprb42")
    ap.add_argument("--level", type=int, default=None, help="grid level override (C4: 9 or 10)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=0,
                    help="steps of the e2e replay (default: all timed steps)")
    ap.add_argument("--sweep-steps", type=int, default=0,
                    help="timed steps replayed for the sweep roofline (default: all)")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    return FALLBACK_HBM, "fallback"


def b_alg_per_iter(ops):
    """N*(96+64+24) + 8*W_coef, W_coef = nnz of the distinct
    CSR arrays among Gx..Vz, L."""
    seen, wc = [], 0
    for name in ("Gx", "Gy", "Gz", "Dx", "Dy", "Dz", "Vx", "Vy", "Vz", "L"):
        c = getattr(ops, name).csr
        key = (c.nnz, c.data[:8].tobytes(), c.data[-8:].tobytes() if c.nnz else b"")
        if key in seen:
            continue
        seen.append(key)
        wc += c.nnz
    return ops.n_g * (96 + 64 + 24) + 8 * wc


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None
        self.tmp = None

    def start(self):
        try:
            self.tmp = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=self.tmp, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.tmp.flush()
        with open(self.tmp.name) as fh:
            lines = [l.strip() for l in fh if l.strip()]
        os.unlink(self.tmp.name)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


EPISODE = 2  # trajectory steps timed by both arms (the reference arm's bounded sample)


def workload(cfg, ops, spec, scheme):
    """One workload string for both arms (the driver compares them)."""
    return (f"{cfg}: L{ops.level} icosahedral ({ops.n_g} cells) {scheme} dt={spec.dt}s "
            f"tol={spec.tol}; trajectory steps 1-{EPISODE} from the seeded initial state "
            f"(cold engine seeds), replayed")


def cpu_baseline_oracle(ops, u0, spec, scheme, nsteps):
    """The oracle port (numpy/scipy restatement of the reference) on the host
    cores: trajectory steps 1..nsteps from the config's initial state."""
    from oracle import integrate_oracle, swe_problem
    t = time.perf_counter()
    integrate_oracle(swe_problem(ops), scheme, u0, spec.dt, nsteps * spec.dt, tol=spec.tol)
    return time.perf_counter() - t


def run_reference(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = str(threads)
    from paper_1805_02144_b200.states import make_config
    ops, u0, spec = make_config(args.config, level=args.level)
    nsteps = EPISODE
    secs = cpu_baseline_oracle(ops, u0, spec, args.scheme, nsteps)
    value = nsteps / secs
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "steps/s",
        "n_gpus": ws, "steps": nsteps, "warmup": 0, "ms_per_step": 1e3 * secs / nsteps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded BASELINE C3 jet state on our icosahedral grid)",
        "config": {"workload": workload(args.config, ops, spec, args.scheme),
                   "cells": ops.n_g},
        "cpu_baseline": {"value": value, "unit": "steps/s", "cores": threads,
                         "kind": "port",
                         "sample": f"trajectory steps 1-{nsteps} of {args.config} "
                                   f"{args.scheme} from the seeded initial state (cold engine "
                                   "seeds), timed once; scipy csr_matvec is "
                                   "single-threaded, BLAS uses all cores"},
        "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def self_launch(args):
    """--gpus N without torchrun: re-run this script under torch.distributed.run
    with N processes on this node (127.0.0.1 rendezvous)."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    ws, rank, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    if ws != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}\n")
        return 2
    if args.impl == "reference":
        return run_reference(args)
    dist = None
    if ws > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    import torch
    from paper_1805_02144_b200 import _native as nat
    from paper_1805_02144_b200 import swe as gswe
    from paper_1805_02144_b200.states import make_config

    ops, u0, spec = make_config(args.config, level=args.level)
    scheme = args.scheme
    ctx = gswe.SweContext(ops, device=local)
    ctx.set_state(u0)
    ctx.set_prev(None)
    ctx.reset_seeds()
    ctx.snapshot()  # trajectory start: initial state, cold seeds

    def step(i):
        """Timed unit: trajectory step (i mod EPISODE) + 1; the episode
        restarts from the device snapshot of the initial state."""
        k = i % EPISODE
        if k == 0:
            ctx.snapshot(restore=True)
        sch = "rb_euler" if (scheme == "epi3" and k == 0) else scheme
        return ctx.step(sch, spec.dt, spec.tol)

    for w in range(args.warmup):
        step(w)
    torch.cuda.synchronize(local)
    if dist:
        dist.barrier()
    clk = ClockSampler(local)
    clk.start()
    l0 = ctx.launches()
    k0 = ctx.krylov_iters()
    dev_ms = 0.0
    mv = 0
    t0 = time.perf_counter()
    step_ms = []
    for i in range(args.steps):
        calls = step(i)
        step_ms.append(ctx.last_kernel_ms())
        dev_ms += step_ms[-1]
        mv += sum(int(c.matvecs) for c in calls)
    torch.cuda.synchronize(local)
    wall = time.perf_counter() - t0
    if dist:
        dist.barrier()
    clocks = clk.stop()
    launches = ctx.launches() - l0
    kiters = ctx.krylov_iters() - k0
    from paper_1805_02144_b200.replicas import aggregate_throughput
    value, ms = aggregate_throughput(args.steps, dev_ms, dist, f"cuda:{local}")
    ms_per_step = ms / args.steps

    # end to end through the C ABI: the same steps, each step's input state
    # copied in from pinned host memory and its result copied back (step k's
    # result is step k+1's input; an episode starts from the host initial
    # state with cold seeds)
    pins = [torch.empty(4 * ops.n_g, dtype=torch.float64).pin_memory() for _ in range(3)]
    bufs = [p.numpy() for p in pins]
    bufs[2][:] = u0
    args.e2e_steps = args.steps if args.e2e_steps <= 0 else min(args.e2e_steps, args.steps)
    torch.cuda.synchronize(local)
    e2e_dev_ms = 0.0
    te = time.perf_counter()
    for i in range(args.e2e_steps):
        k = i % EPISODE
        hin = bufs[2] if k == 0 else bufs[(i - 1) & 1]
        hout = bufs[i & 1]
        if k == 0:
            ctx.set_prev(None)
            ctx.reset_seeds()
        nat.check(nat.load().eik_swe_set_state(ctx.h, nat.dptr(hin)), "set_state")
        sch = "rb_euler" if (scheme == "epi3" and k == 0) else scheme
        ctx.step(sch, spec.dt, spec.tol)
        e2e_dev_ms += ctx.last_kernel_ms()
        nat.check(nat.load().eik_swe_get_state(ctx.h, nat.dptr(hout)), "get_state")
    e2e_wall = time.perf_counter() - te
    e2e, _ = aggregate_throughput(args.e2e_steps, 1e3 * e2e_wall, dist, f"cuda:{local}")

    # the dominant kernel alone: the timed steps replayed kernel by kernel
    # (host-loop mode, identical results), every Krylov sweep kernel
    # bracketed by CUDA events on the libeik stream
    nsw_steps = args.steps if args.sweep_steps <= 0 else min(args.sweep_steps, args.steps)
    ctx.set_hostloop(True)
    ctx.sweep_timing(reset=True)
    k1 = ctx.krylov_iters()
    for i in range(nsw_steps):
        step(i)
    torch.cuda.synchronize(local)
    sweep_ms, nsweeps = ctx.sweep_timing(reset=True)
    sweep_iters = ctx.krylov_iters() - k1
    ctx.set_hostloop(False)

    # the config's whole stated run (C3: 144 steps = 1 day) from the initial
    # state, graph-replayed: the representative average over the trajectory
    ctx.snapshot(restore=True)
    day_ms, day_mv = 0.0, 0
    kd = ctx.krylov_iters()
    for k in range(spec.steps):
        sch = "rb_euler" if (scheme == "epi3" and k == 0) else scheme
        calls = ctx.step(sch, spec.dt, spec.tol)
        day_ms += ctx.last_kernel_ms()
        day_mv += sum(int(c.matvecs) for c in calls)
    day_iters = ctx.krylov_iters() - kd

    hbm, src = peaks()
    balg = b_alg_per_iter(ops)
    it_per_step = kiters / args.steps
    # roofline of k_swe_sweep: algorithmic bytes per launch (B_alg x the
    # launch's Krylov iterations) / average launch duration
    achieved = balg * sweep_iters / (sweep_ms / 1e3) / 1e9
    iters_per_launch = sweep_iters / max(nsweeps, 1)
    # whole step: every J*v pass at B_alg + the candidate's basis reads
    step_bytes = balg * mv + 32.0 * ops.n_g * kiters
    step_achieved = step_bytes / (dev_ms / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as fh:
            tr = json.load(fh)
        if tr.get("cells") == ops.n_g and tr.get("kernel") == "k_swe_sweep":
            traffic = tr["dram_bytes_per_iter"] * iters_per_launch
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return 0
    line = {
        "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded BASELINE C3 jet state on our icosahedral grid)",
        "config": {"workload": workload(args.config, ops, spec, scheme),
                   "cells": ops.n_g, "parallelism": f"replicas x{ws}",
                   "l2": "no flush: inputs > L2 (each Krylov iteration streams ~0.5 GB)"},
        "krylov_iters_per_step": it_per_step, "matvecs_per_step": mv / args.steps,
        "wall_ms_per_step": 1e3 * wall / args.steps,
        "full_run": {"steps": spec.steps, "device_ms": day_ms,
                     "steps_per_s": 1e3 * spec.steps / day_ms,
                     "matvecs_per_step": day_mv / spec.steps,
                     "krylov_iters_per_step": day_iters / spec.steps,
                     "note": f"the config's whole stated run ({spec.steps} x {spec.dt}s) from "
                             "the initial state, device time of the step graphs"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": traffic,
                     "kernel": "k_swe_sweep",
                     "launches": nsweeps, "iters_per_launch": iters_per_launch,
                     "us_per_iter": 1e3 * sweep_ms / max(sweep_iters, 1),
                     "sweep_share_of_step": sweep_ms / sum(step_ms[:nsw_steps]),
                     "step_achieved": step_achieved, "step_frac": step_achieved / hbm,
                     "note": f"kernel = k_swe_sweep (one IOM2 Krylov sweep per launch, "
                             f"{iters_per_launch:.1f} iterations avg); achieved = B_alg "
                             f"{balg / 1e6:.1f} MB x iterations / CUDA-event time of the "
                             f"sweep launches ({nsweeps} launches over the "
                             f"{nsw_steps} timed steps replayed in host-loop "
                             f"mode); traffic = ncu DRAM bytes per iteration of one captured "
                             f"launch (profiles/traffic.json) x iterations per launch; "
                             f"step_* = every J*v pass + candidate reads over the whole "
                             f"graph-replayed step; peak {src} (MEASURED_PEAKS.json hbm_gbs)"},
        "e2e": {"value": e2e, "unit": "steps/s", "h2d_bytes_per_step": 8 * 4 * ops.n_g,
                "d2h_bytes_per_step": 8 * 4 * ops.n_g, "steps": args.e2e_steps,
                "wall_ms_per_step": 1e3 * e2e_wall / args.e2e_steps,
                "device_ms_per_step": e2e_dev_ms / args.e2e_steps},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if ws == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        secs = cpu_baseline_oracle(ops, u0, spec, scheme, 1)
        line["cpu_baseline"] = {
            "value": 1.0 / secs, "unit": "steps/s", "cores": threads, "kind": "port",
            "sample": f"trajectory step 1 of {args.config} {scheme} from the initial state "
                      "(oracle port, cold seeds); scipy csr_matvec single-threaded"}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
