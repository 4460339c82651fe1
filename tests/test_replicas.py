"""Multi-rank (world_size 2, gloo, CPU) coverage of the replica path used by
bench.py --gpus N: independent trajectories, max-over-ranks time, summed
throughput."""

import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1805_02144_b200.replicas import aggregate_throughput, max_over_ranks


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        local_ms = 100.0 + 50.0 * rank          # rank 1 is the slow one
        value, ms = aggregate_throughput(10, local_ms, dist)
        # each replica runs the same workload independently (oracle on a small
        # grid stands in for the device step on CPU)
        from oracle import integrate_oracle, swe_problem
        from paper_1805_02144_b200.states import make_config
        ops, u0, spec = make_config("C0", level=2)
        u, steps, _, _ = integrate_oracle(swe_problem(ops), "exprb42", u0, spec.dt,
                                          2 * spec.dt, tol=1e-6)
        digest = float(np.linalg.norm(u))
        dg = max_over_ranks(digest, dist)
        out[rank] = (value, ms, digest, dg)
    finally:
        dist.destroy_process_group()


def test_two_rank_replicas():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    (v0, ms0, d0, g0), (v1, ms1, d1, g1) = out[0], out[1]
    assert ms0 == ms1 == 150.0                     # max over ranks
    assert v0 == v1 == pytest.approx(2 * 10 / 0.150)
    assert d0 == d1 == g0 == g1                    # identical independent replicas


def test_single_process_identity():
    assert max_over_ranks(3.5) == 3.5
    v, ms = aggregate_throughput(4, 200.0)
    assert ms == 200.0 and v == pytest.approx(20.0)


def test_bench_gpus_flag_self_launches_ranks():
    """`bench.py --gpus 2` without torchrun re-launches itself with two ranks
    (127.0.0.1 rendezvous); the reference arm prints one line from rank 0
    with n_gpus = 2 (CPU-only: the reference arm needs no device)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env["OMP_NUM_THREADS"] = "1"
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2",
                        "--impl", "reference", "--config", "C0", "--steps", "2",
                        "--warmup", "1"], capture_output=True, text=True, timeout=600,
                       env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0


def test_bench_rejects_world_size_mismatch():
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2",
                        "--impl", "reference", "--config", "C0"], capture_output=True,
                       text=True, timeout=300, env=env, cwd=root)
    assert r.returncode == 2 and "WORLD_SIZE" in r.stderr
