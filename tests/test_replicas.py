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
