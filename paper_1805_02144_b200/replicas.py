"""Replica-parallel timing helpers (the path does not shard).

Every rank integrates its own trajectory on its own GPU with no data-path
collective; only the timing is combined: the job time is the max of the
per-rank device times and the throughput counts every rank's steps.
"""


def max_over_ranks(x, dist=None, device="cpu"):
    """Max of a scalar over all ranks (identity without a process group)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_throughput(steps_per_rank, local_ms, dist=None, device="cpu"):
    """(value steps/s over the whole job, max-over-ranks ms) for `steps_per_rank`
    steps timed as `local_ms` milliseconds of device time on this rank."""
    ws = 1 if dist is None or not dist.is_initialized() else dist.get_world_size()
    ms = max_over_ranks(local_ms, dist, device)
    return ws * steps_per_rank / (ms / 1e3), ms
