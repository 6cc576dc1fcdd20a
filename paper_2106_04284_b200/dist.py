"""Multi-GPU plumbing for the data-parallel copy: one process
per GPU, torch.distributed for barriers and the over-ranks reductions of one
timing number only -- there is no data-path collective, every rank relayouts
its own records.  bench.py's rank context calls these."""
import os


def env_rank():
    """(rank, world size, local rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def _active():
    import torch.distributed as dist
    return dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1


def _reduce(value, op, device):
    import torch
    import torch.distributed as dist
    if not _active():
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=op)
    return float(t.item())


def max_over_ranks(value, device=None):
    """All-reduce(MAX) of one float (the slowest rank's time); identity when not distributed."""
    import torch.distributed as dist
    return _reduce(value, dist.ReduceOp.MAX, device)


def sum_over_ranks(value, device=None):
    """All-reduce(SUM) of one float (bytes moved by all ranks); identity when not distributed."""
    import torch.distributed as dist
    return _reduce(value, dist.ReduceOp.SUM, device)


def barrier():
    import torch.distributed as dist
    if _active():
        dist.barrier()
