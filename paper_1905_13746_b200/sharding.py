"""Multi-GPU plumbing: one process per GPU, rows sharded contiguously.

Predict needs no collective (samples are independent; the <= 100 KB model
tables are replicated).  Fit has exactly one exchange: the packed fp64
statistics buffer {sums | sumsq | counts} is all-reduced (SUM) once.  Every
value in it is an integer < 2^53, so the reduction is exact and
order-independent and the fitted bundle is bit-identical for any number of
GPUs (engine.classify_parallel's chunking, engine.py:264-268, restated per GPU).
"""

from __future__ import annotations


def shard_bounds(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [lo, hi) of rank's rows: ceil(n/world)-sized chunks (engine.py:267-268)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    chunk = -(-n_total // world) if n_total else 0
    lo = min(rank * chunk, n_total)
    return lo, min(lo + chunk, n_total)


def allreduce_stats(stats, group=None):
    """SUM-all-reduce a dense.FitStats (or any object with packed()/unpack_()) in place.

    One collective per fit: NCCL over NVLink on GPUs, gloo in the CPU tests."""
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return stats
    flat = stats.packed()
    if dist.get_backend(group) == "gloo" and flat.is_cuda:   # gloo reduces host tensors
        host = flat.cpu()
        dist.all_reduce(host, op=dist.ReduceOp.SUM, group=group)
        return stats.unpack_(host.to(flat.device))
    dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    return stats.unpack_(flat)
