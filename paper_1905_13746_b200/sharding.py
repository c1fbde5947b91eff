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


class Comms:
    """The library's own NCCL communicator (gnb_comms_* in include/gnb.h), for
    callers without torch.distributed: one process driving several GPUs
    (`Comms.local([0, 1, ...])`, ncclCommInitAll) or one process per GPU
    (`Comms.rank(nranks, rank, uid, device)` with `uid = Comms.unique_id()`
    from rank 0).  `allreduce(stats_per_device, streams)` is the fit's one
    exchange: every device's packed statistics summed in place."""

    def __init__(self, handle: int):
        self._h = handle

    @staticmethod
    def unique_id() -> bytes:
        import ctypes as C
        from . import _native as N
        buf = (C.c_uint8 * 128)()
        N.check(N.lib.gnb_comms_unique_id(buf), "gnb_comms_unique_id")
        return bytes(buf)

    @classmethod
    def local(cls, devices) -> "Comms":
        import ctypes as C
        from . import _native as N
        devs = (C.c_int32 * len(devices))(*devices)
        h = C.c_void_p()
        N.check(N.lib.gnb_comms_init(C.byref(h), len(devices), devs), "gnb_comms_init")
        return cls(h.value)

    @classmethod
    def rank(cls, nranks: int, rank: int, uid: bytes, device: int) -> "Comms":
        import ctypes as C
        from . import _native as N
        if len(uid) != 128:
            raise ValueError("uid must be the 128 bytes of Comms.unique_id()")
        h = C.c_void_p()
        N.check(N.lib.gnb_comms_init_rank(C.byref(h), nranks, rank,
                                          (C.c_uint8 * 128).from_buffer_copy(uid), device),
                "gnb_comms_init_rank")
        return cls(h.value)

    def __len__(self) -> int:
        from . import _native as N
        return int(N.lib.gnb_comms_size(self._h))

    def allreduce(self, stats_per_device, streams=None):
        """SUM-all-reduce one dense.FitStats per local device, in place."""
        import ctypes as C
        import torch
        from . import _native as N
        if len(stats_per_device) != len(self):
            raise ValueError(f"need one FitStats per local device ({len(self)})")
        flats = [s.packed() for s in stats_per_device]
        if len({f.numel() for f in flats}) != 1:
            raise ValueError("statistics buffers differ in size")
        if streams is None:
            streams = [torch.cuda.current_stream(f.device) for f in flats]
        bufs = (C.c_void_p * len(flats))(*[f.data_ptr() for f in flats])
        strs = (C.c_size_t * len(flats))(*[int(s.cuda_stream) for s in streams])
        N.check(N.lib.gnb_fit_allreduce(self._h, bufs, flats[0].numel(), strs),
                "gnb_fit_allreduce")
        for s, f in zip(stats_per_device, flats):
            s.unpack_(f)
        return stats_per_device

    def close(self) -> None:
        h, self._h = self._h, None
        if h:
            from . import _native as N
            N.lib.gnb_comms_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
