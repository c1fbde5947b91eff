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


# ---------------------------------------------------------------- one process per GPU
def fit_distributed(x, size_bytes, labels, *, n_classes: int, group_size_bytes: int,
                    max_size_bytes: int, sumsq: bool = True, group=None, fit=None):
    """This rank's row shard -> K-FIT -> the fit's one exchange (SUM all-reduce
    of the packed statistics).  Every rank returns the statistics of ALL rows,
    identical to a single-device fit of the concatenated shards.
    `fit` (default dense.fit_stats) produces the local statistics."""
    if fit is None:
        from .dense import fit_stats as fit
    st = fit(x, size_bytes, labels, n_classes=n_classes, group_size_bytes=group_size_bytes,
             max_size_bytes=max_size_bytes, sumsq=sumsq)
    return allreduce_stats(st, group=group)


def train_distributed(x, size_bytes, labels, *, k: int, alpha: float, group_size_bytes: int,
                      max_size_bytes: int, min_per_class: int, group=None, fit=None):
    """fit_distributed (2 classes) + the host finalize (scores, top-k, libm
    logs): every rank gets the same FinResult, bit-identical for any world size
    (train_bundle's dense form, engine.py:157-177)."""
    from .dense import fin_train
    st = fit_distributed(x, size_bytes, labels, n_classes=2, group_size_bytes=group_size_bytes,
                         max_size_bytes=max_size_bytes, sumsq=False, group=group, fit=fit)
    return fin_train(st.sums.cpu().numpy(), st.counts.cpu().numpy(), k=k, alpha=alpha,
                     min_per_class=min_per_class)


def gather_rows(local, group=None):
    """Concatenate every rank's rows of `local` (a tensor) in rank order -- the
    sharded predict's optional output collection (predict itself needs no
    collective).  Shards may differ in length (ceil chunking)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return local
    world = dist.get_world_size(group)
    dev = local.device if dist.get_backend(group) == "nccl" else torch.device("cpu")
    n = torch.tensor([local.shape[0]], dtype=torch.int64, device=dev)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    ns = [int(v.item()) for v in ns]
    m = max(ns)
    buf = torch.zeros((m,) + tuple(local.shape[1:]), dtype=local.dtype, device=dev)
    buf[:local.shape[0]] = local.to(dev)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([p[:c] for p, c in zip(parts, ns)]).to(local.device)


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

    _local_cache: dict = {}

    @classmethod
    def local_cached(cls, devices) -> "Comms":
        """Comms.local for a device tuple, created once per process (ncclCommInitAll
        costs far more than the all-reduce it serves)."""
        key = tuple(int(d) for d in devices)
        c = cls._local_cache.get(key)
        if c is None:
            c = cls._local_cache[key] = cls.local(list(key))
        return c

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
