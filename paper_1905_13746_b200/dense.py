"""Dense device API over libgnb.so: the throughput boundary of the hot path.

Tensors are torch CUDA tensors (torch is only the allocator / stream carrier);
every call enqueues one of the hand-written sm_100a kernels on the current
(or given) stream through the C ABI in include/gnb.h.  No CPU fallback: a
non-CUDA tensor is an error.

  fit_stats  -> K-FIT   (features.py:48-53, classifier.py:94-101, corpus.py:302-305)
  fin_train  -> FIN     (features.py:59-86, classifier.py:103-120)  [host C++]
  predict    -> K-PRED  (classifier.py:132-158, engine.py:187-206)
  generate   -> GEN     (synth.py:64-116 law, counter-based)
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .errors import InvalidConfigError


def _stream(stream) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _dev(t: torch.Tensor, name: str, dtype) -> int:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise InvalidConfigError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != dtype:
        raise InvalidConfigError(f"{name} must be {dtype}, got {t.dtype}")
    return t.data_ptr()


_X_TYPES = {torch.int32: N.X_I32, torch.uint16: N.X_U16, torch.uint8: N.X_U8}
_ORDERS = {"auto": N.GNB_ORDER_AUTO, "grouped": N.GNB_ORDER_GROUPED, "mixed": N.GNB_ORDER_MIXED}


def _rows(x: torch.Tensor, name: str = "x", dtypes=(torch.int32,)):
    if isinstance(x, torch.Tensor) and x.dtype in dtypes:
        ptr = _dev(x, name, x.dtype)
    else:
        ptr = _dev(x, name, dtypes[0])
    if x.dim() != 2 or (x.numel() > 0 and x.shape[1] > 1 and x.stride(1) != 1):
        raise InvalidConfigError(f"{name} must be a row-major [N, F] int32 matrix")
    return ptr, x.shape[0], x.shape[1], max(x.stride(0), x.shape[1])


def _vec(t: torch.Tensor, n: int, name: str, dtype=torch.int32) -> int:
    ptr = _dev(t, name, dtype)
    if t.dim() != 1 or t.shape[0] != n or (n > 1 and t.stride(0) != 1):
        raise InvalidConfigError(f"{name} must be a contiguous vector of length {n}")
    return ptr


# ---------------------------------------------------------------- predict
@dataclass
class DeviceTables:
    """A model bundle resident on one device, in the K-PRED layout.

    route[group_count] maps size group -> slot; packed holds the per-slot
    log priors and (ll, -2^52 ll) feature tables (gnb_pack_tables).
    """

    route: torch.Tensor
    packed: torch.Tensor
    n_slots: int
    n_classes: int
    n_features: int
    group_size_bytes: int
    max_size_bytes: int

    @classmethod
    def build(cls, log_prior, log_lik, route, *, group_size_bytes: int, max_size_bytes: int,
              device=None, stream=None) -> "DeviceTables":
        """log_prior [S, C], log_lik [S, C, F] (fp64), route [max/width] -> slot."""
        device = torch.device(device or "cuda")
        lp = torch.as_tensor(log_prior, dtype=torch.float64).to(device).contiguous()
        ll = torch.as_tensor(log_lik, dtype=torch.float64).to(device).contiguous()
        rt = torch.as_tensor(route, dtype=torch.int32).to(device).contiguous()
        if lp.dim() != 2 or ll.dim() != 3 or ll.shape[:2] != lp.shape:
            raise InvalidConfigError("need log_prior [S, C] and log_lik [S, C, F]")
        S, Cn, F = ll.shape
        if rt.numel() != max_size_bytes // group_size_bytes:
            raise InvalidConfigError("route must have one entry per size group")
        if S > 0 and (int(rt.min()) < 0 or int(rt.max()) >= S):
            raise InvalidConfigError("route entries must be valid slots")
        nbytes = N.lib.gnb_packed_table_bytes(S, Cn, F)
        if nbytes == 0:
            raise InvalidConfigError(f"unsupported table shape S={S} C={Cn} F={F}")
        packed = torch.empty(nbytes // 8, dtype=torch.float64, device=device)
        N.check(N.lib.gnb_pack_tables(lp.data_ptr(), ll.data_ptr(), S, Cn, F, packed.data_ptr(),
                                      _stream(stream)), "gnb_pack_tables")
        return cls(rt, packed, S, Cn, F, group_size_bytes, max_size_bytes)


def needs_slot_sort(x_dtype: torch.dtype, tables: DeviceTables) -> bool:
    """True when a ragged batch in arbitrary row order should go through
    slot_sort + predict(perm=...): K-PRED's mixed-slot kernel (every slot's table
    resident in shared memory, rows sorted by slot inside each tile) scores any
    row order at streaming speed whenever gnb_predict_mixed_rows() > 0."""
    if tables.n_slots < 2:
        return False
    return N.lib.gnb_predict_mixed_rows(tables.n_features, _X_TYPES[x_dtype],
                                        tables.n_classes, tables.n_slots) == 0


def slot_sort(size_bytes: torch.Tensor, tables: DeviceTables, *, stream=None) -> torch.Tensor:
    """perm[n]: row indices grouped by routed model slot (device counting sort)."""
    n = size_bytes.shape[0]
    sp = _vec(size_bytes, n, "size_bytes")
    dev = size_bytes.device
    perm = torch.empty(n, dtype=torch.int32, device=dev)
    ws_bytes = N.lib.gnb_slot_sort_workspace_bytes(n, tables.n_slots)
    ws = torch.empty(max(ws_bytes, 4), dtype=torch.uint8, device=dev)
    N.check(N.lib.gnb_slot_sort(sp, n, tables.group_size_bytes, tables.max_size_bytes,
                                tables.route.data_ptr(), tables.n_slots, perm.data_ptr(),
                                ws.data_ptr(), ws.numel(), _stream(stream)), "gnb_slot_sort")
    return perm


def predict(x: torch.Tensor, size_bytes: torch.Tensor, tables: DeviceTables, *,
            logpost: bool = True, label_out=None, logpost_out=None, stream=None,
            generic: bool = False, perm: torch.Tensor | None = None, mode: str = "exact",
            order: str = "auto"):
    """Score every row: label[N] int32 (class index, or -1 size out of range,
    -2 negative count) and, if requested, log-posteriors [N, C] fp64.

    Row n of x holds its routed model's feature counts in FeatureSet order
    (extra columns beyond the model's features must be 0).  x may be int32,
    uint16 or uint8 (the same counts in fewer bytes; identical results).
    perm (from slot_sort): score in slot-grouped order -- for ragged batches
    whose rows are not grouped by size group; results are identical.
    mode: "exact" (default; the reference's mul-then-add roundings, bit-identical
    log-posteriors) or "fma" (one fused rounding per term, ~1e-12 relative).
    order: "auto" (default: the device counts the tiles that mix models and picks
    the kernel, no host sync), "grouped" (rows grouped by size group) or "mixed"
    (rows in any order: the mixed-slot kernel) -- a speed hint; results are
    identical."""
    if mode not in ("exact", "fma"):
        raise InvalidConfigError(f"mode must be 'exact' or 'fma', got {mode!r}")
    if order not in _ORDERS:
        raise InvalidConfigError(f"order must be one of {sorted(_ORDERS)}, got {order!r}")
    if order == "mixed" and perm is None and not generic and needs_slot_sort(x.dtype, tables):
        perm = slot_sort(size_bytes, tables, stream=stream)  # no mixed-slot kernel for this shape
    xp, n, F, ldx = _rows(x, dtypes=tuple(_X_TYPES))
    if F != tables.n_features:
        raise InvalidConfigError(f"x has {F} columns, tables have {tables.n_features} features")
    sp = _vec(size_bytes, n, "size_bytes")
    dev = x.device
    label = label_out if label_out is not None else torch.empty(n, dtype=torch.int32, device=dev)
    lp = None
    if logpost:
        lp = logpost_out if logpost_out is not None else torch.empty(
            (n, tables.n_classes), dtype=torch.float64, device=dev)
    args = (n, F, ldx, sp, tables.group_size_bytes, tables.max_size_bytes,
            tables.route.data_ptr(), tables.n_slots, tables.n_classes, tables.packed.data_ptr(),
            _vec(label, n, "label_out"), lp.data_ptr() if lp is not None else None,
            _stream(stream))
    if mode == "fma" or order != "auto":
        pp = _vec(perm, n, "perm") if perm is not None else None
        a = list(args)
        flags = (N.GNB_MODE_FMA if mode == "fma" else N.GNB_MODE_EXACT) | _ORDERS[order]
        a[10:10] = [pp, flags]   # after packed
        N.check(N.lib.gnb_predict_mode(xp, _X_TYPES[x.dtype], *a), "gnb_predict_mode")
    elif generic:
        if x.dtype != torch.int32:
            raise InvalidConfigError("generic=True is the int32 L1 test path")
        N.check(N.lib.gnb_predict_generic(xp, *args), "gnb_predict_generic")
    elif perm is not None:
        pp = _vec(perm, n, "perm")
        a = list(args)
        a.insert(10, pp)   # after packed
        N.check(N.lib.gnb_predict_permuted(xp, _X_TYPES[x.dtype], *a), "gnb_predict_permuted")
    else:
        N.check(N.lib.gnb_predict_typed(xp, _X_TYPES[x.dtype], *args), "gnb_predict_typed")
    return label, lp


def narrowest(x: torch.Tensor) -> torch.Tensor:
    """The same non-negative counts in the narrowest lossless dtype (uint8 /
    uint16 / int32) -- 4x / 2x fewer bytes for K-PRED to stream."""
    if x.numel() == 0:
        return x
    lo, hi = int(x.min()), int(x.max())
    if lo < 0:
        return x
    if hi < 256:
        return x.to(torch.uint8)
    if hi < 65536:
        return x.to(torch.uint16)
    return x


def pack_u4(x: torch.Tensor, out: torch.Tensor = None) -> torch.Tensor:
    """Host rows of counts < 16 packed two per byte (GNB_X_U4: feature 2j in the
    low nibble of byte j, 2j+1 in the high nibble), each row padded to a
    multiple of 8 bytes -- the layout gnb_predict_host_typed copies in one piece
    and unpacks on the device.  Pass `ldx = 2 * result.shape[1]` (features).
    Raises if a count is outside [0, 16): the storage is lossless or refused."""
    n, F = x.shape
    if x.numel() and (int(x.min()) < 0 or int(x.max()) > 15):
        raise ValueError("pack_u4: counts must be in [0, 16)")
    pb = (F + 15) // 16 * 8
    if out is None:
        out = torch.empty((n, pb), dtype=torch.uint8, pin_memory=torch.cuda.is_available())
    if out.shape != (n, pb) or out.dtype != torch.uint8:
        raise ValueError(f"pack_u4: out must be uint8 [{n}, {pb}]")
    w = torch.zeros((n, 2 * pb), dtype=torch.uint8)
    w[:, :F] = x
    out.copy_(w[:, 0::2] | (w[:, 1::2] << 4))
    return out


def gather_features(x_vocab: torch.Tensor, size_bytes: torch.Tensor, tables: DeviceTables,
                    features, n_features, *, out=None, stream=None) -> torch.Tensor:
    """[N, V] full-vocabulary counts -> [N, F] predict layout (routed FeatureSet order),
    in x_vocab's storage (int32 / uint16 / uint8).

    features: [S, F] vocabulary column per (slot, feature); n_features: [S]."""
    xp, n, V, ldx = _rows(x_vocab, "x_vocab", dtypes=tuple(_X_TYPES))
    dev = x_vocab.device
    feats = torch.as_tensor(features, dtype=torch.int32).to(dev).contiguous()
    nf = torch.as_tensor(n_features, dtype=torch.int32).to(dev).contiguous()
    F = tables.n_features
    if feats.shape != (tables.n_slots, F) or nf.shape != (tables.n_slots,):
        raise InvalidConfigError("features must be [n_slots, F] and n_features [n_slots]")
    if out is None:
        eb = x_vocab.element_size()
        ld = (F * eb + 15) // 16 * 16 // eb     # 16-B row pitch (TMA path of K-PRED)
        full = torch.empty((n, ld), dtype=x_vocab.dtype, device=dev)
        if ld > F:
            full[:, F:].zero_()   # pitch padding: defined bytes for every consumer
        out = full[:, :F]
    if out.dtype != x_vocab.dtype:
        raise InvalidConfigError("out must have x_vocab's dtype")
    op, _, Fo, ldo = _rows(out, "out", dtypes=(x_vocab.dtype,))
    if Fo != F:
        raise InvalidConfigError("out must have F columns")
    N.check(N.lib.gnb_gather_features_typed(
        xp, _X_TYPES[x_vocab.dtype], n, V, ldx, _vec(size_bytes, n, "size_bytes"),
        tables.group_size_bytes, tables.max_size_bytes, tables.route.data_ptr(), feats.data_ptr(),
        nf.data_ptr(), tables.n_slots, F, op, ldo, _stream(stream)), "gnb_gather_features_typed")
    return out


# ---------------------------------------------------------------- fit
@dataclass
class FitStats:
    sums: torch.Tensor      # [G, C, V] fp64 (exact integers)
    sumsq: torch.Tensor | None
    counts: torch.Tensor    # [G, C] fp64
    status: torch.Tensor    # [2] int64: rows with bad label, rows out of size range

    def packed(self) -> torch.Tensor:
        """One flat fp64 buffer {S | Q | n} for a single all-reduce."""
        parts = [self.sums.reshape(-1)]
        if self.sumsq is not None:
            parts.append(self.sumsq.reshape(-1))
        parts.append(self.counts.reshape(-1))
        return torch.cat(parts)

    def unpack_(self, flat: torch.Tensor) -> "FitStats":
        o = 0
        for t in (self.sums, self.sumsq, self.counts):
            if t is None:
                continue
            t.copy_(flat[o:o + t.numel()].view_as(t))
            o += t.numel()
        return self


def fit_stats(x: torch.Tensor, size_bytes: torch.Tensor, labels: torch.Tensor, *,
              n_classes: int, group_size_bytes: int, max_size_bytes: int, sumsq: bool = True,
              out: FitStats | None = None, accumulate: bool = False, stream=None) -> FitStats:
    """Per-(size group, class, column) sums / sums of squares / row counts.
    x may be int32, uint16 or uint8 (same counts, fewer bytes)."""
    xp, n, V, ldx = _rows(x, dtypes=tuple(_X_TYPES))
    if max_size_bytes <= 0 or group_size_bytes <= 0 or max_size_bytes % group_size_bytes:
        raise InvalidConfigError("group_size_bytes must divide max_size_bytes")
    G = max_size_bytes // group_size_bytes
    dev = x.device
    if out is None:
        out = FitStats(
            torch.zeros((G, n_classes, V), dtype=torch.float64, device=dev),
            torch.zeros((G, n_classes, V), dtype=torch.float64, device=dev) if sumsq else None,
            torch.zeros((G, n_classes), dtype=torch.float64, device=dev),
            torch.zeros(2, dtype=torch.int64, device=dev))
    N.check(N.lib.gnb_fit_stats_typed(
        xp, _X_TYPES[x.dtype], n, V, ldx, _vec(size_bytes, n, "size_bytes"),
        _vec(labels, n, "labels"),
        group_size_bytes, max_size_bytes, n_classes, out.sums.data_ptr(),
        out.sumsq.data_ptr() if out.sumsq is not None else None, out.counts.data_ptr(),
        out.status.data_ptr(), 1 if accumulate else 0, _stream(stream)), "gnb_fit_stats_typed")
    return out


# ---------------------------------------------------------------- several GPUs, one process
def fit_stats_sharded(xs, sizes, labels, *, n_classes: int, group_size_bytes: int,
                      max_size_bytes: int, sumsq: bool = True, comms=None) -> list[FitStats]:
    """K-FIT on every device's row shard (xs[d] / sizes[d] / labels[d] resident on
    device d, launched back to back so the devices run concurrently), then the
    fit's one exchange: the library's NCCL communicator all-reduces the packed
    statistics in place over NVLink (gnb_fit_allreduce).  Returns one FitStats
    per device, all equal to a single-device fit of the concatenated rows."""
    from .sharding import Comms
    if not (len(xs) == len(sizes) == len(labels)) or not xs:
        raise InvalidConfigError("need one x / sizes / labels shard per device")
    devs = [x.device.index for x in xs]
    if len(set(devs)) != len(devs):
        raise InvalidConfigError("one shard per device (devices must differ)")
    out = []
    for x, sz, lb in zip(xs, sizes, labels):
        with torch.cuda.device(x.device):
            out.append(fit_stats(x, sz, lb, n_classes=n_classes,
                                 group_size_bytes=group_size_bytes,
                                 max_size_bytes=max_size_bytes, sumsq=sumsq))
    if len(out) > 1:
        (comms or Comms.local_cached(devs)).allreduce(out)
    return out


def predict_sharded(xs, sizes, tables, **kw):
    """K-PRED on every device's shard with that device's replica of the tables
    (tables[d], DeviceTables.build(..., device=d)); no exchange.  Returns
    [(label, logpost)] per device, launched back to back (concurrent)."""
    if not (len(xs) == len(sizes) == len(tables)) or not xs:
        raise InvalidConfigError("need one x / sizes / tables per device")
    out = []
    for x, sz, t in zip(xs, sizes, tables):
        if t.route.device != x.device:
            raise InvalidConfigError("tables[d] must live on shard d's device")
        with torch.cuda.device(x.device):
            out.append(predict(x, sz, t, **kw))
    return out


# ---------------------------------------------------------------- finalize (host C++)
@dataclass
class FinResult:
    state: np.ndarray        # [G] 1 trained, 0 untrainable, -1/-2 insufficient class
    n_features: np.ndarray   # [G]
    features: np.ndarray     # [G, k] column indices (FeatureSet order)
    log_prior: np.ndarray    # [G, 2]  (benign, malware)
    log_lik: np.ndarray      # [G, 2, k]


def fin_train(sums, counts, *, k: int, alpha: float, min_per_class: int) -> FinResult:
    """Feature selection + smoothed log-parameters for every group (C = 2)."""
    S = np.ascontiguousarray(np.asarray(sums, dtype=np.float64))
    n = np.ascontiguousarray(np.asarray(counts, dtype=np.float64))
    if S.ndim != 3 or S.shape[1] != 2 or n.shape != S.shape[:2]:
        raise InvalidConfigError("fin_train needs sums [G, 2, V] and counts [G, 2]")
    G, _, V = S.shape
    res = FinResult(np.zeros(G, np.int32), np.zeros(G, np.int32), np.zeros((G, k), np.int32),
                    np.zeros((G, 2)), np.zeros((G, 2, k)))
    ptr = lambda a: a.ctypes.data  # noqa: E731
    N.check(N.lib.gnb_fin_train(ptr(S), ptr(n), G, V, k, float(alpha), min_per_class,
                                ptr(res.state), ptr(res.n_features), ptr(res.features),
                                ptr(res.log_prior), ptr(res.log_lik)), "gnb_fin_train")
    return res


def fin_train_device(stats: FitStats, *, k: int, alpha: float, min_per_class: int,
                     stream=None) -> FinResult:
    """fin_train with scoring + top-k on the device (C = 2, V <= 16384)."""
    S, n = stats.sums, stats.counts
    if S.dim() != 3 or S.shape[1] != 2:
        raise InvalidConfigError("fin_train_device needs 2-class statistics")
    G, _, V = S.shape
    res = FinResult(np.zeros(G, np.int32), np.zeros(G, np.int32), np.zeros((G, k), np.int32),
                    np.zeros((G, 2)), np.zeros((G, 2, k)))
    ptr = lambda a: a.ctypes.data  # noqa: E731
    N.check(N.lib.gnb_fin_train_device(
        S.contiguous().data_ptr(), n.contiguous().data_ptr(), G, V, k, float(alpha),
        min_per_class, ptr(res.state), ptr(res.n_features), ptr(res.features),
        ptr(res.log_prior), ptr(res.log_lik), _stream(stream)), "gnb_fin_train_device")
    return res


def fin_tables(sums_g, counts_g, features, alpha: float):
    """train_group for one group with a given feature list; any class count."""
    S = np.ascontiguousarray(np.asarray(sums_g, dtype=np.float64))
    n = np.ascontiguousarray(np.asarray(counts_g, dtype=np.float64))
    f = np.ascontiguousarray(np.asarray(features, dtype=np.int32))
    Cn, V = S.shape
    prior = np.zeros(Cn)
    ll = np.zeros((Cn, len(f)))
    N.check(N.lib.gnb_fin_tables(S.ctypes.data, n.ctypes.data, Cn, V, f.ctypes.data, len(f),
                                 float(alpha), prior.ctypes.data, ll.ctypes.data),
            "gnb_fin_tables")
    return prior, ll


# ---------------------------------------------------------------- synthetic data
def generate(n_rows: int, n_cols: int, *, n_classes: int = 2, group_rows=None,
             group_size_bytes: int = 5120, divergence: float = 0.8, seed: int = 0,
             row_offset: int = 0, ldx: int | None = None, col_map=None, out=None,
             device=None, stream=None):
    """Synthetic (x [n, V] int32, size [n], label [n]) following the reference law.

    group_rows: rows per size group of the GLOBAL index space (default: all in
    group 0); rows [row_offset, row_offset + n_rows) are materialised.
    col_map: output column j holds vocabulary column col_map[j] (vocabulary of
    `vocab_cols` = max(col_map)+1 columns) -- i.e. the same samples gathered
    into a FeatureSet order.  out: reuse (x, size, label) buffers."""
    device = torch.device(device or "cuda")
    if out is not None:
        x, size, lab = out
        ld = max(x.stride(0), x.shape[1])
    else:
        ld = ldx or (n_cols + 3) // 4 * 4
        full = torch.empty((n_rows, ld), dtype=torch.int32, device=device)
        if ld > n_cols:
            full[:, n_cols:].zero_()   # pitch padding: defined bytes for every consumer
        x = full[:, :n_cols]
        size = torch.empty(n_rows, dtype=torch.int32, device=device)
        lab = torch.empty(n_rows, dtype=torch.int32, device=device)
    cmap = None
    vocab_cols = n_cols
    if col_map is not None:
        cm = np.asarray(col_map, dtype=np.int32)
        if cm.shape != (n_cols,) or cm.min() < 0:
            raise InvalidConfigError("col_map must give one vocabulary column per output column")
        vocab_cols = int(cm.max()) + 1
        cmap = torch.from_numpy(cm).to(device)
    if group_rows is None:
        group_rows = [row_offset + n_rows]
    ends = np.cumsum(np.asarray(group_rows, dtype=np.int64))
    N.check(N.lib.gnb_generate(x.data_ptr(), n_rows, n_cols, ld, size.data_ptr(),
                               lab.data_ptr(), row_offset, ends.ctypes.data, len(ends),
                               group_size_bytes, n_classes, float(divergence), seed,
                               cmap.data_ptr() if cmap is not None else None, vocab_cols,
                               _stream(stream)), "gnb_generate")
    return x, size, lab
