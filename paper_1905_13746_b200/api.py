"""The reference's fit / classify operation contract, executed on the GPU.

Drop-in for the hot path of `groupnb` (reference pkg/src/groupnb):

  train_bundle(train, k, alpha=1.0, *, seed=0, created_at=None)  engine.py:157-177
  train_bundles(train, k_values, alpha=1.0, *, seed=0, created_at="")
                                                                  bench.py:91-111
  train_group(samples, features, alpha=1.0, *, group=0)           classifier.py:68-129
  classify_parallel(bundle, workload, *, warmup=True)   (Tp)      engine.py:250-296
  classify_sequential(bundle, workload, *, warmup=True) (Tc)      engine.py:209-226
  log_posterior(model, histogram) / predict(model, histogram)     classifier.py:132-158

Same arguments, same results (bit-identical log-scores and bundles), same
exception types and messages.  Every function accepts EITHER this package's
object model (model.py) OR the reference's own `groupnb` objects, and answers
in the caller's types (`_ns.of`): a `groupnb.GroupedCorpus` trains into a
`groupnb.ModelBundle` of `groupnb.GroupModel`s, a `groupnb` bundle classifies
into `groupnb.TimedRun`s of `groupnb.Prediction`s, and errors are
`groupnb.errors.*` -- so `backend.install()` can put these functions behind the
reference's own API.

Where the work runs:
  * fit (`train_*`) and Tp (`classify_parallel` / `classify_gpu`): the GPU --
    the histograms are densified on the host by `_adapt` (C API, threaded)
    and handed to libgnb.so's host-buffer entry points (K-FIT + FIN,
    K-PRED), one device or several (`devices=`, contiguous row shards).
  * Tc (`classify_sequential`) and the per-sample `log_posterior` / `predict`:
    one host thread (`_adapt.classify_slice` / `score_packed`, C), because the
    reference defines Tc as "never parallelized internally" (engine.py:212-215)
    -- it is the baseline side of `speedup(Tc, Tp)` -- and a single histogram
    costs less on the host than a device round trip.  Same arithmetic and
    order as the kernel, so Tc and Tp agree bit for bit.
"""

from __future__ import annotations

import ctypes
import time
import weakref
from datetime import datetime, timezone
from typing import Sequence

import numpy as np

from . import _adapt
from . import _native as N
from . import _ns
from .model import GroupingConfig, oversize_message

_I32_MAX = 2**31 - 1


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _device_ordinal(device) -> int:
    if device is None:
        return 0
    if isinstance(device, int):
        return device
    idx = getattr(device, "index", None)
    return 0 if idx is None else int(idx)


def _device_list(device, devices) -> list[int]:
    """devices=None -> [device]; an int N -> the first N GPUs; else the ordinals."""
    if devices is None:
        return [_device_ordinal(device)]
    if isinstance(devices, int) and not isinstance(devices, bool):
        if devices < 1:
            raise ValueError(f"devices must be >= 1, got {devices}")
        return list(range(devices))
    out = [_device_ordinal(d) for d in devices]
    if not out:
        raise ValueError("devices must not be empty")
    return out


def _labels(samples, ns) -> np.ndarray:
    """Class codes by identity with the caller's Label members: benign 0,
    malware 1, anything else (UNKNOWN, foreign objects) -1."""
    size = np.empty(len(samples), dtype=np.int32)
    label = np.empty(len(samples), dtype=np.int32)
    _adapt.meta_into(samples, 1, ns.MALWARE, ns.BENIGN, size, label)
    return label


def _densify(samples: Sequence, columns: dict[str, int], width: int) -> np.ndarray:
    """[N, width] int32 counts of the opcodes in `columns` (others ignored)."""
    x = np.zeros((len(samples), width), dtype=np.int32)
    _adapt.densify_into(samples, columns, x, width)
    return x


def _dense_vocab(samples: Sequence):
    """[N, max(V, 1)] int32 counts over the sorted union of opcodes (the
    vocabulary score_opcodes ranges over, features.py:71) and that vocabulary:
    one C-API walk of the histograms discovers the opcodes (first-seen columns)
    while densifying; the columns are then put in mnemonic order."""
    fast = _adapt.vocab_dense(samples)          # threaded walk (None: serial rules apply)
    if fast is not None:
        ops, buf = fast
        return np.frombuffer(buf, dtype=np.int32).reshape(len(samples), max(len(ops), 1)), ops
    width = 512
    while True:
        columns: dict[str, int] = {}
        ops: list[str] = []
        raw = np.zeros((len(samples), width), dtype=np.int32)
        if _adapt.discover_into(samples, columns, ops, raw, width):
            break
        width *= 4
    order = np.asarray(sorted(range(len(ops)), key=ops.__getitem__), dtype=np.int64)
    x = np.zeros((len(samples), max(len(ops), 1)), dtype=np.int32)
    if len(ops):
        _adapt.permute_columns(raw, width, order, x)
    return x, [ops[j] for j in order.tolist()]


def _fit_stats_host(x: np.ndarray, gid: np.ndarray, label: np.ndarray, *, n_classes: int,
                    n_groups: int, devices: list[int]):
    """K-FIT over rows keyed by size-group id gid (-1 = skip): sums [G, C, V],
    counts [G, C] (exact integers in fp64), status [bad label rows, skipped]."""
    V = x.shape[1]
    S = np.zeros((n_groups, n_classes, V))
    n = np.zeros((n_groups, n_classes))
    status = np.zeros(2, dtype=np.uint64)
    if len(devices) == 1:
        N.check(N.lib.gnb_fit_stats_host(_ptr(x), x.shape[0], V, V, _ptr(gid), _ptr(label), 1,
                                         n_groups, n_classes, _ptr(S), None, _ptr(n),
                                         _ptr(status), devices[0]), "gnb_fit_stats_host")
    else:
        devs = np.asarray(devices, dtype=np.int32)
        N.check(N.lib.gnb_fit_stats_host_sharded(
            _ptr(x), x.shape[0], V, V, _ptr(gid), _ptr(label), 1, n_groups, n_classes, _ptr(S),
            None, _ptr(n), _ptr(status), len(devs), _ptr(devs)), "gnb_fit_stats_host_sharded")
    return S, n, status


# ---------------------------------------------------------------- fit
def train_group(samples: Sequence, features, alpha: float = 1.0, *, group: int = 0,
                device=None):
    """One group's model on its samples (classifier.py:68-129), counted on the GPU."""
    ns = _ns.of(features)
    E = ns.errors
    if not (isinstance(alpha, (int, float)) and not isinstance(alpha, bool)) or alpha <= 0:
        raise E.InvalidConfigError(f"alpha must be positive, got {alpha!r}")
    if not features.opcodes:
        raise E.InvalidConfigError("feature set is empty")
    labels = _labels(samples, ns)
    bad = np.flatnonzero(labels < 0)
    if len(bad):
        raise E.IntegrityError(f"sample {samples[int(bad[0])].id!r} has no training label")
    ops = features.opcodes
    cols = {op: j for j, op in enumerate(dict.fromkeys(ops))}
    x = _densify(samples, cols, max(len(cols), 1))
    gid = np.zeros(len(samples), dtype=np.int32)
    S, n, _ = _fit_stats_host(x, gid, labels, n_classes=2, n_groups=1,
                              devices=[_device_ordinal(device)])
    ci = ns.class_index()
    for c in ns.CLASSES:
        if n[0, ci[c]] == 0:
            raise E.InsufficientClassError(f"group {group}: no {c.value} samples to train on")
    from .dense import fin_tables
    feat_cols = np.array([cols[op] for op in ops], dtype=np.int32)
    prior, ll = fin_tables(S[0], n[0], feat_cols, float(alpha))
    return _model(ns, group, features, prior, ll, n[0], float(alpha))


def _model(ns, group, features, prior, ll, counts, alpha):
    ops = features.opcodes
    ci = ns.class_index()
    return ns.GroupModel(
        group=group, features=features,
        log_prior={c: float(prior[ci[c]]) for c in ns.CLASSES},
        log_likelihood={c: {op: float(ll[ci[c], j]) for j, op in enumerate(ops)}
                        for c in ns.CLASSES},
        alpha=alpha,
        train_counts={c: int(counts[ci[c]]) for c in ns.CLASSES})


def _corpus_rows(train):
    """(samples in ascending group order, group id per sample) of a GroupedCorpus:
    a sample trains the group whose dict key holds it (engine.py:170-172)."""
    samples, gids = [], []
    for g in sorted(train.groups):
        part = train.groups[g]
        samples.extend(part)
        gids.append(np.full(len(part), g, dtype=np.int64))
    return samples, (np.concatenate(gids) if gids else np.zeros(0, np.int64))


class _Fit:
    """One K-FIT pass over a corpus (every group, full vocabulary)."""

    def __init__(self, x, gid64, label, vocab, config, devices, ids):
        G = config.group_count
        self.config, self.vocab, self.ids = config, vocab, ids
        self.label = label
        ok = (gid64 >= 0) & (gid64 < G)
        self.gid = np.where(ok, gid64, -1).astype(np.int32)
        self.S, self.n, self.status = _fit_stats_host(
            np.ascontiguousarray(x, dtype=np.int32), self.gid, label, n_classes=2, n_groups=G,
            devices=devices)
        # group keys outside [0, group_count) (a hand-built GroupedCorpus): the
        # reference trains them if they have enough of each class, and then
        # build_bundle rejects the model (engine.py:108-109)
        self.out_of_range = []
        for g in sorted(set(gid64[~ok].tolist())):
            m = int(np.count_nonzero((gid64 == g) & (label == 1)))
            b = int(np.count_nonzero((gid64 == g) & (label == 0)))
            if m >= config.min_per_class and b >= config.min_per_class:
                self.out_of_range.append(g)

    def _fin(self, k, alpha):
        from .dense import fin_train
        return fin_train(self.S, self.n, k=k, alpha=alpha, min_per_class=self.config.min_per_class)

    @staticmethod
    def _score_error(ns, fin, g):
        if fin.state[g] == -1:
            raise ns.errors.InsufficientClassError(
                f"group {g}: no malware opcode occurrences to score")
        if fin.state[g] == -2:
            raise ns.errors.InsufficientClassError(
                f"group {g}: no benign opcode occurrences to score")

    def check_scores(self, ns):
        """score_opcodes of every trainable group, ascending (bench.py:101-102)."""
        fin = self._fin(1, 1.0)
        for g in np.nonzero(fin.state != 0)[0].tolist():
            self._score_error(ns, fin, g)

    def models(self, ns, k, alpha):
        """Per trainable group, in ascending order, exactly as train_bundle runs
        score_opcodes -> select_top_k -> train_group (engine.py:170-173): the
        same error for the same first failing group."""
        E = ns.errors
        k_ok = isinstance(k, int) and not isinstance(k, bool) and k >= 1
        a_ok = isinstance(alpha, (int, float)) and not isinstance(alpha, bool) and alpha > 0
        fin = self._fin(k if k_ok else 1, float(alpha) if a_ok else 1.0)
        out = []
        for g in np.nonzero(fin.state != 0)[0].tolist():
            self._score_error(ns, fin, g)
            if not k_ok:
                raise E.InvalidConfigError(f"k must be a positive integer, got {k!r}")
            if not a_ok:
                raise E.InvalidConfigError(f"alpha must be positive, got {alpha!r}")
            bad = np.nonzero((self.gid == g) & (self.label < 0))[0]
            if len(bad):
                raise E.IntegrityError(f"sample {self.ids[int(bad[0])]!r} has no training label")
            F = int(fin.n_features[g])
            feats = ns.FeatureSet(tuple(self.vocab[j] for j in fin.features[g, :F]), k)
            out.append(_model(ns, g, feats, fin.log_prior[g], fin.log_lik[g, :, :F], self.n[g],
                              float(alpha)))
        return out

    def check_out_of_range(self, ns):
        gc = self.config.group_count
        for g in self.out_of_range:
            raise ns.errors.BundleValidationError(
                f"model for group {g}: group id outside [0, {gc})")


def _fit_corpus(train, ns, devices) -> _Fit:
    samples, gid64 = _corpus_rows(train)
    x, vocab = _dense_vocab(samples)
    label = _labels(samples, ns)
    return _Fit(x, gid64, label, vocab, train.config, devices, [s.id for s in samples])


def train_bundle(train, k: int, alpha: float = 1.0, *, seed: int = 0,
                 created_at: str | None = None, device=None, devices=None):
    """Select features and train every trainable group (engine.py:157-177).

    One K-FIT pass over the whole corpus (every group, full vocabulary; on
    several GPUs when `devices` is given), then the host finalize (scores,
    top-k, libm logs) per group."""
    ns = _ns.of(train)
    fit = _fit_corpus(train, ns, _device_list(device, devices))
    models = fit.models(ns, k, alpha)
    fit.check_out_of_range(ns)
    if created_at is None:
        created_at = datetime.now(timezone.utc).isoformat(timespec="seconds")
    meta = ns.BundleMeta(k=k, alpha=float(alpha), seed=seed, created_at=created_at)
    return ns.build_bundle(models, train.config, meta)


def train_bundles(train, k_values: Sequence[int], alpha: float = 1.0, *, seed: int = 0,
                  created_at: str = "", device=None, devices=None) -> dict:
    """One bundle per k sharing one fit (bench.train_bundles, bench.py:91-111):
    K-FIT once, then FIN per k.  Errors in the reference's order: every
    group's scoring first, then per k the top-k and train_group checks."""
    ns = _ns.of(train)
    fit = _fit_corpus(train, ns, _device_list(device, devices))
    fit.check_scores(ns)
    bundles = {}
    for k in k_values:
        models = fit.models(ns, k, alpha)
        fit.check_out_of_range(ns)
        meta = ns.BundleMeta(k=k, alpha=float(alpha), seed=seed, created_at=created_at)
        bundles[k] = ns.build_bundle(models, train.config, meta)
    return bundles


# ---------------------------------------------------------------- predict
class _PackedBundle:
    """Dense tables of a bundle: slot order = trained_ids order."""

    def __init__(self, bundle, ns):
        ids = bundle.trained_ids
        slot = {g: i for i, g in enumerate(ids)}
        ci = ns.class_index()
        self.ids = ids
        self.route = np.array([slot[g] for g in bundle._route_table], dtype=np.int32)
        self.F = max(len(bundle.models[g].features.opcodes) for g in ids)
        S = len(ids)
        self.prior = np.zeros((S, 2))
        self.lik = np.zeros((S, 2, self.F))
        self.columns = []
        for i, g in enumerate(ids):
            m = bundle.models[g]
            for c in ns.CLASSES:
                self.prior[i, ci[c]] = m.log_prior[c]
                self.lik[i, ci[c], :len(m.features.opcodes)] = [
                    m.log_likelihood[c][op] for op in m.features.opcodes]
            self.columns.append({op: j for j, op in enumerate(m.features.opcodes)})
        self.eff = np.asarray([bundle.models[g].group for g in ids], dtype=np.int32)


_packed_cache: dict[int, tuple] = {}


def _packed_of(bundle, ns) -> _PackedBundle:
    """Bundles are immutable (engine.py:45-59): pack once, keep while alive."""
    hit = _packed_cache.get(id(bundle))
    if hit is not None and hit[0]() is bundle:
        return hit[1]
    pb = _PackedBundle(bundle, ns)
    key = id(bundle)
    try:
        ref = weakref.ref(bundle, lambda _r, k=key: _packed_cache.pop(k, None))
    except TypeError:
        return pb
    _packed_cache[key] = (ref, pb)
    return pb


def _gather(samples, packed: _PackedBundle, config):
    """Row i = counts of its routed model's features, FeatureSet order
    (engine.py:198-202), plus its size group id (-1 outside [0, limit))."""
    x = np.zeros((len(samples), packed.F), dtype=np.int32)
    gid = np.empty(len(samples), dtype=np.int32)
    _adapt.gather_into(samples, packed.route, packed.columns, packed.F,
                       config.group_size_bytes, config.max_size_bytes, x, gid)
    return x, gid


def _predict_host(x, gid, packed: _PackedBundle, group_count: int, devices: list[int]):
    """K-PRED through the host-buffer ABI; rows routed by group id (width 1)."""
    n = x.shape[0]
    label = np.empty(n, dtype=np.int32)
    lp = np.empty((n, 2))
    elapsed = ctypes.c_int64(0)
    if len(devices) == 1:
        N.check(N.lib.gnb_predict_host(
            _ptr(x), n, packed.F, packed.F, _ptr(gid), 1, group_count, _ptr(packed.route),
            len(packed.ids), 2, _ptr(packed.prior), _ptr(packed.lik), _ptr(label), _ptr(lp),
            devices[0], ctypes.addressof(elapsed)), "gnb_predict_host")
    else:
        devs = np.asarray(devices, dtype=np.int32)
        N.check(N.lib.gnb_predict_host_sharded(
            _ptr(x), N.X_I32, n, packed.F, packed.F, _ptr(gid), 1, group_count,
            _ptr(packed.route), len(packed.ids), 2, _ptr(packed.prior), _ptr(packed.lik),
            _ptr(label), _ptr(lp), len(devs), _ptr(devs), ctypes.addressof(elapsed)),
            "gnb_predict_host_sharded")
    return label, lp, int(elapsed.value)


def classify_gpu(bundle, workload, *, warmup: bool = True, device=None, devices=None):
    """Classify a workload on the GPU (or several: `devices`); the TimedRun is
    identical to classify_sequential's.

    elapsed_ns covers the device call only (host->device copy, the K-PRED
    kernel, device->host copy; the slowest device when sharded), like the
    reference's kernel-only timing: densifying the objects
    happens before the clock starts."""
    ns = _ns.of(bundle)
    if not bundle.trained_ids:
        raise ns.errors.EmptyBundleError("bundle has no trained models")
    samples = workload.samples
    config = bundle.config
    if not samples:
        return ns.TimedRun((), (), 0)
    packed = _packed_of(bundle, ns)
    x, gid = _gather(samples, packed, config)
    devs = _device_list(device, devices)
    if warmup:
        _predict_host(x, gid, packed, config.group_count, devs)
    label, lp, elapsed = _predict_host(x, gid, packed, config.group_count, devs)
    bad = np.flatnonzero(label < 0)
    errors: list[tuple[int, str]] = []
    lim = config.max_size_bytes
    for i in bad.tolist():
        if label[i] != N.ROW_OUT_OF_RANGE:
            raise ns.errors.IntegrityError(f"sample {samples[i].id!r}: negative opcode count")
        errors.append((i, oversize_message(samples[i].size_bytes, lim)))
    # effective group of every in-range row (the routed model's `group`,
    # engine.py:202 + classifier.py:158); the Prediction objects are built in C
    eff = packed.eff[packed.route[np.maximum(gid, 0)]]
    preds = _adapt.predictions(label, lp, np.ascontiguousarray(eff, dtype=np.int32), ns.Prediction,
                               ns.INDEX_CLASS, ns.MALWARE, ns.BENIGN)
    return ns.TimedRun(tuple(preds), tuple(errors), max(elapsed, 1))


def classify_parallel(bundle, workload, *, warmup: bool = True, device=None, devices=None):
    """engine.py:250 contract (Tp): the GPU is the parallel backend.
    `workload.lanes` is validated by Workload; the device decides the
    parallelism within a GPU, `devices` across GPUs."""
    return classify_gpu(bundle, workload, warmup=warmup, device=device, devices=devices)


def classify_sequential(bundle, workload, *, warmup: bool = True):
    """engine.py:209-226 contract (Tc): one host thread, never parallelised.

    `_classify_slice` (engine.py:187-206) in C over the reference's objects:
    route by size, score the model's `_packed` rows in order (mul, then add),
    malware iff strictly higher.  The unmeasured warmup pass and the timed
    pass are the reference's; results equal classify_parallel's bit for bit."""
    ns = _ns.of(bundle)
    if not bundle.trained_ids:
        raise ns.errors.EmptyBundleError("bundle has no trained models")
    samples = workload.samples
    cfg = bundle.config
    args = (samples, bundle._route_table, bundle.models, cfg.group_size_bytes,
            cfg.max_size_bytes, ns.Prediction, ns.MALWARE, ns.BENIGN)
    if warmup:
        _adapt.classify_slice(*args)
    t0 = time.perf_counter_ns()
    preds, bad = _adapt.classify_slice(*args)
    elapsed = time.perf_counter_ns() - t0
    errors = tuple((i, oversize_message(samples[i].size_bytes, cfg.max_size_bytes)) for i in bad)
    return ns.TimedRun(tuple(preds), errors, elapsed)


def log_posterior(model, histogram) -> dict:
    """Unnormalised joint log-score per class (classifier.py:132-148), host."""
    ns = _ns.of(model)
    m, b = _adapt.score_packed(model._packed, model.log_prior[ns.MALWARE],
                               model.log_prior[ns.BENIGN], histogram.entries)
    return {ns.MALWARE: m, ns.BENIGN: b}


def predict(model, histogram):
    """Malware iff strictly higher, ties -> benign (classifier.py:151-158), host."""
    ns = _ns.of(model)
    scores = log_posterior(model, histogram)
    label = ns.MALWARE if scores[ns.MALWARE] > scores[ns.BENIGN] else ns.BENIGN
    return ns.Prediction(label=label, log_posterior=scores, effective_group=model.group)


# ---------------------------------------------------------------- dense corpus paths
def train_bundle_corpus(corpus, config: GroupingConfig, k: int, alpha: float = 1.0, *,
                        seed: int = 0, created_at: str | None = None, device=None,
                        devices=None):
    """train_bundle (engine.py:157-177) on an ingest.DenseCorpus: no per-record
    Python work; rows outside the size range are skipped like partition_by_group."""
    ns = _ns.OWN
    size = corpus.size.astype(np.int64)
    ok = (size >= 0) & (size < config.max_size_bytes)
    gid64 = np.where(ok, size // config.group_size_bytes, -1)
    fit = _Fit(corpus.dense(), gid64, corpus.label.astype(np.int32), corpus.vocab, config,
               _device_list(device, devices), corpus.ids)
    models = fit.models(ns, k, alpha)
    if created_at is None:
        created_at = datetime.now(timezone.utc).isoformat(timespec="seconds")
    meta = ns.BundleMeta(k=k, alpha=float(alpha), seed=seed, created_at=created_at)
    return ns.build_bundle(models, config, meta)


def classify_corpus(bundle, corpus, *, device=None, warmup: bool = True):
    """classify_parallel on an ingest.DenseCorpus: rows go to the device in the
    corpus's full-vocabulary layout (narrowest lossless storage); route +
    FeatureSet gather (gnb_gather_features, any storage), an optional slot sort
    and K-PRED run on the device.  Returns (label[N] int8: 1 malware / 0 benign /
    -1 error, log_posterior [N, 2] (benign, malware), effective_group[N],
    errors, elapsed_ns)."""
    import torch
    from . import dense
    ns = _ns.of(bundle)
    if not bundle.trained_ids:
        raise ns.errors.EmptyBundleError("bundle has no trained models")
    dev = torch.device("cuda", _device_ordinal(device))
    packed = _packed_of(bundle, ns)
    col = {op: j for j, op in enumerate(corpus.vocab)}
    feats = np.full((len(packed.ids), packed.F), -1, dtype=np.int32)
    nfeat = np.zeros(len(packed.ids), dtype=np.int32)
    for i, g in enumerate(packed.ids):
        ops = bundle.models[g].features.opcodes
        feats[i, :len(ops)] = [col.get(op, -1) for op in ops]
        nfeat[i] = len(ops)
    cfg = bundle.config
    lim = cfg.max_size_bytes
    size64 = corpus.size.astype(np.int64)
    gid = np.where((size64 >= 0) & (size64 < lim), size64 // cfg.group_size_bytes,
                   -1).astype(np.int32)
    tables = dense.DeviceTables.build(packed.prior, packed.lik, packed.route,
                                      group_size_bytes=1, max_size_bytes=cfg.group_count,
                                      device=dev)
    n = len(corpus)
    V = max(len(corpus.vocab), 1)
    dt = np.dtype(corpus.narrowest_dtype())
    pitch = (V * dt.itemsize + 15) // 16 * 16 // dt.itemsize
    host = torch.zeros((n, pitch), dtype=getattr(torch, dt.name), pin_memory=True)
    corpus.dense(dt, out=host.numpy()[:, :V])

    def run():
        t0 = time.perf_counter_ns()
        xv = host.to(dev, non_blocking=True)[:, :V]
        sd = torch.from_numpy(gid).to(dev, non_blocking=True)
        xg = dense.gather_features(xv, sd, tables, feats, nfeat)
        perm = dense.slot_sort(sd, tables) if dense.needs_slot_sort(xg.dtype, tables) else None
        lab, lp = dense.predict(xg, sd, tables, perm=perm)
        out = lab.cpu().numpy(), lp.cpu().numpy()
        return out, time.perf_counter_ns() - t0

    if warmup:
        run()
    (lab, lp), elapsed = run()
    eff = np.where(lab >= 0, packed.eff[packed.route[np.maximum(gid, 0)]], -1)
    errors = [(int(i), oversize_message(int(corpus.size[i]), lim)) for i in np.nonzero(lab < 0)[0]]
    return lab.astype(np.int8), lp, eff, errors, elapsed


def speedup(tc_ns: int, tp_ns: int) -> float:
    """Sequential-over-parallel time ratio (engine.py:299-305)."""
    from .errors import MeasurementError
    if tp_ns <= 0:
        raise MeasurementError(f"parallel time must be positive, got {tp_ns}")
    if tc_ns < 0:
        raise MeasurementError(f"sequential time must be non-negative, got {tc_ns}")
    return tc_ns / tp_ns
