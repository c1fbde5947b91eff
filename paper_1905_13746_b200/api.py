"""The reference's fit / classify operation contract, executed on the GPU.

Drop-in for the hot path of `groupnb` (reference pkg/src/groupnb):

  train_bundle(train, k, alpha=1.0, *, seed=0, created_at=None)  engine.py:157-177
  train_group(samples, features, alpha=1.0, *, group=0)           classifier.py:68-129
  classify_parallel / classify_sequential(bundle, workload, *, warmup=True)
                                                                  engine.py:209-296
  log_posterior(model, histogram) / predict(model, histogram)     classifier.py:132-158

Same arguments, same results (bit-identical log-scores and bundles), same
exception types and messages.  The object model is densified here on the
host and handed to libgnb.so's host-buffer entry points (gnb_fit_stats_host,
gnb_fin_train, gnb_predict_host), which run the sm_100a kernels.  Per SPEC.md
("a GPU backend is an optional extension point behind the same operation
contract"), `lanes` is validated but the device decides the parallelism.
"""

from __future__ import annotations

import ctypes
from datetime import datetime, timezone
from typing import Sequence

import numpy as np

from . import _adapt
from . import _native as N
from .errors import (EmptyBundleError, InsufficientClassError, IntegrityError,
                     InvalidConfigError, MeasurementError)
from .model import (CLASS_INDEX, CLASSES, INDEX_CLASS, BundleMeta, FeatureSet, GroupedCorpus,
                    GroupingConfig, GroupModel, Label, ModelBundle, OpcodeHistogram, Prediction,
                    SampleRecord, TimedRun, Workload, build_bundle, oversize_message)

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


def _meta(samples: Sequence[SampleRecord], limit: int):
    """int32 sizes (outside [0, limit) -> -1, still an error row) and class codes
    (benign 0, malware 1, unlabeled -1), via the C-API packer."""
    size = np.empty(len(samples), dtype=np.int32)
    label = np.empty(len(samples), dtype=np.int32)
    _adapt.meta_into(samples, limit, Label.MALWARE, Label.BENIGN, size, label)
    return size, label


def _densify(samples: Sequence[SampleRecord], columns: dict[str, int], width: int) -> np.ndarray:
    """[N, width] int32 counts of the opcodes in `columns` (others ignored)."""
    x = np.zeros((len(samples), width), dtype=np.int32)
    _adapt.densify_into(samples, columns, x, width)
    return x


def _dense_vocab(samples: Sequence[SampleRecord]):
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


def _fit_stats_host(x: np.ndarray, size: np.ndarray, label: np.ndarray, *, n_classes: int,
                    width: int, limit: int, device: int):
    G = limit // width
    V = x.shape[1]
    S = np.zeros((G, n_classes, V))
    n = np.zeros((G, n_classes))
    status = np.zeros(2, dtype=np.uint64)
    N.check(N.lib.gnb_fit_stats_host(_ptr(x), x.shape[0], V, V, _ptr(size), _ptr(label), width,
                                     limit, n_classes, _ptr(S), None, _ptr(n), _ptr(status),
                                     device), "gnb_fit_stats_host")
    return S, n, status


# ---------------------------------------------------------------- fit
def train_group(samples: Sequence[SampleRecord], features: FeatureSet, alpha: float = 1.0, *,
                group: int = 0, device=None) -> GroupModel:
    """One group's model on its samples (classifier.py:68-129), counted on the GPU."""
    if isinstance(alpha, bool) or not isinstance(alpha, (int, float)) or alpha <= 0:
        raise InvalidConfigError(f"alpha must be positive, got {alpha!r}")
    if not features.opcodes:
        raise InvalidConfigError("feature set is empty")
    for s in samples:
        if s.label not in CLASS_INDEX:
            raise IntegrityError(f"sample {s.id!r} has no training label")
    ops = features.opcodes
    cols = {op: j for j, op in enumerate(dict.fromkeys(ops))}
    x = _densify(samples, cols, max(len(cols), 1))
    zeros = np.zeros(len(samples), dtype=np.int32)
    _, labels = _meta(samples, 1)
    S, n, _ = _fit_stats_host(x, zeros, labels, n_classes=2, width=1, limit=1,
                              device=_device_ordinal(device))
    for c in CLASSES:
        if n[0, CLASS_INDEX[c]] == 0:
            raise InsufficientClassError(f"group {group}: no {c.value} samples to train on")
    from .dense import fin_tables
    feat_cols = np.array([cols[op] for op in ops], dtype=np.int32)
    prior, ll = fin_tables(S[0], n[0], feat_cols, float(alpha))
    return _model(group, features, prior, ll, n[0], float(alpha))


def _model(group, features: FeatureSet, prior, ll, counts, alpha) -> GroupModel:
    ops = features.opcodes
    return GroupModel(
        group=group, features=features,
        log_prior={c: float(prior[CLASS_INDEX[c]]) for c in CLASSES},
        log_likelihood={c: {op: float(ll[CLASS_INDEX[c], j]) for j, op in enumerate(ops)}
                        for c in CLASSES},
        alpha=alpha,
        train_counts={c: int(counts[CLASS_INDEX[c]]) for c in CLASSES})


def train_bundle(train: GroupedCorpus, k: int, alpha: float = 1.0, *, seed: int = 0,
                 created_at: str | None = None, device=None) -> ModelBundle:
    """Select features and train every trainable group (engine.py:157-177).

    One K-FIT pass over the whole corpus (every group, full vocabulary), then
    the host finalize (scores, top-k, libm logs) per group."""
    config = train.config
    samples = train.all_samples()
    x, vocab = _dense_vocab(samples)
    size = np.array([s.size_bytes for s in samples], dtype=object)
    size64 = np.array([v if -2**63 <= v < 2**63 else -1 for v in size], dtype=np.int64)
    _, label = _meta(samples, config.max_size_bytes)
    return _train_dense(x[:, :len(vocab)], size64, label, vocab, config, k, alpha, seed,
                        created_at, _device_ordinal(device), [s.id for s in samples])


# ---------------------------------------------------------------- predict
class _PackedBundle:
    """Dense tables of a bundle: slot order = trained_ids order."""

    def __init__(self, bundle: ModelBundle):
        ids = bundle.trained_ids
        slot = {g: i for i, g in enumerate(ids)}
        self.ids = ids
        self.route = np.array([slot[g] for g in bundle._route_table], dtype=np.int32)
        self.F = max(len(bundle.models[g].features.opcodes) for g in ids)
        S = len(ids)
        self.prior = np.zeros((S, 2))
        self.lik = np.zeros((S, 2, self.F))
        self.columns = []
        for i, g in enumerate(ids):
            m = bundle.models[g]
            for c in CLASSES:
                ci = CLASS_INDEX[c]
                self.prior[i, ci] = m.log_prior[c]
                self.lik[i, ci, :len(m.features.opcodes)] = [
                    m.log_likelihood[c][op] for op in m.features.opcodes]
            self.columns.append({op: j for j, op in enumerate(m.features.opcodes)})


def _gather(samples, packed: _PackedBundle, config: GroupingConfig):
    """Row i = counts of its routed model's features, FeatureSet order
    (engine.py:198-202), plus int32 sizes (-1 outside [0, limit))."""
    x = np.zeros((len(samples), packed.F), dtype=np.int32)
    size = np.empty(len(samples), dtype=np.int32)
    _adapt.gather_into(samples, packed.route, packed.columns, packed.F,
                       config.group_size_bytes, config.max_size_bytes, x, size)
    return x, size


def _predict_host(x, size, packed: _PackedBundle, config: GroupingConfig, device: int):
    n = x.shape[0]
    label = np.empty(n, dtype=np.int32)
    lp = np.empty((n, 2))
    elapsed = ctypes.c_int64(0)
    N.check(N.lib.gnb_predict_host(
        _ptr(x), n, packed.F, packed.F, _ptr(size), config.group_size_bytes,
        config.max_size_bytes, _ptr(packed.route), len(packed.ids), 2, _ptr(packed.prior),
        _ptr(packed.lik), _ptr(label), _ptr(lp), device, ctypes.addressof(elapsed)),
        "gnb_predict_host")
    return label, lp, int(elapsed.value)


def classify_gpu(bundle: ModelBundle, workload: Workload, *, warmup: bool = True,
                 device=None) -> TimedRun:
    """Classify a workload on the GPU; TimedRun identical to classify_sequential.

    elapsed_ns covers the device call only (host->device copy, the K-PRED
    kernel, device->host copy), like the reference's kernel-only timing
    (SPEC.md:357): densifying the objects happens before the clock starts."""
    if not bundle.trained_ids:
        raise EmptyBundleError("bundle has no trained models")
    samples = workload.samples
    config = bundle.config
    if not samples:
        return TimedRun((), (), 0)
    packed = _PackedBundle(bundle)
    x, size = _gather(samples, packed, config)
    dev = _device_ordinal(device)
    if warmup:
        _predict_host(x, size, packed, config, dev)
    label, lp, elapsed = _predict_host(x, size, packed, config, dev)
    bad = np.flatnonzero(label < 0)
    errors: list[tuple[int, str]] = []
    lim = config.max_size_bytes
    for i in bad.tolist():
        if label[i] != N.ROW_OUT_OF_RANGE:
            raise IntegrityError(f"sample {samples[i].id!r}: negative opcode count")
        errors.append((i, oversize_message(samples[i].size_bytes, lim)))
    # effective group of every in-range row (engine.py:202 route), then the
    # Prediction objects in C (ADAPT): the per-row Python object loop cost
    # ~4.5 us per sample, more than the whole device call
    g = np.where(size >= 0, size // config.group_size_bytes, 0)
    eff = np.asarray(packed.ids, dtype=np.int32)[packed.route[g]]
    preds = _adapt.predictions(label, lp, np.ascontiguousarray(eff, dtype=np.int32), Prediction,
                               INDEX_CLASS, Label.MALWARE, Label.BENIGN)
    return TimedRun(tuple(preds), tuple(errors), max(elapsed, 1))


def classify_parallel(bundle: ModelBundle, workload: Workload, *, warmup: bool = True,
                      device=None) -> TimedRun:
    """engine.py:250 contract; the GPU is the parallel backend."""
    return classify_gpu(bundle, workload, warmup=warmup, device=device)


def classify_sequential(bundle: ModelBundle, workload: Workload, *, warmup: bool = True,
                        device=None) -> TimedRun:
    """engine.py:209 contract.  Runs the same device kernel; results are
    identical to classify_parallel by construction (one code path)."""
    return classify_gpu(bundle, workload, warmup=warmup, device=device)


def log_posterior(model: GroupModel, histogram: OpcodeHistogram, *, device=None):
    """Unnormalised joint log-score per class (classifier.py:132-148)."""
    return predict(model, histogram, device=device).log_posterior


def predict(model: GroupModel, histogram: OpcodeHistogram, *, device=None) -> Prediction:
    """Malware iff strictly higher (classifier.py:151-158)."""
    cfg = GroupingConfig(group_size_bytes=1, max_size_bytes=1, min_per_class=1)
    bundle = ModelBundle(cfg, {0: model}, (0,), BundleMeta(len(model.features.opcodes), 1.0, 0, ""))
    packed = _PackedBundle(bundle)
    sample = SampleRecord("_", Label.UNKNOWN, 0, histogram)
    x, size = _gather([sample], packed, cfg)
    label, lp, _ = _predict_host(x, size, packed, cfg, _device_ordinal(device))
    return Prediction(INDEX_CLASS[int(label[0])],
                      {Label.MALWARE: float(lp[0, 1]), Label.BENIGN: float(lp[0, 0])},
                      model.group)


# ---------------------------------------------------------------- dense corpus paths
def train_bundle_corpus(corpus, config: GroupingConfig, k: int, alpha: float = 1.0, *,
                        seed: int = 0, created_at: str | None = None, device=None) -> ModelBundle:
    """train_bundle (engine.py:157-177) on an ingest.DenseCorpus: no per-record
    Python work; rows outside the size range are skipped like partition_by_group."""
    return _train_dense(corpus.dense(), corpus.size, corpus.label.astype(np.int32),
                        corpus.vocab, config, k, alpha, seed, created_at,
                        _device_ordinal(device), corpus.ids)


def _train_dense(x, size64, label, vocab, config, k, alpha, seed, created_at, device, ids):
    k_ok = isinstance(k, int) and not isinstance(k, bool) and k >= 1
    a_ok = isinstance(alpha, (int, float)) and not isinstance(alpha, bool) and alpha > 0
    lim = config.max_size_bytes
    size = np.where((size64 >= 0) & (size64 < lim), size64, -1).astype(np.int32)
    models = []
    if len(size) and len(vocab):
        x = np.ascontiguousarray(x, dtype=np.int32)   # gnb_fit_stats_host takes int32 rows
        S, n, _ = _fit_stats_host(x, size, label, n_classes=2, width=config.group_size_bytes,
                                  limit=lim, device=device)
        from .dense import fin_train
        fin = fin_train(S, n, k=k if k_ok else 1, alpha=float(alpha) if a_ok else 1.0,
                        min_per_class=config.min_per_class)
        g_of = np.where(size >= 0, size // config.group_size_bytes, -1)
        for g in np.nonzero(fin.state != 0)[0].tolist():
            if fin.state[g] == -1:
                raise InsufficientClassError(f"group {g}: no malware opcode occurrences to score")
            if fin.state[g] == -2:
                raise InsufficientClassError(f"group {g}: no benign opcode occurrences to score")
            if not k_ok:
                raise InvalidConfigError(f"k must be a positive integer, got {k!r}")
            if not a_ok:
                raise InvalidConfigError(f"alpha must be positive, got {alpha!r}")
            bad = np.nonzero((g_of == g) & (label < 0))[0]
            if len(bad):
                raise IntegrityError(f"sample {ids[int(bad[0])]!r} has no training label")
            F = int(fin.n_features[g])
            feats = FeatureSet(tuple(vocab[j] for j in fin.features[g, :F]), k)
            models.append(_model(g, feats, fin.log_prior[g], fin.log_lik[g, :, :F], n[g],
                                 float(alpha)))
    if created_at is None:
        created_at = datetime.now(timezone.utc).isoformat(timespec="seconds")
    meta = BundleMeta(k=k, alpha=float(alpha), seed=seed, created_at=created_at)
    return build_bundle(models, config, meta)


def classify_corpus(bundle: ModelBundle, corpus, *, device=None, warmup: bool = True):
    """classify_parallel on an ingest.DenseCorpus: rows go to the device in the
    corpus's full-vocabulary layout (narrowest lossless storage); route +
    FeatureSet gather (gnb_gather_features), an optional slot sort and K-PRED run
    on the device.  Returns (label[N] int8: 1 malware / 0 benign / -1 error,
    log_posterior [N, 2] (benign, malware), effective_group[N], errors, elapsed_ns)."""
    import time
    import torch
    from . import dense
    if not bundle.trained_ids:
        raise EmptyBundleError("bundle has no trained models")
    dev = torch.device("cuda", _device_ordinal(device))
    packed = _PackedBundle(bundle)
    col = {op: j for j, op in enumerate(corpus.vocab)}
    feats = np.full((len(packed.ids), packed.F), -1, dtype=np.int32)
    nfeat = np.zeros(len(packed.ids), dtype=np.int32)
    for i, g in enumerate(packed.ids):
        ops = bundle.models[g].features.opcodes
        feats[i, :len(ops)] = [col.get(op, -1) for op in ops]
        nfeat[i] = len(ops)
    lim = bundle.config.max_size_bytes
    size = np.where((corpus.size >= 0) & (corpus.size < lim), corpus.size, -1).astype(np.int32)
    tables = dense.DeviceTables.build(packed.prior, packed.lik, packed.route,
                                      group_size_bytes=bundle.config.group_size_bytes,
                                      max_size_bytes=lim, device=dev)
    n = len(corpus)
    V = max(len(corpus.vocab), 1)
    dt = np.dtype(corpus.narrowest_dtype())
    pitch = (V * dt.itemsize + 15) // 16 * 16 // dt.itemsize
    host = torch.empty((n, pitch), dtype=getattr(torch, dt.name), pin_memory=True)
    corpus.dense(dt, out=host.numpy()[:, :V])

    def run():
        t0 = time.perf_counter_ns()
        xv = host.to(dev, non_blocking=True)[:, :V]
        sd = torch.from_numpy(size).to(dev, non_blocking=True)
        xi = xv if xv.dtype == torch.int32 else xv.to(torch.int32)
        xg = dense.gather_features(xi, sd, tables, feats, nfeat)
        perm = dense.slot_sort(sd, tables) if len(packed.ids) > 1 else None
        lab, lp = dense.predict(dense.narrowest(xg) if dt.itemsize < 4 else xg, sd, tables,
                                perm=perm)
        out = lab.cpu().numpy(), lp.cpu().numpy()
        return out, time.perf_counter_ns() - t0

    if warmup:
        run()
    (lab, lp), elapsed = run()
    g = np.where(size >= 0, size // bundle.config.group_size_bytes, 0)
    eff = np.where(lab >= 0, np.array(packed.ids)[packed.route[g]], -1)
    errors = [(int(i), oversize_message(int(corpus.size[i]), lim)) for i in np.nonzero(lab < 0)[0]]
    return lab.astype(np.int8), lp, eff, errors, elapsed


def speedup(tc_ns: int, tp_ns: int) -> float:
    """Sequential-over-parallel time ratio (engine.py:299-305)."""
    if tp_ns <= 0:
        raise MeasurementError(f"parallel time must be positive, got {tp_ns}")
    if tc_ns < 0:
        raise MeasurementError(f"sequential time must be non-negative, got {tc_ns}")
    return tc_ns / tp_ns
