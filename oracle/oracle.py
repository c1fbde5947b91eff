"""CPU oracle for the group-wise Naive Bayes hot path -- TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import this module, and only as the checker (or
the timed CPU baseline).  The product package `paper_1905_13746_b200` never
imports it and has no CPU fallback.

This is a dense numpy restatement of the reference algorithm
(/root/reference/pkg/src/groupnb, pure Python).  Parity is PINNED: every
function below is checked bit-for-bit against golden vectors produced by
running the reference itself (`tests/golden/make_golden.py`, fixtures
`tests/golden/*.npz`, test `tests/test_oracle.py`).

Dense conventions (shared with the CUDA path):
  * class index 0 = benign, 1 = malware (extra classes 2.. are malware
    families for the multi-class fit); argmax ties go to the lowest index,
    which reproduces "malware iff strictly higher" (classifier.py:154-157).
  * vocabulary columns are sorted by mnemonic, so column order == the
    reference's `sorted()` order (features.py:71, :85).
  * predict input row n holds the counts of its routed model's features in
    FeatureSet order (classifier.py:143 `_packed` order), zero-padded to F.
"""

from __future__ import annotations

import math
from bisect import bisect_left
from dataclasses import dataclass

import numpy as np

BENIGN, MALWARE = 0, 1


# ---------------------------------------------------------------- routing
def group_of(size: np.ndarray, width: int, limit: int) -> np.ndarray:
    """size // width on [0, limit); -1 outside (corpus.py:222-232, engine.py:201)."""
    size = np.asarray(size, dtype=np.int64)
    g = np.where((size >= 0) & (size < limit), size // width, -1)
    return g.astype(np.int64)


def route_table(trained_ids, group_count: int) -> np.ndarray:
    """Smallest trained id >= g, else the largest (engine.py:56-59, 87-91)."""
    ids = sorted(trained_ids)
    out = np.empty(group_count, dtype=np.int32)
    for g in range(group_count):
        i = bisect_left(ids, g)
        out[g] = ids[i] if i < len(ids) else ids[-1]
    return out


# ---------------------------------------------------------------- fit stats
def fit_stats(x, size, label, n_classes: int, width: int, limit: int):
    """Per-(group, class, column) sums S, sums of squares Q and row counts n.

    S restates the count loops of class_frequency (features.py:48-53) and
    train_group (classifier.py:94-101) over the full vocabulary; n restates
    trainable_groups (corpus.py:302-305) and train_group's n_samples
    (classifier.py:97).  Q (sum of x^2) is the north-star extra with no
    reference counterpart.  Integer arithmetic, exact.  Rows outside the
    size range are skipped (partition_by_group, corpus.py:247-251); rows
    with a label outside [0, C) are counted in `bad_label`
    (classifier.py:95-96 raises IntegrityError for them).
    """
    x = np.asarray(x, dtype=np.int64)
    g = group_of(size, width, limit)
    label = np.asarray(label, dtype=np.int64)
    n_groups = limit // width
    ok = g >= 0
    good = ok & (label >= 0) & (label < n_classes)
    key = g[good] * n_classes + label[good]
    keys = n_groups * n_classes
    xs = x[good]
    S = np.zeros((keys, x.shape[1]), dtype=np.int64)
    Q = np.zeros((keys, x.shape[1]), dtype=np.int64)
    for k in np.unique(key):
        rows = xs[key == k]
        S[k] = rows.sum(0)
        Q[k] = (rows * rows).sum(0)
    n = np.bincount(key, minlength=keys).astype(np.int64)
    shape = (n_groups, n_classes, x.shape[1])
    return (S.reshape(shape), Q.reshape(shape), n.reshape(n_groups, n_classes),
            int((ok & ~good).sum()), int((~ok).sum()))


# ---------------------------------------------------------------- finalize
class OracleError(Exception):
    def __init__(self, kind: str, message: str):
        super().__init__(message)
        self.kind = kind


@dataclass
class GroupTables:
    group: int
    features: np.ndarray      # vocab column indices, FeatureSet order
    log_prior: np.ndarray     # [C]
    log_lik: np.ndarray       # [C, F]
    train_counts: np.ndarray  # [C]


def trainable(n, min_per_class: int):
    """Groups with >= min_per_class rows of every class (corpus.py:295-307)."""
    return [g for g in range(n.shape[0]) if bool((n[g] >= min_per_class).all())]


def select_features(S_g, k: int, group: int):
    """score_opcodes + select_top_k on one group's [2, V] sums (features.py:59-86)."""
    t_b = int(S_g[BENIGN].sum())
    t_m = int(S_g[MALWARE].sum())
    if t_m == 0:
        raise OracleError("InsufficientClassError",
                          f"group {group}: no malware opcode occurrences to score")
    if t_b == 0:
        raise OracleError("InsufficientClassError",
                          f"group {group}: no benign opcode occurrences to score")
    cand = [v for v in range(S_g.shape[1]) if S_g[MALWARE, v] or S_g[BENIGN, v]]
    scores = {v: abs(int(S_g[MALWARE, v]) / t_m - int(S_g[BENIGN, v]) / t_b) for v in cand}
    ordered = sorted(cand, key=lambda v: (-scores[v], v))
    return np.array(ordered[:k], dtype=np.int64), scores


def train_tables(S_g, n_g, features, alpha: float, group: int) -> GroupTables:
    """train_group on dense sums (classifier.py:84-129); libm log via math.log."""
    if not (alpha > 0):
        raise OracleError("InvalidConfigError", f"alpha must be positive, got {alpha!r}")
    if len(features) == 0:
        raise OracleError("InvalidConfigError", "feature set is empty")
    C = S_g.shape[0]
    for c in range(C):
        if n_g[c] == 0:
            raise OracleError("InsufficientClassError", f"group {group}: no samples of class {c}")
    n_total = int(sum(int(v) for v in n_g))
    log_prior = np.array([math.log(int(n_g[c]) / n_total) for c in range(C)])
    F = len(features)
    alpha = float(alpha)
    ll = np.empty((C, F))
    for c in range(C):
        counts = [int(S_g[c, v]) for v in features]
        # total_c over DISTINCT features (the reference's count dict is keyed
        # by opcode, classifier.py:91-93, 116); |F| counts repeats (:112)
        denom = sum(int(S_g[c, v]) for v in dict.fromkeys(int(f) for f in features)) + alpha * F
        for j, cnt in enumerate(counts):
            ll[c, j] = math.log((cnt + alpha) / denom)
    return GroupTables(group, np.asarray(features), log_prior, ll,
                       np.array([int(v) for v in n_g]))


def train_bundle_dense(x, size, label, vocab_size: int, *, width: int, limit: int,
                       min_per_class: int, k: int, alpha: float = 1.0):
    """train_bundle (engine.py:157-177) on dense arrays; returns {group: GroupTables}."""
    S, _, n, bad, _ = fit_stats(x, size, label, 2, width, limit)
    if bad:
        raise OracleError("IntegrityError", "training row without a class label")
    out = {}
    for g in trainable(n, min_per_class):
        feats, _ = select_features(S[g], k, g)
        out[g] = train_tables(S[g], n[g], feats, alpha, g)
    return out


# ---------------------------------------------------------------- predict
def pack_models(models: dict, group_count: int, n_features: int | None = None):
    """Slot tables: route[group_count] -> slot, log_prior[S, C], log_lik[S, C, F] (0-padded)."""
    ids = sorted(models)
    slot_of = {g: i for i, g in enumerate(ids)}
    route = np.array([slot_of[int(g)] for g in route_table(ids, group_count)], dtype=np.int32)
    C = len(models[ids[0]].log_prior)
    F = n_features or max(len(models[g].features) for g in ids)
    prior = np.stack([models[g].log_prior for g in ids])
    ll = np.zeros((len(ids), C, F))
    for i, g in enumerate(ids):
        ll[i, :, : len(models[g].features)] = models[g].log_lik
    return ids, route, prior, ll


def gather_rows(x_vocab, size, models: dict, *, width: int, limit: int, n_features: int):
    """Dense [N, V] -> [N, F] in each row's routed FeatureSet order (engine.py:198-202)."""
    ids = sorted(models)
    table = route_table(ids, limit // width)
    g = group_of(size, width, limit)
    out = np.zeros((len(size), n_features), dtype=np.int32)
    for r in range(len(size)):
        if g[r] < 0:
            continue
        feats = models[int(table[g[r]])].features
        out[r, : len(feats)] = x_vocab[r, feats]
    return out


def predict_dense(x, size, route, prior, ll, *, width: int, limit: int):
    """log_posterior + predict + _classify_slice (classifier.py:132-158, engine.py:187-206).

    One fp64 accumulator per class seeded with the prior, then for every
    feature in order `acc = acc + x * ll` as a separate multiply and add
    (two roundings, no FMA) -- bit-identical to the reference's Python loop
    (zeros contribute -0.0 / +0.0 and leave the sum unchanged).
    Returns label[N] (-1 = size out of range) and logpost[N, C] (NaN there).
    """
    x = np.asarray(x)
    N = x.shape[0]
    g = group_of(size, width, limit)
    ok = g >= 0
    slot = np.zeros(N, dtype=np.int64)
    slot[ok] = np.asarray(route)[g[ok]]
    C = prior.shape[1]
    F = ll.shape[2]
    acc = prior[slot].copy()                       # [N, C]
    xf = x.astype(np.float64)
    for j in range(F):
        acc = acc + xf[:, j : j + 1] * ll[slot, :, j]   # numpy: mul then add, no FMA
    label = np.zeros(N, dtype=np.int32)
    best = acc[:, 0].copy()
    for c in range(1, C):
        better = acc[:, c] > best
        label[better] = c
        best = np.where(better, acc[:, c], best)
    label[~ok] = -1
    acc[~ok] = np.nan
    return label, acc


def oversize_message(size: int, limit: int) -> str:
    """engine.py:183-184."""
    return f"size_bytes {size} outside [0, {limit})"


# ---------------------------------------------------------------- C restatement
_C_LIB = None


def c_oracle():
    """ctypes handle on oracle/build/liboracle.so (built by `make -C oracle`)."""
    global _C_LIB
    if _C_LIB is None:
        import ctypes as C
        import os
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "build", "liboracle.so")
        lib = C.CDLL(path)
        p, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        lib.oracle_predict.argtypes = [p, i64, i32, i64, p, i32, i32, p, i32, p, p, p, p, i32]
        lib.oracle_predict_typed.argtypes = [p, i32, i64, i32, i64, p, i32, i32, p, i32, p, p, p,
                                             p, i32]
        lib.oracle_fit_stats.argtypes = [p, i64, i32, i64, p, p, i32, i32, i32, p, p, p, p]
        _C_LIB = lib
    return _C_LIB


def c_predict(x, size, route, prior, ll, *, width: int, limit: int, threads: int = 1,
              logpost: bool = True):
    """Same contract as predict_dense, in C (pthreads over contiguous row chunks
    -- the reference's classify_parallel chunking, engine.py:264-268).  x may be
    int32, uint16 or uint8 (same counts, narrower storage)."""
    x = np.asarray(x)
    xt = {np.dtype(np.uint8): 2, np.dtype(np.uint16): 1}.get(x.dtype, 0)
    x = np.ascontiguousarray(x, dtype=x.dtype if xt else np.int32)
    size = np.ascontiguousarray(size, dtype=np.int32)
    route = np.ascontiguousarray(route, dtype=np.int32)
    prior = np.ascontiguousarray(prior, dtype=np.float64)
    ll = np.ascontiguousarray(ll, dtype=np.float64)
    n, F = x.shape
    C = prior.shape[1]
    label = np.empty(n, dtype=np.int32)
    lp = np.empty((n, C)) if logpost else None
    rc = c_oracle().oracle_predict_typed(x.ctypes.data, xt, n, F, F, size.ctypes.data, width,
                                         limit, route.ctypes.data, C, prior.ctypes.data,
                                         ll.ctypes.data, label.ctypes.data,
                                         lp.ctypes.data if lp is not None else None, threads)
    assert rc == 0
    return label, lp


def c_fit_stats(x, size, label, n_classes: int, width: int, limit: int):
    x = np.ascontiguousarray(x, dtype=np.int32)
    size = np.ascontiguousarray(size, dtype=np.int32)
    label = np.ascontiguousarray(label, dtype=np.int32)
    n, V = x.shape
    G = limit // width
    S = np.empty((G, n_classes, V), dtype=np.int64)
    Q = np.empty_like(S)
    cnt = np.empty((G, n_classes), dtype=np.int64)
    status = np.zeros(2, dtype=np.int64)
    c_oracle().oracle_fit_stats(x.ctypes.data, n, V, V, size.ctypes.data, label.ctypes.data,
                                width, limit, n_classes, S.ctypes.data, Q.ctypes.data,
                                cnt.ctypes.data, status.ctypes.data)
    return S, Q, cnt, int(status[0]), int(status[1])


# ---------------------------------------------------------------- synthetic (CPU)
def synth_dense(n: int, V: int, *, seed: int = 0, divergence: float = 0.8, width: int = 5120,
                n_classes: int = 2):
    """The reference's synthetic law (synth.py:64-116) as dense numpy arrays,
    one size group, per-cell Poisson counts (the multinomial's cell limit).
    Used by the CPU reference arm, which may not touch the GPU generator."""
    rng = np.random.default_rng(seed)
    label = (np.arange(n) % n_classes).astype(np.int32)
    size = rng.integers(0, width, size=n).astype(np.int32)
    draws = 64 + size // 64
    low = 1.0 - divergence
    bounds = [-(-b * V // n_classes) for b in range(n_classes + 1)]
    w = np.full((n_classes, V), low)
    for c in range(n_classes):
        b = n_classes - 1 - c
        w[c, bounds[b]:bounds[b + 1]] = 1.0
    p = w / w.sum(1, keepdims=True)
    x = rng.poisson(draws[:, None] * p[label]).astype(np.int32)
    return x, size, label
