"""Object model of the reference's hot-path API, restated for the GPU engine.

Same class names, fields, invariants and error types as the reference
(pkg/src/groupnb/corpus.py:23-124, features.py:33-38, classifier.py:18-65,
engine.py:37-154), so code written against `groupnb` can switch to this
package for the fit / classify path.  Only what that path touches is here;
JSONL parsing, splitting, bundle JSON and the CLI stay in the reference.
"""

from __future__ import annotations

import math
import sys
from bisect import bisect_left
from dataclasses import dataclass, field
from enum import Enum
from typing import Iterable, Mapping

from .errors import BundleValidationError, EmptyBundleError, IntegrityError, InvalidConfigError


def _positive_int(value) -> bool:
    return isinstance(value, int) and not isinstance(value, bool) and value > 0


class Label(Enum):
    """Sample class (corpus.py:23-28).  Dense class index: BENIGN 0, MALWARE 1."""

    MALWARE = "malware"
    BENIGN = "benign"
    UNKNOWN = "unknown"


CLASSES = (Label.MALWARE, Label.BENIGN)  # classifier.py:18 order
CLASS_INDEX = {Label.BENIGN: 0, Label.MALWARE: 1}
INDEX_CLASS = (Label.BENIGN, Label.MALWARE)


@dataclass(frozen=True)
class OpcodeHistogram:
    """mnemonic -> positive count, lower-case keys (corpus.py:31-59)."""

    entries: dict[str, int]

    @classmethod
    def from_counts(cls, counts: Mapping[str, int]) -> "OpcodeHistogram":
        merged: dict[str, int] = {}
        for op, n in counts.items():
            if not isinstance(op, str) or op == "":
                raise ValueError(f"opcode mnemonic must be a non-empty string, got {op!r}")
            if isinstance(n, bool) or not isinstance(n, int) or n < 0:
                raise ValueError(f"count for {op!r} must be a non-negative integer, got {n!r}")
            if n:
                key = sys.intern(op.lower())  # shared key objects: identity hits in lookups
                merged[key] = merged.get(key, 0) + n
        return cls(merged)

    def total(self) -> int:
        return sum(self.entries.values())

    def get(self, mnemonic: str, default: int = 0) -> int:
        return self.entries.get(mnemonic, default)


@dataclass(frozen=True)
class SampleRecord:
    id: str
    label: Label
    size_bytes: int
    histogram: OpcodeHistogram


@dataclass(frozen=True)
class GroupingConfig:
    """Size-group geometry (corpus.py:72-98): 5120-B groups below 512000 B."""

    group_size_bytes: int = 5120
    max_size_bytes: int = 512000
    min_per_class: int = 6

    def __post_init__(self):
        for name in ("group_size_bytes", "max_size_bytes", "min_per_class"):
            if not _positive_int(getattr(self, name)):
                raise InvalidConfigError(
                    f"{name} must be a positive integer, got {getattr(self, name)!r}")
        if self.max_size_bytes % self.group_size_bytes:
            raise InvalidConfigError(
                f"max_size_bytes ({self.max_size_bytes}) must be divisible by "
                f"group_size_bytes ({self.group_size_bytes})")

    @property
    def group_count(self) -> int:
        return self.max_size_bytes // self.group_size_bytes


@dataclass(frozen=True)
class GroupedCorpus:
    config: GroupingConfig
    groups: dict[int, list[SampleRecord]]

    def sample_count(self) -> int:
        return sum(map(len, self.groups.values()))

    def all_samples(self) -> list[SampleRecord]:
        return [s for g in sorted(self.groups) for s in self.groups[g]]


def partition_by_group(samples: Iterable[SampleRecord], config: GroupingConfig):
    """(GroupedCorpus, rejected) by size (corpus.py:235-252)."""
    groups: dict[int, list[SampleRecord]] = {}
    rejected: list[SampleRecord] = []
    for s in samples:
        if 0 <= s.size_bytes < config.max_size_bytes:
            groups.setdefault(s.size_bytes // config.group_size_bytes, []).append(s)
        else:
            rejected.append(s)
    return GroupedCorpus(config, groups), rejected


@dataclass(frozen=True)
class FeatureSet:
    """Top-k opcodes in score order (features.py:33-38)."""

    opcodes: tuple[str, ...]
    k: int


@dataclass(frozen=True)
class GroupModel:
    """One size group's NB parameters (classifier.py:21-52)."""

    group: int
    features: FeatureSet
    log_prior: dict[Label, float]
    log_likelihood: dict[Label, dict[str, float]]
    alpha: float
    train_counts: dict[Label, int]
    # (opcode, ll_malware, ll_benign) rows in FeatureSet order: the summation
    # order every scoring path follows (classifier.py:36-52)
    _packed: tuple[tuple[str, float, float], ...] = field(init=False, repr=False, compare=False)

    def __post_init__(self):
        ll_m = self.log_likelihood.get(Label.MALWARE, {})
        ll_b = self.log_likelihood.get(Label.BENIGN, {})
        packed = []
        for op in self.features.opcodes:
            if op not in ll_m or op not in ll_b:
                raise IntegrityError(f"group {self.group}: log_likelihood missing feature {op!r}")
            packed.append((op, ll_m[op], ll_b[op]))
        object.__setattr__(self, "_packed", tuple(packed))


@dataclass(frozen=True)
class Prediction:
    label: Label
    log_posterior: dict[Label, float]
    effective_group: int


@dataclass(frozen=True)
class BundleMeta:
    k: int
    alpha: float
    seed: int
    created_at: str


def _route_ids(ids, group: int) -> int:
    i = bisect_left(ids, group)
    return ids[i] if i < len(ids) else ids[-1]


@dataclass(frozen=True)
class ModelBundle:
    """Immutable per-group models + routing table (engine.py:45-59)."""

    config: GroupingConfig
    models: dict[int, GroupModel]
    trained_ids: tuple[int, ...]
    meta: BundleMeta
    _route_table: tuple[int, ...] = field(init=False, repr=False, compare=False)

    def __post_init__(self):
        ids = self.trained_ids
        table = tuple(_route_ids(ids, g) for g in range(self.config.group_count)) if ids else ()
        object.__setattr__(self, "_route_table", table)


def route(bundle: ModelBundle, group: int) -> int:
    """Trained group serving `group`: itself, else the next trained id above,
    else the largest trained id (engine.py:87-103)."""
    if not bundle.trained_ids:
        raise EmptyBundleError("bundle has no trained models")
    return _route_ids(bundle.trained_ids, group)


_SUM_TOL = 1e-9


def validate_model(model: GroupModel, config: GroupingConfig, meta: BundleMeta) -> None:
    """Bundle invariants (engine.py:106-135)."""
    where = f"model for group {model.group}"
    n = len(model.features.opcodes)
    if not 0 <= model.group < config.group_count:
        raise BundleValidationError(f"{where}: group id outside [0, {config.group_count})")
    if n == 0:
        raise BundleValidationError(f"{where}: empty feature set")
    if n > meta.k:
        raise BundleValidationError(f"{where}: {n} features exceeds k={meta.k}")
    if len(set(model.features.opcodes)) != n:
        raise BundleValidationError(f"{where}: duplicate features")
    if not (model.alpha > 0 and math.isfinite(model.alpha)):
        raise BundleValidationError(f"{where}: alpha must be positive and finite")
    prior_sum = sum(math.exp(model.log_prior[c]) for c in CLASSES)
    if abs(prior_sum - 1.0) > _SUM_TOL:
        raise BundleValidationError(f"{where}: priors sum to {prior_sum!r}, not 1")
    for c in CLASSES:
        if model.train_counts.get(c, 0) < 1:
            raise BundleValidationError(f"{where}: no {c.value} training samples recorded")
        total = 0.0
        for op in model.features.opcodes:
            v = model.log_likelihood[c][op]
            if not math.isfinite(v):
                raise BundleValidationError(f"{where}: non-finite likelihood for {op!r}")
            total += math.exp(v)
        if abs(total - 1.0) > _SUM_TOL:
            raise BundleValidationError(f"{where}: {c.value} likelihoods sum to {total!r}, not 1")


def build_bundle(models: Iterable[GroupModel], config: GroupingConfig,
                 meta: BundleMeta) -> ModelBundle:
    """Validate and assemble; trained_ids ascending (engine.py:138-154)."""
    by_group: dict[int, GroupModel] = {}
    for m in models:
        if m.group in by_group:
            raise IntegrityError(f"duplicate model for group {m.group}")
        validate_model(m, config, meta)
        by_group[m.group] = m
    ids = tuple(sorted(by_group))
    return ModelBundle(config=config, models={g: by_group[g] for g in ids}, trained_ids=ids,
                       meta=meta)


@dataclass(frozen=True)
class Workload:
    samples: tuple[SampleRecord, ...]
    lanes: int

    def __post_init__(self):
        if not _positive_int(self.lanes):
            raise InvalidConfigError(f"lanes must be a positive integer, got {self.lanes!r}")


@dataclass(frozen=True)
class TimedRun:
    """Predictions in input order (None where errors has the index) + elapsed ns."""

    predictions: tuple[Prediction | None, ...]
    errors: tuple[tuple[int, str], ...]
    elapsed_ns: int


def oversize_message(size_bytes: int, limit: int) -> str:
    """engine.py:183-184."""
    return f"size_bytes {size_bytes} outside [0, {limit})"


def trainable_groups(train: GroupedCorpus, config: GroupingConfig) -> set[int]:
    """Groups with >= min_per_class of each class (corpus.py:295-307)."""
    out = set()
    for g, samples in train.groups.items():
        m = sum(s.label is Label.MALWARE for s in samples)
        b = sum(s.label is Label.BENIGN for s in samples)
        if m >= config.min_per_class and b >= config.min_per_class:
            out.add(g)
    return out


def normalized_posterior(scores: Mapping[Label, float]) -> dict[Label, float]:
    """Diagnostic softmax of joint log-scores (classifier.py:161-166)."""
    top = max(scores.values())
    ex = {c: math.exp(v - top) for c, v in scores.items()}
    z = sum(ex.values())
    return {c: e / z for c, e in ex.items()}
