"""Which object model a call speaks, resolved from the caller's own objects.

The drop-in is used two ways:

* through this package's restated object model (`model.py`, `errors.py`), or
* behind the reference package itself: `groupnb`'s own `GroupedCorpus`,
  `SampleRecord`, `ModelBundle`, `GroupModel`, `Label` ... (pkg/src/groupnb/
  corpus.py:23-124, classifier.py:18-65, engine.py:37-84), e.g. after
  `backend.install()` has rebound the reference's fit / classify_parallel.

Either way the GPU path must read the caller's enums and dict keys and hand
back -- and raise -- the caller's own types: a reference test asserting
`isinstance(run, groupnb.engine.TimedRun)` or `pytest.raises(
groupnb.errors.InsufficientClassError)` must pass.  `of(obj)` finds the
package that defines `type(obj)` and returns its classes; classes are matched
by the reference's public names, labels by identity with that package's
`Label` members (`_adapt` compares identities).
"""

from __future__ import annotations

import importlib
import sys
from dataclasses import dataclass
from typing import Any

from . import errors as _own_errors
from . import model as _own_model

_ERRORS = ("BundleValidationError", "EmptyBundleError", "GroupNBError", "InsufficientClassError",
           "IntegrityError", "InvalidConfigError", "MeasurementError", "ParseError",
           "SizeRangeError")
_TYPES = ("Label", "Prediction", "TimedRun", "Workload", "GroupModel", "FeatureSet",
          "BundleMeta", "ModelBundle", "GroupingConfig", "SampleRecord", "OpcodeHistogram")


@dataclass(frozen=True)
class Namespace:
    """The classes / functions of one object model (this package's or groupnb's)."""

    name: str
    Label: Any
    Prediction: Any
    TimedRun: Any
    Workload: Any
    GroupModel: Any
    FeatureSet: Any
    BundleMeta: Any
    ModelBundle: Any
    GroupingConfig: Any
    SampleRecord: Any
    OpcodeHistogram: Any
    build_bundle: Any
    errors: Any      # module-like: .InsufficientClassError, .IntegrityError, ...

    @property
    def MALWARE(self):
        return self.Label.MALWARE

    @property
    def BENIGN(self):
        return self.Label.BENIGN

    @property
    def CLASSES(self):
        """classifier.py:18 order (malware, benign)."""
        return (self.Label.MALWARE, self.Label.BENIGN)

    @property
    def INDEX_CLASS(self):
        """Dense class index -> label: 0 benign, 1 malware."""
        return (self.Label.BENIGN, self.Label.MALWARE)

    def class_index(self):
        return {self.Label.BENIGN: 0, self.Label.MALWARE: 1}


class _Errors:
    def __init__(self, src):
        for n in _ERRORS:
            setattr(self, n, getattr(src, n))


OWN = Namespace("paper_1905_13746_b200", *(getattr(_own_model, n) for n in _TYPES),
                _own_model.build_bundle, _Errors(_own_errors))

_cache: dict[str, Namespace] = {}
_ROOT = __name__.split(".")[0]


def _load(root: str) -> Namespace | None:
    mod = sys.modules.get(root)
    if mod is None:
        try:
            mod = importlib.import_module(root)
        except Exception:  # noqa: BLE001 -- an unknown module is simply not a namespace
            return None
    try:
        errs = getattr(mod, "errors", None) or importlib.import_module(root + ".errors")
        ns = Namespace(root, *(getattr(mod, n) for n in _TYPES), getattr(mod, "build_bundle"),
                       _Errors(errs))
    except (AttributeError, ImportError):
        return None
    return ns


def of(obj) -> Namespace:
    """The object model `obj` belongs to (this package's when unknown)."""
    root = type(obj).__module__.split(".")[0]
    if root == _ROOT:
        return OWN
    ns = _cache.get(root)
    if ns is None:
        ns = _load(root) or OWN
        _cache[root] = ns
    return ns


def of_samples(samples, default: Namespace = OWN) -> Namespace:
    """Namespace of the first sample (labels are what matters for a fit)."""
    for s in samples:
        return of(s)
    return default
