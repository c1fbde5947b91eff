"""B200-native group-wise Naive Bayes hot path (arXiv 1905.13746).

Hand-written sm_100a CUDA kernels (libgnb.so, C ABI in include/gnb.h) behind
the reference package's fit / classify operation contract.

    from paper_1905_13746_b200 import train_bundle, classify_parallel   # object API
    from paper_1905_13746_b200 import dense                             # device tensors
    from paper_1905_13746_b200 import backend; backend.install()        # behind groupnb itself
"""

from . import _native  # noqa: F401  -- fails loudly if libgnb.so is missing
from .api import (classify_gpu, classify_parallel, classify_sequential, log_posterior, predict,
                  speedup, train_bundle, train_bundles, train_group)
from .errors import (BundleValidationError, EmptyBundleError, GroupNBError,
                     InsufficientClassError, IntegrityError, InvalidConfigError,
                     MeasurementError, ParseError, SizeRangeError)
from .model import (CLASSES, BundleMeta, FeatureSet, GroupedCorpus, GroupingConfig, GroupModel,
                    Label, ModelBundle, OpcodeHistogram, Prediction, SampleRecord, TimedRun,
                    Workload, build_bundle, normalized_posterior, partition_by_group, route,
                    trainable_groups)

__all__ = [
    "BundleMeta", "BundleValidationError", "CLASSES", "EmptyBundleError", "FeatureSet",
    "GroupModel", "GroupNBError", "GroupedCorpus", "GroupingConfig", "InsufficientClassError",
    "IntegrityError", "InvalidConfigError", "Label", "MeasurementError", "ModelBundle",
    "OpcodeHistogram", "ParseError", "Prediction", "SampleRecord", "SizeRangeError", "TimedRun",
    "Workload", "build_bundle", "classify_gpu", "classify_parallel", "classify_sequential",
    "log_posterior", "normalized_posterior", "partition_by_group", "predict", "route",
    "speedup", "train_bundle", "train_bundles", "train_group", "trainable_groups",
]
