"""ctypes binding of libgnb.so (include/gnb.h).

The library is the product: there is no CPU fallback.  Importing this module
raises if the shared object is missing, and every call that fails raises with
the library's own message.
"""

from __future__ import annotations

import ctypes as C
import os
import re

from .errors import EmptyBundleError, InvalidConfigError

_HERE = os.path.dirname(os.path.abspath(__file__))
# GNB_LIB: load an alternative in-tree build (kernel experiments / profiling)
LIB_PATH = os.path.join(_HERE, os.environ.get("GNB_LIB", "libgnb.so"))
HEADER = os.path.join(os.path.dirname(_HERE), "include", "gnb.h")

GNB_OK, GNB_EINVAL, GNB_ECUDA, GNB_EUNSUPPORTED, GNB_ENOMEM = 0, 1, 2, 3, 4
GNB_MODE_EXACT, GNB_MODE_FMA = 0, 1
GNB_ORDER_AUTO, GNB_ORDER_GROUPED, GNB_ORDER_MIXED = 0, 0x10, 0x20
ROW_OUT_OF_RANGE = -1
ROW_NEGATIVE_COUNT = -2
MAX_CLASSES = 16
X_I32, X_U16, X_U8, X_U4 = 0, 1, 2, 3


class NativeError(RuntimeError):
    """A CUDA / library failure inside libgnb.so."""


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make` or __graft_entry__.build() "
            "(there is no CPU fallback)")
    return C.CDLL(LIB_PATH)


lib = _load()

_p = C.c_void_p
_i32, _i64, _u64, _f64, _sz, _up = C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_size_t, C.c_size_t

_SIGS = {
    "gnb_abi_version": ([], C.c_int),
    "gnb_strerror": ([C.c_int], C.c_char_p),
    "gnb_last_error": ([], C.c_char_p),
    "gnb_packed_table_bytes": ([_i32, _i32, _i32], _sz),
    "gnb_pack_tables": ([_p, _p, _i32, _i32, _i32, _p, _up], C.c_int),
    "gnb_predict": ([_p, _i64, _i32, _i64, _p, _i32, _i32, _p, _i32, _i32, _p, _p, _p, _up],
                    C.c_int),
    "gnb_predict_typed": ([_p, _i32, _i64, _i32, _i64, _p, _i32, _i32, _p, _i32, _i32, _p, _p,
                           _p, _up], C.c_int),
    "gnb_predict_mixed_rows": ([_i32, _i32, _i32, _i32], _i32),
    "gnb_slot_sort_workspace_bytes": ([_i64, _i32], _sz),
    "gnb_slot_sort": ([_p, _i64, _i32, _i32, _p, _i32, _p, _p, _sz, _up], C.c_int),
    "gnb_predict_permuted": ([_p, _i32, _i64, _i32, _i64, _p, _i32, _i32, _p, _i32, _i32, _p, _p,
                              _p, _p, _up], C.c_int),
    "gnb_predict_mode": ([_p, _i32, _i64, _i32, _i64, _p, _i32, _i32, _p, _i32, _i32, _p, _p,
                          _i32, _p, _p, _up], C.c_int),
    "gnb_predict_generic": ([_p, _i64, _i32, _i64, _p, _i32, _i32, _p, _i32, _i32, _p, _p, _p,
                             _up], C.c_int),
    "gnb_predict_host": ([_p, _i64, _i32, _i64, _p, _i32, _i32, _p, _i32, _i32, _p, _p, _p, _p,
                          _i32, _p], C.c_int),
    "gnb_gather_features": ([_p, _i64, _i32, _i64, _p, _i32, _i32, _p, _p, _p, _i32, _i32, _p,
                             _i64, _up], C.c_int),
    "gnb_gather_features_typed": ([_p, _i32, _i64, _i32, _i64, _p, _i32, _i32, _p, _p, _p,
                                   _i32, _i32, _p, _i64, _up], C.c_int),
    "gnb_predict_host_typed": ([_p, _i32, _i64, _i32, _i64, _p, _i32, _i32, _p, _i32, _i32, _p,
                                _p, _p, _p, _i32, _p], C.c_int),
    "gnb_predict_host_sharded": ([_p, _i32, _i64, _i32, _i64, _p, _i32, _i32, _p, _i32, _i32,
                                  _p, _p, _p, _p, _i32, _p, _p], C.c_int),
    "gnb_fit_stats_host_sharded": ([_p, _i64, _i32, _i64, _p, _p, _i32, _i32, _i32, _p, _p, _p,
                                    _p, _i32, _p], C.c_int),
    "gnb_fit_stats": ([_p, _i64, _i32, _i64, _p, _p, _i32, _i32, _i32, _p, _p, _p, _p, _i32, _up],
                      C.c_int),
    "gnb_fit_stats_typed": ([_p, _i32, _i64, _i32, _i64, _p, _p, _i32, _i32, _i32, _p, _p, _p,
                             _p, _i32, _up], C.c_int),
    "gnb_fit_stats_host": ([_p, _i64, _i32, _i64, _p, _p, _i32, _i32, _i32, _p, _p, _p, _p, _i32],
                           C.c_int),
    "gnb_fin_train": ([_p, _p, _i32, _i32, _i32, _f64, _i32, _p, _p, _p, _p, _p], C.c_int),
    "gnb_fin_train_device": ([_p, _p, _i32, _i32, _i32, _f64, _i32, _p, _p, _p, _p, _p, _up],
                             C.c_int),
    "gnb_fin_tables": ([_p, _p, _i32, _i32, _p, _i32, _f64, _p, _p], C.c_int),
    "gnb_generate": ([_p, _i64, _i32, _i64, _p, _p, _i64, _p, _i32, _i32, _i32, _f64, _u64, _p,
                      _i32, _up],
                     C.c_int),
    "gnb_comms_unique_id": ([_p], C.c_int),
    "gnb_comms_init": ([C.POINTER(_p), _i32, _p], C.c_int),
    "gnb_comms_init_rank": ([C.POINTER(_p), _i32, _i32, _p, _i32], C.c_int),
    "gnb_comms_size": ([_p], _i32),
    "gnb_comms_destroy": ([_p], None),
    "gnb_fit_allreduce": ([_p, _p, _i64, _p], C.c_int),
}

for _name, (_args, _res) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.argtypes = _args
    _fn.restype = _res


def declared_symbols() -> list[str]:
    """Every function name include/gnb.h declares (for the ABI completeness test)."""
    with open(HEADER) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(gnb_\w+)\(", text, flags=re.M)))


def check(rc: int, what: str = "") -> None:
    if rc == GNB_OK:
        return
    msg = lib.gnb_last_error().decode(errors="replace")
    if rc == GNB_EINVAL:
        if "EmptyBundleError" in msg:
            raise EmptyBundleError("bundle has no trained models")
        raise InvalidConfigError(f"{what}: {msg}" if what else msg)
    raise NativeError(f"{what}: {lib.gnb_strerror(rc).decode()}: {msg}")
