"""Dense ingestion: JSONL corpus -> vocabulary + count matrix (C++, multithreaded).

`read_corpus` is the dense counterpart of the reference's `parse_corpus`
(pkg/src/groupnb/corpus.py:133-189): same record schema, same error types,
line numbers and messages (JSON syntax errors: "invalid JSON: <reason>"),
implemented by `gnb_corpus_parse` in libgnb.so.  The vocabulary is the sorted
union of (lower-cased) mnemonics, i.e. the reference's column / tie order.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import IntegrityError, InvalidConfigError, ParseError
from .model import Label, OpcodeHistogram, SampleRecord

_L = N.lib
_p, _i32, _i64, _sz = C.c_void_p, C.c_int32, C.c_int64, C.c_size_t
_L.gnb_corpus_parse.argtypes = [C.c_void_p, _sz, _i32, _i32, C.POINTER(C.c_void_p)]
# a str's UTF-8 bytes without a copy (for ASCII text CPython's own buffer)
_utf8 = C.pythonapi.PyUnicode_AsUTF8AndSize
_utf8.restype = C.c_void_p
_utf8.argtypes = [C.py_object, C.POINTER(C.c_ssize_t)]
_L.gnb_corpus_parse.restype = C.c_int
_L.gnb_corpus_free.argtypes = [_p]
_L.gnb_corpus_free.restype = None
for _n, _r in (("gnb_corpus_rows", _i64), ("gnb_corpus_vocab_size", _i32),
               ("gnb_corpus_max_count", _i64), ("gnb_corpus_nnz", _i64)):
    getattr(_L, _n).argtypes = [_p]
    getattr(_L, _n).restype = _r
_L.gnb_corpus_vocab.argtypes = [_p, _i32]
_L.gnb_corpus_vocab.restype = C.c_char_p
_L.gnb_corpus_id.argtypes = [_p, _i64]
_L.gnb_corpus_id.restype = C.c_char_p
_L.gnb_corpus_error.argtypes = [_p, C.POINTER(_i64), C.POINTER(C.c_char_p)]
_L.gnb_corpus_error.restype = _i32
_L.gnb_corpus_meta.argtypes = [_p, _p, _p]
_L.gnb_corpus_meta.restype = C.c_int
_L.gnb_corpus_dense.argtypes = [_p, _i32, _p, _i64, _i64, _i64, _i32]
_L.gnb_corpus_dense.restype = C.c_int

_L.gnb_corpus_write_predictions.argtypes = [_p, _p, _p, _p, _i64, _i32,
                                            C.POINTER(C.c_void_p), C.POINTER(_sz)]
_L.gnb_corpus_write_predictions.restype = C.c_int
_L.gnb_free_text.argtypes = [_p]
_L.gnb_free_text.restype = None

_DTYPES = {np.dtype(np.int32): N.X_I32, np.dtype(np.uint16): N.X_U16, np.dtype(np.uint8): N.X_U8}


class DenseCorpus:
    """A parsed corpus held by the C++ library; `dense()` materialises rows."""

    def __init__(self, handle: int):
        self._h = handle
        n = _L.gnb_corpus_rows(handle)
        self.vocab = [_L.gnb_corpus_vocab(handle, k).decode() for k in
                      range(_L.gnb_corpus_vocab_size(handle))]
        self.size = np.empty(n, dtype=np.int64)
        self.label = np.empty(n, dtype=np.int8)     # 1 malware, 0 benign, -1 unlabeled
        _L.gnb_corpus_meta(handle, self.size.ctypes.data, self.label.ctypes.data)
        self.max_count = _L.gnb_corpus_max_count(handle)
        self.nnz = _L.gnb_corpus_nnz(handle)
        self._ids = None
        self._merge = None
        # The C++ parser lower-cases ASCII only; the reference lower-cases with
        # str.lower() (corpus.py:51), which also folds non-ASCII letters and so
        # can merge mnemonics the parser kept apart.  Fold those here: columns
        # whose Python-lowered keys coincide are summed (like from_counts does).
        if not all(v.isascii() for v in self.vocab):
            lowered = [v.lower() for v in self.vocab]
            if lowered != self.vocab:
                new_vocab = sorted(set(lowered))
                col = {v: j for j, v in enumerate(new_vocab)}
                self._merge = np.array([col[v] for v in lowered], dtype=np.int64)
                mult = int(np.bincount(self._merge).max())
                self.vocab = new_vocab
                self.max_count = self.max_count * mult     # bound on merged counts

    def __len__(self) -> int:
        return len(self.size)

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            _L.gnb_corpus_free(h)

    @property
    def ids(self) -> list[str]:
        if self._ids is None:
            self._ids = [_L.gnb_corpus_id(self._h, r).decode() for r in range(len(self))]
        return self._ids

    def narrowest_dtype(self):
        return np.uint8 if self.max_count < 256 else (
            np.uint16 if self.max_count < 65536 else np.int32)

    def dense(self, dtype=None, rows: slice | None = None, out: np.ndarray | None = None,
              threads: int = 0) -> np.ndarray:
        """Rows as a dense [n, V] matrix (int32 / uint16 / uint8; default: narrowest
        lossless).  `out` may be a pinned host buffer with a wider pitch."""
        dtype = np.dtype(dtype or self.narrowest_dtype())
        if dtype not in _DTYPES:
            raise InvalidConfigError(f"unsupported dense dtype {dtype}")
        lo, hi, _ = (rows or slice(0, len(self))).indices(len(self))
        V = max(len(self.vocab), 1)
        if out is None:
            out = np.empty((hi - lo, V), dtype=dtype)
        if self._merge is not None:   # fold case-variant columns (see __init__)
            raw = np.empty((hi - lo, max(len(self._merge), 1)), dtype=np.int32)
            if _L.gnb_corpus_dense(self._h, N.X_I32, raw.ctypes.data, raw.shape[1], lo,
                                   hi - lo, threads) != N.GNB_OK:
                raise InvalidConfigError("gnb_corpus_dense failed")
            merged = np.zeros((hi - lo, V), dtype=np.int64)
            np.add.at(merged.T, self._merge, raw.T)
            if merged.size and int(merged.max()) > np.iinfo(dtype).max:
                raise InvalidConfigError(f"merged counts do not fit {dtype}")
            out[:, :V] = merged
            return out
        ldx = out.strides[0] // out.itemsize
        if _L.gnb_corpus_dense(self._h, _DTYPES[dtype], out.ctypes.data, ldx, lo, hi - lo,
                               threads) != N.GNB_OK:
            raise InvalidConfigError(f"counts up to {self.max_count} do not fit {dtype}")
        return out

    def predictions_jsonl(self, label, logpost, effective_group, max_size_bytes: int,
                          threads: int = 0) -> str:
        """engine.write_predictions (engine.py:466-481) text for this corpus:
        label 1/0/<0 (error), logpost [N, 2] (benign, malware)."""
        lab = np.ascontiguousarray(label, dtype=np.int8)
        lp = np.ascontiguousarray(logpost, dtype=np.float64)
        eff = np.ascontiguousarray(effective_group, dtype=np.int32)
        if lab.shape != (len(self),) or lp.shape != (len(self), 2) or eff.shape != lab.shape:
            raise InvalidConfigError("need label [N], logpost [N, 2], effective_group [N]")
        buf, n = C.c_void_p(), _sz()
        rc = _L.gnb_corpus_write_predictions(self._h, lab.ctypes.data, lp.ctypes.data,
                                             eff.ctypes.data, max_size_bytes, threads,
                                             C.byref(buf), C.byref(n))
        if rc != N.GNB_OK:
            raise InvalidConfigError("gnb_corpus_write_predictions failed")
        try:
            return C.string_at(buf.value, n.value).decode()
        finally:
            _L.gnb_free_text(buf)

    def records(self) -> list[SampleRecord]:
        """The reference's object model (slow path, for object-API callers)."""
        x = self.dense()
        labels = {1: Label.MALWARE, 0: Label.BENIGN, -1: Label.UNKNOWN}
        out = []
        for r in range(len(self)):
            nz = np.nonzero(x[r])[0]
            out.append(SampleRecord(self.ids[r], labels[int(self.label[r])], int(self.size[r]),
                                    OpcodeHistogram({self.vocab[j]: int(x[r, j]) for j in nz})))
        return out


def read_corpus(source, *, allow_unlabeled: bool = False, threads: int = 0) -> DenseCorpus:
    """Parse JSONL text / bytes / a path into a DenseCorpus (parse_corpus contract)."""
    if isinstance(source, os.PathLike) or (
            isinstance(source, str) and "\n" not in source[:4096]
            and not source[:4096].lstrip().startswith("{") and os.path.exists(source)):
        with open(source, "rb") as fh:     # a path (text is JSONL: '{' or several lines)
            data = fh.read()
    elif isinstance(source, str):
        data = source                  # kept alive across the call
    else:
        data = bytes(source)
    if isinstance(data, str):
        n = C.c_ssize_t()
        addr = _utf8(data, C.byref(n))   # raises UnicodeEncodeError on lone surrogates
        ptr, size = addr, n.value
    else:
        ptr, size = data, len(data)
    h = C.c_void_p()
    rc = _L.gnb_corpus_parse(ptr, size, 1 if allow_unlabeled else 0, threads, C.byref(h))
    if rc != N.GNB_OK:
        line, msg = _i64(), C.c_char_p()
        kind = _L.gnb_corpus_error(h, C.byref(line), C.byref(msg))
        text = msg.value.decode(errors="replace")
        _L.gnb_corpus_free(h)
        if kind == 2:
            raise IntegrityError(text)
        if kind == 1:
            raise ParseError(int(line.value), text)
        raise InvalidConfigError("gnb_corpus_parse failed")
    return DenseCorpus(h.value)


def parse_corpus(stream, *, allow_unlabeled: bool = False) -> list[SampleRecord]:
    """corpus.parse_corpus (corpus.py:133-189) through the C++ parser."""
    if not isinstance(stream, (str, bytes)):
        stream = "\n".join(line.rstrip("\r\n") for line in stream)
    return read_corpus(stream, allow_unlabeled=allow_unlabeled).records()
