// ADAPT (CPython extension `_adapt`): the reference's object model -> dense
// arrays, in C ("C++ ADAPT packer for Workload").
//
// The GPU path consumes dense rows; the reference hands it SampleRecord
// objects whose histograms are dicts (pkg/src/groupnb/corpus.py:31-69).
// Walking those dicts from Python costs ~1 us per entry; here the same walk is
// plain C-API dict iteration.  Semantics are those of the Python packers in
// api.py (column maps, routing by size as engine._classify_slice does,
// engine.py:198-202); counts must fit int32.
#define PY_SSIZE_T_CLEAN
#include <Python.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

namespace {

struct Buf {
  Py_buffer view{};
  bool ok = false;
  ~Buf() {
    if (ok) PyBuffer_Release(&view);
  }
  bool get(PyObject* o, Py_ssize_t itemsize, Py_ssize_t want_len) {
    if (PyObject_GetBuffer(o, &view, PyBUF_WRITABLE | PyBUF_C_CONTIGUOUS) != 0) return false;
    ok = true;
    if (view.itemsize != itemsize || view.len < want_len * itemsize) {
      PyErr_SetString(PyExc_ValueError, "output buffer has the wrong item size or length");
      return false;
    }
    return true;
  }
};

PyObject* s_histogram = nullptr;
PyObject* s_entries = nullptr;
PyObject* s_size_bytes = nullptr;
PyObject* s_label = nullptr;

// entries dict of sample i (borrowed from a new reference we release)
PyObject* entries_of(PyObject* sample) {
  PyObject* h = PyObject_GetAttr(sample, s_histogram);
  if (!h) return nullptr;
  PyObject* e = PyObject_GetAttr(h, s_entries);
  Py_DECREF(h);
  if (e && !PyDict_Check(e)) {
    Py_DECREF(e);
    PyErr_SetString(PyExc_TypeError, "histogram.entries must be a dict");
    return nullptr;
  }
  return e;
}

bool put_count(int32_t* row, Py_ssize_t j, PyObject* v) {
  const long long n = PyLong_AsLongLong(v);
  if (n == -1 && PyErr_Occurred()) return false;
  if (n < 0 || n > 2147483647LL) {
    PyErr_SetString(PyExc_OverflowError, "opcode counts must be in [0, 2^31) for the GPU path");
    return false;
  }
  row[j] = static_cast<int32_t>(n);
  return true;
}

// densify_into(samples, columns: dict[str, int], out: int32 buffer [N, width], width)
PyObject* densify_into_serial(PyObject*, PyObject* args) {
  PyObject *samples, *columns, *out;
  Py_ssize_t width;
  if (!PyArg_ParseTuple(args, "OO!On", &samples, &PyDict_Type, &columns, &out, &width))
    return nullptr;
  PyObject* seq = PySequence_Fast(samples, "samples must be a sequence");
  if (!seq) return nullptr;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(seq);
  Buf b;
  if (!b.get(out, 4, n * width)) {
    Py_DECREF(seq);
    return nullptr;
  }
  int32_t* x = static_cast<int32_t*>(b.view.buf);
  for (Py_ssize_t i = 0; i < n; ++i) {
    PyObject* e = entries_of(PySequence_Fast_GET_ITEM(seq, i));
    if (!e) {
      Py_DECREF(seq);
      return nullptr;
    }
    Py_ssize_t pos = 0;
    PyObject *k, *v;
    while (PyDict_Next(e, &pos, &k, &v)) {
      PyObject* col = PyDict_GetItemWithError(columns, k);
      if (!col) {
        if (PyErr_Occurred()) {
          Py_DECREF(e);
          Py_DECREF(seq);
          return nullptr;
        }
        continue;
      }
      const Py_ssize_t j = PyLong_AsSsize_t(col);
      if (j < 0 || j >= width || !put_count(x + i * width, j, v)) {
        if (!PyErr_Occurred()) PyErr_SetString(PyExc_IndexError, "column out of range");
        Py_DECREF(e);
        Py_DECREF(seq);
        return nullptr;
      }
    }
    Py_DECREF(e);
  }
  Py_DECREF(seq);
  Py_RETURN_NONE;
}

PyObject* gather_into_serial(PyObject*, PyObject* args);

// ------------------------------------------------------------------ parallel gather
// The dict walk of gather_into is ~3 us per sample (~85 entries) on one core,
// 20x the device call.  gather_into splits it in two:
//   1. serial, GIL held: per sample size_bytes -> slot, and a new reference
//      to its entries dict (the only steps that touch reference counts);
//   2. host threads walk the dicts with PyDict_Next and look each key up in a
//      C++ table built from the model column maps (exact str keys compared by
//      identity, then by cached hash + code points).
// The calling thread keeps the GIL for the whole call, so no Python code runs
// while the workers read: they only read dict storage, str data and compact
// int values -- no reference counts, no allocation, no exceptions.  Anything
// outside that (non-str keys, uncached hashes, non-int or out-of-range
// counts) makes the call redo the rows with the serial walk above, which
// raises exactly the serial path's errors.
struct KeyTable {
  std::vector<PyObject*> slot_key;  // open addressing, power-of-two size
  std::vector<int32_t> slot_id;
  size_t mask = 0;

  static Py_hash_t cached_hash(PyObject* k) {
    return reinterpret_cast<PyASCIIObject*>(k)->hash;
  }
  static bool same(PyObject* a, PyObject* b) {
    if (a == b) return true;
    const Py_ssize_t n = PyUnicode_GET_LENGTH(a);
    const int kind = PyUnicode_KIND(a);
    return n == PyUnicode_GET_LENGTH(b) && kind == PyUnicode_KIND(b) &&
           memcmp(PyUnicode_DATA(a), PyUnicode_DATA(b), size_t(n) * kind) == 0;
  }
  void reserve(size_t n) {
    size_t cap = 16;
    while (cap < 2 * n) cap <<= 1;
    slot_key.assign(cap, nullptr);
    slot_id.assign(cap, -1);
    mask = cap - 1;
  }
  // GIL held; k exact str with its hash computed.  Returns the id of k.
  int32_t insert(PyObject* k, int32_t next_id) {
    for (size_t i = size_t(cached_hash(k)) & mask;; i = (i + 1) & mask) {
      if (!slot_key[i]) {
        slot_key[i] = k;
        slot_id[i] = next_id;
        return next_id;
      }
      if (same(slot_key[i], k)) return slot_id[i];
    }
  }
  // insert with growth (worker-local tables): keys get ids 0, 1, ... in
  // first-seen order, recorded in `order`
  std::vector<PyObject*> order;
  int32_t add(PyObject* k) {
    if (2 * (order.size() + 1) > slot_key.size()) {
      std::vector<PyObject*> old = order;
      reserve(2 * old.size() + 8);
      order.clear();
      for (PyObject* q : old) add(q);
    }
    const int32_t id = insert(k, static_cast<int32_t>(order.size()));
    if (id == static_cast<int32_t>(order.size())) order.push_back(k);
    return id;
  }
  // worker-safe (reads only); -1 = not present
  int32_t find(PyObject* k, Py_hash_t h) const {
    for (size_t i = size_t(h) & mask;; i = (i + 1) & mask) {
      PyObject* q = slot_key[i];
      if (!q) return -1;
      if (q == k || (cached_hash(q) == h && same(q, k))) return slot_id[i];
    }
  }
};

// Threads walk rows' entries dicts (null = skip) and write each count at
// slot_col[slots[i]][id(key)]; false when any entry is outside the read-only
// rules (the caller then redoes the call serially).
bool walk_rows(const std::vector<PyObject*>& ents, const std::vector<int32_t>& slots,
               const KeyTable& tab, const std::vector<int32_t>& slot_col, int32_t uids,
               int32_t* x, Py_ssize_t width, int W) {
  const Py_ssize_t n = static_cast<Py_ssize_t>(ents.size());
  std::atomic<int> bad{0};
  auto work = [&](int w) {
    const Py_ssize_t lo = n * w / W, hi = n * (w + 1) / W;
    for (Py_ssize_t i = lo; i < hi && !bad.load(std::memory_order_relaxed); ++i) {
      PyObject* e = ents[size_t(i)];
      if (!e) continue;
      const int32_t* cols = slot_col.data() + size_t(slots[size_t(i)]) * uids;
      int32_t* row = x + i * width;
      Py_ssize_t pos = 0;
      PyObject *k, *v;
      while (PyDict_Next(e, &pos, &k, &v)) {
        if (!PyUnicode_CheckExact(k) || !PyLong_CheckExact(v)) {
          bad.store(1);
          return;
        }
        const Py_hash_t h = KeyTable::cached_hash(k);
        if (h == -1) {
          bad.store(1);
          return;
        }
        const int32_t id = tab.find(k, h);
        if (id < 0) continue;
        const int32_t j = cols[id];
        if (j < 0) continue;
        int overflow = 0;
        const long long c = PyLong_AsLongLongAndOverflow(v, &overflow);
        if (overflow || c < 0 || c > 2147483647LL) {
          bad.store(1);
          return;
        }
        row[j] = static_cast<int32_t>(c);
      }
    }
  };
  std::vector<std::thread> th;
  th.reserve(size_t(W - 1));
  for (int w = 1; w < W; ++w) th.emplace_back(work, w);
  work(0);
  for (auto& t : th) t.join();
  return bad.load() == 0;
}

// Column map (exact str keys -> int columns in [0, width)) as a key table
// plus uid -> column; false if the map is outside those rules.
bool column_table(PyObject* columns, Py_ssize_t width, KeyTable& tab, std::vector<int32_t>& col,
                  int32_t& uids) {
  tab.reserve(size_t(PyDict_GET_SIZE(columns)) + 1);
  uids = 0;
  std::vector<int32_t> tmp;
  Py_ssize_t pos = 0;
  PyObject *k, *v;
  while (PyDict_Next(columns, &pos, &k, &v)) {
    if (!PyUnicode_CheckExact(k) || !PyLong_CheckExact(v) || PyObject_Hash(k) == -1) {
      PyErr_Clear();
      return false;
    }
    const Py_ssize_t j = PyLong_AsSsize_t(v);
    if (j < 0 || j >= width) {
      PyErr_Clear();
      return false;
    }
    const int32_t id = tab.insert(k, uids);
    if (id == uids) {
      ++uids;
      tmp.push_back(static_cast<int32_t>(j));
    } else {
      tmp[size_t(id)] = static_cast<int32_t>(j);
    }
  }
  col = std::move(tmp);
  if (col.empty()) col.push_back(-1);
  return true;
}

// densify_into for >= 8192 samples: every row, one column map, threaded walk
// (same rules as gather_into); anything unusual -> the serial densify walk.
PyObject* densify_into_serial(PyObject*, PyObject* args);
PyObject* densify_into(PyObject* self, PyObject* args) {
  PyObject *samples, *columns, *out;
  Py_ssize_t width;
  if (!PyArg_ParseTuple(args, "OO!On", &samples, &PyDict_Type, &columns, &out, &width))
    return nullptr;
  const unsigned hw = std::thread::hardware_concurrency();
  const int W = static_cast<int>(std::min(hw ? hw : 1u, 32u));
  const Py_ssize_t n_hint = PyObject_Length(samples);
  if (n_hint < 0) PyErr_Clear();
  KeyTable tab;
  std::vector<int32_t> col;
  int32_t uids = 0;
  if (W < 2 || n_hint < 8192 || !column_table(columns, width, tab, col, uids))
    return densify_into_serial(self, args);
  PyObject* seq = PySequence_Fast(samples, "samples must be a sequence");
  if (!seq) return nullptr;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(seq);
  Buf b;
  if (!b.get(out, 4, n * width)) {
    Py_DECREF(seq);
    return nullptr;
  }
  std::vector<PyObject*> ents(size_t(n), nullptr);
  std::vector<int32_t> slots(size_t(n), 0);
  auto release = [&] {
    for (PyObject* e : ents) Py_XDECREF(e);
    Py_DECREF(seq);
  };
  for (Py_ssize_t i = 0; i < n; ++i) {
    PyObject* e = entries_of(PySequence_Fast_GET_ITEM(seq, i));
    if (!e) {
      release();
      return nullptr;
    }
    ents[size_t(i)] = e;
  }
  const bool ok = walk_rows(ents, slots, tab, col, uids, static_cast<int32_t*>(b.view.buf),
                            width, W);
  release();
  if (!ok) return densify_into_serial(self, args);
  Py_RETURN_NONE;
}

PyObject* gather_into(PyObject* self, PyObject* args) {
  PyObject *samples, *route_o, *colmaps, *out, *sizes_o;
  Py_ssize_t width, group_width, limit;
  if (!PyArg_ParseTuple(args, "OOO!nnnOO", &samples, &route_o, &PyList_Type, &colmaps, &width,
                        &group_width, &limit, &out, &sizes_o))
    return nullptr;
  const unsigned hw = std::thread::hardware_concurrency();
  const int W = static_cast<int>(std::min(hw ? hw : 1u, 32u));
  const Py_ssize_t n_hint = PyObject_Length(samples);
  if (n_hint < 0) PyErr_Clear();
  if (W < 2 || n_hint < 8192 || group_width <= 0) return gather_into_serial(self, args);

  // column maps -> one key table (union of every model's features) and a
  // per-slot uid -> column array; anything but exact str keys / int columns:
  // serial path
  const Py_ssize_t S = PyList_GET_SIZE(colmaps);
  Py_ssize_t total = 0;
  for (Py_ssize_t s = 0; s < S; ++s) {
    PyObject* cm = PyList_GET_ITEM(colmaps, s);
    if (!PyDict_Check(cm)) return gather_into_serial(self, args);
    total += PyDict_GET_SIZE(cm);
  }
  KeyTable tab;
  tab.reserve(size_t(total) + 1);
  std::vector<std::vector<std::pair<int32_t, int32_t>>> slot_pairs(static_cast<size_t>(S));
  int32_t uids = 0;
  for (Py_ssize_t s = 0; s < S; ++s) {
    Py_ssize_t pos = 0;
    PyObject *k, *v;
    while (PyDict_Next(PyList_GET_ITEM(colmaps, s), &pos, &k, &v)) {
      if (!PyUnicode_CheckExact(k) || !PyLong_CheckExact(v)) return gather_into_serial(self, args);
      if (PyObject_Hash(k) == -1) return nullptr;
      const Py_ssize_t j = PyLong_AsSsize_t(v);
      if (j < 0 || j >= width) return gather_into_serial(self, args);  // raises IndexError
      const int32_t id = tab.insert(k, uids);
      if (id == uids) ++uids;
      slot_pairs[size_t(s)].emplace_back(id, static_cast<int32_t>(j));
    }
  }
  std::vector<int32_t> slot_col(size_t(S) * std::max<int32_t>(uids, 1), -1);
  for (Py_ssize_t s = 0; s < S; ++s)
    for (auto [id, j] : slot_pairs[size_t(s)]) slot_col[size_t(s) * uids + id] = j;

  PyObject* seq = PySequence_Fast(samples, "samples must be a sequence");
  if (!seq) return nullptr;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(seq);
  Buf bx, bs, br;
  const Py_ssize_t G = limit / group_width;
  if (!bx.get(out, 4, n * width) || !bs.get(sizes_o, 4, n) || !br.get(route_o, 4, G)) {
    Py_DECREF(seq);
    return nullptr;
  }
  int32_t* x = static_cast<int32_t*>(bx.view.buf);
  int32_t* sz = static_cast<int32_t*>(bs.view.buf);
  const int32_t* route = static_cast<const int32_t*>(br.view.buf);

  // 1. serial: sizes, slots, entries dicts (new references, released below)
  std::vector<PyObject*> ents(size_t(n), nullptr);
  std::vector<int32_t> slots(size_t(n), -1);
  auto release = [&] {
    for (PyObject* e : ents) Py_XDECREF(e);
    Py_DECREF(seq);
  };
  bool serial = false;
  for (Py_ssize_t i = 0; i < n && !serial; ++i) {
    PyObject* s = PySequence_Fast_GET_ITEM(seq, i);
    PyObject* so = PyObject_GetAttr(s, s_size_bytes);
    if (!so) {
      release();
      return nullptr;
    }
    int overflow = 0;
    const long long size = PyLong_AsLongLongAndOverflow(so, &overflow);
    Py_DECREF(so);
    if (size == -1 && PyErr_Occurred()) {
      release();
      return nullptr;
    }
    if (overflow || size < 0 || size >= limit) continue;  // row stays zero, sz = -1 below
    const int32_t slot = route[size / group_width];
    if (slot < 0 || slot >= S) {
      serial = true;  // the serial walk raises the IndexError
      break;
    }
    PyObject* e = entries_of(s);
    if (!e) {
      release();
      return nullptr;
    }
    ents[size_t(i)] = e;
    slots[size_t(i)] = slot;
    sz[i] = static_cast<int32_t>(size / group_width);  // size group id (any size range)
  }
  // 2. parallel dict walks (reads only; see above)
  const bool bad = !serial && !walk_rows(ents, slots, tab, slot_col, uids, x, width, W);
  // rows outside [0, limit) (their ents entry is null) get size -1
  for (Py_ssize_t i = 0; i < n; ++i)
    if (!ents[size_t(i)] && !serial) sz[i] = -1;
  release();
  if (serial || bad) return gather_into_serial(self, args);
  Py_RETURN_NONE;
}

// vocab_dense(samples) -> (ops, bytearray) | None: _dense_vocab in one call --
// the sorted union of the histograms' opcodes and the [N, max(V, 1)] int32
// counts in that column order, built by host threads (same read-only rules
// as gather_into: the GIL stays held, the serial phase takes the references).
//   A. threads collect the distinct keys of their rows;
//   B. serial: union, sorted by code point (Python's str order);
//   C. threads zero their rows and write each count at its sorted column.
// None = an input outside the fast path's rules (non-str keys, non-int or
// out-of-range counts, fewer than 8192 samples): the caller uses the serial
// discover_into walk, which raises the serial errors.
PyObject* vocab_dense(PyObject*, PyObject* args) {
  PyObject* samples;
  if (!PyArg_ParseTuple(args, "O", &samples)) return nullptr;
  const unsigned hw = std::thread::hardware_concurrency();
  const int W = static_cast<int>(std::min(hw ? hw : 1u, 32u));
  PyObject* seq = PySequence_Fast(samples, "samples must be a sequence");
  if (!seq) return nullptr;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(seq);
  if (W < 2 || n < 8192) {
    Py_DECREF(seq);
    Py_RETURN_NONE;
  }
  std::vector<PyObject*> ents(size_t(n), nullptr);
  auto release = [&] {
    for (PyObject* e : ents) Py_XDECREF(e);
    Py_DECREF(seq);
  };
  for (Py_ssize_t i = 0; i < n; ++i) {
    PyObject* e = entries_of(PySequence_Fast_GET_ITEM(seq, i));
    if (!e) {
      release();
      return nullptr;
    }
    ents[size_t(i)] = e;
  }
  auto run = [&](auto&& fn) {
    std::vector<std::thread> th;
    th.reserve(size_t(W - 1));
    for (int w = 1; w < W; ++w) th.emplace_back(fn, w);
    fn(0);
    for (auto& t : th) t.join();
  };
  // A. distinct keys per thread
  std::atomic<int> bad{0};
  std::vector<KeyTable> local(static_cast<size_t>(W));
  run([&](int w) {
    KeyTable& t = local[size_t(w)];
    t.reserve(64);
    const Py_ssize_t lo = n * w / W, hi = n * (w + 1) / W;
    for (Py_ssize_t i = lo; i < hi; ++i) {
      Py_ssize_t pos = 0;
      PyObject *k, *v;
      while (PyDict_Next(ents[size_t(i)], &pos, &k, &v)) {
        if (!PyUnicode_CheckExact(k) || !PyLong_CheckExact(v) || KeyTable::cached_hash(k) == -1) {
          bad.store(1);
          return;
        }
        t.add(k);
      }
    }
  });
  if (bad.load()) {
    release();
    Py_RETURN_NONE;
  }
  // B. union, code-point order
  KeyTable all;
  all.reserve(64);
  for (const KeyTable& t : local)
    for (PyObject* k : t.order) all.add(k);
  std::vector<PyObject*> ops = all.order;
  std::sort(ops.begin(), ops.end(),
            [](PyObject* a, PyObject* b) { return PyUnicode_Compare(a, b) < 0; });
  KeyTable col;  // key -> sorted column
  col.reserve(ops.size() + 1);
  for (size_t j = 0; j < ops.size(); ++j) col.insert(ops[j], static_cast<int32_t>(j));
  const Py_ssize_t V = std::max<Py_ssize_t>(static_cast<Py_ssize_t>(ops.size()), 1);
  PyObject* buf = PyByteArray_FromStringAndSize(nullptr, n * V * 4);
  if (!buf) {
    release();
    return nullptr;
  }
  int32_t* x = reinterpret_cast<int32_t*>(PyByteArray_AS_STRING(buf));
  // C. rows
  run([&](int w) {
    const Py_ssize_t lo = n * w / W, hi = n * (w + 1) / W;
    memset(x + lo * V, 0, size_t(hi - lo) * V * 4);
    for (Py_ssize_t i = lo; i < hi; ++i) {
      Py_ssize_t pos = 0;
      PyObject *k, *v;
      int32_t* row = x + i * V;
      while (PyDict_Next(ents[size_t(i)], &pos, &k, &v)) {
        int overflow = 0;
        const long long c = PyLong_AsLongLongAndOverflow(v, &overflow);
        if (overflow || c < 0 || c > 2147483647LL) {
          bad.store(1);
          return;
        }
        row[col.find(k, KeyTable::cached_hash(k))] = static_cast<int32_t>(c);
      }
    }
  });
  if (bad.load()) {
    Py_DECREF(buf);
    release();
    Py_RETURN_NONE;
  }
  PyObject* names = PyList_New(static_cast<Py_ssize_t>(ops.size()));
  if (!names) {
    Py_DECREF(buf);
    release();
    return nullptr;
  }
  for (size_t j = 0; j < ops.size(); ++j) {
    Py_INCREF(ops[j]);
    PyList_SET_ITEM(names, static_cast<Py_ssize_t>(j), ops[j]);
  }
  release();
  PyObject* r = PyTuple_Pack(2, names, buf);
  Py_DECREF(names);
  Py_DECREF(buf);
  return r;
}

// gather_into(samples, route: int32 buffer [G], colmaps: list[dict], width, limit,
//             out: int32 [N, width], sizes_out: int32 [N])
// Row i gets the counts of its routed model's features (FeatureSet order);
// sizes_out[i] = its size group (size // group_width), or -1 (row left zero)
// for sizes outside [0, limit): callers score with width 1 / limit G, so
// size ranges beyond int32 route exactly.
PyObject* gather_into_serial(PyObject*, PyObject* args) {
  PyObject *samples, *route_o, *colmaps, *out, *sizes_o;
  Py_ssize_t width, group_width, limit;
  if (!PyArg_ParseTuple(args, "OOO!nnnOO", &samples, &route_o, &PyList_Type, &colmaps, &width,
                        &group_width, &limit, &out, &sizes_o))
    return nullptr;
  PyObject* seq = PySequence_Fast(samples, "samples must be a sequence");
  if (!seq) return nullptr;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(seq);
  Buf bx, bs, br;
  const Py_ssize_t G = limit / group_width;
  if (!bx.get(out, 4, n * width) || !bs.get(sizes_o, 4, n) || !br.get(route_o, 4, G)) {
    Py_DECREF(seq);
    return nullptr;
  }
  int32_t* x = static_cast<int32_t*>(bx.view.buf);
  int32_t* sz = static_cast<int32_t*>(bs.view.buf);
  const int32_t* route = static_cast<const int32_t*>(br.view.buf);
  const Py_ssize_t S = PyList_GET_SIZE(colmaps);
  for (Py_ssize_t i = 0; i < n; ++i) {
    PyObject* s = PySequence_Fast_GET_ITEM(seq, i);
    PyObject* so = PyObject_GetAttr(s, s_size_bytes);
    if (!so) {
      Py_DECREF(seq);
      return nullptr;
    }
    int overflow = 0;
    const long long size = PyLong_AsLongLongAndOverflow(so, &overflow);
    Py_DECREF(so);
    if (size == -1 && PyErr_Occurred()) {
      Py_DECREF(seq);
      return nullptr;
    }
    if (overflow || size < 0 || size >= limit) {
      sz[i] = -1;
      continue;
    }
    sz[i] = static_cast<int32_t>(size / group_width);  // size group id (any size range)
    const int32_t slot = route[size / group_width];
    if (slot < 0 || slot >= S) {
      PyErr_SetString(PyExc_IndexError, "route entry out of range");
      Py_DECREF(seq);
      return nullptr;
    }
    PyObject* columns = PyList_GET_ITEM(colmaps, slot);
    PyObject* e = entries_of(s);
    if (!e) {
      Py_DECREF(seq);
      return nullptr;
    }
    // Walk the smaller of the two dicts: the model's k features looked up in
    // the histogram (the reference's own `hist.get(op)` per feature,
    // classifier.py:143-147) when k < nnz, else the histogram's entries looked
    // up in the column map.  Same counts either way.
    const bool by_feature = PyDict_GET_SIZE(columns) < PyDict_GET_SIZE(e);
    PyObject* walk = by_feature ? columns : e;
    PyObject* probe = by_feature ? e : columns;
    Py_ssize_t pos = 0;
    PyObject *k, *v;
    while (PyDict_Next(walk, &pos, &k, &v)) {
      PyObject* hit = PyDict_GetItemWithError(probe, k);
      if (!hit) {
        if (PyErr_Occurred()) {
          Py_DECREF(e);
          Py_DECREF(seq);
          return nullptr;
        }
        continue;
      }
      PyObject* col = by_feature ? v : hit;
      PyObject* cnt = by_feature ? hit : v;
      const Py_ssize_t j = PyLong_AsSsize_t(col);
      if (j < 0 || j >= width || !put_count(x + i * width, j, cnt)) {
        if (!PyErr_Occurred()) PyErr_SetString(PyExc_IndexError, "column out of range");
        Py_DECREF(e);
        Py_DECREF(seq);
        return nullptr;
      }
    }
    Py_DECREF(e);
  }
  Py_DECREF(seq);
  Py_RETURN_NONE;
}

// predictions(label int32 [N], logpost float64 [N, 2], eff int32 [N], Prediction,
//             classes (index -> Label), MALWARE, BENIGN) -> list
// The TimedRun.predictions of classify_* (engine.py:187-206): None where the
// row's label is negative (error rows), else Prediction(label,
// {MALWARE: lp[i,1], BENIGN: lp[i,0]}, eff[i]).  Instances are made like the
// frozen dataclass's own __init__ makes them (object.__setattr__ per field).
PyObject* s_f_label = nullptr;
PyObject* s_f_logpost = nullptr;
PyObject* s_f_group = nullptr;

PyObject* predictions(PyObject*, PyObject* args) {
  PyObject *lab_o, *lp_o, *eff_o, *type_o, *classes, *malware, *benign;
  if (!PyArg_ParseTuple(args, "OOOO!O!OO", &lab_o, &lp_o, &eff_o, &PyType_Type, &type_o,
                        &PyTuple_Type, &classes, &malware, &benign))
    return nullptr;
  Py_buffer bl{}, bp{}, be{};
  if (PyObject_GetBuffer(lab_o, &bl, PyBUF_C_CONTIGUOUS) != 0) return nullptr;
  const Py_ssize_t n = bl.len / 4;
  if (PyObject_GetBuffer(lp_o, &bp, PyBUF_C_CONTIGUOUS) != 0) {
    PyBuffer_Release(&bl);
    return nullptr;
  }
  if (PyObject_GetBuffer(eff_o, &be, PyBUF_C_CONTIGUOUS) != 0) {
    PyBuffer_Release(&bl);
    PyBuffer_Release(&bp);
    return nullptr;
  }
  PyObject* out = nullptr;
  PyTypeObject* tp = reinterpret_cast<PyTypeObject*>(type_o);
  PyObject* empty = PyTuple_New(0);
  const Py_ssize_t nc = PyTuple_GET_SIZE(classes);
  if (bl.itemsize != 4 || be.itemsize != 4 || bp.itemsize != 8 || bp.len < n * 16 ||
      be.len < n * 4 || !empty) {
    if (!PyErr_Occurred()) PyErr_SetString(PyExc_ValueError, "bad prediction buffers");
  } else {
    // no cyclic-GC passes while allocating ~2 containers per row (they cost
    // more than the construction itself); the previous state is restored
    // Label is an Enum: its __hash__ is Python code (~250 ns a call), so the
    // two class keys are hashed once here, not twice per Prediction
    const Py_hash_t h_malware = PyObject_Hash(malware), h_benign = PyObject_Hash(benign);
    const int gc_was_on = PyGC_Disable();
    out = (h_malware == -1 || h_benign == -1) ? nullptr : PyList_New(n);
    const int32_t* lab = static_cast<const int32_t*>(bl.buf);
    const double* lp = static_cast<const double*>(bp.buf);
    const int32_t* eff = static_cast<const int32_t*>(be.buf);
    for (Py_ssize_t i = 0; out && i < n; ++i) {
      if (lab[i] < 0 || lab[i] >= nc) {
        Py_INCREF(Py_None);
        PyList_SET_ITEM(out, i, Py_None);
        continue;
      }
      PyObject* obj = tp->tp_new(tp, empty, nullptr);
      PyObject* d = PyDict_New();
      PyObject* fm = PyFloat_FromDouble(lp[2 * i + 1]);
      PyObject* fb = PyFloat_FromDouble(lp[2 * i]);
      PyObject* g = PyLong_FromLong(eff[i]);
      bool ok = obj && d && fm && fb && g &&
                _PyDict_SetItem_KnownHash(d, malware, fm, h_malware) == 0 &&
                _PyDict_SetItem_KnownHash(d, benign, fb, h_benign) == 0 &&
                PyObject_GenericSetAttr(obj, s_f_label, PyTuple_GET_ITEM(classes, lab[i])) == 0 &&
                PyObject_GenericSetAttr(obj, s_f_logpost, d) == 0 &&
                PyObject_GenericSetAttr(obj, s_f_group, g) == 0;
      Py_XDECREF(d);
      Py_XDECREF(fm);
      Py_XDECREF(fb);
      Py_XDECREF(g);
      if (!ok) {
        Py_XDECREF(obj);
        Py_CLEAR(out);
        break;
      }
      PyList_SET_ITEM(out, i, obj);
    }
    if (gc_was_on) PyGC_Enable();
  }
  Py_XDECREF(empty);
  PyBuffer_Release(&bl);
  PyBuffer_Release(&bp);
  PyBuffer_Release(&be);
  return out;
}

// ------------------------------------------------------------------ sequential scoring (Tc)
// classifier.log_posterior (pkg/src/groupnb/classifier.py:132-148) over a
// model's `_packed` rows, exactly: score_c = log_prior[c]; for (op, ll_m,
// ll_b) in feature order: n = entries.get(op); if n is not None:
// score_m += n * ll_m; score_b += n * ll_b.  For an int count CPython computes
// `n * ll` as float(n) (correctly rounded; OverflowError past the double
// range) times ll, one rounding, then one rounding for the add -- the doubles
// below do the same (built without FMA contraction).  Anything else (a float
// count, a non-float parameter) switches to the generic number protocol, i.e.
// literally the reference's expressions.
PyObject* s_packed = nullptr;
PyObject* s_log_prior = nullptr;
PyObject* s_group = nullptr;

struct Score {
  PyObject* m = nullptr;  // new references
  PyObject* b = nullptr;
};

bool score_packed_impl(PyObject* packed, PyObject* prior_m, PyObject* prior_b, PyObject* entries,
                       Score* out) {
  if (!PyTuple_Check(packed) || !PyDict_Check(entries)) {
    PyErr_SetString(PyExc_TypeError, "_packed must be a tuple and entries a dict");
    return false;
  }
  const Py_ssize_t F = PyTuple_GET_SIZE(packed);
  bool fast = PyFloat_CheckExact(prior_m) && PyFloat_CheckExact(prior_b);
  double dm = fast ? PyFloat_AS_DOUBLE(prior_m) : 0.0, db = fast ? PyFloat_AS_DOUBLE(prior_b) : 0.0;
  PyObject* om = nullptr;  // generic accumulators (owned) once !fast
  PyObject* ob = nullptr;
  if (!fast) {
    Py_INCREF(prior_m);
    Py_INCREF(prior_b);
    om = prior_m;
    ob = prior_b;
  }
  for (Py_ssize_t j = 0; j < F; ++j) {
    PyObject* row = PyTuple_GET_ITEM(packed, j);
    if (!PyTuple_Check(row) || PyTuple_GET_SIZE(row) != 3) {
      PyErr_SetString(PyExc_TypeError, "_packed rows must be (op, ll_m, ll_b)");
      Py_XDECREF(om);
      Py_XDECREF(ob);
      return false;
    }
    PyObject* n = PyDict_GetItemWithError(entries, PyTuple_GET_ITEM(row, 0));
    if (!n) {
      if (PyErr_Occurred()) {
        Py_XDECREF(om);
        Py_XDECREF(ob);
        return false;
      }
      continue;
    }
    PyObject* lm = PyTuple_GET_ITEM(row, 1);
    PyObject* lb = PyTuple_GET_ITEM(row, 2);
    if (fast && PyLong_CheckExact(n) && PyFloat_CheckExact(lm) && PyFloat_CheckExact(lb)) {
      const double x = PyLong_AsDouble(n);
      if (x == -1.0 && PyErr_Occurred()) return false;
      const double pm = x * PyFloat_AS_DOUBLE(lm);
      const double pb = x * PyFloat_AS_DOUBLE(lb);
      dm = dm + pm;
      db = db + pb;
      continue;
    }
    if (fast) {  // switch to objects from here on
      fast = false;
      om = PyFloat_FromDouble(dm);
      ob = PyFloat_FromDouble(db);
      if (!om || !ob) {
        Py_XDECREF(om);
        Py_XDECREF(ob);
        return false;
      }
    }
    PyObject* tm = PyNumber_Multiply(n, lm);
    PyObject* nm = tm ? PyNumber_Add(om, tm) : nullptr;
    Py_XDECREF(tm);
    PyObject* tb = nm ? PyNumber_Multiply(n, lb) : nullptr;
    PyObject* nb = tb ? PyNumber_Add(ob, tb) : nullptr;
    Py_XDECREF(tb);
    Py_DECREF(om);
    Py_DECREF(ob);
    om = nm;
    ob = nb;
    if (!om || !ob) {
      Py_XDECREF(om);
      Py_XDECREF(ob);
      return false;
    }
  }
  if (fast) {
    out->m = PyFloat_FromDouble(dm);
    out->b = PyFloat_FromDouble(db);
    if (!out->m || !out->b) {
      Py_CLEAR(out->m);
      Py_CLEAR(out->b);
      return false;
    }
  } else {
    out->m = om;
    out->b = ob;
  }
  return true;
}

// score_packed(packed, prior_m, prior_b, entries) -> (score_m, score_b)
PyObject* score_packed(PyObject*, PyObject* args) {
  PyObject *packed, *pm, *pb, *entries;
  if (!PyArg_ParseTuple(args, "OOOO", &packed, &pm, &pb, &entries)) return nullptr;
  Score sc;
  if (!score_packed_impl(packed, pm, pb, entries, &sc)) return nullptr;
  return Py_BuildValue("(NN)", sc.m, sc.b);
}

struct ModelPrep {
  PyObject* packed;  // borrowed from the model (kept alive by `models`)
  PyObject* prior_m;
  PyObject* prior_b;
  PyObject* group;   // owned
};

// classify_slice(samples, route_table: tuple, models: dict, width, limit,
//                Prediction, malware, benign) -> (predictions list, error indices list)
// engine._classify_slice (pkg/src/groupnb/engine.py:187-206) on ONE thread --
// the Tc side of the reference's speedup ratio, "never parallelized
// internally" (engine.py:212-215): per sample the range check, the route
// table lookup, the log_posterior above and `malware iff strictly higher`
// (classifier.py:151-158); None + an error index outside [0, limit).
PyObject* classify_slice(PyObject*, PyObject* args) {
  PyObject *samples, *table, *models, *type_o, *malware, *benign;
  Py_ssize_t width;
  long long limit;
  if (!PyArg_ParseTuple(args, "OO!O!nLO!OO", &samples, &PyTuple_Type, &table, &PyDict_Type,
                        &models, &width, &limit, &PyType_Type, &type_o, &malware, &benign))
    return nullptr;
  if (width <= 0) {
    PyErr_SetString(PyExc_ValueError, "width must be positive");
    return nullptr;
  }
  PyObject* seq = PySequence_Fast(samples, "samples must be a sequence");
  if (!seq) return nullptr;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(seq);
  PyTypeObject* tp = reinterpret_cast<PyTypeObject*>(type_o);
  PyObject* out = PyList_New(n);
  PyObject* errs = PyList_New(0);
  PyObject* empty = PyTuple_New(0);
  std::vector<std::pair<PyObject*, ModelPrep>> cache;  // model -> prepared rows (few models)
  bool ok = out && errs && empty;
  for (Py_ssize_t i = 0; ok && i < n; ++i) {
    PyObject* s = PySequence_Fast_GET_ITEM(seq, i);
    PyObject* so = PyObject_GetAttr(s, s_size_bytes);
    if (!so) {
      ok = false;
      break;
    }
    if (!PyLong_Check(so)) {
      Py_DECREF(so);
      PyErr_SetString(PyExc_TypeError, "size_bytes must be an int");
      ok = false;
      break;
    }
    int overflow = 0;
    const long long size = PyLong_AsLongLongAndOverflow(so, &overflow);
    Py_DECREF(so);
    if (size == -1 && PyErr_Occurred()) {
      ok = false;
      break;
    }
    if (overflow || size < 0 || size >= limit) {
      Py_INCREF(Py_None);
      PyList_SET_ITEM(out, i, Py_None);
      PyObject* idx = PyLong_FromSsize_t(i);
      ok = idx && PyList_Append(errs, idx) == 0;
      Py_XDECREF(idx);
      continue;
    }
    const long long g = size / width;
    if (g >= PyTuple_GET_SIZE(table)) {
      PyErr_SetString(PyExc_IndexError, "tuple index out of range");
      ok = false;
      break;
    }
    PyObject* model = PyDict_GetItemWithError(models, PyTuple_GET_ITEM(table, g));
    if (!model) {
      if (!PyErr_Occurred()) PyErr_SetObject(PyExc_KeyError, PyTuple_GET_ITEM(table, g));
      ok = false;
      break;
    }
    const ModelPrep* mp = nullptr;
    for (auto& c : cache)
      if (c.first == model) mp = &c.second;
    if (!mp) {
      ModelPrep np{};
      PyObject* lp = PyObject_GetAttr(model, s_log_prior);
      np.packed = PyObject_GetAttr(model, s_packed);
      np.group = PyObject_GetAttr(model, s_group);
      np.prior_m = lp ? PyObject_GetItem(lp, malware) : nullptr;
      np.prior_b = np.prior_m ? PyObject_GetItem(lp, benign) : nullptr;
      Py_XDECREF(lp);
      if (!np.packed || !np.group || !np.prior_m || !np.prior_b) {
        Py_XDECREF(np.packed);
        Py_XDECREF(np.group);
        Py_XDECREF(np.prior_m);
        Py_XDECREF(np.prior_b);
        ok = false;
        break;
      }
      cache.emplace_back(model, np);
      mp = &cache.back().second;
    }
    PyObject* e = entries_of(s);
    if (!e) {
      ok = false;
      break;
    }
    Score sc;
    ok = score_packed_impl(mp->packed, mp->prior_m, mp->prior_b, e, &sc);
    Py_DECREF(e);
    if (!ok) break;
    const int gt = PyObject_RichCompareBool(sc.m, sc.b, Py_GT);
    PyObject* obj = gt < 0 ? nullptr : tp->tp_new(tp, empty, nullptr);
    PyObject* d = obj ? PyDict_New() : nullptr;
    ok = d && PyDict_SetItem(d, malware, sc.m) == 0 && PyDict_SetItem(d, benign, sc.b) == 0 &&
         PyObject_GenericSetAttr(obj, s_f_label, gt ? malware : benign) == 0 &&
         PyObject_GenericSetAttr(obj, s_f_logpost, d) == 0 &&
         PyObject_GenericSetAttr(obj, s_f_group, mp->group) == 0;
    Py_XDECREF(d);
    Py_DECREF(sc.m);
    Py_DECREF(sc.b);
    if (!ok) {
      Py_XDECREF(obj);
      break;
    }
    PyList_SET_ITEM(out, i, obj);
  }
  for (auto& c : cache) {
    Py_DECREF(c.second.packed);
    Py_DECREF(c.second.group);
    Py_DECREF(c.second.prior_m);
    Py_DECREF(c.second.prior_b);
  }
  Py_XDECREF(empty);
  Py_DECREF(seq);
  if (!ok) {
    Py_XDECREF(out);
    Py_XDECREF(errs);
    return nullptr;
  }
  return Py_BuildValue("(NN)", out, errs);
}

// discover_into(samples, columns: dict (grown), ops: list (grown), out int32 [N, width], width)
//   -> bool.  densify_into that also discovers the vocabulary: an opcode not
// yet in `columns` gets the next column (first-seen order, appended to `ops`).
// One walk of the histograms for the fit's union-of-opcodes + densify; False
// (out is then incomplete) when more than `width` distinct opcodes turn up.
PyObject* discover_into(PyObject*, PyObject* args) {
  PyObject *samples, *columns, *ops, *out;
  Py_ssize_t width;
  if (!PyArg_ParseTuple(args, "OO!O!On", &samples, &PyDict_Type, &columns, &PyList_Type, &ops,
                        &out, &width))
    return nullptr;
  PyObject* seq = PySequence_Fast(samples, "samples must be a sequence");
  if (!seq) return nullptr;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(seq);
  Buf b;
  if (!b.get(out, 4, n * width)) {
    Py_DECREF(seq);
    return nullptr;
  }
  int32_t* x = static_cast<int32_t*>(b.view.buf);
  for (Py_ssize_t i = 0; i < n; ++i) {
    PyObject* e = entries_of(PySequence_Fast_GET_ITEM(seq, i));
    if (!e) {
      Py_DECREF(seq);
      return nullptr;
    }
    Py_ssize_t pos = 0;
    PyObject *k, *v;
    while (PyDict_Next(e, &pos, &k, &v)) {
      PyObject* col = PyDict_GetItemWithError(columns, k);
      Py_ssize_t j;
      if (col) {
        j = PyLong_AsSsize_t(col);
      } else {
        if (PyErr_Occurred()) {
          Py_DECREF(e);
          Py_DECREF(seq);
          return nullptr;
        }
        j = PyList_GET_SIZE(ops);
        if (j >= width) {  // the caller retries with a wider buffer
          Py_DECREF(e);
          Py_DECREF(seq);
          Py_RETURN_FALSE;
        }
        PyObject* jo = PyLong_FromSsize_t(j);
        const bool ok = jo && PyDict_SetItem(columns, k, jo) == 0 && PyList_Append(ops, k) == 0;
        Py_XDECREF(jo);
        if (!ok) {
          Py_DECREF(e);
          Py_DECREF(seq);
          return nullptr;
        }
      }
      if (!put_count(x + i * width, j, v)) {
        Py_DECREF(e);
        Py_DECREF(seq);
        return nullptr;
      }
    }
    Py_DECREF(e);
  }
  Py_DECREF(seq);
  Py_RETURN_TRUE;
}

// permute_columns(src int32 [N, ws], order int64 [V], dst int32 [N, V]):
// dst[:, j] = src[:, order[j]] (numpy's column fancy-indexing is ~30 ns/element).
PyObject* permute_columns(PyObject*, PyObject* args) {
  PyObject *src_o, *order_o, *dst_o;
  Py_ssize_t ws;
  if (!PyArg_ParseTuple(args, "OnOO", &src_o, &ws, &order_o, &dst_o)) return nullptr;
  Py_buffer bs{}, bo{};
  if (PyObject_GetBuffer(src_o, &bs, PyBUF_C_CONTIGUOUS) != 0) return nullptr;
  if (PyObject_GetBuffer(order_o, &bo, PyBUF_C_CONTIGUOUS) != 0) {
    PyBuffer_Release(&bs);
    return nullptr;
  }
  Buf bd;
  const Py_ssize_t V = bo.len / 8, n = ws > 0 ? bs.len / 4 / ws : 0;
  PyObject* ret = nullptr;
  if (bs.itemsize == 4 && bo.itemsize == 8 && bd.get(dst_o, 4, n * V)) {
    const int32_t* src = static_cast<const int32_t*>(bs.buf);
    const int64_t* order = static_cast<const int64_t*>(bo.buf);
    int32_t* dst = static_cast<int32_t*>(bd.view.buf);
    bool ok = true;
    for (Py_ssize_t j = 0; j < V; ++j) ok = ok && order[j] >= 0 && order[j] < ws;
    if (!ok) {
      PyErr_SetString(PyExc_IndexError, "column order out of range");
    } else {
      Py_BEGIN_ALLOW_THREADS
      for (Py_ssize_t r = 0; r < n; ++r)
        for (Py_ssize_t j = 0; j < V; ++j) dst[r * V + j] = src[r * ws + order[j]];
      Py_END_ALLOW_THREADS
      Py_INCREF(Py_None);
      ret = Py_None;
    }
  } else if (!PyErr_Occurred()) {
    PyErr_SetString(PyExc_ValueError, "bad permute_columns buffers");
  }
  PyBuffer_Release(&bs);
  PyBuffer_Release(&bo);
  return ret;
}

// meta_into(samples, limit, malware, benign, sizes_out int32 [N], labels_out int32 [N])
// sizes outside [0, limit) -> -1; labels: malware 1, benign 0, anything else -1.
PyObject* meta_into(PyObject*, PyObject* args) {
  PyObject *samples, *malware, *benign, *sizes_o, *labels_o;
  Py_ssize_t limit;
  if (!PyArg_ParseTuple(args, "OnOOOO", &samples, &limit, &malware, &benign, &sizes_o, &labels_o))
    return nullptr;
  PyObject* seq = PySequence_Fast(samples, "samples must be a sequence");
  if (!seq) return nullptr;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(seq);
  Buf bs, bl;
  if (!bs.get(sizes_o, 4, n) || !bl.get(labels_o, 4, n)) {
    Py_DECREF(seq);
    return nullptr;
  }
  int32_t* sz = static_cast<int32_t*>(bs.view.buf);
  int32_t* lab = static_cast<int32_t*>(bl.view.buf);
  for (Py_ssize_t i = 0; i < n; ++i) {
    PyObject* s = PySequence_Fast_GET_ITEM(seq, i);
    PyObject* so = PyObject_GetAttr(s, s_size_bytes);
    PyObject* lo = so ? PyObject_GetAttr(s, s_label) : nullptr;
    if (!so || !lo) {
      Py_XDECREF(so);
      Py_DECREF(seq);
      return nullptr;
    }
    int overflow = 0;
    const long long size = PyLong_AsLongLongAndOverflow(so, &overflow);
    Py_DECREF(so);
    sz[i] = (!overflow && size >= 0 && size < limit) ? static_cast<int32_t>(size) : -1;
    lab[i] = lo == malware ? 1 : lo == benign ? 0 : -1;
    Py_DECREF(lo);
    if (size == -1 && PyErr_Occurred()) {
      Py_DECREF(seq);
      return nullptr;
    }
  }
  Py_DECREF(seq);
  Py_RETURN_NONE;
}

PyMethodDef kMethods[] = {
    {"densify_into", densify_into, METH_VARARGS,
     "densify_into(samples, columns, out, width): counts of `columns` per sample."},
    {"gather_into", gather_into, METH_VARARGS,
     "gather_into(samples, route, colmaps, width, group_width, limit, out, group_ids_out)."},
    {"vocab_dense", vocab_dense, METH_VARARGS,
     "vocab_dense(samples) -> (sorted opcodes, int32 bytearray [N, max(V, 1)]) or None."},
    {"densify_into_serial", densify_into_serial, METH_VARARGS,
     "densify_into on the calling thread only (the reference walk for tests)."},
    {"gather_into_serial", gather_into_serial, METH_VARARGS,
     "gather_into on the calling thread only (the reference walk for tests)."},
    {"meta_into", meta_into, METH_VARARGS,
     "meta_into(samples, limit, MALWARE, BENIGN, sizes_out, labels_out)."},
    {"discover_into", discover_into, METH_VARARGS,
     "discover_into(samples, columns, ops, out, width) -> bool (vocabulary fit in width)."},
    {"permute_columns", permute_columns, METH_VARARGS,
     "permute_columns(src, src_width, order, dst): dst[:, j] = src[:, order[j]]."},
    {"score_packed", score_packed, METH_VARARGS,
     "score_packed(model._packed, prior_m, prior_b, entries) -> (score_m, score_b)."},
    {"classify_slice", classify_slice, METH_VARARGS,
     "classify_slice(samples, route_table, models, width, limit, Prediction, malware, benign)"
     " -> (predictions, error_indices): engine._classify_slice on one thread."},
    {"predictions", predictions, METH_VARARGS,
     "predictions(label, logpost, eff, Prediction, classes, MALWARE, BENIGN) -> list."},
    {nullptr, nullptr, 0, nullptr}};

PyModuleDef kModule = {PyModuleDef_HEAD_INIT, "_adapt",
                       "SampleRecord -> dense arrays (ADAPT, C API).", -1, kMethods};

}  // namespace

PyMODINIT_FUNC PyInit__adapt(void) {
  s_histogram = PyUnicode_InternFromString("histogram");
  s_entries = PyUnicode_InternFromString("entries");
  s_size_bytes = PyUnicode_InternFromString("size_bytes");
  s_label = PyUnicode_InternFromString("label");
  s_f_label = s_label;
  s_f_logpost = PyUnicode_InternFromString("log_posterior");
  s_f_group = PyUnicode_InternFromString("effective_group");
  s_packed = PyUnicode_InternFromString("_packed");
  s_log_prior = PyUnicode_InternFromString("log_prior");
  s_group = PyUnicode_InternFromString("group");
  return PyModule_Create(&kModule);
}
