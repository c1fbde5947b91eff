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

#include <cstdint>
#include <cstring>

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
PyObject* densify_into(PyObject*, PyObject* args) {
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

// gather_into(samples, route: int32 buffer [G], colmaps: list[dict], width, limit,
//             out: int32 [N, width], sizes_out: int32 [N])
// Row i gets the counts of its routed model's features (FeatureSet order);
// sizes outside [0, limit) become -1 and leave the row zero.
PyObject* gather_into(PyObject*, PyObject* args) {
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
    sz[i] = static_cast<int32_t>(size);
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
     "gather_into(samples, route, colmaps, width, group_width, limit, out, sizes_out)."},
    {"meta_into", meta_into, METH_VARARGS,
     "meta_into(samples, limit, MALWARE, BENIGN, sizes_out, labels_out)."},
    {nullptr, nullptr, 0, nullptr}};

PyModuleDef kModule = {PyModuleDef_HEAD_INIT, "_adapt",
                       "SampleRecord -> dense arrays (ADAPT, C API).", -1, kMethods};

}  // namespace

PyMODINIT_FUNC PyInit__adapt(void) {
  s_histogram = PyUnicode_InternFromString("histogram");
  s_entries = PyUnicode_InternFromString("entries");
  s_size_bytes = PyUnicode_InternFromString("size_bytes");
  s_label = PyUnicode_InternFromString("label");
  return PyModule_Create(&kModule);
}
