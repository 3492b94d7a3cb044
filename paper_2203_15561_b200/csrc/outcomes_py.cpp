// outcomes_py.cpp -- CPython extension `_outcomes`: builds the drop-in API's
// result objects (window.py's AlignmentResult / AccessCounters / BatchOutcome,
// the reference's pkg/src/bitalign/window.py:73-82 and :132-141) for every
// aligned pair of a batch in one call, straight from the C-ABI output arrays.
//
// It is what window.outcomes_from_packed does per pair in Python -- create the
// frozen instances without running __init__ and fill their __dict__ -- minus
// the interpreter loop: each CIGAR is one PyUnicode_New + memcpy from the op
// bytes, each window-distance tuple is built from the small-int cache.  Host
// object construction only; no alignment work happens here.
#define PY_SSIZE_T_CLEAN
#include <Python.h>

#include <cstdint>
#include <cstring>

namespace {

PyObject* new_instance(PyTypeObject* cls) {
    return cls->tp_alloc(cls, 0);  // object.__new__(cls): no __init__, no __setattr__
}

// obj.__dict__[key] = value (steals value)
bool put(PyObject* obj, PyObject* key, PyObject* value) {
    if (!value) return false;
    PyObject* d = PyObject_GenericGetDict(obj, nullptr);
    if (!d) {
        Py_DECREF(value);
        return false;
    }
    const int rc = PyDict_SetItem(d, key, value);
    Py_DECREF(d);
    Py_DECREF(value);
    return rc == 0;
}

template <class T>
const T* ptr(unsigned long long a) {
    return reinterpret_cast<const T*>(static_cast<uintptr_t>(a));
}

// build(result_cls, counters_cls, outcome_cls, n, status, cost, text_consumed,
//       rows_computed, entry_reads, entry_writes, words_allocated, ops_len,
//       ops_off, win_off, n_windows, ops, dists) -> list
// Array arguments are addresses (numpy .ctypes.data): status int32, the
// counters and offsets int64, ops / dists uint8.  Slot q is a BatchOutcome for
// status 0, None otherwise (the caller fills the error slots).
PyObject* build(PyObject*, PyObject* args) {
    PyObject *rcls, *ccls, *bcls;
    Py_ssize_t n;
    unsigned long long a_status, a_cost, a_tcons, a_rows, a_reads, a_writes, a_words, a_olen, a_ooff,
        a_woff, a_nwin, a_ops, a_dists;
    if (!PyArg_ParseTuple(args, "OOOnKKKKKKKKKKKKK", &rcls, &ccls, &bcls, &n, &a_status, &a_cost,
                          &a_tcons, &a_rows, &a_reads, &a_writes, &a_words, &a_olen, &a_ooff,
                          &a_woff, &a_nwin, &a_ops, &a_dists))
        return nullptr;
    if (!PyType_Check(rcls) || !PyType_Check(ccls) || !PyType_Check(bcls)) {
        PyErr_SetString(PyExc_TypeError, "build: the first three arguments must be classes");
        return nullptr;
    }
    auto* rt = reinterpret_cast<PyTypeObject*>(rcls);
    auto* ct = reinterpret_cast<PyTypeObject*>(ccls);
    auto* bt = reinterpret_cast<PyTypeObject*>(bcls);
    const int32_t* status = ptr<int32_t>(a_status);
    const int64_t *cost = ptr<int64_t>(a_cost), *tcons = ptr<int64_t>(a_tcons),
                  *rows = ptr<int64_t>(a_rows), *reads = ptr<int64_t>(a_reads),
                  *writes = ptr<int64_t>(a_writes), *words = ptr<int64_t>(a_words),
                  *olen = ptr<int64_t>(a_olen), *ooff = ptr<int64_t>(a_ooff),
                  *woff = ptr<int64_t>(a_woff), *nwin = ptr<int64_t>(a_nwin);
    const uint8_t *ops = ptr<uint8_t>(a_ops), *dists = ptr<uint8_t>(a_dists);

    static const char* kNames[] = {"entry_reads", "entry_writes", "words_allocated", "cigar",
                                   "cost", "text_consumed", "window_distances", "counters",
                                   "rows_computed", "result", "error"};
    PyObject* key[11];
    for (int i = 0; i < 11; ++i) {
        key[i] = PyUnicode_InternFromString(kNames[i]);
        if (!key[i]) {
            for (int k = 0; k < i; ++k) Py_DECREF(key[k]);
            return nullptr;
        }
    }
    PyObject* out = PyList_New(n);
    bool ok = out != nullptr;
    for (Py_ssize_t q = 0; ok && q < n; ++q) {
        if (status[q] != 0) {
            Py_INCREF(Py_None);
            PyList_SET_ITEM(out, q, Py_None);
            continue;
        }
        PyObject* c = new_instance(ct);
        PyObject* r = c ? new_instance(rt) : nullptr;
        PyObject* b = r ? new_instance(bt) : nullptr;
        ok = b != nullptr;
        if (ok) {
            ok = put(c, key[0], PyLong_FromLongLong(reads[q])) &&
                 put(c, key[1], PyLong_FromLongLong(writes[q])) &&
                 put(c, key[2], PyLong_FromLongLong(words[q]));
        }
        if (ok) {
            PyObject* s = PyUnicode_New((Py_ssize_t)olen[q], 127);
            if (s) memcpy(PyUnicode_DATA(s), ops + ooff[q], (size_t)olen[q]);
            ok = put(r, key[3], s);
        }
        if (ok) {
            PyObject* t = PyTuple_New((Py_ssize_t)nwin[q]);
            for (int64_t w = 0; t && w < nwin[q]; ++w) {
                PyObject* v = PyLong_FromLong(dists[woff[q] + w]);
                if (!v) {
                    Py_CLEAR(t);
                    break;
                }
                PyTuple_SET_ITEM(t, (Py_ssize_t)w, v);
            }
            // the dataclass's field order: cigar, cost, text_consumed, window_distances
            ok = put(r, key[4], PyLong_FromLongLong(cost[q])) &&
                 put(r, key[5], PyLong_FromLongLong(tcons[q]));
            if (ok) ok = put(r, key[6], t);
            else Py_XDECREF(t);
        }
        if (ok) {
            Py_INCREF(c);
            ok = put(r, key[7], c) && put(r, key[8], PyLong_FromLongLong(rows[q]));
        }
        if (ok) {
            Py_INCREF(r);
            Py_INCREF(Py_None);
            ok = put(b, key[9], r) && put(b, key[10], Py_None);
        }
        Py_XDECREF(c);
        Py_XDECREF(r);
        if (ok) {
            PyList_SET_ITEM(out, q, b);
        } else {
            Py_XDECREF(b);
        }
    }
    for (int i = 0; i < 11; ++i) Py_DECREF(key[i]);
    if (!ok) {
        Py_XDECREF(out);
        if (!PyErr_Occurred()) PyErr_NoMemory();
        return nullptr;
    }
    return out;
}

PyMethodDef kMethods[] = {
    {"build", build, METH_VARARGS,
     "build(result_cls, counters_cls, outcome_cls, n, *array_addresses) -> list"},
    {nullptr, nullptr, 0, nullptr}};

PyModuleDef kModule = {PyModuleDef_HEAD_INIT, "_outcomes",
                       "Bulk construction of the drop-in API's result objects.", -1, kMethods,
                       nullptr, nullptr, nullptr, nullptr};

}  // namespace

PyMODINIT_FUNC PyInit__outcomes(void) { return PyModule_Create(&kModule); }
