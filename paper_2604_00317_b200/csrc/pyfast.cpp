// Python fast path for the per-call data-path entry point (comm.py).
//
// ctypes costs ~4 us per nimbleAlltoAllv call (four count lists converted
// element by element, argument marshalling), about as much as the C call
// itself -- for small exchanges that is the difference between a host-bound
// and a device-bound call rate.  This module converts the count sequences on
// the stack and calls nimbleAlltoAllv through the function pointer comm.py
// hands it from the ctypes-loaded library, so both always bind the same
// libnimble_b200.so.  It returns the nimbleResult_t; comm.py raises on errors.
#define PY_SSIZE_T_CLEAN
#include <Python.h>

#include <cstddef>
#include <cstdint>

namespace {

constexpr Py_ssize_t kMaxRanks = 32;
using AlltoAllvFn = int (*)(const void*, const size_t*, const size_t*, void*, const size_t*, const size_t*, int,
                            void*, void*);
AlltoAllvFn g_alltoallv = nullptr;

// init(address of nimbleAlltoAllv)
PyObject* init(PyObject*, PyObject* arg) {
    const unsigned long long p = PyLong_AsUnsignedLongLong(arg);
    if (PyErr_Occurred()) return nullptr;
    g_alltoallv = reinterpret_cast<AlltoAllvFn>(static_cast<uintptr_t>(p));
    Py_RETURN_NONE;
}

bool to_sizes(PyObject* seq, Py_ssize_t n, size_t* out) {
    PyObject* fast = PySequence_Fast(seq, "counts / displacements must be a sequence");
    if (!fast) return false;
    const bool ok_len = PySequence_Fast_GET_SIZE(fast) == n;
    if (ok_len) {
        PyObject** items = PySequence_Fast_ITEMS(fast);
        for (Py_ssize_t i = 0; i < n; ++i) {
            out[i] = static_cast<size_t>(PyLong_AsUnsignedLongLong(items[i]));
            if (PyErr_Occurred()) {
                Py_DECREF(fast);
                return false;
            }
        }
    } else {
        PyErr_SetString(PyExc_ValueError, "counts / displacements: one entry per rank");
    }
    Py_DECREF(fast);
    return ok_len;
}

// alltoallv(comm, sendptr, sendcounts, sdispls, recvptr, recvcounts, rdispls, dtype, stream) -> int
PyObject* alltoallv(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
    if (nargs != 9) {
        PyErr_SetString(PyExc_TypeError, "alltoallv takes 9 arguments");
        return nullptr;
    }
    if (!g_alltoallv) {
        PyErr_SetString(PyExc_RuntimeError, "_fast.init() was not called");
        return nullptr;
    }
    const Py_ssize_t n = PySequence_Size(args[2]);
    if (n < 0) return nullptr;
    if (n > kMaxRanks) {
        PyErr_SetString(PyExc_ValueError, "more than 32 ranks");
        return nullptr;
    }
    size_t sc[kMaxRanks], sd[kMaxRanks], rc[kMaxRanks], rd[kMaxRanks];
    if (!to_sizes(args[2], n, sc) || !to_sizes(args[3], n, sd) || !to_sizes(args[5], n, rc) ||
        !to_sizes(args[6], n, rd))
        return nullptr;
    const unsigned long long comm = PyLong_AsUnsignedLongLong(args[0]);
    const unsigned long long sp = PyLong_AsUnsignedLongLong(args[1]);
    const unsigned long long rp = PyLong_AsUnsignedLongLong(args[4]);
    const long dtype = PyLong_AsLong(args[7]);
    const unsigned long long st = PyLong_AsUnsignedLongLong(args[8]);
    if (PyErr_Occurred()) return nullptr;
    int rcode;
    Py_BEGIN_ALLOW_THREADS
    rcode = g_alltoallv(reinterpret_cast<const void*>(sp), sc, sd, reinterpret_cast<void*>(rp), rc, rd,
                        static_cast<int>(dtype), reinterpret_cast<void*>(comm), reinterpret_cast<void*>(st));
    Py_END_ALLOW_THREADS
    return PyLong_FromLong(rcode);
}

PyMethodDef methods[] = {
    {"init", init, METH_O, "init(address of nimbleAlltoAllv)"},
    {"alltoallv", reinterpret_cast<PyCFunction>(reinterpret_cast<void (*)()>(alltoallv)), METH_FASTCALL,
     "alltoallv(comm, sendptr, sendcounts, sdispls, recvptr, recvcounts, rdispls, dtype, stream) -> result code"},
    {nullptr, nullptr, 0, nullptr},
};

PyModuleDef module = {PyModuleDef_HEAD_INIT, "_fast", "nimbleAlltoAllv fast call for comm.py", -1, methods,
                      nullptr, nullptr, nullptr, nullptr};

}  // namespace

PyMODINIT_FUNC PyInit__fast(void) { return PyModule_Create(&module); }
