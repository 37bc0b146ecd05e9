/*
 * hostptr.c -- CPython extension _hostptr: the pointer table of a
 * ScatteredPatchSet (memory.py:60-96), i.e. the data addresses of T
 * independently allocated numpy arrays, in one C loop (a Python-level loop
 * costs ~1 us per array, ~1 s at 2^20 patches).
 *
 *   pointer_table(arrays, count, out, writable) -> None
 *     arrays:   sequence of float64 C-contiguous numpy arrays, each `count`
 *               elements (ShapeMismatchError semantics: ValueError naming
 *               the first offending index)
 *     out:      writable uint64 numpy array of len(arrays) entries
 *     writable: demand writable arrays (outputs)
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#define NPY_NO_DEPRECATED_API NPY_1_7_API_VERSION
#include <numpy/arrayobject.h>

#include <stdint.h>

static PyObject* pointer_table(PyObject* self, PyObject* args) {
    PyObject* seq;
    Py_ssize_t count;
    PyObject* out_obj;
    int writable;
    (void)self;
    if (!PyArg_ParseTuple(args, "OnOp", &seq, &count, &out_obj, &writable)) return NULL;
    if (!PyArray_Check(out_obj)) {
        PyErr_SetString(PyExc_TypeError, "out must be a numpy array");
        return NULL;
    }
    PyArrayObject* out = (PyArrayObject*)out_obj;
    PyObject* fast = PySequence_Fast(seq, "arrays must be a sequence");
    if (fast == NULL) return NULL;
    const Py_ssize_t n = PySequence_Fast_GET_SIZE(fast);
    if (PyArray_TYPE(out) != NPY_UINT64 || PyArray_NDIM(out) != 1 || PyArray_DIM(out, 0) != n ||
        !PyArray_ISCARRAY(out)) {
        Py_DECREF(fast);
        PyErr_SetString(PyExc_ValueError, "out must be a writable contiguous uint64 array of len(arrays)");
        return NULL;
    }
    uint64_t* dst = (uint64_t*)PyArray_DATA(out);
    PyObject** items = PySequence_Fast_ITEMS(fast);
    for (Py_ssize_t i = 0; i < n; ++i) {
        PyObject* o = items[i];
        if (!PyArray_Check(o)) {
            Py_DECREF(fast);
            PyErr_Format(PyExc_ValueError, "patch %zd is not a numpy array", i);
            return NULL;
        }
        PyArrayObject* a = (PyArrayObject*)o;
        if (PyArray_TYPE(a) != NPY_FLOAT64 || !PyArray_IS_C_CONTIGUOUS(a) || PyArray_SIZE(a) != count ||
            (writable && !PyArray_ISWRITEABLE(a)) || !PyArray_ISALIGNED(a)) {
            Py_DECREF(fast);
            PyErr_Format(PyExc_ValueError,
                         "patch %zd: expected an aligned C-contiguous float64 array of %zd entries%s", i, count,
                         writable ? " (writable)" : "");
            return NULL;
        }
        dst[i] = (uint64_t)(uintptr_t)PyArray_DATA(a);
    }
    Py_DECREF(fast);
    Py_RETURN_NONE;
}

static PyMethodDef methods[] = {
    {"pointer_table", pointer_table, METH_VARARGS, "data addresses of a sequence of float64 arrays"},
    {NULL, NULL, 0, NULL},
};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_hostptr", NULL, -1, methods};

PyMODINIT_FUNC PyInit__hostptr(void) {
    import_array();
    return PyModule_Create(&module);
}
