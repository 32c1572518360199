/* bdk_pyhost.c -- a CPython fast path for the host decode entry point.
 *
 * bitkv.decode_step with host float32 arrays calls bdk_decode_step_host
 * (include/bitdecode_b200.h) once per step.  Through ctypes the Python side
 * of that call (four buffer addresses, argument conversion) costs ~7 us, the
 * same order as the GPU work of a short step; here the buffers are taken with
 * the buffer protocol and the C-ABI function (its address comes from the
 * ctypes-loaded library, so this module links against nothing) is called
 * with the GIL released.
 *
 * step(fn, cache, cfg, q, k, v, out, nq, nkv) -> status, or -1000 when a
 * buffer is not a C-contiguous float32 of the expected element count (the
 * caller then takes its general path, which converts or raises).
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <string.h>

typedef int (*step_fn)(void*, const void*, const float*, const float*, const float*, float*);

static int take(PyObject* o, Py_buffer* b, Py_ssize_t n, int writable) {
  if (PyObject_GetBuffer(o, b, PyBUF_C_CONTIGUOUS | PyBUF_FORMAT | (writable ? PyBUF_WRITABLE : 0)) != 0) {
    PyErr_Clear();
    return 0;
  }
  if (b->itemsize != 4 || b->len != n * 4 || b->format == NULL || strcmp(b->format, "f") != 0) {
    PyBuffer_Release(b);
    return 0;
  }
  return 1;
}

static PyObject* step(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  if (nargs != 9) {
    PyErr_SetString(PyExc_TypeError, "step(fn, cache, cfg, q, k, v, out, nq, nkv)");
    return NULL;
  }
  step_fn fn = (step_fn)PyLong_AsVoidPtr(args[0]);
  void* cache = PyLong_AsVoidPtr(args[1]);
  const void* cfg = PyLong_AsVoidPtr(args[2]);
  const Py_ssize_t nq = PyLong_AsSsize_t(args[7]), nkv = PyLong_AsSsize_t(args[8]);
  if (PyErr_Occurred()) return NULL;
  Py_buffer bq, bk, bv, bo;
  if (!take(args[3], &bq, nq, 0)) return PyLong_FromLong(-1000);
  if (!take(args[4], &bk, nkv, 0)) {
    PyBuffer_Release(&bq);
    return PyLong_FromLong(-1000);
  }
  if (!take(args[5], &bv, nkv, 0)) {
    PyBuffer_Release(&bq);
    PyBuffer_Release(&bk);
    return PyLong_FromLong(-1000);
  }
  if (!take(args[6], &bo, nq, 1)) {
    PyBuffer_Release(&bq);
    PyBuffer_Release(&bk);
    PyBuffer_Release(&bv);
    return PyLong_FromLong(-1000);
  }
  int st;
  Py_BEGIN_ALLOW_THREADS
  st = fn(cache, cfg, (const float*)bq.buf, (const float*)bk.buf, (const float*)bv.buf, (float*)bo.buf);
  Py_END_ALLOW_THREADS
  PyBuffer_Release(&bq);
  PyBuffer_Release(&bk);
  PyBuffer_Release(&bv);
  PyBuffer_Release(&bo);
  return PyLong_FromLong(st);
}

static PyMethodDef methods[] = {
    {"step", (PyCFunction)(void (*)(void))step, METH_FASTCALL, "host decode step (see module doc)"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef mod = {PyModuleDef_HEAD_INIT, "_bdk_pyhost",
                                 "CPython fast path for bdk_decode_step_host", -1, methods};

PyMODINIT_FUNC PyInit__bdk_pyhost(void) { return PyModule_Create(&mod); }
