/* drs_host.c -- the per-call host path of the samplers as a CPython extension
 * (module paper_2604_01356_b200._drshost).
 *
 * dac_sampler / ccf_sampler (samplers.py:255-266) cost ~40 us end to end at
 * config 3, of which the kernel is ~11.5 us and the 512 KB of indices over
 * the host link ~10 us; the rest is host time.  ctypes converts the 15
 * arguments of dr_sample_dac through their argtypes on every call (~2 us);
 * here they arrive as a vectorcall (METH_FASTCALL) and go straight to the C
 * ABI of libdrs.so, and the stream synchronisation of a host result runs in
 * the same call with the GIL released.  The entry points are bound once from
 * the addresses of the library ctypes already loaded (no second dlopen, so
 * exactly one copy of libdrs.so and its state exists in the process).
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>

typedef int (*sample_dac_fn)(const double*, const double*, int64_t, uint64_t, uint64_t, uint64_t, uint64_t*,
                             int64_t, double*, int64_t*, int32_t*, int32_t, void*, size_t, void*);
typedef int (*sample_ccf_fn)(const double*, const double*, int64_t, uint64_t, uint64_t, uint64_t, uint64_t*,
                             int64_t, double*, int64_t*, int32_t*, void*, size_t, void*);
typedef int (*sync_fn)(void*);

static sample_dac_fn p_dac = NULL;
static sample_dac_fn p_dac_sync = NULL;
static sample_ccf_fn p_ccf = NULL;
static sync_fn p_sync = NULL;

/* bind(addr_dr_sample_dac, addr_dr_sample_dac_sync, addr_dr_sample_ccf, addr_dr_stream_synchronize) */
static PyObject* drs_bind(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  if (nargs != 4) {
    PyErr_SetString(PyExc_TypeError, "bind() takes 4 addresses");
    return NULL;
  }
  void* a[4];
  for (int i = 0; i < 4; ++i) {
    a[i] = PyLong_AsVoidPtr(args[i]);
    if (!a[i]) {
      if (!PyErr_Occurred()) PyErr_SetString(PyExc_ValueError, "null entry point");
      return NULL;
    }
  }
  p_dac = (sample_dac_fn)a[0];
  p_dac_sync = (sample_dac_fn)a[1];
  p_ccf = (sample_ccf_fn)a[2];
  p_sync = (sync_fn)a[3];
  Py_RETURN_NONE;
}

/* sorted_sample(kind, W, idx, M, k0, k1, offset, n, U, out, status, mode, ws, ws_bytes, stream, sync) -> rc
 * kind 0: dr_sample_dac (mode), 1: dr_sample_ccf; sync != 0: wait for the stream (the result is host
 * memory the kernel wrote) with the GIL released -- dr_sample_dac_sync for kind 0, else
 * dr_stream_synchronize after a successful launch. */
static PyObject* drs_sorted_sample(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  if (nargs != 16) {
    PyErr_SetString(PyExc_TypeError, "sorted_sample() takes 16 arguments");
    return NULL;
  }
  if (!p_dac || !p_dac_sync || !p_ccf || !p_sync) {
    PyErr_SetString(PyExc_RuntimeError, "_drshost.bind() was not called");
    return NULL;
  }
  const long kind = PyLong_AsLong(args[0]);
  void* W = PyLong_AsVoidPtr(args[1]);
  void* idx = PyLong_AsVoidPtr(args[2]);
  const long long M = PyLong_AsLongLong(args[3]);
  const unsigned long long k0 = PyLong_AsUnsignedLongLong(args[4]);
  const unsigned long long k1 = PyLong_AsUnsignedLongLong(args[5]);
  const unsigned long long off = PyLong_AsUnsignedLongLong(args[6]);
  const long long n = PyLong_AsLongLong(args[7]);
  void* U = PyLong_AsVoidPtr(args[8]);
  void* out = PyLong_AsVoidPtr(args[9]);
  void* status = PyLong_AsVoidPtr(args[10]);
  const long mode = PyLong_AsLong(args[11]);
  void* ws = PyLong_AsVoidPtr(args[12]);
  const size_t wsb = PyLong_AsSize_t(args[13]);
  void* stream = PyLong_AsVoidPtr(args[14]);
  const long sync = PyLong_AsLong(args[15]);
  if (PyErr_Occurred()) return NULL;
  int rc;
  if (kind == 0 && sync) {  /* launch + wait in the library (its host-result launch path) */
    Py_BEGIN_ALLOW_THREADS
    rc = p_dac_sync((const double*)W, (const double*)idx, (int64_t)M, k0, k1, off, NULL, (int64_t)n, (double*)U,
                    (int64_t*)out, (int32_t*)status, (int32_t)mode, ws, wsb, stream);
    Py_END_ALLOW_THREADS
    return PyLong_FromLong(rc);
  }
  if (kind == 0)
    rc = p_dac((const double*)W, (const double*)idx, (int64_t)M, k0, k1, off, NULL, (int64_t)n, (double*)U,
               (int64_t*)out, (int32_t*)status, (int32_t)mode, ws, wsb, stream);
  else
    rc = p_ccf((const double*)W, (const double*)idx, (int64_t)M, k0, k1, off, NULL, (int64_t)n, (double*)U,
               (int64_t*)out, (int32_t*)status, ws, wsb, stream);
  if (rc == 0 && sync) {
    Py_BEGIN_ALLOW_THREADS
    rc = p_sync(stream);
    Py_END_ALLOW_THREADS
  }
  return PyLong_FromLong(rc);
}

static PyMethodDef methods[] = {
    {"bind", (PyCFunction)(void (*)(void))drs_bind, METH_FASTCALL, "bind the libdrs.so entry points"},
    {"sorted_sample", (PyCFunction)(void (*)(void))drs_sorted_sample, METH_FASTCALL,
     "dr_sample_dac / dr_sample_ccf (+ stream synchronisation) in one call"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_drshost", NULL, -1, methods};

PyMODINIT_FUNC PyInit__drshost(void) { return PyModule_Create(&module); }
