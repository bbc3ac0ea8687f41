/* sjb_pack.c -- host-side token packing for the device embedding kernels
 * (subword model, synthetic-model hashing): a Python sequence of str ->
 * (UTF-8 bytes of all tokens back to back + a trailing NUL, int64 offsets
 * [n + 1]) in one pass over the sequence.  For compact ASCII strings
 * PyUnicode_AsUTF8AndSize returns CPython's own buffer, so a token costs one
 * memcpy.  Replaces device.pack_tokens' pure-Python path (~10 ms per 200k
 * tokens on the GPU box host). */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>
#include <string.h>

static PyObject* pack(PyObject* self, PyObject* arg) {
  (void)self;
  PyObject* fast = PySequence_Fast(arg, "tokens must be a sequence of str");
  if (!fast) return NULL;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(fast);
  PyObject** items = PySequence_Fast_ITEMS(fast);
  PyObject* offs = PyBytes_FromStringAndSize(NULL, (n + 1) * (Py_ssize_t)sizeof(int64_t));
  size_t cap = (size_t)n * 16 + 64, pos = 0;
  char* buf = (char*)PyMem_RawMalloc(cap);
  if (!offs || !buf) {
    Py_XDECREF(offs);
    PyMem_RawFree(buf);
    Py_DECREF(fast);
    return PyErr_NoMemory();
  }
  int64_t* o = (int64_t*)PyBytes_AS_STRING(offs);
  o[0] = 0;
  /* one pass: each string object is touched once (they are scattered in the
     heap; a second pass doubled the cache misses) */
  for (Py_ssize_t i = 0; i < n; i++) {
    /* the string objects are scattered over the heap: fetch a few ahead so
       their cache misses overlap (a compact ASCII str keeps its bytes right
       after the 40-byte header, in the same or the next line) */
    if (i + 16 < n) {
      __builtin_prefetch(items[i + 16]);
      __builtin_prefetch((const char*)items[i + 16] + 64);
    }
    if (!PyUnicode_Check(items[i])) {
      PyErr_Format(PyExc_TypeError, "token %zd is not a str", i);
      goto fail;
    }
    Py_ssize_t len = 0;
    const char* s;
    if (PyUnicode_IS_COMPACT_ASCII(items[i])) {   /* the bytes are the object's own */
      len = PyUnicode_GET_LENGTH(items[i]);
      s = (const char*)PyUnicode_DATA(items[i]);
    } else {
      s = PyUnicode_AsUTF8AndSize(items[i], &len);
      if (!s) goto fail;
    }
    if (pos + (size_t)len + 1 > cap) {
      while (pos + (size_t)len + 1 > cap) cap *= 2;
      char* nb = (char*)PyMem_RawRealloc(buf, cap);
      if (!nb) {
        PyErr_NoMemory();
        goto fail;
      }
      buf = nb;
    }
    memcpy(buf + pos, s, (size_t)len);
    pos += (size_t)len;
    o[i + 1] = (int64_t)pos;
  }
  buf[pos] = 0;
  {
    PyObject* data = PyBytes_FromStringAndSize(buf, (Py_ssize_t)pos + 1);
    PyMem_RawFree(buf);
    Py_DECREF(fast);
    if (!data) {
      Py_DECREF(offs);
      return NULL;
    }
    return Py_BuildValue("NN", data, offs);
  }
fail:
  PyMem_RawFree(buf);
  Py_DECREF(offs);
  Py_DECREF(fast);
  return NULL;
}

/* lookup(index, tokens) -> int64 bytearray (writable, so numpy/torch views
 * of it are too): index[token] for every token, -1
 * where absent (LookupModel.indices: the reference's per-token table probe,
 * embedding.py:143-152, as one C loop -- str objects cache their hash, so a
 * probe is a table read; the next tokens' objects are prefetched). */
static PyObject* lookup(PyObject* self, PyObject* args) {
  (void)self;
  PyObject *index, *seq;
  if (!PyArg_ParseTuple(args, "O!O", &PyDict_Type, &index, &seq)) return NULL;
  PyObject* fast = PySequence_Fast(seq, "tokens must be a sequence of str");
  if (!fast) return NULL;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(fast);
  PyObject** items = PySequence_Fast_ITEMS(fast);
  PyObject* out = PyByteArray_FromStringAndSize(NULL, n * (Py_ssize_t)sizeof(int64_t));
  if (!out) {
    Py_DECREF(fast);
    return NULL;
  }
  int64_t* o = (int64_t*)PyByteArray_AS_STRING(out);
  for (Py_ssize_t i = 0; i < n; i++) {
    if (i + 8 < n) __builtin_prefetch(items[i + 8]);
    PyObject* v = PyDict_GetItemWithError(index, items[i]);   /* borrowed */
    if (v == NULL) {
      if (PyErr_Occurred()) goto fail;
      o[i] = -1;
      continue;
    }
    const long long x = PyLong_AsLongLong(v);
    if (x == -1 && PyErr_Occurred()) goto fail;
    o[i] = (int64_t)x;
  }
  Py_DECREF(fast);
  return out;
fail:
  Py_DECREF(out);
  Py_DECREF(fast);
  return NULL;
}

static PyMethodDef methods[] = {
    {"pack", pack, METH_O, "pack(tokens) -> (utf8 bytes + NUL, int64 offsets bytes)"},
    {"lookup", lookup, METH_VARARGS, "lookup(index dict, tokens) -> int64 bytearray (-1: absent)"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_sjbpack", NULL, -1, methods};

PyMODINIT_FUNC PyInit__sjbpack(void) { return PyModule_Create(&module); }
