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

/* ---- multithreaded token -> row lookup (LookupModel.indices).  A C hash
 * table of the model's vocabulary (FNV-1a-64 of the UTF-8 bytes, linear
 * probing, the bytes copied into one arena) is built once per model; the
 * probes then run on several threads without the GIL.  Compact-ASCII str
 * objects expose their bytes directly (immutable, kept alive by the caller's
 * list); other tokens are left at -2 and resolved by the caller's dict. */
#include <pthread.h>
#include <stdlib.h>

typedef struct {
  uint64_t* hash;      /* 0 = empty slot */
  int64_t* row;
  uint64_t* off;       /* token bytes at arena + off, length len */
  uint32_t* len;
  char* arena;
  uint64_t mask;
} VocabIndex;

static uint64_t fnv1a(const char* s, size_t n) {
  uint64_t h = 1469598103934665603ull;
  for (size_t i = 0; i < n; i++) h = (h ^ (unsigned char)s[i]) * 1099511628211ull;
  return h | 1ull;   /* never 0 (0 marks an empty slot) */
}

static void vocab_free(PyObject* cap) {
  VocabIndex* v = (VocabIndex*)PyCapsule_GetPointer(cap, "sjb.vocab");
  if (!v) return;
  free(v->hash);
  free(v->row);
  free(v->off);
  free(v->len);
  free(v->arena);
  free(v);
}

/* build_index(dict token -> row) -> capsule */
static PyObject* build_index(PyObject* self, PyObject* arg) {
  (void)self;
  if (!PyDict_Check(arg)) {
    PyErr_SetString(PyExc_TypeError, "build_index wants a dict");
    return NULL;
  }
  const Py_ssize_t n = PyDict_Size(arg);
  uint64_t cap = 16;
  while (cap < (uint64_t)(2 * n + 16)) cap <<= 1;
  VocabIndex* v = (VocabIndex*)calloc(1, sizeof(VocabIndex));
  size_t acap = (size_t)n * 16 + 64, apos = 0;
  if (v) {
    v->hash = (uint64_t*)calloc(cap, 8);
    v->row = (int64_t*)malloc(cap * 8);
    v->off = (uint64_t*)malloc(cap * 8);
    v->len = (uint32_t*)malloc(cap * 4);
    v->arena = (char*)malloc(acap);
    v->mask = cap - 1;
  }
  if (!v || !v->hash || !v->row || !v->off || !v->len || !v->arena) goto nomem;
  {
    Py_ssize_t pos = 0;
    PyObject *k, *val;
    while (PyDict_Next(arg, &pos, &k, &val)) {
      Py_ssize_t len = 0;
      const char* b = PyUnicode_Check(k) ? PyUnicode_AsUTF8AndSize(k, &len) : NULL;
      if (!b) {
        if (!PyErr_Occurred()) PyErr_SetString(PyExc_TypeError, "vocabulary keys must be str");
        goto fail;
      }
      const long long r = PyLong_AsLongLong(val);
      if (r == -1 && PyErr_Occurred()) goto fail;
      if (apos + (size_t)len > acap) {
        while (apos + (size_t)len > acap) acap *= 2;
        char* na = (char*)realloc(v->arena, acap);
        if (!na) goto nomem;
        v->arena = na;
      }
      memcpy(v->arena + apos, b, (size_t)len);
      const uint64_t h = fnv1a(b, (size_t)len);
      uint64_t i = h & v->mask;
      while (v->hash[i]) i = (i + 1) & v->mask;   /* dict keys are distinct */
      v->hash[i] = h;
      v->row[i] = (int64_t)r;
      v->off[i] = apos;
      v->len[i] = (uint32_t)len;
      apos += (size_t)len;
    }
  }
  {
    PyObject* c = PyCapsule_New(v, "sjb.vocab", vocab_free);
    if (!c) goto fail;
    return c;
  }
nomem:
  PyErr_NoMemory();
fail:
  if (v) {
    free(v->hash);
    free(v->row);
    free(v->off);
    free(v->len);
    free(v->arena);
    free(v);
  }
  return NULL;
}

typedef struct {
  const VocabIndex* v;
  PyObject** items;
  int64_t* out;
  Py_ssize_t b, e;
} ProbeJob;

static void* probe_range(void* arg) {
  ProbeJob* j = (ProbeJob*)arg;
  const VocabIndex* v = j->v;
  for (Py_ssize_t t = j->b; t < j->e; t++) {
    if (t + 8 < j->e) __builtin_prefetch(j->items[t + 8]);
    PyObject* o = j->items[t];
    if (!PyUnicode_Check(o) || !PyUnicode_IS_COMPACT_ASCII(o)) {
      j->out[t] = -2;   /* the caller resolves it with the GIL */
      continue;
    }
    const size_t len = (size_t)PyUnicode_GET_LENGTH(o);
    const char* s = (const char*)PyUnicode_DATA(o);
    const uint64_t h = fnv1a(s, len);
    uint64_t i = h & v->mask;
    int64_t r = -1;
    while (v->hash[i]) {
      if (v->hash[i] == h && v->len[i] == len && memcmp(v->arena + v->off[i], s, len) == 0) {
        r = v->row[i];
        break;
      }
      i = (i + 1) & v->mask;
    }
    j->out[t] = r;
  }
  return NULL;
}

/* lookup_mt(capsule, tokens, threads) -> int64 bytearray (-1 absent, -2 not
 * compact ASCII: resolve with the dict) */
static PyObject* lookup_mt(PyObject* self, PyObject* args) {
  (void)self;
  PyObject *cap, *seq;
  int nthr = 1;
  if (!PyArg_ParseTuple(args, "OOi", &cap, &seq, &nthr)) return NULL;
  const VocabIndex* v = (const VocabIndex*)PyCapsule_GetPointer(cap, "sjb.vocab");
  if (!v) return NULL;
  PyObject* fast = PySequence_Fast(seq, "tokens must be a sequence of str");
  if (!fast) return NULL;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(fast);
  PyObject* out = PyByteArray_FromStringAndSize(NULL, n * (Py_ssize_t)sizeof(int64_t));
  if (!out) {
    Py_DECREF(fast);
    return NULL;
  }
  int64_t* o = (int64_t*)PyByteArray_AS_STRING(out);
  PyObject** items = PySequence_Fast_ITEMS(fast);
  if (nthr < 1) nthr = 1;
  if (nthr > 64) nthr = 64;
  if ((Py_ssize_t)nthr > n / 4096 + 1) nthr = (int)(n / 4096 + 1);
  ProbeJob jobs[64];
  pthread_t tid[64];
  int created[64];
  Py_BEGIN_ALLOW_THREADS
  for (int k = 0; k < nthr; k++) {
    jobs[k].v = v;
    jobs[k].items = items;
    jobs[k].out = o;
    jobs[k].b = n * k / nthr;
    jobs[k].e = n * (k + 1) / nthr;
    created[k] = 0;
  }
  for (int k = 1; k < nthr; k++) {
    created[k] = pthread_create(&tid[k], NULL, probe_range, &jobs[k]) == 0;
    if (!created[k]) probe_range(&jobs[k]);   /* no thread: run it here */
  }
  probe_range(&jobs[0]);
  for (int k = 1; k < nthr; k++)
    if (created[k]) pthread_join(tid[k], NULL);
  Py_END_ALLOW_THREADS
  Py_DECREF(fast);
  return out;
}

static PyMethodDef methods[] = {
    {"pack", pack, METH_O, "pack(tokens) -> (utf8 bytes + NUL, int64 offsets bytes)"},
    {"lookup", lookup, METH_VARARGS, "lookup(index dict, tokens) -> int64 bytearray (-1: absent)"},
    {"build_index", build_index, METH_O, "build_index(dict str -> row) -> vocabulary capsule"},
    {"lookup_mt", lookup_mt, METH_VARARGS,
     "lookup_mt(capsule, tokens, threads) -> int64 bytearray (-1 absent, -2 non-ASCII)"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_sjbpack", NULL, -1, methods};

PyMODINIT_FUNC PyInit__sjbpack(void) { return PyModule_Create(&module); }
