/*
 * _pack -- CPython extension: the pair-batching layer of the drop-in API.
 *
 * Packs a list of (a, b[, payload]) items -- what the reference's
 * AlignEngine.submit / align_batch receive (align.py:223-246, 327-335;
 * pipeline.py:305-310) -- into the C ABI's inputs: one flat byte arena holding
 * every DISTINCT sequence object once (the pipeline passes residues[i] for
 * every pair of sequence i, so identity dedup shares them) and a sw_pair_t
 * table in input order.  Per-pair input errors follow the reference's order
 * of checks (align.py:81-84: empty -> AlignmentError, then a.encode("ascii"),
 * then b.encode("ascii")), plus the GPU aligner's one domain limit (65,000
 * residues per sequence -> ValueError); a failing pair is reported, not
 * packed, and never fails the batch (align.py:235-241).
 *
 * Phase A (worker threads; the calling thread keeps the GIL, so no Python
 *   code runs and every object stays alive -- the workers only read object
 *   memory): items that are tuples of two non-empty ASCII str objects of at
 *   most 65,000 characters (the pipeline's case) are resolved in place and
 *   deduplicated through a lock-free open-addressing map keyed by object
 *   address; every other item is left to phase B.
 * Phase B (calling thread, Python semantics): the remaining items, in input
 *   order, with the reference's exact checks and exceptions.
 * Then arena offsets are a prefix sum over the pieces in input order (a
 *   shared object's bytes sit at the piece of whichever of its users the
 *   threads resolved first; phase D rewrites the table's piece ids).
 * Phase C: the arena buffer comes from the caller's alloc(nbytes) (pinned host
 *   memory from the engine's pool) and the distinct sequences are copied into
 *   it by the worker threads with the GIL released.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <pthread.h>
#include <stdint.h>
#include <string.h>
#include <stdio.h>
#include <stdlib.h>
#include <time.h>

static double now_ms(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

#define MAX_RESIDUES 65000u
#define CHUNK 4096

typedef struct { uint64_t a_off, b_off; uint32_t a_len, b_len; } pair_t;
typedef struct { const char *src; uint64_t len, dst; } piece_t;

typedef struct {               /* one slot of the map: object address -> piece id */
  uintptr_t key;               /* 0 = empty */
  uint64_t pid;                /* piece id + 1 once published (0 = being inserted) */
} slot_t;

typedef struct {               /* lock-free open-addressing map */
  slot_t *slot;
  size_t mask;
} omap_t;

static inline size_t hash_ptr(uintptr_t p) {
  uint64_t x = (uint64_t)p >> 4;
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33;
  return (size_t)x;
}

/* find or insert object `s`, whose bytes would become piece `pid`; returns
 * the piece id holding its bytes (== pid when this call inserted it).  No
 * shared counter: arena offsets are assigned afterwards by a prefix sum over
 * the pieces in input order. */
static uint64_t omap_get(omap_t *M, uintptr_t s, uint64_t pid) {
  size_t i = hash_ptr(s) & M->mask;
  for (;;) {
    slot_t *e = &M->slot[i];
    uintptr_t k = __atomic_load_n(&e->key, __ATOMIC_ACQUIRE);
    if (k == 0) {
      uintptr_t z = 0;
      if (__atomic_compare_exchange_n(&e->key, &z, s, 0, __ATOMIC_ACQ_REL, __ATOMIC_ACQUIRE)) {
        __atomic_store_n(&e->pid, pid + 1, __ATOMIC_RELEASE);
        return pid;
      }
      k = z;
    }
    if (k == s) {
      uint64_t v;
      while ((v = __atomic_load_n(&e->pid, __ATOMIC_ACQUIRE)) == 0) { }
      return v - 1;
    }
    i = (i + 1) & M->mask;
  }
}

/* Maps are kept between calls (a fresh 64 MB calloc costs its page faults
 * on every call) and cleared by the worker threads after use; a small pool,
 * since two batches may be packed concurrently (AlignEngine's two threads). */
#define MAP_POOL 4
static pthread_mutex_t map_mu = PTHREAD_MUTEX_INITIALIZER;
static slot_t *map_free[MAP_POOL];
static size_t map_cap[MAP_POOL];

static slot_t *map_get(size_t cap) {
  pthread_mutex_lock(&map_mu);
  for (int i = 0; i < MAP_POOL; ++i)
    if (map_free[i] && map_cap[i] == cap) {
      slot_t *m = map_free[i];
      map_free[i] = NULL;
      pthread_mutex_unlock(&map_mu);
      return m;
    }
  pthread_mutex_unlock(&map_mu);
  return (slot_t *)calloc(cap, sizeof(slot_t));
}

static void map_put(slot_t *m, size_t cap) {   /* m must be all-zero */
  pthread_mutex_lock(&map_mu);
  for (int i = 0; i < MAP_POOL; ++i)
    if (!map_free[i]) {
      map_free[i] = m;
      map_cap[i] = cap;
      pthread_mutex_unlock(&map_mu);
      return;
    }
  pthread_mutex_unlock(&map_mu);
  free(m);
}

typedef struct {
  PyObject **items;
  Py_ssize_t n;
  omap_t *M;
  pair_t *tmp;                 /* per input item (the caller's table, compacted later) */
  uint8_t *state;              /* 0 packed in phase A, 1 left to phase B */
  piece_t *pc;                 /* bytes to copy: slots 2k, 2k+1 belong to item k */
  Py_ssize_t next;
  pthread_mutex_t mu;
  uint8_t *arena;              /* phase C destination */
  size_t map_cap;              /* phase C also clears the map */
  size_t clear_next;
  int map_cleared;
  uint64_t *blk;               /* prefix sum: per-block totals, then offsets */
  Py_ssize_t nblk;
  int prefix_write;
} job_t;

static inline int fast_str(PyObject *s) {
  return PyUnicode_CheckExact(s) && PyUnicode_IS_COMPACT_ASCII(s) && PyUnicode_GET_LENGTH(s) > 0 &&
         (size_t)PyUnicode_GET_LENGTH(s) <= MAX_RESIDUES;
}

static void *phase_a(void *arg) {
  job_t *J = (job_t *)arg;
  for (;;) {
    pthread_mutex_lock(&J->mu);
    const Py_ssize_t k0 = J->next;
    J->next += CHUNK;
    pthread_mutex_unlock(&J->mu);
    if (k0 >= J->n) break;
    const Py_ssize_t k1 = k0 + CHUNK < J->n ? k0 + CHUNK : J->n;
    for (Py_ssize_t k = k0; k < k1; ++k) {
      /* software prefetch, three items deep per level: the tuple 12 ahead,
       * its two str objects 6 ahead, their map slots 3 ahead (each item
       * touches ~4 cold cache lines) */
      if (k + 12 < k1) __builtin_prefetch(J->items[k + 12]);
      if (k + 6 < k1) {
        PyObject *t = J->items[k + 6];
        if (PyTuple_CheckExact(t) && PyTuple_GET_SIZE(t) >= 2) {
          __builtin_prefetch(PyTuple_GET_ITEM(t, 0));
          __builtin_prefetch(PyTuple_GET_ITEM(t, 1));
        }
      }
      if (k + 3 < k1) {
        PyObject *t = J->items[k + 3];
        if (PyTuple_CheckExact(t) && PyTuple_GET_SIZE(t) >= 2) {
          __builtin_prefetch(&J->M->slot[hash_ptr((uintptr_t)PyTuple_GET_ITEM(t, 0)) & J->M->mask]);
          __builtin_prefetch(&J->M->slot[hash_ptr((uintptr_t)PyTuple_GET_ITEM(t, 1)) & J->M->mask]);
        }
      }
      PyObject *item = J->items[k];
      J->pc[2 * k].len = 0;
      J->pc[2 * k + 1].len = 0;
      if (!PyTuple_CheckExact(item) || PyTuple_GET_SIZE(item) < 2) { J->state[k] = 1; continue; }
      PyObject *a = PyTuple_GET_ITEM(item, 0), *b = PyTuple_GET_ITEM(item, 1);
      if (!fast_str(a) || !fast_str(b)) { J->state[k] = 1; continue; }
      const char *pa = (const char *)PyUnicode_DATA(a), *pb = (const char *)PyUnicode_DATA(b);
      const uint32_t la = (uint32_t)PyUnicode_GET_LENGTH(a), lb = (uint32_t)PyUnicode_GET_LENGTH(b);
      /* pieces 2k / 2k+1: this item's a / b bytes if it is their first user */
      const uint64_t qa = omap_get(J->M, (uintptr_t)a, 2 * (uint64_t)k);
      const uint64_t qb = omap_get(J->M, (uintptr_t)b, 2 * (uint64_t)k + 1);
      if (qa == 2 * (uint64_t)k) { J->pc[2 * k].src = pa; J->pc[2 * k].len = la; }
      if (qb == 2 * (uint64_t)k + 1) { J->pc[2 * k + 1].src = pb; J->pc[2 * k + 1].len = lb; }
      J->tmp[k].a_off = qa; J->tmp[k].b_off = qb;   /* piece ids until phase D */
      J->tmp[k].a_len = la; J->tmp[k].b_len = lb;
      J->state[k] = 0;
    }
  }
  return NULL;
}

static void *phase_c(void *arg) {
  job_t *J = (job_t *)arg;
  /* clear the map for its next use, 1/threads of it per call of this function */
  for (;;) {
    pthread_mutex_lock(&J->mu);
    const size_t s0 = J->clear_next;
    J->clear_next += 1u << 16;
    pthread_mutex_unlock(&J->mu);
    if (s0 >= J->map_cap) break;
    const size_t s1 = s0 + (1u << 16) < J->map_cap ? s0 + (1u << 16) : J->map_cap;
    memset(J->M->slot + s0, 0, (s1 - s0) * sizeof(slot_t));
  }
  const Py_ssize_t np = 2 * J->n;
  for (;;) {
    pthread_mutex_lock(&J->mu);
    const Py_ssize_t k0 = J->next;
    J->next += 2 * CHUNK;
    pthread_mutex_unlock(&J->mu);
    if (k0 >= np) break;
    const Py_ssize_t k1 = k0 + 2 * CHUNK < np ? k0 + 2 * CHUNK : np;
    for (Py_ssize_t k = k0; k < k1; ++k)
      if (J->pc[k].len) memcpy(J->arena + J->pc[k].dst, J->pc[k].src, J->pc[k].len);
  }
  return NULL;
}

#define PREFIX_BLK 65536
/* pass 1 (prefix_write 0): blk[b] = total length of block b's pieces;
 * pass 2: dst of every piece = blk[b] (the block's offset) + running sum */
static void *prefix_sum_pass(void *arg) {
  job_t *J = (job_t *)arg;
  for (;;) {
    pthread_mutex_lock(&J->mu);
    const Py_ssize_t b = J->next;
    J->next += 1;
    pthread_mutex_unlock(&J->mu);
    if (b >= J->nblk) break;
    const Py_ssize_t q0 = b * PREFIX_BLK, q1 = q0 + PREFIX_BLK < 2 * J->n ? q0 + PREFIX_BLK : 2 * J->n;
    if (!J->prefix_write) {
      uint64_t s = 0;
      for (Py_ssize_t q = q0; q < q1; ++q) s += J->pc[q].len;
      J->blk[b] = s;
    } else {
      uint64_t o = J->blk[b];
      for (Py_ssize_t q = q0; q < q1; ++q) {
        J->pc[q].dst = o;
        o += J->pc[q].len;
      }
    }
  }
  return NULL;
}

static void *phase_d(void *arg) {
  job_t *J = (job_t *)arg;
  for (;;) {
    pthread_mutex_lock(&J->mu);
    const Py_ssize_t k0 = J->next;
    J->next += CHUNK;
    pthread_mutex_unlock(&J->mu);
    if (k0 >= J->n) break;
    const Py_ssize_t k1 = k0 + CHUNK < J->n ? k0 + CHUNK : J->n;
    for (Py_ssize_t k = k0; k < k1; ++k) {
      if (J->state[k]) continue;
      J->tmp[k].a_off = J->pc[J->tmp[k].a_off].dst;
      J->tmp[k].b_off = J->pc[J->tmp[k].b_off].dst;
    }
  }
  return NULL;
}

static void run_threads(void *(*fn)(void *), job_t *J, int threads) {
  J->next = 0;
  if (threads <= 1) { fn(J); return; }
  pthread_t th[64];
  int started = 0;
  for (int t = 0; t < threads - 1; ++t)
    if (pthread_create(&th[started], NULL, fn, J) == 0) ++started;
  fn(J);
  for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
}

/* resolve one sequence object the reference's way: its .encode("ascii")
 * bytes (kept alive in `keep`); -1 with the Python exception set */
static int resolve(PyObject *s, PyObject *keep, const char **ptr, Py_ssize_t *len) {
  if (PyUnicode_Check(s) && PyUnicode_IS_ASCII(s)) {
    *ptr = (const char *)PyUnicode_DATA(s);
    *len = PyUnicode_GET_LENGTH(s);
    return 0;
  }
  PyObject *enc = PyObject_CallMethod(s, "encode", "s", "ascii");
  if (!enc) return -1;
  if (!PyBytes_Check(enc)) {
    Py_DECREF(enc);
    PyErr_SetString(PyExc_TypeError, "encode() did not return bytes");
    return -1;
  }
  if (PyList_Append(keep, enc) < 0) { Py_DECREF(enc); return -1; }
  Py_DECREF(enc);
  *ptr = PyBytes_AS_STRING(enc);
  *len = PyBytes_GET_SIZE(enc);
  return 0;
}

static int is_empty(PyObject *s) {
  if (PyUnicode_Check(s)) return PyUnicode_GET_LENGTH(s) == 0;
  int t = PyObject_IsTrue(s);
  return t < 0 ? -1 : !t;
}

static int add_error(PyObject *errors, Py_ssize_t idx) {
  PyObject *exc = PyErr_GetRaisedException();
  if (!exc) return -1;
  PyObject *t = Py_BuildValue("(nN)", idx, exc);
  if (!t) return -1;
  int rc = PyList_Append(errors, t);
  Py_DECREF(t);
  return rc;
}

/* phase B: one item with the reference's semantics; 0 packed, 1 error
 * recorded, -1 fatal (a malformed item raises, like the reference's tuple
 * unpacking would) */
static int slow_item(job_t *J, Py_ssize_t k, PyObject *keep, PyObject *errors, PyObject *err_cls) {
  PyObject *item = J->items[k];
  PyObject *ab[2];
  ab[0] = PySequence_GetItem(item, 0);
  ab[1] = ab[0] ? PySequence_GetItem(item, 1) : NULL;
  if (!ab[0] || !ab[1]) { Py_XDECREF(ab[0]); return -1; }
  /* objects handed out by a non-tuple/list container may be temporaries:
   * keep them alive so their addresses stay unique map keys */
  const int keep_refs = !(PyTuple_Check(item) || PyList_Check(item));
  int bad = 0;
  const int ea = is_empty(ab[0]), eb = ea > 0 ? 0 : is_empty(ab[1]);
  if (ea < 0 || eb < 0) bad = 1;
  else if (ea || eb) { PyErr_SetString(err_cls, "cannot align an empty sequence"); bad = 1; }
  uint64_t o[2] = {0, 0};
  uint32_t L[2] = {0, 0};
  for (int h = 0; h < 2 && !bad; ++h) {
    const char *ptr;
    Py_ssize_t len;
    if (resolve(ab[h], keep, &ptr, &len) < 0) { bad = 1; break; }
    if ((uint64_t)len > MAX_RESIDUES) {
      PyErr_SetString(PyExc_ValueError,
                      "sequence longer than 65,000 residues: outside the GPU aligner's domain");
      bad = 1;
      break;
    }
    if (keep_refs && PyList_Append(keep, ab[h]) < 0) { bad = 1; break; }
    const uint64_t pid = 2 * (uint64_t)k + h;
    o[h] = omap_get(J->M, (uintptr_t)ab[h], pid);
    L[h] = (uint32_t)len;
    /* a sequence inserted for a pair that then fails keeps its arena bytes */
    if (o[h] == pid) { J->pc[pid].src = ptr; J->pc[pid].len = (uint64_t)len; }
  }
  Py_DECREF(ab[0]);
  Py_DECREF(ab[1]);
  if (bad) return add_error(errors, k) < 0 ? -1 : 1;
  J->tmp[k].a_off = o[0]; J->tmp[k].b_off = o[1];
  J->tmp[k].a_len = L[0]; J->tmp[k].b_len = L[1];
  J->state[k] = 0;
  return 0;
}

/* pack(pairs, table_buf, index_buf, alloc, AlignmentError, threads)
 *   -> (n_kept, arena, arena_bytes, errors) */
static PyObject *pack(PyObject *self, PyObject *args) {
  (void)self;
  PyObject *pairs, *table_obj, *index_obj, *alloc, *err_cls;
  int threads = 4;
  if (!PyArg_ParseTuple(args, "OOOOO|i", &pairs, &table_obj, &index_obj, &alloc, &err_cls, &threads))
    return NULL;
  if (threads < 1) threads = 1;
  if (threads > 64) threads = 64;
  PyObject *seq = PySequence_Fast(pairs, "pairs must be a sequence");
  if (!seq) return NULL;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(seq);
  Py_buffer tb, ib;
  if (PyObject_GetBuffer(table_obj, &tb, PyBUF_WRITABLE) < 0) { Py_DECREF(seq); return NULL; }
  if (PyObject_GetBuffer(index_obj, &ib, PyBUF_WRITABLE) < 0) {
    PyBuffer_Release(&tb); Py_DECREF(seq); return NULL;
  }
  PyObject *errors = PyList_New(0), *keep = PyList_New(0), *result = NULL, *arena_obj = NULL;
  omap_t M;
  memset(&M, 0, sizeof(M));
  job_t J;
  memset(&J, 0, sizeof(J));
  pthread_mutex_init(&J.mu, NULL);
  if (!errors || !keep) goto out;
  if ((size_t)tb.len < (size_t)n * sizeof(pair_t) || (size_t)ib.len < (size_t)n * 8) {
    PyErr_SetString(PyExc_ValueError, "table/index buffers too small");
    goto out;
  }
  const double t_0 = now_ms();
  size_t cap = 64;
  while (cap < (size_t)n * 4 + 16) cap <<= 1;
  M.slot = map_get(cap);
  J.map_cap = cap;
  M.mask = cap - 1;
  J.items = PySequence_Fast_ITEMS(seq);
  J.n = n;
  J.M = &M;
  J.tmp = (pair_t *)tb.buf;
  J.state = (uint8_t *)PyMem_Malloc((size_t)n + 1);
  J.pc = (piece_t *)PyMem_Malloc(((size_t)n * 2 + 1) * sizeof(piece_t));
  if (!M.slot || !J.state || !J.pc) { PyErr_NoMemory(); goto out; }
  const double t_alloc = now_ms();
  /* phase A: no Python calls; the GIL stays with this thread throughout */
  run_threads(phase_a, &J, n >= 2 * CHUNK ? threads : 1);
  const double t_a = now_ms();
  /* phase B */
  for (Py_ssize_t k = 0; k < n; ++k)
    if (J.state[k] && slow_item(&J, k, keep, errors, err_cls) < 0) goto out;
  /* arena offsets: prefix sum over the pieces in input order (two threaded
   * passes over blocks of pieces: block sums, then offsets) */
  uint64_t off = 0;
  {
    const Py_ssize_t np = 2 * n, nblk = (np + PREFIX_BLK - 1) / PREFIX_BLK;
    J.blk = (uint64_t *)PyMem_Malloc(((size_t)nblk + 1) * sizeof(uint64_t));
    if (!J.blk) { PyErr_NoMemory(); goto out; }
    J.nblk = nblk;
    run_threads(prefix_sum_pass, &J, nblk >= 8 ? threads : 1);
    for (Py_ssize_t b = 0; b < nblk; ++b) {
      const uint64_t t = J.blk[b];
      J.blk[b] = off;
      off += t;
    }
    J.prefix_write = 1;
    run_threads(prefix_sum_pass, &J, nblk >= 8 ? threads : 1);
    PyMem_Free(J.blk);
    J.blk = NULL;
  }
  const double t_b = now_ms();
  /* phase D: piece ids -> offsets */
  run_threads(phase_d, &J, n >= 2 * CHUNK ? threads : 1);
  const double t_d = now_ms();
  /* compaction (only when some pair failed) */
  int64_t *index = (int64_t *)ib.buf;
  pair_t *table = (pair_t *)tb.buf;
  Py_ssize_t kept = 0;
  if (PyList_GET_SIZE(errors) == 0) {
    for (Py_ssize_t k = 0; k < n; ++k) index[k] = k;
    kept = n;
  } else {
    for (Py_ssize_t k = 0; k < n; ++k) {
      if (J.state[k]) continue;
      table[kept] = table[k];
      index[kept] = k;
      ++kept;
    }
  }
  {
    const uint64_t nbytes = off ? off : 1;
    arena_obj = PyObject_CallFunction(alloc, "K", (unsigned long long)nbytes);
    if (!arena_obj) goto out;
    Py_buffer ab;
    if (PyObject_GetBuffer(arena_obj, &ab, PyBUF_WRITABLE) < 0) goto out;
    if ((uint64_t)ab.len < nbytes) {
      PyBuffer_Release(&ab);
      PyErr_SetString(PyExc_ValueError, "alloc() returned a buffer that is too small");
      goto out;
    }
    J.arena = (uint8_t *)ab.buf;
    const int tc = off >= (1u << 20) ? threads : 1;
    const double t_c0 = now_ms();
    J.clear_next = 0;
    Py_BEGIN_ALLOW_THREADS
    run_threads(phase_c, &J, tc);
    Py_END_ALLOW_THREADS
    J.map_cleared = 1;
    if (getenv("PASTIS_PACK_DEBUG"))
      fprintf(stderr, "pack: n=%zd threads=%d alloc=%.2f A=%.2f B+prefix=%.2f D=%.2f arena_alloc=%.2f C=%.2f ms\n",
              n, threads, t_alloc - t_0, t_a - t_alloc, t_b - t_a, t_d - t_b, t_c0 - t_d, now_ms() - t_c0);
    PyBuffer_Release(&ab);
    result = Py_BuildValue("(nOKO)", kept, arena_obj, (unsigned long long)off, errors);
  }
out:
  pthread_mutex_destroy(&J.mu);
  Py_XDECREF(arena_obj);
  if (M.slot) {
    if (!J.map_cleared) memset(M.slot, 0, J.map_cap * sizeof(slot_t));
    map_put(M.slot, J.map_cap);
  }
  PyMem_Free(J.state);
  PyMem_Free(J.pc);
  Py_XDECREF(errors);
  Py_XDECREF(keep);
  PyBuffer_Release(&tb);
  PyBuffer_Release(&ib);
  Py_DECREF(seq);
  return result;
}

static PyMethodDef methods[] = {
    {"pack", pack, METH_VARARGS, "pack(pairs, table, index, alloc, AlignmentError[, threads])"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef mod = {PyModuleDef_HEAD_INIT, "_pack", NULL, -1, methods,
                                 NULL, NULL, NULL, NULL};

PyMODINIT_FUNC PyInit__pack(void) { return PyModule_Create(&mod); }
