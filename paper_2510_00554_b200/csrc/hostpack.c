/* _hostpack: host-side packing for the reference-shaped entry points (CPython extension, plain C).
 *
 * The reference's hash_blocks (merkle.py:93-114) takes a SEQUENCE of bytes-like blocks and its loader
 * protocol (dataset.py:74-86) a Batch of SampleRecord objects. The GPU wants ONE contiguous block per
 * launch in page-locked memory. Walking such sequences in Python costs 0.4-2 us per item (frombuffer,
 * attribute reads, b"".join, a second copy into the pinned block); here it is one pass over the buffer
 * protocol and one memcpy per item straight into the pinned destination, the copies outside the GIL and
 * on several threads when the pack is large.
 *
 * No hashing happens here: this is host plumbing above the C ABI of include/sentinel_b200.h.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    const char *src;
    char *dst;
    size_t len;
} Piece;

typedef struct {
    const Piece *pieces;
    size_t begin, end;
    int stream;           /* large packs: streaming stores (the copy engine reads the block next) */
} Span;

static void copy_to_staging(char *dst, const char *src, size_t n);      /* streaming stores, defined with the pool */

static void *copy_span(void *arg) {
    const Span *s = (const Span *)arg;
    for (size_t i = s->begin; i < s->end; ++i) {
        if (!s->pieces[i].len) continue;
        if (s->stream) copy_to_staging(s->pieces[i].dst, s->pieces[i].src, s->pieces[i].len);
        else memcpy(s->pieces[i].dst, s->pieces[i].src, s->pieces[i].len);
    }
    return NULL;
}

#define MAX_COPY_THREADS 16
#define BYTES_PER_THREAD ((size_t)4 << 20)

/* Copy all pieces; caller has released the GIL. Threads split the pieces by bytes. */
static void copy_pieces(const Piece *pieces, size_t n, size_t total, int max_threads) {
    int threads = (int)(total / BYTES_PER_THREAD);
    if (threads > max_threads) threads = max_threads;
    if (threads > MAX_COPY_THREADS) threads = MAX_COPY_THREADS;
    /* streaming stores pay for packs the copy engine reads from DRAM anyway (128 MiB of 8 KiB blocks: 9.1 -> 7.5 ms);
     * a loader batch of a few hundred KB on one thread is faster with ordinary stores (391 batches: 35 vs 41 ms) */
    const int stream = total >= ((size_t)8 << 20);
    if (threads < 2) {
        Span all = {pieces, 0, n, stream};
        copy_span(&all);
        return;
    }
    Span spans[MAX_COPY_THREADS];
    pthread_t tids[MAX_COPY_THREADS];
    int started[MAX_COPY_THREADS];
    size_t share = total / (size_t)threads + 1, i = 0;
    for (int t = 0; t < threads; ++t) {
        size_t acc = 0, b = i;
        while (i < n && (acc < share || t == threads - 1)) acc += pieces[i++].len;
        spans[t].pieces = pieces; spans[t].begin = b; spans[t].end = i; spans[t].stream = stream;
    }
    for (int t = 1; t < threads; ++t)
        started[t] = pthread_create(&tids[t], NULL, copy_span, &spans[t]) == 0;
    copy_span(&spans[0]);
    for (int t = 1; t < threads; ++t) {
        if (started[t]) pthread_join(tids[t], NULL);
        else copy_span(&spans[t]);
    }
}

static void release_views(Py_buffer *views, size_t n) {
    for (size_t i = 0; i < n; ++i) PyBuffer_Release(&views[i]);
    PyMem_Free(views);
}

/* gather(seq, dst_addr, capacity, lens_addr, threads) -> total
 *
 * lens_addr (if non-zero) receives len(seq) uint64 lengths. When total <= capacity the items are copied
 * back to back to dst_addr; otherwise nothing is copied (capacity 0 = measure only). */
static PyObject *hp_gather(PyObject *self, PyObject *args) {
    PyObject *seq_in;
    unsigned long long dst_addr, capacity, lens_addr;
    int threads = 8;
    if (!PyArg_ParseTuple(args, "OKKK|i", &seq_in, &dst_addr, &capacity, &lens_addr, &threads)) return NULL;
    PyObject *seq = PySequence_Fast(seq_in, "gather expects a sequence of bytes-like objects");
    if (!seq) return NULL;
    size_t n = (size_t)PySequence_Fast_GET_SIZE(seq);
    PyObject **items = PySequence_Fast_ITEMS(seq);
    uint64_t *lens = (uint64_t *)(uintptr_t)lens_addr;
    Py_buffer *views = (Py_buffer *)PyMem_Malloc((n ? n : 1) * sizeof(Py_buffer));
    Piece *pieces = (Piece *)PyMem_Malloc((n ? n : 1) * sizeof(Piece));
    if (!views || !pieces) {
        PyMem_Free(views); PyMem_Free(pieces); Py_DECREF(seq);
        return PyErr_NoMemory();
    }
    size_t total = 0;
    for (size_t i = 0; i < n; ++i) {
        if (PyObject_GetBuffer(items[i], &views[i], PyBUF_SIMPLE) != 0) {
            release_views(views, i); PyMem_Free(pieces); Py_DECREF(seq);
            return NULL;
        }
        pieces[i].src = (const char *)views[i].buf;
        pieces[i].len = (size_t)views[i].len;
        pieces[i].dst = (char *)(uintptr_t)dst_addr + total;
        if (lens) lens[i] = (uint64_t)views[i].len;
        total += (size_t)views[i].len;
    }
    if (total <= capacity && total) {
        Py_BEGIN_ALLOW_THREADS
        copy_pieces(pieces, n, total, threads);
        Py_END_ALLOW_THREADS
    }
    release_views(views, n);
    PyMem_Free(pieces);
    Py_DECREF(seq);
    return PyLong_FromSize_t(total);
}

static PyObject *s_data, *s_label, *s_sample_id, *s_source_id;

/* pack_records(samples, cover_labels, slot_of, declared, dst_addr, capacity) -> (code, a, b)
 *
 * Lays a batch out as  offsets[n] u64 | lengths[n] u64 | ids[n] u64 | slots[n] i32 | pad to 16 | payload
 * (payload of sample i = label ‖ data when cover_labels, else data).
 *   (0, total, header)  packed
 *   (1, needed, 0)      capacity too small, nothing written
 *   (2, index, 0)       samples[index].source_id is not in `declared`
 *   (3, index, 0)       samples[index].sample_id does not fit an unsigned 64-bit tag
 *   (4, index, 0)       samples[index].source_id has no slot in `slot_of` yet
 * Checks run in that order over the whole batch, as the Python path does. */
static PyObject *hp_pack_records(PyObject *self, PyObject *args) {
    PyObject *seq_in, *slot_of, *declared;
    int cover_labels;
    unsigned long long dst_addr, capacity;
    if (!PyArg_ParseTuple(args, "OpOOKK", &seq_in, &cover_labels, &slot_of, &declared, &dst_addr, &capacity)) return NULL;
    if (!PyDict_Check(slot_of)) { PyErr_SetString(PyExc_TypeError, "slot_of must be a dict"); return NULL; }
    PyObject *seq = PySequence_Fast(seq_in, "pack_records expects a sequence of records");
    if (!seq) return NULL;
    size_t n = (size_t)PySequence_Fast_GET_SIZE(seq);
    PyObject **items = PySequence_Fast_ITEMS(seq);
    size_t nviews = 0, cap_views = (cover_labels ? 2 : 1) * (n ? n : 1);
    Py_buffer *views = (Py_buffer *)PyMem_Malloc(cap_views * sizeof(Py_buffer));
    Piece *pieces = (Piece *)PyMem_Malloc(cap_views * sizeof(Piece));
    uint64_t *meta = (uint64_t *)PyMem_Malloc((n ? n : 1) * 3 * sizeof(uint64_t));   /* len, id, slot */
    PyObject *result = NULL;
    long code = 0; size_t a = 0, b = 0;
    if (!views || !pieces || !meta) { PyErr_NoMemory(); goto done; }

    if (declared != Py_None) {
        for (size_t i = 0; i < n; ++i) {
            PyObject *src = PyObject_GetAttr(items[i], s_source_id);
            if (!src) goto done;
            int has = PySet_Check(declared) || PyFrozenSet_Check(declared) ? PySet_Contains(declared, src)
                                                                          : PySequence_Contains(declared, src);
            Py_DECREF(src);
            if (has < 0) goto done;
            if (!has) { code = 2; a = i; goto answer; }
        }
    }
    for (size_t i = 0; i < n; ++i) {
        PyObject *idobj = PyObject_GetAttr(items[i], s_sample_id);
        if (!idobj) goto done;
        unsigned long long id = PyLong_Check(idobj) ? PyLong_AsUnsignedLongLong(idobj) : (unsigned long long)-1;
        int bad = !PyLong_Check(idobj) || (id == (unsigned long long)-1 && PyErr_Occurred());
        Py_DECREF(idobj);
        if (bad) { PyErr_Clear(); code = 3; a = i; goto answer; }
        meta[3 * i + 1] = id;
    }
    size_t total = 0;
    for (size_t i = 0; i < n; ++i) {
        PyObject *src = PyObject_GetAttr(items[i], s_source_id);
        if (!src) goto done;
        PyObject *slot = PyDict_GetItemWithError(slot_of, src);      /* borrowed */
        Py_DECREF(src);
        if (!slot) {
            if (PyErr_Occurred()) goto done;
            code = 4; a = i; goto answer;
        }
        long s = PyLong_AsLong(slot);
        if (s == -1 && PyErr_Occurred()) goto done;
        meta[3 * i + 2] = (uint64_t)s;
        size_t len = 0;
        for (int part = cover_labels ? 0 : 1; part < 2; ++part) {
            PyObject *obj = PyObject_GetAttr(items[i], part ? s_data : s_label);
            if (!obj) goto done;
            int rc = PyObject_GetBuffer(obj, &views[nviews], PyBUF_SIMPLE);
            Py_DECREF(obj);                                          /* the view keeps its exporter alive */
            if (rc != 0) goto done;
            pieces[nviews].src = (const char *)views[nviews].buf;
            pieces[nviews].len = (size_t)views[nviews].len;
            len += (size_t)views[nviews].len;
            ++nviews;
        }
        meta[3 * i] = len;
        total += len;
    }
    {
        size_t header = (28 * n + 15) / 16 * 16;
        size_t needed = header + (total > 16 ? total : 16);
        if (needed > capacity) { code = 1; a = needed; goto answer; }
        char *base = (char *)(uintptr_t)dst_addr;
        uint64_t *offs = (uint64_t *)base, *lens = offs + n, *ids = lens + n;
        int32_t *slots = (int32_t *)(ids + n);
        size_t off = 0;
        for (size_t i = 0; i < n; ++i) {
            offs[i] = off; lens[i] = meta[3 * i]; ids[i] = meta[3 * i + 1]; slots[i] = (int32_t)meta[3 * i + 2];
            off += meta[3 * i];
        }
        char *p = base + header;
        for (size_t v = 0; v < nviews; ++v) { pieces[v].dst = p; p += pieces[v].len; }
        Py_BEGIN_ALLOW_THREADS
        copy_pieces(pieces, nviews, total, 8);
        Py_END_ALLOW_THREADS
        code = 0; a = total; b = header;
    }
answer:
    result = Py_BuildValue("(lnn)", code, (Py_ssize_t)a, (Py_ssize_t)b);
done:
    if (views) { for (size_t v = 0; v < nviews; ++v) PyBuffer_Release(&views[v]); PyMem_Free(views); }
    PyMem_Free(pieces);
    PyMem_Free(meta);
    Py_DECREF(seq);
    return result;
}

/* manifest_columns(rows, ids_addr, src_addr, off_addr, len_addr) -> (code, index)
 *
 * rows: sequence of (sample_id, source_id, label, offset, length) tuples (DatasetManifest.samples). Writes the
 * four integer columns (u64 ids, i64 the rest) in one pass.
 *   (0, n)      done
 *   (3, index)  rows[index].sample_id does not fit an unsigned 64-bit tag
 *   (5, index)  another field of rows[index] is not an integer that fits 64 bits (caller takes its Python path) */
static PyObject *hp_manifest_columns(PyObject *self, PyObject *args) {
    PyObject *seq_in;
    unsigned long long a_ids, a_src, a_off, a_len;
    if (!PyArg_ParseTuple(args, "OKKKK", &seq_in, &a_ids, &a_src, &a_off, &a_len)) return NULL;
    PyObject *seq = PySequence_Fast(seq_in, "manifest_columns expects a sequence of rows");
    if (!seq) return NULL;
    size_t n = (size_t)PySequence_Fast_GET_SIZE(seq);
    PyObject **items = PySequence_Fast_ITEMS(seq);
    uint64_t *ids = (uint64_t *)(uintptr_t)a_ids;
    int64_t *cols[3] = {(int64_t *)(uintptr_t)a_src, (int64_t *)(uintptr_t)a_off, (int64_t *)(uintptr_t)a_len};
    static const int field[3] = {1, 3, 4};
    long code = 0; size_t at = n;
    for (size_t i = 0; i < n && !code; ++i) {
        PyObject *row = items[i];
        if (!PyTuple_Check(row) || PyTuple_GET_SIZE(row) < 5) { code = 5; at = i; break; }
        PyObject *idobj = PyTuple_GET_ITEM(row, 0);
        if (!PyLong_Check(idobj)) { code = 3; at = i; break; }
        unsigned long long id = PyLong_AsUnsignedLongLong(idobj);
        if (id == (unsigned long long)-1 && PyErr_Occurred()) { PyErr_Clear(); code = 3; at = i; break; }
        ids[i] = id;
        for (int c = 0; c < 3; ++c) {
            PyObject *v = PyTuple_GET_ITEM(row, field[c]);
            long long x = PyLong_Check(v) ? PyLong_AsLongLong(v) : -1;
            if (!PyLong_Check(v) || (x == -1 && PyErr_Occurred())) { PyErr_Clear(); code = 5; at = i; break; }
            cols[c][i] = x;
        }
    }
    Py_DECREF(seq);
    return Py_BuildValue("(ln)", code, (Py_ssize_t)at);
}

/* ---- a persistent pool of copy threads ---------------------------------------------------------------------------
 * Fills pinned staging buffers from pageable memory (streaming stores) or from a file (pread). The Python version
 * queued one task per 4 MB piece on a ThreadPoolExecutor and copied with ordinary stores. Here the threads live in C,
 * take 1 MB jobs from a queue of batches and never touch the GIL; a batch is submitted without blocking
 * (copy_submit) and waited for later (copy_wait), so the caller can queue the next staging buffer and issue transfers
 * while the threads copy. */
#include <immintrin.h>
#include <stdatomic.h>
#include <sys/types.h>
#include <unistd.h>

#define POOL_MAX 16
#define QUEUE_MAX 16
#define JOB_BYTES ((size_t)1 << 20)

typedef struct {
    char *dst;
    const char *src;      /* memory source, or NULL when the batch reads a file */
    long long file_off;
    size_t len;
} Job;

typedef struct {
    Job *jobs;
    size_t njobs, next, unfinished;
    int fd, failed, done, in_use;
    unsigned long id;
} Batch;

static struct {
    pthread_mutex_t mu;
    pthread_cond_t work, finished;
    int nthreads;
    pid_t owner;
    Batch q[QUEUE_MAX];
    unsigned long next_id;
} pool = {PTHREAD_MUTEX_INITIALIZER, PTHREAD_COND_INITIALIZER, PTHREAD_COND_INITIALIZER};

/* memcpy whose stores bypass the caches. The destination is a page-locked staging buffer that the GPU's copy engine
 * reads next: with ordinary stores its lines sit dirty in the L2s of a dozen cores and every DMA read has to snoop
 * them out (64 MB through the ring: 3.8 ms; with streaming stores 1.8 ms), and every store costs a
 * read-for-ownership (12 threads: 60 -> 75 GB/s). tools/ring_probe.py, SNT_CACHED_STAGING=1 for the A/B. */
__attribute__((target("avx2"))) static void copy_stream_avx2(char *dst, const char *src, size_t n) {
    size_t head = (32 - ((uintptr_t)dst & 31)) & 31;
    if (head > n) head = n;
    if (head) { memcpy(dst, src, head); dst += head; src += head; n -= head; }
    size_t i = 0;
    for (; i + 128 <= n; i += 128) {
        __m256i a = _mm256_loadu_si256((const __m256i *)(src + i)), b = _mm256_loadu_si256((const __m256i *)(src + i + 32)),
                c = _mm256_loadu_si256((const __m256i *)(src + i + 64)), d = _mm256_loadu_si256((const __m256i *)(src + i + 96));
        _mm256_stream_si256((__m256i *)(dst + i), a); _mm256_stream_si256((__m256i *)(dst + i + 32), b);
        _mm256_stream_si256((__m256i *)(dst + i + 64), c); _mm256_stream_si256((__m256i *)(dst + i + 96), d);
    }
    for (; i + 32 <= n; i += 32) _mm256_stream_si256((__m256i *)(dst + i), _mm256_loadu_si256((const __m256i *)(src + i)));
    if (i < n) memcpy(dst + i, src + i, n - i);
    _mm_sfence();
}

static int g_stream_stores = -1;      /* -1: not decided yet */

static void copy_to_staging(char *dst, const char *src, size_t n) {
    if (g_stream_stores < 0) {
        const char *e = getenv("SNT_CACHED_STAGING");
        g_stream_stores = (!e || !*e || *e == '0') && __builtin_cpu_supports("avx2");
    }
    if (g_stream_stores && n >= 1024) copy_stream_avx2(dst, src, n);
    else memcpy(dst, src, n);
}

static int run_job(const Job *j, int fd) {
    if (fd < 0) { copy_to_staging(j->dst, j->src, j->len); return 0; }
    size_t got = 0;
    while (got < j->len) {
        ssize_t r = pread(fd, j->dst + got, j->len - got, (off_t)(j->file_off + (long long)got));
        if (r <= 0) return -1;
        got += (size_t)r;
    }
    return 0;
}

/* Oldest batch that still has a job to hand out (pool.mu held). */
static Batch *next_batch(void) {
    Batch *best = NULL;
    for (int i = 0; i < QUEUE_MAX; ++i) {
        Batch *b = &pool.q[i];
        if (b->in_use && b->next < b->njobs && (!best || b->id < best->id)) best = b;
    }
    return best;
}

static void *pool_worker(void *arg) {
    (void)arg;
    pthread_mutex_lock(&pool.mu);
    for (;;) {
        Batch *b = next_batch();
        if (!b) { pthread_cond_wait(&pool.work, &pool.mu); continue; }
        const Job *j = &b->jobs[b->next++];
        const int fd = b->fd;
        pthread_mutex_unlock(&pool.mu);
        const int rc = run_job(j, fd);
        pthread_mutex_lock(&pool.mu);
        if (rc) b->failed = 1;
        if (--b->unfinished == 0) { b->done = 1; pthread_cond_broadcast(&pool.finished); }
    }
    return NULL;
}

/* Queue a batch (takes ownership of jobs). Returns its id (> 0), or 0 when the queue is full / no thread could be made. */
static unsigned long pool_submit(Job *jobs, size_t njobs, int fd, int threads) {
    if (threads > POOL_MAX) threads = POOL_MAX;
    if (threads < 1) threads = 1;
    pthread_mutex_lock(&pool.mu);
    if (pool.owner != getpid()) {                     /* first use, or the child of a fork(): no threads, no batches */
        pool.owner = getpid(); pool.nthreads = 0;
        memset(pool.q, 0, sizeof pool.q);
    }
    while (pool.nthreads < threads) {
        pthread_t t;
        if (pthread_create(&t, NULL, pool_worker, NULL) != 0) break;
        pthread_detach(t);
        ++pool.nthreads;
    }
    Batch *b = NULL;
    for (int i = 0; i < QUEUE_MAX && !b; ++i) if (!pool.q[i].in_use) b = &pool.q[i];
    if (!b || pool.nthreads == 0) { pthread_mutex_unlock(&pool.mu); return 0; }
    b->jobs = jobs; b->njobs = njobs; b->next = 0; b->unfinished = njobs; b->fd = fd;
    b->failed = 0; b->done = njobs == 0; b->in_use = 1; b->id = ++pool.next_id;
    const unsigned long id = b->id;
    pthread_cond_broadcast(&pool.work);
    pthread_mutex_unlock(&pool.mu);
    return id;
}

/* Wait for a batch and release it. 0 = copied, -1 = short read, -2 = unknown id. GIL must be released. */
static int pool_wait(unsigned long id) {
    pthread_mutex_lock(&pool.mu);
    Batch *b = NULL;
    for (int i = 0; i < QUEUE_MAX; ++i) if (pool.q[i].in_use && pool.q[i].id == id) b = &pool.q[i];
    if (!b) { pthread_mutex_unlock(&pool.mu); return -2; }
    while (!b->done) pthread_cond_wait(&pool.finished, &pool.mu);
    const int rc = b->failed ? -1 : 0;
    Job *jobs = b->jobs;
    b->in_use = 0; b->jobs = NULL;
    pthread_mutex_unlock(&pool.mu);
    free(jobs);
    return rc;
}

/* pieces: flat sequence of ints  dst_addr, src, len, ...  -> malloc'ed 1 MB jobs */
static Job *parse_pieces(PyObject *seq_in, int fd, size_t *njobs_out, size_t *total_out) {
    PyObject *seq = PySequence_Fast(seq_in, "expected a flat sequence of integers");
    if (!seq) return NULL;
    size_t n = (size_t)PySequence_Fast_GET_SIZE(seq);
    PyObject **items = PySequence_Fast_ITEMS(seq);
    if (n % 3) { Py_DECREF(seq); PyErr_SetString(PyExc_ValueError, "pieces come in (dst, src, len) triples"); return NULL; }
    size_t njobs = 0, total = 0;
    for (size_t i = 0; i < n; i += 3) {
        unsigned long long len = PyLong_AsUnsignedLongLong(items[i + 2]);
        if (len == (unsigned long long)-1 && PyErr_Occurred()) { Py_DECREF(seq); return NULL; }
        njobs += (size_t)((len + JOB_BYTES - 1) / JOB_BYTES);
        total += (size_t)len;
    }
    Job *jobs = (Job *)malloc((njobs ? njobs : 1) * sizeof(Job));
    if (!jobs) { Py_DECREF(seq); PyErr_NoMemory(); return NULL; }
    size_t k = 0;
    for (size_t i = 0; i < n; i += 3) {
        unsigned long long dst = PyLong_AsUnsignedLongLong(items[i]), src = PyLong_AsUnsignedLongLong(items[i + 1]),
                           len = PyLong_AsUnsignedLongLong(items[i + 2]);
        if (PyErr_Occurred()) { free(jobs); Py_DECREF(seq); return NULL; }
        for (unsigned long long o = 0; o < len; o += JOB_BYTES) {
            jobs[k].dst = (char *)(uintptr_t)(dst + o);
            jobs[k].src = fd < 0 ? (const char *)(uintptr_t)(src + o) : NULL;
            jobs[k].file_off = (long long)(src + o);
            jobs[k].len = (size_t)(len - o < JOB_BYTES ? len - o : JOB_BYTES);
            ++k;
        }
    }
    Py_DECREF(seq);
    *njobs_out = njobs; *total_out = total;
    return jobs;
}

/* copy_submit(pieces, fd=-1, threads=12) -> batch id (0: nothing to copy). The memory the pieces name (and the
 * file) must stay valid until copy_wait(id) returns. */
static PyObject *hp_copy_submit(PyObject *self, PyObject *args) {
    PyObject *seq_in;
    int fd = -1, threads = 12;
    if (!PyArg_ParseTuple(args, "O|ii", &seq_in, &fd, &threads)) return NULL;
    size_t njobs = 0, total = 0;
    Job *jobs = parse_pieces(seq_in, fd, &njobs, &total);
    if (!jobs) return NULL;
    if (njobs == 0) { free(jobs); return PyLong_FromLong(0); }
    unsigned long id = pool_submit(jobs, njobs, fd, threads);
    if (id == 0) {                                    /* queue full or no threads: copy here and now */
        int rc = 0;
        Py_BEGIN_ALLOW_THREADS
        for (size_t i = 0; i < njobs; ++i) rc |= run_job(&jobs[i], fd);
        Py_END_ALLOW_THREADS
        free(jobs);
        if (rc) { PyErr_SetString(PyExc_OSError, "short read while staging a file"); return NULL; }
        return PyLong_FromLong(0);
    }
    return PyLong_FromUnsignedLong(id);
}

/* copy_wait(id): returns when the batch has been copied; OSError on a short read. id 0 is a no-op. */
static PyObject *hp_copy_wait(PyObject *self, PyObject *args) {
    unsigned long id;
    if (!PyArg_ParseTuple(args, "k", &id)) return NULL;
    if (id == 0) Py_RETURN_NONE;
    int rc;
    Py_BEGIN_ALLOW_THREADS
    rc = pool_wait(id);
    Py_END_ALLOW_THREADS
    if (rc == -1) { PyErr_SetString(PyExc_OSError, "short read while staging a file"); return NULL; }
    if (rc == -2) { PyErr_SetString(PyExc_ValueError, "unknown copy batch"); return NULL; }
    Py_RETURN_NONE;
}

/* copy_many(pieces, fd=-1, threads=12) -> bytes copied: copy_submit + copy_wait. */
static PyObject *hp_copy_many(PyObject *self, PyObject *args) {
    PyObject *seq_in;
    int fd = -1, threads = 12;
    if (!PyArg_ParseTuple(args, "O|ii", &seq_in, &fd, &threads)) return NULL;
    size_t njobs = 0, total = 0;
    Job *jobs = parse_pieces(seq_in, fd, &njobs, &total);
    if (!jobs) return NULL;
    int rc = 0;
    if (njobs) {
        Py_BEGIN_ALLOW_THREADS
        unsigned long id = pool_submit(jobs, njobs, fd, threads);
        if (id) rc = pool_wait(id);
        else { for (size_t i = 0; i < njobs; ++i) rc |= run_job(&jobs[i], fd); free(jobs); }
        Py_END_ALLOW_THREADS
    } else {
        free(jobs);
    }
    if (rc != 0) { PyErr_SetString(PyExc_OSError, "short read while staging a file"); return NULL; }
    return PyLong_FromSize_t(total);
}

static PyMethodDef methods[] = {
    {"copy_many", hp_copy_many, METH_VARARGS, "copy_many(pieces, fd=-1, threads=12) -> bytes copied"},
    {"copy_submit", hp_copy_submit, METH_VARARGS, "copy_submit(pieces, fd=-1, threads=12) -> batch id"},
    {"copy_wait", hp_copy_wait, METH_VARARGS, "copy_wait(batch id)"},
    {"manifest_columns", hp_manifest_columns, METH_VARARGS,
     "manifest_columns(rows, ids_addr, src_addr, off_addr, len_addr) -> (code, index)"},
    {"gather", hp_gather, METH_VARARGS, "gather(seq, dst_addr, capacity, lens_addr, threads=8) -> total bytes"},
    {"pack_records", hp_pack_records, METH_VARARGS,
     "pack_records(samples, cover_labels, slot_of, declared, dst_addr, capacity) -> (code, a, b)"},
    {NULL, NULL, 0, NULL},
};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_hostpack", "host-side packing helpers", -1, methods};

PyMODINIT_FUNC PyInit__hostpack(void) {
    s_data = PyUnicode_InternFromString("data");
    s_label = PyUnicode_InternFromString("label");
    s_sample_id = PyUnicode_InternFromString("sample_id");
    s_source_id = PyUnicode_InternFromString("source_id");
    return PyModule_Create(&module);
}
