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
#include <string.h>

typedef struct {
    const char *src;
    char *dst;
    size_t len;
} Piece;

typedef struct {
    const Piece *pieces;
    size_t begin, end;
} Span;

static void *copy_span(void *arg) {
    const Span *s = (const Span *)arg;
    for (size_t i = s->begin; i < s->end; ++i)
        if (s->pieces[i].len) memcpy(s->pieces[i].dst, s->pieces[i].src, s->pieces[i].len);
    return NULL;
}

#define MAX_COPY_THREADS 16
#define BYTES_PER_THREAD ((size_t)4 << 20)

/* Copy all pieces; caller has released the GIL. Threads split the pieces by bytes. */
static void copy_pieces(const Piece *pieces, size_t n, size_t total, int max_threads) {
    int threads = (int)(total / BYTES_PER_THREAD);
    if (threads > max_threads) threads = max_threads;
    if (threads > MAX_COPY_THREADS) threads = MAX_COPY_THREADS;
    if (threads < 2) {
        Span all = {pieces, 0, n};
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
        spans[t].pieces = pieces; spans[t].begin = b; spans[t].end = i;
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

static PyMethodDef methods[] = {
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
