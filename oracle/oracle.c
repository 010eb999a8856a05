/*
 * oracle.c -- plain-C CPU restatement of the reference's hashing path.
 *
 * TEST INFRASTRUCTURE. Only tests/, __graft_entry__.smoke() and bench.py's
 * CPU-baseline / --impl reference legs load this library; the product package
 * never does (it has no CPU fallback).
 *
 * The reference (/root/reference/pkg/src/sentinel) delegates its arithmetic to
 * CPython hashlib, a third-party dependency not vendored under /root/reference
 * (pyproject.toml:10-14 pins nothing tighter than python>=3.10; this container
 * has Python 3.12.3 / OpenSSL 3.0.13). The three primitives are therefore
 * restated here from their published specifications:
 *   SHA-256      FIPS 180-4 sec. 6.2        (hashlib.sha256,   compression.py:45-49)
 *   BLAKE2b-512  RFC 7693 sec. 3, unkeyed    (hashlib.blake2b,  compression.py:45-49, lattice.py:99)
 *   SHA3-256     FIPS 202 sec. 3-6           (hashlib.sha3_256, compression.py:45-49)
 * and the constructions follow the reference's own code:
 *   orc_hash_blocks      merkle.py:93-114   entry i = H(block i), contiguous ranges per worker (workers.py:30-57)
 *   orc_merkle_root      merkle.py:117-165  pair neighbours, zero-pad an odd level, one leaf = root
 *   orc_inplace_*        model.py:137-146, :298-315   block table over fragmented tensors, ragged tails unpadded
 *   orc_lthash_samples   lattice.py:97-119, dataset.py:41-49, :74-91   BLAKE2b(LE64(id) || data), u16 lane sums per source
 *
 * Parity is PINNED: tests/test_oracle.py checks every function against the
 * golden vectors in tests/golden/ (the reference suite's known answers and
 * golden digest, and fixtures produced by the unmodified reference package).
 *
 * SHA-256 uses the x86 SHA extensions when the CPU has them (runtime check),
 * as OpenSSL does for the reference; the portable path is otherwise identical.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#if defined(__x86_64__)
#include <cpuid.h>
#include <immintrin.h>
#define ORC_X86 1
#else
#define ORC_X86 0
#endif

enum { ORC_SHA256 = 0, ORC_BLAKE2B = 1, ORC_SHA3_256 = 2 };

static int digest_len(int alg) { return alg == ORC_BLAKE2B ? 64 : 32; }

/* ------------------------------------------------------------------ SHA-256 */

static const uint32_t K256[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
    0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
    0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
    0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
    0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
    0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
    0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};

static inline uint32_t ror32(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }

static void sha256_blocks_portable(uint32_t st[8], const uint8_t* p, size_t nblk) {
    uint32_t w[64];
    while (nblk--) {
        for (int i = 0; i < 16; ++i)
            w[i] = ((uint32_t)p[4 * i] << 24) | ((uint32_t)p[4 * i + 1] << 16) | ((uint32_t)p[4 * i + 2] << 8) | p[4 * i + 3];
        for (int i = 16; i < 64; ++i) {
            uint32_t s0 = ror32(w[i - 15], 7) ^ ror32(w[i - 15], 18) ^ (w[i - 15] >> 3);
            uint32_t s1 = ror32(w[i - 2], 17) ^ ror32(w[i - 2], 19) ^ (w[i - 2] >> 10);
            w[i] = w[i - 16] + s0 + w[i - 7] + s1;
        }
        uint32_t a = st[0], b = st[1], c = st[2], d = st[3], e = st[4], f = st[5], g = st[6], h = st[7];
        for (int i = 0; i < 64; ++i) {
            uint32_t t1 = h + (ror32(e, 6) ^ ror32(e, 11) ^ ror32(e, 25)) + ((e & f) ^ (~e & g)) + K256[i] + w[i];
            uint32_t t2 = (ror32(a, 2) ^ ror32(a, 13) ^ ror32(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
            h = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
        }
        st[0] += a; st[1] += b; st[2] += c; st[3] += d; st[4] += e; st[5] += f; st[6] += g; st[7] += h;
        p += 64;
    }
}

#if ORC_X86
__attribute__((target("sha,sse4.1,ssse3")))
static void sha256_blocks_shani(uint32_t st[8], const uint8_t* p, size_t nblk) {
    const __m128i bswap = _mm_set_epi64x(0x0c0d0e0f08090a0bULL, 0x0405060700010203ULL);
    __m128i tmp = _mm_loadu_si128((const __m128i*)&st[0]);      /* DCBA */
    __m128i s1 = _mm_loadu_si128((const __m128i*)&st[4]);       /* HGFE */
    tmp = _mm_shuffle_epi32(tmp, 0xB1);                          /* CDAB */
    s1 = _mm_shuffle_epi32(s1, 0x1B);                            /* EFGH */
    __m128i s0 = _mm_alignr_epi8(tmp, s1, 8);                    /* ABEF */
    s1 = _mm_blend_epi16(s1, tmp, 0xF0);                         /* CDGH */
    while (nblk--) {
        const __m128i save0 = s0, save1 = s1;
        __m128i m[4];
        for (int i = 0; i < 4; ++i) m[i] = _mm_shuffle_epi8(_mm_loadu_si128((const __m128i*)(p + 16 * i)), bswap);
        for (int r = 0; r < 16; ++r) {
            __m128i cur = m[r & 3];
            __m128i wk = _mm_add_epi32(cur, _mm_loadu_si128((const __m128i*)&K256[4 * r]));
            s1 = _mm_sha256rnds2_epu32(s1, s0, wk);
            wk = _mm_shuffle_epi32(wk, 0x0E);
            s0 = _mm_sha256rnds2_epu32(s0, s1, wk);
            if (r < 12) {
                /* schedule words 4(r+4) .. 4(r+4)+3 from the four most recent groups */
                __m128i w0 = m[r & 3], w1 = m[(r + 1) & 3], w2 = m[(r + 2) & 3], w3 = m[(r + 3) & 3];
                __m128i x = _mm_sha256msg1_epu32(w0, w1);
                x = _mm_add_epi32(x, _mm_alignr_epi8(w3, w2, 4));
                m[r & 3] = _mm_sha256msg2_epu32(x, w3);
            }
        }
        s0 = _mm_add_epi32(s0, save0);
        s1 = _mm_add_epi32(s1, save1);
        p += 64;
    }
    tmp = _mm_shuffle_epi32(s0, 0x1B);                           /* FEBA */
    s1 = _mm_shuffle_epi32(s1, 0xB1);                            /* DCHG */
    s0 = _mm_blend_epi16(tmp, s1, 0xF0);                         /* DCBA */
    s1 = _mm_alignr_epi8(s1, tmp, 8);                            /* HGFE */
    _mm_storeu_si128((__m128i*)&st[0], s0);
    _mm_storeu_si128((__m128i*)&st[4], s1);
}

static int have_shani(void) {
    static int cached = -1;
    if (cached < 0) {
        unsigned a, b, c, d;
        cached = 0;
        if (__get_cpuid_count(7, 0, &a, &b, &c, &d)) cached = (b >> 29) & 1;
        if (cached) {
            if (__get_cpuid(1, &a, &b, &c, &d)) cached = ((c >> 19) & 1) && ((c >> 9) & 1); /* sse4.1, ssse3 */
        }
    }
    return cached;
}
#endif

int orc_sha256_uses_shani(void) {
#if ORC_X86
    return have_shani();
#else
    return 0;
#endif
}

static void sha256_blocks(uint32_t st[8], const uint8_t* p, size_t nblk) {
#if ORC_X86
    if (have_shani()) { sha256_blocks_shani(st, p, nblk); return; }
#endif
    sha256_blocks_portable(st, p, nblk);
}

static void sha256(const uint8_t* data, uint64_t len, uint8_t out[32]) {
    uint32_t st[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a, 0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
    size_t nblk = (size_t)(len / 64);
    sha256_blocks(st, data, nblk);
    uint8_t tail[128];
    size_t rem = (size_t)(len % 64);
    memset(tail, 0, sizeof(tail));
    if (rem) memcpy(tail, data + 64 * nblk, rem);
    tail[rem] = 0x80;
    size_t tl = rem < 56 ? 64 : 128;
    uint64_t bits = len * 8;
    for (int i = 0; i < 8; ++i) tail[tl - 1 - i] = (uint8_t)(bits >> (8 * i));
    sha256_blocks(st, tail, tl / 64);
    for (int i = 0; i < 8; ++i) {
        out[4 * i] = (uint8_t)(st[i] >> 24); out[4 * i + 1] = (uint8_t)(st[i] >> 16);
        out[4 * i + 2] = (uint8_t)(st[i] >> 8); out[4 * i + 3] = (uint8_t)st[i];
    }
}

/* ------------------------------------------------------------------ BLAKE2b */

static const uint64_t B2_IV[8] = {0x6a09e667f3bcc908ULL, 0xbb67ae8584caa73bULL, 0x3c6ef372fe94f82bULL,
                                  0xa54ff53a5f1d36f1ULL, 0x510e527fade682d1ULL, 0x9b05688c2b3e6c1fULL,
                                  0x1f83d9abfb41bd6bULL, 0x5be0cd19137e2179ULL};
static const uint8_t B2_SIGMA[12][16] = {
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
    {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4}, {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
    {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13}, {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
    {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11}, {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
    {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5}, {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};

static inline uint64_t ror64(uint64_t x, int n) { return (x >> n) | (x << (64 - n)); }

static void b2_compress(uint64_t h[8], const uint8_t blk[128], uint64_t t, int last) {
    uint64_t m[16], v[16];
    memcpy(m, blk, 128); /* little-endian host */
    for (int i = 0; i < 8; ++i) { v[i] = h[i]; v[8 + i] = B2_IV[i]; }
    v[12] ^= t;
    if (last) v[14] = ~v[14];
    for (int r = 0; r < 12; ++r) {
        const uint8_t* s = B2_SIGMA[r];
#define B2G(a, b, c, d, x, y)                                          \
        v[a] += v[b] + m[x]; v[d] = ror64(v[d] ^ v[a], 32);            \
        v[c] += v[d];        v[b] = ror64(v[b] ^ v[c], 24);            \
        v[a] += v[b] + m[y]; v[d] = ror64(v[d] ^ v[a], 16);            \
        v[c] += v[d];        v[b] = ror64(v[b] ^ v[c], 63);
        B2G(0, 4, 8, 12, s[0], s[1]) B2G(1, 5, 9, 13, s[2], s[3]) B2G(2, 6, 10, 14, s[4], s[5]) B2G(3, 7, 11, 15, s[6], s[7])
        B2G(0, 5, 10, 15, s[8], s[9]) B2G(1, 6, 11, 12, s[10], s[11]) B2G(2, 7, 8, 13, s[12], s[13]) B2G(3, 4, 9, 14, s[14], s[15])
#undef B2G
    }
    for (int i = 0; i < 8; ++i) h[i] ^= v[i] ^ v[8 + i];
}

/* BLAKE2b-512 over prefix || data (prefix may be empty) */
static void blake2b_2part(const uint8_t* pre, size_t pre_len, const uint8_t* data, uint64_t len, uint8_t out[64]) {
    uint64_t h[8];
    for (int i = 0; i < 8; ++i) h[i] = B2_IV[i];
    h[0] ^= 0x01010040ULL;
    uint8_t buf[128];
    size_t fill = 0;
    uint64_t t = 0;
    /* buffer-and-flush: a block is compressed only when more input follows it */
    const uint8_t* parts[2] = {pre, data};
    uint64_t lens[2] = {pre_len, len};
    for (int k = 0; k < 2; ++k) {
        const uint8_t* p = parts[k];
        uint64_t n = lens[k];
        while (n) {
            if (fill == 128) { t += 128; b2_compress(h, buf, t, 0); fill = 0; }
            size_t take = 128 - fill;
            if (take > n) take = (size_t)n;
            memcpy(buf + fill, p, take);
            fill += take; p += take; n -= take;
        }
    }
    t += fill;
    memset(buf + fill, 0, 128 - fill);
    b2_compress(h, buf, t, 1);
    memcpy(out, h, 64);
}

/* ------------------------------------------------------------------ SHA3-256 */

static const uint64_t KECCAK_RC[24] = {
    0x0000000000000001ULL, 0x0000000000008082ULL, 0x800000000000808aULL, 0x8000000080008000ULL,
    0x000000000000808bULL, 0x0000000080000001ULL, 0x8000000080008081ULL, 0x8000000000008009ULL,
    0x000000000000008aULL, 0x0000000000000088ULL, 0x0000000080008009ULL, 0x000000008000000aULL,
    0x000000008000808bULL, 0x800000000000008bULL, 0x8000000000008089ULL, 0x8000000000008003ULL,
    0x8000000000008002ULL, 0x8000000000000080ULL, 0x000000000000800aULL, 0x800000008000000aULL,
    0x8000000080008081ULL, 0x8000000000008080ULL, 0x0000000080000001ULL, 0x8000000080008008ULL};
static const int KECCAK_ROT[24] = {1, 3, 6, 10, 15, 21, 28, 36, 45, 55, 2, 14, 27, 41, 56, 8, 25, 43, 62, 18, 39, 61, 20, 44};
static const int KECCAK_PIL[24] = {10, 7, 11, 17, 18, 3, 5, 16, 8, 21, 24, 4, 15, 23, 19, 13, 12, 2, 20, 14, 22, 9, 6, 1};

static void keccak_f(uint64_t s[25]) {
    for (int round = 0; round < 24; ++round) {
        uint64_t bc[5];
        for (int i = 0; i < 5; ++i) bc[i] = s[i] ^ s[i + 5] ^ s[i + 10] ^ s[i + 15] ^ s[i + 20];
        for (int i = 0; i < 5; ++i) {
            uint64_t t = bc[(i + 4) % 5] ^ ((bc[(i + 1) % 5] << 1) | (bc[(i + 1) % 5] >> 63));
            for (int j = 0; j < 25; j += 5) s[j + i] ^= t;
        }
        uint64_t t = s[1];
        for (int i = 0; i < 24; ++i) {
            int j = KECCAK_PIL[i];
            uint64_t x = s[j];
            s[j] = (t << KECCAK_ROT[i]) | (t >> (64 - KECCAK_ROT[i]));
            t = x;
        }
        for (int j = 0; j < 25; j += 5) {
            for (int i = 0; i < 5; ++i) bc[i] = s[j + i];
            for (int i = 0; i < 5; ++i) s[j + i] ^= (~bc[(i + 1) % 5]) & bc[(i + 2) % 5];
        }
        s[0] ^= KECCAK_RC[round];
    }
}

static void sha3_256(const uint8_t* data, uint64_t len, uint8_t out[32]) {
    uint64_t s[25];
    memset(s, 0, sizeof(s));
    const size_t rate = 136;
    while (len >= rate) {
        uint64_t lane[17];
        memcpy(lane, data, rate);
        for (int i = 0; i < 17; ++i) s[i] ^= lane[i];
        keccak_f(s);
        data += rate; len -= rate;
    }
    uint8_t tail[136];
    memset(tail, 0, rate);
    if (len) memcpy(tail, data, (size_t)len);
    tail[len] ^= 0x06;
    tail[rate - 1] ^= 0x80;
    uint64_t lane[17];
    memcpy(lane, tail, rate);
    for (int i = 0; i < 17; ++i) s[i] ^= lane[i];
    keccak_f(s);
    memcpy(out, s, 32);
}

/* ------------------------------------------------------------------ dispatch */

static void hash_one(int alg, const uint8_t* data, uint64_t len, uint8_t* out) {
    switch (alg) {
        case ORC_SHA256: sha256(data, len, out); break;
        case ORC_BLAKE2B: blake2b_2part(NULL, 0, data, len, out); break;
        default: sha3_256(data, len, out); break;
    }
}

int orc_hash(int alg, const uint8_t* data, uint64_t len, uint8_t* out) {
    if (alg < 0 || alg > 2) return -1;
    hash_one(alg, data, len, out);
    return 0;
}

/* BLAKE2b(tag || data), lattice.py:97-101 */
int orc_lt_hash_tagged(const uint8_t* tag, uint64_t tag_len, const uint8_t* data, uint64_t len, uint8_t* out) {
    blake2b_2part(tag, (size_t)tag_len, data, len, out);
    return 0;
}

/* ------------------------------------------------------------------ worker pool (workers.py:30-57) */

typedef void (*range_fn)(void* ctx, uint64_t begin, uint64_t end, int worker);

typedef struct {
    range_fn fn;
    void* ctx;
    uint64_t begin, end;
    int worker;
} job_t;

static void* job_main(void* arg) {
    job_t* j = (job_t*)arg;
    j->fn(j->ctx, j->begin, j->end, j->worker);
    return NULL;
}

/* contiguous ranges, sizes differing by at most one; results written by index */
static int run_chunked(uint64_t n, int workers, range_fn fn, void* ctx) {
    if (n == 0) return 0;
    if (workers < 1) workers = 1;
    if ((uint64_t)workers > n) workers = (int)n;
    if (workers == 1) { fn(ctx, 0, n, 0); return 0; }
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * workers);
    job_t* jobs = (job_t*)malloc(sizeof(job_t) * workers);
    if (!th || !jobs) { free(th); free(jobs); return -1; }
    uint64_t base = n / workers, extra = n % workers, start = 0;
    for (int i = 0; i < workers; ++i) {
        uint64_t stop = start + base + ((uint64_t)i < extra ? 1 : 0);
        jobs[i].fn = fn; jobs[i].ctx = ctx; jobs[i].begin = start; jobs[i].end = stop; jobs[i].worker = i;
        start = stop;
    }
    int started = 0;
    for (; started < workers; ++started)
        if (pthread_create(&th[started], NULL, job_main, &jobs[started]) != 0) break;
    for (int i = started; i < workers; ++i) job_main(&jobs[i]);   /* fall back to inline */
    for (int i = 0; i < started; ++i) pthread_join(th[i], NULL);
    free(th); free(jobs);
    return 0;
}

/* ------------------------------------------------------------------ merkle */

typedef struct {
    int alg;
    const uint8_t* base;
    const uint64_t* off;
    const uint64_t* len;
    uint8_t* out;
} blocks_ctx;

static void blocks_range(void* c, uint64_t a, uint64_t b, int w) {
    (void)w;
    blocks_ctx* x = (blocks_ctx*)c;
    int dl = digest_len(x->alg);
    for (uint64_t i = a; i < b; ++i) hash_one(x->alg, x->base + x->off[i], x->len[i], x->out + i * dl);
}

int orc_hash_blocks(int alg, const uint8_t* base, const uint64_t* off, const uint64_t* len, uint64_t n, uint8_t* out, int threads) {
    if (alg < 0 || alg > 2 || n == 0) return -1;
    blocks_ctx c = {alg, base, off, len, out};
    return run_chunked(n, threads, blocks_range, &c);
}

typedef struct {
    int alg;
    const uint8_t* in;
    uint64_t count;
    uint8_t* out;
} level_ctx;

static void level_range(void* c, uint64_t a, uint64_t b, int w) {
    (void)w;
    level_ctx* x = (level_ctx*)c;
    int dl = digest_len(x->alg);
    uint8_t msg[128];
    for (uint64_t j = a; j < b; ++j) {
        memcpy(msg, x->in + 2 * j * dl, dl);
        if (2 * j + 1 < x->count) memcpy(msg + dl, x->in + (2 * j + 1) * dl, dl);
        else memset(msg + dl, 0, dl);                       /* zero padding node, merkle.py:131,139-140 */
        hash_one(x->alg, msg, 2 * (uint64_t)dl, x->out + j * dl);
    }
}

int orc_merkle_root(int alg, const uint8_t* leaves, uint64_t count, uint8_t* root, int threads) {
    if (alg < 0 || alg > 2 || count == 0) return -1;
    int dl = digest_len(alg);
    if (count == 1) { memcpy(root, leaves, dl); return 0; } /* merkle.py:159-160 */
    uint64_t cap = (count + 1) / 2;
    uint8_t* a = (uint8_t*)malloc(cap * dl);
    uint8_t* b = (uint8_t*)malloc(((cap + 1) / 2 + 1) * dl);
    if (!a || !b) { free(a); free(b); return -1; }
    const uint8_t* in = leaves;
    uint8_t* outb = a;
    while (count > 1) {
        level_ctx c = {alg, in, count, outb};
        run_chunked((count + 1) / 2, threads, level_range, &c);
        count = (count + 1) / 2;
        in = outb;
        outb = (outb == a) ? b : a;
    }
    memcpy(root, in, dl);
    free(a); free(b);
    return 0;
}

/* ------------------------------------------------------------------ in-place model (model.py:137-146, 298-315) */

uint64_t orc_leaf_count(const uint64_t* nbytes, uint32_t n_tensors, uint32_t block_size) {
    uint64_t k = 0;
    for (uint32_t t = 0; t < n_tensors; ++t) k += (nbytes[t] + block_size - 1) / block_size;
    return k;
}

typedef struct {
    int alg;
    const uint8_t* const* tensors;
    const uint64_t* nbytes;
    const uint64_t* first;     /* first leaf of tensor t; n_tensors + 1 entries */
    uint32_t n_tensors;
    uint32_t block_size;
    uint8_t* out;              /* leaf digests, or NULL */
    uint16_t* lanes;           /* per-worker 32 lanes (lattice), or NULL */
} leaves_ctx;

static uint32_t tensor_of(const leaves_ctx* x, uint64_t k) {
    uint32_t lo = 0, hi = x->n_tensors;
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) / 2;
        if (x->first[mid] <= k) lo = mid; else hi = mid;
    }
    return lo;
}

static void leaves_range(void* c, uint64_t a, uint64_t b, int w) {
    leaves_ctx* x = (leaves_ctx*)c;
    int dl = digest_len(x->alg);
    uint32_t t = tensor_of(x, a);
    for (uint64_t k = a; k < b; ++k) {
        while (x->first[t + 1] <= k) ++t;                   /* skips empty tensors */
        uint64_t off = (k - x->first[t]) * x->block_size;
        uint64_t len = x->nbytes[t] - off;
        if (len > x->block_size) len = x->block_size;       /* ragged tail hashed at true length */
        const uint8_t* p = x->tensors[t] + off;
        if (x->out) {
            hash_one(x->alg, p, len, x->out + k * dl);
        } else {
            uint8_t tag[8], d[64];
            for (int i = 0; i < 8; ++i) tag[i] = (uint8_t)(k >> (8 * i));   /* LE64(k), model.py:312 */
            blake2b_2part(tag, 8, p, len, d);
            uint16_t* acc = x->lanes + 32 * (size_t)w;
            for (int i = 0; i < 32; ++i) acc[i] = (uint16_t)(acc[i] + (uint16_t)(d[2 * i] | (d[2 * i + 1] << 8)));
        }
    }
}

static uint64_t* build_first(const uint64_t* nbytes, uint32_t n, uint32_t bs) {
    uint64_t* first = (uint64_t*)malloc(sizeof(uint64_t) * ((size_t)n + 1));
    if (!first) return NULL;
    uint64_t k = 0;
    for (uint32_t t = 0; t < n; ++t) { first[t] = k; k += (nbytes[t] + bs - 1) / bs; }
    first[n] = k;
    return first;
}

int orc_inplace_leaves(int alg, const uint8_t* const* tensors, const uint64_t* nbytes, uint32_t n_tensors,
                       uint32_t block_size, uint8_t* leaves_out, int threads) {
    if (alg < 0 || alg > 2 || n_tensors == 0) return -1;
    uint64_t* first = build_first(nbytes, n_tensors, block_size);
    if (!first) return -1;
    uint64_t n = first[n_tensors];
    if (n == 0) { free(first); return -1; }
    leaves_ctx c = {alg, tensors, nbytes, first, n_tensors, block_size, leaves_out, NULL};
    int rc = run_chunked(n, threads, leaves_range, &c);
    free(first);
    return rc;
}

int orc_inplace_merkle(int alg, const uint8_t* const* tensors, const uint64_t* nbytes, uint32_t n_tensors,
                       uint32_t block_size, uint8_t* root, int threads) {
    uint64_t n = orc_leaf_count(nbytes, n_tensors, block_size);
    if (n == 0) return -1;
    uint8_t* leaves = (uint8_t*)malloc(n * digest_len(alg));
    if (!leaves) return -1;
    int rc = orc_inplace_leaves(alg, tensors, nbytes, n_tensors, block_size, leaves, threads);
    if (rc == 0) rc = orc_merkle_root(alg, leaves, n, root, threads);
    free(leaves);
    return rc;
}

int orc_inplace_lattice(const uint8_t* const* tensors, const uint64_t* nbytes, uint32_t n_tensors,
                        uint32_t block_size, uint8_t out[64], int threads) {
    if (n_tensors == 0) return -1;
    uint64_t* first = build_first(nbytes, n_tensors, block_size);
    if (!first) return -1;
    uint64_t n = first[n_tensors];
    if (threads < 1) threads = 1;
    uint16_t* lanes = (uint16_t*)calloc((size_t)threads * 32, sizeof(uint16_t));
    if (!lanes) { free(first); return -1; }
    leaves_ctx c = {ORC_BLAKE2B, tensors, nbytes, first, n_tensors, block_size, NULL, lanes};
    int rc = run_chunked(n, threads, leaves_range, &c);
    uint16_t sum[32];
    memset(sum, 0, sizeof(sum));
    for (int w = 0; w < threads; ++w)
        for (int i = 0; i < 32; ++i) sum[i] = (uint16_t)(sum[i] + lanes[32 * (size_t)w + i]);
    for (int i = 0; i < 32; ++i) { out[2 * i] = (uint8_t)sum[i]; out[2 * i + 1] = (uint8_t)(sum[i] >> 8); }
    free(lanes); free(first);
    return rc;
}

/* ------------------------------------------------------------------ dataset LtHash (dataset.py:41-49, 74-91) */

typedef struct {
    const uint8_t* shard;
    const uint64_t* off;
    const uint64_t* len;
    const uint64_t* ids;
    const uint32_t* slot;
    uint32_t n_sources;
    uint16_t* lanes;      /* per worker: n_sources x 32 */
    uint64_t* counts;     /* per worker: n_sources */
    uint8_t* digests;     /* optional n x 64 */
    int bad;
} lt_ctx;

static void lt_range(void* c, uint64_t a, uint64_t b, int w) {
    lt_ctx* x = (lt_ctx*)c;
    uint16_t* lanes = x->lanes + (size_t)w * x->n_sources * 32;
    uint64_t* counts = x->counts + (size_t)w * x->n_sources;
    for (uint64_t i = a; i < b; ++i) {
        if (x->slot[i] >= x->n_sources) { x->bad = 1; continue; }
        uint8_t tag[8], d[64];
        for (int k = 0; k < 8; ++k) tag[k] = (uint8_t)(x->ids[i] >> (8 * k));
        blake2b_2part(tag, 8, x->shard + x->off[i], x->len[i], d);
        if (x->digests) memcpy(x->digests + i * 64, d, 64);
        uint16_t* acc = lanes + 32 * (size_t)x->slot[i];
        for (int k = 0; k < 32; ++k) acc[k] = (uint16_t)(acc[k] + (uint16_t)(d[2 * k] | (d[2 * k + 1] << 8)));
        counts[x->slot[i]] += 1;
    }
}

/* sums: n_sources x 32 u16 lanes (little-endian host), counts: n_sources. Both are overwritten. */
int orc_lthash_samples(const uint8_t* shard, const uint64_t* off, const uint64_t* len, const uint64_t* ids,
                       const uint32_t* slot, uint64_t n, uint32_t n_sources, uint16_t* sums, uint64_t* counts,
                       uint8_t* digests, int threads) {
    if (n_sources == 0) return -1;
    if (threads < 1) threads = 1;
    uint16_t* lanes = (uint16_t*)calloc((size_t)threads * n_sources * 32, sizeof(uint16_t));
    uint64_t* cnt = (uint64_t*)calloc((size_t)threads * n_sources, sizeof(uint64_t));
    if (!lanes || !cnt) { free(lanes); free(cnt); return -1; }
    lt_ctx c = {shard, off, len, ids, slot, n_sources, lanes, cnt, digests, 0};
    int rc = run_chunked(n, threads, lt_range, &c);
    memset(sums, 0, sizeof(uint16_t) * n_sources * 32);
    memset(counts, 0, sizeof(uint64_t) * n_sources);
    for (int w = 0; w < threads; ++w) {                     /* commutative merge, dataset.py:67-71 */
        for (size_t i = 0; i < (size_t)n_sources * 32; ++i) sums[i] = (uint16_t)(sums[i] + lanes[(size_t)w * n_sources * 32 + i]);
        for (size_t i = 0; i < n_sources; ++i) counts[i] += cnt[(size_t)w * n_sources + i];
    }
    free(lanes); free(cnt);
    if (rc == 0 && c.bad) rc = -4;                          /* undeclared source, dataset.py:78-80 */
    return rc;
}
