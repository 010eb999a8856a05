// SHA-256 (FIPS 180-4) for one thread: state and the rolling 16-word message
// schedule live in registers; rounds are fully unrolled so every K[t] becomes
// an immediate operand.
//
// Pipe placement (tools/pipe_mix.cu, tools/sha_variants.cu, profiles/r1s2_*): the rotations, shifts
// and three-input logic ops can only run on the ALU pipe (SHF / LOP3, 64 lanes/clk/SM), which is what
// bounds the kernel. Every addition is therefore issued as an IMAD on the FMA pipe. The two pipes
// issue concurrently only while the register file keeps up: it delivers about two vector operands
// per cycle per scheduler, a three-vector-register instruction takes two read cycles, and a pair
// (ALU op, IMAD) that reads more than four vector registers no longer dual-issues (pipe_mix: 36 Tops/s
// for 2+2 operands, 24 for 3+3). So the IMADs are written to read at most two vector registers:
// a + b  = a * ONE.u + b   with ONE.u = 1 in a *uniform* register (kernel parameter), and
// K + h  = ONE.v * K + h   with ONE.v = 1 in a per-thread register and K in the immediate slot.
//
// Role in the reference: the arithmetic hashlib.sha256 performs for
// compression.py:45-49 / merkle.py:106-110 (leaf) and merkle.py:134-144 (node).
#pragma once
#include "common.cuh"

namespace snt {

#define SNT_SHA256_K                                                                            \
    0x428a2f98u, 0x71374491u, 0xb5c0fbcfu, 0xe9b5dba5u, 0x3956c25bu, 0x59f111f1u, 0x923f82a4u, \
    0xab1c5ed5u, 0xd807aa98u, 0x12835b01u, 0x243185beu, 0x550c7dc3u, 0x72be5d74u, 0x80deb1feu, \
    0x9bdc06a7u, 0xc19bf174u, 0xe49b69c1u, 0xefbe4786u, 0x0fc19dc6u, 0x240ca1ccu, 0x2de92c6fu, \
    0x4a7484aau, 0x5cb0a9dcu, 0x76f988dau, 0x983e5152u, 0xa831c66du, 0xb00327c8u, 0xbf597fc7u, \
    0xc6e00bf3u, 0xd5a79147u, 0x06ca6351u, 0x14292967u, 0x27b70a85u, 0x2e1b2138u, 0x4d2c6dfcu, \
    0x53380d13u, 0x650a7354u, 0x766a0abbu, 0x81c2c92eu, 0x92722c85u, 0xa2bfe8a1u, 0xa81a664bu, \
    0xc24b8b70u, 0xc76c51a3u, 0xd192e819u, 0xd6990624u, 0xf40e3585u, 0x106aa070u, 0x19a4c116u, \
    0x1e376c08u, 0x2748774cu, 0x34b0bcb5u, 0x391c0cb3u, 0x4ed8aa4au, 0x5b9cca4fu, 0x682e6ff3u, \
    0x748f82eeu, 0x78a5636fu, 0x84c87814u, 0x8cc70208u, 0x90befffau, 0xa4506cebu, 0xbef9a3f7u, \
    0xc67178f2u

#if defined(__CUDACC__)
__constant__ uint32_t c_sha256_k[64] = {SNT_SHA256_K};      // for the rolled compression (compress_rolled)
#endif

struct Sha256 {
    static constexpr int DIGEST_BYTES = 32;
    static constexpr int STATE_WORDS = 8;     // 32-bit words carried between compressions
    static constexpr int BLOCK_BYTES = 64;

    SNT_HD static uint32_t bsig0(uint32_t x) { return rotr32(x, 2) ^ rotr32(x, 13) ^ rotr32(x, 22); }
    SNT_HD static uint32_t bsig1(uint32_t x) { return rotr32(x, 6) ^ rotr32(x, 11) ^ rotr32(x, 25); }
    SNT_HD static uint32_t ssig0(uint32_t x) { return rotr32(x, 7) ^ rotr32(x, 18) ^ (x >> 3); }
    SNT_HD static uint32_t ssig1(uint32_t x) { return rotr32(x, 17) ^ rotr32(x, 19) ^ (x >> 10); }
    SNT_HD static uint32_t ch(uint32_t e, uint32_t f, uint32_t g) { return (e & f) ^ (~e & g); }
    SNT_HD static uint32_t maj(uint32_t a, uint32_t b, uint32_t c) { return (a & b) ^ (a & c) ^ (b & c); }

    // The runtime 1 the compiler cannot fold, in the two register classes the IMAD forms need:
    // `u` comes straight from the kernel parameter block (uniform register or constant operand),
    // `v` is loaded per thread (vector register). On the host both are plain 1.
    struct One {
        uint32_t u, v;
        SNT_HD One() : u(1u), v(1u) {}
        SNT_HD One(uint32_t uu, uint32_t vv) : u(uu), v(vv) {}
    };

    // a + b on the FMA pipe: IMAD R, Ra, UR(one), Rb -- two vector operands.
    SNT_HD static uint32_t add_fma(uint32_t a, uint32_t b, uint32_t one_u) {
#ifdef __CUDA_ARCH__
        uint32_t r;
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(one_u), "r"(b));
        return r;
#else
        return a * one_u + b;
#endif
    }
    // k + x on the FMA pipe with k a compile-time constant (immediate) or a constant-bank word:
    // IMAD R, R(one), k, Rx -- `one_v` must live in a vector register for this encoding to exist.
    SNT_HD static uint32_t addk_fma(uint32_t k, uint32_t x, uint32_t one_v) {
#ifdef __CUDA_ARCH__
        uint32_t r;
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(one_v), "r"(k), "r"(x));
        return r;
#else
        return one_v * k + x;
#endif
    }

    // One round with every addition on the FMA pipe; kw is K[t] (+ W[t] for a constant block).
    SNT_HD static void round_fma(uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d, uint32_t& e, uint32_t& f,
                                 uint32_t& g, uint32_t& h, uint32_t kw, const uint32_t* w, const One& one) {
        uint32_t hk = addk_fma(kw, h, one.v);
        if (w) hk = add_fma(hk, *w, one.u);
        const uint32_t t1 = add_fma(hk, add_fma(bsig1(e), ch(e, f, g), one.u), one.u);
        const uint32_t t2 = add_fma(bsig0(a), maj(a, b, c), one.u);
        h = g; g = f; f = e; e = add_fma(d, t1, one.u); d = c; c = b; b = a; a = add_fma(t1, t2, one.u);
    }

    SNT_HD static void init(uint32_t s[8]) {
        s[0] = 0x6a09e667u; s[1] = 0xbb67ae85u; s[2] = 0x3c6ef372u; s[3] = 0xa54ff53au;
        s[4] = 0x510e527fu; s[5] = 0x9b05688cu; s[6] = 0x1f83d9abu; s[7] = 0x5be0cd19u;
    }


    // One compression. w[16] holds the block as big-endian-decoded words and
    // is overwritten by the rolling schedule.
    SNT_HD static void compress(uint32_t s[8], uint32_t w[16], const One& one = One()) {
        const uint32_t K[64] = {SNT_SHA256_K};
        uint32_t a = s[0], b = s[1], c = s[2], d = s[3], e = s[4], f = s[5], g = s[6], h = s[7];
#pragma unroll
        for (int t = 0; t < 64; ++t) {
            if (t >= 16) {
                const uint32_t x = add_fma(w[t & 15], w[(t - 7) & 15], one.u);
                const uint32_t y = add_fma(ssig1(w[(t - 2) & 15]), ssig0(w[(t - 15) & 15]), one.u);
                w[t & 15] = add_fma(x, y, one.u);
            }
            round_fma(a, b, c, d, e, f, g, h, K[t], &w[t & 15], one);
        }
        s[0] += a; s[1] += b; s[2] += c; s[3] += d; s[4] += e; s[5] += f; s[6] += g; s[7] += h;
    }

    // One compression with the rounds rolled four times over a 16-round body and the round constants
    // read from a table: a quarter of the code of compress() (7 KB instead of 26 KB). For the cold paths
    // that share a kernel with the unrolled leaf loop (tree nodes, closing blocks, leaves at odd addresses)
    // and must not push that loop out of the instruction cache.
    SNT_HD static void compress_rolled(uint32_t s[8], uint32_t w[16]) {
#ifdef __CUDA_ARCH__
        const uint32_t* K = c_sha256_k;
#else
        static const uint32_t K[64] = {SNT_SHA256_K};
#endif
        uint32_t a = s[0], b = s[1], c = s[2], d = s[3], e = s[4], f = s[5], g = s[6], h = s[7];
#pragma unroll 1
        for (int t0 = 0; t0 < 64; t0 += 16) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                if (t0) w[i] += ssig1(w[(i + 14) & 15]) + w[(i + 9) & 15] + ssig0(w[(i + 1) & 15]);
                const uint32_t t1 = h + bsig1(e) + ch(e, f, g) + K[t0 + i] + w[i];
                const uint32_t t2 = bsig0(a) + maj(a, b, c);
                h = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
            }
        }
        s[0] += a; s[1] += b; s[2] += c; s[3] += d; s[4] += e; s[5] += f; s[6] += g; s[7] += h;
    }

    // Compression of a block that is the same for every message of a given
    // length (the padding block of a block-multiple message): kw[t] = K[t] +
    // W[t] is precomputed on the host, so only the 64 rounds remain.
    SNT_HD static void compress_const(uint32_t s[8], const uint32_t* __restrict__ kw, const One& one = One()) {
        uint32_t a = s[0], b = s[1], c = s[2], d = s[3], e = s[4], f = s[5], g = s[6], h = s[7];
#pragma unroll
        for (int t = 0; t < 64; ++t) round_fma(a, b, c, d, e, f, g, h, kw[t], nullptr, one);
        s[0] += a; s[1] += b; s[2] += c; s[3] += d; s[4] += e; s[5] += f; s[6] += g; s[7] += h;
    }

    // Host helper: K[t] + W[t] for the padding block that follows a message of
    // `msg_bytes` bytes when msg_bytes is a multiple of 64.
    static inline void pad_schedule(uint64_t msg_bytes, uint32_t kw[64]) {
        const uint32_t K[64] = {SNT_SHA256_K};
        uint32_t w[64];
        w[0] = 0x80000000u;
        for (int i = 1; i < 14; ++i) w[i] = 0;
        const uint64_t bits = msg_bytes * 8;
        w[14] = static_cast<uint32_t>(bits >> 32);
        w[15] = static_cast<uint32_t>(bits);
        for (int t = 16; t < 64; ++t) {
            const uint32_t x = w[t - 15], y = w[t - 2];
            const uint32_t s0 = ((x >> 7) | (x << 25)) ^ ((x >> 18) | (x << 14)) ^ (x >> 3);
            const uint32_t s1 = ((y >> 17) | (y << 15)) ^ ((y >> 19) | (y << 13)) ^ (y >> 10);
            w[t] = w[t - 16] + s0 + w[t - 7] + s1;
        }
        for (int t = 0; t < 64; ++t) kw[t] = K[t] + w[t];
    }

    // The one or two closing blocks of a message of `len` bytes whose last `rem` (< 64) bytes start at t
    // (any alignment): the tail bytes, 0x80, zeros, the 64-bit big-endian bit length.
    SNT_HD static void finish(const uint8_t* t, uint32_t rem, uint64_t len, uint32_t s[8], const One& one = One()) {
        const uint64_t bits = len << 3;
        const int nb = rem >= 56 ? 2 : 1;
#pragma unroll 1
        for (int b = 0; b < nb; ++b) {
            uint32_t w[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                uint32_t v = 0;
                if (b == 0) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint32_t idx = 4 * i + j;
                        uint32_t byte = tail_byte(t, idx, rem);
                        if (idx == rem) byte = 0x80u;
                        v = (v << 8) | byte;
                    }
                }
                w[i] = v;
            }
            if (b == nb - 1) {
                w[14] = static_cast<uint32_t>(bits >> 32);
                w[15] = static_cast<uint32_t>(bits);
            }
            compress(s, w, one);
        }
    }

    // Whole message at p[0..len), any alignment, any length (generic path): the full 64-byte blocks,
    // then the closing blocks.
    SNT_HD static void hash_message(const uint8_t* p, uint64_t len, uint32_t s[8], const One& one = One()) {
        init(s);
        const uint64_t nfull = len >> 6;
        for (uint64_t b = 0; b < nfull; ++b) {
            uint32_t w[16];
            load_words<16>(p + (b << 6), w);
#pragma unroll
            for (int i = 0; i < 16; ++i) w[i] = bswap32(w[i]);
            compress(s, w, one);
        }
        finish(p + (nfull << 6), static_cast<uint32_t>(len & 63), len, s, one);
    }

    // Tree node: H(left || right) where both children are given as state
    // words (= the digest read as big-endian words). 64-byte message: one
    // data compression plus the constant padding block.
    SNT_HD static void hash_pair(const uint32_t l[8], const uint32_t r[8],
                                 const uint32_t* __restrict__ pad64_kw, uint32_t out[8], const One& one = One()) {
        uint32_t w[16];
#pragma unroll
        for (int i = 0; i < 8; ++i) { w[i] = l[i]; w[8 + i] = r[i]; }
        uint32_t s[8];
        init(s);
        compress(s, w, one);
        compress_const(s, pad64_kw, one);
#pragma unroll
        for (int i = 0; i < 8; ++i) out[i] = s[i];
    }

    // hash_pair with the rolled compression: the second block is the padding of a 64-byte message.
    SNT_HD static void hash_pair_rolled(const uint32_t l[8], const uint32_t r[8], uint32_t out[8]) {
        uint32_t w[16];
#pragma unroll
        for (int i = 0; i < 8; ++i) { w[i] = l[i]; w[8 + i] = r[i]; }
        init(out);
        compress_rolled(out, w);
        w[0] = 0x80000000u;
#pragma unroll
        for (int i = 1; i < 15; ++i) w[i] = 0;
        w[15] = 512;
        compress_rolled(out, w);
    }

    // Digest bytes <-> state words (big-endian words).
    SNT_HD static void state_to_bytes_words(const uint32_t s[8], uint32_t le[8]) {
#pragma unroll
        for (int i = 0; i < 8; ++i) le[i] = bswap32(s[i]);
    }
    SNT_HD static void bytes_words_to_state(const uint32_t le[8], uint32_t s[8]) {
#pragma unroll
        for (int i = 0; i < 8; ++i) s[i] = bswap32(le[i]);
    }
};

}  // namespace snt
