// BLAKE2b-512 (RFC 7693), unkeyed, default parameters, one message per thread.
// 64-bit lanes are kept as uint64_t; the rotations are spelled with PRMT / SHF
// on the device so each costs two 32-bit instructions (rot32 is a register
// rename).
//
// Role in the reference: hashlib.blake2b at compression.py:45-49 (Merkle leaf
// and node variant) and lattice.py:97-101 (LtHash of tag || data).
#pragma once
#include "common.cuh"

namespace snt {

#define SNT_B2B_SIGMA                                          \
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},   \
    {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},   \
    {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4},   \
    {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},   \
    {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13},   \
    {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},   \
    {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11},   \
    {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},   \
    {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5},   \
    {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},   \
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},   \
    {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}

#if defined(__CUDACC__)
__constant__ uint8_t c_b2b_sigma[12][16] = {SNT_B2B_SIGMA};      // for the rolled compression (compress_rolled)
#endif

struct Blake2b {
    static constexpr int DIGEST_BYTES = 64;
    static constexpr int BLOCK_BYTES = 128;

    SNT_HD static uint64_t ror32(uint64_t x) {
#ifdef __CUDA_ARCH__
        const uint32_t lo = static_cast<uint32_t>(x), hi = static_cast<uint32_t>(x >> 32);
        return (static_cast<uint64_t>(lo) << 32) | hi;
#else
        return rotr64(x, 32);
#endif
    }
    SNT_HD static uint64_t ror24(uint64_t x) {
#ifdef __CUDA_ARCH__
        const uint32_t lo = static_cast<uint32_t>(x), hi = static_cast<uint32_t>(x >> 32);
        const uint32_t nlo = __byte_perm(lo, hi, 0x6543), nhi = __byte_perm(lo, hi, 0x2107);
        return (static_cast<uint64_t>(nhi) << 32) | nlo;
#else
        return rotr64(x, 24);
#endif
    }
    SNT_HD static uint64_t ror16(uint64_t x) {
#ifdef __CUDA_ARCH__
        const uint32_t lo = static_cast<uint32_t>(x), hi = static_cast<uint32_t>(x >> 32);
        const uint32_t nlo = __byte_perm(lo, hi, 0x5432), nhi = __byte_perm(lo, hi, 0x1076);
        return (static_cast<uint64_t>(nhi) << 32) | nlo;
#else
        return rotr64(x, 16);
#endif
    }
    SNT_HD static uint64_t ror63(uint64_t x) {
#ifdef __CUDA_ARCH__
        const uint32_t lo = static_cast<uint32_t>(x), hi = static_cast<uint32_t>(x >> 32);
        const uint32_t nlo = __funnelshift_l(hi, lo, 1), nhi = __funnelshift_l(lo, hi, 1);
        return (static_cast<uint64_t>(nhi) << 32) | nlo;
#else
        return rotr64(x, 63);
#endif
    }

#define SNT_B2B_IV0 0x6a09e667f3bcc908ull
#define SNT_B2B_IV1 0xbb67ae8584caa73bull
#define SNT_B2B_IV2 0x3c6ef372fe94f82bull
#define SNT_B2B_IV3 0xa54ff53a5f1d36f1ull
#define SNT_B2B_IV4 0x510e527fade682d1ull
#define SNT_B2B_IV5 0x9b05688c2b3e6c1full
#define SNT_B2B_IV6 0x1f83d9abfb41bd6bull
#define SNT_B2B_IV7 0x5be0cd19137e2179ull

    SNT_HD static void init(uint64_t h[8]) {
        // parameter block word 0: digest_length=64, key_length=0, fanout=1, depth=1
        h[0] = SNT_B2B_IV0 ^ 0x01010040ull;
        h[1] = SNT_B2B_IV1; h[2] = SNT_B2B_IV2; h[3] = SNT_B2B_IV3;
        h[4] = SNT_B2B_IV4; h[5] = SNT_B2B_IV5; h[6] = SNT_B2B_IV6; h[7] = SNT_B2B_IV7;
    }

#define SNT_B2B_G(a, b, c, d, x, y)   \
    a = a + b + (x); d = ror32(d ^ a); \
    c = c + d;       b = ror24(b ^ c); \
    a = a + b + (y); d = ror16(d ^ a); \
    c = c + d;       b = ror63(b ^ c);

    // One compression: t = bytes absorbed so far including this block
    // (messages here are < 2^64 bytes, so the high counter word is zero).
    SNT_HD static void compress(uint64_t h[8], const uint64_t m[16], uint64_t t, bool last) {
        const uint8_t S[12][16] = {SNT_B2B_SIGMA};
        uint64_t v0 = h[0], v1 = h[1], v2 = h[2], v3 = h[3], v4 = h[4], v5 = h[5], v6 = h[6], v7 = h[7];
        uint64_t v8 = SNT_B2B_IV0, v9 = SNT_B2B_IV1, v10 = SNT_B2B_IV2, v11 = SNT_B2B_IV3;
        uint64_t v12 = SNT_B2B_IV4 ^ t, v13 = SNT_B2B_IV5;
        uint64_t v14 = last ? ~SNT_B2B_IV6 : SNT_B2B_IV6, v15 = SNT_B2B_IV7;
#pragma unroll
        for (int r = 0; r < 12; ++r) {
            SNT_B2B_G(v0, v4, v8, v12, m[S[r][0]], m[S[r][1]]);
            SNT_B2B_G(v1, v5, v9, v13, m[S[r][2]], m[S[r][3]]);
            SNT_B2B_G(v2, v6, v10, v14, m[S[r][4]], m[S[r][5]]);
            SNT_B2B_G(v3, v7, v11, v15, m[S[r][6]], m[S[r][7]]);
            SNT_B2B_G(v0, v5, v10, v15, m[S[r][8]], m[S[r][9]]);
            SNT_B2B_G(v1, v6, v11, v12, m[S[r][10]], m[S[r][11]]);
            SNT_B2B_G(v2, v7, v8, v13, m[S[r][12]], m[S[r][13]]);
            SNT_B2B_G(v3, v4, v9, v14, m[S[r][14]], m[S[r][15]]);
        }
        h[0] ^= v0 ^ v8;  h[1] ^= v1 ^ v9;  h[2] ^= v2 ^ v10; h[3] ^= v3 ^ v11;
        h[4] ^= v4 ^ v12; h[5] ^= v5 ^ v13; h[6] ^= v6 ^ v14; h[7] ^= v7 ^ v15;
    }

    // One compression with the twelve rounds rolled and the message schedule read from a table: ~3 KB
    // of code instead of 34 KB, for the cold paths that share a kernel with the unrolled leaf loop (tree
    // nodes) and must not push that loop out of the instruction cache. m is indexed dynamically, so it
    // lives in local memory.
    SNT_HD static void compress_rolled(uint64_t h[8], const uint64_t m[16], uint64_t t, bool last) {
#ifdef __CUDA_ARCH__
        const uint8_t (*S)[16] = c_b2b_sigma;
#else
        static const uint8_t S[12][16] = {SNT_B2B_SIGMA};
#endif
        uint64_t v0 = h[0], v1 = h[1], v2 = h[2], v3 = h[3], v4 = h[4], v5 = h[5], v6 = h[6], v7 = h[7];
        uint64_t v8 = SNT_B2B_IV0, v9 = SNT_B2B_IV1, v10 = SNT_B2B_IV2, v11 = SNT_B2B_IV3;
        uint64_t v12 = SNT_B2B_IV4 ^ t, v13 = SNT_B2B_IV5;
        uint64_t v14 = last ? ~SNT_B2B_IV6 : SNT_B2B_IV6, v15 = SNT_B2B_IV7;
#pragma unroll 1
        for (int r = 0; r < 12; ++r) {
            SNT_B2B_G(v0, v4, v8, v12, m[S[r][0]], m[S[r][1]]);
            SNT_B2B_G(v1, v5, v9, v13, m[S[r][2]], m[S[r][3]]);
            SNT_B2B_G(v2, v6, v10, v14, m[S[r][4]], m[S[r][5]]);
            SNT_B2B_G(v3, v7, v11, v15, m[S[r][6]], m[S[r][7]]);
            SNT_B2B_G(v0, v5, v10, v15, m[S[r][8]], m[S[r][9]]);
            SNT_B2B_G(v1, v6, v11, v12, m[S[r][10]], m[S[r][11]]);
            SNT_B2B_G(v2, v7, v8, v13, m[S[r][12]], m[S[r][13]]);
            SNT_B2B_G(v3, v4, v9, v14, m[S[r][14]], m[S[r][15]]);
        }
        h[0] ^= v0 ^ v8;  h[1] ^= v1 ^ v9;  h[2] ^= v2 ^ v10; h[3] ^= v3 ^ v11;
        h[4] ^= v4 ^ v12; h[5] ^= v5 ^ v13; h[6] ^= v6 ^ v14; h[7] ^= v7 ^ v15;
    }

    // Load `NW` 64-bit little-endian words from p (any alignment, all valid).
    template <int NW>
    SNT_HD static void load_words64(const uint8_t* p, uint64_t* m) {
        uint32_t w[2 * NW];
        load_words<2 * NW>(p, w);
#pragma unroll
        for (int i = 0; i < NW; ++i) m[i] = (static_cast<uint64_t>(w[2 * i + 1]) << 32) | w[2 * i];
    }

    // 64-bit LE word j of a tail of `rem` valid bytes at t, zero beyond.
    SNT_HD static uint64_t tail_word64(const uint8_t* t, uint32_t j, uint32_t rem) {
        if (8 * j + 8 <= rem) {
            uint64_t m;
            load_words64<1>(t + 8 * j, &m);
            return m;
        }
        uint64_t v = 0;
        if (8 * j < rem) {
#pragma unroll
            for (int k = 7; k >= 0; --k) v = (v << 8) | tail_byte(t, 8 * j + k, rem);
        }
        return v;
    }

    // H(tag words || data): the message is T little-endian 64-bit tag words
    // (T = 0 for plain hashing, 1 for LE64(index), 2 for LE64(i)||LE64(j))
    // followed by data[0..len). Mirrors lattice.py:92-101 and, with T = 0,
    // compression.py:70-74.
    template <int T>
    SNT_HD static void hash_message(uint64_t tag0, uint64_t tag1, const uint8_t* p, uint64_t len,
                                    uint64_t h[8]) {
        init(h);
        const uint64_t total = len + 8ull * T;
        // A message ending on a block boundary keeps its last block as the
        // final one; the empty message is one all-zero final block.
        const uint64_t nblocks = total == 0 ? 1 : ((total + 127) >> 7);
        for (uint64_t b = 0; b < nblocks; ++b) {
            uint64_t m[16];
            const bool last = (b == nblocks - 1);
            if (!last) {
                if (T > 0 && b == 0) {
                    if (T >= 1) m[0] = tag0;
                    if (T >= 2) m[1] = tag1;
                    load_words64<16 - T>(p, m + T);
                } else {
                    load_words64<16>(p + (b << 7) - 8 * T, m);
                }
            } else if (b == 0) {
                // tag words (if any) sit at the front of the only block
                if (T >= 1) m[0] = tag0;
                if (T >= 2) m[1] = tag1;
                const uint32_t rem = static_cast<uint32_t>(len);
#pragma unroll
                for (int j = 0; j < 16 - T; ++j) m[T + j] = tail_word64(p, j, rem);
            } else {
                const uint8_t* t = p + (b << 7) - 8 * T;
                const uint32_t rem = static_cast<uint32_t>(total - (b << 7));   // 1..128
#pragma unroll
                for (int j = 0; j < 16; ++j) m[j] = tail_word64(t, j, rem);
            }
            compress(h, m, last ? total : ((b + 1) << 7), last);
        }
    }

    // Tree node: H(left || right), 128-byte message = exactly one final block.
    SNT_HD static void hash_pair(const uint64_t l[8], const uint64_t r[8], uint64_t out[8]) {
        uint64_t m[16];
#pragma unroll
        for (int i = 0; i < 8; ++i) { m[i] = l[i]; m[8 + i] = r[i]; }
        init(out);
        compress(out, m, 128, true);
    }
    SNT_HD static void hash_pair_rolled(const uint64_t l[8], const uint64_t r[8], uint64_t out[8]) {
        uint64_t m[16];
#pragma unroll
        for (int i = 0; i < 8; ++i) { m[i] = l[i]; m[8 + i] = r[i]; }
        init(out);
        compress_rolled(out, m, 128, true);
    }
};

}  // namespace snt
