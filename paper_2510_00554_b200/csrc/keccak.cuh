// SHA3-256 (FIPS 202): Keccak-f[1600] sponge, rate 136 bytes, one message per
// thread, the 25-lane state in registers.
//
// Role in the reference: hashlib.sha3_256 at compression.py:45-49 (Merkle leaf
// and node variant).
#pragma once
#include "common.cuh"

namespace snt {

#define SNT_KECCAK_RC                                                                             \
    0x0000000000000001ull, 0x0000000000008082ull, 0x800000000000808aull, 0x8000000080008000ull, \
    0x000000000000808bull, 0x0000000080000001ull, 0x8000000080008081ull, 0x8000000000008009ull, \
    0x000000000000008aull, 0x0000000000000088ull, 0x0000000080008009ull, 0x000000008000000aull, \
    0x000000008000808bull, 0x800000000000008bull, 0x8000000000008089ull, 0x8000000000008003ull, \
    0x8000000000008002ull, 0x8000000000000080ull, 0x000000000000800aull, 0x800000008000000aull, \
    0x8000000080008081ull, 0x8000000000008080ull, 0x0000000080000001ull, 0x8000000080008008ull

#if defined(__CUDACC__)
__constant__ uint64_t c_keccak_rc[24] = {SNT_KECCAK_RC};
#endif
static const uint64_t h_keccak_rc[24] = {SNT_KECCAK_RC};

struct Sha3_256 {
    static constexpr int DIGEST_BYTES = 32;
    static constexpr int RATE_BYTES = 136;
    static constexpr int RATE_LANES = 17;

    SNT_HD static uint64_t rol(uint64_t x, int n) {
#ifdef __CUDA_ARCH__
        const uint32_t lo = static_cast<uint32_t>(x), hi = static_cast<uint32_t>(x >> 32);
        uint32_t nlo, nhi;
        if (n == 0) return x;
        if (n < 32) {
            nlo = __funnelshift_l(hi, lo, n);
            nhi = __funnelshift_l(lo, hi, n);
        } else if (n == 32) {
            nlo = hi; nhi = lo;
        } else {
            nlo = __funnelshift_l(lo, hi, n - 32);
            nhi = __funnelshift_l(hi, lo, n - 32);
        }
        return (static_cast<uint64_t>(nhi) << 32) | nlo;
#else
        return n ? rotl64(x, n) : x;
#endif
    }

    // a ^ b ^ c as one LOP3 per 32-bit half. Spelled out so that the compiler does not regroup the
    // theta step into an explicit D[x] = C[x-1] ^ rol(C[x+1], 1) followed by 25 two-input XORs
    // (10 + 50 LOP3 per round); folding D into each lane's XOR needs 50 (192 -> 182 ALU ops per round).
    SNT_HD static uint64_t xor3(uint64_t a, uint64_t b, uint64_t c) {
#ifdef __CUDA_ARCH__
        uint32_t lo, hi;
        asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(lo)
            : "r"(static_cast<uint32_t>(a)), "r"(static_cast<uint32_t>(b)), "r"(static_cast<uint32_t>(c)));
        asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(hi)
            : "r"(static_cast<uint32_t>(a >> 32)), "r"(static_cast<uint32_t>(b >> 32)), "r"(static_cast<uint32_t>(c >> 32)));
        return (static_cast<uint64_t>(hi) << 32) | lo;
#else
        return a ^ b ^ c;
#endif
    }

    SNT_HD static uint64_t round_constant(int round) {
#ifdef __CUDA_ARCH__
        return c_keccak_rc[round];
#else
        return h_keccak_rc[round];
#endif
    }

    SNT_HD static void permute(uint64_t a[25]) {
        // rho rotation of lane (x, y) stored at index x + 5*y
        const int RHO[25] = {0,  1,  62, 28, 27, 36, 44, 6,  55, 20, 3,  10, 43,
                             25, 39, 41, 45, 15, 21, 8,  18, 2,  61, 56, 14};
#pragma unroll 1
        for (int round = 0; round < 24; ++round) {
            uint64_t c[5], c1[5], b[25];
#pragma unroll
            for (int x = 0; x < 5; ++x) c[x] = xor3(xor3(a[x], a[x + 5], a[x + 10]), a[x + 15], a[x + 20]);
#pragma unroll
            for (int x = 0; x < 5; ++x) c1[x] = rol(c[x], 1);
            // theta + rho + pi: B[y, 2x+3y] = rol(A[x, y] ^ D[x], r[x, y]) with D[x] = C[x-1] ^ rol(C[x+1], 1)
            // folded into the lane's XOR
#pragma unroll
            for (int y = 0; y < 5; ++y) {
#pragma unroll
                for (int x = 0; x < 5; ++x) {
                    const int nx = y, ny = (2 * x + 3 * y) % 5;
                    b[nx + 5 * ny] = rol(xor3(a[x + 5 * y], c[(x + 4) % 5], c1[(x + 1) % 5]), RHO[x + 5 * y]);
                }
            }
            // chi
#pragma unroll
            for (int y = 0; y < 5; ++y) {
#pragma unroll
                for (int x = 0; x < 5; ++x) {
                    a[x + 5 * y] = b[x + 5 * y] ^ (~b[(x + 1) % 5 + 5 * y] & b[(x + 2) % 5 + 5 * y]);
                }
            }
            a[0] ^= round_constant(round);
        }
    }

    SNT_HD static uint64_t tail_lane(const uint8_t* t, uint32_t j, uint32_t rem) {
        if (8 * j + 8 <= rem) {
            uint32_t w[2];
            load_words<2>(t + 8 * j, w);
            return (static_cast<uint64_t>(w[1]) << 32) | w[0];
        }
        uint64_t v = 0;
        if (8 * j < rem) {
#pragma unroll
            for (int k = 7; k >= 0; --k) v = (v << 8) | tail_byte(t, 8 * j + k, rem);
        }
        return v;
    }

    // Number of permutations a message of `len` bytes takes: its full rate blocks plus the padded tail.
    SNT_HD static uint64_t block_count(uint64_t len) { return len / RATE_BYTES + 1; }

    // Absorb rate blocks [u0, u1) (clipped to block_count(len)) into the sponge state a. One loop,
    // one permute call site: full rate blocks, then the padded tail (0x06 after the last byte,
    // 0x80 in the last rate byte). Slices of one message may run in different threads: the 25
    // lanes are all that travels.
    SNT_HD static void absorb_blocks(uint64_t a[25], const uint8_t* p, uint64_t len, uint64_t u0, uint64_t u1) {
        const uint64_t nfull = len / RATE_BYTES;
        const uint32_t rem = static_cast<uint32_t>(len - nfull * RATE_BYTES);   // 0..135
        if (u1 > nfull + 1) u1 = nfull + 1;
        for (uint64_t blk = u0; blk < u1; ++blk) {
            const uint8_t* q = p + blk * RATE_BYTES;
            if (blk < nfull) {
                uint32_t w[2 * RATE_LANES];
                load_words<2 * RATE_LANES>(q, w);
#pragma unroll
                for (int i = 0; i < RATE_LANES; ++i)
                    a[i] ^= (static_cast<uint64_t>(w[2 * i + 1]) << 32) | w[2 * i];
            } else {
#pragma unroll
                for (int j = 0; j < RATE_LANES; ++j) {
                    uint64_t lane = tail_lane(q, j, rem);
                    if ((rem >> 3) == static_cast<uint32_t>(j)) lane ^= 0x06ull << (8 * (rem & 7));
                    a[j] ^= lane;
                }
                a[RATE_LANES - 1] ^= 0x8000000000000000ull;
            }
            permute(a);
        }
    }

    // Whole message; out = first four lanes = the 32 digest bytes little-endian.
    SNT_HD static void hash_message(const uint8_t* p, uint64_t len, uint64_t out[4]) {
        uint64_t a[25];
#pragma unroll
        for (int i = 0; i < 25; ++i) a[i] = 0;
        absorb_blocks(a, p, len, 0, ~0ull);
#pragma unroll
        for (int i = 0; i < 4; ++i) out[i] = a[i];
    }

    // Tree node: H(left || right), 64-byte message = one permutation.
    SNT_HD static void hash_pair(const uint64_t l[4], const uint64_t r[4], uint64_t out[4]) {
        uint64_t a[25];
#pragma unroll
        for (int i = 0; i < 4; ++i) { a[i] = l[i]; a[4 + i] = r[i]; }
        a[8] = 0x06ull;
#pragma unroll
        for (int i = 9; i < 25; ++i) a[i] = 0;
        a[RATE_LANES - 1] ^= 0x8000000000000000ull;
        permute(a);
#pragma unroll
        for (int i = 0; i < 4; ++i) out[i] = a[i];
    }
};

}  // namespace snt
