// BLAKE2b-512 with four lanes per message ("quad"): lane c owns column c of the
// 4x4 state (a = v[c], b = v[4+c], c = v[8+c], d = v[12+c]). A round is a column
// step (G on the own column), a lane rotation of b/c/d inside the quad with
// warp shuffles, a diagonal step, and the rotation back. The 128-byte message
// block is staged in shared memory by the quad (32 contiguous bytes per lane,
// coalesced), and each lane fetches the four words its G functions need with
// LDS.64 at offsets picked from compile-time immediates by one PRMT.
//
// Why: LATENCY. One thread per message is the throughput-optimal form (the four G functions of a step are that
// thread's instruction-level parallelism; measured on the CIFAR-shaped set the quad form is 0.28 vs 0.22 ms), but
// a loader batch of 128 samples is four warps of serial compressions, one warp alone on its scheduler: 2.6-3 us
// per 128-byte block, 70 us for 128 CIFAR-sized rows with the GPU 99.9 % idle. With four lanes per message a
// compression is a quarter of the instructions per lane plus 12 shuffles per round: about half the time per
// block. Used for launches of at most a few thousand items (lthash_quad_kernel); the arithmetic is the same
// RFC 7693 function as blake2b.cuh (lattice.py:97-101 in the reference).
#pragma once
#include "blake2b.cuh"

namespace snt {

constexpr int QUAD_REGION_BYTES = 144;   // 128-byte block + padding that spreads quads over banks

// byte offsets (8 * sigma index) of message word `slot` (0..3) of round R for the 4 lanes, packed
// one byte per lane. slot 0,1: column step words sigma[R][2c], sigma[R][2c+1];
// slot 2,3: diagonal step words sigma[R][8+2c], sigma[R][9+2c].
__host__ __device__ constexpr uint32_t quad_moff(int round, int slot) {
    const uint8_t S[12][16] = {
        {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},
        {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
        {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4},
        {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
        {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13},
        {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
        {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11},
        {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
        {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5},
        {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
        {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},
        {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};
    uint32_t packed = 0;
    for (int c = 0; c < 4; ++c) {
        const int pos = (slot < 2) ? (2 * c + slot) : (8 + 2 * c + (slot - 2));
        packed |= static_cast<uint32_t>(8 * S[round][pos]) << (8 * c);
    }
    return packed;
}

struct QuadLane {
    uint32_t c;          // lane within the quad, 0..3
    uint32_t sel;        // PRMT selector that extracts byte c
    uint32_t qmask;      // the quad's four lanes in the warp
    uint32_t base;       // lane id of the quad's lane 0
};

SNT_D QuadLane quad_lane() {
    QuadLane q;
    const uint32_t lane = threadIdx.x & 31;
    q.c = lane & 3;
    q.sel = 0x4440u | q.c;
    q.base = lane & ~3u;
    q.qmask = 0xFu << q.base;
    return q;
}

SNT_D uint64_t quad_shfl(uint64_t v, uint32_t src_lane, uint32_t qmask) {
    const uint32_t lo = __shfl_sync(qmask, static_cast<uint32_t>(v), src_lane);
    const uint32_t hi = __shfl_sync(qmask, static_cast<uint32_t>(v >> 32), src_lane);
    return (static_cast<uint64_t>(hi) << 32) | lo;
}

SNT_D uint64_t quad_word(const uint8_t* region, uint32_t packed, uint32_t sel) {
    const uint32_t off = __byte_perm(packed, 0, sel);
    return *reinterpret_cast<const uint64_t*>(region + off);
}

// Uses SNT_B2B_G's ror helpers, which are members of Blake2b.
struct Blake2bQuad : Blake2b {
    template <int R>
    SNT_D static void round(uint64_t& a, uint64_t& b, uint64_t& c, uint64_t& d, const uint8_t* region,
                            const QuadLane& q) {
        constexpr uint32_t o0 = quad_moff(R, 0), o1 = quad_moff(R, 1), o2 = quad_moff(R, 2), o3 = quad_moff(R, 3);
        {
            const uint64_t x = quad_word(region, o0, q.sel), y = quad_word(region, o1, q.sel);
            SNT_B2B_G(a, b, c, d, x, y);
        }
        b = quad_shfl(b, q.base + ((q.c + 1) & 3), q.qmask);
        c = quad_shfl(c, q.base + ((q.c + 2) & 3), q.qmask);
        d = quad_shfl(d, q.base + ((q.c + 3) & 3), q.qmask);
        {
            const uint64_t x = quad_word(region, o2, q.sel), y = quad_word(region, o3, q.sel);
            SNT_B2B_G(a, b, c, d, x, y);
        }
        b = quad_shfl(b, q.base + ((q.c + 3) & 3), q.qmask);
        c = quad_shfl(c, q.base + ((q.c + 2) & 3), q.qmask);
        d = quad_shfl(d, q.base + ((q.c + 1) & 3), q.qmask);
    }

    SNT_D static uint64_t iv(uint32_t i) {
        // IV word i for i in 0..7 without indexing a local array
        uint64_t v = SNT_B2B_IV0;
        v = i == 1 ? SNT_B2B_IV1 : v; v = i == 2 ? SNT_B2B_IV2 : v; v = i == 3 ? SNT_B2B_IV3 : v;
        v = i == 4 ? SNT_B2B_IV4 : v; v = i == 5 ? SNT_B2B_IV5 : v; v = i == 6 ? SNT_B2B_IV6 : v;
        v = i == 7 ? SNT_B2B_IV7 : v;
        return v;
    }

    // Stream words [16*blk + 4*c, +4) of (T tag words || data): this lane's 32 bytes of message block blk.
    template <int T>
    SNT_D static void fetch(const QuadLane& q, uint64_t blk, uint64_t tag0, uint64_t tag1, const uint8_t* p, uint64_t len,
                            uint64_t m[4]) {
        const uint64_t sw0 = (blk << 4) + 4 * q.c;                 // first stream word of this lane
        const uint64_t d0 = (sw0 - T) << 3;                        // data byte offset of stream word sw0 (if sw0 >= T)
        if (sw0 >= static_cast<uint64_t>(T) && d0 + 32 <= len) {
            load_words64<4>(p + d0, m);
        } else {
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                const uint64_t sw = sw0 + w;
                uint64_t v = 0;
                if (sw < static_cast<uint64_t>(T)) {
                    v = sw == 0 ? tag0 : tag1;
                } else {
                    const uint64_t off = (sw - T) << 3;
                    if (off + 8 <= len) {
                        load_words64<1>(p + off, &v);
                    } else if (off < len) {
                        const uint32_t rem = static_cast<uint32_t>(len - off);
#pragma unroll
                        for (int k = 7; k >= 0; --k) v = (v << 8) | tail_byte(p + off, k, rem);
                    }
                }
                m[w] = v;
            }
        }
    }
    SNT_D static void put(uint8_t* region, const QuadLane& q, const uint64_t m[4]) {
        uint64_t* dst = reinterpret_cast<uint64_t*>(region + 32 * q.c);
#pragma unroll
        for (int w = 0; w < 4; ++w) dst[w] = m[w];
    }

    // Whole message (T tag words || data[0..len)). On return lane c holds digest
    // words c and 4 + c in h_lo / h_hi.
    template <int T>
    SNT_D static void hash_message(uint8_t* region, const QuadLane& q, uint64_t tag0, uint64_t tag1,
                                   const uint8_t* p, uint64_t len, uint64_t& h_lo, uint64_t& h_hi) {
        h_lo = iv(q.c) ^ (q.c == 0 ? 0x01010040ull : 0ull);
        h_hi = iv(4 + q.c);
        const uint64_t total = len + 8ull * T;
        const uint64_t nblocks = total == 0 ? 1 : ((total + 127) >> 7);
        uint64_t m[4];
        fetch<T>(q, 0, tag0, tag1, p, len, m);
        for (uint64_t blk = 0; blk < nblocks; ++blk) {
            const bool last = blk == nblocks - 1;
            __syncwarp(q.qmask);                       // previous block's words have been consumed
            put(region, q, m);
            __syncwarp(q.qmask);
            if (!last) fetch<T>(q, blk + 1, tag0, tag1, p, len, m);     // in flight while this block is compressed
            const uint64_t t = last ? total : ((blk + 1) << 7);
            uint64_t a = h_lo, b = h_hi, c = iv(q.c), d = iv(4 + q.c);
            if (q.c == 0) d ^= t;                      // v12 ^= t (low counter word)
            if (q.c == 2 && last) d = ~d;              // v14 ^= f0
            round<0>(a, b, c, d, region, q);  round<1>(a, b, c, d, region, q);
            round<2>(a, b, c, d, region, q);  round<3>(a, b, c, d, region, q);
            round<4>(a, b, c, d, region, q);  round<5>(a, b, c, d, region, q);
            round<6>(a, b, c, d, region, q);  round<7>(a, b, c, d, region, q);
            round<8>(a, b, c, d, region, q);  round<9>(a, b, c, d, region, q);
            round<10>(a, b, c, d, region, q); round<11>(a, b, c, d, region, q);
            h_lo ^= a ^ c;
            h_hi ^= b ^ d;
        }
    }
};

}  // namespace snt
