// BLAKE2b-512 with the message streamed through shared memory.
//
// The register-resident formulation (blake2b.cuh) keeps the 16 message words of
// a block in 32 registers and unrolls all 12 rounds so that the sigma
// permutation becomes register names: ~165 registers per thread and 36 KB of
// straight-line code per compression -- three warps per scheduler, no room to
// prefetch, and an instruction stream larger than the SM's 32 KB instruction
// cache (ncu: long-scoreboard and no-instruction stalls, ALU pipe 68-90 % busy).
//
// Here every thread owns two 17-slot staging buffers in shared memory, laid out
// word-major ([slot][thread], 8 bytes per thread: conflict-free LDS.64). The
// next 128-byte chunk of the thread's message is copied in with cp.async while
// the current block is compressed (prefetch without registers), the rounds are
// a rolled loop that reads message word sigma[r][i] straight from the staging
// buffer (the index is warp-uniform, so the address arithmetic runs on the
// uniform datapath), and the 8-byte LtHash tag is absorbed by sliding the
// window one slot: slot 0 of a buffer holds the word carried over from the
// previous chunk (or the tag), slots 1..16 the chunk.
//
// The algorithm (block/tail/carry bookkeeping) is __host__ __device__: on the
// host the stager is a memcpy and tests/hostcheck runs it against hashlib.
#pragma once
#include "blake2b.cuh"

namespace snt {

#define SNT_B2B_SIGMA_ROWS                                                              \
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},                             \
    {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},                             \
    {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4},                             \
    {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},                             \
    {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13},                             \
    {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},                             \
    {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11},                             \
    {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},                             \
    {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5},                             \
    {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},                             \
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},                             \
    {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}

#if defined(__CUDACC__)
__constant__ uint8_t c_b2b_sigma[12][16] = {SNT_B2B_SIGMA_ROWS};
#endif
static const uint8_t h_b2b_sigma[12][16] = {SNT_B2B_SIGMA_ROWS};

constexpr int B2S_MAX_TAG_WORDS = 2;
constexpr int B2S_SLOTS = 16 + B2S_MAX_TAG_WORDS;     // carried/tag words + 16 chunk words

// STRIDE = number of 8-byte words between consecutive slots of one thread
// (= threads per CTA on the device, 1 on the host).
template <int STRIDE>
struct Blake2bStream : Blake2b {
    SNT_HD static const uint8_t* sigma_row(int r) {
#ifdef __CUDA_ARCH__
        return c_b2b_sigma[r];
#else
        return h_b2b_sigma[r];
#endif
    }

    // One compression; message word i is win[i * STRIDE].
    SNT_HD static void compress_window(uint64_t h[8], const uint64_t* win, uint64_t t, bool last) {
        uint64_t v0 = h[0], v1 = h[1], v2 = h[2], v3 = h[3], v4 = h[4], v5 = h[5], v6 = h[6], v7 = h[7];
        uint64_t v8 = SNT_B2B_IV0, v9 = SNT_B2B_IV1, v10 = SNT_B2B_IV2, v11 = SNT_B2B_IV3;
        uint64_t v12 = SNT_B2B_IV4 ^ t, v13 = SNT_B2B_IV5;
        uint64_t v14 = last ? ~SNT_B2B_IV6 : SNT_B2B_IV6, v15 = SNT_B2B_IV7;
#pragma unroll 1
        for (int r = 0; r < 12; ++r) {
            const uint8_t* s = sigma_row(r);
#define SNT_W(k) win[static_cast<int>(s[k]) * STRIDE]
            SNT_B2B_G(v0, v4, v8, v12, SNT_W(0), SNT_W(1));
            SNT_B2B_G(v1, v5, v9, v13, SNT_W(2), SNT_W(3));
            SNT_B2B_G(v2, v6, v10, v14, SNT_W(4), SNT_W(5));
            SNT_B2B_G(v3, v7, v11, v15, SNT_W(6), SNT_W(7));
            SNT_B2B_G(v0, v5, v10, v15, SNT_W(8), SNT_W(9));
            SNT_B2B_G(v1, v6, v11, v12, SNT_W(10), SNT_W(11));
            SNT_B2B_G(v2, v7, v8, v13, SNT_W(12), SNT_W(13));
            SNT_B2B_G(v3, v4, v9, v14, SNT_W(14), SNT_W(15));
#undef SNT_W
        }
        h[0] ^= v0 ^ v8;  h[1] ^= v1 ^ v9;  h[2] ^= v2 ^ v10; h[3] ^= v3 ^ v11;
        h[4] ^= v4 ^ v12; h[5] ^= v5 ^ v13; h[6] ^= v6 ^ v14; h[7] ^= v7 ^ v15;
    }

    // Copy the 128-byte chunk at g into slots T..T+15 of `buf`: asynchronously (cp.async,
    // 8 bytes at a time) when g is 8-byte aligned, through registers otherwise.
    template <int T>
    SNT_HD static void stage_chunk(uint64_t* buf, const uint8_t* g) {
#ifdef __CUDA_ARCH__
        if ((reinterpret_cast<uintptr_t>(g) & 7) == 0) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(buf + (T + i) * STRIDE));
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(g + 8 * i) : "memory");
            }
            return;
        }
#endif
        uint64_t m[16];
        load_words64<16>(g, m);
#pragma unroll
        for (int i = 0; i < 16; ++i) buf[(T + i) * STRIDE] = m[i];
    }
    SNT_HD static void commit() {
#ifdef __CUDA_ARCH__
        asm volatile("cp.async.commit_group;" ::: "memory");
#endif
    }
    // wait until at most `N` of this thread's committed groups are still in flight
    template <int N>
    SNT_HD static void wait_pending() {
#ifdef __CUDA_ARCH__
        asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
#endif
    }

    // H(T tag words || data[0..len)), any data alignment. `bufs` points at this thread's
    // slot 0 of buffer 0; buffer 1 starts B2S_SLOTS * STRIDE words later.
    // T = 0: plain BLAKE2b (Merkle leaves, hash_blocks); T = 1: LE64(index) in front (LtHash,
    // lattice.py:92-94); T = 2: LE64(layer) || LE64(block) (per-layer lattice, model.py:259).
    //
    // Block b of the message is T words carried over from the previous chunk (the tag for
    // b = 0) followed by the first 16 - T words of data chunk b: with the chunk staged at
    // slots T..T+15 the block is simply slots 0..15, and slots 16..16+T-1 are the carry.
    template <int T>
    SNT_HD static void hash_message(uint64_t* bufs, uint64_t tag0, uint64_t tag1, const uint8_t* p, uint64_t len,
                                    uint64_t h[8]) {
        static_assert(T >= 0 && T <= B2S_MAX_TAG_WORDS, "unsupported tag width");
        init(h);
        uint64_t* const buf0 = bufs;
        uint64_t* const buf1 = bufs + B2S_SLOTS * STRIDE;
        const uint64_t nfull = len >> 7;                 // whole 128-byte chunks of data
        const uint32_t r = static_cast<uint32_t>(len & 127);
        const uint64_t total = len + 8ull * T;
        if (nfull > 0) stage_chunk<T>(buf0, p);
        commit();
        if (T >= 1) buf0[0] = tag0;
        if (T >= 2) buf0[STRIDE] = tag1;
        for (uint64_t b = 0; b < nfull; ++b) {
            uint64_t* cur = (b & 1) ? buf1 : buf0;
            uint64_t* nxt = (b & 1) ? buf0 : buf1;
            if (b + 1 < nfull) stage_chunk<T>(nxt, p + ((b + 1) << 7));
            commit();
            wait_pending<1>();                            // chunk b has landed
            // a full data chunk is followed by at least the carried words, so with T > 0 this
            // block is never the final one; with T = 0 it is final when the data ends here
            const bool last = T == 0 && (b + 1 == nfull) && r == 0;
            compress_window(h, cur, (b + 1) << 7, last);
#pragma unroll
            for (int i = 0; i < T; ++i) nxt[i * STRIDE] = cur[(16 + i) * STRIDE];
        }
        wait_pending<0>();
        if (T == 0 && r == 0 && len != 0) return;         // ended exactly on a block boundary
        // tail: the T carried words (already in slots 0..T-1) and the r remaining data bytes
        const uint8_t* q = p + (nfull << 7);
        uint64_t* win = (nfull & 1) ? buf1 : buf0;
#pragma unroll 1
        for (int j = 0; j < 16 - T; ++j) win[(T + j) * STRIDE] = tail_word64(q, j, r);
        if (8u * T + r <= 128u) {
            compress_window(h, win, total, true);
        } else {
            compress_window(h, win, (nfull + 1) << 7, false);
#pragma unroll 1
            for (int j = 0; j < 16; ++j) win[j * STRIDE] = j < T ? tail_word64(q, 16 - T + j, r) : 0ull;
            compress_window(h, win, total, true);
        }
    }
};

}  // namespace snt
