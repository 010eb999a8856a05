// BLAKE2b-512 with the message prefetched through shared memory.
//
// Blake2b::hash_message (blake2b.cuh) loads each 128-byte block with ordinary
// loads right before compressing it: with ~165 registers per thread only three
// warps fit per scheduler, nothing hides the load latency (ncu: long-scoreboard
// is the top stall of the LtHash kernel) and the four alignment variants of the
// loader bloat an already 36 KB instruction stream.
//
// Here every thread owns two staging buffers in shared memory, word-major
// ([slot][thread], 8 bytes per thread: conflict-free LDS.64/STS.64). While block
// b is compressed from registers, data chunk b+1 is already on its way into the
// other buffer with cp.async (no registers involved). The T tag words of LtHash
// (LE64(index), or LE64(layer) || LE64(block)) are absorbed by sliding the
// window: a buffer's slots 0..T-1 hold the words carried over from the previous
// chunk (the tag for the first block), slots T..T+15 the chunk, and the message
// block is simply slots 0..15. One loop, one compress call site.
//
// The block/tail/carry bookkeeping is __host__ __device__; on the host the
// stager is a memcpy and tests/hostcheck runs it against hashlib.
#pragma once
#include "blake2b.cuh"

namespace snt {

constexpr int B2S_MAX_TAG_WORDS = 2;
constexpr int B2S_SLOTS = 16 + B2S_MAX_TAG_WORDS;     // carried/tag words + 16 chunk words

#if defined(__CUDACC__)
// 8 * sigma[r][j]: byte offset of message word sigma[r][j] in a staging buffer of stride 1 (compress_staged)
#define SNT_B2S_ROW(a, b, c, d, e, f, g, h, i, j, k, l, m, n, o, p) \
    {8 * a, 8 * b, 8 * c, 8 * d, 8 * e, 8 * f, 8 * g, 8 * h, 8 * i, 8 * j, 8 * k, 8 * l, 8 * m, 8 * n, 8 * o, 8 * p}
__constant__ uint32_t c_b2s_sigma8[13][16] = {
    SNT_B2S_ROW(0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15),
    SNT_B2S_ROW(14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3),
    SNT_B2S_ROW(11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4),
    SNT_B2S_ROW(7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8),
    SNT_B2S_ROW(9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13),
    SNT_B2S_ROW(2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9),
    SNT_B2S_ROW(12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11),
    SNT_B2S_ROW(13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10),
    SNT_B2S_ROW(6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5),
    SNT_B2S_ROW(10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0),
    SNT_B2S_ROW(0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15),
    SNT_B2S_ROW(14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3),
    SNT_B2S_ROW(0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15)};
#undef SNT_B2S_ROW
#endif

// STRIDE = 8-byte words between consecutive slots of one thread (= threads per CTA on the
// device, 1 on the host).
template <int STRIDE>
struct Blake2bStaged : Blake2b {
    // One compression with the message block LEFT in the staging buffer `cur` (this thread's slot 0): on the
    // device the twelve rounds are one loop body that fetches its sixteen message words in sigma order with
    // LDS at offsets from the constant bank -- 3 KB of code instead of the 34 KB of the unrolled rounds, and
    // no 32 registers of message. Kernels whose warps sit at many different places of a large instruction
    // stream (LtHash over short ragged samples: ncu showed no_instruction as the top stall, 22 % of the
    // samples, instruction-cache hit rate 74 %) run faster this way; the long regular leaf loop of the Merkle
    // kernel keeps the unrolled form.
    SNT_HD static void compress_staged(uint64_t h[8], const uint64_t* cur, uint64_t t, bool last) {
#ifdef __CUDA_ARCH__
        uint64_t v0 = h[0], v1 = h[1], v2 = h[2], v3 = h[3], v4 = h[4], v5 = h[5], v6 = h[6], v7 = h[7];
        uint64_t v8 = SNT_B2B_IV0, v9 = SNT_B2B_IV1, v10 = SNT_B2B_IV2, v11 = SNT_B2B_IV3;
        uint64_t v12 = SNT_B2B_IV4 ^ t, v13 = SNT_B2B_IV5;
        uint64_t v14 = last ? ~SNT_B2B_IV6 : SNT_B2B_IV6, v15 = SNT_B2B_IV7;
        const char* base = reinterpret_cast<const char*>(cur);
#define SNT_B2S_LOAD(m, r) \
    _Pragma("unroll") for (int j = 0; j < 16; ++j) m[j] = *reinterpret_cast<const uint64_t*>(base + c_b2s_sigma8[r][j] * STRIDE)
#define SNT_B2S_ROUND(m)                         \
    SNT_B2B_G(v0, v4, v8, v12, m[0], m[1]);      \
    SNT_B2B_G(v1, v5, v9, v13, m[2], m[3]);      \
    SNT_B2B_G(v2, v6, v10, v14, m[4], m[5]);     \
    SNT_B2B_G(v3, v7, v11, v15, m[6], m[7]);     \
    SNT_B2B_G(v0, v5, v10, v15, m[8], m[9]);     \
    SNT_B2B_G(v1, v6, v11, v12, m[10], m[11]);   \
    SNT_B2B_G(v2, v7, v8, v13, m[12], m[13]);    \
    SNT_B2B_G(v3, v4, v9, v14, m[14], m[15])
        // two rounds per trip, the message words of a round fetched while the round before it runs
        uint64_t ma[16], mb[16];
        SNT_B2S_LOAD(ma, 0);
#pragma unroll 1
        for (int r = 0; r < 12; r += 2) {
            SNT_B2S_LOAD(mb, r + 1);
            SNT_B2S_ROUND(ma);
            SNT_B2S_LOAD(ma, r + 2);             // (row 12 of the table repeats row 0: loaded, never used)
            SNT_B2S_ROUND(mb);
        }
#undef SNT_B2S_LOAD
#undef SNT_B2S_ROUND
        h[0] ^= v0 ^ v8;  h[1] ^= v1 ^ v9;  h[2] ^= v2 ^ v10; h[3] ^= v3 ^ v11;
        h[4] ^= v4 ^ v12; h[5] ^= v5 ^ v13; h[6] ^= v6 ^ v14; h[7] ^= v7 ^ v15;
#else
        uint64_t m[16];
        for (int i = 0; i < 16; ++i) m[i] = cur[i * STRIDE];
        compress(h, m, t, last);
#endif
    }

    // Copy the 128-byte chunk at g into slots T..T+15 of `buf`: asynchronously (cp.async, 8
    // bytes at a time) when g is 8-byte aligned, through registers otherwise.
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
    // wait until at most N of this thread's committed copy groups are still in flight
    template <int N>
    SNT_HD static void wait_pending() {
#ifdef __CUDA_ARCH__
        asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
#endif
    }

    // H(T tag words || data[0..len)), any data alignment. `bufs` points at this thread's slot
    // 0 of buffer 0; buffer 1 starts B2S_SLOTS * STRIDE words later.
    //   T = 0  plain BLAKE2b                      (Merkle leaves, hash_blocks; compression.py:70-74)
    //   T = 1  LE64(index) in front               (LtHash, lattice.py:92-94)
    //   T = 2  LE64(layer) || LE64(block) in front (per-layer lattice, model.py:259)
    template <int T>
    SNT_HD static uint64_t block_count(uint64_t len) {
        const uint64_t total = len + 8ull * T;
        return total == 0 ? 1 : ((total + 127) >> 7);
    }

    // Compress message blocks [b0, b1) (clipped to the message's block count) into h, which holds
    // the chaining value after block b0 - 1 (init(h) for b0 = 0). A message can therefore be hashed
    // in slices, by different threads if need be: nothing but h travels between slices -- the T
    // carried words of block b0 are re-read from the message itself.
    // ROLLED: compress straight from the staging buffer (compress_staged) instead of from registers.
    template <int T, bool ROLLED = false>
    SNT_HD static void hash_blocks(uint64_t* bufs, uint64_t tag0, uint64_t tag1, const uint8_t* p, uint64_t len,
                                   uint64_t b0, uint64_t b1, uint64_t h[8]) {
        static_assert(T >= 0 && T <= B2S_MAX_TAG_WORDS, "unsupported tag width");
        uint64_t* const buf0 = bufs;
        uint64_t* const buf1 = bufs + B2S_SLOTS * STRIDE;
        const uint64_t nfull = len >> 7;                 // whole 128-byte chunks of data
        const uint32_t r = static_cast<uint32_t>(len & 127);
        const uint64_t total = len + 8ull * T;
        const uint64_t nblocks = total == 0 ? 1 : ((total + 127) >> 7);
        const uint8_t* q = p + (nfull << 7);             // the ragged tail, r bytes
        if (b1 > nblocks) b1 = nblocks;
        if (b0 >= b1) return;
        uint64_t* const first = (b0 & 1) ? buf1 : buf0;
        if (b0 < nfull) stage_chunk<T>(first, p + (b0 << 7));
        commit();
        if (b0 == 0) {
            if (T >= 1) first[0] = tag0;
            if (T >= 2) first[STRIDE] = tag1;
        } else if (T > 0 && b0 <= nfull) {
            // resuming: the words carried into block b0 are the last T words of data chunk b0 - 1
            uint64_t carry[T > 0 ? T : 1];
            load_words64<(T > 0 ? T : 1)>(p + (b0 << 7) - 8 * T, carry);
#pragma unroll
            for (int i = 0; i < T; ++i) first[i * STRIDE] = carry[i];
        }
        for (uint64_t b = b0; b < b1; ++b) {
            uint64_t* cur = (b & 1) ? buf1 : buf0;
            uint64_t* nxt = (b & 1) ? buf0 : buf1;
            if (b + 1 < nfull && b + 1 < b1) stage_chunk<T>(nxt, p + ((b + 1) << 7));
            commit();
            if (b < nfull) {
                wait_pending<1>();                        // chunk b has landed in slots T..T+15
            } else if (b == nfull) {
                // first tail block: the carried words are in slots 0..T-1 already
#pragma unroll 1
                for (int j = 0; j < 16 - T; ++j) cur[(T + j) * STRIDE] = tail_word64(q, j, r);
            } else {
                // second tail block (8T + r > 128): the tail words that did not fit
#pragma unroll 1
                for (int j = 0; j < 16; ++j) cur[j * STRIDE] = j < T ? tail_word64(q, 16 - T + j, r) : 0ull;
            }
            const bool last = b + 1 == nblocks;
            if (ROLLED) {
#pragma unroll
                for (int i = 0; i < T; ++i) nxt[i * STRIDE] = cur[(16 + i) * STRIDE];   // carry for the next block
                compress_staged(h, cur, last ? total : ((b + 1) << 7), last);
            } else {
                uint64_t m[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) m[i] = cur[i * STRIDE];
#pragma unroll
                for (int i = 0; i < T; ++i) nxt[i * STRIDE] = cur[(16 + i) * STRIDE];   // carry for the next block
                compress(h, m, last ? total : ((b + 1) << 7), last);
            }
        }
    }

    template <int T, bool ROLLED = false>
    SNT_HD static void hash_message(uint64_t* bufs, uint64_t tag0, uint64_t tag1, const uint8_t* p, uint64_t len,
                                    uint64_t h[8]) {
        init(h);
        hash_blocks<T, ROLLED>(bufs, tag0, tag1, p, len, 0, ~0ull, h);
    }
};

}  // namespace snt
