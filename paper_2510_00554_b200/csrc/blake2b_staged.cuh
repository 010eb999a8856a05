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

// STRIDE = 8-byte words between consecutive slots of one thread (= threads per CTA on the
// device, 1 on the host).
template <int STRIDE>
struct Blake2bStaged : Blake2b {
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
    template <int T>
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
            uint64_t m[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) m[i] = cur[i * STRIDE];
#pragma unroll
            for (int i = 0; i < T; ++i) nxt[i * STRIDE] = cur[(16 + i) * STRIDE];   // carry for the next block
            const bool last = b + 1 == nblocks;
            compress(h, m, last ? total : ((b + 1) << 7), last);
        }
    }

    template <int T>
    SNT_HD static void hash_message(uint64_t* bufs, uint64_t tag0, uint64_t tag1, const uint8_t* p, uint64_t len,
                                    uint64_t h[8]) {
        init(h);
        hash_blocks<T>(bufs, tag0, tag1, p, len, 0, ~0ull, h);
    }
};

}  // namespace snt
