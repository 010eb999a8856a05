// LtHash kernels: BLAKE2b-512 of (index tag || bytes) per item, the 64 digest
// bytes read as 32 little-endian u16 lanes, lanes summed per source modulo
// 2^16. Sums are carried wider and masked to 16 bits at the end (exact modulo
// 2^16 for any count): in u32 in shared memory per CTA, in u64 in the global
// accumulator -- u64 because lanes, counts and the status word then form ONE
// array of one type, and a single 64-bit sum all-reduce combines the partial
// accumulators of several GPUs with nothing to pack or unpack.
//
// Reference behaviour reproduced:
//   lattice.py:92-101   lt_hash_block / lt_hash_tagged
//   lattice.py:69-82    lt_add (per-lane add mod 2^16), :104-119 lt_reduce
//   dataset.py:41-49    hash_sample, :74-86 process_batch (group by source, sum)
//   model.py:183-193    _lattice_sum_blocks with tag LE64(k) (model.py:312)
#pragma once
#include "algs.cuh"
#include "blake2b_staged.cuh"
#include "chain_sched.cuh"

namespace snt {

#ifndef SNT_LT_GRID_ROLLED
#define SNT_LT_GRID_ROLLED 0
#endif
// 1 = the grid kernel compresses from the staging buffer with rolled rounds (Blake2bStaged::compress_staged). Measured:
// better on ragged samples (2 M: 2.94 -> 2.06 ms), worse on samples of one length (CIFAR 194 -> 220 us) -- and ragged
// samples take the lane kernel anyway, so the grid keeps the unrolled rounds.
constexpr bool LT_GRID_ROLLED = SNT_LT_GRID_ROLLED != 0;
#ifndef SNT_LT_THREADS
#define SNT_LT_THREADS 64
#endif
constexpr int LT_THREADS = SNT_LT_THREADS;
constexpr int LT_LANES = 32;                 // u16 lanes per digest
constexpr int LT_SMEM_SOURCES = 128;         // per-CTA shared accumulators: 128 x 32 x 4 B = 16 KiB

struct LtItem {
    const uint8_t* ptr;
    uint64_t len;
    uint64_t tag;         // first tag word: LE64(index)
    uint64_t tag1;        // second tag word (per-layer tags LE64(layer) || LE64(block)), else unused
    uint32_t slot;
};

// Dataset samples: a flat shard plus (offset, length, sample_id, source slot)
// rows -- the manifest layout of dataset.py:94-100 moved to device arrays.
struct SampleItems {
    const uint8_t* __restrict__ shard;
    const uint64_t* __restrict__ off;
    const uint64_t* __restrict__ len;
    const uint64_t* __restrict__ ids;
    const uint32_t* __restrict__ slot;
    static constexpr int TAG_WORDS = 1;
    static constexpr bool LONG_ITEMS = false;          // samples: tens of BLAKE2b blocks at most (see launch_lthash)
    SNT_HD LtItem get(uint64_t i) const {
        LtItem it;
        it.ptr = shard + off[i];
        it.len = len[i];
        it.tag = ids[i];
        it.tag1 = 0;
        it.slot = slot[i];
        return it;
    }
};

// Loader batches (dataset.StreamingDatasetHasher): n fixed-size rows of ONE tensor, as a GPU data loader holds a
// batch. The source slot of a row is found INSIDE the kernel, by binary search of its source id in the sorted
// table of declared ids (an id that is not there gets slot n_table = undeclared, counted in the status word,
// dataset.py:78-80) -- one launch per batch and no index arithmetic around it.
struct RowItems {
    const uint8_t* __restrict__ rows;
    uint64_t row_bytes;
    const uint64_t* __restrict__ ids;
    const long long* __restrict__ src;
    const long long* __restrict__ table;
    uint32_t n_table;
    static constexpr int TAG_WORDS = 1;
    static constexpr bool LONG_ITEMS = false;
    SNT_HD LtItem get(uint64_t i) const {
        LtItem it;
        it.ptr = rows + i * row_bytes;
        it.len = row_bytes;
        it.tag = ids[i];
        it.tag1 = 0;
        const long long want = src[i];
        uint32_t lo = 0, hi = n_table;                 // first entry >= want
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (table[mid] < want) lo = mid + 1; else hi = mid;
        }
        it.slot = (lo < n_table && table[lo] == want) ? lo : n_table;
        return it;
    }
};

// Model blocks hashed in place: item i is leaf k = leaf_begin + i of the block
// table, tagged with the global block counter k (model.py:312).
struct LeafItems {
    TensorTable tab;
    uint64_t leaf_begin;
    static constexpr int TAG_WORDS = 1;
    static constexpr bool LONG_ITEMS = true;           // model blocks: 8 KiB = 65 BLAKE2b blocks each
    SNT_HD LtItem get(uint64_t i) const {
        const uint64_t k = leaf_begin + i;
        const LeafRef r = locate_leaf(tab, k);
        LtItem it;
        it.ptr = r.ptr;
        it.len = r.len;
        it.tag = k;
        it.tag1 = 0;
        it.slot = 0;
        return it;
    }
};

// Per-layer lattice hashing (model.py:255-262): block j of tensor i is tagged
// LE64(i) || LE64(j) and summed into accumulator slot i (one slot per tensor).
struct LayerLeafItems {
    TensorTable tab;
    uint64_t leaf_begin;
    static constexpr int TAG_WORDS = 2;
    static constexpr bool LONG_ITEMS = true;
    SNT_HD LtItem get(uint64_t i) const {
        const LeafRef r = locate_leaf(tab, leaf_begin + i);
        LtItem it;
        it.ptr = r.ptr;
        it.len = r.len;
        it.tag = r.tensor;
        it.tag1 = r.block;
        it.slot = r.tensor;
        return it;
    }
};

// Dynamic shared memory: the per-thread message staging buffers (blake2b_staged.cuh), then
// (SMEM_ACC) the per-CTA accumulators [n_sources][32] lanes + [n_sources] counts.
constexpr size_t LT_STAGE_BYTES = 2ull * B2S_SLOTS * LT_THREADS * sizeof(uint64_t);

template <class Items, bool SMEM_ACC>
__global__ void __launch_bounds__(LT_THREADS)
lthash_kernel(const Items items, uint64_t n, uint32_t n_sources, unsigned long long* __restrict__ acc,
              unsigned long long* __restrict__ counts, uint8_t* __restrict__ digests,
              unsigned long long* __restrict__ status) {
    extern __shared__ __align__(16) uint8_t lt_smem[];
    uint64_t* stage = reinterpret_cast<uint64_t*>(lt_smem) + threadIdx.x;
    uint32_t* sacc = reinterpret_cast<uint32_t*>(lt_smem + LT_STAGE_BYTES);
    uint32_t* scnt = sacc + static_cast<size_t>(n_sources) * LT_LANES;
    if (SMEM_ACC) {
        for (uint32_t i = threadIdx.x; i < n_sources * (LT_LANES + 1); i += LT_THREADS) sacc[i] = 0;
        __syncthreads();
    }
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * LT_THREADS + threadIdx.x;
    if (i < n) {
        const LtItem it = items.get(i);
        if (it.slot >= n_sources) {
            if (status) atomicAdd(status, 1ull);       // undeclared source (dataset.py:78-80): counted, skipped
        } else {
            uint64_t h[8];
            Blake2bStaged<LT_THREADS>::template hash_message<Items::TAG_WORDS, LT_GRID_ROLLED>(stage, it.tag, it.tag1, it.ptr, it.len, h);
            if (digests) {
                uint4* o = reinterpret_cast<uint4*>(digests + i * 64);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    o[q] = make_uint4(static_cast<uint32_t>(h[2 * q]), static_cast<uint32_t>(h[2 * q] >> 32),
                                      static_cast<uint32_t>(h[2 * q + 1]), static_cast<uint32_t>(h[2 * q + 1] >> 32));
                }
            }

            // rotate the lane order by the thread's lane id: at every step the
            // 32 threads of a warp hit 32 different shared-memory banks
            // whatever their sources are.
            const uint32_t rot = threadIdx.x & 31;
#pragma unroll
            for (int l = 0; l < LT_LANES; ++l) {
                const uint32_t lane = (l + rot) & 31;
                // u16 lane number (lane & 3) of 64-bit word (lane >> 2); the word is
                // picked with a select chain because h[] lives in registers
                uint64_t w = h[0];
#pragma unroll
                for (int q = 1; q < 8; ++q) w = (lane >> 2) == static_cast<uint32_t>(q) ? h[q] : w;
                const uint32_t v = static_cast<uint32_t>(w >> (16 * (lane & 3))) & 0xffffu;
                if (SMEM_ACC) atomicAdd(sacc + static_cast<size_t>(it.slot) * LT_LANES + lane, v);
                else atomicAdd(acc + static_cast<size_t>(it.slot) * LT_LANES + lane, static_cast<unsigned long long>(v));
            }
            if (SMEM_ACC) atomicAdd(scnt + it.slot, 1u);
            else atomicAdd(counts + it.slot, 1ull);
        }
    }
    if (SMEM_ACC) {
        __syncthreads();
        for (uint32_t j = threadIdx.x; j < n_sources * LT_LANES; j += LT_THREADS) {
            const uint32_t v = sacc[j];
            if (v) atomicAdd(acc + j, static_cast<unsigned long long>(v));
        }
        for (uint32_t j = threadIdx.x; j < n_sources; j += LT_THREADS) {
            const uint32_t v = scnt[j];
            if (v) atomicAdd(counts + j, static_cast<unsigned long long>(v));
        }
    }
}

// ---- persistent, time-sliced variant -----------------------------------------------------------
//
// The same per-item work scheduled like the Merkle leaf stage (chain_sched.cuh): one persistent CTA per
// SM owns a contiguous run of CHAINS (one warp x 32 consecutive items), W worker warps share them, and
// the last W + (count mod W) chains are executed in slices so that every scheduler keeps W/4 runnable
// warps until the SM is done. Used for model blocks in launches of a wave or two (LATTICE hashing of a
// GPT-2-sized model: 0.713 -> 0.664 ms); dataset samples are too short to pay for the per-slice queue
// operation and pipeline restart and keep the plain grid above (launch_lthash in capi.cu has the numbers).
// Only the BLAKE2b chaining value (16 words per lane) is parked between slices; the item itself is
// looked up again by the warp that resumes it. A chain is as long as its longest item.
constexpr int LT_CHAIN_MAXW = 8;                                     // worker warps (256 threads): BLAKE2b wants registers
constexpr int LT_CHAIN_STATE_WORDS = 16;
constexpr size_t LT_CHAIN_STAGE_BYTES = 2ull * B2S_SLOTS * LT_CHAIN_MAXW * 32 * sizeof(uint64_t);
constexpr size_t LT_CHAIN_PARK_BYTES = (2ull * LT_CHAIN_MAXW - 1) * LT_CHAIN_STATE_WORDS * 32 * sizeof(uint32_t);

template <class Items, bool SMEM_ACC>
__global__ void __launch_bounds__(LT_CHAIN_MAXW * 32, 1)
lthash_chain_kernel(const Items items, uint64_t n, uint32_t n_sources, unsigned long long* __restrict__ acc,
                    unsigned long long* __restrict__ counts, uint8_t* __restrict__ digests,
                    unsigned long long* __restrict__ status) {
    // dynamic shared memory: [message staging][parked chaining values][per-CTA accumulators + counts]
    extern __shared__ __align__(16) uint8_t lt_smem[];
    __shared__ FusedSched sc;
    constexpr int T = Items::TAG_WORDS;
    uint64_t* const stage = reinterpret_cast<uint64_t*>(lt_smem) + threadIdx.x;
    uint32_t* const park = reinterpret_cast<uint32_t*>(lt_smem + LT_CHAIN_STAGE_BYTES);
    uint32_t* const sacc = reinterpret_cast<uint32_t*>(lt_smem + LT_CHAIN_STAGE_BYTES + LT_CHAIN_PARK_BYTES);
    uint32_t* const scnt = sacc + static_cast<size_t>(n_sources) * LT_LANES;
    const int lane = threadIdx.x & 31;
    const int W = blockDim.x >> 5;
    if (SMEM_ACC)
        for (uint32_t i = threadIdx.x; i < n_sources * (LT_LANES + 1); i += blockDim.x) sacc[i] = 0;
    sched_init(&sc);                                                  // (ends with a barrier)

    const uint64_t R = (n + 31) >> 5;
    const uint64_t q = R / gridDim.x, rem = R % gridDim.x;
    const uint64_t first = blockIdx.x * q + (blockIdx.x < rem ? blockIdx.x : rem);
    const int count = static_cast<int>(q + (blockIdx.x < rem ? 1 : 0));
    const int first_sliced = sched_first_sliced(count, W);

    for (;;) {
        const int ch = sched_pop(&sc, count, lane);
        if (ch < 0) break;
        const bool sliced = ch >= first_sliced;
        const int slot = sliced ? ch - first_sliced : 0;
        uint32_t u0 = sliced ? static_cast<uint32_t>(*reinterpret_cast<volatile int*>(&sc.prog[slot])) : 0u;
        uint32_t* const st = park + static_cast<size_t>(slot) * LT_CHAIN_STATE_WORDS * 32 + lane;
        const uint64_t i = ((first + static_cast<uint64_t>(ch)) << 5) + lane;
        bool valid = i < n;
        LtItem it;
        it.ptr = nullptr; it.len = 0; it.tag = 0; it.tag1 = 0; it.slot = 0;
        if (valid) {
            it = items.get(i);
            if (it.slot >= n_sources) {                    // undeclared source (dataset.py:78-80): skipped, counted once
                valid = false;
                if (status && u0 == 0) atomicAdd(status, 1ull);
            }
        }
        const uint32_t mine = valid ? static_cast<uint32_t>(Blake2bStaged<1>::template block_count<T>(it.len)) : 0u;
        uint32_t units = mine;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint32_t other = __shfl_xor_sync(0xffffffffu, units, o);
            units = other > units ? other : units;
        }
        const uint32_t slice = (units + W - 1) / W > 4 ? (units + W - 1) / W : 4;   // at least 4 blocks between two parkings

        uint64_t h[8];
        if (u0 == 0) {
            Blake2b::init(h);
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) h[k] = (static_cast<uint64_t>(st[(2 * k + 1) * 32]) << 32) | st[2 * k * 32];
        }
        bool parked = false;
        for (;;) {
            const uint32_t u1 = sliced ? (u0 + slice < units ? u0 + slice : units) : units;
            if (valid) Blake2bStaged<LT_CHAIN_MAXW * 32>::template hash_blocks<T>(stage, it.tag, it.tag1, it.ptr, it.len, u0, u1, h);
            __syncwarp();
            if (u1 >= units) break;
            u0 = u1;
            if (!sched_waiting(&sc, count, lane)) continue;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                st[2 * k * 32] = static_cast<uint32_t>(h[k]);
                st[(2 * k + 1) * 32] = static_cast<uint32_t>(h[k] >> 32);
            }
            sched_park(&sc, ch, slot, u0, lane);
            parked = true;
            break;
        }
        if (parked || !valid) continue;

        // ---- item done: digest out (if asked for), lanes into the accumulators
        if (digests) {
            uint4* o = reinterpret_cast<uint4*>(digests + i * 64);
#pragma unroll
            for (int k = 0; k < 4; ++k)
                o[k] = make_uint4(static_cast<uint32_t>(h[2 * k]), static_cast<uint32_t>(h[2 * k] >> 32),
                                  static_cast<uint32_t>(h[2 * k + 1]), static_cast<uint32_t>(h[2 * k + 1] >> 32));
        }
#pragma unroll
        for (int l = 0; l < LT_LANES; ++l) {
            const uint32_t ln = (l + lane) & 31;           // rotated by the lane id: 32 different banks per step
            uint64_t w = h[0];
#pragma unroll
            for (int k = 1; k < 8; ++k) w = (ln >> 2) == static_cast<uint32_t>(k) ? h[k] : w;
            const uint32_t v = static_cast<uint32_t>(w >> (16 * (ln & 3))) & 0xffffu;
            if (SMEM_ACC) atomicAdd(sacc + static_cast<size_t>(it.slot) * LT_LANES + ln, v);
            else atomicAdd(acc + static_cast<size_t>(it.slot) * LT_LANES + ln, static_cast<unsigned long long>(v));
        }
        if (SMEM_ACC) atomicAdd(scnt + it.slot, 1u);
        else atomicAdd(counts + it.slot, 1ull);
    }
    if (SMEM_ACC) {
        __syncthreads();
        for (uint32_t j = threadIdx.x; j < n_sources * LT_LANES; j += blockDim.x) {
            const uint32_t v = sacc[j];
            if (v) atomicAdd(acc + j, static_cast<unsigned long long>(v));
        }
        for (uint32_t j = threadIdx.x; j < n_sources; j += blockDim.x) {
            const uint32_t v = scnt[j];
            if (v) atomicAdd(counts + j, static_cast<unsigned long long>(v));
        }
    }
}

// lt_reduce (lattice.py:104-119): sum n 64-byte digests into acc[32].
__global__ void __launch_bounds__(256)
lt_reduce_kernel(const uint8_t* __restrict__ digests, uint64_t n, unsigned long long* __restrict__ acc) {
    __shared__ uint32_t sacc[LT_LANES];
    if (threadIdx.x < LT_LANES) sacc[threadIdx.x] = 0;
    __syncthreads();
    // thread (j, q): 16-byte quarter q of digest j -> 8 lanes
    const uint32_t q = threadIdx.x & 3;
    uint32_t s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 2);
    for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * (blockDim.x >> 2) + (threadIdx.x >> 2); j < n;
         j += stride) {
        const uint4 v = *reinterpret_cast<const uint4*>(digests + j * 64 + q * 16);
        s[0] += v.x & 0xffffu; s[1] += v.x >> 16;
        s[2] += v.y & 0xffffu; s[3] += v.y >> 16;
        s[4] += v.z & 0xffffu; s[5] += v.z >> 16;
        s[6] += v.w & 0xffffu; s[7] += v.w >> 16;
    }
    // lanes with equal q sit 4 apart: fold them with shuffles, then one
    // shared atomic per warp and lane
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        uint32_t v = s[i];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        if ((threadIdx.x & 31) < 4) atomicAdd(&sacc[q * 8 + i], v);
    }
    __syncthreads();
    if (threadIdx.x < LT_LANES && sacc[threadIdx.x])
        atomicAdd(acc + threadIdx.x, static_cast<unsigned long long>(sacc[threadIdx.x]));
}

// Mask the widened sums to 16 bits and pack them little-endian: n_sources x 64
// bytes, the LatticeDigest layout of lattice.py:37-58.
__global__ void lt_finalize_kernel(const unsigned long long* __restrict__ acc, uint32_t n_words,
                                   uint32_t* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;   // output word = 2 lanes
    if (i < n_words)
        out[i] = (static_cast<uint32_t>(acc[2 * i]) & 0xffffu) | (static_cast<uint32_t>(acc[2 * i + 1]) << 16);
}

}  // namespace snt
