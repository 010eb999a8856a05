// LtHash for SMALL launches: four lanes per item (blake2b_quad.cuh). A loader batch of 128 rows, a process_batch of
// 128 host records, a single hash_sample -- a few warps of work on a 148-SM GPU -- are pure latency: one thread per
// item needs 2.6-3 us per 128-byte block (one warp alone on its scheduler, ALU pipe at half rate), 70 us for 128
// CIFAR-sized rows. Four lanes share an item's compression (a quarter of the G functions each, 12 shuffles per
// round) and halve that. Throughput per SM is LOWER than lthash_kernel's (0.28 vs 0.22 ms on 50,000 samples), so
// launch_lthash uses this kernel only up to LT_QUAD_MAX_ITEMS items (one launch over 128 rows of 3 KB: 47 us
// instead of 76; over 128 ragged token arrays: 21 instead of 35-45).
//
// Reference behaviour as lthash_kernel: lattice.py:92-101, dataset.py:41-49, :74-86 (per-source sums, counts,
// undeclared sources skipped and counted).
#pragma once
#include "blake2b_quad.cuh"
#include "lthash_kernels.cuh"

namespace snt {

constexpr int LT_QUAD_THREADS = 128;                           // 32 items per CTA
// Above this the one-thread-per-item kernels take over. tools/small_batch_probe.py, one launch, microseconds
// (quad / grid or lanes): 3 KB rows 47 / 76 up to 4,096 items, 54 / 82 at 8,192, 70 / 82 at 12,288, 92 / 90 at
// 16,384, 174 / 139 at 32,768; ragged token arrays 21 / 35 at 128, 24 / 36 at 8,192, 27 / 36 at 12,288, 34 / 36 at
// 16,384, 54 / 52 at 32,768.
constexpr uint64_t LT_QUAD_MAX_ITEMS = 12288;

template <class Items, bool SMEM_ACC>
__global__ void __launch_bounds__(LT_QUAD_THREADS)
lthash_quad_kernel(const Items items, uint64_t n, uint32_t n_sources, unsigned long long* __restrict__ acc,
                   unsigned long long* __restrict__ counts, uint8_t* __restrict__ digests,
                   unsigned long long* __restrict__ status) {
    // dynamic shared memory: one message-block region per quad, then (SMEM_ACC) the per-CTA accumulators
    extern __shared__ __align__(16) uint8_t lt_smem[];
    constexpr int QUADS = LT_QUAD_THREADS / 4;
    uint8_t* const region = lt_smem + (threadIdx.x >> 2) * QUAD_REGION_BYTES;
    uint32_t* const sacc = reinterpret_cast<uint32_t*>(lt_smem + QUADS * QUAD_REGION_BYTES);
    uint32_t* const scnt = sacc + static_cast<size_t>(n_sources) * LT_LANES;
    if (SMEM_ACC) {
        for (uint32_t i = threadIdx.x; i < n_sources * (LT_LANES + 1); i += LT_QUAD_THREADS) sacc[i] = 0;
        __syncthreads();
    }
    const QuadLane q = quad_lane();
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * QUADS + (threadIdx.x >> 2);
    if (i < n) {
        const LtItem it = items.get(i);                        // (all four lanes of the quad: the same item)
        if (it.slot >= n_sources) {
            if (status && q.c == 0) atomicAdd(status, 1ull);   // undeclared source (dataset.py:78-80): counted once, skipped
        } else {
            uint64_t h_lo, h_hi;                               // digest words c and 4 + c
            Blake2bQuad::template hash_message<Items::TAG_WORDS>(region, q, it.tag, it.tag1, it.ptr, it.len, h_lo, h_hi);
            if (digests) {
                uint64_t* o = reinterpret_cast<uint64_t*>(digests + i * 64);
                o[q.c] = h_lo;
                o[4 + q.c] = h_hi;
            }
            // u16 lanes 4c .. 4c+3 (from word c) and 16+4c .. 16+4c+3 (from word 4 + c)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t lo = static_cast<uint32_t>(h_lo >> (16 * k)) & 0xffffu;
                const uint32_t hi = static_cast<uint32_t>(h_hi >> (16 * k)) & 0xffffu;
                const size_t a = static_cast<size_t>(it.slot) * LT_LANES + 4 * q.c + k;
                if (SMEM_ACC) {
                    atomicAdd(sacc + a, lo);
                    atomicAdd(sacc + a + 16, hi);
                } else {
                    atomicAdd(acc + a, static_cast<unsigned long long>(lo));
                    atomicAdd(acc + a + 16, static_cast<unsigned long long>(hi));
                }
            }
            if (q.c == 0) {
                if (SMEM_ACC) atomicAdd(scnt + it.slot, 1u);
                else atomicAdd(counts + it.slot, 1ull);
            }
        }
    }
    if (SMEM_ACC) {
        __syncthreads();
        for (uint32_t j = threadIdx.x; j < n_sources * LT_LANES; j += LT_QUAD_THREADS) {
            const uint32_t v = sacc[j];
            if (v) atomicAdd(acc + j, static_cast<unsigned long long>(v));
        }
        for (uint32_t j = threadIdx.x; j < n_sources; j += LT_QUAD_THREADS) {
            const uint32_t v = scnt[j];
            if (v) atomicAdd(counts + j, static_cast<unsigned long long>(v));
        }
    }
}

}  // namespace snt
