// Span gather: copy n byte spans that live anywhere in HBM into one destination buffer, optionally
// zero-padding every span to a multiple of `pad_block` bytes. One launch replaces the per-tensor copies
// of the two strategies that move data before hashing:
//   coalesce_hash   model.py:203-228  every tensor packed back to back (pad_block = 0)
//   per_layer_hash  model.py:245-253  the ragged last block of a tensor, zero-padded to the block size
//                                     (only the tails are copied; the full blocks are hashed in place)
// Work unit = one 32 KiB chunk of one span; chunk c belongs to the span s with
// chunk_first[s] <= c < chunk_first[s + 1] (binary search, like the leaf locator).
#pragma once
#include "common.cuh"

namespace snt {

constexpr uint32_t GATHER_CHUNK_BYTES = 32u << 10;
constexpr int GATHER_THREADS = 256;

__global__ void __launch_bounds__(GATHER_THREADS)
gather_spans_kernel(const uint64_t* __restrict__ src_addr, const uint64_t* __restrict__ len,
                    const uint64_t* __restrict__ dst_off, const uint64_t* __restrict__ chunk_first,
                    uint32_t n_spans, uint32_t pad_block, uint8_t* __restrict__ dst) {
    const uint64_t chunk = blockIdx.x;
    uint32_t lo = 0, hi = n_spans;                 // invariant: chunk_first[lo] <= chunk < chunk_first[hi]
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (chunk_first[mid] <= chunk) lo = mid; else hi = mid;
    }
    const uint64_t n = len[lo];
    const uint64_t padded = pad_block ? (n + pad_block - 1) / pad_block * pad_block : n;
    const uint64_t begin = (chunk - chunk_first[lo]) * GATHER_CHUNK_BYTES;
    const uint64_t end = begin + GATHER_CHUNK_BYTES < padded ? begin + GATHER_CHUNK_BYTES : padded;
    const uint8_t* s = reinterpret_cast<const uint8_t*>(src_addr[lo]);
    uint8_t* d = dst + dst_off[lo];
    const uint64_t data_end = end < n ? end : n;                       // bytes of this chunk that come from the span
    uint64_t q0 = begin;                                               // first byte not yet copied
    if (data_end > begin) {
        const uintptr_t sa = reinterpret_cast<uintptr_t>(s + begin), da = reinterpret_cast<uintptr_t>(d + begin);
        if (((sa | da) & 15) == 0) {
            // source and destination 16-byte aligned: 128-bit units, four independent loads in flight
            const uint32_t units = static_cast<uint32_t>((data_end - begin) >> 4);
            const uint4* s4 = reinterpret_cast<const uint4*>(s + begin);
            uint4* d4 = reinterpret_cast<uint4*>(d + begin);
            uint32_t u = threadIdx.x;
            for (; u + 3 * GATHER_THREADS < units; u += 4 * GATHER_THREADS) {
                const uint4 a = __ldg(s4 + u), b = __ldg(s4 + u + GATHER_THREADS),
                            c = __ldg(s4 + u + 2 * GATHER_THREADS), e = __ldg(s4 + u + 3 * GATHER_THREADS);
                d4[u] = a; d4[u + GATHER_THREADS] = b; d4[u + 2 * GATHER_THREADS] = c; d4[u + 3 * GATHER_THREADS] = e;
            }
            for (; u < units; u += GATHER_THREADS) d4[u] = __ldg(s4 + u);
            q0 = begin + (static_cast<uint64_t>(units) << 4);
        } else {
            // general case: the destination decides the word grid (4-byte stores); a source that sits at a
            // different byte phase is read as aligned words and funnel-shifted. The first and last aligned
            // source words each hold at least one byte of the span, so the reads stay inside its granules.
            const uint32_t head = static_cast<uint32_t>((4 - (da & 3)) & 3);
            const uint64_t body = begin + head;
            if (body + 8 <= data_end) {
                const uint32_t words = static_cast<uint32_t>((data_end - body) >> 2) - 1;   // keeps sp[w + 1] in range
                const uint32_t a = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(s + body) & 3);
                const uint32_t* sp = reinterpret_cast<const uint32_t*>(s + body - a);
                uint32_t* dp = reinterpret_cast<uint32_t*>(d + body);
                for (uint32_t w = threadIdx.x; w < words; w += GATHER_THREADS) {
                    const uint32_t lo = __ldg(sp + w);
                    dp[w] = a ? funnel_bytes(lo, __ldg(sp + w + 1), a) : lo;
                }
                for (uint64_t q = begin + threadIdx.x; q < body; q += GATHER_THREADS) d[q] = __ldg(s + q);
                q0 = body + (static_cast<uint64_t>(words) << 2);
            }
        }
    }
    // edges: the last few bytes of the data and the zero padding
    for (uint64_t q = q0 + threadIdx.x; q < end; q += GATHER_THREADS) d[q] = q < n ? __ldg(s + q) : uint8_t(0);
}

}  // namespace snt
