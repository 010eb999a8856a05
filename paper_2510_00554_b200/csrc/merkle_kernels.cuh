// Merkle kernels: leaf hashing (one thread per leaf, fragmented tensors hashed
// where they lie) and the level reducer (thread-local subtree, then warp
// shuffles, then one shared-memory hop).
//
// Reference behaviour reproduced:
//   leaf stage   merkle.py:93-114 (hash_blocks) over model.py:137-146 (BlockTable)
//   level rule   merkle.py:117-149 (reduce_level): out[j] = H(in[2j] || in[2j+1]),
//                an odd level pairs its last node with dlen zero bytes
//   root         merkle.py:152-165 (single leaf is returned unchanged)
#pragma once
#include "algs.cuh"

namespace snt {

constexpr int LEAF_THREADS = 128;
constexpr int REDUCE_THREADS = 256;
constexpr int REDUCE_LOCAL_LEVELS = 2;                       // 4 digests per thread
constexpr int REDUCE_MAX_LEVELS = REDUCE_LOCAL_LEVELS + 8;   // 1024 digests per CTA

// ---- leaf hashing -----------------------------------------------------------

// SHA-256 of a full leaf whose length is a multiple of 64 and whose address is
// 16-byte aligned: 4 x LDG.128 per compression with the next block's loads
// issued before the current block's rounds, then the constant padding block.
SNT_HD void sha256_leaf_aligned(const uint8_t* __restrict__ p, uint32_t nblk,
                               const uint32_t* __restrict__ pad_kw, uint32_t s[8]) {
    Sha256::init(s);
    U4 q0 = ld128(p), q1 = ld128(p + 16), q2 = ld128(p + 32), q3 = ld128(p + 48);
#pragma unroll 1
    for (uint32_t b = 0; b < nblk; ++b) {
        uint32_t w[16];
        w[0] = bswap32(q0.x);  w[1] = bswap32(q0.y);  w[2] = bswap32(q0.z);  w[3] = bswap32(q0.w);
        w[4] = bswap32(q1.x);  w[5] = bswap32(q1.y);  w[6] = bswap32(q1.z);  w[7] = bswap32(q1.w);
        w[8] = bswap32(q2.x);  w[9] = bswap32(q2.y);  w[10] = bswap32(q2.z); w[11] = bswap32(q2.w);
        w[12] = bswap32(q3.x); w[13] = bswap32(q3.y); w[14] = bswap32(q3.z); w[15] = bswap32(q3.w);
        if (b + 1 < nblk) {
            const uint8_t* n = p + (static_cast<size_t>(b + 1) << 6);
            q0 = ld128(n); q1 = ld128(n + 16); q2 = ld128(n + 32); q3 = ld128(n + 48);
        }
        Sha256::compress(s, w);
    }
    Sha256::compress_const(s, pad_kw);
}

template <int ALG>
SNT_D void store_digest(uint8_t* out, const uint32_t* d) {
    using A = AlgTraits<ALG>;
    uint4* o = reinterpret_cast<uint4*>(out);
#pragma unroll
    for (int i = 0; i < A::DW / 4; ++i) {
        o[i] = make_uint4(A::to_mem(d[4 * i]), A::to_mem(d[4 * i + 1]), A::to_mem(d[4 * i + 2]),
                          A::to_mem(d[4 * i + 3]));
    }
}

template <int ALG>
SNT_D void load_digest(const uint8_t* in, uint32_t* d) {
    using A = AlgTraits<ALG>;
    const uint4* q = reinterpret_cast<const uint4*>(in);
#pragma unroll
    for (int i = 0; i < A::DW / 4; ++i) {
        const uint4 v = q[i];
        d[4 * i] = A::from_mem(v.x); d[4 * i + 1] = A::from_mem(v.y);
        d[4 * i + 2] = A::from_mem(v.z); d[4 * i + 3] = A::from_mem(v.w);
    }
}

// One thread per leaf of [leaf_begin, leaf_end); digest k is written at
// d_leaves + (k - leaf_begin) * DIGEST_BYTES.
template <int ALG>
__global__ void __launch_bounds__(LEAF_THREADS)
merkle_leaf_kernel(const TensorTable tab, const __grid_constant__ MerkleConsts c,
                   uint64_t leaf_begin, uint64_t leaf_end, uint8_t* __restrict__ d_leaves) {
    using A = AlgTraits<ALG>;
    const uint64_t k = leaf_begin + static_cast<uint64_t>(blockIdx.x) * LEAF_THREADS + threadIdx.x;
    const bool exists = k < leaf_end;
    LeafRef leaf{nullptr, 0};
    if (exists) leaf = locate_leaf(tab, k);
    uint32_t d[A::DW];
    if (ALG == ALG_SHA256) {
        const bool fast = exists && leaf.len == (1ull << tab.block_shift) &&
                          (reinterpret_cast<uintptr_t>(leaf.ptr) & 15) == 0;
        if (__all_sync(0xffffffffu, fast)) {
            sha256_leaf_aligned(leaf.ptr, 1u << (tab.block_shift - 6), c.sha256_pad_leaf, d);
        } else if (exists) {
            A::leaf(leaf.ptr, leaf.len, d);
        }
    } else {
        if (exists) A::leaf(leaf.ptr, leaf.len, d);
    }
    if (exists) store_digest<ALG>(d_leaves + (k - leaf_begin) * A::DIGEST_BYTES, d);
}

// hash_blocks over an explicit (address, length) list: entry i = H(block i)
// (merkle.py:93-114). Blocks may be empty, ragged and unaligned.
template <int ALG>
__global__ void __launch_bounds__(LEAF_THREADS)
hash_blocks_kernel(const uint8_t* __restrict__ base, const uint64_t* __restrict__ off,
                   const uint64_t* __restrict__ len, uint64_t n, uint8_t* __restrict__ out) {
    using A = AlgTraits<ALG>;
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * LEAF_THREADS + threadIdx.x;
    if (i >= n) return;
    uint32_t d[A::DW];
    A::leaf(base + off[i], len[i], d);
    store_digest<ALG>(out + i * A::DIGEST_BYTES, d);
}

// ---- level reducer ------------------------------------------------------------
//
// Input: nodes of one tree level with global indices [first, first + n_in);
// `level_count` is the number of nodes the whole tree has at that level (a
// node index >= level_count does not exist and pairs as zeros). Each CTA
// applies `levels` (1..REDUCE_MAX_LEVELS) levels to its aligned group of
// 2^levels inputs and writes one node. Levels are never skipped: a group that
// is down to one node keeps pairing it with zeros, which is exactly what the
// reference tree does to the last node of every odd level and what makes
// per-shard roots combine into the reference root.

template <int ALG>
SNT_D void pair_or_pad(uint32_t* left, const uint32_t* right, bool right_exists,
                       const MerkleConsts& c) {
    using A = AlgTraits<ALG>;
    uint32_t r[A::DW];
#pragma unroll
    for (int i = 0; i < A::DW; ++i) r[i] = right_exists ? right[i] : 0u;
    uint32_t out[A::DW];
    A::pair(left, r, c, out);
#pragma unroll
    for (int i = 0; i < A::DW; ++i) left[i] = out[i];
}

// `nlev` shuffle levels inside a warp. Lane l holds node index g (at relative
// level t) when l is a multiple of `stride`; holders that are multiples of
// 2*stride become the parents.
template <int ALG>
SNT_D void warp_levels(uint32_t* d, uint64_t& g, uint32_t& t, uint32_t nlev, uint32_t stride0,
                       uint64_t level_count, const MerkleConsts& c) {
    using A = AlgTraits<ALG>;
    uint32_t stride = stride0;
    for (uint32_t s = 0; s < nlev; ++s) {
        uint32_t r[A::DW];
#pragma unroll
        for (int i = 0; i < A::DW; ++i) r[i] = __shfl_down_sync(0xffffffffu, d[i], stride);
        const bool right_exists = (g + 1) < ceil_shift(level_count, t);
        pair_or_pad<ALG>(d, r, right_exists, c);
        g >>= 1;
        t += 1;
        stride <<= 1;
    }
}

template <int ALG>
__global__ void __launch_bounds__(REDUCE_THREADS)
merkle_reduce_kernel(const uint8_t* __restrict__ in, uint64_t first, uint64_t n_in,
                     uint64_t level_count, uint32_t levels, const __grid_constant__ MerkleConsts c,
                     uint8_t* __restrict__ out) {
    using A = AlgTraits<ALG>;
    constexpr int DW = A::DW;
    __shared__ uint32_t xwarp[REDUCE_THREADS / 32][DW];

    const uint32_t a = levels < REDUCE_LOCAL_LEVELS ? levels : REDUCE_LOCAL_LEVELS;  // thread-local levels
    const uint32_t r = levels - a;                                                    // cooperative levels
    const uint32_t nthreads = 1u << r;                                                // threads holding data
    const uint32_t tid = threadIdx.x;
    const uint32_t lane = tid & 31;

    // node index (at the input level) of this thread's first input
    const uint64_t gi = first + (static_cast<uint64_t>(blockIdx.x) << levels) +
                        (static_cast<uint64_t>(tid) << a);
    const uint64_t in_end = first + n_in;

    uint32_t d[DW];
#pragma unroll
    for (int i = 0; i < DW; ++i) d[i] = 0;
    uint64_t g = gi;      // index of the node this thread holds, at relative level t
    uint32_t t = 0;

    if (tid < nthreads) {
        // thread-local subtree over 2^a consecutive inputs
        uint32_t n1[DW], n2[DW], n3[DW];
        const bool e0 = gi < in_end;
        if (e0) load_digest<ALG>(in + (gi - first) * A::DIGEST_BYTES, d);
        if (a >= 1) {
            const bool e1 = gi + 1 < in_end;
            if (e1) load_digest<ALG>(in + (gi + 1 - first) * A::DIGEST_BYTES, n1);
            if (a >= 2) {
                const bool e2 = gi + 2 < in_end, e3 = gi + 3 < in_end;
                if (e2) load_digest<ALG>(in + (gi + 2 - first) * A::DIGEST_BYTES, n2);
                if (e3) load_digest<ALG>(in + (gi + 3 - first) * A::DIGEST_BYTES, n3);
                if (e2) pair_or_pad<ALG>(n2, n3, e3, c);
            }
            if (e0) pair_or_pad<ALG>(d, n1, e1, c);
            if (a >= 2) {
                // level 1 -> 2: right child (gi>>1)+1 exists iff it is inside the tree
                const bool r_exists = ((gi >> 1) + 1) < ceil_shift(level_count, 1);
                if (e0) pair_or_pad<ALG>(d, n2, r_exists, c);
            }
        }
    }
    g = gi >> a;
    t = a;

    if (r > 0) {
        const uint32_t wl = r < 5 ? r : 5;
        warp_levels<ALG>(d, g, t, wl, 1, level_count, c);
        if (r > 5) {
            if (lane == 0) {
#pragma unroll
                for (int i = 0; i < DW; ++i) xwarp[tid >> 5][i] = d[i];
            }
            __syncthreads();
            if (tid < 32) {
                const uint32_t nw = nthreads >> 5;    // warps that held data (2, 4 or 8)
#pragma unroll
                for (int i = 0; i < DW; ++i) d[i] = lane < nw ? xwarp[lane][i] : 0u;
                g = ((first + (static_cast<uint64_t>(blockIdx.x) << levels)) >> t) + lane;
                warp_levels<ALG>(d, g, t, r - 5, 1, level_count, c);
            }
        }
    }
    if (tid == 0) store_digest<ALG>(out + static_cast<uint64_t>(blockIdx.x) * A::DIGEST_BYTES, d);
}

}  // namespace snt
