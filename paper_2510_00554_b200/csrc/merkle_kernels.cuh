// Merkle kernels of the multi-launch path: leaf hashing (one thread per leaf, fragmented tensors hashed
// where they lie) and the level reducer (level by level through shared memory with the active threads
// compacted). The single-launch path (merkle_fused.cuh) reuses the per-thread pieces defined here.
//
// Reference behaviour reproduced:
//   leaf stage   merkle.py:93-114 (hash_blocks) over model.py:137-146 (BlockTable)
//   level rule   merkle.py:117-149 (reduce_level): out[j] = H(in[2j] || in[2j+1]),
//                an odd level pairs its last node with dlen zero bytes
//   root         merkle.py:152-165 (single leaf is returned unchanged)
#pragma once
#include "algs.cuh"
#include "blake2b_staged.cuh"

namespace snt {

constexpr int LEAF_THREADS = 128;
// Minimum resident CTAs per SM the SHA-256 leaf kernel is compiled for. Occupancy itself does
// not matter (the kernel runs at the same speed with 2 to 8 CTAs per SM); the register cap
// selects among ptxas allocations whose bank-conflict behaviour differs by ~3%
// (profiles/r1_leafbench_occ.jsonl: 71 regs 7.23 ms, 64 regs 7.47 ms, 56 regs 7.27 ms).
#ifndef SNT_LEAF_MINB
#define SNT_LEAF_MINB 1
#endif
constexpr int REDUCE_THREADS = 256;       // default CTA size of the level reducer (see launch_reduce)

// ---- leaf hashing -----------------------------------------------------------

// SHA-256 blocks [b0, b1) of a leaf at a 16-byte aligned address: 4 x LDG.128 per 64-byte block, the next
// block's loads issued before the current block's rounds.
SNT_HD void sha256_blocks_aligned(const uint8_t* __restrict__ p, uint32_t b0, uint32_t b1, uint32_t s[8],
                                  const Sha256::One& one = Sha256::One()) {
    if (b0 >= b1) return;
    const uint8_t* q = p + (static_cast<size_t>(b0) << 6);
    U4 q0 = ld128(q), q1 = ld128(q + 16), q2 = ld128(q + 32), q3 = ld128(q + 48);
#pragma unroll 1
    for (uint32_t b = b0; b < b1; ++b) {
        uint32_t w[16];
        w[0] = bswap32(q0.x);  w[1] = bswap32(q0.y);  w[2] = bswap32(q0.z);  w[3] = bswap32(q0.w);
        w[4] = bswap32(q1.x);  w[5] = bswap32(q1.y);  w[6] = bswap32(q1.z);  w[7] = bswap32(q1.w);
        w[8] = bswap32(q2.x);  w[9] = bswap32(q2.y);  w[10] = bswap32(q2.z); w[11] = bswap32(q2.w);
        w[12] = bswap32(q3.x); w[13] = bswap32(q3.y); w[14] = bswap32(q3.z); w[15] = bswap32(q3.w);
        if (b + 1 < b1) {
            const uint8_t* n = p + (static_cast<size_t>(b + 1) << 6);
            q0 = ld128(n); q1 = ld128(n + 16); q2 = ld128(n + 32); q3 = ld128(n + 48);
        }
        Sha256::compress(s, w, one);
    }
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

// Dynamic shared memory a leaf-hashing CTA needs: BLAKE2b prefetches its message through two
// staging buffers per thread (blake2b_staged.cuh); the other algorithms load straight to registers.
template <int ALG>
constexpr size_t leaf_stage_bytes() {
    return ALG == ALG_BLAKE2B ? 2ull * B2S_SLOTS * LEAF_THREADS * sizeof(uint64_t) : 0;
}

// One leaf / block with the algorithm's preferred formulation.
template <int ALG>
SNT_D void hash_one_leaf(const uint8_t* p, uint64_t len, const MerkleConsts& c, uint32_t* d) {
    using A = AlgTraits<ALG>;
    if (ALG == ALG_BLAKE2B) {
        extern __shared__ __align__(16) uint8_t leaf_smem[];
        uint64_t* stage = reinterpret_cast<uint64_t*>(leaf_smem) + threadIdx.x;
        uint64_t h[8];
        Blake2bStaged<LEAF_THREADS>::template hash_message<0>(stage, 0, 0, p, len, h);
#pragma unroll
        for (int i = 0; i < 8; ++i) { d[2 * i] = static_cast<uint32_t>(h[i]); d[2 * i + 1] = static_cast<uint32_t>(h[i] >> 32); }
    } else {
        A::leaf(p, len, c, d);
    }
}

// The paths that are not the aligned block loop are kept out of line so that they do not take part in
// the register allocation and instruction scheduling of that loop.
//   sha256_leaf_generic  a leaf at an address that is not 16-byte aligned (tensor views at odd offsets)
//   sha256_finish_cold   the closing blocks of an aligned leaf that is shorter than the block size
//                        (the ragged last block of a tensor); a full leaf closes with the constant
//                        padding block instead (Sha256::compress_const)
__device__ __noinline__ void sha256_finish_cold(const uint8_t* t, uint32_t rem, uint64_t len, uint32_t one_u,
                                                uint32_t one_v, uint32_t s[8]) {
    Sha256::finish(t, rem, len, s, Sha256::One(one_u, one_v));
}

__device__ __noinline__ void sha256_leaf_generic(const uint8_t* p, uint64_t len, uint32_t one_u, uint32_t one_v,
                                                 uint32_t d[8]) {
    Sha256::init(d);
    const uint64_t nfull = len >> 6;
    const Sha256::One one(one_u, one_v);
    for (uint64_t b = 0; b < nfull; ++b) {
        uint32_t w[16];
        load_words<16>(p + (b << 6), w);
#pragma unroll
        for (int i = 0; i < 16; ++i) w[i] = bswap32(w[i]);
        Sha256::compress(d, w, one);
    }
    sha256_finish_cold(p + (nfull << 6), static_cast<uint32_t>(len & 63), len, one_u, one_v, d);
}

// Close an aligned SHA-256 leaf after its full 64-byte blocks: the constant padding block when the leaf
// is a whole block, the closing blocks built from its tail bytes otherwise.
SNT_D void sha256_close_leaf(const LeafRef& leaf, uint32_t block_shift, const MerkleConsts& c, const Sha256::One& one,
                             uint32_t s[8]) {
    if (leaf.len == (1ull << block_shift)) {
        Sha256::compress_const(s, c.sha256_pad_leaf, one);
    } else {
        sha256_finish_cold(leaf.ptr + ((leaf.len >> 6) << 6), static_cast<uint32_t>(leaf.len & 63), leaf.len, one.u, one.v, s);
    }
}

// One thread per leaf of [leaf_begin, leaf_end); digest k is written at
// d_leaves + (k - leaf_begin) * DIGEST_BYTES.
//
// SHA-256 splits the leaves in two classes at plan time. "Regular" leaves (16-byte aligned address --
// in practice all of them: allocators align tensors far more strictly) run the aligned block loop in the
// main part of the grid, a ragged last block of a tensor simply with fewer blocks and its own closing
// blocks. Leaves of tensors that sit at odd addresses (views at byte offsets) are listed in `irregular`
// and hashed by the first `irr_ctas` CTAs of the same grid with the generic path, concurrently with the
// rest; a warp's irregular lanes sit the main part out.
template <int ALG>
__global__ void __launch_bounds__(LEAF_THREADS, (ALG == ALG_SHA256) ? SNT_LEAF_MINB : 1)
merkle_leaf_kernel(const TensorTable tab, const __grid_constant__ MerkleConsts c,
                   uint64_t leaf_begin, uint64_t leaf_end, const uint64_t* __restrict__ irregular,
                   uint32_t n_irregular, uint32_t irr_ctas, uint8_t* __restrict__ d_leaves) {
    using A = AlgTraits<ALG>;
    uint32_t d[A::DW];
    if (ALG == ALG_SHA256) {
        const Sha256::One one = sha256_one(c);
        if (blockIdx.x < irr_ctas) {
            const uint32_t j = blockIdx.x * LEAF_THREADS + threadIdx.x;
            if (j >= n_irregular) return;
            const uint64_t k = irregular[j];
            if (k < leaf_begin || k >= leaf_end) return;
            const LeafRef leaf = locate_leaf(tab, k);
            sha256_leaf_generic(leaf.ptr, leaf.len, one.u, one.v, d);
            store_digest<ALG>(d_leaves + (k - leaf_begin) * A::DIGEST_BYTES, d);
            return;
        }
        const uint64_t k = leaf_begin + static_cast<uint64_t>(blockIdx.x - irr_ctas) * LEAF_THREADS + threadIdx.x;
        if (k >= leaf_end) return;
        const LeafRef leaf = locate_leaf(tab, k);
        if (reinterpret_cast<uintptr_t>(leaf.ptr) & 15) return;   // hashed by the irregular CTAs
        Sha256::init(d);
        sha256_blocks_aligned(leaf.ptr, 0, static_cast<uint32_t>(leaf.len >> 6), d, one);
        sha256_close_leaf(leaf, tab.block_shift, c, one, d);
        store_digest<ALG>(d_leaves + (k - leaf_begin) * A::DIGEST_BYTES, d);
    } else {
        const uint64_t k = leaf_begin + static_cast<uint64_t>(blockIdx.x) * LEAF_THREADS + threadIdx.x;
        if (k >= leaf_end) return;
        const LeafRef leaf = locate_leaf(tab, k);
        hash_one_leaf<ALG>(leaf.ptr, leaf.len, c, d);
        store_digest<ALG>(d_leaves + (k - leaf_begin) * A::DIGEST_BYTES, d);
    }
}

// hash_blocks over an explicit (address, length) list: entry i = H(block i)
// (merkle.py:93-114). Blocks may be empty, ragged and unaligned.
template <int ALG>
__global__ void __launch_bounds__(LEAF_THREADS)
hash_blocks_kernel(const uint8_t* __restrict__ base, const uint64_t* __restrict__ off,
                   const uint64_t* __restrict__ len, uint64_t n, const __grid_constant__ MerkleConsts c,
                   uint8_t* __restrict__ out) {
    using A = AlgTraits<ALG>;
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * LEAF_THREADS + threadIdx.x;
    if (i >= n) return;
    uint32_t d[A::DW];
    hash_one_leaf<ALG>(base + off[i], len[i], c, d);
    store_digest<ALG>(out + i * A::DIGEST_BYTES, d);
}

// ---- level reducer ------------------------------------------------------------
//
// Input: nodes of one tree level with global indices [first, first + n_in);
// `level_count` is the number of nodes the whole tree has at that level (a
// node index >= level_count does not exist and pairs as zeros). Each CTA
// applies `levels` (1..reduce_max_levels) levels to its aligned group of
// 2^levels inputs and writes one node. Levels are never skipped: a group that
// is down to one node keeps pairing it with zeros, which is exactly what the
// reference tree does to the last node of every odd level and what makes
// per-shard roots combine into the reference root.
//
// Work layout: level by level through shared memory with the active threads
// compacted -- at every level thread p hashes pair p, so the wide bottom
// levels (where almost all the node hashes are) run with full warps: a
// 1024-node group costs 36 warp-hash-times against the ideal 32, and the
// critical path is one node hash per level. Digests sit in shared memory word
// by word ([word][node]) so that the pair loads are conflict-free 64-bit reads.

template <int ALG>
struct ReduceShape {
    static constexpr int DW = AlgTraits<ALG>::DW;
    static constexpr int CAP = (DW == 8) ? 512 : 256;     // level-1 outputs held per CTA
    static constexpr int MAX_LEVELS = (DW == 8) ? 10 : 9; // 2 * CAP inputs per CTA
};

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

// The reduction of 2^glog adjacent aligned groups of 2^levels inputs each, starting at global node index
// `base` (see above); writes one output node per group to out_digests (nodes that do not exist in the tree
// are skipped). glog = 0 is the narrowing walk down to one node; glog > 0 with few levels is the wide
// first launch of a big tree: every thread stays busy on every level, so the launch is throughput-bound
// instead of ending in the latency-bound narrow levels. Called by every thread of the CTA.
template <int ALG, int THREADS>
SNT_D void reduce_group(const uint8_t* __restrict__ in, uint64_t first, uint64_t n_in, uint64_t base,
                        uint64_t level_count, uint32_t levels, uint32_t glog, const MerkleConsts& c,
                        uint8_t* __restrict__ out_digests, uint32_t* buf_a, uint32_t* buf_b) {
    using A = AlgTraits<ALG>;
    constexpr int DW = A::DW;
    constexpr int CAP = ReduceShape<ALG>::CAP;
    const uint32_t tid = threadIdx.x;
    const uint64_t in_end = first + n_in;
    const uint32_t width = 1u << (levels + glog);

    // level 0 -> 1 straight from global memory: pair p = inputs base + 2p, base + 2p + 1
    for (uint32_t p = tid; p < (width >> 1); p += THREADS) {
        const uint64_t g = base + 2ull * p;
        if (g < in_end) {
            uint32_t l[DW], r[DW];
            load_digest<ALG>(in + (g - first) * A::DIGEST_BYTES, l);
            const bool r_exists = g + 1 < in_end;
            if (r_exists) load_digest<ALG>(in + (g + 1 - first) * A::DIGEST_BYTES, r);
            pair_or_pad<ALG>(l, r, r_exists, c);
#pragma unroll
            for (int i = 0; i < DW; ++i) buf_a[i * CAP + p] = l[i];
        }
    }
    __syncthreads();

    uint32_t* src = buf_a;
    uint32_t* dst = buf_b;
    uint32_t src_stride = CAP, dst_stride = CAP / 2;
    for (uint32_t t = 1; t < levels; ++t) {
        if (glog == 0 && (width >> t) <= 32) {
            // The level fits one warp: warp 0 finishes the walk on its own, children fetched from the neighbouring
            // lanes by shuffles -- no shared-memory round trip and no CTA barrier per level any more (a level
            // costs one node-hash latency, 3.1 us, instead of ~4.3).
            if (tid < 32) {
                uint32_t x[DW];
#pragma unroll
                for (int i = 0; i < DW; ++i) x[i] = tid < (width >> t) ? src[i * src_stride + tid] : 0u;
                for (uint32_t tt = t; tt < levels; ++tt) {
                    const uint64_t cnt = ceil_shift(level_count, tt);
                    const uint64_t g = (base >> tt) + 2ull * tid;
                    uint32_t l[DW], r[DW];
#pragma unroll
                    for (int i = 0; i < DW; ++i) {
                        l[i] = __shfl_sync(0xffffffffu, x[i], (2 * tid) & 31);
                        r[i] = __shfl_sync(0xffffffffu, x[i], (2 * tid + 1) & 31);
                    }
                    pair_or_pad<ALG>(l, r, g + 1 < cnt, c);       // lanes past the level's nodes compute garbage nobody reads
#pragma unroll
                    for (int i = 0; i < DW; ++i) x[i] = l[i];
                }
                if (tid == 0 && (base >> levels) < ceil_shift(level_count, levels)) store_digest<ALG>(out_digests, x);
            }
            return;
        }
        const uint32_t n_out = width >> (t + 1);
        const uint64_t cnt = ceil_shift(level_count, t);          // nodes the tree has at this level
        const uint64_t gbase = base >> t;
        for (uint32_t p = tid; p < n_out; p += THREADS) {
            const uint64_t g = gbase + 2ull * p;
            if (g < cnt) {
                uint32_t l[DW], r[DW];
#pragma unroll
                for (int i = 0; i < DW; ++i) {
                    const uint2 v = *reinterpret_cast<const uint2*>(src + i * src_stride + 2 * p);
                    l[i] = v.x;
                    r[i] = v.y;
                }
                pair_or_pad<ALG>(l, r, g + 1 < cnt, c);
#pragma unroll
                for (int i = 0; i < DW; ++i) dst[i * dst_stride + p] = l[i];
            }
        }
        __syncthreads();
        uint32_t* tp = src; src = dst; dst = tp;
        const uint32_t ts = src_stride; src_stride = dst_stride; dst_stride = ts;
    }
    const uint64_t out_cnt = ceil_shift(level_count, levels);     // nodes the tree has at the output level
    const uint64_t obase = base >> levels;
    for (uint32_t p = tid; p < (1u << glog); p += THREADS) {
        if (obase + p < out_cnt) {
            uint32_t d[DW];
#pragma unroll
            for (int i = 0; i < DW; ++i) d[i] = src[i * src_stride + p];
            store_digest<ALG>(out_digests + static_cast<uint64_t>(p) * A::DIGEST_BYTES, d);
        }
    }
}

template <int ALG, int THREADS>
__global__ void __launch_bounds__(THREADS)
merkle_reduce_kernel(const uint8_t* __restrict__ in, uint64_t first, uint64_t n_in,
                     uint64_t level_count, uint32_t levels, uint32_t glog, const __grid_constant__ MerkleConsts c,
                     uint8_t* __restrict__ out) {
    using A = AlgTraits<ALG>;
    constexpr int CAP = ReduceShape<ALG>::CAP;
    __shared__ uint32_t buf_a[A::DW * CAP];
    __shared__ uint32_t buf_b[A::DW * CAP / 2];
    const uint64_t base = first + (static_cast<uint64_t>(blockIdx.x) << (levels + glog));   // first input of this CTA
    reduce_group<ALG, THREADS>(in, first, n_in, base, level_count, levels, glog, c,
                               out + (static_cast<uint64_t>(blockIdx.x) << glog) * A::DIGEST_BYTES, buf_a, buf_b);
}

// One tree per segment (per_layer_hash, model.py:245-253), one CTA per segment, one launch for all
// segments of at most 2^MAX_LEVELS nodes: segment j covers the seg[2j+1] digests at ADDRESS seg[2j] (the leaf
// digests of a small tensor, or the level-MAX_LEVELS nodes merkle_reduce_groups_kernel left in the workspace for a
// large one) and its root goes to out + seg_out[j] * DIGEST_BYTES. The root of a tree of `count` nodes under
// the reference rule (merkle.py:152-165) is the result of exactly ceil(log2(count)) levels; a single
// digest is its own root and an empty segment takes the digest of the empty message.
template <int ALG, int THREADS>
__global__ void __launch_bounds__(THREADS)
merkle_reduce_segments_kernel(const uint64_t* __restrict__ seg, const uint32_t* __restrict__ seg_out,
                              const uint8_t* __restrict__ empty_digest, const __grid_constant__ MerkleConsts c,
                              uint8_t* __restrict__ out) {
    using A = AlgTraits<ALG>;
    constexpr int CAP = ReduceShape<ALG>::CAP;
    __shared__ uint32_t buf_a[A::DW * CAP];
    __shared__ uint32_t buf_b[A::DW * CAP / 2];
    const uint8_t* in = reinterpret_cast<const uint8_t*>(seg[2ull * blockIdx.x]);
    const uint64_t count = seg[2ull * blockIdx.x + 1];
    uint8_t* dst = out + static_cast<uint64_t>(seg_out[blockIdx.x]) * A::DIGEST_BYTES;
    if (count <= 1) {
        const uint8_t* src = count ? in : empty_digest;
        for (uint32_t i = threadIdx.x; i < A::DIGEST_BYTES; i += THREADS) dst[i] = src[i];
        return;
    }
    uint32_t levels = 0;
    while ((1ull << levels) < count) ++levels;
    reduce_group<ALG, THREADS>(in, 0, count, 0, count, levels, 0, c, dst, buf_a, buf_b);
}

// The bottom MAX_LEVELS levels of MANY large trees in one launch: CTA r reduces group grp[3r+2] (2^MAX_LEVELS
// aligned leaf digests) of the tree whose grp[3r+1] leaf digests start at ADDRESS grp[3r], and writes the
// level-MAX_LEVELS node to out + grp_out[r] * DIGEST_BYTES. Same existence / zero-padding rule as everywhere
// (reduce_group with the tree's own leaf count), so merkle_reduce_segments_kernel can finish every tree from
// these nodes. Before: one chain of launches per large tensor, one after the other (GPT-2 small per-layer:
// 26 tensors above 1,024 blocks, ~52 latency-bound launches, 2.4 ms for a 0.76 ms hash).
template <int ALG, int THREADS>
__global__ void __launch_bounds__(THREADS)
merkle_reduce_groups_kernel(const uint64_t* __restrict__ grp, const uint32_t* __restrict__ grp_out,
                            const __grid_constant__ MerkleConsts c, uint8_t* __restrict__ out) {
    using A = AlgTraits<ALG>;
    constexpr int CAP = ReduceShape<ALG>::CAP;
    constexpr uint32_t LEVELS = ReduceShape<ALG>::MAX_LEVELS;
    __shared__ uint32_t buf_a[A::DW * CAP];
    __shared__ uint32_t buf_b[A::DW * CAP / 2];
    const uint8_t* in = reinterpret_cast<const uint8_t*>(grp[3ull * blockIdx.x]);
    const uint64_t count = grp[3ull * blockIdx.x + 1], group = grp[3ull * blockIdx.x + 2];
    reduce_group<ALG, THREADS>(in, 0, count, group << LEVELS, count, LEVELS, 0, c,
                               out + static_cast<uint64_t>(grp_out[blockIdx.x]) * A::DIGEST_BYTES, buf_a, buf_b);
}

}  // namespace snt
