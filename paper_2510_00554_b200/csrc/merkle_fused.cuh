// The whole in-place Merkle hash in ONE launch: persistent leaf hashing with software time
// slicing, and the tree folded in behind it through completion counters.
//
// Reference behaviour reproduced (same as merkle_kernels.cuh):
//   leaf stage   merkle.py:93-114 (hash_blocks) over model.py:137-146 (BlockTable)
//   level rule   merkle.py:117-149 (reduce_level), root merkle.py:152-165
//
// Leaf stage. A leaf is a serial chain of compressions, so the schedulable unit is a CHAIN: one
// warp x 32 consecutive leaves. A plain grid gives every SM sub-partition an integer number of
// warps -- GPT-2 small: 2,490 warps on 592 schedulers = 4.2 each, so the launch takes 5 warp-times.
// Here one persistent CTA per SM owns a contiguous run of chains (balanced to +-1 across SMs) and
// W worker warps (W/4 per scheduler) share them. Chains are run to completion one after the other,
// except the last W + (count mod W) chains of the SM: those are executed in slices of 1/W of a
// leaf and handed from warp to warp through a FIFO in shared memory, the hash state (8 to 50 words
// per lane) parked in shared memory in between. Until the very end every scheduler therefore has
// W/4 runnable warps, and the SM finishes after count/4 warp-times instead of ceil(count/4)
// (tools/persist_bench.cu: GPT-2 small 0.777 -> 0.649 ms, GPT2-XL 6.25 -> 6.12 ms).
//
// Tree. When a chain is done its warp stores the 32 leaf digests, fences, and adds its leaf count
// to the counter of the 2^m0-leaf group the chain belongs to (m0 = 8 when the tree is that deep).
// The warp that brings a counter to the group's size reduces the group on its own: the wide levels
// 32 pair hashes at a time with the children redistributed by warp shuffles (fold_sets), the last
// five levels inside the warp, all in registers. It stores the node, bumps the counter of the
// next stage's group (2^6 nodes) and, if that completes, carries on upwards; the warp that
// completes the last group writes the root. Levels are never skipped and a missing right child is
// zeros, decided from range-relative node counts exactly like reduce_group, so shard roots
// (levels = k) recombine into the reference root. Counters are returned to zero by the warp that
// consumes them: the workspace is zeroed once (snt_merkle_work_init), never between launches.
//
// SHA-256 keeps its two leaf classes: leaves at 16-byte aligned addresses (in practice all of them)
// run in the chains above with the aligned loader, a tensor's ragged last block simply with fewer
// blocks and its own closing blocks; leaves of tensors at odd addresses (views at byte offsets) are
// packed 32 to a chain of their own, hashed through the out-of-line generic path at the front of an
// SM's queue, and signal their groups leaf by leaf.
#pragma once
#ifndef SNT_MERKLE_B2B_ROLLED
#define SNT_MERKLE_B2B_ROLLED 0      // BLAKE2b leaf loop: unrolled rounds from registers (1) = rolled rounds from the staging buffer
#endif
#include "chain_sched.cuh"
#include "merkle_kernels.cuh"

namespace snt {

constexpr int FUSED_MAX_STAGES = 8;
constexpr uint32_t FUSED_MIN_LEVELS = 5;   // a chain (32 leaves) must lie inside one first-stage group
constexpr uint32_t FUSED_FIRST_STAGE_LEVELS = 8;
constexpr uint32_t FUSED_NEXT_STAGE_LEVELS = 6;

struct FusedTree {
    uint32_t n_stages;                       // 0: leaf digests only
    uint32_t m[FUSED_MAX_STAGES];            // levels folded by stage s
    uint64_t n_in[FUSED_MAX_STAGES];         // nodes entering stage s (stage 0: leaves of the range)
    uint32_t* cnt[FUSED_MAX_STAGES];         // one completion counter per group of stage s
    uint8_t* nodes[FUSED_MAX_STAGES];        // output nodes of stage s; the last stage writes d_out
};

struct FusedArgs {
    TensorTable tab;
    uint64_t leaf_begin;                     // first leaf of the range (global index)
    uint64_t n;                              // leaves in the range
    const uint64_t* irregular;               // SHA-256: global indices of the range's irregular leaves
    uint32_t n_irregular;
    uint8_t* d_leaves;                       // digest of leaf k at (k - leaf_begin) * DIGEST_BYTES
    uint32_t flip;                           // diagnostics: CTA b takes the share of CTA grid - 1 - b
    unsigned long long* trace;               // diagnostics (may be null): per CTA {start ns, last worker exit ns,
                                             // group reductions done here, chain slices run here,
                                             // last chain finished ns, SM id}
    FusedTree tree;
};

SNT_D unsigned long long fused_now_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// A parked chain keeps, per lane, the hash state and where its leaf is (address, length, whether the lane
// takes part), so that the warp that resumes it does not search the tensor table again.
constexpr int FUSED_PARK_EXTRA = 4;

template <int ALG> struct FusedLeaf;
template <> struct FusedLeaf<ALG_SHA256> { static constexpr int STATE_WORDS = 8; };
template <> struct FusedLeaf<ALG_BLAKE2B> { static constexpr int STATE_WORDS = 16; };
template <> struct FusedLeaf<ALG_SHA3_256> { static constexpr int STATE_WORDS = 50; };

// Schedulable units (compressions / permutations of message data) of a full block.
template <int ALG>
SNT_HD uint32_t fused_units(uint32_t block_shift) {
    const uint64_t bs = 1ull << block_shift;
    if (ALG == ALG_SHA256) return static_cast<uint32_t>(bs >> 6);          // + the constant padding block
    if (ALG == ALG_BLAKE2B) return static_cast<uint32_t>((bs + 127) >> 7);
    return static_cast<uint32_t>(bs / Sha3_256::RATE_BYTES + 1);
}

// Dynamic shared memory of the kernel: message staging (BLAKE2b only) and 2 * MAXW - 1 parked states.
template <int ALG, int MAXW>
SNT_HD constexpr size_t fused_stage_bytes() {
    return ALG == ALG_BLAKE2B ? 2ull * B2S_SLOTS * MAXW * 32 * sizeof(uint64_t) : 0;
}
template <int ALG, int MAXW>
SNT_HD constexpr size_t fused_smem_bytes() {
    return fused_stage_bytes<ALG, MAXW>() + (2ull * MAXW - 1) * (FusedLeaf<ALG>::STATE_WORDS + FUSED_PARK_EXTRA) * 32 * sizeof(uint32_t);
}

// ---- tree: one warp reduces one group ---------------------------------------------------------

// A digest another SM may have written a moment ago: read it from L2.
template <int ALG>
SNT_D void load_digest_cg(const uint8_t* in, uint32_t* d) {
    using A = AlgTraits<ALG>;
    const uint4* q = reinterpret_cast<const uint4*>(in);
#pragma unroll
    for (int i = 0; i < A::DW / 4; ++i) {
        const uint4 v = __ldcg(q + i);
        d[4 * i] = A::from_mem(v.x); d[4 * i + 1] = A::from_mem(v.y);
        d[4 * i + 2] = A::from_mem(v.z); d[4 * i + 3] = A::from_mem(v.w);
    }
}

// The node hash, out of line, in two formulations. While leaf chains are running on this SM the tree uses
// the SMALL one (rolled rounds, a few KB): the unrolled node hash is 40 KB of straight-line code, and a warp
// streaming through it evicts the 26 KB leaf loop the other warps are in from the instruction cache --
// measured on GPT2-XL, interleaving the tree that way cost 7 % of the launch for 3 % of its instructions.
// Once the SM has no leaf work left (the tail of the launch, where only the latency of the remaining
// levels counts) the unrolled one runs: 3.7 us per node instead of 4.8 (tools/nodehash_bench.cu).
template <int ALG, bool SMALL>
__device__ __noinline__ void pair_cold(uint32_t* l, const uint32_t* r, uint32_t right_exists, const MerkleConsts* c) {
    using A = AlgTraits<ALG>;
    uint32_t rr[A::DW], out[A::DW];
#pragma unroll
    for (int i = 0; i < A::DW; ++i) rr[i] = right_exists ? r[i] : 0u;
    if (SMALL) A::pair_small(l, rr, *c, out); else A::pair(l, rr, *c, out);
#pragma unroll
    for (int i = 0; i < A::DW; ++i) l[i] = out[i];
}
template <int ALG>
SNT_D void pair_either(uint32_t* l, const uint32_t* r, uint32_t right_exists, const MerkleConsts* c, bool small) {
    if (small) pair_cold<ALG, true>(l, r, right_exists, c); else pair_cold<ALG, false>(l, r, right_exists, c);
}

// a, b: two sets of 32 adjacent nodes of one level, one node per lane (a before b); n_exist of the
// 64 positions hold nodes of the tree. On return a = their 32 parents (lanes 0..15 from a, 16..31
// from b); parent i exists iff child 2i does. Lanes whose node does not exist hold garbage.
template <int ALG>
SNT_D void fold_sets(uint32_t* a, const uint32_t* b, uint32_t n_exist, const MerkleConsts* c, bool small, int lane) {
    constexpr int DW = AlgTraits<ALG>::DW;
    const int src = 2 * (lane & 15);
    uint32_t l[DW], r[DW];
#pragma unroll
    for (int i = 0; i < DW; ++i) {
        const uint32_t la = __shfl_sync(0xffffffffu, a[i], src), lb = __shfl_sync(0xffffffffu, b[i], src);
        const uint32_t ra = __shfl_sync(0xffffffffu, a[i], src + 1), rb = __shfl_sync(0xffffffffu, b[i], src + 1);
        l[i] = lane < 16 ? la : lb;
        r[i] = lane < 16 ? ra : rb;
    }
    pair_either<ALG>(l, r, static_cast<uint32_t>(2 * lane + 1) < n_exist, c, small);
#pragma unroll
    for (int i = 0; i < DW; ++i) a[i] = l[i];
}

// x: up to 32 adjacent nodes in lanes 0..; on return lanes 0..15 hold their parents.
template <int ALG>
SNT_D void narrow_set(uint32_t* x, uint32_t n_exist, const MerkleConsts* c, bool small, int lane) {
    constexpr int DW = AlgTraits<ALG>::DW;
    uint32_t l[DW], r[DW];
#pragma unroll
    for (int i = 0; i < DW; ++i) {
        l[i] = __shfl_sync(0xffffffffu, x[i], (2 * lane) & 31);
        r[i] = __shfl_sync(0xffffffffu, x[i], (2 * lane + 1) & 31);
    }
    pair_either<ALG>(l, r, static_cast<uint32_t>(2 * lane + 1) < n_exist, c, small);
#pragma unroll
    for (int i = 0; i < DW; ++i) x[i] = l[i];
}

template <int ALG>
SNT_D void load_set(const uint8_t* children, uint32_t first, uint32_t n_children, uint32_t* x, int lane) {
    using A = AlgTraits<ALG>;
    const uint32_t i = first + lane;
    if (i < n_children) {
        load_digest_cg<ALG>(children + static_cast<size_t>(i) * A::DIGEST_BYTES, x);
    } else {
#pragma unroll
        for (int w = 0; w < A::DW; ++w) x[w] = 0;
    }
}

// Apply m (1..8) levels to the n_children (>= 1) adjacent nodes at `children`, which are the first
// nodes of an aligned group of 2^m positions; the result ends up in lane 0's `out`. Called by a
// whole warp. m = 8 costs 4 + 2 + 1 full-width pair hashes and 5 narrowing ones.
template <int ALG>
SNT_D void warp_reduce_group(const uint8_t* children, uint32_t n_children, uint32_t m, const MerkleConsts* c,
                             bool small, uint32_t* out, int lane) {
    constexpr int DW = AlgTraits<ALG>::DW;
    uint32_t x[DW];
    uint32_t cnt = n_children;                   // nodes of the tree at the current level
    uint32_t narrow = m;
    if (m > 5) {
        // sets of 32 nodes merged like a binary counter: stack[t] = a finished set of level t + 1 waiting
        // for its right neighbour (dynamically indexed, so it lives in local memory: the per-warp scratch)
        uint32_t stack[FUSED_FIRST_STAGE_LEVELS - 5][DW];
        const uint32_t n_pairs = 1u << (m - 6);
        for (uint32_t i = 0; i < n_pairs; ++i) {
            uint32_t b[DW];
            load_set<ALG>(children, 64 * i, n_children, x, lane);
            load_set<ALG>(children, 64 * i + 32, n_children, b, lane);
            fold_sets<ALG>(x, b, n_children > 64 * i ? n_children - 64 * i : 0, c, small, lane);
            uint32_t t = 0, idx = i;
            while (idx & 1) {
                // x = right set of level t + 1, stack[t] = left set; positions 64 * (idx >> 1) .. of that level
                const uint32_t level_cnt = (n_children + (1u << (t + 1)) - 1) >> (t + 1);
                const uint32_t base = 64 * (idx >> 1);
#pragma unroll
                for (int w = 0; w < DW; ++w) { b[w] = x[w]; x[w] = stack[t][w]; }
                fold_sets<ALG>(x, b, level_cnt > base ? level_cnt - base : 0, c, small, lane);
                ++t;
                idx >>= 1;
            }
#pragma unroll
            for (int w = 0; w < DW; ++w) stack[t][w] = x[w];
        }
        cnt = (n_children + (1u << (m - 5)) - 1) >> (m - 5);
        narrow = 5;
    } else {
        load_set<ALG>(children, 0, n_children, x, lane);
    }
    for (uint32_t t = 0; t < narrow; ++t) {
        narrow_set<ALG>(x, cnt, c, small, lane);
        cnt = (cnt + 1) >> 1;
    }
#pragma unroll
    for (int w = 0; w < DW; ++w) out[w] = x[w];
}

SNT_D uint32_t fused_group_size(const FusedTree& tr, uint32_t stage, uint64_t g) {
    const uint32_t m = tr.m[stage];
    const uint64_t left = tr.n_in[stage] - (g << m);
    return left < (1ull << m) ? static_cast<uint32_t>(left) : (1u << m);
}

// Group g of `stage` is complete (all its children are stored and visible): reduce it, hand the node
// to the next stage, and keep climbing for as long as this warp is the one that completes a group.
template <int ALG>
SNT_D void fused_climb(const FusedArgs& a, const MerkleConsts* c, const FusedSched* sc, int count, uint32_t stage,
                       uint64_t g, int lane) {
    using A = AlgTraits<ALG>;
    for (;;) {
        __threadfence();
        // leaf chains still queued on this SM? then tread lightly on the instruction cache
        const bool small = sched_waiting(sc, count, lane);
        if (a.trace && lane == 0) atomicAdd(a.trace + 6ull * blockIdx.x + 2, 1ull);
        const uint8_t* children = (stage == 0 ? a.d_leaves : a.tree.nodes[stage - 1]) +
                                  ((g << a.tree.m[stage]) * A::DIGEST_BYTES);
        uint32_t node[A::DW];
        warp_reduce_group<ALG>(children, fused_group_size(a.tree, stage, g), a.tree.m[stage], c, small, node, lane);
        int more = 0;
        uint64_t g_next = 0;
        if (lane == 0) {
            store_digest<ALG>(a.tree.nodes[stage] + g * A::DIGEST_BYTES, node);
            if (stage + 1 < a.tree.n_stages) {
                __threadfence();
                g_next = g >> a.tree.m[stage + 1];
                uint32_t* counter = a.tree.cnt[stage + 1] + g_next;
                if (atomicAdd(counter, 1u) + 1u == fused_group_size(a.tree, stage + 1, g_next)) {
                    *counter = 0;                      // back to zero for the next launch
                    more = 1;
                }
            }
        }
        more = __shfl_sync(0xffffffffu, more, 0);
        if (!more) return;
        g = __shfl_sync(0xffffffffu, g_next, 0);
        ++stage;
    }
}

// `n_done` leaves of first-stage group g have just been stored by this warp (lane 0 speaks for a
// regular chain). Returns true in lane 0 when that completed the group.
SNT_D bool fused_leaves_done(const FusedArgs& a, uint64_t g, uint32_t n_done) {
    uint32_t* counter = a.tree.cnt[0] + g;
    if (atomicAdd(counter, n_done) + n_done == fused_group_size(a.tree, 0, g)) {
        *counter = 0;
        return true;
    }
    return false;
}

// ---- the kernel -------------------------------------------------------------------------------

template <int ALG, int MAXW>
__global__ void __launch_bounds__(MAXW * 32, 1)
merkle_fused_kernel(const __grid_constant__ FusedArgs a, const __grid_constant__ MerkleConsts c) {
    using A = AlgTraits<ALG>;
    constexpr int SW = FusedLeaf<ALG>::STATE_WORDS;
    // dynamic shared memory: [BLAKE2b: per-thread message staging][parked chain states: slot, word, lane]
    extern __shared__ __align__(16) uint8_t fused_smem[];
    __shared__ FusedSched sc;
    const int lane = threadIdx.x & 31;
    const int W = blockDim.x >> 5;

    // this CTA's chains: its share of the irregular chains first, then a contiguous run of regular ones
    const uint32_t bid = a.flip ? gridDim.x - 1 - blockIdx.x : blockIdx.x;
    const uint64_t R = (a.n + 31) >> 5;
    const uint64_t q = R / gridDim.x, rem = R % gridDim.x;
    const uint64_t reg_first = bid * q + (bid < rem ? bid : rem);
    const int n_reg = static_cast<int>(q + (bid < rem ? 1 : 0));
    // irregular chain j goes to the j-th of the CTAs that got the smaller share of regular chains
    const uint32_t n_irr_chains = (a.n_irregular + 31) >> 5;
    const uint32_t light_first = rem ? static_cast<uint32_t>(rem) : 0u, n_light = gridDim.x - light_first;
    int n_irr = 0;
    if (bid >= light_first && bid - light_first < n_irr_chains)
        n_irr = static_cast<int>((n_irr_chains - (bid - light_first) + n_light - 1) / n_light);
    const int count = n_irr + n_reg;
    const int first_sliced = sched_first_sliced(count, W);
    const uint32_t units = fused_units<ALG>(a.tab.block_shift);
    const uint32_t slice = (units + W - 1) / W;

    if (threadIdx.x == 0 && a.trace) {
        uint32_t smid;
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
        a.trace[6ull * blockIdx.x] = fused_now_ns();
        a.trace[6ull * blockIdx.x + 5] = smid;
    }
    sched_init(&sc);
    uint32_t* const my_park = reinterpret_cast<uint32_t*>(fused_smem + fused_stage_bytes<ALG, MAXW>());
    const uint32_t m0 = a.tree.n_stages ? a.tree.m[0] : 0;

    for (;;) {
        const int ch = sched_pop(&sc, count, lane);
        if (ch < 0) break;
        if (a.trace && lane == 0) atomicAdd(a.trace + 6ull * blockIdx.x + 3, 1ull);

        if constexpr (ALG == ALG_SHA256) if (ch < n_irr) {
            // ---- a chain of irregular leaves: generic path, never parked
            const uint32_t j = ((bid - light_first) + static_cast<uint32_t>(ch) * n_light) * 32 + lane;
            bool complete = false;
            uint64_t g = 0;
            if (j < a.n_irregular) {
                const uint64_t k = a.irregular[j];
                const LeafRef leaf = locate_leaf(a.tab, k);
                const Sha256::One one = sha256_one(c);
                uint32_t d[A::DW];
                sha256_leaf_generic(leaf.ptr, leaf.len, one.u, one.v, d);
                store_digest<ALG>(a.d_leaves + (k - a.leaf_begin) * A::DIGEST_BYTES, d);
                if (a.tree.n_stages) {
                    __threadfence();
                    g = (k - a.leaf_begin) >> m0;
                    complete = fused_leaves_done(a, g, 1);
                }
            }
            uint32_t todo = __ballot_sync(0xffffffffu, complete);
            while (todo) {
                const int src = __ffs(todo) - 1;
                todo &= todo - 1;
                fused_climb<ALG>(a, &c, &sc, count, 0, __shfl_sync(0xffffffffu, g, src), lane);
            }
            continue;
        }

        // ---- a regular chain: leaves rel .. rel + 31 of the range, one per lane
        const uint64_t rel = ((reg_first + static_cast<uint64_t>(ch - n_irr)) << 5) + lane;
        const bool sliced = ch >= first_sliced;
        const int slot = sliced ? ch - first_sliced : 0;
        uint32_t u0 = sliced ? static_cast<uint32_t>(*reinterpret_cast<volatile int*>(&sc.prog[slot])) : 0u;
        uint32_t* const st = my_park + static_cast<size_t>(slot) * (SW + FUSED_PARK_EXTRA) * 32 + lane;

        bool valid;
        LeafRef leaf;
        leaf.tensor = 0; leaf.block = 0;
        uint32_t s[SW];                              // the hash state as 32-bit words
        if (u0 == 0) {
            valid = rel < a.n;
            leaf.ptr = nullptr; leaf.len = 0;
            if (valid) {
                leaf = locate_leaf(a.tab, a.leaf_begin + rel);
                if constexpr (ALG == ALG_SHA256)      // leaves at odd addresses are hashed by the irregular chains
                    valid = (reinterpret_cast<uintptr_t>(leaf.ptr) & 15) == 0;
            }
            if constexpr (ALG == ALG_SHA256) {
                Sha256::init(s);
            } else if constexpr (ALG == ALG_BLAKE2B) {
                uint64_t h[8];
                Blake2b::init(h);
#pragma unroll
                for (int i = 0; i < 8; ++i) { s[2 * i] = static_cast<uint32_t>(h[i]); s[2 * i + 1] = static_cast<uint32_t>(h[i] >> 32); }
            } else {
#pragma unroll
                for (int i = 0; i < SW; ++i) s[i] = 0;
            }
        } else {
#pragma unroll
            for (int i = 0; i < SW; ++i) s[i] = st[i * 32];
            leaf.ptr = reinterpret_cast<const uint8_t*>((static_cast<uint64_t>(st[(SW + 1) * 32]) << 32) | st[SW * 32]);
            leaf.len = st[(SW + 2) * 32];
            valid = st[(SW + 3) * 32] != 0;
        }

        bool parked = false;
        for (;;) {
            const uint32_t u1 = sliced ? (u0 + slice < units ? u0 + slice : units) : units;
            if (valid) {
                if constexpr (ALG == ALG_SHA256) {
                    const uint32_t mine = static_cast<uint32_t>(leaf.len >> 6);      // a ragged last block has fewer
                    sha256_blocks_aligned(leaf.ptr, u0, u1 < mine ? u1 : mine, s, sha256_one(c));
                } else if constexpr (ALG == ALG_BLAKE2B) {
                    uint64_t h[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) h[i] = (static_cast<uint64_t>(s[2 * i + 1]) << 32) | s[2 * i];
                    uint64_t* stage = reinterpret_cast<uint64_t*>(fused_smem) + threadIdx.x;
                    Blake2bStaged<MAXW * 32>::template hash_blocks<0, SNT_MERKLE_B2B_ROLLED != 0>(stage, 0, 0, leaf.ptr, leaf.len, u0, u1, h);
#pragma unroll
                    for (int i = 0; i < 8; ++i) { s[2 * i] = static_cast<uint32_t>(h[i]); s[2 * i + 1] = static_cast<uint32_t>(h[i] >> 32); }
                } else {
                    uint64_t st64[25];
#pragma unroll
                    for (int i = 0; i < 25; ++i) st64[i] = (static_cast<uint64_t>(s[2 * i + 1]) << 32) | s[2 * i];
                    Sha3_256::absorb_blocks(st64, leaf.ptr, leaf.len, u0, u1);
#pragma unroll
                    for (int i = 0; i < 25; ++i) { s[2 * i] = static_cast<uint32_t>(st64[i]); s[2 * i + 1] = static_cast<uint32_t>(st64[i] >> 32); }
                }
            }
            __syncwarp();
            if (u1 == units) break;
            u0 = u1;
            if (!sched_waiting(&sc, count, lane)) continue;      // nobody is waiting for a warp: keep this chain
#pragma unroll
            for (int i = 0; i < SW; ++i) st[i * 32] = s[i];
            st[SW * 32] = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(leaf.ptr));
            st[(SW + 1) * 32] = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(leaf.ptr) >> 32);
            st[(SW + 2) * 32] = static_cast<uint32_t>(leaf.len);          // a leaf is at most one block (< 2^32 bytes)
            st[(SW + 3) * 32] = valid ? 1u : 0u;
            sched_park(&sc, ch, slot, u0, lane);
            parked = true;
            break;
        }
        if (parked) continue;

        // ---- chain done: digests out, then the tree
        if (a.trace && lane == 0) atomicMax(a.trace + 6ull * blockIdx.x + 4, fused_now_ns());
        if (valid) {
            if constexpr (ALG == ALG_SHA256) sha256_close_leaf(leaf, a.tab.block_shift, c, sha256_one(c), s);
            store_digest<ALG>(a.d_leaves + rel * A::DIGEST_BYTES, s);     // the first DW state words are the digest
        }
        if (a.tree.n_stages) {
            __threadfence();
            const uint32_t n_done = __popc(__ballot_sync(0xffffffffu, valid));
            const uint64_t g = (rel - lane) >> m0;
            int complete = 0;
            if (lane == 0 && n_done) complete = fused_leaves_done(a, g, n_done);
            if (__shfl_sync(0xffffffffu, complete, 0)) fused_climb<ALG>(a, &c, &sc, count, 0, g, lane);
        }
    }
    if (a.trace && lane == 0) atomicMax(a.trace + 6ull * blockIdx.x + 1, fused_now_ns());
}

}  // namespace snt
