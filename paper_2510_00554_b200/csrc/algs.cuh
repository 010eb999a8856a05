// Uniform per-algorithm traits used by the Merkle kernels.
//
// A digest travels through the kernels as DW 32-bit "carrier" words. For
// BLAKE2b and SHA3-256 the carrier is simply the digest bytes read as
// little-endian words; for SHA-256 it is the hash state (the digest bytes read
// big-endian), which saves the byte swaps between a child digest and the
// parent's message schedule.
#pragma once
#include "blake2b.cuh"
#include "keccak.cuh"
#include "sha256.cuh"

namespace snt {

// Per-launch constants (kernel parameter space -> constant bank operands).
struct MerkleConsts {
    uint32_t sha256_pad_leaf[64];   // K+W of the padding block after a full leaf
    uint32_t sha256_pad_node[64];   // K+W of the padding block after a 64-byte node message
    uint32_t one;                   // 1, opaque to the compiler (Sha256::add_fma)
};

// A per-thread register holding 1 that ptxas cannot fold (loaded through a lane-indexed constant
// read), for the IMAD form that carries a round constant in its immediate slot (Sha256::addk_fma).
#ifdef __CUDACC__
__constant__ uint32_t k_lane_ones[32] = {1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1,
                                         1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1};
#endif
SNT_HD Sha256::One sha256_one(const MerkleConsts& c) {
#ifdef __CUDA_ARCH__
    return Sha256::One(c.one, k_lane_ones[threadIdx.x & 31]);
#else
    (void)c;
    return Sha256::One();
#endif
}

template <int ALG> struct AlgTraits;

template <> struct AlgTraits<ALG_SHA256> {
    static constexpr int DIGEST_BYTES = 32;
    static constexpr int DW = 8;
    // carrier words -> little-endian memory words and back
    SNT_HD static uint32_t to_mem(uint32_t w) { return bswap32(w); }
    SNT_HD static uint32_t from_mem(uint32_t w) { return bswap32(w); }
    SNT_HD static void leaf(const uint8_t* p, uint64_t len, const MerkleConsts& c, uint32_t d[DW]) {
        Sha256::hash_message(p, len, d, sha256_one(c));
    }
    SNT_HD static void pair(const uint32_t* l, const uint32_t* r, const MerkleConsts& c, uint32_t* out) {
        // Compile-time ones: the additions fold back to 3-input IADD3. The level reducer is bound by the
        // latency of one node hash per level, and the IMAD formulation has the longer dependency chain
        // (tree of 799,954 digests: 200.8 us vs 206.0 us; 79,672: 68.6 vs 76.8; tools/tree_probe.py).
        Sha256::hash_pair(l, r, c.sha256_pad_node, out);
    }
    // the same node hash in a quarter of the code (rolled rounds): see Sha256::compress_rolled
    // (additions as IMAD were tried here and lost: GPT2-XL 6.53 -> 6.61 ms)
    SNT_HD static void pair_small(const uint32_t* l, const uint32_t* r, const MerkleConsts&, uint32_t* out) {
        Sha256::hash_pair_rolled(l, r, out);
    }
};

template <> struct AlgTraits<ALG_BLAKE2B> {
    static constexpr int DIGEST_BYTES = 64;
    static constexpr int DW = 16;
    SNT_HD static uint32_t to_mem(uint32_t w) { return w; }
    SNT_HD static uint32_t from_mem(uint32_t w) { return w; }
    SNT_HD static void leaf(const uint8_t* p, uint64_t len, const MerkleConsts&, uint32_t d[DW]) {
        uint64_t h[8];
        Blake2b::hash_message<0>(0, 0, p, len, h);
#pragma unroll
        for (int i = 0; i < 8; ++i) { d[2 * i] = static_cast<uint32_t>(h[i]); d[2 * i + 1] = static_cast<uint32_t>(h[i] >> 32); }
    }
    SNT_HD static void pair(const uint32_t* l, const uint32_t* r, const MerkleConsts&, uint32_t* out) {
        uint64_t a[8], b[8], h[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            a[i] = (static_cast<uint64_t>(l[2 * i + 1]) << 32) | l[2 * i];
            b[i] = (static_cast<uint64_t>(r[2 * i + 1]) << 32) | r[2 * i];
        }
        Blake2b::hash_pair(a, b, h);
#pragma unroll
        for (int i = 0; i < 8; ++i) { out[2 * i] = static_cast<uint32_t>(h[i]); out[2 * i + 1] = static_cast<uint32_t>(h[i] >> 32); }
    }
    SNT_HD static void pair_small(const uint32_t* l, const uint32_t* r, const MerkleConsts&, uint32_t* out) {
        uint64_t a[8], b[8], h[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            a[i] = (static_cast<uint64_t>(l[2 * i + 1]) << 32) | l[2 * i];
            b[i] = (static_cast<uint64_t>(r[2 * i + 1]) << 32) | r[2 * i];
        }
        Blake2b::hash_pair_rolled(a, b, h);
#pragma unroll
        for (int i = 0; i < 8; ++i) { out[2 * i] = static_cast<uint32_t>(h[i]); out[2 * i + 1] = static_cast<uint32_t>(h[i] >> 32); }
    }
};

template <> struct AlgTraits<ALG_SHA3_256> {
    static constexpr int DIGEST_BYTES = 32;
    static constexpr int DW = 8;
    SNT_HD static uint32_t to_mem(uint32_t w) { return w; }
    SNT_HD static uint32_t from_mem(uint32_t w) { return w; }
    SNT_HD static void leaf(const uint8_t* p, uint64_t len, const MerkleConsts&, uint32_t d[DW]) {
        uint64_t h[4];
        Sha3_256::hash_message(p, len, h);
#pragma unroll
        for (int i = 0; i < 4; ++i) { d[2 * i] = static_cast<uint32_t>(h[i]); d[2 * i + 1] = static_cast<uint32_t>(h[i] >> 32); }
    }
    SNT_HD static void pair(const uint32_t* l, const uint32_t* r, const MerkleConsts&, uint32_t* out) {
        uint64_t a[4], b[4], h[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            a[i] = (static_cast<uint64_t>(l[2 * i + 1]) << 32) | l[2 * i];
            b[i] = (static_cast<uint64_t>(r[2 * i + 1]) << 32) | r[2 * i];
        }
        Sha3_256::hash_pair(a, b, h);
#pragma unroll
        for (int i = 0; i < 4; ++i) { out[2 * i] = static_cast<uint32_t>(h[i]); out[2 * i + 1] = static_cast<uint32_t>(h[i] >> 32); }
    }
    // Keccak-f is a rolled 24-round loop already
    SNT_HD static void pair_small(const uint32_t* l, const uint32_t* r, const MerkleConsts& c, uint32_t* out) {
        pair(l, r, c, out);
    }
};

// The in-place block table of the reference (model.py:137-146) in the compact
// per-tensor form a kernel can search: leaf k belongs to the tensor t with
// first_leaf[t] <= k < first_leaf[t+1]; empty tensors own no leaves.
struct TensorTable {
    const uint64_t* __restrict__ addr;         // device address of tensor t's bytes
    const uint64_t* __restrict__ nbytes;       // its byte length
    const uint64_t* __restrict__ first_leaf;   // n_tensors + 1 entries
    uint32_t n_tensors;
    uint32_t block_shift;                      // log2(block_size)
    uint64_t n_leaves;
};

struct LeafRef {
    const uint8_t* ptr;
    uint64_t len;
    uint32_t tensor;      // index of the owning tensor
    uint64_t block;       // block index inside that tensor
};

SNT_HD LeafRef locate_leaf(const TensorTable& tab, uint64_t k) {
    uint32_t lo = 0, hi = tab.n_tensors;       // invariant: first_leaf[lo] <= k < first_leaf[hi]
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (tab.first_leaf[mid] <= k) lo = mid; else hi = mid;
    }
    const uint64_t off = (k - tab.first_leaf[lo]) << tab.block_shift;
    const uint64_t bs = 1ull << tab.block_shift;
    const uint64_t left = tab.nbytes[lo] - off;
    LeafRef r;
    r.ptr = reinterpret_cast<const uint8_t*>(tab.addr[lo]) + off;
    r.len = left < bs ? left : bs;
    r.tensor = lo;
    r.block = k - tab.first_leaf[lo];
    return r;
}

SNT_HD uint64_t ceil_shift(uint64_t n, uint32_t s) {
    return s >= 64 ? (n ? 1 : 0) : ((n >> s) + ((n & ((1ull << s) - 1)) ? 1 : 0));
}

}  // namespace snt
