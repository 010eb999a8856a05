// Host build of the per-thread hashing code the kernels run (the SNT_HD
// functions in paper_2510_00554_b200/csrc). Test infrastructure only: it lets
// the CPU suite check message padding, unaligned loads, the leaf locator and
// the pad schedules against hashlib before any GPU time is spent. The product
// never loads this library.
#include <cstring>
#include <vector>

#include "../../paper_2510_00554_b200/csrc/blake2b_staged.cuh"
#include "../../paper_2510_00554_b200/csrc/lthash_kernels.cuh"
#include "../../paper_2510_00554_b200/csrc/merkle_kernels.cuh"

using namespace snt;

template <int ALG>
static void leaf_bytes(const uint8_t* p, uint64_t len, uint8_t* out) {
    using A = AlgTraits<ALG>;
    uint32_t d[A::DW];
    MerkleConsts c;
    memset(&c, 0, sizeof(c));
    c.one = 1;
    A::leaf(p, len, c, d);
    for (int i = 0; i < A::DW; ++i) {
        const uint32_t w = A::to_mem(d[i]);
        memcpy(out + 4 * i, &w, 4);
    }
}

template <int ALG>
static void pair_bytes(const uint8_t* l, const uint8_t* r, const MerkleConsts& c, uint8_t* out, bool small = false) {
    using A = AlgTraits<ALG>;
    uint32_t a[A::DW], b[A::DW], o[A::DW];
    for (int i = 0; i < A::DW; ++i) {
        uint32_t w;
        memcpy(&w, l + 4 * i, 4); a[i] = A::from_mem(w);
        memcpy(&w, r + 4 * i, 4); b[i] = A::from_mem(w);
    }
    if (small) A::pair_small(a, b, c, o); else A::pair(a, b, c, o);
    for (int i = 0; i < A::DW; ++i) {
        const uint32_t w = A::to_mem(o[i]);
        memcpy(out + 4 * i, &w, 4);
    }
}

extern "C" {

int hc_leaf(int alg, const uint8_t* p, uint64_t len, uint8_t* out) {
    switch (alg) {
        case ALG_SHA256: leaf_bytes<ALG_SHA256>(p, len, out); return 0;
        case ALG_BLAKE2B: leaf_bytes<ALG_BLAKE2B>(p, len, out); return 0;
        case ALG_SHA3_256: leaf_bytes<ALG_SHA3_256>(p, len, out); return 0;
    }
    return -1;
}

// small != 0: the rolled formulation of the node hash (AlgTraits::pair_small)
int hc_pair(int alg, const uint8_t* l, const uint8_t* r, uint8_t* out, int small) {
    MerkleConsts c;
    memset(&c, 0, sizeof(c));
    Sha256::pad_schedule(64, c.sha256_pad_node);
    c.one = 1;
    switch (alg) {
        case ALG_SHA256: pair_bytes<ALG_SHA256>(l, r, c, out, small != 0); return 0;
        case ALG_BLAKE2B: pair_bytes<ALG_BLAKE2B>(l, r, c, out, small != 0); return 0;
        case ALG_SHA3_256: pair_bytes<ALG_SHA3_256>(l, r, c, out, small != 0); return 0;
    }
    return -1;
}

// the aligned SHA-256 leaf path of the kernels (p must be 16-byte aligned): the full 64-byte blocks in two
// slices [0, split) and [split, nfull) -- the time-sliced chains resume a leaf like this -- then the
// constant padding block for a leaf that is a whole number of blocks, Sha256::finish for a ragged one
int hc_sha256_aligned(const uint8_t* p, uint64_t len, uint32_t split, uint8_t* out) {
    uint32_t kw[64], s[8];
    const uint32_t nfull = static_cast<uint32_t>(len >> 6);
    if (split > nfull) split = nfull;
    Sha256::init(s);
    sha256_blocks_aligned(p, 0, split, s);
    sha256_blocks_aligned(p, split, nfull, s);
    if ((len & 63) == 0 && len > 0) {
        Sha256::pad_schedule(len, kw);
        Sha256::compress_const(s, kw);
    } else {
        Sha256::finish(p + (static_cast<uint64_t>(nfull) << 6), static_cast<uint32_t>(len & 63), len, s);
    }
    for (int i = 0; i < 8; ++i) {
        const uint32_t w = bswap32(s[i]);
        memcpy(out + 4 * i, &w, 4);
    }
    return 0;
}

// BLAKE2b (T tag words) and SHA3-256 hashed in slices of `slice` blocks, the state carried between slices
// the way the time-sliced chains park it (hash_blocks / absorb_blocks)
int hc_blake2b_sliced(int T, uint64_t tag0, uint64_t tag1, const uint8_t* p, uint64_t len, uint32_t slice, uint8_t* out) {
    uint64_t h[8];
    Blake2b::init(h);
    const uint64_t n = T == 0 ? Blake2bStaged<1>::block_count<0>(len) : T == 1 ? Blake2bStaged<1>::block_count<1>(len)
                                                                               : Blake2bStaged<1>::block_count<2>(len);
    for (uint64_t b = 0; b < n; b += slice) {
        uint64_t bufs[2 * B2S_SLOTS];
        memset(bufs, 0x5A, sizeof(bufs));        // a fresh thread's staging buffers: nothing may be carried in them
        // odd slices through the compress-from-the-staging-buffer form (ROLLED; on the host its rounds are the unrolled
        // ones, what differs is that the carried words are moved before the block is compressed)
        const bool rolled = (b / slice) & 1;
        if (T == 0) rolled ? Blake2bStaged<1>::hash_blocks<0, true>(bufs, tag0, tag1, p, len, b, b + slice, h)
                           : Blake2bStaged<1>::hash_blocks<0>(bufs, tag0, tag1, p, len, b, b + slice, h);
        else if (T == 1) rolled ? Blake2bStaged<1>::hash_blocks<1, true>(bufs, tag0, tag1, p, len, b, b + slice, h)
                                : Blake2bStaged<1>::hash_blocks<1>(bufs, tag0, tag1, p, len, b, b + slice, h);
        else rolled ? Blake2bStaged<1>::hash_blocks<2, true>(bufs, tag0, tag1, p, len, b, b + slice, h)
                    : Blake2bStaged<1>::hash_blocks<2>(bufs, tag0, tag1, p, len, b, b + slice, h);
    }
    memcpy(out, h, 64);
    return 0;
}

int hc_sha3_sliced(const uint8_t* p, uint64_t len, uint32_t slice, uint8_t* out) {
    uint64_t a[25];
    memset(a, 0, sizeof(a));
    const uint64_t n = Sha3_256::block_count(len);
    for (uint64_t u = 0; u < n; u += slice) Sha3_256::absorb_blocks(a, p, len, u, u + slice);
    memcpy(out, a, 32);
    return 0;
}

// BLAKE2b-512(tag words || data), T in {0, 1, 2}
int hc_blake2b_tagged(int T, uint64_t tag0, uint64_t tag1, const uint8_t* p, uint64_t len, uint8_t* out) {
    uint64_t h[8];
    if (T == 0) Blake2b::hash_message<0>(tag0, tag1, p, len, h);
    else if (T == 1) Blake2b::hash_message<1>(tag0, tag1, p, len, h);
    else if (T == 2) Blake2b::hash_message<2>(tag0, tag1, p, len, h);
    else return -1;
    memcpy(out, h, 64);
    return 0;
}

// the shared-memory staged BLAKE2b (blake2b_staged.cuh) with the stager as a memcpy
int hc_blake2b_staged(int T, uint64_t tag0, uint64_t tag1, const uint8_t* p, uint64_t len, uint8_t* out) {
    uint64_t h[8];
    uint64_t bufs[2 * B2S_SLOTS];
    memset(bufs, 0xA5, sizeof(bufs));        // stale slots must never leak into a block
    if (T == 0) Blake2bStaged<1>::hash_message<0>(bufs, tag0, tag1, p, len, h);
    else if (T == 1) Blake2bStaged<1>::hash_message<1>(bufs, tag0, tag1, p, len, h);
    else if (T == 2) Blake2bStaged<1>::hash_message<2>(bufs, tag0, tag1, p, len, h);
    else return -1;
    memcpy(out, h, 64);
    return 0;
}

// leaf locator over a host copy of the tensor table: returns offset within
// the tensor through *off, tensor index through *t, length through *len
int hc_locate(const uint64_t* nbytes, uint32_t n_tensors, uint32_t block_size, uint64_t k, uint32_t* t,
              uint64_t* off, uint64_t* len) {
    uint32_t shift = 0;
    while ((1u << shift) < block_size) ++shift;
    std::vector<uint64_t> addr(n_tensors), first(n_tensors + 1);
    uint64_t leaves = 0, base = 1ull << 40;
    for (uint32_t i = 0; i < n_tensors; ++i) {
        addr[i] = base;
        base += (nbytes[i] + 4095) & ~4095ull;
        base += 4096;
        first[i] = leaves;
        leaves += (nbytes[i] + block_size - 1) >> shift;
    }
    first[n_tensors] = leaves;
    if (k >= leaves) return -1;
    TensorTable tab;
    tab.addr = addr.data();
    tab.nbytes = nbytes;
    tab.first_leaf = first.data();
    tab.n_tensors = n_tensors;
    tab.block_shift = shift;
    tab.n_leaves = leaves;
    const LeafRef r = locate_leaf(tab, k);
    const uint64_t a = reinterpret_cast<uint64_t>(r.ptr);
    for (uint32_t i = 0; i < n_tensors; ++i) {
        if (nbytes[i] && a >= addr[i] && a < addr[i] + nbytes[i]) {
            *t = i;
            *off = a - addr[i];
            *len = r.len;
            return 0;
        }
    }
    return -2;
}

}  // extern "C"
