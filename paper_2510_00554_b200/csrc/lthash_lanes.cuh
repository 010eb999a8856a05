// LtHash with persistent LANES: every lane of a warp walks its own item and takes the next item of the warp's
// slice the moment it finishes one, so that ragged items (token arrays of 64..1024 bytes, say) keep all 32
// lanes compressing -- in lthash_kernel a warp runs as long as its longest sample and the other lanes idle,
// which is why large ragged datasets used to be length-sorted first (dataset.py, BALANCE_MIN_SAMPLES).
//
// One iteration of the warp loop = one BLAKE2b compression per busy lane:
//   * lanes on their last block (or idle) CLAIM the next item from a small shared-memory ring of item rows
//     (ballot + rank, no atomics); the ring is refilled 32 rows at a time by the whole warp, one iteration
//     ahead of need (the rows wait in registers across the compression);
//   * every lane stages the block it will compress NEXT -- chunk b+1 of its item, or chunk 0 of the item it
//     just claimed -- into its other staging buffer with cp.async; a ragged tail is the same copy with a
//     source size (the hardware zero-fills the rest, which is exactly BLAKE2b's padding), so there is no
//     tail path and a lane's blocks follow each other, across items, without a pipeline restart;
//   * wait for the block staged one iteration ago, compress it;
//   * lanes that finished an item push the 64-byte digest into a per-warp queue; when the queue is full the
//     warp adds it to the per-source sums TOGETHER: lane l adds u16 lane l of entry e (one conflict-free
//     shared-memory atomic per entry and warp, instead of 32 per finishing group with a select chain).
//
// Reference behaviour: lattice.py:92-101 (lt_hash_block), dataset.py:74-86 (per-source sums, counts,
// undeclared sources), exactly as lthash_kernel; per-source sums do not depend on the order of the samples.
#pragma once
#include "lthash_kernels.cuh"

namespace snt {

constexpr int LTL_MAXW = 12;                                   // warps per persistent CTA (three per scheduler)
constexpr int LTL_RING = 64;                                   // item rows buffered per warp
constexpr int LTL_QCAP = 32;                                   // finished digests buffered per warp
constexpr size_t LTL_STAGE_BYTES_PER_WARP = 2ull * B2S_SLOTS * 32 * sizeof(uint64_t);
constexpr size_t LTL_QUEUE_BYTES = LTL_QCAP * 64ull + LTL_QCAP * sizeof(uint32_t);
// ring rows: address, length, T tag words, source slot
SNT_HD constexpr size_t ltl_ring_bytes(int tag_words) { return (2ull + tag_words) * LTL_RING * sizeof(uint64_t) + LTL_RING * sizeof(uint32_t); }
SNT_HD constexpr size_t ltl_warp_bytes(int tag_words) { return LTL_STAGE_BYTES_PER_WARP + ltl_ring_bytes(tag_words) + LTL_QUEUE_BYTES; }

SNT_D void ltl_cp8(uint64_t* dst, const uint8_t* src) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
SNT_D void ltl_cp4(uint32_t d, const uint8_t* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}
// 4 bytes of which the first `valid` (0..4) come from src; the rest is zero-filled, src is not read beyond them
SNT_D void ltl_cp4_zfill(uint32_t d, const uint8_t* src, int valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src), "r"(valid) : "memory");
}

// Data chunk at g (`avail` valid bytes, the rest of the 128 zero) into slots T..T+15 of `buf` (lane-strided).
template <int T>
SNT_D void ltl_stage(uint64_t* buf, const uint8_t* g, uint64_t avail) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(g);
    if ((a & 3) == 0) {
        if (avail >= 128) {
            if ((a & 7) == 0) {
#pragma unroll
                for (int i = 0; i < 16; ++i) ltl_cp8(buf + (T + i) * 32, g + 8 * i);
            } else {
                const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(buf + T * 32));
#pragma unroll
                for (int i = 0; i < 32; ++i) ltl_cp4(d + (i >> 1) * 256 + (i & 1) * 4, g + 4 * i);
            }
        } else {
            const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(buf + T * 32));
            const int r = static_cast<int>(avail);
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                int v = r - 4 * i;
                v = v < 0 ? 0 : (v > 4 ? 4 : v);
                ltl_cp4_zfill(d + (i >> 1) * 256 + (i & 1) * 4, g + 4 * i, v);
            }
        }
    } else {
        // items at odd addresses: through registers (rare; same loaders as the grid kernel)
        const uint32_t r = avail >= 128 ? 128u : static_cast<uint32_t>(avail);
#pragma unroll 1
        for (int i = 0; i < 16; ++i) buf[(T + i) * 32] = Blake2b::tail_word64(g, i, r);
    }
}

template <class Items, bool SMEM_ACC>
__global__ void __launch_bounds__(LTL_MAXW * 32, 1)
lthash_lanes_kernel(const Items items, uint64_t n, uint32_t n_sources, unsigned long long* __restrict__ acc,
                    unsigned long long* __restrict__ counts, uint8_t* __restrict__ digests,
                    unsigned long long* __restrict__ status) {
    constexpr int T = Items::TAG_WORDS;
    static_assert(T >= 1 && T <= B2S_MAX_TAG_WORDS, "LtHash items carry one or two tag words");
    constexpr uint32_t FULL = 0xffffffffu;
    extern __shared__ __align__(16) uint8_t lt_smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, W = blockDim.x >> 5;

    // dynamic shared memory: per warp [2 staging buffers | item ring | digest queue], then the CTA's accumulators
    constexpr size_t WARP_BYTES = ltl_warp_bytes(T);
    uint8_t* const wbase = lt_smem + static_cast<size_t>(warp) * WARP_BYTES;
    uint64_t* const stage = reinterpret_cast<uint64_t*>(wbase) + lane;       // slot s of buffer f: stage[(f * B2S_SLOTS + s) * 32]
    uint64_t* const r_ptr = reinterpret_cast<uint64_t*>(wbase + LTL_STAGE_BYTES_PER_WARP);
    uint64_t* const r_len = r_ptr + LTL_RING;
    uint64_t* const r_tag = r_len + LTL_RING;
    uint64_t* const r_tag1 = r_tag + LTL_RING;                               // (T == 2 only)
    uint32_t* const r_slot = reinterpret_cast<uint32_t*>(r_tag + T * LTL_RING);
    uint64_t* const q_dig = reinterpret_cast<uint64_t*>(wbase + LTL_STAGE_BYTES_PER_WARP + ltl_ring_bytes(T));
    uint32_t* const q_slot = reinterpret_cast<uint32_t*>(q_dig + LTL_QCAP * 8);
    uint32_t* const sacc = reinterpret_cast<uint32_t*>(lt_smem + static_cast<size_t>(W) * WARP_BYTES);
    uint32_t* const scnt = sacc + static_cast<size_t>(n_sources) * LT_LANES;
    if (SMEM_ACC) {
        for (uint32_t i = threadIdx.x; i < n_sources * (LT_LANES + 1); i += blockDim.x) sacc[i] = 0;
        __syncthreads();
    }

    // this warp's slice of the items: [wb, we), sizes balanced to +-1 over all warps of the grid
    const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * W + warp, nw = static_cast<uint64_t>(gridDim.x) * W;
    const uint64_t per = n / nw, extra = n % nw;
    const uint64_t wb = gw * per + (gw < extra ? gw : extra);
    const uint64_t we = wb + per + (gw < extra ? 1 : 0);

    // add the queued digests to the per-source sums: lane l owns u16 lane l of every entry
    auto flush = [&](uint32_t count) {
        __syncwarp();
        const uint16_t* q16 = reinterpret_cast<const uint16_t*>(q_dig);
#pragma unroll 4
        for (uint32_t e = 0; e < count; ++e) {
            const uint32_t s = q_slot[e];
            const uint32_t v = q16[e * 32 + lane];
            if (SMEM_ACC) atomicAdd(sacc + static_cast<size_t>(s) * LT_LANES + lane, v);
            else atomicAdd(acc + static_cast<size_t>(s) * LT_LANES + lane, static_cast<unsigned long long>(v));
            if (lane == 0) {
                if (SMEM_ACC) atomicAdd(scnt + s, 1u);
                else atomicAdd(counts + s, 1ull);
            }
        }
        __syncwarp();
    };
    auto put_row = [&](uint64_t i, const LtItem& it) {
        const uint32_t s = static_cast<uint32_t>(i - wb) & (LTL_RING - 1);
        r_ptr[s] = reinterpret_cast<uint64_t>(it.ptr);
        r_len[s] = it.len;
        r_tag[s] = it.tag;
        if (T == 2) r_tag1[s] = it.tag1;
        r_slot[s] = it.slot;
    };

    // ring of item rows: [r_head, r_ready) can be claimed, [r_ready, r_issued) is in flight (registers)
    uint64_t r_head = wb, r_ready = wb, r_issued = wb;
#pragma unroll 1
    for (int k = 0; k < 2; ++k) {                              // first fill: up to 64 rows
        const uint64_t i = r_issued + lane;
        if (i < we) put_row(i, items.get(i));
        r_issued = r_issued + 32 < we ? r_issued + 32 : we;
    }
    r_ready = r_issued;
    __syncwarp();
    LtItem pend;
    pend.ptr = nullptr; pend.len = 0; pend.tag = 0; pend.tag1 = 0; pend.slot = 0;
    uint64_t pend_base = 0;
    bool pend_valid = false;
    uint32_t qcount = 0;

    // lane state: the item being hashed (sp/srem describe the chunk about to be compressed) and the claimed next one
    bool have = false, have_nxt = false;
    uint32_t bufsel = 0;
    uint64_t h[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) h[k] = 0;
    const uint8_t* sp = nullptr;
    uint64_t srem = 0, left = 0, tcnt = 0, total = 0;
    uint32_t slot = 0, idx = 0;
    const uint8_t* nptr = nullptr;
    uint64_t nlen = 0;
    uint32_t nslot = 0, nidx = 0;

    for (;;) {
        // (1) the rows fetched during the previous iteration land in the ring
        if (pend_valid) {
            const uint64_t i = pend_base + lane;
            if (i < we) put_row(i, pend);
            r_ready = r_issued;
            pend_valid = false;
            __syncwarp();
        }

        // (2) lanes on their last block, and idle lanes, claim the next items of the slice
        uint64_t* const other = stage + (bufsel ^ 1) * (B2S_SLOTS * 32);
        const bool want = !have_nxt && (!have || left == 1);
        const uint32_t wmask = __ballot_sync(FULL, want);
        bool claimed = false;
        if (wmask) {
            const uint32_t avail = static_cast<uint32_t>(r_ready - r_head);
            const uint32_t rank = __popc(wmask & ((1u << lane) - 1u));
            if (want && rank < avail) {
                const uint64_t i = r_head + rank;
                const uint32_t s = static_cast<uint32_t>(i - wb) & (LTL_RING - 1);
                const uint32_t sl = r_slot[s];
                if (sl >= n_sources) {                         // undeclared source (dataset.py:78-80): counted, skipped
                    if (status) atomicAdd(status, 1ull);
                } else {
                    nptr = reinterpret_cast<const uint8_t*>(r_ptr[s]);
                    nlen = r_len[s];
                    nslot = sl;
                    nidx = static_cast<uint32_t>(i - wb);
                    other[0] = r_tag[s];                       // block 0 of the new item starts with its tag words
                    if (T == 2) other[32] = r_tag1[s];
                    have_nxt = true;
                    claimed = true;
                }
            }
            const uint32_t wn = __popc(wmask);
            r_head += wn < avail ? wn : avail;
        }

        // (3) stage the block this lane compresses NEXT iteration: chunk b+1 of its item, or chunk 0 of the new one
        {
            const bool cont = have && left > 1;
            const uint8_t* g = cont ? sp + 128 : nptr;
            const uint64_t av = cont ? (srem > 128 ? srem - 128 : 0) : nlen;
            if (cont || claimed) ltl_stage<T>(other, g, av);
        }

        // (4) refill the ring one iteration ahead: the loads complete while the block is compressed
        if (r_issued < we && r_issued - r_head <= 32) {
            pend_base = r_issued;
            const uint64_t i = r_issued + lane;
            if (i < we) pend = items.get(i);
            r_issued = r_issued + 32 < we ? r_issued + 32 : we;
            pend_valid = true;
        }

        // (5) everything staged one iteration ago has landed
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 1;" ::: "memory");

        // (6) one compression per busy lane
        const bool busy = have;
        if (busy) {
            const uint64_t* cur = stage + bufsel * (B2S_SLOTS * 32);
            const bool last = left == 1;
            if (!last) {
#pragma unroll
                for (int i = 0; i < T; ++i) other[i * 32] = cur[(16 + i) * 32];   // words carried into the next block
            }
            tcnt += 128;
            Blake2bStaged<32>::compress_staged(h, cur, last ? total : tcnt, last);
            sp += 128;
            srem = srem > 128 ? srem - 128 : 0;
            --left;
        }

        // (7) finished items: digest into the warp's queue (and out, if asked for)
        const bool fin = busy && left == 0;
        const uint32_t fmask = __ballot_sync(FULL, fin);
        if (fmask) {
            const uint32_t nf = __popc(fmask);
            if (qcount + nf > LTL_QCAP) {
                flush(qcount);
                qcount = 0;
            }
            if (fin) {
                const uint32_t pos = qcount + __popc(fmask & ((1u << lane) - 1u));
#pragma unroll
                for (int k = 0; k < 8; ++k) q_dig[pos * 8 + k] = h[k];
                q_slot[pos] = slot;
                if (digests) {
                    uint4* o = reinterpret_cast<uint4*>(digests + (wb + idx) * 64);
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        o[k] = make_uint4(static_cast<uint32_t>(h[2 * k]), static_cast<uint32_t>(h[2 * k] >> 32),
                                          static_cast<uint32_t>(h[2 * k + 1]), static_cast<uint32_t>(h[2 * k + 1] >> 32));
                }
                have = false;
            }
            qcount += nf;
        }

        // (8) the claimed item becomes the current one; its block 0 is what (3) staged this iteration
        const bool promoted = !have && have_nxt;
        if (promoted) {
            sp = nptr;
            srem = nlen;
            total = nlen + 8ull * T;
            left = (total + 127) >> 7;
            tcnt = 0;
            slot = nslot;
            idx = nidx;
            Blake2b::init(h);
            have = true;
            have_nxt = false;
        }
        if (busy || promoted) bufsel ^= 1;

        if (!__any_sync(FULL, have) && r_head >= we) break;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    flush(qcount);

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

}  // namespace snt
