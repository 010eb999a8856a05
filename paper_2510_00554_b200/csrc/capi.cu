// C ABI of the B200 hashing engine (see include/sentinel_b200.h).
// Host-side orchestration only: argument checks, launch geometry, the chain of
// level-reducer launches. No torch types, no allocation on the hashing path.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/sentinel_b200.h"
#include "gather_kernels.cuh"
#include "lthash_kernels.cuh"
#include "lthash_lanes.cuh"
#include "lthash_quad.cuh"
#include "merkle_fused.cuh"
#include "merkle_kernels.cuh"

using namespace snt;

namespace {

thread_local char g_cuda_err[256] = "";

// diagnostic only: number of kernels this library has launched in this process
std::atomic<uint64_t> g_launches{0};
// how snt_merkle_inplace / snt_merkle_leaves schedule their work (snt_merkle_schedule)
std::atomic<int> g_schedule{SNT_SCHEDULE_PERSISTENT};
// diagnostic only: device buffer of 6 x u64 per CTA the fused kernel writes its timeline into
std::atomic<unsigned long long*> g_fused_trace{nullptr};

int cuda_fail(cudaError_t e, const char* where) {
    snprintf(g_cuda_err, sizeof(g_cuda_err), "%s: %s", where, cudaGetErrorString(e));
    return SNT_ERR_RESOURCE;
}

#define SNT_CUDA(call)                                        \
    do {                                                      \
        cudaError_t e__ = (call);                             \
        if (e__ != cudaSuccess) return cuda_fail(e__, #call); \
    } while (0)

uint32_t ceil_log2(uint64_t n) {
    uint32_t l = 0;
    while ((1ull << l) < n) ++l;
    return l;
}

uint64_t cdiv_shift(uint64_t n, uint32_t s) { return ceil_shift(n, s); }

bool valid_alg(int alg) { return alg == SNT_SHA256 || alg == SNT_BLAKE2B || alg == SNT_SHA3_256; }

uint32_t max_levels(int alg) {
    return alg == SNT_BLAKE2B ? ReduceShape<ALG_BLAKE2B>::MAX_LEVELS : ReduceShape<ALG_SHA256>::MAX_LEVELS;
}

// A big level starts with a WIDE launch: WIDE_LEVELS levels over full-width CTAs that each emit
// 2^(max_levels - WIDE_LEVELS) nodes, so the bulk of the node hashes (7/8 of them) run with every thread
// busy; the narrowing launches that follow see an 8x smaller level.
#ifndef SNT_WIDE_LEVELS
#define SNT_WIDE_LEVELS 3
#endif
constexpr uint32_t WIDE_LEVELS = SNT_WIDE_LEVELS;
#ifndef SNT_FUSED_MAXW_SHA256
#define SNT_FUSED_MAXW_SHA256 24
#endif
constexpr uint64_t WIDE_MIN_NODES = 1ull << 18;    // below this the extra launch costs more than it saves (tools/tree_probe.py)

const MerkleConsts& node_consts() {
    static const MerkleConsts c = [] {
        MerkleConsts k;
        memset(&k, 0, sizeof(k));
        Sha256::pad_schedule(64, k.sha256_pad_node);
        k.one = 1;
        return k;
    }();
    return c;
}

// SMs of the current device (one persistent CTA each in the fused kernel); 148 when there is no device
// to ask, so that the size queries of the ABI work on a machine without a GPU.
int sm_count() {
    static const int n = [] {
        int dev = 0, sms = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) {
            cudaGetLastError();
            return 148;
        }
        return sms;
    }();
    return n;
}

// Worker warps per persistent CTA, upper bound per algorithm (registers: 65,536 / (32 * W)).
constexpr int FUSED_MAXW_SHA256 = SNT_FUSED_MAXW_SHA256;
constexpr int FUSED_MAXW_WIDE = 16;      // SHA3-256
#ifndef SNT_FUSED_MAXW_BLAKE2B
#define SNT_FUSED_MAXW_BLAKE2B 8
#endif
constexpr int FUSED_MAXW_BLAKE2B = SNT_FUSED_MAXW_BLAKE2B;    // fewer, fatter warps: 34 KB of unrolled rounds per warp position, 128+ registers
size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

// Workspace of one (algorithm, node count): [ping-pong levels of the multi-launch reducer | completion
// counters | stage nodes]. The last two belong to the fused kernel; the counters must be zero before
// its first launch (snt_merkle_work_init) and it hands them back zeroed.
struct WorkLayout {
    size_t pingpong, counters_off, counters_bytes, nodes_off, nodes_bytes, total;
};

size_t pingpong_bytes(int alg, uint64_t count) {
    // two ping-pong buffers, each able to hold the widest intermediate level:
    // every launch but the last folds max_levels(alg) levels, so the widest
    // intermediate has ceil(count / 2^max_levels) nodes
    // -- or, for a level big enough for the wide first launch, ceil(count / 2^WIDE_LEVELS) nodes
    const uint64_t widest = count >= WIDE_MIN_NODES ? cdiv_shift(count, WIDE_LEVELS) : cdiv_shift(count, max_levels(alg));
    return align256(2 * static_cast<size_t>(widest + 1) * snt_digest_len(alg));
}

WorkLayout work_layout(int alg, uint64_t count) {
    WorkLayout w;
    w.pingpong = pingpong_bytes(alg, count);
    // groups of stage 0 <= ceil(count / 32), every later stage at most halves: < 2 * that + one per stage
    const size_t n_groups = 2 * static_cast<size_t>(cdiv_shift(count, FUSED_MIN_LEVELS)) + 2 * FUSED_MAX_STAGES;
    w.counters_off = w.pingpong;
    w.counters_bytes = align256(n_groups * sizeof(uint32_t));
    w.nodes_off = w.counters_off + w.counters_bytes;
    w.nodes_bytes = align256(n_groups * snt_digest_len(alg));
    w.total = w.nodes_off + w.nodes_bytes;
    return w;
}

}  // namespace

struct snt_model_plan {
    uint64_t* d_table = nullptr;     // addr[n] | nbytes[n] | first_leaf[n + 1] | irregular[n_irregular]
    uint32_t n_irregular = 0;        // leaves of tensors that are not 16-byte aligned (SHA-256 generic path)
    cudaStream_t stream = nullptr;   // the stream the table was allocated and filled on
    std::vector<uint64_t> host;      // staging copy of the table (kept alive until destroy)
    uint32_t n_tensors = 0;
    uint32_t block_shift = 0;
    uint64_t n_leaves = 0;
    uint64_t total_bytes = 0;
    MerkleConsts consts;
    TensorTable table() const {
        TensorTable t;
        t.addr = d_table;
        t.nbytes = d_table + n_tensors;
        t.first_leaf = d_table + 2ull * n_tensors;
        t.n_tensors = n_tensors;
        t.block_shift = block_shift;
        t.n_leaves = n_leaves;
        return t;
    }
};

extern "C" {

const char* snt_strerror(int status) {
    switch (status) {
        case SNT_OK: return "ok";
        case SNT_ERR_INVALID_INPUT: return "invalid input";
        case SNT_ERR_INVALID_STATE: return "invalid state";
        case SNT_ERR_CONFIG: return "bad hashing configuration";
        case SNT_ERR_VALIDATION: return "validation failed";
        case SNT_ERR_RESOURCE: return "CUDA resource error";
        default: return "unknown status";
    }
}

const char* snt_last_cuda_error(void) { return g_cuda_err; }

uint32_t snt_abi_version(void) { return 3; }

uint64_t snt_debug_launch_count(void) { return g_launches.load(); }

int snt_merkle_schedule(int schedule) {
    const int old = g_schedule.load();
    if (schedule == SNT_SCHEDULE_PERSISTENT || schedule == SNT_SCHEDULE_FUSED || schedule == SNT_SCHEDULE_GRID)
        g_schedule.store(schedule);
    return old;
}

void snt_debug_fused_trace(void* d_trace) { g_fused_trace.store(static_cast<unsigned long long*>(d_trace)); }

uint32_t snt_digest_len(int alg) {
    switch (alg) {
        case SNT_SHA256: return 32;
        case SNT_BLAKE2B: return 64;
        case SNT_SHA3_256: return 32;
        default: return 0;
    }
}

int snt_model_plan_create(const void* const* d_tensor_ptrs, const uint64_t* tensor_nbytes,
                          uint32_t n_tensors, uint32_t block_size, snt_stream_t stream,
                          snt_model_plan** out_plan) {
    if (!out_plan) return SNT_ERR_INVALID_INPUT;
    *out_plan = nullptr;
    if (block_size < 64 || (block_size & (block_size - 1))) return SNT_ERR_CONFIG;   // model.py:94-95
    if (n_tensors == 0 || !d_tensor_ptrs || !tensor_nbytes) return SNT_ERR_INVALID_INPUT;
    uint32_t shift = 0;
    while ((1u << shift) < block_size) ++shift;
    std::vector<uint64_t> host(3ull * n_tensors + 1);
    std::vector<uint64_t> irregular;
    uint64_t leaves = 0, total = 0;
    for (uint32_t t = 0; t < n_tensors; ++t) {
        const uint64_t addr = reinterpret_cast<uint64_t>(d_tensor_ptrs[t]);
        const uint64_t nb = tensor_nbytes[t];
        host[t] = addr;
        host[n_tensors + t] = nb;
        host[2ull * n_tensors + t] = leaves;
        const uint64_t count = (nb + block_size - 1) >> shift;
        if (nb && !d_tensor_ptrs[t]) return SNT_ERR_INVALID_INPUT;
        if (addr & 15) {
            for (uint64_t j = 0; j < count; ++j) irregular.push_back(leaves + j);
        }
        leaves += count;
        total += nb;
    }
    if (irregular.size() > 0xffffffffull) return SNT_ERR_INVALID_INPUT;
    host[3ull * n_tensors] = leaves;
    host.insert(host.end(), irregular.begin(), irregular.end());
    if (total == 0) return SNT_ERR_INVALID_INPUT;                                     // model.py:166-168
    snt_model_plan* p = new (std::nothrow) snt_model_plan();
    if (!p) return SNT_ERR_RESOURCE;
    p->n_tensors = n_tensors;
    p->block_shift = shift;
    p->n_leaves = leaves;
    p->total_bytes = total;
    p->n_irregular = static_cast<uint32_t>(irregular.size());
    p->consts = node_consts();
    Sha256::pad_schedule(block_size, p->consts.sha256_pad_leaf);
    // stream-ordered allocation and copy: no device-wide synchronisation on the hashing path
    p->stream = static_cast<cudaStream_t>(stream);
    p->host.swap(host);
    const size_t bytes = p->host.size() * sizeof(uint64_t);
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&p->d_table), bytes, p->stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(p->d_table, p->host.data(), bytes, cudaMemcpyHostToDevice, p->stream);
    if (e != cudaSuccess) {
        if (p->d_table) cudaFreeAsync(p->d_table, p->stream);
        delete p;
        return cuda_fail(e, "snt_model_plan_create");
    }
    *out_plan = p;
    return SNT_OK;
}

void snt_model_plan_destroy(snt_model_plan* plan) {
    if (!plan) return;
    if (plan->d_table) cudaFreeAsync(plan->d_table, plan->stream);   // ordered after the launches on that stream
    delete plan;
}

uint64_t snt_model_plan_leaf_count(const snt_model_plan* plan) { return plan ? plan->n_leaves : 0; }
uint64_t snt_model_plan_total_bytes(const snt_model_plan* plan) { return plan ? plan->total_bytes : 0; }

size_t snt_merkle_work_bytes(int alg, uint64_t count) {
    if (!valid_alg(alg)) return 0;
    return work_layout(alg, count).total;
}

int snt_merkle_work_init(void* d_work, size_t work_bytes, snt_stream_t stream) {
    if (!d_work || work_bytes == 0) return SNT_ERR_INVALID_INPUT;
    SNT_CUDA(cudaMemsetAsync(d_work, 0, work_bytes, static_cast<cudaStream_t>(stream)));
    return SNT_OK;
}

}  // extern "C"

namespace {

// CTA size of the level reducer, by grid size. Every CTA walks its levels one barrier at a
// time, so a launch is as slow as (critical path of one CTA) x (number of waves):
//   <= 5/SM   -> 256 threads (512 threads were measured no faster: with 16 warps per CTA the
//                first level is ALU-bound instead of latency-bound, same time);
//   more      -> 128 threads: twice as many CTAs fit per SM (registers), fewer waves
//                (BLAKE2b / SHA3-256 trees of 800k leaves: -8% / -4%; SHA-256 neutral).
template <int ALG, int THREADS>
int launch_reduce_t(const uint8_t* in, uint64_t first, uint64_t n_in, uint64_t level_count, uint32_t levels,
                    uint32_t glog, const MerkleConsts& c, uint8_t* out, uint64_t n_ctas, cudaStream_t s) {
    static const cudaError_t carve = cudaFuncSetAttribute(
        merkle_reduce_kernel<ALG, THREADS>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    (void)carve;
    merkle_reduce_kernel<ALG, THREADS><<<static_cast<unsigned>(n_ctas), THREADS, 0, s>>>(
        in, first, n_in, level_count, levels, glog, c, out);
    SNT_CUDA(cudaGetLastError());
    ++g_launches;
    return SNT_OK;
}

template <int ALG>
int launch_reduce(const uint8_t* in, uint64_t first, uint64_t n_in, uint64_t level_count,
                  uint32_t levels, uint32_t glog, const MerkleConsts& c, uint8_t* out, cudaStream_t s) {
    const uint64_t n_ctas = cdiv_shift(n_in, levels + glog);
    if (n_ctas > 0x7fffffffull) return SNT_ERR_INVALID_INPUT;
    if (glog == 0 && n_ctas <= 5 * 148)
        return launch_reduce_t<ALG, 256>(in, first, n_in, level_count, levels, glog, c, out, n_ctas, s);
    return launch_reduce_t<ALG, 128>(in, first, n_in, level_count, levels, glog, c, out, n_ctas, s);
}

int launch_reduce_alg(int alg, const uint8_t* in, uint64_t first, uint64_t n_in, uint64_t level_count,
                      uint32_t levels, uint32_t glog, const MerkleConsts& c, uint8_t* out, cudaStream_t s) {
    switch (alg) {
        case SNT_SHA256: return launch_reduce<ALG_SHA256>(in, first, n_in, level_count, levels, glog, c, out, s);
        case SNT_BLAKE2B: return launch_reduce<ALG_BLAKE2B>(in, first, n_in, level_count, levels, glog, c, out, s);
        default: return launch_reduce<ALG_SHA3_256>(in, first, n_in, level_count, levels, glog, c, out, s);
    }
}

// Apply `levels` levels to the node range, max_levels(alg) at a time,
// ping-ponging intermediates through `work`; the last launch writes `out`.
int reduce_chain(int alg, const uint8_t* in, uint64_t first, uint64_t n_in, uint64_t level_count,
                 uint32_t levels, uint8_t* work, size_t work_bytes, uint8_t* out,
                 const MerkleConsts& c, cudaStream_t s) {
    const uint32_t dlen = snt_digest_len(alg);
    // only the ping-pong part of a full workspace: what lies behind it belongs to the fused kernel
    const size_t pp = pingpong_bytes(alg, n_in);
    const size_t half = (work_bytes < pp ? work_bytes : pp) / 2;
    int flip = 0;
    const uint8_t* src = in;
    while (levels > 0) {
        const uint32_t cap = max_levels(alg);
        uint32_t m = levels < cap ? levels : cap;
        uint32_t glog = 0;
        if (n_in >= WIDE_MIN_NODES && levels > WIDE_LEVELS && work &&
            cdiv_shift(n_in, WIDE_LEVELS) * dlen <= half) {          // (a caller with a small workspace keeps the old schedule)
            m = WIDE_LEVELS;
            glog = cap - WIDE_LEVELS;
        }
        const uint64_t n_out = cdiv_shift(n_in, m);
        uint8_t* dst = out;
        if (levels > m) {
            if (!work || n_out * dlen > half) return SNT_ERR_RESOURCE;
            dst = work + (flip ? half : 0);
            flip ^= 1;
        }
        const int rc = launch_reduce_alg(alg, src, first, n_in, level_count, m, glog, c, dst, s);
        if (rc != SNT_OK) return rc;
        src = dst;
        first >>= m;
        n_in = n_out;
        level_count = cdiv_shift(level_count, m);
        levels -= m;
    }
    return SNT_OK;
}

template <int ALG>
int launch_leaves(const snt_model_plan* plan, uint64_t begin, uint64_t end, uint8_t* d_leaves,
                  cudaStream_t s) {
    const uint64_t n = end - begin;
    const uint32_t irr_ctas = ALG == ALG_SHA256 ? (plan->n_irregular + LEAF_THREADS - 1) / LEAF_THREADS : 0;
    const uint64_t grid = (n + LEAF_THREADS - 1) / LEAF_THREADS + irr_ctas;
    if (grid > 0x7fffffffull) return SNT_ERR_INVALID_INPUT;
    const uint64_t* irregular = plan->d_table + 3ull * plan->n_tensors + 1;
    merkle_leaf_kernel<ALG><<<static_cast<unsigned>(grid), LEAF_THREADS, leaf_stage_bytes<ALG>(), s>>>(
        plan->table(), plan->consts, begin, end, irregular, plan->n_irregular, irr_ctas, d_leaves);
    SNT_CUDA(cudaGetLastError());
    ++g_launches;
    return SNT_OK;
}

// The whole hash of leaves [begin, end) down to level `levels` in one launch (merkle_fused.cuh).
template <int ALG, int MAXW>
int launch_fused(const snt_model_plan* plan, uint64_t begin, uint64_t end, uint32_t levels, int warps, uint8_t* d_leaves,
                 uint8_t* work, const WorkLayout& wl, uint8_t* d_out, cudaStream_t s) {
    constexpr size_t stage_bytes = fused_smem_bytes<ALG, MAXW>();
    static const cudaError_t attr = cudaFuncSetAttribute(
        merkle_fused_kernel<ALG, MAXW>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(stage_bytes));
    if (attr != cudaSuccess) return cuda_fail(attr, "cudaFuncSetAttribute(merkle_fused_kernel)");
    FusedArgs a;
    memset(&a, 0, sizeof(a));
    a.tab = plan->table();
    a.leaf_begin = begin;
    a.n = end - begin;
    if (ALG == ALG_SHA256 && plan->n_irregular) {
        const uint64_t* irr = plan->host.data() + 3ull * plan->n_tensors + 1;
        const uint64_t* lo = std::lower_bound(irr, irr + plan->n_irregular, begin);
        const uint64_t* hi = std::lower_bound(lo, irr + plan->n_irregular, end);
        a.irregular = plan->d_table + 3ull * plan->n_tensors + 1 + (lo - irr);
        a.n_irregular = static_cast<uint32_t>(hi - lo);
    }
    a.d_leaves = d_leaves;
    a.trace = g_fused_trace.load();
    a.flip = getenv("SNT_FUSED_FLIP") ? 1u : 0u;
    // stages: 8 levels from the leaves, then 6 at a time
    uint32_t left = levels;
    uint64_t n_in = a.n;
    uint32_t* cnt = reinterpret_cast<uint32_t*>(work + wl.counters_off);
    uint8_t* nodes = work + wl.nodes_off;
    const uint32_t dlen = AlgTraits<ALG>::DIGEST_BYTES;
    while (left > 0) {
        const uint32_t st = a.tree.n_stages++;
        const uint32_t m = st == 0 ? (left < FUSED_FIRST_STAGE_LEVELS ? left : FUSED_FIRST_STAGE_LEVELS)
                                   : (left < FUSED_NEXT_STAGE_LEVELS ? left : FUSED_NEXT_STAGE_LEVELS);
        const uint64_t groups = cdiv_shift(n_in, m);
        a.tree.m[st] = m;
        a.tree.n_in[st] = n_in;
        a.tree.cnt[st] = cnt;
        a.tree.nodes[st] = left == m ? d_out : nodes;
        cnt += groups;
        nodes += groups * dlen;
        n_in = groups;
        left -= m;
    }
    const uint64_t chains = ((a.n + 31) >> 5) + ((a.n_irregular + 31) >> 5);
    const uint64_t sms = static_cast<uint64_t>(sm_count());
    const unsigned grid = static_cast<unsigned>(chains < sms ? chains : sms);
    if (getenv("SNT_FUSED_NOTREE")) a.tree.n_stages = 0;          // diagnostics: leaf phase alone (no root)
    merkle_fused_kernel<ALG, MAXW><<<grid, warps * 32, stage_bytes, s>>>(a, plan->consts);
    SNT_CUDA(cudaGetLastError());
    ++g_launches;
    return SNT_OK;
}

// Worker warps per persistent CTA: a multiple of four (one per scheduler) not above the chains every SM
// gets, so that the time-sliced tail keeps every scheduler equally busy.
int fused_warps(const snt_model_plan* plan, int alg, uint64_t begin, uint64_t end, int maxw) {
    uint64_t chains = (end - begin + 31) >> 5;
    if (alg == SNT_SHA256) chains += (plan->n_irregular + 31) >> 5;      // an upper bound is good enough here
    const uint64_t sms = static_cast<uint64_t>(sm_count());
    const uint64_t grid = chains < sms ? chains : sms;
    int warps = static_cast<int>((chains / (grid ? grid : 1)) & ~3ull);
    if (const char* force = getenv("SNT_FUSED_WARPS")) warps = atoi(force) & ~3;
    return warps < 4 ? 4 : (warps > maxw ? maxw : warps);
}

// Can the fused kernel take this job? It needs the full workspace, a tree deep enough for a chain of 32
// leaves to sit inside one first-stage group, and no more stages than FusedTree holds.
bool fused_applies(uint64_t n, uint32_t levels, size_t work_bytes, const WorkLayout& wl) {
    if (levels < FUSED_MIN_LEVELS || work_bytes < wl.total || n == 0) return false;
    const uint32_t rest = levels > FUSED_FIRST_STAGE_LEVELS ? levels - FUSED_FIRST_STAGE_LEVELS : 0;
    return 1 + (rest + FUSED_NEXT_STAGE_LEVELS - 1) / FUSED_NEXT_STAGE_LEVELS <= FUSED_MAX_STAGES;
}

// The persistent kernel for [begin, end): leaves only (levels = 0) or with the tree folded in.
int fused_dispatch(const snt_model_plan* plan, int alg, uint64_t begin, uint64_t end, uint32_t levels, uint8_t* leaves,
                   uint8_t* work, const WorkLayout& wl, uint8_t* out, cudaStream_t s) {
    const int warps = fused_warps(plan, alg, begin, end, alg == SNT_SHA256 ? FUSED_MAXW_SHA256
                                                          : alg == SNT_BLAKE2B ? FUSED_MAXW_BLAKE2B : FUSED_MAXW_WIDE);
    switch (alg) {
        case SNT_SHA256:
            // two builds of the SHA-256 kernel: up to 16 warps with the registers ptxas likes best (~96),
            // up to 24 warps capped at 80 registers for the models that have that many chains per SM
            if (warps <= 16) return launch_fused<ALG_SHA256, 16>(plan, begin, end, levels, warps, leaves, work, wl, out, s);
            return launch_fused<ALG_SHA256, FUSED_MAXW_SHA256>(plan, begin, end, levels, warps, leaves, work, wl, out, s);
        case SNT_BLAKE2B:
            return launch_fused<ALG_BLAKE2B, FUSED_MAXW_BLAKE2B>(plan, begin, end, levels, warps, leaves, work, wl, out, s);
        default:
            return launch_fused<ALG_SHA3_256, FUSED_MAXW_WIDE>(plan, begin, end, levels, warps, leaves, work, wl, out, s);
    }
}

// The leaf stage alone, scheduled as asked: the persistent time-sliced kernel with the tree switched off, or
// the plain one-thread-per-leaf grid.
int leaf_stage(const snt_model_plan* plan, int alg, uint64_t begin, uint64_t end, uint8_t* leaves, cudaStream_t s) {
    if (g_schedule.load() == SNT_SCHEDULE_GRID) {
        switch (alg) {
            case SNT_SHA256: return launch_leaves<ALG_SHA256>(plan, begin, end, leaves, s);
            case SNT_BLAKE2B: return launch_leaves<ALG_BLAKE2B>(plan, begin, end, leaves, s);
            default: return launch_leaves<ALG_SHA3_256>(plan, begin, end, leaves, s);
        }
    }
    return fused_dispatch(plan, alg, begin, end, 0, leaves, nullptr, WorkLayout{}, nullptr, s);
}

template <int ALG>
int launch_blocks(const uint8_t* base, const uint64_t* off, const uint64_t* len, uint64_t n,
                  uint8_t* out, cudaStream_t s) {
    const uint64_t grid = (n + LEAF_THREADS - 1) / LEAF_THREADS;
    if (grid > 0x7fffffffull) return SNT_ERR_INVALID_INPUT;
    hash_blocks_kernel<ALG><<<static_cast<unsigned>(grid), LEAF_THREADS, leaf_stage_bytes<ALG>(), s>>>(
        base, off, len, n, node_consts(), out);
    SNT_CUDA(cudaGetLastError());
    ++g_launches;
    return SNT_OK;
}

// Largest launch that takes the four-lanes-per-item kernel (SNT_LT_QUAD_MAX overrides it for the probes).
uint64_t quad_max_items() {
    static const uint64_t v = [] {
        const char* e = getenv("SNT_LT_QUAD_MAX");
        return e ? static_cast<uint64_t>(strtoull(e, nullptr, 10)) : LT_QUAD_MAX_ITEMS;
    }();
    return v;
}

// Four lanes per item (lthash_quad.cuh): small launches, where latency is everything.
template <class Items>
int launch_lthash_quad(const Items& items, uint64_t n, uint32_t n_sources, unsigned long long* acc,
                       unsigned long long* counts, uint8_t* dig, unsigned long long* status, cudaStream_t s) {
    if (n == 0) return SNT_OK;
    constexpr int quads = LT_QUAD_THREADS / 4;
    const unsigned grid = static_cast<unsigned>((n + quads - 1) / quads);
    const size_t regions = static_cast<size_t>(quads) * QUAD_REGION_BYTES;
    if (n_sources <= static_cast<uint32_t>(LT_SMEM_SOURCES)) {
        const size_t smem = regions + static_cast<size_t>(n_sources) * (LT_LANES + 1) * sizeof(uint32_t);
        lthash_quad_kernel<Items, true><<<grid, LT_QUAD_THREADS, smem, s>>>(items, n, n_sources, acc, counts, dig, status);
    } else {
        lthash_quad_kernel<Items, false><<<grid, LT_QUAD_THREADS, regions, s>>>(items, n, n_sources, acc, counts, dig, status);
    }
    SNT_CUDA(cudaGetLastError());
    ++g_launches;
    return SNT_OK;
}

// One thread per item on a plain grid (lthash_kernel).
template <class Items>
int launch_lthash_grid(const Items& items, uint64_t n, uint32_t n_sources, unsigned long long* acc,
                       unsigned long long* counts, uint8_t* dig, unsigned long long* status, cudaStream_t s) {
    if (n == 0) return SNT_OK;
    const uint64_t grid = (n + LT_THREADS - 1) / LT_THREADS;
    if (grid > 0x7fffffffull) return SNT_ERR_INVALID_INPUT;
    if (n_sources <= static_cast<uint32_t>(LT_SMEM_SOURCES)) {
        const size_t smem = LT_STAGE_BYTES + static_cast<size_t>(n_sources) * (LT_LANES + 1) * sizeof(uint32_t);
        lthash_kernel<Items, true><<<static_cast<unsigned>(grid), LT_THREADS, smem, s>>>(
            items, n, n_sources, acc, counts, dig, status);
    } else {
        lthash_kernel<Items, false><<<static_cast<unsigned>(grid), LT_THREADS, LT_STAGE_BYTES, s>>>(
            items, n, n_sources, acc, counts, dig, status);
    }
    SNT_CUDA(cudaGetLastError());
    ++g_launches;
    return SNT_OK;
}

template <class Items, bool SMEM_ACC>
int launch_lthash_chains(const Items& items, uint64_t n, uint32_t n_sources, unsigned long long* acc,
                         unsigned long long* counts, uint8_t* dig, unsigned long long* status, cudaStream_t s) {
    const size_t smem = LT_CHAIN_STAGE_BYTES + LT_CHAIN_PARK_BYTES +
                        (SMEM_ACC ? static_cast<size_t>(n_sources) * (LT_LANES + 1) * sizeof(uint32_t) : 0);
    static const cudaError_t attr = cudaFuncSetAttribute(
        lthash_chain_kernel<Items, SMEM_ACC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
        static_cast<int>(LT_CHAIN_STAGE_BYTES + LT_CHAIN_PARK_BYTES + LT_SMEM_SOURCES * (LT_LANES + 1) * sizeof(uint32_t)));
    if (attr != cudaSuccess) return cuda_fail(attr, "cudaFuncSetAttribute(lthash_chain_kernel)");
    const uint64_t chains = (n + 31) >> 5;
    const uint64_t sms = static_cast<uint64_t>(sm_count());
    const unsigned grid = static_cast<unsigned>(chains < sms ? chains : sms);
    int warps = static_cast<int>((chains / grid) & ~3ull);
    warps = warps < 4 ? 4 : (warps > LT_CHAIN_MAXW ? LT_CHAIN_MAXW : warps);
    lthash_chain_kernel<Items, SMEM_ACC><<<grid, warps * 32, smem, s>>>(items, n, n_sources, acc, counts, dig, status);
    SNT_CUDA(cudaGetLastError());
    ++g_launches;
    return SNT_OK;
}

// Persistent lanes (lthash_lanes.cuh): W warps per CTA, one CTA per SM, every warp a contiguous slice of the items.
template <class Items, bool SMEM_ACC>
int launch_lthash_lanes(const Items& items, uint64_t n, uint32_t n_sources, unsigned long long* acc,
                        unsigned long long* counts, uint8_t* dig, unsigned long long* status, cudaStream_t s) {
    constexpr size_t acc_max = LT_SMEM_SOURCES * (LT_LANES + 1) * sizeof(uint32_t);
    static const cudaError_t attr = cudaFuncSetAttribute(
        lthash_lanes_kernel<Items, SMEM_ACC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
        static_cast<int>(LTL_MAXW * ltl_warp_bytes(Items::TAG_WORDS) + acc_max));
    if (attr != cudaSuccess) return cuda_fail(attr, "cudaFuncSetAttribute(lthash_lanes_kernel)");
    const uint64_t sms = static_cast<uint64_t>(sm_count());
    // at least two items per lane (a lane that holds one sample cannot even out the ragged lengths: 40 k samples
    // 61.7 us at 8 warps, 57.8 at 4), a multiple of four warps per CTA, at most three per scheduler
    int warps = static_cast<int>((n / (sms * 64)) & ~3ull);
    if (const char* force = getenv("SNT_LT_LANES_WARPS")) warps = atoi(force);
    warps = warps < 4 ? 4 : (warps > LTL_MAXW ? LTL_MAXW : warps);
    const uint64_t want_ctas = (n + static_cast<uint64_t>(warps) * 32 - 1) / (static_cast<uint64_t>(warps) * 32);
    const unsigned grid = static_cast<unsigned>(want_ctas < sms ? want_ctas : sms);
    const size_t smem = warps * ltl_warp_bytes(Items::TAG_WORDS) +
                        (SMEM_ACC ? static_cast<size_t>(n_sources) * (LT_LANES + 1) * sizeof(uint32_t) : 0);
    lthash_lanes_kernel<Items, SMEM_ACC><<<grid, warps * 32, smem, s>>>(items, n, n_sources, acc, counts, dig, status);
    SNT_CUDA(cudaGetLastError());
    ++g_launches;
    return SNT_OK;
}

template <class Items>
int launch_lthash(const Items& items, uint64_t n, uint32_t n_sources, uint64_t* d_acc,
                  uint64_t* d_counts, void* d_digests, uint64_t* d_status, cudaStream_t s,
                  uint32_t shape = SNT_SAMPLES_UNKNOWN) {
    if (n == 0) return SNT_OK;
    auto* counts = reinterpret_cast<unsigned long long*>(d_counts);
    auto* acc = reinterpret_cast<unsigned long long*>(d_acc);
    auto* status = reinterpret_cast<unsigned long long*>(d_status);
    auto* dig = static_cast<uint8_t*>(d_digests);
    const bool smem_acc = n_sources <= static_cast<uint32_t>(LT_SMEM_SOURCES);
    // Persistent CTAs with warp-wide chains and a time-sliced tail (lthash_chain_kernel) pay a queue operation
    // and a pipeline restart per slice. That is worth it only for long items in a launch of a wave or two --
    // model blocks (8 KiB = 65 BLAKE2b blocks each), where the plain grid loses a whole warp-time to
    // quantisation: GPT-2 small LATTICE 0.713 -> 0.664 ms. Dataset samples are short (CIFAR 25 blocks,
    // hellaswag ~3): there the plain grid wins (CIFAR 194 vs 210 us, 2 M ragged samples 1.26 vs 2.82 ms;
    // tools/lthash_probe.py, tools/lthash_big_probe.py), so samples always take it.
    const uint64_t chains_per_sm = ((n + 31) >> 5) / static_cast<uint64_t>(sm_count());
    const int schedule = g_schedule.load();           // FUSED forces the chain kernel (tests, A/B timing), GRID the grid
    if (schedule == SNT_SCHEDULE_FUSED || (Items::LONG_ITEMS && chains_per_sm < 32 && schedule != SNT_SCHEDULE_GRID)) {
        if (smem_acc) return launch_lthash_chains<Items, true>(items, n, n_sources, acc, counts, dig, status, s);
        return launch_lthash_chains<Items, false>(items, n, n_sources, acc, counts, dig, status, s);
    }
    // Samples of unknown or ragged length take the persistent lanes (a lane fetches its next sample the moment it
    // finishes one: 2 M hellaswag-shaped samples 2.94 -> 1.09 ms unsorted, 40 k 93 -> 65 us); samples the caller
    // declares to be of ONE length keep the plain grid, which has less bookkeeping per block (CIFAR 194 vs 217 us).
    if constexpr (!Items::LONG_ITEMS) if (schedule == SNT_SCHEDULE_PERSISTENT && n <= quad_max_items())
        return launch_lthash_quad(items, n, n_sources, acc, counts, dig, status, s);     // a loader batch: latency, not throughput
    if constexpr (!Items::LONG_ITEMS) if (schedule == SNT_SCHEDULE_PERSISTENT && shape != SNT_SAMPLES_UNIFORM) {
        if (smem_acc) return launch_lthash_lanes<Items, true>(items, n, n_sources, acc, counts, dig, status, s);
        return launch_lthash_lanes<Items, false>(items, n, n_sources, acc, counts, dig, status, s);
    }
    return launch_lthash_grid(items, n, n_sources, acc, counts, dig, status, s);
}

}  // namespace

extern "C" {

int snt_merkle_leaves(const snt_model_plan* plan, int alg, uint64_t leaf_begin, uint64_t leaf_end,
                      void* d_leaves, snt_stream_t stream) {
    if (!plan || !d_leaves) return SNT_ERR_INVALID_INPUT;
    if (!valid_alg(alg)) return SNT_ERR_CONFIG;
    if (leaf_begin >= leaf_end || leaf_end > plan->n_leaves) return SNT_ERR_INVALID_INPUT;
    return leaf_stage(plan, alg, leaf_begin, leaf_end, static_cast<uint8_t*>(d_leaves), static_cast<cudaStream_t>(stream));
}

int snt_merkle_inplace(const snt_model_plan* plan, int alg, uint64_t leaf_begin, uint64_t leaf_end,
                       uint32_t levels, void* d_leaves, void* d_work, size_t work_bytes, void* d_out,
                       snt_stream_t stream) {
    if (!plan || !d_leaves || !d_out) return SNT_ERR_INVALID_INPUT;
    if (!valid_alg(alg)) return SNT_ERR_CONFIG;
    const uint64_t n = plan->n_leaves;
    if (leaf_begin >= leaf_end || leaf_end > n) return SNT_ERR_INVALID_INPUT;
    if (levels == SNT_LEVELS_TO_ROOT) {
        if (leaf_begin != 0 || leaf_end != n) return SNT_ERR_INVALID_INPUT;
        levels = ceil_log2(n);
    } else {
        if (levels > 63) return SNT_ERR_INVALID_INPUT;
        const uint64_t mask = (1ull << levels) - 1;
        if ((leaf_begin & mask) || ((leaf_end & mask) && leaf_end != n)) return SNT_ERR_INVALID_INPUT;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    uint8_t* leaves = static_cast<uint8_t*>(d_leaves);
    if (d_work && g_schedule.load() == SNT_SCHEDULE_FUSED) {
        const WorkLayout wl = work_layout(alg, leaf_end - leaf_begin);
        if (fused_applies(leaf_end - leaf_begin, levels, work_bytes, wl))
            return fused_dispatch(plan, alg, leaf_begin, leaf_end, levels, leaves, static_cast<uint8_t*>(d_work), wl,
                                  static_cast<uint8_t*>(d_out), s);
    }
    const int rc = leaf_stage(plan, alg, leaf_begin, leaf_end, leaves, s);
    if (rc != SNT_OK) return rc;
    const uint32_t dlen = snt_digest_len(alg);
    if (levels == 0) {
        SNT_CUDA(cudaMemcpyAsync(d_out, leaves, static_cast<size_t>(leaf_end - leaf_begin) * dlen,
                                 cudaMemcpyDefault, s));
        return SNT_OK;
    }
    return reduce_chain(alg, leaves, leaf_begin, leaf_end - leaf_begin, n, levels,
                        static_cast<uint8_t*>(d_work), work_bytes, static_cast<uint8_t*>(d_out),
                        plan->consts, s);
}

int snt_hash_blocks(int alg, const void* d_base, const uint64_t* d_off, const uint64_t* d_len, uint64_t n,
                    void* d_out, snt_stream_t stream) {
    if (!valid_alg(alg)) return SNT_ERR_CONFIG;
    if (n == 0 || !d_off || !d_len || !d_out) return SNT_ERR_INVALID_INPUT;          // merkle.py:100-101
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const uint8_t* base = static_cast<const uint8_t*>(d_base);
    uint8_t* out = static_cast<uint8_t*>(d_out);
    switch (alg) {
        case SNT_SHA256: return launch_blocks<ALG_SHA256>(base, d_off, d_len, n, out, s);
        case SNT_BLAKE2B: return launch_blocks<ALG_BLAKE2B>(base, d_off, d_len, n, out, s);
        default: return launch_blocks<ALG_SHA3_256>(base, d_off, d_len, n, out, s);
    }
}

int snt_merkle_reduce_levels(int alg, const void* d_in, uint64_t first, uint64_t n_in, uint64_t level_count,
                             uint32_t levels, void* d_work, size_t work_bytes, void* d_out,
                             snt_stream_t stream) {
    if (!valid_alg(alg)) return SNT_ERR_CONFIG;
    if (!d_in || !d_out || n_in == 0 || levels == 0 || levels > 63) return SNT_ERR_INVALID_INPUT;
    const uint64_t mask = (1ull << levels) - 1;
    const uint64_t end = first + n_in;
    if ((first & mask) || end > level_count || ((end & mask) && end != level_count))
        return SNT_ERR_INVALID_INPUT;
    return reduce_chain(alg, static_cast<const uint8_t*>(d_in), first, n_in, level_count, levels,
                        static_cast<uint8_t*>(d_work), work_bytes, static_cast<uint8_t*>(d_out),
                        node_consts(), static_cast<cudaStream_t>(stream));
}

int snt_merkle_root(int alg, const void* d_nodes, uint64_t count, void* d_work, size_t work_bytes,
                    void* d_root, snt_stream_t stream) {
    if (!valid_alg(alg)) return SNT_ERR_CONFIG;
    if (count == 0 || !d_nodes || !d_root) return SNT_ERR_INVALID_INPUT;              // merkle.py:156-157
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (count == 1) {                                                                 // merkle.py:159-160
        SNT_CUDA(cudaMemcpyAsync(d_root, d_nodes, snt_digest_len(alg), cudaMemcpyDefault, s));
        return SNT_OK;
    }
    return reduce_chain(alg, static_cast<const uint8_t*>(d_nodes), 0, count, count, ceil_log2(count),
                        static_cast<uint8_t*>(d_work), work_bytes, static_cast<uint8_t*>(d_root),
                        node_consts(), s);
}

int snt_lthash_samples(const void* d_shard, const uint64_t* d_off, const uint64_t* d_len,
                       const uint64_t* d_ids, const uint32_t* d_slot, uint64_t n, uint32_t n_sources,
                       uint64_t* d_acc, uint64_t* d_counts, void* d_digests, uint64_t* d_status,
                       snt_stream_t stream) {
    return snt_lthash_samples_shaped(d_shard, d_off, d_len, d_ids, d_slot, n, n_sources, d_acc, d_counts, d_digests,
                                     d_status, SNT_SAMPLES_UNKNOWN, stream);
}

int snt_lthash_samples_shaped(const void* d_shard, const uint64_t* d_off, const uint64_t* d_len,
                              const uint64_t* d_ids, const uint32_t* d_slot, uint64_t n, uint32_t n_sources,
                              uint64_t* d_acc, uint64_t* d_counts, void* d_digests, uint64_t* d_status,
                              uint32_t shape, snt_stream_t stream) {
    if (shape > SNT_SAMPLES_RAGGED) return SNT_ERR_INVALID_INPUT;
    if (n_sources == 0 || !d_acc || !d_counts) return SNT_ERR_INVALID_INPUT;
    if (n && (!d_off || !d_len || !d_ids || !d_slot)) return SNT_ERR_INVALID_INPUT;
    SampleItems items;
    items.shard = static_cast<const uint8_t*>(d_shard);
    items.off = d_off;
    items.len = d_len;
    items.ids = d_ids;
    items.slot = d_slot;
    return launch_lthash(items, n, n_sources, d_acc, d_counts, d_digests, d_status,
                         static_cast<cudaStream_t>(stream), shape);
}

int snt_lthash_rows(const void* d_rows, uint64_t row_bytes, uint64_t n, const uint64_t* d_ids,
                    const int64_t* d_src_ids, const int64_t* d_table, uint32_t n_sources, uint64_t* d_acc,
                    uint64_t* d_counts, void* d_digests, uint64_t* d_status, snt_stream_t stream) {
    if (n_sources == 0 || !d_acc || !d_counts || !d_table) return SNT_ERR_INVALID_INPUT;
    if (n && (!d_ids || !d_src_ids || (row_bytes && !d_rows))) return SNT_ERR_INVALID_INPUT;
    RowItems items;
    items.rows = static_cast<const uint8_t*>(d_rows);
    items.row_bytes = row_bytes;
    items.ids = d_ids;
    items.src = reinterpret_cast<const long long*>(d_src_ids);
    items.table = reinterpret_cast<const long long*>(d_table);
    items.n_table = n_sources;
    auto* acc = reinterpret_cast<unsigned long long*>(d_acc);
    auto* counts = reinterpret_cast<unsigned long long*>(d_counts);
    auto* status = reinterpret_cast<unsigned long long*>(d_status);
    auto* dig = static_cast<uint8_t*>(d_digests);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (n <= quad_max_items() && g_schedule.load() == SNT_SCHEDULE_PERSISTENT)
        return launch_lthash_quad(items, n, n_sources, acc, counts, dig, status, s);
    return launch_lthash_grid(items, n, n_sources, acc, counts, dig, status, s);
}

int snt_lthash_model(const snt_model_plan* plan, uint64_t leaf_begin, uint64_t leaf_end, uint64_t* d_acc,
                     uint64_t* d_counts, void* d_digests, snt_stream_t stream) {
    if (!plan || !d_acc || !d_counts) return SNT_ERR_INVALID_INPUT;
    if (leaf_begin > leaf_end || leaf_end > plan->n_leaves) return SNT_ERR_INVALID_INPUT;
    LeafItems items;
    items.tab = plan->table();
    items.leaf_begin = leaf_begin;
    return launch_lthash(items, leaf_end - leaf_begin, 1, d_acc, d_counts, d_digests, nullptr,
                         static_cast<cudaStream_t>(stream));
}

int snt_lthash_model_layers(const snt_model_plan* plan, uint64_t leaf_begin, uint64_t leaf_end, uint64_t* d_acc,
                            uint64_t* d_counts, void* d_digests, snt_stream_t stream) {
    if (!plan || !d_acc || !d_counts) return SNT_ERR_INVALID_INPUT;
    if (leaf_begin > leaf_end || leaf_end > plan->n_leaves) return SNT_ERR_INVALID_INPUT;
    LayerLeafItems items;
    items.tab = plan->table();
    items.leaf_begin = leaf_begin;
    return launch_lthash(items, leaf_end - leaf_begin, plan->n_tensors, d_acc, d_counts, d_digests, nullptr,
                         static_cast<cudaStream_t>(stream));
}

int snt_merkle_roots_segmented(int alg, const void* d_digests, const uint64_t* seg_first, uint32_t n_segments,
                               const void* d_empty_digest, void* d_work, size_t work_bytes, void* d_out,
                               snt_stream_t stream) {
    if (!valid_alg(alg)) return SNT_ERR_CONFIG;
    if (!d_digests || !seg_first || !d_out || n_segments == 0) return SNT_ERR_INVALID_INPUT;
    const uint32_t dlen = snt_digest_len(alg);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const uint8_t* in = static_cast<const uint8_t*>(d_digests);
    uint8_t* out = static_cast<uint8_t*>(d_out);
    // Segments that fit one CTA (<= 2^max_levels digests) are finished by ONE launch, one CTA each. Larger ones (up
    // to 2^(2 * max_levels) digests, as far as the workspace goes) first lose their bottom max_levels levels in ONE
    // launch over all their groups (merkle_reduce_groups_kernel, nodes into the workspace) and then join that same
    // launch. Anything larger goes through the ordinary reducer chain, one tree after the other.
    const uint32_t cap = max_levels(alg);
    const uint64_t cta_cap = 1ull << cap;
    const uint64_t work_nodes = d_work ? work_bytes / dlen : 0;
    std::vector<uint64_t> seg_rows;        // [address, count] per segment of the final launch
    std::vector<uint32_t> seg_out;
    std::vector<uint64_t> grp_rows;        // [address, count, group] per group of the first launch
    std::vector<uint32_t> grp_out;
    std::vector<uint32_t> chained;         // segments left to the reducer chain
    uint64_t inter = 0;                    // workspace nodes handed out so far
    const uint64_t in_addr = reinterpret_cast<uint64_t>(in), work_addr = reinterpret_cast<uint64_t>(d_work);
    for (uint32_t t = 0; t < n_segments; ++t) {
        if (seg_first[t + 1] < seg_first[t]) return SNT_ERR_INVALID_INPUT;
        const uint64_t count = seg_first[t + 1] - seg_first[t];
        if (count == 0 && !d_empty_digest) return SNT_ERR_INVALID_INPUT;
        const uint64_t addr = in_addr + seg_first[t] * dlen;
        if (count <= cta_cap) {
            seg_rows.push_back(addr);
            seg_rows.push_back(count);
            seg_out.push_back(t);
            continue;
        }
        const uint64_t groups = (count + cta_cap - 1) >> cap;
        if (groups > cta_cap || inter + groups > work_nodes || grp_out.size() + groups > 0x7fffffffull) {
            chained.push_back(t);
            continue;
        }
        for (uint64_t g = 0; g < groups; ++g) {
            grp_rows.push_back(addr);
            grp_rows.push_back(count);
            grp_rows.push_back(g);
            grp_out.push_back(static_cast<uint32_t>(inter + g));
        }
        seg_rows.push_back(work_addr + inter * dlen);
        seg_rows.push_back(groups);
        seg_out.push_back(t);
        inter += groups;
    }
    // the reducer chain uses the workspace too: those trees go first, before the group nodes are written into it
    for (uint32_t t : chained) {
        const int rc = snt_merkle_root(alg, in + seg_first[t] * dlen, seg_first[t + 1] - seg_first[t], d_work, work_bytes,
                                       out + static_cast<size_t>(t) * dlen, stream);
        if (rc != SNT_OK) return rc;
    }
    // both tables in one upload: [group rows | segment rows | group outputs | segment outputs]
    const size_t n_grp = grp_out.size(), n_seg = seg_out.size();
    if (n_seg) {
        std::vector<uint64_t> table(grp_rows);
        table.insert(table.end(), seg_rows.begin(), seg_rows.end());
        const size_t rows_words = table.size();
        table.resize(rows_words + (n_grp + n_seg + 1) / 2);
        uint32_t* idx = reinterpret_cast<uint32_t*>(table.data() + rows_words);
        memcpy(idx, grp_out.data(), n_grp * sizeof(uint32_t));
        memcpy(idx + n_grp, seg_out.data(), n_seg * sizeof(uint32_t));
        uint64_t* d_table = nullptr;
        SNT_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_table), table.size() * sizeof(uint64_t), s));
        // pageable source: the call returns once the bytes sit in the driver's staging buffer
        cudaError_t e = cudaMemcpyAsync(d_table, table.data(), table.size() * sizeof(uint64_t), cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess) {
            const uint64_t* d_grp = d_table;
            const uint64_t* d_seg = d_table + grp_rows.size();
            const uint32_t* d_grp_out = reinterpret_cast<const uint32_t*>(d_table + rows_words);
            const uint32_t* d_seg_out = d_grp_out + n_grp;
            const uint8_t* empty = static_cast<const uint8_t*>(d_empty_digest);
            uint8_t* work = static_cast<uint8_t*>(d_work);
            const MerkleConsts& c = node_consts();
            const unsigned g_grid = static_cast<unsigned>(n_grp), s_grid = static_cast<unsigned>(n_seg);
            switch (alg) {
                case SNT_SHA256:
                    if (n_grp) merkle_reduce_groups_kernel<ALG_SHA256, 256><<<g_grid, 256, 0, s>>>(d_grp, d_grp_out, c, work);
                    merkle_reduce_segments_kernel<ALG_SHA256, 256><<<s_grid, 256, 0, s>>>(d_seg, d_seg_out, empty, c, out);
                    break;
                case SNT_BLAKE2B:
                    if (n_grp) merkle_reduce_groups_kernel<ALG_BLAKE2B, 256><<<g_grid, 256, 0, s>>>(d_grp, d_grp_out, c, work);
                    merkle_reduce_segments_kernel<ALG_BLAKE2B, 256><<<s_grid, 256, 0, s>>>(d_seg, d_seg_out, empty, c, out);
                    break;
                default:
                    if (n_grp) merkle_reduce_groups_kernel<ALG_SHA3_256, 256><<<g_grid, 256, 0, s>>>(d_grp, d_grp_out, c, work);
                    merkle_reduce_segments_kernel<ALG_SHA3_256, 256><<<s_grid, 256, 0, s>>>(d_seg, d_seg_out, empty, c, out);
            }
            e = cudaGetLastError();
            g_launches += n_grp ? 2 : 1;
        }
        cudaFreeAsync(d_table, s);
        if (e != cudaSuccess) return cuda_fail(e, "snt_merkle_roots_segmented");
    }
    return SNT_OK;
}

int snt_memcpy_h2d_batch(void* const* d_dst, const void* const* h_src, const uint64_t* nbytes, uint32_t n,
                         snt_stream_t stream) {
    if (n && (!d_dst || !h_src || !nbytes)) return SNT_ERR_INVALID_INPUT;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    for (uint32_t i = 0; i < n; ++i) {
        if (!nbytes[i]) continue;
        if (!d_dst[i] || !h_src[i]) return SNT_ERR_INVALID_INPUT;
        SNT_CUDA(cudaMemcpyAsync(d_dst[i], h_src[i], nbytes[i], cudaMemcpyHostToDevice, s));
    }
    return SNT_OK;
}

uint32_t snt_gather_chunk_bytes(void) { return GATHER_CHUNK_BYTES; }

int snt_device_reads_pinned_host(void) {
    static const int ok = [] {
        int dev = 0, unified = 0, same_ptr = 0;
        if (cudaGetDevice(&dev) != cudaSuccess) return 0;
        if (cudaDeviceGetAttribute(&unified, cudaDevAttrUnifiedAddressing, dev) != cudaSuccess) return 0;
        if (cudaDeviceGetAttribute(&same_ptr, cudaDevAttrCanUseHostPointerForRegisteredMem, dev) != cudaSuccess) return 0;
        return (unified && same_ptr) ? 1 : 0;
    }();
    return ok;
}

int snt_gather_spans(const uint64_t* d_src_addr, const uint64_t* d_len, const uint64_t* d_dst_off,
                     const uint64_t* d_chunk_first, uint32_t n_spans, uint64_t n_chunks,
                     uint32_t pad_block, void* d_dst, snt_stream_t stream) {
    if (n_spans == 0 || n_chunks == 0) return SNT_OK;
    if (!d_src_addr || !d_len || !d_dst_off || !d_chunk_first || !d_dst) return SNT_ERR_INVALID_INPUT;
    if (n_chunks > 0x7fffffffull) return SNT_ERR_INVALID_INPUT;
    gather_spans_kernel<<<static_cast<unsigned>(n_chunks), GATHER_THREADS, 0, static_cast<cudaStream_t>(stream)>>>(
        d_src_addr, d_len, d_dst_off, d_chunk_first, n_spans, pad_block, static_cast<uint8_t*>(d_dst));
    SNT_CUDA(cudaGetLastError());
    ++g_launches;
    return SNT_OK;
}

int snt_lt_reduce(const void* d_digests, uint64_t n, uint64_t* d_acc, snt_stream_t stream) {
    if (!d_acc || (n && !d_digests)) return SNT_ERR_INVALID_INPUT;
    if (n == 0) return SNT_OK;                                                        // lattice.py:112-113
    uint64_t grid = (n + 63) / 64;
    if (grid > 148 * 8) grid = 148 * 8;
    lt_reduce_kernel<<<static_cast<unsigned>(grid), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint8_t*>(d_digests), n, reinterpret_cast<unsigned long long*>(d_acc));
    SNT_CUDA(cudaGetLastError());
    ++g_launches;
    return SNT_OK;
}

int snt_lt_finalize(const uint64_t* d_acc, uint32_t n_sources, void* d_out, snt_stream_t stream) {
    if (!d_acc || !d_out || n_sources == 0) return SNT_ERR_INVALID_INPUT;
    const uint32_t n_words = n_sources * (LT_LANES / 2);
    lt_finalize_kernel<<<(n_words + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<const unsigned long long*>(d_acc), n_words, static_cast<uint32_t*>(d_out));
    SNT_CUDA(cudaGetLastError());
    ++g_launches;
    return SNT_OK;
}

}  // extern "C"
