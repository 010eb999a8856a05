// Scheduling experiment for the SHA-256 leaf stage: one persistent CTA per SM whose warps share the
// SM's leaf-warps ("chains" of 32 consecutive 8 KiB leaves) by software time slicing.
//
// Why: a leaf is a serial Merkle-Damgard chain, so the unit of work is one warp x 129 compressions.
// With the plain grid (one thread per leaf, 128-thread CTAs) the SM sub-partitions end up with an
// integer number of warps each -- GPT-2 small: 2,490 warps on 592 schedulers = 4.2 -> the kernel
// takes 5 warp-times. Here every SM gets a contiguous run of chains (balanced to +-1); W worker
// warps (W/4 per scheduler) run them, and the last W + (count mod W) chains of an SM are executed in
// slices of nblk/W blocks through a FIFO, the chain state (8 words per lane) parked in global
// memory between slices. Every scheduler then always has W/4 runnable warps until the very end:
// makespan = count/4 warp-times instead of ceil(count/4).
//
// Prints one JSON line per variant; digests are checked against the plain kernel.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_2510_00554_b200/csrc/sha256.cuh"

using namespace snt;

#define CHECK(x)                                                                      \
    do {                                                                              \
        cudaError_t e = (x);                                                          \
        if (e != cudaSuccess) {                                                       \
            fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));                   \
            exit(1);                                                                  \
        }                                                                             \
    } while (0)

struct Params {
    uint32_t pad_kw[64];
    uint32_t one;
};

__constant__ uint32_t k_ones[32] = {1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1};

__device__ __forceinline__ void to_words(const U4& q0, const U4& q1, const U4& q2, const U4& q3, uint32_t w[16]) {
    w[0] = bswap32(q0.x);  w[1] = bswap32(q0.y);  w[2] = bswap32(q0.z);  w[3] = bswap32(q0.w);
    w[4] = bswap32(q1.x);  w[5] = bswap32(q1.y);  w[6] = bswap32(q1.z);  w[7] = bswap32(q1.w);
    w[8] = bswap32(q2.x);  w[9] = bswap32(q2.y);  w[10] = bswap32(q2.z); w[11] = bswap32(q2.w);
    w[12] = bswap32(q3.x); w[13] = bswap32(q3.y); w[14] = bswap32(q3.z); w[15] = bswap32(q3.w);
}

// blocks [b0, b1) of the leaf at p
__device__ __forceinline__ void run_blocks(const uint8_t* p, uint32_t b0, uint32_t b1, uint32_t s[8], const Sha256::One& one) {
    const uint8_t* q = p + (static_cast<size_t>(b0) << 6);
    U4 q0 = ld128(q), q1 = ld128(q + 16), q2 = ld128(q + 32), q3 = ld128(q + 48);
#pragma unroll 1
    for (uint32_t b = b0; b < b1; ++b) {
        uint32_t w[16];
        to_words(q0, q1, q2, q3, w);
        if (b + 1 < b1) {
            const uint8_t* n = p + (static_cast<size_t>(b + 1) << 6);
            q0 = ld128(n); q1 = ld128(n + 16); q2 = ld128(n + 32); q3 = ld128(n + 48);
        }
        Sha256::compress(s, w, one);
    }
}

// ---- baseline: the product's grid (one thread per leaf, 128 threads per CTA) ---------------
__global__ void __launch_bounds__(128, 1)
plain_kernel(const uint8_t* __restrict__ data, uint64_t n_leaves, const __grid_constant__ Params prm,
             uint8_t* __restrict__ out) {
    const uint64_t k = static_cast<uint64_t>(blockIdx.x) * 128 + threadIdx.x;
    if (k >= n_leaves) return;
    const Sha256::One one(prm.one, k_ones[threadIdx.x & 31]);
    uint32_t s[8];
    Sha256::init(s);
    run_blocks(data + (k << 13), 0, 128, s, one);
    Sha256::compress_const(s, prm.pad_kw, one);
    uint4* o = reinterpret_cast<uint4*>(out + k * 32);
    o[0] = make_uint4(bswap32(s[0]), bswap32(s[1]), bswap32(s[2]), bswap32(s[3]));
    o[1] = make_uint4(bswap32(s[4]), bswap32(s[5]), bswap32(s[6]), bswap32(s[7]));
}

// ---- persistent, time-sliced --------------------------------------------------------------
constexpr int RING = 32;          // >= 2 * max workers - 1 parked chains
constexpr uint32_t NBLK = 128;

struct Sched {
    int lock;
    int fresh;                // next chain of this CTA that has not been started
    int head, tail;           // FIFO of parked chains (ring indices)
    int ring[RING];
    int prog[RING];           // blocks done, per slot of the time-sliced group
};

__device__ __forceinline__ void sched_lock(Sched* sc) {
    while (atomicCAS(&sc->lock, 0, 1) != 0) {}
    __threadfence_block();
}
__device__ __forceinline__ void sched_unlock(Sched* sc) {
    __threadfence_block();
    atomicExch(&sc->lock, 0);
}

template <int MAXW, int MAXREG>
__global__ void __launch_bounds__(MAXW * 32, 1) __maxnreg__(MAXREG)
persist_kernel(const uint8_t* __restrict__ data, uint64_t n_leaves, const __grid_constant__ Params prm,
               uint8_t* __restrict__ out, uint32_t* __restrict__ park, int slicing) {
    __shared__ Sched sc;
    const int lane = threadIdx.x & 31;
    const int W = blockDim.x >> 5;
    const uint64_t R = (n_leaves + 31) >> 5;                      // chains in total
    const uint64_t q = R / gridDim.x, rem = R % gridDim.x;
    const uint64_t first = blockIdx.x * q + (blockIdx.x < rem ? blockIdx.x : rem);
    const int count = static_cast<int>(q + (blockIdx.x < rem ? 1 : 0));
    // the last W + (count mod W) chains are time-sliced (none when count <= W or W divides count)
    int first_sliced = count;
    if (slicing && count > W && (count % W) != 0) first_sliced = count - (W + count % W);
    const uint32_t Q = (NBLK + W - 1) / W;
    if (threadIdx.x == 0) {
        sc.lock = 0; sc.fresh = 0; sc.head = 0; sc.tail = 0;
    }
    if (threadIdx.x < RING) sc.prog[threadIdx.x] = 0;
    __syncthreads();
    const Sha256::One one(prm.one, k_ones[lane]);
    uint32_t* my_park = park + static_cast<size_t>(blockIdx.x) * RING * 8 * 32;

    for (;;) {
        int c = -1;
        if (lane == 0) {
            sched_lock(&sc);
            if (sc.fresh < count) c = sc.fresh++;
            else if (sc.head != sc.tail) c = sc.ring[(sc.head++) & (RING - 1)];
            sched_unlock(&sc);
        }
        c = __shfl_sync(0xffffffffu, c, 0);
        if (c < 0) break;
        const bool sliced = c >= first_sliced;
        const int slot = c - first_sliced;
        const uint64_t k = ((first + c) << 5) + lane;
        const bool valid = k < n_leaves;
        const uint8_t* p = data + (k << 13);
        uint32_t b0 = sliced ? static_cast<uint32_t>(*reinterpret_cast<volatile int*>(&sc.prog[slot & (RING - 1)])) : 0u;
        uint32_t s[8];
        uint32_t* st = my_park + static_cast<size_t>(slot & (RING - 1)) * 8 * 32 + lane;
        if (b0 == 0) {
            Sha256::init(s);
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) s[i] = __ldcg(st + i * 32);
        }
        for (;;) {
            uint32_t b1 = sliced ? (b0 + Q < NBLK ? b0 + Q : NBLK) : NBLK;
            if (valid) run_blocks(p, b0, b1, s, one);
            __syncwarp();
            if (b1 == NBLK) break;
            b0 = b1;
            // somebody waiting? if not, keep going with this chain
            int waiting = 0;
            if (lane == 0) waiting = (*reinterpret_cast<volatile int*>(&sc.fresh) < count) ||
                                     (*reinterpret_cast<volatile int*>(&sc.head) != *reinterpret_cast<volatile int*>(&sc.tail));
            waiting = __shfl_sync(0xffffffffu, waiting, 0);
            if (!waiting) continue;
#pragma unroll
            for (int i = 0; i < 8; ++i) __stcg(st + i * 32, s[i]);
            __threadfence_block();
            __syncwarp();
            if (lane == 0) {
                sched_lock(&sc);
                sc.prog[slot & (RING - 1)] = static_cast<int>(b0);
                sc.ring[(sc.tail++) & (RING - 1)] = c;
                sched_unlock(&sc);
            }
            b0 = NBLK + 1;     // parked
            break;
        }
        if (b0 == NBLK + 1) continue;
        if (valid) {
            Sha256::compress_const(s, prm.pad_kw, one);
            uint4* o = reinterpret_cast<uint4*>(out + k * 32);
            o[0] = make_uint4(bswap32(s[0]), bswap32(s[1]), bswap32(s[2]), bswap32(s[3]));
            o[1] = make_uint4(bswap32(s[4]), bswap32(s[5]), bswap32(s[6]), bswap32(s[7]));
        }
    }
}

static uint8_t* g_data;
static uint8_t* g_out;
static uint8_t* g_ref;
static uint32_t* g_park;
static uint64_t g_leaves;
static Params g_prm;
static std::vector<uint8_t> h_ref, h_out;
static int g_sms;

template <class F>
static void bench(const char* name, int warps, int regs, int slicing, F launch) {
    CHECK(cudaMemset(g_out, 0, g_leaves * 32));
    launch(g_out);
    CHECK(cudaDeviceSynchronize());
    CHECK(cudaMemcpy(h_out.data(), g_out, g_leaves * 32, cudaMemcpyDeviceToHost));
    const int ok = memcmp(h_out.data(), h_ref.data(), g_leaves * 32) == 0;
    cudaEvent_t e0, e1;
    CHECK(cudaEventCreate(&e0));
    CHECK(cudaEventCreate(&e1));
    float best = 1e30f, sum = 0;
    const int reps = 7;
    for (int r = 0; r < reps; ++r) {
        CHECK(cudaEventRecord(e0));
        launch(g_out);
        CHECK(cudaEventRecord(e1));
        CHECK(cudaEventSynchronize(e1));
        float ms;
        CHECK(cudaEventElapsedTime(&ms, e0, e1));
        best = ms < best ? ms : best;
        sum += ms;
    }
    CHECK(cudaGetLastError());
    const double bytes = double(g_leaves) * 8192;
    printf("{\"leaves\": %llu, \"variant\": \"%s\", \"warps\": %d, \"regs\": %d, \"slicing\": %d, \"ok\": %d, "
           "\"best_ms\": %.4f, \"avg_ms\": %.4f, \"gbs_best\": %.1f}\n",
           (unsigned long long)g_leaves, name, warps, regs, slicing, ok, best, sum / reps, bytes / (best * 1e-3) / 1e9);
    fflush(stdout);
}

template <int MAXW, int MAXREG>
static void run_persist(int warps, int slicing) {
    cudaFuncAttributes attr;
    CHECK(cudaFuncGetAttributes(&attr, persist_kernel<MAXW, MAXREG>));
    // > half of the shared memory: one CTA per SM
    CHECK(cudaFuncSetAttribute(persist_kernel<MAXW, MAXREG>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024));
    char name[64];
    snprintf(name, sizeof(name), "persist<%d,%d>", MAXW, MAXREG);
    bench(name, warps, attr.numRegs, slicing, [&](uint8_t* out) {
        persist_kernel<MAXW, MAXREG><<<g_sms, warps * 32, 120 * 1024>>>(g_data, g_leaves, g_prm, out, g_park, slicing);
    });
}

int main(int argc, char** argv) {
    g_leaves = argc > 1 ? strtoull(argv[1], nullptr, 10) : 79672ull;
    cudaDeviceProp prop;
    CHECK(cudaGetDeviceProperties(&prop, 0));
    g_sms = prop.multiProcessorCount;
    CHECK(cudaMalloc(&g_data, g_leaves * 8192));
    CHECK(cudaMalloc(&g_out, g_leaves * 32));
    CHECK(cudaMalloc(&g_ref, g_leaves * 32));
    CHECK(cudaMalloc(&g_park, static_cast<size_t>(g_sms) * RING * 8 * 32 * 4));
    h_ref.resize(g_leaves * 32);
    h_out.resize(g_leaves * 32);
    {
        std::vector<uint32_t> buf(16u << 20);
        uint32_t x = 12345;
        for (uint64_t off = 0; off < g_leaves * 8192; off += buf.size() * 4) {
            for (auto& v : buf) { x = x * 1664525u + 1013904223u; v = x; }
            uint64_t n = g_leaves * 8192 - off;
            if (n > buf.size() * 4) n = buf.size() * 4;
            CHECK(cudaMemcpy(g_data + off, buf.data(), n, cudaMemcpyHostToDevice));
        }
    }
    Sha256::pad_schedule(8192, g_prm.pad_kw);
    g_prm.one = 1;

    const unsigned grid = static_cast<unsigned>((g_leaves + 127) / 128);
    plain_kernel<<<grid, 128>>>(g_data, g_leaves, g_prm, g_ref);
    CHECK(cudaDeviceSynchronize());
    CHECK(cudaMemcpy(h_ref.data(), g_ref, g_leaves * 32, cudaMemcpyDeviceToHost));
    {
        cudaFuncAttributes attr;
        CHECK(cudaFuncGetAttributes(&attr, plain_kernel));
        bench("plain", 4, attr.numRegs, 0, [&](uint8_t* out) { plain_kernel<<<grid, 128>>>(g_data, g_leaves, g_prm, out); });
    }
    for (int slicing : {0, 1}) {
        for (int w : {8, 12, 16}) {
            run_persist<16, 128>(w, slicing);
            run_persist<16, 80>(w, slicing);
            run_persist<16, 72>(w, slicing);
            run_persist<16, 64>(w, slicing);
        }
        run_persist<20, 96>(20, slicing);
        run_persist<24, 80>(24, slicing);
    }
    return 0;
}
