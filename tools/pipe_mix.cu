// ALU-pipe / FMA-pipe co-issue curve on sm_100a.
//
// tools/intpeak shows LOP3 and IMAD each at 18.5 Tops/s and a 1:1 mix at 36 Tops/s, but the SHA-256
// leaf kernel loses ALU throughput as soon as more of its additions are moved to IMAD
// (profiles/r1_sha256_variants*). This program measures how the ALU-pipe rate behaves as a function of
// the ALU:FMA instruction ratio and of the number of resident warps, with the instruction stream of each
// warp a fixed repeating pattern of A (ALU: SHF with one register operand, or LOP3 with three) and
// F (IMAD, three registers) slots over independent dependency chains.
//
// Output: one JSON object per (pattern, warps/SM) with the achieved ALU-pipe and FMA-pipe Tops/s.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CHECK(x)                                                                      \
    do {                                                                              \
        cudaError_t e = (x);                                                          \
        if (e != cudaSuccess) {                                                       \
            fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));                   \
            exit(1);                                                                  \
        }                                                                             \
    } while (0)

constexpr int CHAINS = 8;

// One pattern period = NA ALU slots followed/interleaved by NF FMA slots. Slot k of the period is an
// FMA slot when (k * NF) / (NA + NF) changes, i.e. the F slots are spread evenly through the period.
// ALU slots alternate SHF (1 register) and LOP3 (3 registers) in the ratio the SHA-256 round has (2:1).
// FORM selects the F-slot instruction: 0 = IMAD with three per-chain registers, 1 = multiplier is one
// shared vector register (the "runtime 1" of Sha256::add_fma), 2 = shared multiplier + immediate addend,
// 3 = multiplier in a uniform register (kernel parameter).
template <int NA, int NF, int REPS, int THREADS, int FORM>
__global__ void __launch_bounds__(THREADS) mix_kernel(uint32_t* out, int iters, uint32_t seed, uint32_t uone) {
    uint32_t x[CHAINS], yy[CHAINS], zz[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
        x[c] = seed + c * 0x9e3779b9u + threadIdx.x;
        yy[c] = (seed ^ threadIdx.x) * (2 * c + 3);
        zz[c] = (seed * 2654435761u + blockIdx.x + c) ^ (threadIdx.x * 40503u);
    }
    constexpr int P = NA + NF;
    const uint32_t vone = uone + (threadIdx.x >> 20);      // a per-thread (vector) register holding 1
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < REPS; ++r) {
#pragma unroll
            for (int k = 0; k < P; ++k) {
                const int c = (r * P + k) % CHAINS;
                const bool fslot = ((k + 1) * NF) / P != (k * NF) / P;
                if (fslot) {
                    if (FORM == 0) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(yy[c]), "r"(zz[c]));
                    else if (FORM == 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(vone), "r"(zz[c]));
                    else if (FORM == 2) asm volatile("mad.lo.u32 %0, %0, %1, 0x5be0cd19;" : "+r"(x[c]) : "r"(vone));
                    else asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(uone), "r"(zz[c]));
                } else if ((k % 3) == 2) {
                    asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(yy[c]), "r"(zz[c]));
                } else {
                    asm volatile("shf.r.wrap.b32 %0, %0, %0, 7;" : "+r"(x[c]));
                }
            }
        }
    }
    uint32_t r = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) r ^= x[c] ^ yy[c] ^ zz[c];
    if (r == 0x12345678u) out[blockIdx.x * THREADS + threadIdx.x] = r;
}

// Register-operand experiment: A slots are ALU instructions reading AR vector registers (1: SHF x,x;
// 2: LOP3 x,y,RZ; 3: LOP3 x,y,z), F slots are IMADs reading FR vector registers (1: x*imm+imm;
// 2: x*y+imm; 3: x*y+z), strictly alternating A F A F over 8 independent chains; every operand is a true
// per-thread register (nothing the compiler can move to the uniform datapath).
template <int AR, int FR, int THREADS>
__global__ void __launch_bounds__(THREADS) regs_kernel(uint32_t* out, int iters, uint32_t seed) {
    uint32_t x[CHAINS], yy[CHAINS], zz[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
        x[c] = seed + c * 0x9e3779b9u + threadIdx.x;
        yy[c] = ((seed ^ threadIdx.x) * (2 * c + 3)) | 1u;
        zz[c] = (seed * 2654435761u + blockIdx.x + c) ^ (threadIdx.x * 40503u);
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 64; ++r) {
            const int ca = (2 * r) % CHAINS, cf = (2 * r + 1) % CHAINS;
            if (AR == 1) asm volatile("shf.r.wrap.b32 %0, %0, %0, 7;" : "+r"(x[ca]));
            else if (AR == 2) asm volatile("lop3.b32 %0, %0, %1, 0, 0x96;" : "+r"(x[ca]) : "r"(yy[ca]));
            else if (AR == 3) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[ca]) : "r"(yy[ca]), "r"(zz[ca]));
            if (FR == 1) asm volatile("mad.lo.u32 %0, %0, 0x01000193, 0x5be0cd19;" : "+r"(x[cf]));
            else if (FR == 2) asm volatile("mad.lo.u32 %0, %0, %1, 0x5be0cd19;" : "+r"(x[cf]) : "r"(yy[cf]));
            else if (FR == 3) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[cf]) : "r"(yy[cf]), "r"(zz[cf]));
        }
    }
    uint32_t r = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) r ^= x[c] ^ yy[c] ^ zz[c];
    if (r == 0x12345678u) out[blockIdx.x * THREADS + threadIdx.x] = r;
}

// Does a warp instruction cost less when only half of the warp's lanes are active? `active` lanes per
// warp run a pure ALU (SHF) loop; the rest exit at once. Rate is reported per *warp instruction*.
template <int THREADS>
__global__ void __launch_bounds__(THREADS) lanes_kernel(uint32_t* out, int iters, uint32_t seed, int active) {
    if (static_cast<int>(threadIdx.x & 31) >= active) return;
    uint32_t x[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = seed + c * 0x9e3779b9u + threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 64; ++r) asm volatile("shf.r.wrap.b32 %0, %0, %0, 7;" : "+r"(x[r % CHAINS]));
    }
    uint32_t r = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) r ^= x[c];
    if (r == 0x12345678u) out[blockIdx.x * THREADS + threadIdx.x] = r;
}

static uint32_t* g_out;

static void run_lanes(int sms, int warps_per_sm, int active) {
    constexpr int THREADS = 128;
    const int grid = sms * (warps_per_sm / 4);
    const int iters = 400;
    cudaEvent_t a, b;
    CHECK(cudaEventCreate(&a));
    CHECK(cudaEventCreate(&b));
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        CHECK(cudaEventRecord(a));
        lanes_kernel<THREADS><<<grid, THREADS>>>(g_out, iters, 12345u, active);
        CHECK(cudaEventRecord(b));
        CHECK(cudaEventSynchronize(b));
        float ms;
        CHECK(cudaEventElapsedTime(&ms, a, b));
        if (r > 0 && ms < best) best = ms;
    }
    CHECK(cudaGetLastError());
    const double warp_instr = double(grid) * (THREADS / 32) * double(iters) * 64;
    printf("{\"active_lanes\": %d, \"warps_per_sm\": %d, \"warp_instr_per_clk_per_smsp\": %.4f}\n", active, warps_per_sm,
           warp_instr / (best * 1e-3) / (sms * 4.0) / 1.965e9);
}

template <int AR, int FR>
static void run_regs(int sms, int warps_per_sm) {
    constexpr int THREADS = 128;
    const int grid = sms * (warps_per_sm / 4);
    const int iters = 400;
    cudaEvent_t a, b;
    CHECK(cudaEventCreate(&a));
    CHECK(cudaEventCreate(&b));
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        CHECK(cudaEventRecord(a));
        regs_kernel<AR, FR, THREADS><<<grid, THREADS>>>(g_out, iters, 12345u);
        CHECK(cudaEventRecord(b));
        CHECK(cudaEventSynchronize(b));
        float ms;
        CHECK(cudaEventElapsedTime(&ms, a, b));
        if (r > 0 && ms < best) best = ms;
    }
    CHECK(cudaGetLastError());
    const double slots = double(grid) * THREADS * double(iters) * 64;
    const int n = (AR > 0) + (FR > 0);
    printf("{\"alu_regs\": %d, \"fma_regs\": %d, \"warps_per_sm\": %d, \"total_tops\": %.3f}\n", AR, FR, warps_per_sm,
           slots * n / (best * 1e-3) / 1e12);
}

template <int NA, int NF, int REPS, int FORM = 0>
static void run(int sms, int warps_per_sm) {
    constexpr int THREADS = 128;
    const int grid = sms * (warps_per_sm / 4);
    const int iters = 400;
    cudaEvent_t a, b;
    CHECK(cudaEventCreate(&a));
    CHECK(cudaEventCreate(&b));
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        CHECK(cudaEventRecord(a));
        mix_kernel<NA, NF, REPS, THREADS, FORM><<<grid, THREADS>>>(g_out, iters, 12345u, 1u);
        CHECK(cudaEventRecord(b));
        CHECK(cudaEventSynchronize(b));
        float ms;
        CHECK(cudaEventElapsedTime(&ms, a, b));
        if (r > 0 && ms < best) best = ms;
    }
    CHECK(cudaGetLastError());
    const double slots = double(grid) * THREADS * double(iters) * REPS;
    printf("{\"form\": %d, \"na\": %d, \"nf\": %d, \"warps_per_sm\": %d, \"alu_tops\": %.3f, \"fma_tops\": %.3f, \"total_tops\": %.3f}\n",
           FORM, NA, NF, warps_per_sm, slots * NA / (best * 1e-3) / 1e12, slots * NF / (best * 1e-3) / 1e12,
           slots * (NA + NF) / (best * 1e-3) / 1e12);
}

int main() {
    cudaDeviceProp prop;
    CHECK(cudaGetDeviceProperties(&prop, 0));
    const int sms = prop.multiProcessorCount;
    CHECK(cudaMalloc(&g_out, sizeof(uint32_t) * sms * 32 * 128));
    for (int act : {32, 24, 16, 8}) run_lanes(sms, 32, act);
    for (int w : {32, 64}) {
        run_regs<1, 0>(sms, w); run_regs<2, 0>(sms, w); run_regs<3, 0>(sms, w);
        run_regs<0, 1>(sms, w); run_regs<0, 2>(sms, w); run_regs<0, 3>(sms, w);
        run_regs<1, 1>(sms, w); run_regs<1, 2>(sms, w); run_regs<1, 3>(sms, w);
        run_regs<2, 1>(sms, w); run_regs<2, 2>(sms, w); run_regs<2, 3>(sms, w);
        run_regs<3, 1>(sms, w); run_regs<3, 2>(sms, w); run_regs<3, 3>(sms, w);
    }
    for (int w : {16, 32, 64}) {
        run<12, 0, 8>(sms, w);
        run<12, 1, 8>(sms, w);
        run<8, 1, 10>(sms, w);
        run<6, 1, 12>(sms, w);
        run<5, 1, 16>(sms, w);
        run<4, 1, 16>(sms, w);
        run<3, 1, 24>(sms, w);
        run<5, 2, 12>(sms, w);
        run<2, 1, 32>(sms, w);
        run<5, 3, 12>(sms, w);
        run<3, 2, 16>(sms, w);
        run<4, 3, 12>(sms, w);
        run<1, 1, 48>(sms, w);
        run<3, 4, 12>(sms, w);
        run<1, 2, 32>(sms, w);
    }
    for (int w : {32}) {
        run<3, 1, 24, 1>(sms, w); run<2, 1, 32, 1>(sms, w); run<3, 2, 16, 1>(sms, w); run<1, 1, 48, 1>(sms, w);
        run<3, 1, 24, 2>(sms, w); run<2, 1, 32, 2>(sms, w); run<3, 2, 16, 2>(sms, w); run<1, 1, 48, 2>(sms, w);
        run<3, 1, 24, 3>(sms, w); run<2, 1, 32, 3>(sms, w); run<3, 2, 16, 3>(sms, w); run<1, 1, 48, 3>(sms, w);
    }
    return 0;
}
