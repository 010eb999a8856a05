// Integer-pipe peak microbenchmark for the B200 (sm_100a).
//
// MEASURED_PEAKS.json carries HBM and tensor peaks only; the hashing kernels
// are bound by the 32-bit integer pipes. This program measures, on the box:
//   * per-instruction issue rates (LOP3, SHF, IADD3, PRMT on the ALU pipe;
//     IMAD on the FMA pipe) with 8 independent dependency chains per thread,
//   * an ALU+FMA mix (can adds ride on the FMA pipe while logic saturates ALU?),
//   * the three compression functions fed from registers (no memory traffic):
//     the compute-only ceiling of the leaf kernels (SHA-256 both as the compiler
//     places it -- additions on the ALU pipe -- and in the product's formulation
//     with every addition an IMAD on the FMA pipe).
// Output: one JSON object on stdout. Rates are in 10^12 thread-instructions/s
// ("Tops/s") over the whole GPU at the clocks the run saw.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "../paper_2510_00554_b200/csrc/blake2b.cuh"
#include "../paper_2510_00554_b200/csrc/keccak.cuh"
#include "../paper_2510_00554_b200/csrc/sha256.cuh"

#define CHECK(x)                                                                      \
    do {                                                                              \
        cudaError_t e = (x);                                                          \
        if (e != cudaSuccess) {                                                       \
            fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));                   \
            exit(1);                                                                  \
        }                                                                             \
    } while (0)

constexpr int THREADS = 256;
constexpr int CHAINS = 8;
constexpr int INNER = 64;      // ops per chain per loop iteration

enum Op { OP_LOP3, OP_SHF, OP_IADD3, OP_PRMT, OP_IMAD, OP_MIX_LOP3_IMAD, OP_MIX_SHF_LOP3_IADD, OP_IMAD_WIDE, OP_MIX_LOP3_WIDE, OP_IMAD_HI,
          OP_DEP_LOP3_IMAD, OP_MIX21_DISTINCT, OP_MIX11_DISTINCT, OP_LOP3_DISTINCT, OP_IMAD_DISTINCT, OP_SHF_IMAD_DISTINCT };

template <int OP>
__global__ void __launch_bounds__(THREADS) op_kernel(uint32_t* out, int iters, uint32_t seed) {
    uint32_t x[CHAINS], y = seed ^ threadIdx.x, z = seed * 2654435761u + blockIdx.x;
    uint32_t yy[CHAINS], zz[CHAINS];      // per-chain operands: no operand-reuse-cache help
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
        x[c] = seed + c * 0x9e3779b9u + threadIdx.x;
        yy[c] = (seed ^ threadIdx.x) * (2 * c + 3);
        zz[c] = seed * 2654435761u + blockIdx.x + c;
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < INNER; ++k) {
#pragma unroll
            for (int c = 0; c < CHAINS; ++c) {
                if (OP == OP_LOP3) {
                    asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(y), "r"(z));
                } else if (OP == OP_SHF) {
                    asm volatile("shf.r.wrap.b32 %0, %0, %1, 7;" : "+r"(x[c]) : "r"(y));
                } else if (OP == OP_IADD3) {
                    asm volatile("{ .reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %2; }" : "+r"(x[c]) : "r"(y), "r"(z));
                } else if (OP == OP_PRMT) {
                    asm volatile("prmt.b32 %0, %0, %1, 0x2103;" : "+r"(x[c]) : "r"(y));
                } else if (OP == OP_IMAD) {
                    asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(y), "r"(z));
                } else if (OP == OP_IMAD_WIDE) {
                    // x = lo(x * y) ^ hi(x * y): one IMAD.WIDE + one LOP3 per step; counted as 1 wide
                    asm volatile("{ .reg .u64 t; .reg .u32 a, b; mul.wide.u32 t, %0, %1; mov.b64 {a, b}, t; xor.b32 %0, a, b; }"
                                 : "+r"(x[c]) : "r"(y));
                } else if (OP == OP_IMAD_HI) {
                    asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(x[c]) : "r"(y));
                } else if (OP == OP_MIX_LOP3_WIDE) {
                    if (c & 1) asm volatile("{ .reg .u64 t; .reg .u32 a, b; mul.wide.u32 t, %0, %1; mov.b64 {a, b}, t; add.u32 %0, a, b; }"
                                            : "+r"(x[c]) : "r"(y));
                    else asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(y), "r"(z));
                } else if (OP == OP_DEP_LOP3_IMAD) {
                    // one dependent chain hopping between the pipes: counted as 2 ops
                    asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(yy[c]), "r"(zz[c]));
                    asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(yy[c]), "r"(zz[c]));
                } else if (OP == OP_MIX21_DISTINCT) {
                    if (c % 3 == 2) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(yy[c]), "r"(zz[c]));
                    else asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(yy[c]), "r"(zz[c]));
                } else if (OP == OP_MIX11_DISTINCT) {
                    if (c & 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(yy[c]), "r"(zz[c]));
                    else asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(yy[c]), "r"(zz[c]));
                } else if (OP == OP_LOP3_DISTINCT) {
                    asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(yy[c]), "r"(zz[c]));
                } else if (OP == OP_IMAD_DISTINCT) {
                    asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(yy[c]), "r"(zz[c]));
                } else if (OP == OP_SHF_IMAD_DISTINCT) {
                    if (c & 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(yy[c]), "r"(zz[c]));
                    else asm volatile("shf.r.wrap.b32 %0, %0, %0, 7;" : "+r"(x[c]));
                } else if (OP == OP_MIX_LOP3_IMAD) {
                    if (c & 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(y), "r"(z));
                    else asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(y), "r"(z));
                } else {
                    // the SHA-256 ALU mix: ~6 SHF : 4 LOP3 : 4 IADD3 per round
                    if ((k % 7) < 3) asm volatile("shf.r.wrap.b32 %0, %0, %1, 11;" : "+r"(x[c]) : "r"(y));
                    else if ((k % 7) < 5) asm volatile("lop3.b32 %0, %0, %1, %2, 0xca;" : "+r"(x[c]) : "r"(y), "r"(z));
                    else asm volatile("{ .reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %2; }" : "+r"(x[c]) : "r"(y), "r"(z));
                }
            }
        }
    }
    uint32_t r = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) r ^= x[c] ^ yy[c] ^ zz[c];
    if (r == 0x12345678u) out[blockIdx.x * THREADS + threadIdx.x] = r;
}

// compression functions from registers: `iters` compressions per thread
__global__ void __launch_bounds__(128) sha256_kernel(uint32_t* out, int iters, uint32_t seed) {
    uint32_t s[8], w[16];
    snt::Sha256::init(s);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) w[i] = s[i & 7] ^ (seed + i + it + threadIdx.x * 977u);
        snt::Sha256::compress(s, w);
    }
    if (s[0] == 0x12345678u) out[blockIdx.x * 128 + threadIdx.x] = s[1];
}

// the product's formulation: every addition an IMAD with at most two vector operands (sha256.cuh)
__constant__ uint32_t k_ones[32] = {1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1};
__global__ void __launch_bounds__(128) sha256_fma_kernel(uint32_t* out, int iters, uint32_t seed, uint32_t one) {
    uint32_t s[8], w[16];
    snt::Sha256::init(s);
    const snt::Sha256::One o(one, k_ones[threadIdx.x & 31]);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) w[i] = s[i & 7] ^ (seed + i + it + threadIdx.x * 977u);
        snt::Sha256::compress(s, w, o);
    }
    if (s[0] == 0x12345678u) out[blockIdx.x * 128 + threadIdx.x] = s[1];
}

__global__ void __launch_bounds__(128) blake2b_kernel(uint32_t* out, int iters, uint32_t seed) {
    uint64_t h[8], m[16];
    snt::Blake2b::init(h);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) m[i] = h[i & 7] ^ (static_cast<uint64_t>(seed + i + threadIdx.x * 977u) << 13) ^ it;
        snt::Blake2b::compress(h, m, 128ull * (it + 1), false);
    }
    if (h[0] == 0x12345678ull) out[blockIdx.x * 128 + threadIdx.x] = static_cast<uint32_t>(h[1]);
}

__global__ void __launch_bounds__(128) keccak_kernel(uint32_t* out, int iters, uint32_t seed) {
    uint64_t a[25];
#pragma unroll
    for (int i = 0; i < 25; ++i) a[i] = (seed + threadIdx.x) * (i + 1);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 17; ++i) a[i] ^= (static_cast<uint64_t>(seed + i) << 7) ^ it;
        snt::Sha3_256::permute(a);
    }
    if (a[0] == 0x12345678ull) out[blockIdx.x * 128 + threadIdx.x] = static_cast<uint32_t>(a[1]);
}

template <class F>
static float time_ms(F launch, int reps) {
    cudaEvent_t a, b;
    CHECK(cudaEventCreate(&a));
    CHECK(cudaEventCreate(&b));
    launch();
    launch();
    CHECK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        CHECK(cudaEventRecord(a));
        launch();
        CHECK(cudaEventRecord(b));
        CHECK(cudaEventSynchronize(b));
        float ms;
        CHECK(cudaEventElapsedTime(&ms, a, b));
        if (ms < best) best = ms;
    }
    CHECK(cudaGetLastError());
    return best;
}

int main() {
    cudaDeviceProp prop;
    CHECK(cudaGetDeviceProperties(&prop, 0));
    const int sms = prop.multiProcessorCount;
    uint32_t* out;
    CHECK(cudaMalloc(&out, sizeof(uint32_t) * sms * 16 * THREADS));
    const int iters = 200;
    const int grid = sms * 8;     // 8 CTAs x 256 threads = 64 warps per SM

    printf("{\"gpu\": \"%s\", \"sms\": %d", prop.name, sms);
#define RUN_OP(name, OP, count_per_slot)                                                       \
    {                                                                                          \
        float ms = time_ms([&] { op_kernel<OP><<<grid, THREADS>>>(out, iters, 12345u); }, 5);  \
        double ops = double(grid) * THREADS * double(iters) * INNER * CHAINS * (count_per_slot); \
        printf(", \"%s_tops\": %.3f", name, ops / (ms * 1e-3) / 1e12);                       \
    }
    RUN_OP("lop3", OP_LOP3, 1.0)
    RUN_OP("shf", OP_SHF, 1.0)
    RUN_OP("iadd3", OP_IADD3, 1.0)
    RUN_OP("prmt", OP_PRMT, 1.0)
    RUN_OP("imad", OP_IMAD, 1.0)
    RUN_OP("mix_lop3_imad", OP_MIX_LOP3_IMAD, 1.0)
    RUN_OP("mix_sha_alu", OP_MIX_SHF_LOP3_IADD, 1.0)
    RUN_OP("imad_wide_plus_lop3", OP_IMAD_WIDE, 1.0)
    RUN_OP("imad_hi", OP_IMAD_HI, 1.0)
    RUN_OP("mix_lop3_widepair", OP_MIX_LOP3_WIDE, 1.0)
    RUN_OP("dep_lop3_imad", OP_DEP_LOP3_IMAD, 2.0)
    RUN_OP("mix21_distinct", OP_MIX21_DISTINCT, 1.0)
    RUN_OP("mix11_distinct", OP_MIX11_DISTINCT, 1.0)
    RUN_OP("lop3_distinct", OP_LOP3_DISTINCT, 1.0)
    RUN_OP("imad_distinct", OP_IMAD_DISTINCT, 1.0)
    RUN_OP("shf_imad_distinct", OP_SHF_IMAD_DISTINCT, 1.0)

    {
        const int it = 256;
        const int g = sms * 16;
        float ms = time_ms([&] { sha256_kernel<<<g, 128>>>(out, it, 7u); }, 5);
        double comp = double(g) * 128 * it;
        printf(", \"sha256_regs_gcomp_s\": %.3f, \"sha256_regs_gbs\": %.1f", comp / (ms * 1e-3) / 1e9,
               comp * 64 / (ms * 1e-3) / 1e9);
        ms = time_ms([&] { sha256_fma_kernel<<<g, 128>>>(out, it, 7u, 1u); }, 5);
        printf(", \"sha256_fma_regs_gcomp_s\": %.3f, \"sha256_fma_regs_gbs\": %.1f", comp / (ms * 1e-3) / 1e9,
               comp * 64 / (ms * 1e-3) / 1e9);
        ms = time_ms([&] { blake2b_kernel<<<g, 128>>>(out, it, 7u); }, 5);
        printf(", \"blake2b_regs_gcomp_s\": %.3f, \"blake2b_regs_gbs\": %.1f", comp / (ms * 1e-3) / 1e9,
               comp * 128 / (ms * 1e-3) / 1e9);
        ms = time_ms([&] { keccak_kernel<<<g, 128>>>(out, it, 7u); }, 5);
        printf(", \"keccak_regs_gperm_s\": %.3f, \"sha3_regs_gbs\": %.1f", comp / (ms * 1e-3) / 1e9,
               comp * 136 / (ms * 1e-3) / 1e9);
    }
    printf("}\n");
    return 0;
}
