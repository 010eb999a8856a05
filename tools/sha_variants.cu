// SHA-256 formulation experiments (compute-only, message from registers).
//
// The ALU pipe (LOP3/SHF/IADD3/PRMT, 64 lanes/clk/SM) and the FMA pipe (IMAD,
// 64 lanes/clk/SM) issue concurrently on sm_100a (tools/intpeak: 18.5 + 18.5 =
// 36 Tops/s). The stock compilation of SHA-256 puts ~1280 of its ~1410
// instructions per compression on the ALU pipe. These variants move work to
// the FMA pipe and report GB/s per variant so the best one can be adopted:
//   rotations as IMAD.WIDE: x * 2^(32-n) = (x >> n) : (x << (32-n)); the two
//   halves are bit-disjoint, so rotr(x, n) = hi ^ lo and the XOR folds into the
//   LOP3 that combines the sigma terms;
//   additions as IMAD (a * 1 + b) with the 1 hidden from the compiler.
// Every variant is checked against the stock compression on the same input.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <string>

#include "../paper_2510_00554_b200/csrc/sha256.cuh"

#define CHECK(x)                                                                      \
    do {                                                                              \
        cudaError_t e = (x);                                                          \
        if (e != cudaSuccess) {                                                       \
            fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));                   \
            exit(1);                                                                  \
        }                                                                             \
    } while (0)

struct Consts {
    uint32_t one;
    uint32_t p[32];    // p[n] = 2^(32-n) for n in 1..31
    const uint32_t* ones;   // device array of 1s: a load the compiler cannot see through (per-thread register)
};

__device__ __forceinline__ uint64_t mulwide(uint32_t x, uint32_t m) {
    uint64_t r;
    asm("mul.wide.u32 %0, %1, %2;" : "=l"(r) : "r"(x), "r"(m));
    return r;
}
__device__ __forceinline__ uint32_t lo32(uint64_t v) { return static_cast<uint32_t>(v); }
__device__ __forceinline__ uint32_t hi32(uint64_t v) { return static_cast<uint32_t>(v >> 32); }
__device__ __forceinline__ uint32_t madd(uint32_t a, uint32_t one, uint32_t b) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(one), "r"(b));
    return r;
}

// SS: small sigmas via IMAD.WIDE; SB: big sigmas via IMAD.WIDE;
// AD: 0 = compiler's choice, 1 = every add on the FMA pipe, 2 = schedule adds on FMA,
//     3 = (h + K + w) and (d + t1) on FMA
template <int SS, int SB, int AD>
struct V {
    const Consts& c;
    uint32_t vone;
    __device__ V(const Consts& cc) : c(cc), vone(cc.ones[threadIdx.x & 31]) {}
    static __device__ __forceinline__ uint32_t maddk(uint32_t one_v, uint32_t k, uint32_t x) {
        uint32_t r;
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(one_v), "r"(k), "r"(x));   // k folds to an immediate
        return r;
    }
    // x >> n as the high half of x * 2^(32-n): IMAD.HI on the FMA pipe (half rate), one vector operand
    __device__ __forceinline__ uint32_t shr_hi(uint32_t x, int n) const {
        uint32_t r;
        asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(c.p[n]));
        return r;
    }
    __device__ __forceinline__ uint32_t ssig0(uint32_t x) const {
        if (AD == 6 || AD == 7 || AD == 10) return snt::rotr32(x, 7) ^ snt::rotr32(x, 18) ^ shr_hi(x, 3);
        if (SS) {
            const uint64_t a = mulwide(x, c.p[7]), b = mulwide(x, c.p[18]), d = mulwide(x, c.p[3]);
            return lo32(a) ^ hi32(a) ^ lo32(b) ^ hi32(b) ^ hi32(d);
        }
        return snt::Sha256::ssig0(x);
    }
    __device__ __forceinline__ uint32_t ssig1(uint32_t x) const {
        if (AD == 6 || AD == 7 || AD == 10 || AD == 11) return snt::rotr32(x, 17) ^ snt::rotr32(x, 19) ^ shr_hi(x, 10);
        if (SS) {
            const uint64_t a = mulwide(x, c.p[17]), b = mulwide(x, c.p[19]), d = mulwide(x, c.p[10]);
            return lo32(a) ^ hi32(a) ^ lo32(b) ^ hi32(b) ^ hi32(d);
        }
        return snt::Sha256::ssig1(x);
    }
    __device__ __forceinline__ uint32_t bsig0(uint32_t x) const {
        if (SB) {
            const uint64_t a = mulwide(x, c.p[2]), b = mulwide(x, c.p[13]), d = mulwide(x, c.p[22]);
            return lo32(a) ^ hi32(a) ^ lo32(b) ^ hi32(b) ^ lo32(d) ^ hi32(d);
        }
        return snt::Sha256::bsig0(x);
    }
    __device__ __forceinline__ uint32_t bsig1(uint32_t x) const {
        if (SB) {
            const uint64_t a = mulwide(x, c.p[6]), b = mulwide(x, c.p[11]), d = mulwide(x, c.p[25]);
            return lo32(a) ^ hi32(a) ^ lo32(b) ^ hi32(b) ^ lo32(d) ^ hi32(d);
        }
        return snt::Sha256::bsig1(x);
    }
    __device__ __forceinline__ uint32_t add_sched(uint32_t a, uint32_t b) const {
        return (AD == 1 || AD == 2 || AD >= 4) ? madd(a, c.one, b) : a + b;
    }
    __device__ __forceinline__ uint32_t add_fma(uint32_t a, uint32_t b) const {
        return (AD == 1 || AD == 3) ? madd(a, c.one, b) : a + b;
    }
    __device__ __forceinline__ uint32_t add_any(uint32_t a, uint32_t b) const {
        return (AD == 1) ? madd(a, c.one, b) : a + b;
    }
    __device__ __forceinline__ void compress(uint32_t s[8], uint32_t w[16]) const {
        const uint32_t K[64] = {SNT_SHA256_K};
        uint32_t a = s[0], b = s[1], cc = s[2], d = s[3], e = s[4], f = s[5], g = s[6], h = s[7];
#pragma unroll
        for (int t = 0; t < 64; ++t) {
            if (t >= 16) {
                const uint32_t x = add_sched(w[t & 15], w[(t - 7) & 15]);
                const uint32_t y = add_sched(ssig1(w[(t - 2) & 15]), ssig0(w[(t - 15) & 15]));
                w[t & 15] = add_sched(x, y);
            }
            if (AD >= 8) {
                // 8: only (h + K + w) stays an ALU IADD3 (K in its immediate slot); 9: K enters through
                // IMAD(vone, K, h) with a per-thread register holding 1, so no addition is left on the ALU pipe
                const uint32_t hkw = (AD == 8) ? h + K[t] + w[t & 15]
                                               : madd(maddk(vone, K[t], h), c.one, w[t & 15]);
                const uint32_t t1 = madd(hkw, c.one, madd(bsig1(e), c.one, snt::Sha256::ch(e, f, g)));
                const uint32_t na = madd(t1, c.one, madd(bsig0(a), c.one, snt::Sha256::maj(a, b, cc)));
                h = g; g = f; f = e; e = madd(d, c.one, t1); d = cc; cc = b; b = a; a = na;
                continue;
            }
            if (AD >= 4) {
                // K rides in the immediate slot of an ALU IADD3; the two-input additions go to IMAD with
                // the multiplier in a uniform register (two vector operands per instruction)
                const uint32_t t1 = (h + K[t] + w[t & 15]) + (bsig1(e) + snt::Sha256::ch(e, f, g));
                uint32_t na;
                if (AD == 5 || AD == 6) na = madd(t1, c.one, madd(bsig0(a), c.one, snt::Sha256::maj(a, b, cc)));
                else na = t1 + bsig0(a) + snt::Sha256::maj(a, b, cc);
                h = g; g = f; f = e; e = (AD == 7) ? d + t1 : madd(d, c.one, t1); d = cc; cc = b; b = a; a = na;
                continue;
            }
            const uint32_t hk = add_fma(add_fma(h, K[t]), w[t & 15]);          // off the critical path
            const uint32_t t1 = add_any(add_any(hk, snt::Sha256::ch(e, f, g)), bsig1(e));
            const uint32_t t2 = add_any(bsig0(a), snt::Sha256::maj(a, b, cc));
            h = g; g = f; f = e; e = add_fma(d, t1); d = cc; cc = b; b = a; a = add_any(t1, t2);
        }
        s[0] += a; s[1] += b; s[2] += cc; s[3] += d; s[4] += e; s[5] += f; s[6] += g; s[7] += h;
    }
};

template <int SS, int SB, int AD>
__global__ void __launch_bounds__(128) variant_kernel(uint32_t* out, int iters, uint32_t seed,
                                                      const __grid_constant__ Consts c, int check) {
    V<SS, SB, AD> v(c);
    uint32_t s[8], w[16];
    snt::Sha256::init(s);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) w[i] = s[i & 7] ^ (seed + i + it + threadIdx.x * 977u);
        v.compress(s, w);
    }
    if (check) {
        uint32_t r = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) r ^= s[i] * (i + 1);
        out[blockIdx.x * 128 + threadIdx.x] = r;
    } else if (s[0] == 0x12345678u) {
        out[blockIdx.x * 128 + threadIdx.x] = s[1];
    }
}

static uint32_t* g_out;
static uint32_t* g_ref;
static Consts g_c;

template <int SS, int SB, int AD>
static void run(const char* name, int sms, int ctas_per_sm) {
    const int g = sms * ctas_per_sm, it = 256;
    // correctness against the stock formulation
    variant_kernel<SS, SB, AD><<<4, 128>>>(g_out, 3, 99u, g_c, 1);
    CHECK(cudaDeviceSynchronize());
    uint32_t a[512], b[512];
    CHECK(cudaMemcpy(a, g_out, sizeof(a), cudaMemcpyDeviceToHost));
    CHECK(cudaMemcpy(b, g_ref, sizeof(b), cudaMemcpyDeviceToHost));
    int ok = 1;
    for (int i = 0; i < 512; ++i) ok &= (a[i] == b[i]);
    cudaEvent_t e0, e1;
    CHECK(cudaEventCreate(&e0));
    CHECK(cudaEventCreate(&e1));
    float best = 1e30f;
    for (int r = 0; r < 6; ++r) {
        CHECK(cudaEventRecord(e0));
        variant_kernel<SS, SB, AD><<<g, 128>>>(g_out, it, 7u, g_c, 0);
        CHECK(cudaEventRecord(e1));
        CHECK(cudaEventSynchronize(e1));
        float ms;
        CHECK(cudaEventElapsedTime(&ms, e0, e1));
        if (r > 0 && ms < best) best = ms;
    }
    CHECK(cudaGetLastError());
    const double comp = double(g) * 128 * it;
    printf("{\"variant\": \"%s\", \"ss\": %d, \"sb\": %d, \"ad\": %d, \"warps_per_sm\": %d, \"ok\": %d, \"gbs\": %.1f}\n",
           name, SS, SB, AD, ctas_per_sm * 4, ok, comp * 64 / (best * 1e-3) / 1e9);
}

int main(int argc, char** argv) {
    cudaDeviceProp prop;
    CHECK(cudaGetDeviceProperties(&prop, 0));
    const int sms = prop.multiProcessorCount;
    CHECK(cudaMalloc(&g_out, sizeof(uint32_t) * sms * 16 * 128));
    CHECK(cudaMalloc(&g_ref, sizeof(uint32_t) * 512));
    g_c.one = 1;
    for (int n = 1; n < 32; ++n) g_c.p[n] = 1u << (32 - n);
    g_c.p[0] = 0;
    {
        uint32_t h_ones[32];
        for (int i = 0; i < 32; ++i) h_ones[i] = 1;
        uint32_t* d_ones;
        CHECK(cudaMalloc(&d_ones, sizeof(h_ones)));
        CHECK(cudaMemcpy(d_ones, h_ones, sizeof(h_ones), cudaMemcpyHostToDevice));
        g_c.ones = d_ones;
    }
    variant_kernel<0, 0, 0><<<4, 128>>>(g_ref, 3, 99u, g_c, 1);
    CHECK(cudaDeviceSynchronize());
    if (argc > 1) {      // one variant only (for ncu): sha_variants <name> [ctas_per_sm]
        const std::string v = argv[1];
        const int occ = argc > 2 ? atoi(argv[2]) : 8;
        if (v == "stock") run<0, 0, 0>("stock", sms, occ);
        else if (v == "adds_imad") run<0, 0, 1>("adds_imad", sms, occ);
        else if (v == "sched_adds_imad") run<0, 0, 2>("sched_adds_imad", sms, occ);
        else if (v == "hkw_adds_imad") run<0, 0, 3>("hkw_adds_imad", sms, occ);
        else if (v == "sched_e") run<0, 0, 4>("sched_e", sms, occ);
        else if (v == "sched_e_a") run<0, 0, 5>("sched_e_a", sms, occ);
        else if (v == "sched_e_a_shr") run<0, 0, 6>("sched_e_a_shr", sms, occ);
        else if (v == "sched_shr") run<0, 0, 7>("sched_shr", sms, occ);
        else if (v == "all_but_hkw") run<0, 0, 8>("all_but_hkw", sms, occ);
        else if (v == "all_adds_ur") run<0, 0, 9>("all_adds_ur", sms, occ);
        else if (v == "all_adds_ur_shr") run<0, 0, 10>("all_adds_ur_shr", sms, occ);
        else if (v == "all_adds_ur_shr1") run<0, 0, 11>("all_adds_ur_shr1", sms, occ);
        else { fprintf(stderr, "unknown variant\n"); return 2; }
        return 0;
    }
    for (int occ : {8, 16}) {
        run<0, 0, 0>("stock", sms, occ);
        run<0, 0, 1>("adds_imad", sms, occ);
        run<0, 0, 2>("sched_adds_imad", sms, occ);
        run<0, 0, 3>("hkw_adds_imad", sms, occ);
        run<0, 0, 4>("sched_e", sms, occ);
        run<0, 0, 5>("sched_e_a", sms, occ);
        run<0, 0, 6>("sched_e_a_shr", sms, occ);
        run<0, 0, 7>("sched_shr", sms, occ);
        run<0, 0, 8>("all_but_hkw", sms, occ);
        run<0, 0, 9>("all_adds_ur", sms, occ);
        run<0, 0, 10>("all_adds_ur_shr", sms, occ);
        run<0, 0, 11>("all_adds_ur_shr1", sms, occ);
        run<1, 0, 0>("ssig_wide", sms, occ);
        run<1, 0, 3>("ssig_wide+hkw_imad", sms, occ);
        run<1, 0, 2>("ssig_wide+sched_imad", sms, occ);
        run<0, 1, 0>("bsig_wide", sms, occ);
        run<1, 1, 0>("all_sig_wide", sms, occ);
        run<1, 1, 3>("all_sig_wide+hkw_imad", sms, occ);
    }
    return 0;
}
