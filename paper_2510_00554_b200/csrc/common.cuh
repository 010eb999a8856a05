// Shared helpers for the sm_100a hashing kernels.
//
// Everything marked SNT_HD compiles for both host and device: the per-thread
// hashing logic is exercised on the CPU by tests/hostcheck (no GPU in the
// build container) and runs unchanged inside the kernels on the B200.
#pragma once
#include <stdint.h>
#include <stddef.h>

#if defined(__CUDACC__)
#define SNT_HD __host__ __device__ __forceinline__
#define SNT_D __device__ __forceinline__
#else
#define SNT_HD inline
#define SNT_D inline
#endif

namespace snt {

enum Alg : int { ALG_SHA256 = 0, ALG_BLAKE2B = 1, ALG_SHA3_256 = 2 };

SNT_HD uint32_t rotr32(uint32_t x, int n) {
#ifdef __CUDA_ARCH__
    return __funnelshift_r(x, x, n);   // SHF.R.W
#else
    return (x >> n) | (x << ((32 - n) & 31));
#endif
}

SNT_HD uint32_t bswap32(uint32_t x) {
#ifdef __CUDA_ARCH__
    return __byte_perm(x, 0, 0x0123);  // PRMT
#else
    return __builtin_bswap32(x);
#endif
}

SNT_HD uint64_t rotr64(uint64_t x, int n) {
    return (x >> n) | (x << ((64 - n) & 63));
}
SNT_HD uint64_t rotl64(uint64_t x, int n) {
    return (x << n) | (x >> ((64 - n) & 63));
}

// r = low 32 bits of ((hi:lo) >> (8*a)), a in 0..3 (byte funnel).
SNT_HD uint32_t funnel_bytes(uint32_t lo, uint32_t hi, uint32_t a) {
#ifdef __CUDA_ARCH__
    return __funnelshift_r(lo, hi, a * 8);
#else
    return a ? ((lo >> (8 * a)) | (hi << (32 - 8 * a))) : lo;
#endif
}

// ---- global loads ---------------------------------------------------------
// Input bytes are read exactly once: use the read-only path and do not
// allocate in L1 (streaming).

SNT_HD uint32_t ld32(const void* p) {
#ifdef __CUDA_ARCH__
    return __ldg(reinterpret_cast<const uint32_t*>(p));
#else
    return *reinterpret_cast<const uint32_t*>(p);
#endif
}

SNT_HD uint8_t ld8(const void* p) {
#ifdef __CUDA_ARCH__
    return __ldg(reinterpret_cast<const uint8_t*>(p));
#else
    return *reinterpret_cast<const uint8_t*>(p);
#endif
}

struct alignas(8) U2 { uint32_t x, y; };
struct alignas(16) U4 { uint32_t x, y, z, w; };

SNT_HD U2 ld64(const void* p) {
    U2 r;
#ifdef __CUDA_ARCH__
    uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
    r.x = v.x; r.y = v.y;
#else
    r = *reinterpret_cast<const U2*>(p);
#endif
    return r;
}

SNT_HD U4 ld128(const void* p) {
    U4 r;
#ifdef __CUDA_ARCH__
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
#else
    r = *reinterpret_cast<const U4*>(p);
#endif
    return r;
}

// Load N little-endian 32-bit words starting at byte address p (any
// alignment; all N*4 bytes must be valid message bytes). Picks the widest
// load the address allows. When p is not 4-byte aligned the N+1 aligned words
// that cover the range are read and byte-funnelled; the first and last of
// those words each contain at least one valid byte, so the reads stay inside
// the 4-byte granules the buffer occupies.
template <int N>
SNT_HD void load_words(const uint8_t* p, uint32_t* w) {
    const uintptr_t addr = reinterpret_cast<uintptr_t>(p);
    if ((N % 4 == 0) && (addr & 15) == 0) {
#pragma unroll
        for (int i = 0; i < N / 4; ++i) {
            U4 v = ld128(p + 16 * i);
            w[4 * i + 0] = v.x; w[4 * i + 1] = v.y; w[4 * i + 2] = v.z; w[4 * i + 3] = v.w;
        }
    } else if ((N % 2 == 0) && (addr & 7) == 0) {
#pragma unroll
        for (int i = 0; i < N / 2; ++i) {
            U2 v = ld64(p + 8 * i);
            w[2 * i + 0] = v.x; w[2 * i + 1] = v.y;
        }
    } else if ((addr & 3) == 0) {
#pragma unroll
        for (int i = 0; i < N; ++i) w[i] = ld32(p + 4 * i);
    } else {
        const uint32_t a = static_cast<uint32_t>(addr & 3);
        const uint8_t* q = p - a;
        uint32_t lo = ld32(q);
#pragma unroll
        for (int i = 0; i < N; ++i) {
            uint32_t hi = ld32(q + 4 * (i + 1));
            w[i] = funnel_bytes(lo, hi, a);
            lo = hi;
        }
    }
}

// Byte `i` of a message tail, zero beyond `n`. Tails are < one hash block.
SNT_HD uint32_t tail_byte(const uint8_t* p, uint32_t i, uint32_t n) {
    return i < n ? static_cast<uint32_t>(ld8(p + i)) : 0u;
}

}  // namespace snt
