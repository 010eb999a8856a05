// Latency of one SHA-256 tree-node hash computed by ONE warp alone on its SM (the situation of the last
// levels of the tree): a chain of dependent node hashes, one variant per formulation.
//   unrolled        Sha256::hash_pair, 64 rounds unrolled twice (26 + 16 KB of code), additions on the ALU pipe
//   unrolled_imad   the same with the additions as IMAD (the leaf loop's formulation)
//   rolled          Sha256::hash_pair_rolled: 16-round body x 4, constants from a table (7 KB)
//   *_noinline      called out of line with the operands in local memory, as in the fused kernel
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include "../paper_2510_00554_b200/csrc/algs.cuh"
using namespace snt;

#define CHECK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __noinline__ void pair_unrolled_ni(uint32_t* l, const uint32_t* r, const MerkleConsts* c) {
    uint32_t o[8];
    Sha256::hash_pair(l, r, c->sha256_pad_node, o);
    for (int i = 0; i < 8; ++i) l[i] = o[i];
}
__device__ __noinline__ void pair_rolled_ni(uint32_t* l, const uint32_t* r) {
    uint32_t o[8];
    Sha256::hash_pair_rolled(l, r, o);
    for (int i = 0; i < 8; ++i) l[i] = o[i];
}

template <int V>
__global__ void chain_kernel(const __grid_constant__ MerkleConsts c, int n, uint32_t* out) {
    uint32_t l[8], r[8];
    for (int i = 0; i < 8; ++i) { l[i] = threadIdx.x * 7 + i; r[i] = threadIdx.x * 13 + i; }
    for (int k = 0; k < n; ++k) {
        if (V == 0) { uint32_t o[8]; Sha256::hash_pair(l, r, c.sha256_pad_node, o); for (int i = 0; i < 8; ++i) l[i] = o[i]; }
        if (V == 1) { uint32_t o[8]; Sha256::hash_pair(l, r, c.sha256_pad_node, o, sha256_one(c)); for (int i = 0; i < 8; ++i) l[i] = o[i]; }
        if (V == 2) { uint32_t o[8]; Sha256::hash_pair_rolled(l, r, o); for (int i = 0; i < 8; ++i) l[i] = o[i]; }
        if (V == 3) pair_unrolled_ni(l, r, &c);
        if (V == 4) pair_rolled_ni(l, r);
        // what the narrowing levels do between two hashes: fetch the children from the neighbouring lanes
        for (int i = 0; i < 8; ++i) r[i] = __shfl_sync(0xffffffffu, l[i], (threadIdx.x + 1) & 31);
    }
    for (int i = 0; i < 8; ++i) out[threadIdx.x * 8 + i] = l[i];
}

template <int V>
static void run(const char* name, const MerkleConsts& c, uint32_t* d_out) {
    const int n = 2000;
    chain_kernel<V><<<1, 32>>>(c, 10, d_out);
    CHECK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    CHECK(cudaEventCreate(&e0)); CHECK(cudaEventCreate(&e1));
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        CHECK(cudaEventRecord(e0));
        chain_kernel<V><<<1, 32>>>(c, n, d_out);
        CHECK(cudaEventRecord(e1));
        CHECK(cudaEventSynchronize(e1));
        float ms; CHECK(cudaEventElapsedTime(&ms, e0, e1));
        best = ms < best ? ms : best;
    }
    uint32_t h[8];
    CHECK(cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost));
    printf("{\"variant\": \"%s\", \"us_per_node_hash\": %.3f, \"check\": \"%08x\"}\n", name, best * 1000.0 / n, h[0]);
}

int main() {
    MerkleConsts c;
    memset(&c, 0, sizeof(c));
    Sha256::pad_schedule(64, c.sha256_pad_node);
    c.one = 1;
    uint32_t* d_out;
    CHECK(cudaMalloc(&d_out, 32 * 8 * 4));
    run<0>("unrolled", c, d_out);
    run<1>("unrolled_imad", c, d_out);
    run<2>("rolled", c, d_out);
    run<3>("unrolled_noinline", c, d_out);
    run<4>("rolled_noinline", c, d_out);
    return 0;
}
