// row_probe.cu -- bandwidth of reading whole 4 KB rows of a large matrix, a
// warp per row, in sequential, random and block-random order (the CELF wide
// evaluation reads candidate rows of the 17 GB label matrix in stale-gain
// order, i.e. random row ids).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/row_probe tools/row_probe.cu
//   tools/row_probe  -> one JSON line per (order, quads in flight, via)
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

// mode 0: row = i; 1: row = hash(i) % rows; 2: sorted within groups of G (row = group-random base + j)
template <int Q>
__global__ void k_rows(const uint4 *__restrict__ a, uint64_t rows, uint64_t count, int mode, uint32_t *out) {
    const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    uint32_t acc = 0;
    for (uint64_t i = w; i < count; i += nw) {
        uint64_t r = i;
        if (mode == 1) r = ((uint64_t)mix((uint32_t)i * 0x9E3779B9u + 12345u) * rows) >> 32;
        if (mode == 2) r = ((((uint64_t)mix((uint32_t)(i >> 6) * 0x9E3779B9u + 12345u) * (rows >> 6)) >> 32) << 6) + (i & 63);
        const uint4 *row = a + r * 256;
        for (int q0 = lane; q0 < 256; q0 += 32 * Q) {
            uint4 v[Q];
#pragma unroll
            for (int k = 0; k < Q; ++k) v[k] = row[q0 + 32 * k];
#pragma unroll
            for (int k = 0; k < Q; ++k) acc += v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
        }
    }
    if (acc == 0x12345678u) out[0] = acc;
}

int main() {
    const uint64_t rows = 4u << 20;                    // 4 M rows x 4 KB = 16 GB
    uint4 *a = nullptr;
    uint32_t *out = nullptr;
    if (cudaMalloc(&a, rows * 4096) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMalloc(&out, 4);
    cudaMemset(a, 1, rows * 4096);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const uint64_t count = 1u << 21;                   // 2 M rows = 8 GB per run
    const char *names[] = {"sequential", "random", "random-groups-of-64"};
    for (int mode = 0; mode < 3; ++mode)
        for (int q : {1, 2, 8})
            for (int bpsm : {4, 8}) {
                float best = 1e30f;
                for (int rep = 0; rep < 3; ++rep) {
                    cudaEventRecord(e0);
                    if (q == 1) k_rows<1><<<148 * bpsm, 256>>>(a, rows, count, mode, out);
                    else if (q == 2) k_rows<2><<<148 * bpsm, 256>>>(a, rows, count, mode, out);
                    else k_rows<8><<<148 * bpsm, 256>>>(a, rows, count, mode, out);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    if (ms < best) best = ms;
                }
                printf("{\"order\": \"%s\", \"quads_in_flight\": %d, \"blocks_per_sm\": %d, \"ms\": %.3f, \"GBps\": %.0f}\n",
                       names[mode], q, bpsm, best, count * 4096.0 / (best * 1e-3) / 1e9);
            }
    return 0;
}
