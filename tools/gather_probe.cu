// gather_probe.cu -- random 4-byte access roofline of this GPU.
//
// The union-find passes (hook, compress) are bound by random single-word
// accesses to the label matrix, not by streaming bandwidth.  This probe
// measures, for working sets from L2-resident to far beyond L2:
//   gather  independent random 4-byte loads (ld.relaxed.gpu, like the hook)
//   cas     independent random atomicCAS on 4-byte words
//   chase   dependent random loads (a pointer chase) -- latency under load
// Addresses come from a counter-based hash in registers (no index stream).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_probe tools/gather_probe.cu
//   tools/gather_probe            -> one JSON line per (kind, bytes)
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// K independent loads per thread, 8 in flight at a time
__global__ void k_gather(const uint32_t *__restrict__ a, uint64_t words, int K, uint32_t salt, uint32_t *out) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (int k = 0; k < K; k += 8) {
        uint32_t v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint64_t idx = ((uint64_t)mix(t * 0x9E3779B9u + (k + i) * 0x85EBCA6Bu + salt) * words) >> 32;
            v[i] = ld_relaxed(a + idx);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) acc += v[i];
    }
    if (acc == 0x12345678u) out[0] = acc;
}

__global__ void k_cas(uint32_t *__restrict__ a, uint64_t words, int K, uint32_t salt, uint32_t *out) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (int k = 0; k < K; k += 4) {
        uint32_t v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint64_t idx = ((uint64_t)mix(t * 0x9E3779B9u + (k + i) * 0x85EBCA6Bu + salt) * words) >> 32;
            v[i] = atomicCAS(a + idx, 0xFFFFFFFFu, t);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) acc += v[i];
    }
    if (acc == 0x12345678u) out[0] = acc;
}

// a[i] holds the next index of a random cycle-free walk: one chain per thread
__global__ void k_fill_chase(uint32_t *a, uint64_t words) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < words; i += (uint64_t)gridDim.x * blockDim.x)
        a[i] = (uint32_t)(((uint64_t)mix((uint32_t)i * 0x27d4eb2dU + 7u) * words) >> 32);
}
__global__ void k_chase(const uint32_t *__restrict__ a, uint64_t words, int K, uint32_t *out) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t p = (uint32_t)(((uint64_t)mix(t) * words) >> 32);
    for (int k = 0; k < K; ++k) p = ld_relaxed(a + p);
    if (p == 0x12345678u) out[0] = p;
}

int main(int argc, char **argv) {
    // optional argument: cudaLimitMaxL2FetchGranularity (32 / 64 / 128 bytes)
    if (argc > 1) {
        cudaError_t le = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(argv[1]));
        if (le != cudaSuccess) printf("set limit: %s\n", cudaGetErrorString(le));
    }
    size_t gran = 0;
    cudaDeviceGetLimit(&gran, cudaLimitMaxL2FetchGranularity);
    printf("{\"l2_fetch_granularity\": %zu}\n", gran);
    const uint64_t sizes_mb[] = {16, 64, 256, 1024, 4096, 16384};
    uint32_t *a = nullptr, *out = nullptr;
    const uint64_t maxw = sizes_mb[5] << 18;
    if (cudaMalloc(&a, maxw * 4) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMalloc(&out, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int threads = 256, blocks = 148 * 8;
    for (uint64_t mb : sizes_mb) {
        const uint64_t words = mb << 18;
        cudaMemset(a, 0xFF, words * 4);
        struct { const char *kind; int K; } kinds[] = {{"gather", 256}, {"cas", 64}, {"chase", 64}};
        for (auto &kd : kinds) {
            if (kd.kind[1] == 'h') k_fill_chase<<<148 * 16, 256>>>(a, words);
            float best = 1e30f;
            for (int rep = 0; rep < 4; ++rep) {
                if (kd.kind[0] == 'c' && kd.kind[1] == 'a') cudaMemset(a, 0xFF, words * 4);
                cudaEventRecord(e0);
                if (kd.kind[0] == 'g') k_gather<<<blocks, threads>>>(a, words, kd.K, rep * 77u, out);
                else if (kd.kind[1] == 'a') k_cas<<<blocks, threads>>>(a, words, kd.K, rep * 77u, out);
                else k_chase<<<blocks, threads>>>(a, words, kd.K, out);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (rep > 0 && ms < best) best = ms;
            }
            const double acc = (double)blocks * threads * kd.K;
            const double rate = acc / (best * 1e-3);
            // chase: every thread's loads are dependent -> latency = time / K
            const double lat_ns = kd.kind[1] == 'h' ? best * 1e6 / kd.K : 0.0;
            printf("{\"kind\": \"%s\", \"bytes\": %llu, \"accesses\": %.0f, \"ms\": %.4f, \"g_accesses_per_s\": %.2f, "
                   "\"sector_gbs\": %.1f, \"latency_ns\": %.1f, \"in_flight_threads\": %d}\n",
                   kd.kind, (unsigned long long)(words * 4), acc, best, rate / 1e9, rate * 32 / 1e9, lat_ns,
                   blocks * threads);
        }
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
    return 0;
}
