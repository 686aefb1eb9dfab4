// common.cuh -- shared device helpers and error plumbing for libinfuser_b200.
#pragma once
#include <cstdint>
#include <cstdio>
#include <string>
#include <cuda_runtime.h>

#include "../../include/infuser_b200.h"

namespace imx {

void set_error(const char *fmt, ...);
int cuda_fail(cudaError_t e, const char *what, const char *file, int line);

#define IMX_CUDA(call)                                                       \
    do {                                                                     \
        cudaError_t _e = (call);                                             \
        if (_e != cudaSuccess) return ::imx::cuda_fail(_e, #call, __FILE__, __LINE__); \
    } while (0)

#define IMX_CHECK_LAUNCH() IMX_CUDA(cudaGetLastError())

#define IMX_TRY(expr)                                                        \
    do { int _r = (expr); if (_r != IMX_OK) return _r; } while (0)

// H_MAX = 2^31 - 1 (hashing.py:23)
constexpr int32_t H_MAX = 0x7FFFFFFF;

// ---------------------------------------------------------------------------
// MurmurHash3 x86_32 of the 8-byte key LE32(lo) || LE32(hi), seed 0:
// two full blocks, no tail, length 8 (hashing.py:65-86).
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint32_t rotl32(uint32_t x, int r) {
    return (x << r) | (x >> (32 - r));
}
__host__ __device__ __forceinline__ uint32_t murmur3_pair(uint32_t lo, uint32_t hi) {
    const uint32_t c1 = 0xCC9E2D51u, c2 = 0x1B873593u;
    uint32_t h = 0u;
    uint32_t k = lo * c1; k = rotl32(k, 15); k *= c2;
    h ^= k; h = rotl32(h, 13); h = h * 5u + 0xE6546B64u;
    k = hi * c1; k = rotl32(k, 15); k *= c2;
    h ^= k; h = rotl32(h, 13); h = h * 5u + 0xE6546B64u;
    h ^= 8u;
    h ^= h >> 16; h *= 0x85EBCA6Bu;
    h ^= h >> 13; h *= 0xC2B2AE35u;
    h ^= h >> 16;
    return h;
}
// build_hash_table: digest of (min, max) masked to 31 bits (hashing.py:97-101)
__host__ __device__ __forceinline__ int32_t edge_hash(int32_t u, int32_t v) {
    uint32_t lo = (uint32_t)(u < v ? u : v), hi = (uint32_t)(u < v ? v : u);
    return (int32_t)(murmur3_pair(lo, hi) & 0x7FFFFFFFu);
}

// Relaxed, L2-coherent accesses for the concurrent union-find.
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t *p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// process-wide count of this library's kernel launches (imx_launch_count)
void note_launch(int64_t k = 1);
// recycled non-blocking streams (graph.cu)
cudaError_t acquire_stream(int dev, cudaStream_t *st);
void release_stream(int dev, cudaStream_t st);
// host->device copy of a pageable buffer, staged through pinned memory by
// host threads when large (upload.cu)
cudaError_t upload_h2d(void *dst, const void *src, size_t bytes, cudaStream_t st);
bool host_pinned_ptr(const void *p);
// recycled pinned host buffers (ctx.cu)
cudaError_t pinned_get(void **p, size_t bytes);
void pinned_put(void *p, size_t bytes);
// stream-ordered allocation from the device's pool (ctx.cu)
cudaError_t pool_alloc(void **p, size_t bytes, cudaStream_t st);

}  // namespace imx
