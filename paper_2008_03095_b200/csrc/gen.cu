// gen.cu -- seeded synthetic graphs generated on the device (SURVEY 8(f)
// rank 1: the reference's numpy R-MAT takes 266 s / 32.5 GB at scale 22).
//
// Every random number is a counter-based SplitMix64 value rnd(seed, index),
// so candidate i of a stream is the same no matter how many candidates are
// drawn (a larger draw extends the same sequence) and the numpy restatement
// in paper_2008_03095_b200/generators.py produces bit-identical edges:
//   Erdos-Renyi  u = hi64(rnd(s, 2i) * n), v = hi64(rnd(s, 2i+1) * n)
//   R-MAT        level l of candidate i: x = unit(rnd(s, 64 i + l)) picks the
//                quadrant (a | b | c | d) by the cumulative probabilities
//   Chung-Lu     u = #{cdf <= unit(rnd(s, 2i))}, v likewise with 2i+1
//                (cdf: normalised cumulative expected degrees, from the host)
// Self-loops are dropped and unordered pairs deduplicated on the device
// (radix sort of (min, max) keys, first draw of each pair kept); with m > 0
// the first m distinct pairs in draw order form the graph, with m == 0 every
// distinct pair of the draws.  The edges never leave the device: the CSR
// builder (graph.cu) turns them into the graph.
#include <algorithm>
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "common.cuh"
#include "graph.cuh"

namespace imx {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t rnd(uint64_t seed_mixed, uint64_t idx) { return mix64(seed_mixed ^ idx); }
__host__ __device__ __forceinline__ double unit(uint64_t r) { return (double)(r >> 11) * 0x1.0p-53; }
// floor(r * n / 2^64) for n < 2^32, exact in 64-bit arithmetic
__host__ __device__ __forceinline__ uint64_t below(uint64_t r, uint64_t n) {
    return ((r >> 32) * n + (((r & 0xffffffffull) * n) >> 32)) >> 32;
}

enum { GEN_ER = 0, GEN_RMAT = 1, GEN_CL = 2 };

__global__ void k_gen_candidates(int kind, int64_t n, int scale, uint64_t smix, int64_t first, int64_t count,
                                 double ca, double cb, double cc, const double *__restrict__ cdf,
                                 uint64_t *__restrict__ keys, uint32_t *__restrict__ idx) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < count;
         j += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t i = (uint64_t)(first + j);
        uint64_t u = 0, v = 0;
        if (kind == GEN_ER) {
            u = below(rnd(smix, 2 * i), (uint64_t)n);
            v = below(rnd(smix, 2 * i + 1), (uint64_t)n);
        } else if (kind == GEN_RMAT) {
            for (int l = 0; l < scale; ++l) {
                const double x = unit(rnd(smix, 64 * i + l));
                const uint64_t down = x >= cb, right = (x >= ca && x < cb) || x >= cc;
                u = (u << 1) | down;
                v = (v << 1) | right;
            }
        } else {
            const double x1 = unit(rnd(smix, 2 * i)), x2 = unit(rnd(smix, 2 * i + 1));
            int64_t lo = 0, hi = n;                  // number of cdf entries <= x
            while (lo < hi) { const int64_t mid = (lo + hi) >> 1; if (cdf[mid] <= x1) lo = mid + 1; else hi = mid; }
            u = (uint64_t)(lo < n ? lo : n - 1);
            lo = 0; hi = n;
            while (lo < hi) { const int64_t mid = (lo + hi) >> 1; if (cdf[mid] <= x2) lo = mid + 1; else hi = mid; }
            v = (uint64_t)(lo < n ? lo : n - 1);
        }
        keys[j] = u == v ? ~0ull : (u < v ? u * (uint64_t)n + v : v * (uint64_t)n + u);
        idx[j] = (uint32_t)i;
    }
}

__global__ void k_first_of_run(const uint64_t *__restrict__ keys, int64_t cnt, uint8_t *__restrict__ flag) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < cnt;
         j += (int64_t)gridDim.x * blockDim.x)
        flag[j] = keys[j] != ~0ull && (j == 0 || keys[j] != keys[j - 1]);
}

__global__ void k_keys_to_edges(const uint64_t *__restrict__ keys, int64_t cnt, int64_t n, int64_t *__restrict__ e) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < cnt;
         j += (int64_t)gridDim.x * blockDim.x) {
        e[2 * j] = (int64_t)(keys[j] / (uint64_t)n);
        e[2 * j + 1] = (int64_t)(keys[j] % (uint64_t)n);
    }
}

static int gen_grid(int64_t w) { int64_t b = (w + 255) / 256; return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 16)); }

// distinct non-loop pairs of candidates [0, draws): sorted by key in ukeys,
// their first draw index in uidx; returns the count
static int gen_distinct(cudaStream_t st, int kind, int64_t n, int scale, uint64_t smix, int64_t draws, double ca,
                        double cb, double cc, const double *dcdf, uint64_t **ukeys, uint32_t **uidx, int64_t *count) {
    uint64_t *k0 = nullptr, *k1 = nullptr;
    uint32_t *i0 = nullptr, *i1 = nullptr;
    uint8_t *flag = nullptr;
    int64_t *dcnt = nullptr;
    void *tmp = nullptr;
    size_t tb = 0, tb2 = 0;
    int rc = IMX_OK;
    int endbit = 1;
    while (endbit < 64 && ((uint64_t)n * (uint64_t)n >> endbit)) ++endbit;
#define GG(call) do { cudaError_t _e = (call); if (_e != cudaSuccess) { rc = cuda_fail(_e, #call, __FILE__, __LINE__); goto out; } } while (0)
    GG(pool_alloc((void **)&k0, sizeof(uint64_t) * draws, st));
    GG(pool_alloc((void **)&k1, sizeof(uint64_t) * draws, st));
    GG(pool_alloc((void **)&i0, sizeof(uint32_t) * draws, st));
    GG(pool_alloc((void **)&i1, sizeof(uint32_t) * draws, st));
    GG(pool_alloc((void **)&flag, draws, st));
    GG(pool_alloc((void **)&dcnt, sizeof(int64_t), st));
    k_gen_candidates<<<gen_grid(draws), 256, 0, st>>>(kind, n, scale, smix, 0, draws, ca, cb, cc, dcdf, k0, i0);
    note_launch();
    GG(cudaGetLastError());
    // self-loop keys (~0) must sort last: sort over all 64 bits then
    GG(cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, k1, i0, i1, draws, 0, 64, st));
    GG(cub::DeviceSelect::Flagged(nullptr, tb2, k1, flag, k0, dcnt, draws, st));
    GG(pool_alloc(&tmp, std::max(tb, tb2), st));
    GG(cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, i0, i1, draws, 0, 64, st));
    k_first_of_run<<<gen_grid(draws), 256, 0, st>>>(k1, draws, flag);
    note_launch();
    GG(cudaGetLastError());
    GG(cub::DeviceSelect::Flagged(tmp, tb2, k1, flag, k0, dcnt, draws, st));
    GG(cub::DeviceSelect::Flagged(tmp, tb2, i1, flag, i0, dcnt, draws, st));
    GG(cudaMemcpyAsync(count, dcnt, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    GG(cudaStreamSynchronize(st));
    *ukeys = k0; k0 = nullptr;
    *uidx = i0; i0 = nullptr;
out:
    for (void *p : {(void *)k0, (void *)k1, (void *)i0, (void *)i1, (void *)flag, (void *)dcnt, tmp})
        if (p) cudaFreeAsync(p, st);
#undef GG
    (void)endbit;
    return rc;
}

}  // namespace imx

using namespace imx;

extern "C" int imx_graph_generate(int32_t device, int32_t kind, int64_t n, int64_t m, int64_t draws,
                                  uint64_t seed, const double *params, const double *cdf, imx_graph **out) {
    if (!out) { set_error("out is NULL"); return IMX_EINVAL; }
    *out = nullptr;
    if (kind < GEN_ER || kind > GEN_CL) { set_error("unknown generator kind %d", kind); return IMX_EINVAL; }
    int scale = 0;
    if (kind == GEN_RMAT) {
        while ((int64_t(1) << scale) < n) ++scale;
        if ((int64_t(1) << scale) != n) { set_error("R-MAT needs n = 2^scale, got %lld", (long long)n); return IMX_EINVAL; }
        if (!params) { set_error("R-MAT needs probs[4]"); return IMX_EINVAL; }
    }
    if (kind == GEN_CL && !cdf) { set_error("Chung-Lu needs the cdf"); return IMX_EINVAL; }
    if (n < 2 || n >= (int64_t(1) << 31)) { set_error("vertex count %lld outside [2, 2^31)", (long long)n); return IMX_ECONSTRAINT; }
    if (m < 0 || (m == 0 && draws <= 0) || draws >= (int64_t(1) << 32)) { set_error("bad m/draws"); return IMX_EINVAL; }
    double ca = 0, cb = 0, cc = 0;
    if (kind == GEN_RMAT) {
        const double tot = params[0] + params[1] + params[2] + params[3];
        ca = params[0] / tot; cb = (params[0] + params[1]) / tot; cc = (params[0] + params[1] + params[2]) / tot;
    }
    IMX_TRY(select_device(device));
    cudaStream_t st;
    IMX_CUDA(acquire_stream(device, &st));
    double *dcdf = nullptr;
    uint64_t *ukeys = nullptr;
    uint32_t *uidx = nullptr;
    int64_t *dedges = nullptr;
    int64_t cnt = 0, k = 0;
    int rc = IMX_OK;
    imx_graph *g = nullptr;
    const uint64_t smix = mix64(seed);
    if (m > 0 && draws <= 0) draws = m + m / 4 + 4096;
    if (kind == GEN_CL) {
        if (pool_alloc((void **)&dcdf, sizeof(double) * n, st) != cudaSuccess ||
            cudaMemcpyAsync(dcdf, cdf, sizeof(double) * n, cudaMemcpyHostToDevice, st) != cudaSuccess)
            rc = cuda_fail(cudaGetLastError(), "upload cdf", __FILE__, __LINE__);
    }
    for (; rc == IMX_OK;) {
        rc = gen_distinct(st, kind, n, scale, smix, draws, ca, cb, cc, dcdf, &ukeys, &uidx, &cnt);
        if (rc != IMX_OK || m == 0 || cnt >= m) break;
        cudaFreeAsync(ukeys, st); cudaFreeAsync(uidx, st);
        ukeys = nullptr; uidx = nullptr;
        if (draws >= (int64_t(1) << 31)) { set_error("cannot draw %lld distinct pairs", (long long)m); rc = IMX_EINVAL; break; }
        draws = std::min<int64_t>(draws + draws / 2, (int64_t(1) << 31));   // same streams, extended
    }
    if (rc == IMX_OK) {
        k = m > 0 ? m : cnt;
        if (m > 0) {
            // first m distinct pairs in draw order: sort the uniques by first draw
            uint32_t *i2 = nullptr;
            uint64_t *k2 = nullptr;
            void *tmp = nullptr;
            size_t tb = 0;
            cudaError_t e = pool_alloc((void **)&i2, sizeof(uint32_t) * cnt, st);
            if (e == cudaSuccess) e = pool_alloc((void **)&k2, sizeof(uint64_t) * cnt, st);
            if (e == cudaSuccess) e = cub::DeviceRadixSort::SortPairs(nullptr, tb, uidx, i2, ukeys, k2, cnt, 0, 32, st);
            if (e == cudaSuccess) e = pool_alloc(&tmp, tb, st);
            if (e == cudaSuccess) e = cub::DeviceRadixSort::SortPairs(tmp, tb, uidx, i2, ukeys, k2, cnt, 0, 32, st);
            if (e == cudaSuccess) { std::swap(ukeys, k2); }
            for (void *p : {(void *)i2, (void *)k2, tmp}) if (p) cudaFreeAsync(p, st);
            if (e != cudaSuccess) rc = cuda_fail(e, "first-m selection", __FILE__, __LINE__);
        }
    }
    if (rc == IMX_OK) {
        if (pool_alloc((void **)&dedges, sizeof(int64_t) * 2 * (k > 0 ? k : 1), st) != cudaSuccess) rc = IMX_ENOMEM;
        else {
            k_keys_to_edges<<<gen_grid(k), 256, 0, st>>>(ukeys, k, n, dedges);
            note_launch();
            if (cudaStreamSynchronize(st) != cudaSuccess) rc = cuda_fail(cudaGetLastError(), "keys to edges", __FILE__, __LINE__);
        }
    }
    if (rc == IMX_OK) rc = graph_create(device, n, 2 * k, &g);
    if (rc == IMX_OK) rc = graph_build_from_device_edges(g, dedges, k, nullptr, 1.0);
    for (void *p : {(void *)dcdf, (void *)ukeys, (void *)uidx, (void *)dedges}) if (p) cudaFreeAsync(p, st);
    release_stream(device, st);
    if (rc != IMX_OK) { if (g) graph_free(g); return rc; }
    *out = g;
    return IMX_OK;
}
