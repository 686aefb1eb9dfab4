// graph.cu -- K1 (CSR builder) and K2 (slot hashes / thresholds) on sm_100a.
//
// Replaces, bit for bit:
//   Graph.from_edges        graph.py:124-155  (validation :134-146, lexsort :149, cumsum :150-151)
//   Graph.sources           graph.py:75-78
//   Graph.canonical_slots   graph.py:80-83
//   Graph.reciprocal_slots  graph.py:85-99
//   Graph.with_weights      graph.py:112-119
//   build_hash_table        hashing.py:97-101
//   slot_thresholds         hashing.py:153-165
//
// The CSR lives on the device for the whole pipeline: the per-slot hash and
// symmetrized threshold are computed here once, and the canonical
// (lo < hi) edge list in slot order is the work list of the hook kernel.
#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstring>
#include <vector>
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "common.cuh"
#include "graph.cuh"

namespace imx {

static thread_local std::string g_err;
static std::atomic<long long> g_launches{0};
void note_launch(int64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

void set_error(const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
}

int cuda_fail(cudaError_t e, const char *what, const char *file, int line) {
    set_error("CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e),
              cudaGetErrorString(e), what, file, line);
    if (e == cudaErrorMemoryAllocation) return IMX_ENOMEM;
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) return IMX_ENODEV;
    return IMX_ECUDA;
}

int select_device(int32_t device) {
    int cnt = 0;
    cudaError_t e = cudaGetDeviceCount(&cnt);
    if (e != cudaSuccess || cnt == 0) {
        cudaGetLastError();
        set_error("no CUDA device available (libinfuser_b200 needs an sm_100 GPU; "
                  "there is no CPU fallback)");
        return IMX_ENODEV;
    }
    if (device < 0 || device >= cnt) {
        set_error("device %d out of range (%d visible)", device, cnt);
        return IMX_EINVAL;
    }
    IMX_CUDA(cudaSetDevice(device));
    return IMX_OK;
}

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
// error flags: bit0 endpoint out of range, bit1 self-loop, bit2 duplicate
__global__ void k_edges_check_and_keys(const int64_t *__restrict__ edges, int64_t k, int64_t n,
                                       int nb, uint64_t *__restrict__ keys,
                                       uint32_t *__restrict__ vals, unsigned *__restrict__ flags) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t u = edges[2 * i], v = edges[2 * i + 1];
        unsigned f = 0;
        if (u < 0 || v < 0 || u >= n || v >= n) f |= 1u;
        else if (u == v) f |= 2u;
        if (f) { atomicOr(flags, f); u = 0; v = 0; }
        keys[i] = ((uint64_t)u << nb) | (uint64_t)v;
        keys[i + k] = ((uint64_t)v << nb) | (uint64_t)u;
        vals[i] = (uint32_t)i;
        vals[i + k] = (uint32_t)i;
    }
}

__global__ void k_csr_from_sorted(const uint64_t *__restrict__ keys, const uint32_t *__restrict__ vals,
                                  int64_t m2, int nb, const double *__restrict__ w_edge,
                                  double w_scalar, int32_t *__restrict__ adj,
                                  int32_t *__restrict__ src, double *__restrict__ w,
                                  unsigned *__restrict__ flags) {
    const uint64_t mask = (nb >= 64) ? ~0ull : ((1ull << nb) - 1);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m2;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t key = keys[i];
        adj[i] = (int32_t)(key & mask);
        src[i] = (int32_t)(key >> nb);
        w[i] = w_edge ? w_edge[vals[i]] : w_scalar;
        if (i > 0 && keys[i - 1] == key) atomicOr(flags, 4u);
    }
}

// xadj[v] = lower_bound(src, v)  (src sorted ascending)
__global__ void k_xadj_from_src(const int32_t *__restrict__ src, int64_t m2, int64_t n,
                                int64_t *__restrict__ xadj) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v <= n;
         v += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = m2;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (src[mid] < v) lo = mid + 1; else hi = mid;
        }
        xadj[v] = lo;
    }
}

// src[s] = row of slot s (np.repeat over degrees, graph.py:75-78)
__global__ void k_src_from_xadj(const int64_t *__restrict__ xadj, int64_t n, int64_t m2,
                                int32_t *__restrict__ src) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < m2;
         s += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = n;  // largest v with xadj[v] <= s
        while (hi - lo > 1) {
            int64_t mid = (lo + hi) >> 1;
            if (xadj[mid] <= s) lo = mid; else hi = mid;
        }
        src[s] = (int32_t)lo;
    }
}

// reciprocal slot of (u, v): position of u in row v (rows sorted ascending)
__global__ void k_reciprocal(const int64_t *__restrict__ xadj, const int32_t *__restrict__ adj,
                             const int32_t *__restrict__ src, int64_t m2,
                             int64_t *__restrict__ recip, unsigned *__restrict__ flags) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < m2;
         s += (int64_t)gridDim.x * blockDim.x) {
        int32_t u = src[s], v = adj[s];
        int64_t lo = xadj[v], hi = xadj[v + 1];
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (adj[mid] < u) lo = mid + 1; else hi = mid;
        }
        if (lo < xadj[v + 1] && adj[lo] == u && lo != s) recip[s] = lo;
        else { recip[s] = -1; atomicOr(flags, 8u); }
    }
}

__global__ void k_slot_hashes(const int32_t *__restrict__ src, const int32_t *__restrict__ adj,
                              int64_t m2, int32_t *__restrict__ hash) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < m2;
         s += (int64_t)gridDim.x * blockDim.x)
        hash[s] = edge_hash(src[s], adj[s]);
}

// thr = int32(int64(w * H_MAX)) (hashing.py:135-138, :162); IEEE f64 multiply
// and truncation toward zero match numpy's astype(np.int64).
__device__ __forceinline__ int32_t thr_of(double w) {
    return (int32_t)(int64_t)(w * 2147483647.0);
}
__global__ void k_thresholds(const double *__restrict__ w, const int64_t *__restrict__ recip,
                             int64_t m2, int32_t *__restrict__ thr,
                             int32_t *__restrict__ tmin, int32_t *__restrict__ tmax) {
    int32_t lmin = INT32_MAX, lmax = INT32_MIN;
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < m2;
         s += (int64_t)gridDim.x * blockDim.x) {
        int32_t t = thr_of(w[s]);
        if (recip) { int32_t t2 = thr_of(w[recip[s]]); t = t2 > t ? t2 : t; }
        thr[s] = t;
        lmin = min(lmin, t); lmax = max(lmax, t);
    }
    for (int o = 16; o; o >>= 1) {
        lmin = min(lmin, __shfl_xor_sync(0xffffffffu, lmin, o));
        lmax = max(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
    }
    if ((threadIdx.x & 31) == 0) { atomicMin(tmin, lmin); atomicMax(tmax, lmax); }
}

__global__ void k_weights_range(const double *__restrict__ w, int64_t m2, unsigned *flags) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < m2;
         s += (int64_t)gridDim.x * blockDim.x) {
        double x = w[s];
        if (x < 0.0 || x > 1.0) atomicOr(flags, 16u);
    }
}

// canonical slots (src < adj) in slot order -> edge list for the hook kernel
__global__ void k_canon_flags(const int32_t *__restrict__ src, const int32_t *__restrict__ adj,
                              int64_t m2, uint8_t *__restrict__ flag) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < m2;
         s += (int64_t)gridDim.x * blockDim.x)
        flag[s] = src[s] < adj[s];
}
__global__ void k_fill_edges(const int64_t *__restrict__ cslot, int64_t me,
                             const int32_t *__restrict__ src, const int32_t *__restrict__ adj,
                             const int32_t *__restrict__ hash, const int32_t *__restrict__ thr,
                             int2 *__restrict__ E, int32_t *__restrict__ EH,
                             int32_t *__restrict__ ET) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < me;
         e += (int64_t)gridDim.x * blockDim.x) {
        int64_t s = cslot[e];
        E[e] = make_int2(src[s], adj[s]);
        EH[e] = hash[s];
        ET[e] = thr[s];
    }
}

// sorted-index construction --------------------------------------------------
__global__ void k_iota_thr_keys(const int32_t *__restrict__ ET, int64_t me, uint32_t *__restrict__ keys,
                                uint32_t *__restrict__ vals) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < me;
         e += (int64_t)gridDim.x * blockDim.x) {
        keys[e] = (uint32_t)ET[e];
        vals[e] = (uint32_t)e;
    }
}
// position p of the threshold-sorted order -> bucket p*nb/me; key = bucket<<32 | hash
__global__ void k_bucket_hash_keys(const uint32_t *__restrict__ by_thr, int64_t me, int nb,
                                   const int32_t *__restrict__ EH, uint64_t *__restrict__ keys,
                                   uint32_t *__restrict__ vals) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < me;
         p += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t e = by_thr ? by_thr[p] : (uint32_t)p;
        const uint64_t b = (uint64_t)((p * nb) / me);
        keys[p] = (b << 32) | (uint32_t)EH[e];
        vals[p] = e;
    }
}
__global__ void k_permute_edges(const uint32_t *__restrict__ perm, int64_t me,
                                const int2 *__restrict__ E0, const int32_t *__restrict__ EH0,
                                const int32_t *__restrict__ ET0, int2 *__restrict__ E,
                                int32_t *__restrict__ EH, int32_t *__restrict__ ET) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < me;
         j += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t e = perm[j];
        E[j] = E0[e];
        EH[j] = EH0[e];
        ET[j] = ET0[e];
    }
}
// bucket offsets from the sorted keys; per-bucket max threshold
__global__ void k_bucket_meta(const uint64_t *__restrict__ keys, int64_t me, int nb,
                              const int32_t *__restrict__ ET, int64_t *__restrict__ boff,
                              int32_t *__restrict__ btmax) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < me;
         j += (int64_t)gridDim.x * blockDim.x) {
        const int b = (int)(keys[j] >> 32);
        const int bp = j ? (int)(keys[j - 1] >> 32) : -1;
        for (int q = bp + 1; q <= b; ++q) boff[q] = j;
        if (j == me - 1)
            for (int q = b + 1; q <= nb; ++q) boff[q] = me;
        atomicMax(btmax + b, ET[j]);
    }
}

// number of neighbours smaller than v = lower_bound(row v, v) - xadj[v]
__global__ void k_max_prefix(const int64_t *__restrict__ xadj, const int32_t *__restrict__ adj, int64_t n,
                             unsigned long long *__restrict__ out) {
    unsigned long long best = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = xadj[v], hi = xadj[v + 1];
        const int64_t s0 = lo;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (adj[mid] < v) lo = mid + 1; else hi = mid;
        }
        const unsigned long long k = (unsigned long long)(lo - s0);
        best = k > best ? k : best;
    }
    for (int o = 16; o; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(0xffffffffu, best, o);
        best = y > best ? y : best;
    }
    if ((threadIdx.x & 31) == 0 && best) atomicMax(out, best);
}

__global__ void k_sum_thr(const int32_t *__restrict__ ET, int64_t me, unsigned long long *__restrict__ out) {
    unsigned long long acc = 0;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < me;
         e += (int64_t)gridDim.x * blockDim.x)
        acc += (unsigned long long)(uint32_t)ET[e];
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

__global__ void k_murmur_pairs(const uint32_t *__restrict__ lo, const uint32_t *__restrict__ hi,
                               int64_t cnt, uint32_t *__restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = murmur3_pair(lo[i], hi[i]);
}

// ---------------------------------------------------------------------------
// host helpers
// ---------------------------------------------------------------------------
static int grid_for(int64_t work, int threads = 256) {
    int64_t b = ceil_div(work > 0 ? work : 1, threads);
    if (b > 148 * 32) b = 148 * 32;
    return (int)b;
}

// Every device buffer comes from the stream-ordered pool (pool_alloc, a
// high release threshold), so building/dropping graphs and contexts back to
// back does not pay cudaMalloc/cudaFree each time.
template <class T>
static int dalloc(imx_graph *g, T **p, int64_t count) {
    *p = nullptr;
    if (count <= 0) count = 1;
    IMX_CUDA(pool_alloc((void **)p, sizeof(T) * (size_t)count, g->stream));
    return IMX_OK;
}

void graph_free(imx_graph *g) {
    if (!g) return;
    cudaSetDevice(g->dev);
    void *ptrs[] = {g->xadj, g->adj, g->w, g->src, g->hash, g->thr, g->recip,
                    g->cslot, g->E, g->EH, g->ET, g->btmax, g->boff};
    for (void *p : ptrs) if (p) cudaFreeAsync(p, g->stream);
    if (g->stream) {
        cudaStreamSynchronize(g->stream);
        cudaStreamDestroy(g->stream);
    }
    delete g;
}

static int read_flags(imx_graph *g, unsigned *dflags, unsigned *out) {
    IMX_CUDA(cudaMemcpyAsync(out, dflags, sizeof(unsigned), cudaMemcpyDeviceToHost, g->stream));
    IMX_CUDA(cudaStreamSynchronize(g->stream));
    return IMX_OK;
}

// Derived per-slot data: sources (if missing), reciprocal, hashes, thresholds,
// canonical edge list.
static int graph_finish(imx_graph *g) {
    cudaStream_t st = g->stream;
    const int64_t m2 = g->m2, n = g->n;
    if (!g->src) {
        IMX_TRY(dalloc(g, &g->src, m2));
        if (m2) { k_src_from_xadj<<<grid_for(m2), 256, 0, st>>>(g->xadj, n, m2, g->src); IMX_CHECK_LAUNCH(); }
    }
    IMX_TRY(dalloc(g, &g->hash, m2));
    IMX_TRY(dalloc(g, &g->thr, m2));
    IMX_TRY(dalloc(g, &g->recip, m2));
    unsigned *dflags;
    IMX_CUDA(cudaMallocAsync((void **)&dflags, sizeof(unsigned), st));
    IMX_CUDA(cudaMemsetAsync(dflags, 0, sizeof(unsigned), st));
    if (m2) {
        k_reciprocal<<<grid_for(m2), 256, 0, st>>>(g->xadj, g->adj, g->src, m2, g->recip, dflags); note_launch();
        IMX_CHECK_LAUNCH();
        k_slot_hashes<<<grid_for(m2), 256, 0, st>>>(g->src, g->adj, m2, g->hash); note_launch();
        IMX_CHECK_LAUNCH();
    }
    unsigned flags = 0;
    IMX_TRY(read_flags(g, dflags, &flags));
    g->symmetric = (flags & 8u) == 0 && (m2 % 2 == 0);
    cudaFreeAsync(dflags, st);
    if (m2) {
        unsigned long long *dmax, hmax = 0;
        IMX_CUDA(cudaMallocAsync((void **)&dmax, sizeof(unsigned long long), st));
        IMX_CUDA(cudaMemsetAsync(dmax, 0, sizeof(unsigned long long), st));
        k_max_prefix<<<grid_for(n), 256, 0, st>>>(g->xadj, g->adj, n, dmax); note_launch();
        IMX_CHECK_LAUNCH();
        IMX_CUDA(cudaMemcpyAsync(&hmax, dmax, sizeof hmax, cudaMemcpyDeviceToHost, st));
        IMX_CUDA(cudaStreamSynchronize(st));
        cudaFreeAsync(dmax, st);
        g->max_prefix = (int64_t)hmax;
    }
    // canonical edge list
    g->me = 0;
    if (m2) {
        uint8_t *flag;
        int64_t *cslot, *dcount;
        IMX_CUDA(cudaMallocAsync((void **)&flag, m2, st));
        IMX_CUDA(pool_alloc((void **)&cslot, sizeof(int64_t) * m2, st));
        IMX_CUDA(cudaMallocAsync((void **)&dcount, sizeof(int64_t), st));
        k_canon_flags<<<grid_for(m2), 256, 0, st>>>(g->src, g->adj, m2, flag); note_launch();
        IMX_CHECK_LAUNCH();
        size_t tmp_bytes = 0;
        thrust::counting_iterator<int64_t> it(0);
        IMX_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp_bytes, it, flag, cslot, dcount, m2, st));
        void *tmp;
        IMX_CUDA(cudaMallocAsync(&tmp, tmp_bytes, st));
        IMX_CUDA(cub::DeviceSelect::Flagged(tmp, tmp_bytes, it, flag, cslot, dcount, m2, st));
        int64_t me = 0;
        IMX_CUDA(cudaMemcpyAsync(&me, dcount, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        IMX_CUDA(cudaStreamSynchronize(st));
        g->me = me;
        IMX_TRY(dalloc(g, &g->E, me));
        IMX_TRY(dalloc(g, &g->EH, me));
        IMX_TRY(dalloc(g, &g->ET, me));
        g->cslot = cslot;
        cudaFreeAsync(tmp, st);
        cudaFreeAsync(flag, st);
        cudaFreeAsync(dcount, st);
    }
    return IMX_OK;
}

// Sort the undirected edges by (threshold bucket, hash) so the sampler can
// enumerate the edges live in a lane as at most 31 hash intervals per bucket
// (the reference's index sweep, propagation.py:104-163, on the device).
static int graph_build_index(imx_graph *g) {
    cudaStream_t st = g->stream;
    const int64_t me = g->me;
    const int nb = g->uniform ? 1 : (int)std::min<int64_t>(64, std::max<int64_t>(1, me));
    if (g->btmax) { cudaFreeAsync(g->btmax, st); g->btmax = nullptr; }
    if (g->boff) { cudaFreeAsync(g->boff, st); g->boff = nullptr; }
    g->nb = nb;
    IMX_CUDA(pool_alloc((void **)&g->btmax, sizeof(int32_t) * nb, st));
    IMX_CUDA(pool_alloc((void **)&g->boff, sizeof(int64_t) * (nb + 1), st));
    IMX_CUDA(cudaMemsetAsync(g->btmax, 0, sizeof(int32_t) * nb, st));
    IMX_CUDA(cudaMemsetAsync(g->boff, 0, sizeof(int64_t) * (nb + 1), st));
    if (me == 0) return IMX_OK;
    uint32_t *k32 = nullptr, *k32b = nullptr, *v32 = nullptr, *v32b = nullptr;
    uint64_t *k64 = nullptr, *k64b = nullptr;
    int2 *E0 = nullptr;
    int32_t *EH0 = nullptr, *ET0 = nullptr;
    void *tmp = nullptr;
    size_t tb = 0, tb2 = 0;
    int rc = IMX_OK;
#define GI(call) do { cudaError_t _e = (call); if (_e != cudaSuccess) { rc = cuda_fail(_e, #call, __FILE__, __LINE__); goto done; } } while (0)
    GI(cudaMallocAsync((void **)&v32, sizeof(uint32_t) * me, st));
    GI(cudaMallocAsync((void **)&v32b, sizeof(uint32_t) * me, st));
    GI(cudaMallocAsync((void **)&k64, sizeof(uint64_t) * me, st));
    GI(cudaMallocAsync((void **)&k64b, sizeof(uint64_t) * me, st));
    GI(cub::DeviceRadixSort::SortPairs(nullptr, tb, k64, k64b, v32, v32b, me, 0, 64, st));
    if (nb > 1) {
        GI(cudaMallocAsync((void **)&k32, sizeof(uint32_t) * me, st));
        GI(cudaMallocAsync((void **)&k32b, sizeof(uint32_t) * me, st));
        GI(cub::DeviceRadixSort::SortPairs(nullptr, tb2, k32, k32b, v32, v32b, me, 0, 32, st));
    }
    GI(cudaMallocAsync(&tmp, std::max(tb, tb2), st));
    if (nb > 1) {
        k_iota_thr_keys<<<grid_for(me), 256, 0, st>>>(g->ET, me, k32, v32); note_launch();
        GI(cudaGetLastError());
        GI(cub::DeviceRadixSort::SortPairs(tmp, tb2, k32, k32b, v32, v32b, me, 0, 32, st));
        k_bucket_hash_keys<<<grid_for(me), 256, 0, st>>>(v32b, me, nb, g->EH, k64, v32); note_launch();
    } else {
        k_bucket_hash_keys<<<grid_for(me), 256, 0, st>>>(nullptr, me, 1, g->EH, k64, v32); note_launch();
    }
    GI(cudaGetLastError());
    GI(cub::DeviceRadixSort::SortPairs(tmp, tb, k64, k64b, v32, v32b, me, 0, 40, st));
    GI(cudaMallocAsync((void **)&E0, sizeof(int2) * me, st));
    GI(cudaMallocAsync((void **)&EH0, sizeof(int32_t) * me, st));
    GI(cudaMallocAsync((void **)&ET0, sizeof(int32_t) * me, st));
    GI(cudaMemcpyAsync(E0, g->E, sizeof(int2) * me, cudaMemcpyDeviceToDevice, st));
    GI(cudaMemcpyAsync(EH0, g->EH, sizeof(int32_t) * me, cudaMemcpyDeviceToDevice, st));
    GI(cudaMemcpyAsync(ET0, g->ET, sizeof(int32_t) * me, cudaMemcpyDeviceToDevice, st));
    k_permute_edges<<<grid_for(me), 256, 0, st>>>(v32b, me, E0, EH0, ET0, g->E, g->EH, g->ET); note_launch();
    GI(cudaGetLastError());
    k_bucket_meta<<<grid_for(me), 256, 0, st>>>(k64b, me, nb, g->ET, g->boff, g->btmax); note_launch();
    GI(cudaGetLastError());
    {
        unsigned long long *dsum = reinterpret_cast<unsigned long long *>(k64);   // reuse scratch
        GI(cudaMemsetAsync(dsum, 0, sizeof(unsigned long long), st));
        k_sum_thr<<<grid_for(me), 256, 0, st>>>(g->ET, me, dsum); note_launch();
        unsigned long long hs = 0;
        GI(cudaMemcpyAsync(&hs, dsum, sizeof hs, cudaMemcpyDeviceToHost, st));
        GI(cudaStreamSynchronize(st));
        g->thr_mean = (double)hs / (double)me / 2147483647.0;
    }
done:
    for (void *p : {(void *)k32, (void *)k32b, (void *)v32, (void *)v32b, (void *)k64, (void *)k64b,
                    (void *)E0, (void *)EH0, (void *)ET0, tmp})
        if (p) cudaFreeAsync(p, st);
#undef GI
    return rc;
}

// thresholds from current weights (symmetrized over reciprocal slots when the
// graph is symmetric) and refresh the edge list's hash/thr columns
static int graph_refresh_thresholds(imx_graph *g) {
    cudaStream_t st = g->stream;
    const int64_t m2 = g->m2;
    g->uniform = 1;
    g->thr_u = 0;
    if (m2) {
        int32_t *mm;
        IMX_CUDA(cudaMallocAsync((void **)&mm, 2 * sizeof(int32_t), st));
        int32_t init[2] = {INT32_MAX, INT32_MIN};
        IMX_CUDA(cudaMemcpyAsync(mm, init, sizeof init, cudaMemcpyHostToDevice, st));
        k_thresholds<<<grid_for(m2), 256, 0, st>>>(g->w, g->symmetric ? g->recip : nullptr, m2,
                                                   g->thr, mm, mm + 1); note_launch();
        IMX_CHECK_LAUNCH();
        int32_t res[2];
        IMX_CUDA(cudaMemcpyAsync(res, mm, sizeof res, cudaMemcpyDeviceToHost, st));
        IMX_CUDA(cudaStreamSynchronize(st));
        cudaFreeAsync(mm, st);
        g->uniform = res[0] == res[1];
        g->thr_u = res[0];
    }
    if (g->me) {
        k_fill_edges<<<grid_for(g->me), 256, 0, st>>>(g->cslot, g->me, g->src, g->adj, g->hash,
                                                      g->thr, g->E, g->EH, g->ET); note_launch();
        IMX_CHECK_LAUNCH();
    }
    IMX_TRY(graph_build_index(g));
    IMX_CUDA(cudaStreamSynchronize(st));
    return IMX_OK;
}

static int graph_new(int32_t device, int64_t n, int64_t m2, imx_graph **out) {
    IMX_TRY(select_device(device));
    imx_graph *g = new imx_graph();
    g->dev = device;
    g->n = n;
    g->m2 = m2;
    if (cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete g;
        set_error("cudaStreamCreate failed");
        return IMX_ECUDA;
    }
    *out = g;
    return IMX_OK;
}

}  // namespace imx

using namespace imx;

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" const char *imx_last_error(void) { return g_err.c_str(); }
extern "C" int imx_version(void) { return 10000; }
extern "C" int64_t imx_launch_count(void) { return g_launches.load(); }

extern "C" int imx_device_count(void) {
    int cnt = 0;
    if (cudaGetDeviceCount(&cnt) != cudaSuccess) { cudaGetLastError(); return 0; }
    int ok = 0;
    for (int d = 0; d < cnt; ++d) {
        cudaDeviceProp p;
        if (cudaGetDeviceProperties(&p, d) == cudaSuccess && p.major == 10) ++ok;
    }
    return ok;
}

namespace imx {

// CSR from k undirected edges already on the device (dedges: 2k int64,
// pairs (u, v)); dw: per-edge weights on the device or NULL (w_scalar).
int graph_build_from_device_edges(imx_graph *g, const int64_t *dedges, int64_t k, const double *dw,
                                  double w_scalar) {
    cudaStream_t st = g->stream;
    const int64_t n = g->n, m2 = 2 * k;
    int rc = IMX_OK;
    if (dalloc(g, &g->xadj, n + 1) || dalloc(g, &g->adj, m2) || dalloc(g, &g->w, m2) || dalloc(g, &g->src, m2))
        return IMX_ENOMEM;
    if (k > 0) {
        int nb = 1;
        while ((int64_t(1) << nb) < n) ++nb;
        uint64_t *keys = nullptr, *keys2 = nullptr;
        uint32_t *vals = nullptr, *vals2 = nullptr;
        unsigned *dflags = nullptr;
        void *tmp = nullptr;
        size_t tmp_bytes = 0;
#define GF(call) do { cudaError_t _e = (call); if (_e != cudaSuccess) { rc = cuda_fail(_e, #call, __FILE__, __LINE__); goto cleanup; } } while (0)
        GF(cudaMallocAsync((void **)&keys, sizeof(uint64_t) * m2, st));
        GF(cudaMallocAsync((void **)&keys2, sizeof(uint64_t) * m2, st));
        GF(cudaMallocAsync((void **)&vals, sizeof(uint32_t) * m2, st));
        GF(cudaMallocAsync((void **)&vals2, sizeof(uint32_t) * m2, st));
        GF(cudaMallocAsync((void **)&dflags, sizeof(unsigned), st));
        GF(cudaMemsetAsync(dflags, 0, sizeof(unsigned), st));
        k_edges_check_and_keys<<<grid_for(k), 256, 0, st>>>(dedges, k, n, nb, keys, vals, dflags); note_launch();
        GF(cudaGetLastError());
        GF(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys2, vals, vals2, m2, 0, 2 * nb, st));
        GF(cudaMallocAsync(&tmp, tmp_bytes, st));
        GF(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys2, vals, vals2, m2, 0, 2 * nb, st));
        k_csr_from_sorted<<<grid_for(m2), 256, 0, st>>>(keys2, vals2, m2, nb, dw, w_scalar, g->adj,
                                                        g->src, g->w, dflags); note_launch();
        GF(cudaGetLastError());
        k_xadj_from_src<<<grid_for(n + 1), 256, 0, st>>>(g->src, m2, n, g->xadj); note_launch();
        GF(cudaGetLastError());
        {
            unsigned flags = 0;
            GF(cudaMemcpyAsync(&flags, dflags, sizeof flags, cudaMemcpyDeviceToHost, st));
            GF(cudaStreamSynchronize(st));
            // graph.py:137-146 check order: range, self-loop, duplicates
            if (flags & 1u) { set_error("edge endpoint outside 0..n-1"); rc = IMX_EINVAL; }
            else if (flags & 2u) { set_error("self-loops are not allowed"); rc = IMX_EINVAL; }
            else if (flags & 4u) { set_error("duplicate undirected edges"); rc = IMX_EINVAL; }
        }
    cleanup:
        if (keys) cudaFreeAsync(keys, st); if (keys2) cudaFreeAsync(keys2, st);
        if (vals) cudaFreeAsync(vals, st); if (vals2) cudaFreeAsync(vals2, st);
        if (dflags) cudaFreeAsync(dflags, st); if (tmp) cudaFreeAsync(tmp, st);
#undef GF
        if (rc != IMX_OK) return rc;
    } else {
        IMX_CUDA(cudaMemsetAsync(g->xadj, 0, sizeof(int64_t) * (n + 1), st));
    }
    IMX_TRY(graph_finish(g));
    return graph_refresh_thresholds(g);
}

int graph_create(int32_t device, int64_t n, int64_t m2, imx_graph **out) { return graph_new(device, n, m2, out); }

}  // namespace imx

extern "C" int imx_graph_from_edges(int32_t device, int64_t n, const int64_t *edges, int64_t k,
                                    const double *w_edge, double w_scalar, imx_graph **out) {
    if (!out) { set_error("out is NULL"); return IMX_EINVAL; }
    *out = nullptr;
    if (n < 0 || n >= (int64_t(1) << 31)) {
        set_error("vertex count %lld outside [0, 2^31)", (long long)n);
        return IMX_ECONSTRAINT;
    }
    if (k < 0 || k >= (int64_t(1) << 31)) { set_error("edge count %lld invalid", (long long)k); return IMX_EINVAL; }
    if (k > 0 && !edges) { set_error("edges is NULL"); return IMX_EINVAL; }
    imx_graph *g;
    IMX_TRY(graph_new(device, n, 2 * k, &g));
    cudaStream_t st = g->stream;
    int64_t *dedges = nullptr;
    double *dw = nullptr;
    int rc = IMX_OK;
    cudaError_t e = cudaSuccess;
    if (k > 0) {
        if ((e = cudaMallocAsync((void **)&dedges, sizeof(int64_t) * 2 * k, st)) == cudaSuccess)
            e = cudaMemcpyAsync(dedges, edges, sizeof(int64_t) * 2 * k, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess && w_edge) {
            if ((e = cudaMallocAsync((void **)&dw, sizeof(double) * k, st)) == cudaSuccess)
                e = cudaMemcpyAsync(dw, w_edge, sizeof(double) * k, cudaMemcpyHostToDevice, st);
        }
    }
    rc = e == cudaSuccess ? graph_build_from_device_edges(g, dedges, k, dw, w_scalar)
                          : cuda_fail(e, "upload edges", __FILE__, __LINE__);
    if (dedges) cudaFreeAsync(dedges, st);
    if (dw) cudaFreeAsync(dw, st);
    if (rc != IMX_OK) { graph_free(g); return rc; }
    *out = g;
    return IMX_OK;
}

extern "C" int imx_graph_from_csr(int32_t device, int64_t n, int64_t m2, const int64_t *xadj,
                                  const int32_t *adj, const double *weights, imx_graph **out) {
    if (!out || !xadj || (m2 && (!adj || !weights))) { set_error("NULL argument"); return IMX_EINVAL; }
    *out = nullptr;
    if (n < 0 || n >= (int64_t(1) << 31)) { set_error("vertex count %lld outside [0, 2^31)", (long long)n); return IMX_ECONSTRAINT; }
    if (xadj[0] != 0 || xadj[n] != m2) { set_error("corrupt CSR offsets"); return IMX_EINVAL; }
    for (int64_t v = 0; v < n; ++v)
        if (xadj[v + 1] < xadj[v]) { set_error("corrupt CSR offsets"); return IMX_EINVAL; }
    imx_graph *g;
    IMX_TRY(graph_new(device, n, m2, &g));
    cudaStream_t st = g->stream;
    auto fail = [&](int code) { graph_free(g); return code; };
    if (dalloc(g, &g->xadj, n + 1) || dalloc(g, &g->adj, m2) || dalloc(g, &g->w, m2)) return fail(IMX_ENOMEM);
    if (cudaMemcpyAsync(g->xadj, xadj, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, st) != cudaSuccess ||
        (m2 && cudaMemcpyAsync(g->adj, adj, sizeof(int32_t) * m2, cudaMemcpyHostToDevice, st) != cudaSuccess) ||
        (m2 && cudaMemcpyAsync(g->w, weights, sizeof(double) * m2, cudaMemcpyHostToDevice, st) != cudaSuccess))
        return fail(cuda_fail(cudaGetLastError(), "upload csr", __FILE__, __LINE__));
    int rc = graph_finish(g);
    if (rc == IMX_OK) rc = graph_refresh_thresholds(g);
    if (rc != IMX_OK) return fail(rc);
    *out = g;
    return IMX_OK;
}

extern "C" void imx_graph_destroy(imx_graph *g) { graph_free(g); }

extern "C" int imx_graph_dims(const imx_graph *g, int64_t *n, int64_t *m2) {
    if (!g) { set_error("graph is NULL"); return IMX_EINVAL; }
    if (n) *n = g->n;
    if (m2) *m2 = g->m2;
    return IMX_OK;
}

extern "C" int imx_graph_get_csr(imx_graph *g, int64_t *xadj, int32_t *adj, double *weights) {
    if (!g) { set_error("graph is NULL"); return IMX_EINVAL; }
    IMX_CUDA(cudaSetDevice(g->dev));
    cudaStream_t st = g->stream;
    if (xadj) IMX_CUDA(cudaMemcpyAsync(xadj, g->xadj, sizeof(int64_t) * (g->n + 1), cudaMemcpyDeviceToHost, st));
    if (adj && g->m2) IMX_CUDA(cudaMemcpyAsync(adj, g->adj, sizeof(int32_t) * g->m2, cudaMemcpyDeviceToHost, st));
    if (weights && g->m2) IMX_CUDA(cudaMemcpyAsync(weights, g->w, sizeof(double) * g->m2, cudaMemcpyDeviceToHost, st));
    IMX_CUDA(cudaStreamSynchronize(st));
    return IMX_OK;
}

extern "C" int imx_graph_reciprocal(imx_graph *g, int64_t *recip) {
    if (!g || (!recip && g->m2)) { set_error("NULL argument"); return IMX_EINVAL; }
    if (!g->symmetric) { set_error("adjacency is not symmetric"); return IMX_EFORMAT; }
    IMX_CUDA(cudaSetDevice(g->dev));
    if (g->m2) {
        IMX_CUDA(cudaMemcpyAsync(recip, g->recip, sizeof(int64_t) * g->m2, cudaMemcpyDeviceToHost, g->stream));
        IMX_CUDA(cudaStreamSynchronize(g->stream));
    }
    return IMX_OK;
}

extern "C" int imx_graph_set_weights(imx_graph *g, const double *weights) {
    if (!g || (!weights && g->m2)) { set_error("NULL argument"); return IMX_EINVAL; }
    IMX_CUDA(cudaSetDevice(g->dev));
    cudaStream_t st = g->stream;
    if (g->m2) {
        double *tmp;
        IMX_CUDA(cudaMallocAsync((void **)&tmp, sizeof(double) * g->m2, st));
        IMX_CUDA(cudaMemcpyAsync(tmp, weights, sizeof(double) * g->m2, cudaMemcpyHostToDevice, st));
        unsigned *dflags;
        IMX_CUDA(cudaMallocAsync((void **)&dflags, sizeof(unsigned), st));
        IMX_CUDA(cudaMemsetAsync(dflags, 0, sizeof(unsigned), st));
        k_weights_range<<<grid_for(g->m2), 256, 0, st>>>(tmp, g->m2, dflags); note_launch();
        IMX_CHECK_LAUNCH();
        unsigned flags = 0;
        IMX_TRY(read_flags(g, dflags, &flags));
        cudaFreeAsync(dflags, st);
        if (flags & 16u) {
            cudaFreeAsync(tmp, st);
            set_error("weights must lie in [0, 1]");
            return IMX_ECONSTRAINT;
        }
        IMX_CUDA(cudaMemcpyAsync(g->w, tmp, sizeof(double) * g->m2, cudaMemcpyDeviceToDevice, st));
        cudaFreeAsync(tmp, st);
    }
    return graph_refresh_thresholds(g);
}

extern "C" int imx_graph_hashes(imx_graph *g, int32_t *out) {
    if (!g || (!out && g->m2)) { set_error("NULL argument"); return IMX_EINVAL; }
    IMX_CUDA(cudaSetDevice(g->dev));
    if (g->m2) {
        IMX_CUDA(cudaMemcpyAsync(out, g->hash, sizeof(int32_t) * g->m2, cudaMemcpyDeviceToHost, g->stream));
        IMX_CUDA(cudaStreamSynchronize(g->stream));
    }
    return IMX_OK;
}

extern "C" int imx_graph_set_hashes(imx_graph *g, const int32_t *hashes) {
    if (!g) { set_error("NULL argument"); return IMX_EINVAL; }
    IMX_CUDA(cudaSetDevice(g->dev));
    if (g->m2) {
        if (hashes) {
            IMX_CUDA(cudaMemcpyAsync(g->hash, hashes, sizeof(int32_t) * g->m2, cudaMemcpyHostToDevice, g->stream));
        } else {
            k_slot_hashes<<<grid_for(g->m2), 256, 0, g->stream>>>(g->src, g->adj, g->m2, g->hash); note_launch();
            IMX_CHECK_LAUNCH();
        }
    }
    return graph_refresh_thresholds(g);
}

extern "C" int imx_graph_thresholds(imx_graph *g, int32_t symmetrize, int32_t *thr_out,
                                    int32_t *uniform_out) {
    if (!g || (!thr_out && g->m2)) { set_error("NULL argument"); return IMX_EINVAL; }
    IMX_CUDA(cudaSetDevice(g->dev));
    cudaStream_t st = g->stream;
    if (symmetrize && !g->symmetric) { set_error("adjacency is not symmetric"); return IMX_EFORMAT; }
    if (g->m2) {
        if (symmetrize) {
            IMX_CUDA(cudaMemcpyAsync(thr_out, g->thr, sizeof(int32_t) * g->m2, cudaMemcpyDeviceToHost, st));
        } else {
            int32_t *tmp, *mm;
            IMX_CUDA(cudaMallocAsync((void **)&tmp, sizeof(int32_t) * g->m2, st));
            IMX_CUDA(cudaMallocAsync((void **)&mm, 2 * sizeof(int32_t), st));
            int32_t init[2] = {INT32_MAX, INT32_MIN};
            IMX_CUDA(cudaMemcpyAsync(mm, init, sizeof init, cudaMemcpyHostToDevice, st));
            k_thresholds<<<grid_for(g->m2), 256, 0, st>>>(g->w, nullptr, g->m2, tmp, mm, mm + 1); note_launch();
            IMX_CHECK_LAUNCH();
            IMX_CUDA(cudaMemcpyAsync(thr_out, tmp, sizeof(int32_t) * g->m2, cudaMemcpyDeviceToHost, st));
            cudaFreeAsync(tmp, st);
            cudaFreeAsync(mm, st);
        }
        IMX_CUDA(cudaStreamSynchronize(st));
    }
    if (uniform_out) *uniform_out = g->uniform;
    return IMX_OK;
}

extern "C" int imx_murmur3_pairs(int32_t device, const uint32_t *lo, const uint32_t *hi,
                                 int64_t count, uint32_t *out) {
    if (count < 0 || (count && (!lo || !hi || !out))) { set_error("bad arguments"); return IMX_EINVAL; }
    IMX_TRY(select_device(device));
    if (!count) return IMX_OK;
    uint32_t *d;
    IMX_CUDA(cudaMalloc((void **)&d, sizeof(uint32_t) * 3 * count));
    cudaError_t e = cudaMemcpy(d, lo, sizeof(uint32_t) * count, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d + count, hi, sizeof(uint32_t) * count, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        k_murmur_pairs<<<grid_for(count), 256>>>(d, d + count, count, d + 2 * count); note_launch();
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(out, d + 2 * count, sizeof(uint32_t) * count, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return cuda_fail(e, "murmur3 pairs", __FILE__, __LINE__);
    return IMX_OK;
}
