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
#include <mutex>
#include <cstdarg>
#include <cstring>
#include <vector>
#include <chrono>
#include <functional>
#include <thread>
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "common.cuh"
#include "graph.cuh"

namespace imx {

static thread_local std::string g_err;
static std::atomic<long long> g_launches{0};
void note_launch(int64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

// Non-blocking streams are recycled per device: graphs and contexts are
// often built and dropped back to back (one per run_fused), and creating a
// stream costs tens of microseconds.
static std::mutex g_stream_mu;
static std::vector<std::pair<int, cudaStream_t>> g_streams;
cudaError_t acquire_stream(int dev, cudaStream_t *st) {
    {
        std::lock_guard<std::mutex> lk(g_stream_mu);
        for (size_t i = 0; i < g_streams.size(); ++i)
            if (g_streams[i].first == dev) {
                *st = g_streams[i].second;
                g_streams.erase(g_streams.begin() + i);
                return cudaSuccess;
            }
    }
    return cudaStreamCreateWithFlags(st, cudaStreamNonBlocking);
}
void release_stream(int dev, cudaStream_t st) {
    if (!st) return;
    cudaStreamSynchronize(st);
    std::lock_guard<std::mutex> lk(g_stream_mu);
    if (g_streams.size() < 64) g_streams.emplace_back(dev, st);
    else cudaStreamDestroy(st);
}

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

// src[s] = row of slot s (np.repeat over degrees, graph.py:75-78): one warp
// per vertex writes its row (coalesced, no search)
__global__ void k_src_rows(const int64_t *__restrict__ xadj, int64_t n, int64_t m2, int32_t *__restrict__ src,
                           int64_t v0 = 0) {
    const int lane = threadIdx.x & 31;
    for (int64_t v = v0 + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); v < n;
         v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t a = xadj[v], b = xadj[v + 1];
        if (a < 0 || b > m2 || a > b) continue;      // corrupt offsets: flagged by k_check_xadj
        for (int64_t s = a + lane; s < b; s += 32) src[s] = (int32_t)v;
    }
}

// (binary-search form, kept for callers that only have the offsets)
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

// Reciprocal slots and symmetrized thresholds in one pass.  Only slots with
// u < v search (u in the larger id's row v); each such pair writes both
// directions of recip and of thr = max(thr(w[s]), thr(w[reciprocal])), and
// the threshold statistics.  recip starts at -1; k_recip_check flags slots
// no search reached and duplicate slots.  flags: 8 = a slot without
// reciprocal, 32 = adjacency entry outside 0..n-1, 64 = corrupt offsets.
struct GStats;
__global__ void k_reciprocal(const int64_t *__restrict__ xadj, const int32_t *__restrict__ adj,
                             const int32_t *__restrict__ src, const double *__restrict__ w, int64_t n,
                             int64_t m2, int64_t *__restrict__ recip, int32_t *__restrict__ thr,
                             GStats *__restrict__ gs);
__global__ void k_recip_check(const int64_t *__restrict__ xadj, const int32_t *__restrict__ adj,
                              const int32_t *__restrict__ src, const int64_t *__restrict__ recip,
                              int64_t m2, unsigned *__restrict__ flags) {
    bool bad = false;
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < m2;
         s += (int64_t)gridDim.x * blockDim.x) {
        // unpaired, or a repeated neighbour in a sorted row (it pairs once)
        bad |= recip[s] < 0 || (s > 0 && s > xadj[src[s]] && adj[s] == adj[s - 1]);
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, 8u);
}

// k_sym_check and k_slot_hashes in one pass over the slots (deferred path)
struct GStats;
__global__ void k_sym_hash(const int64_t *__restrict__ xadj, const int32_t *__restrict__ adj,
                           const int32_t *__restrict__ src, int64_t n, int64_t m2, int32_t *__restrict__ hash,
                           GStats *__restrict__ gs, int64_t s0 = 0);

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
// Build statistics gathered by the analysis kernels and read back with ONE
// device->host copy (graph_analyze).
struct GStats {
    unsigned flags;
    int32_t tmin, tmax;
    int32_t pad;
    unsigned long long maxp;   // max #smaller neighbours (k_max_prefix)
    unsigned long long tsum;   // sum of canonical-slot thresholds
    int64_t me;                // canonical slots (DeviceSelect count)
    unsigned long long symsum; // sum of mix(u, v) - mix(v, u) over slots (k_sym_check)
    int64_t nnz;               // non-isolated vertices (graph_nz_rows_async)
};
__global__ void k_stats_init(GStats *gs) {
    gs->flags = 0; gs->tmin = INT32_MAX; gs->tmax = INT32_MIN; gs->pad = 0;
    gs->maxp = 0; gs->tsum = 0; gs->me = 0; gs->symsum = 0; gs->nnz = 0;
}

__global__ void k_sym_hash(const int64_t *__restrict__ xadj, const int32_t *__restrict__ adj,
                           const int32_t *__restrict__ src, int64_t n, int64_t m2, int32_t *__restrict__ hash,
                           GStats *__restrict__ gs, int64_t s0);

// Symmetry of a large host CSR without the reciprocal search (deferred
// path): rows strictly ascending (no duplicate, no self-loop) and the slot
// multiset equal to its transpose, tested as sum(mix(u, v) - mix(v, u)) == 0
// over all slots mod 2^64 (mix = SplitMix64 of the ordered pair).  The exact
// pairing (k_reciprocal) runs later if anything needs it and re-checks.
// flags: 8 = not symmetric / unsorted, 32 = entry outside 0..n-1.
__device__ __forceinline__ unsigned long long pair_mix(uint32_t a, uint32_t b) {
    unsigned long long z = ((unsigned long long)a << 32 | b) + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__global__ void k_sym_check(const int64_t *__restrict__ xadj, const int32_t *__restrict__ adj,
                            const int32_t *__restrict__ src, int64_t n, int64_t m2, GStats *__restrict__ gs) {
    unsigned long long sum = 0;
    unsigned fl = 0;
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < m2;
         s += (int64_t)gridDim.x * blockDim.x) {
        const int32_t u = src[s], v = adj[s];
        if (v < 0 || v >= n) { fl |= 32u | 8u; continue; }
        if (u == v) fl |= 8u;
        if (s > xadj[u] && adj[s - 1] >= v) fl |= 8u;
        sum += pair_mix((uint32_t)u, (uint32_t)v) - pair_mix((uint32_t)v, (uint32_t)u);
    }
    for (int o = 16; o; o >>= 1) {
        sum += __shfl_xor_sync(0xffffffffu, sum, o);
        fl |= __shfl_xor_sync(0xffffffffu, fl, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (sum) atomicAdd(&gs->symsum, sum);
        if (fl) atomicOr(&gs->flags, fl);
    }
}

// slots [s0, m2): a chunk of a streamed CSR passes its own slot range
__global__ void k_sym_hash(const int64_t *__restrict__ xadj, const int32_t *__restrict__ adj,
                           const int32_t *__restrict__ src, int64_t n, int64_t m2, int32_t *__restrict__ hash,
                           GStats *__restrict__ gs, int64_t s0) {
    unsigned long long sum = 0;
    unsigned fl = 0;
    for (int64_t s = s0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < m2;
         s += (int64_t)gridDim.x * blockDim.x) {
        const int32_t u = src[s], v = adj[s];
        hash[s] = edge_hash(u, v);
        if (v < 0 || v >= n) { fl |= 32u | 8u; continue; }
        if (u == v) fl |= 8u;
        if (s > xadj[u] && adj[s - 1] >= v) fl |= 8u;
        sum += pair_mix((uint32_t)u, (uint32_t)v) - pair_mix((uint32_t)v, (uint32_t)u);
    }
    for (int o = 16; o; o >>= 1) {
        sum += __shfl_xor_sync(0xffffffffu, sum, o);
        fl |= __shfl_xor_sync(0xffffffffu, fl, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (sum) atomicAdd(&gs->symsum, sum);
        if (fl) atomicOr(&gs->flags, fl);
    }
}

// thresholds (symmetrized over valid reciprocal slots when recip != NULL),
// their range over all slots and their sum over the canonical slots
__global__ void k_thresholds(const double *__restrict__ w, const int64_t *__restrict__ recip,
                             const int32_t *__restrict__ src, const int32_t *__restrict__ adj,
                             const int32_t *__restrict__ hash, int64_t m2, int32_t *__restrict__ thr,
                             GStats *__restrict__ gs) {
    int32_t lmin = INT32_MAX, lmax = INT32_MIN;
    unsigned long long lsum = 0;
    bool neg = false;
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < m2;
         s += (int64_t)gridDim.x * blockDim.x) {
        int32_t t = thr_of(w[s]);
        if (recip) {
            const int64_t r = recip[s];
            if (r >= 0) { const int32_t t2 = thr_of(w[r]); t = t2 > t ? t2 : t; }
        }
        thr[s] = t;
        lmin = min(lmin, t); lmax = max(lmax, t);
        if (src[s] < adj[s]) lsum += (unsigned long long)(uint32_t)t;
        if (hash && hash[s] < 0) neg = true;     // a caller's table outside 31 bits
    }
    if (__any_sync(0xffffffffu, neg) && (threadIdx.x & 31) == 0) atomicOr(&gs->flags, 128u);
    for (int o = 16; o; o >>= 1) {
        lmin = min(lmin, __shfl_xor_sync(0xffffffffu, lmin, o));
        lmax = max(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
        lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&gs->tmin, lmin);
        atomicMax(&gs->tmax, lmax);
        if (lsum) atomicAdd(&gs->tsum, lsum);
    }
}

// flag 256: some weight's bit pattern differs from w0's (the deferred graph's
// whole check when the weights are uniform: 8 bytes read per slot instead of
// the 28 read and written by k_thresholds)
__global__ void k_weights_same(const double *__restrict__ w, int64_t m2, unsigned long long w0,
                               unsigned *__restrict__ flags) {
    bool diff = false;
    const unsigned long long *wb = reinterpret_cast<const unsigned long long *>(w);
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < m2; s += (int64_t)gridDim.x * blockDim.x)
        diff |= wb[s] != w0;
    if (__any_sync(0xffffffffu, diff) && (threadIdx.x & 31) == 0) atomicOr(flags, 256u);
}
__global__ void k_fill_i32(int32_t *__restrict__ a, int64_t cnt, int32_t v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = v;
}

__global__ void k_reciprocal(const int64_t *__restrict__ xadj, const int32_t *__restrict__ adj,
                             const int32_t *__restrict__ src, const double *__restrict__ w, int64_t n,
                             int64_t m2, int64_t *__restrict__ recip, int32_t *__restrict__ thr,
                             GStats *__restrict__ gs) {
    int32_t lmin = INT32_MAX, lmax = INT32_MIN;
    unsigned long long lsum = 0;
    unsigned fl = 0;
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < m2;
         s += (int64_t)gridDim.x * blockDim.x) {
        const int32_t u = src[s], v = adj[s];
        if (v < 0 || v >= n) { fl |= 32u | 8u; continue; }
        if (u >= v) { if (u == v) fl |= 8u; continue; }          // paired from the other side
        int64_t lo = xadj[v], hi = xadj[v + 1];
        if (lo < 0 || hi > m2 || lo > hi) { fl |= 64u | 8u; continue; }
        const int64_t end = hi;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (adj[mid] < u) lo = mid + 1; else hi = mid;
        }
        if (lo < end && adj[lo] == u) {
            recip[s] = lo;
            recip[lo] = s;
            if (!w) continue;                 // thresholds later (k_thresholds)
            const int32_t t1 = thr_of(w[s]), t2 = thr_of(w[lo]);
            const int32_t t = t1 > t2 ? t1 : t2;
            thr[s] = t;
            thr[lo] = t;
            lmin = min(lmin, t); lmax = max(lmax, t);
            lsum += (unsigned long long)(uint32_t)t;
        } else {
            fl |= 8u;
        }
    }
    for (int o = 16; o; o >>= 1) {
        lmin = min(lmin, __shfl_xor_sync(0xffffffffu, lmin, o));
        lmax = max(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
        lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
        fl |= __shfl_xor_sync(0xffffffffu, fl, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&gs->tmin, lmin);
        atomicMax(&gs->tmax, lmax);
        if (lsum) atomicAdd(&gs->tsum, lsum);
        if (fl) atomicOr(&gs->flags, fl);
    }
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
                             int32_t *__restrict__ ET, uint32_t *__restrict__ iota) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < me;
         e += (int64_t)gridDim.x * blockDim.x) {
        int64_t s = cslot[e];
        E[e] = make_int2(src[s], adj[s]);
        EH[e] = hash[s];
        ET[e] = thr[s];
        iota[e] = (uint32_t)e;
    }
}

// sorted-index construction --------------------------------------------------
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
// one threshold bucket: the sorted keys are the hashes and every threshold
// is thr_u, so only the endpoints are gathered
__global__ void k_permute_uniform(const uint32_t *__restrict__ perm, const uint32_t *__restrict__ keys, int64_t me,
                                  const int2 *__restrict__ E0, int32_t tu, int2 *__restrict__ E,
                                  int32_t *__restrict__ EH, int32_t *__restrict__ ET) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < me;
         j += (int64_t)gridDim.x * blockDim.x) {
        E[j] = E0[perm[j]];
        EH[j] = (int32_t)keys[j];
        ET[j] = tu;
    }
}
// bucket offsets from the sorted keys; per-bucket max threshold (reduced
// per warp over equal buckets first: the keys are sorted, so a warp sees one
// or two buckets and the atomics do not pile up on 64 addresses)
__global__ void k_bucket_meta(const uint64_t *__restrict__ keys, int64_t me, int nb,
                              const int32_t *__restrict__ ET, int64_t *__restrict__ boff,
                              int32_t *__restrict__ btmax) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j0 = blockIdx.x * (int64_t)blockDim.x; j0 < me; j0 += stride) {
        const int64_t j = j0 + threadIdx.x;
        const bool in = j < me;
        const int b = in ? (int)(keys[j] >> 32) : -1;
        if (in) {
            const int bp = j ? (int)(keys[j - 1] >> 32) : -1;
            for (int q = bp + 1; q <= b; ++q) boff[q] = j;
            if (j == me - 1)
                for (int q = b + 1; q <= nb; ++q) boff[q] = me;
        }
        const unsigned peers = __match_any_sync(0xffffffffu, b);
        const int t = in ? ET[j] : INT32_MIN;
        const int m = __reduce_max_sync(peers, t);
        if (in && (threadIdx.x & 31) == __ffs(peers) - 1) atomicMax(btmax + b, m);
    }
}

__global__ void k_uniform_meta(int64_t me, int32_t thr, int64_t *__restrict__ boff, int32_t *__restrict__ btmax) {
    boff[0] = 0;
    boff[1] = me;
    btmax[0] = thr;
}

// lut[b][k] = lower_bound of (k << shift) among bucket b's sorted hashes
__global__ void k_build_lut(const int32_t *__restrict__ EH, const int64_t *__restrict__ boff, int nb, int bits,
                            int32_t *__restrict__ lut) {
    const int64_t per = ((int64_t)1 << bits) + 1;
    const int shift = 31 - bits;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nb * per;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int b = (int)(i / per);
        const int64_t k = i - b * per;
        const uint64_t key = (uint64_t)k << shift;
        int64_t lo = boff[b], hi = boff[b + 1];
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((uint64_t)(uint32_t)EH[mid] < key) lo = mid + 1; else hi = mid;
        }
        lut[i] = (int32_t)lo;
    }
}

// CSR offsets must be non-decreasing within [0, m2] (flag 64)
__global__ void k_check_xadj(const int64_t *__restrict__ xadj, int64_t n, int64_t m2, unsigned *__restrict__ flags) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x)
        if (xadj[v] < 0 || xadj[v + 1] > m2 || xadj[v + 1] < xadj[v]) atomicOr(flags, 64u);
}

// number of neighbours smaller than v = lower_bound(row v, v) - xadj[v]
__global__ void k_max_prefix(const int64_t *__restrict__ xadj, const int32_t *__restrict__ adj, int64_t n,
                             int64_t m2, unsigned long long *__restrict__ out, int64_t v0 = 0) {
    unsigned long long best = 0;
    for (int64_t v = v0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = xadj[v], hi = xadj[v + 1];
        if (lo < 0 || hi > m2 || lo > hi) continue;     // corrupt offsets: flagged by k_check_xadj
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

__global__ void k_murmur_pairs(const uint32_t *__restrict__ lo, const uint32_t *__restrict__ hi,
                               int64_t cnt, uint32_t *__restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = murmur3_pair(lo[i], hi[i]);
}

// ---------------------------------------------------------------------------
// host helpers
// ---------------------------------------------------------------------------
// IMX_GRAPH_PROFILE=1: host wall time of each graph-build phase (stream
// synchronised at every mark, so the marks themselves add syncs)
struct PhaseClock {
    bool on = false;
    std::chrono::steady_clock::time_point t;
    void start() {
        on = getenv("IMX_GRAPH_PROFILE") != nullptr;
        t = std::chrono::steady_clock::now();
    }
    void mark(const char *what, cudaStream_t st) {
        if (!on) return;
        cudaStreamSynchronize(st);
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[graph] %-22s %8.1f us\n", what,
                std::chrono::duration<double, std::micro>(now - t).count());
        t = now;
    }
};
static PhaseClock g_clock;

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
    if (g->struct_pending) graph_settle_structure(g);   // waits for the chunk uploads
    if (g->thr_pending) graph_settle(g);    // joins the weight upload
    // leftovers of a streamed build that failed half way
    if (g->ust) { cudaStreamSynchronize(g->ust); release_stream(g->dev, g->ust); g->ust = nullptr; }
    for (auto &e : g->chunk_ev) if (e) { cudaEventDestroy(e); e = nullptr; }
    if (g->sev_done) { cudaEventDestroy(g->sev_done); g->sev_done = nullptr; }
    if (g->sstats_h) { cudaStreamSynchronize(g->stream); pinned_put(g->sstats_h, sizeof(GStats)); g->sstats_h = nullptr; }
    if (g->sstats_d) { cudaFreeAsync(g->sstats_d, g->stream); g->sstats_d = nullptr; }
    void *ptrs[] = {g->hv[0].pre, g->hv[0].nsl, g->hv[0].off, g->hv[1].pre, g->hv[1].nsl, g->hv[1].off, g->xadj, g->adj, g->w, g->src, g->hash, g->thr, g->recip, g->nz_rows,
                    g->cslot, g->E, g->EH, g->ET, g->btmax, g->boff, g->lut,
                    g->hv[0].heavy, g->hv[0].hs_v, g->hv[0].hs_a, g->hv[0].hs_len,
                    g->hv[1].heavy, g->hv[1].hs_v, g->hv[1].hs_a, g->hv[1].hs_len};
    for (void *p : ptrs) if (p) cudaFreeAsync(p, g->stream);
    release_stream(g->dev, g->stream);
    delete g;
}

// Sort the undirected edges by (threshold bucket, hash) so the sampler can
// enumerate the edges live in a lane as at most 31 hash intervals per bucket
// (the reference's index sweep, propagation.py:104-163, on the device).
// Stream-ordered, no host synchronisation.
static int graph_build_index(imx_graph *g) {
    IMX_TRY(ensure_thr(g));
    cudaStream_t st = g->stream;
    const int64_t me = g->me;
    const int nb = g->uniform ? 1 : (int)std::min<int64_t>(64, std::max<int64_t>(1, me));
    if (g->btmax) { cudaFreeAsync(g->btmax, st); g->btmax = nullptr; }
    if (g->boff) { cudaFreeAsync(g->boff, st); g->boff = nullptr; }
    if (g->lut) { cudaFreeAsync(g->lut, st); g->lut = nullptr; }
    g->nb = nb;
    if (!g->E) {
        IMX_CUDA(pool_alloc((void **)&g->E, sizeof(int2) * std::max<int64_t>(1, me), st));
        IMX_CUDA(pool_alloc((void **)&g->EH, sizeof(int32_t) * std::max<int64_t>(1, me), st));
        IMX_CUDA(pool_alloc((void **)&g->ET, sizeof(int32_t) * std::max<int64_t>(1, me), st));
    }
    int bits = 6;
    while (bits < 16 && ((int64_t)1 << (bits + 1)) <= me / nb) ++bits;
    g->lut_bits = bits;
    const int64_t lut_n = (int64_t)nb * (((int64_t)1 << bits) + 1);
    IMX_CUDA(pool_alloc((void **)&g->btmax, sizeof(int32_t) * nb, st));
    IMX_CUDA(pool_alloc((void **)&g->boff, sizeof(int64_t) * (nb + 1), st));
    IMX_CUDA(pool_alloc((void **)&g->lut, sizeof(int32_t) * lut_n, st));
    if (me == 0) {
        IMX_CUDA(cudaMemsetAsync(g->btmax, 0, sizeof(int32_t) * nb, st));
        IMX_CUDA(cudaMemsetAsync(g->boff, 0, sizeof(int64_t) * (nb + 1), st));
        IMX_CUDA(cudaMemsetAsync(g->lut, 0, sizeof(int32_t) * lut_n, st));
        return IMX_OK;
    }
    uint32_t *k32b = nullptr, *v32 = nullptr, *v32b = nullptr, *v32c = nullptr;
    uint64_t *k64 = nullptr, *k64b = nullptr;
    int2 *E0 = nullptr;
    int32_t *EH0 = nullptr, *ET0 = nullptr;
    void *tmp = nullptr;
    size_t tb = 0;
    int rc = IMX_OK;
#define GI(call) do { cudaError_t _e = (call); if (_e != cudaSuccess) { rc = cuda_fail(_e, #call, __FILE__, __LINE__); goto done; } } while (0)
    GI(pool_alloc((void **)&E0, sizeof(int2) * me, st));
    GI(pool_alloc((void **)&EH0, sizeof(int32_t) * me, st));
    GI(pool_alloc((void **)&ET0, sizeof(int32_t) * me, st));
    GI(pool_alloc((void **)&v32, sizeof(uint32_t) * me, st));
    GI(pool_alloc((void **)&v32b, sizeof(uint32_t) * me, st));
    GI(pool_alloc((void **)&k32b, sizeof(uint32_t) * me, st));
    k_fill_edges<<<grid_for(me), 256, 0, st>>>(g->cslot, me, g->src, g->adj, g->hash, g->thr, E0, EH0, ET0, v32);
    note_launch();
    GI(cudaGetLastError());
    g_clock.mark("index: alloc+fill", st);
    if (nb == 1) {
        // one bucket: the order is by hash alone (31-bit keys)
        const uint32_t *hk = reinterpret_cast<const uint32_t *>(EH0);
        GI(cub::DeviceRadixSort::SortPairs(nullptr, tb, hk, k32b, v32, v32b, (int)me, 0, 31, st));
        GI(pool_alloc(&tmp, tb, st));
        GI(cub::DeviceRadixSort::SortPairs(tmp, tb, hk, k32b, v32, v32b, (int)me, 0, 31, st));
        note_launch(4);
        g_clock.mark("index: sort", st);
        k_permute_uniform<<<grid_for(me), 256, 0, st>>>(v32b, k32b, me, E0, g->thr_u, g->E, g->EH, g->ET);
        note_launch();
        GI(cudaGetLastError());
        k_uniform_meta<<<1, 1, 0, st>>>(me, g->thr_u, g->boff, g->btmax); note_launch();
        GI(cudaGetLastError());
    } else {
        size_t tb2 = 0;
        GI(pool_alloc((void **)&k64, sizeof(uint64_t) * me, st));
        GI(pool_alloc((void **)&k64b, sizeof(uint64_t) * me, st));
        GI(pool_alloc((void **)&v32c, sizeof(uint32_t) * me, st));
        const uint32_t *tk = reinterpret_cast<const uint32_t *>(ET0);
        GI(cub::DeviceRadixSort::SortPairs(nullptr, tb, tk, k32b, v32, v32b, (int)me, 0, 32, st));
        GI(cub::DeviceRadixSort::SortPairs(nullptr, tb2, k64, k64b, v32, v32c, (int)me, 0, 40, st));
        GI(pool_alloc(&tmp, std::max(tb, tb2), st));
        GI(cub::DeviceRadixSort::SortPairs(tmp, tb, tk, k32b, v32, v32b, (int)me, 0, 32, st));
        g_clock.mark("index: thr sort", st);
        k_bucket_hash_keys<<<grid_for(me), 256, 0, st>>>(v32b, me, nb, EH0, k64, v32); note_launch();
        GI(cudaGetLastError());
        GI(cub::DeviceRadixSort::SortPairs(tmp, tb2, k64, k64b, v32, v32c, (int)me, 0, 40, st));
        note_launch(8);
        g_clock.mark("index: bucket sort", st);
        k_permute_edges<<<grid_for(me), 256, 0, st>>>(v32c, me, E0, EH0, ET0, g->E, g->EH, g->ET); note_launch();
        GI(cudaGetLastError());
        GI(cudaMemsetAsync(g->btmax, 0, sizeof(int32_t) * nb, st));
        GI(cudaMemsetAsync(g->boff, 0, sizeof(int64_t) * (nb + 1), st));
        k_bucket_meta<<<grid_for(me), 256, 0, st>>>(k64b, me, nb, g->ET, g->boff, g->btmax); note_launch();
        GI(cudaGetLastError());
    }
    k_build_lut<<<grid_for(lut_n), 256, 0, st>>>(g->EH, g->boff, nb, bits, g->lut); note_launch();
    GI(cudaGetLastError());
done:
    for (void *p : {(void *)k32b, (void *)v32, (void *)v32b, (void *)v32c, (void *)k64, (void *)k64b,
                    (void *)E0, (void *)EH0, (void *)ET0, tmp})
        if (p) cudaFreeAsync(p, st);
#undef GI
    return rc;
}

// Derived per-slot data and the sampler index, with ONE host round trip for
// the statistics the host needs (symmetry, max prefix, canonical count,
// threshold range and sum).  structure = build sources (if missing),
// reciprocal slots, hashes and the canonical edge list (new CSR); otherwise
// only the thresholds and the index are refreshed (new weights / hashes).
// late_weights (structure pass only): enqueues the weight upload after the
// weight-free structure kernels and makes the graph stream wait for it; the
// pairing then runs without thresholds and k_thresholds follows the upload
static int graph_nz_rows_async(imx_graph *g, GStats *gs);
static void graph_nz_rows_done(imx_graph *g, int64_t nnz);

static int graph_analyze(imx_graph *g, bool structure, const std::function<int()> &late_weights = nullptr) {
    cudaStream_t st = g->stream;
    const int64_t m2 = g->m2, n = g->n;
    GStats *gs = nullptr;
    IMX_CUDA(pool_alloc((void **)&gs, sizeof(GStats), st));
    k_stats_init<<<1, 1, 0, st>>>(gs); note_launch();
    if (structure) {
        if (!g->src) {
            IMX_TRY(dalloc(g, &g->src, m2));
            if (m2) {
                IMX_CUDA(cudaMemsetAsync(g->src, 0, sizeof(int32_t) * m2, st));   // rows of corrupt offsets
                k_src_rows<<<grid_for(n * 32), 256, 0, st>>>(g->xadj, n, m2, g->src);
                note_launch();
            }
        }
        IMX_TRY(dalloc(g, &g->hash, m2));
        IMX_TRY(dalloc(g, &g->thr, m2));
        IMX_TRY(dalloc(g, &g->recip, m2));
        IMX_TRY(dalloc(g, &g->cslot, m2));
        if (m2) {
            IMX_CUDA(cudaMemsetAsync(g->recip, 0xff, sizeof(int64_t) * m2, st));     // -1
            k_reciprocal<<<grid_for(m2), 256, 0, st>>>(g->xadj, g->adj, g->src, late_weights ? nullptr : g->w, n,
                                                        m2, g->recip, g->thr, gs);
            k_recip_check<<<grid_for(m2), 256, 0, st>>>(g->xadj, g->adj, g->src, g->recip, m2, &gs->flags);
            note_launch();
            k_slot_hashes<<<grid_for(m2), 256, 0, st>>>(g->src, g->adj, m2, g->hash);
            k_max_prefix<<<grid_for(n), 256, 0, st>>>(g->xadj, g->adj, n, m2, &gs->maxp);
            k_check_xadj<<<grid_for(n), 256, 0, st>>>(g->xadj, n, m2, &gs->flags);
            note_launch(4);
            IMX_CHECK_LAUNCH();
            uint8_t *flag;
            IMX_CUDA(pool_alloc((void **)&flag, m2, st));
            k_canon_flags<<<grid_for(m2), 256, 0, st>>>(g->src, g->adj, m2, flag); note_launch();
            size_t tmp_bytes = 0;
            thrust::counting_iterator<int64_t> it(0);
            IMX_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp_bytes, it, flag, g->cslot, &gs->me, m2, st));
            void *tmp;
            IMX_CUDA(pool_alloc(&tmp, tmp_bytes, st));
            IMX_CUDA(cub::DeviceSelect::Flagged(tmp, tmp_bytes, it, flag, g->cslot, &gs->me, m2, st));
            note_launch(2);
            cudaFreeAsync(tmp, st);
            cudaFreeAsync(flag, st);
            IMX_TRY(graph_nz_rows_async(g, gs));
        }
    }
    if (late_weights) IMX_TRY(late_weights());
    // thresholds: symmetrized through the reciprocal slots unless the
    // adjacency is known not to be symmetric (a structure pass decides below)
    // (a structure pass computed them with the reciprocal search, unless the
    // weights arrive late)
    const bool sym_try = structure || g->symmetric;
    if (m2 && (!structure || late_weights)) {
        k_thresholds<<<grid_for(m2), 256, 0, st>>>(g->w, sym_try ? g->recip : nullptr, g->src, g->adj, g->hash,
                                                   m2, g->thr, gs);
        note_launch();
        IMX_CHECK_LAUNCH();
    }
    GStats h;
    IMX_CUDA(cudaMemcpyAsync(&h, gs, sizeof h, cudaMemcpyDeviceToHost, st));
    IMX_CUDA(cudaStreamSynchronize(st));
    g_clock.mark("analysis (1 sync)", st);
    if (structure) {
        if (h.flags & 64u) {
            cudaFreeAsync(gs, st);
            set_error("corrupt CSR offsets");
            return IMX_EINVAL;
        }
        if (h.flags & 32u) {
            cudaFreeAsync(gs, st);
            set_error("adjacency entry outside 0..n-1");
            return IMX_EINVAL;
        }
        g->symmetric = (h.flags & 8u) == 0 && (m2 % 2 == 0);
        g->max_prefix = (int64_t)h.maxp;
        g->me = m2 ? h.me : 0;
        if (m2) graph_nz_rows_done(g, h.nnz);
        if (g->me >= (int64_t(1) << 31)) {
            cudaFreeAsync(gs, st);
            set_error("%lld undirected edges exceed 2^31 - 1", (long long)g->me);
            return IMX_ECONSTRAINT;
        }
        if (m2 && !g->symmetric) {        // rare: thresholds without symmetrization
            k_stats_init<<<1, 1, 0, st>>>(gs);
            k_thresholds<<<grid_for(m2), 256, 0, st>>>(g->w, nullptr, g->src, g->adj, g->hash, m2, g->thr, gs);
            note_launch(2);
            IMX_CHECK_LAUNCH();
            IMX_CUDA(cudaMemcpyAsync(&h, gs, sizeof h, cudaMemcpyDeviceToHost, st));
            IMX_CUDA(cudaStreamSynchronize(st));
        }
    }
    cudaFreeAsync(gs, st);
    g->hash_neg = (h.flags & 128u) != 0;
    g->uniform = m2 ? (h.tmin == h.tmax) : 1;
    g->thr_u = m2 ? h.tmin : 0;
    g->thr_mean = g->me ? (double)h.tsum / (double)g->me / 2147483647.0 : 0.0;
    g->index_ready = false;          // built on first use (ensure_index)
    g->thr_ready = true;
    return IMX_OK;
}

// The weight stream of a deferred graph: the upload, then (after everything
// enqueued on the graph stream so far: the structure) the raw per-slot
// thresholds and their statistics, not waited for (graph_settle).
static int deferred_weights_start(imx_graph *g, const double *weights) {
    cudaStream_t st = g->stream;
    const int64_t m2 = g->m2;
    cudaEvent_t ev_struct = nullptr;
    IMX_CUDA(cudaEventCreateWithFlags(&ev_struct, cudaEventDisableTiming));
    IMX_CUDA(cudaEventRecord(ev_struct, st));
    IMX_CUDA(acquire_stream(g->dev, &g->wst));
    IMX_CUDA(cudaEventCreateWithFlags(&g->wev, cudaEventDisableTiming));
    IMX_CUDA(pool_alloc(&g->wstats_d, sizeof(GStats), st));
    IMX_CUDA(pinned_get(&g->wstats_h, sizeof(GStats)));   // recycled: cudaFreeHost synchronises the device
    IMX_CUDA(cudaStreamWaitEvent(g->wst, ev_struct, 0));      // buffers allocated on st
    cudaEventDestroy(ev_struct);
    GStats *wd = static_cast<GStats *>(g->wstats_d);
    GStats *wh = static_cast<GStats *>(g->wstats_h);
    unsigned long long w0_bits;
    memcpy(&w0_bits, weights, sizeof w0_bits);
    auto finish = [g, m2, wd, wh, w0_bits]() -> int {
        cudaStream_t ws = g->wst;
        k_stats_init<<<1, 1, 0, ws>>>(wd);
        // uniform weights (the speculation) need no per-slot pass: only the proof that
        // every weight is weights[0]; anything else is settled by graph_settle
        k_weights_same<<<grid_for(m2), 256, 0, ws>>>(g->w, m2, w0_bits, &wd->flags);
        note_launch(2);
        IMX_CHECK_LAUNCH();
        IMX_CUDA(cudaMemcpyAsync(wh, wd, sizeof(GStats), cudaMemcpyDeviceToHost, ws));
        IMX_CUDA(cudaEventRecord(g->wev, ws));
        return IMX_OK;
    };
    const size_t wbytes = sizeof(double) * (size_t)m2;
    if (host_pinned_ptr(weights)) {
        IMX_CUDA(cudaMemcpyAsync(g->w, weights, wbytes, cudaMemcpyHostToDevice, g->wst));
        IMX_TRY(finish());
    } else {
        // pageable weights: the staged upload blocks its thread, so it runs
        // on its own host thread (joined by graph_settle)
        const int dev = g->dev;
        g->wthread = new std::thread([g, weights, wbytes, finish, dev]() {
            cudaSetDevice(dev);
            cudaError_t e = upload_h2d(g->w, weights, wbytes, g->wst);
            g->wthread_rc = e != cudaSuccess ? cuda_fail(e, "upload weights", __FILE__, __LINE__) : finish();
        });
    }
    g->thr_pending = true;
    return IMX_OK;
}

// imx_graph_from_csr for large graphs: the structure (sources, hashes, max
// prefix, offsets, symmetry, canonical slots) on the graph stream with one
// host sync; the weights and their raw per-slot thresholds on a second
// stream, not waited for (graph_settle).  Until then the graph claims the
// speculative uniform threshold of weights[0].
static int graph_analyze_deferred(imx_graph *g, const double *weights) {
    cudaStream_t st = g->stream;
    const int64_t m2 = g->m2, n = g->n;
    GStats *gs = nullptr;
    IMX_CUDA(pool_alloc((void **)&gs, sizeof(GStats), st));
    k_stats_init<<<1, 1, 0, st>>>(gs); note_launch();
    IMX_TRY(dalloc(g, &g->src, m2));
    IMX_TRY(dalloc(g, &g->hash, m2));
    IMX_TRY(dalloc(g, &g->thr, m2));
    IMX_TRY(dalloc(g, &g->cslot, m2));
    IMX_CUDA(cudaMemsetAsync(g->src, 0, sizeof(int32_t) * m2, st));   // rows of corrupt offsets
    k_src_rows<<<grid_for(n * 32), 256, 0, st>>>(g->xadj, n, m2, g->src);
    k_check_xadj<<<grid_for(n), 256, 0, st>>>(g->xadj, n, m2, &gs->flags);
    k_sym_hash<<<grid_for(m2), 256, 0, st>>>(g->xadj, g->adj, g->src, n, m2, g->hash, gs);
    k_max_prefix<<<grid_for(n), 256, 0, st>>>(g->xadj, g->adj, n, m2, &gs->maxp);
    note_launch(4);
    IMX_CHECK_LAUNCH();
    g->cslot_ready = false;          // canonical slot list on first use (ensure_cslot)
    IMX_TRY(graph_nz_rows_async(g, gs));
    IMX_TRY(deferred_weights_start(g, weights));
    g->thr_pending = true;
    GStats h;
    IMX_CUDA(cudaMemcpyAsync(&h, gs, sizeof h, cudaMemcpyDeviceToHost, st));
    IMX_CUDA(cudaStreamSynchronize(st));
    cudaFreeAsync(gs, st);
    g_clock.mark("structure (1 sync)", st);
    if (h.flags & 64u) { set_error("corrupt CSR offsets"); return IMX_EINVAL; }
    if (h.flags & 32u) { set_error("adjacency entry outside 0..n-1"); return IMX_EINVAL; }
    g->symmetric = (h.flags & 8u) == 0 && h.symsum == 0 && (m2 % 2 == 0);
    g->max_prefix = (int64_t)h.maxp;
    // symmetric, no self-loop: every undirected edge has exactly one canonical slot
    g->me = m2 / 2;
    graph_nz_rows_done(g, h.nnz);
    if (g->me >= (int64_t(1) << 31)) {
        set_error("%lld undirected edges exceed 2^31 - 1", (long long)g->me);
        return IMX_ECONSTRAINT;
    }
    g->recip_ready = false;
    g->index_ready = false;
    g->hash_neg = 0;                     // fresh 31-bit hashes
    // speculation: every slot's threshold is weights[0]'s (hashing.py:135-138)
    const int32_t t0 = (int32_t)(int64_t)(weights[0] * 2147483647.0);
    g->uniform = 1;
    g->thr_u = t0;
    g->thr_mean = (double)t0 / 2147483647.0;
    return IMX_OK;
}

// imx_graph_from_csr for large PINNED host CSRs: returns after the offsets
// are up and checked; the adjacency follows in row-aligned chunks on the
// upload stream, each chunk's structure kernels run on the graph stream as
// soon as it lands (graph.cuh, struct_pending).  The statistics are read by
// graph_settle_structure.  Until then the graph claims what a valid CSR has:
// symmetric, m2 / 2 undirected edges, the speculative uniform threshold.
static int graph_analyze_streamed(imx_graph *g, const int64_t *xadj_h, const int32_t *adj_h, const double *weights) {
    cudaStream_t st = g->stream;
    const int64_t m2 = g->m2, n = g->n;
    GStats *gs = nullptr;
    IMX_CUDA(pool_alloc((void **)&gs, sizeof(GStats), st));
    g->sstats_d = gs;
    IMX_CUDA(pinned_get(&g->sstats_h, sizeof(GStats)));
    k_stats_init<<<1, 1, 0, st>>>(gs); note_launch();
    IMX_TRY(dalloc(g, &g->src, m2));
    IMX_TRY(dalloc(g, &g->hash, m2));
    IMX_TRY(dalloc(g, &g->thr, m2));
    IMX_TRY(dalloc(g, &g->cslot, m2));
    IMX_CUDA(acquire_stream(g->dev, &g->ust));
    cudaEvent_t ev = nullptr;
    IMX_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    IMX_CUDA(cudaEventRecord(ev, st));                       // the buffers were allocated on st
    IMX_CUDA(cudaStreamWaitEvent(g->ust, ev, 0));
    // offsets first: everything below indexes with them
    IMX_CUDA(cudaMemcpyAsync(g->xadj, xadj_h, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, g->ust));
    IMX_CUDA(cudaEventRecord(ev, g->ust));
    // chunks of about equal slot counts, cut at row boundaries (host offsets)
    int want = 16;
    if (const char *e = getenv("IMX_STREAM_CHUNKS")) want = std::max(1, std::min((int)imx_graph::kMaxChunks, atoi(e)));
    g->nchunk = 0;
    g->chunk_row[0] = 0;
    for (int c = 1; c <= want; ++c) {
        int64_t v = c == want ? n : std::upper_bound(xadj_h, xadj_h + n + 1, m2 / want * c) - xadj_h - 1;
        v = std::min(std::max(v, g->chunk_row[g->nchunk]), n);
        if (v > g->chunk_row[g->nchunk] || c == want) g->chunk_row[++g->nchunk] = v;
    }
    // Upload order: the chunks of the highest ids first.  Pass 1 of a chunk
    // writes only that chunk's rows, so any order is valid, and on skewed
    // graphs the high ids hold many low-degree rows -- row stores that outlast
    // their slots' upload (C4: the last sixteenth of the slots took 1.5 ms of
    // pass 1 against 0.6 ms on the link) -- while the hub chunks are all slots
    // and few rows: with the hubs last, almost nothing is left when the link
    // goes quiet.  chunk_row[] / chunk_ev[] are kept in upload order.
    {
        int64_t rows[imx_graph::kMaxChunks + 1];
        for (int c = 0; c <= g->nchunk; ++c) rows[c] = g->chunk_row[c];
        for (int c = 0; c < g->nchunk; ++c) {
            g->chunk_lo[c] = rows[g->nchunk - 1 - c];
            g->chunk_hi[c] = rows[g->nchunk - c];
        }
    }
    for (int c = 0; c < g->nchunk; ++c) {
        const int64_t s0 = xadj_h[g->chunk_lo[c]], s1 = xadj_h[g->chunk_hi[c]];
        if (s0 < 0 || s1 > m2 || s0 > s1) { cudaEventDestroy(ev); set_error("corrupt CSR offsets"); return IMX_EINVAL; }
        if (s1 > s0)
            IMX_CUDA(cudaMemcpyAsync(g->adj + s0, adj_h + s0, sizeof(int32_t) * (s1 - s0), cudaMemcpyHostToDevice, g->ust));
        IMX_CUDA(cudaEventCreateWithFlags(&g->chunk_ev[c], cudaEventDisableTiming));
        IMX_CUDA(cudaEventRecord(g->chunk_ev[c], g->ust));   // re-recorded on st below
    }
    // graph stream: offsets check (read back now), then per chunk its structure
    IMX_CUDA(cudaStreamWaitEvent(st, ev, 0));
    k_check_xadj<<<grid_for(n), 256, 0, st>>>(g->xadj, n, m2, &gs->flags);
    note_launch();
    unsigned xflags = 0;
    IMX_CUDA(cudaMemcpyAsync(&xflags, &gs->flags, sizeof xflags, cudaMemcpyDeviceToHost, st));
    IMX_CUDA(cudaStreamSynchronize(st));
    cudaEventDestroy(ev);
    g_clock.mark("offsets up + checked", st);
    if (xflags & 64u) { set_error("corrupt CSR offsets"); return IMX_EINVAL; }
    IMX_TRY(graph_nz_rows_async(g, gs));
    for (int c = 0; c < g->nchunk; ++c) {
        const int64_t v0 = g->chunk_lo[c], v1 = g->chunk_hi[c];
        const int64_t s0 = xadj_h[v0], s1 = xadj_h[v1];
        IMX_CUDA(cudaStreamWaitEvent(st, g->chunk_ev[c], 0));
        if (s1 > s0) {
            k_src_rows<<<grid_for((v1 - v0) * 32), 256, 0, st>>>(g->xadj, v1, m2, g->src, v0);
            k_sym_hash<<<grid_for(s1 - s0), 256, 0, st>>>(g->xadj, g->adj, g->src, n, s1, g->hash, gs, s0);
            k_max_prefix<<<grid_for(v1 - v0), 256, 0, st>>>(g->xadj, g->adj, v1, m2, &gs->maxp, v0);
            note_launch(3);
            IMX_CHECK_LAUNCH();
        }
        IMX_CUDA(cudaEventRecord(g->chunk_ev[c], st));       // chunk c: adjacency, sources and hashes ready
    }
    IMX_CUDA(cudaMemcpyAsync(g->sstats_h, gs, sizeof(GStats), cudaMemcpyDeviceToHost, st));
    IMX_CUDA(cudaEventCreateWithFlags(&g->sev_done, cudaEventDisableTiming));
    IMX_CUDA(cudaEventRecord(g->sev_done, st));
    g->cslot_ready = false;
    // the weights follow the adjacency on the link (their stream waits for the graph stream)
    IMX_TRY(deferred_weights_start(g, weights));
    g->struct_pending = true;
    g->struct_rc = IMX_OK;
    g->symmetric = 1;
    g->max_prefix = -1;                  // unknown until settled
    g->me = m2 / 2;
    g->n_nz = -1;
    g->recip_ready = false;
    g->index_ready = false;
    g->hash_neg = 0;
    const int32_t t0 = (int32_t)(int64_t)(weights[0] * 2147483647.0);
    g->uniform = 1;
    g->thr_u = t0;
    g->thr_mean = (double)t0 / 2147483647.0;
    g_clock.mark("chunks enqueued", st);
    return IMX_OK;
}

}  // namespace imx

namespace imx {

int graph_settle_structure(imx_graph *g) {
    if (!g->struct_pending) return g->struct_rc;
    g->struct_pending = false;
    cudaError_t e = cudaEventSynchronize(g->sev_done);
    const GStats h = *static_cast<GStats *>(g->sstats_h);
    cudaEventDestroy(g->sev_done);
    g->sev_done = nullptr;
    for (int c = 0; c < g->nchunk; ++c) {
        if (g->chunk_ev[c]) cudaEventDestroy(g->chunk_ev[c]);
        g->chunk_ev[c] = nullptr;
    }
    g->nchunk = 0;
    release_stream(g->dev, g->ust);
    g->ust = nullptr;
    pinned_put(g->sstats_h, sizeof(GStats));
    g->sstats_h = nullptr;
    cudaFreeAsync(g->sstats_d, g->stream);
    g->sstats_d = nullptr;
    int rc = IMX_OK;
    if (e != cudaSuccess) rc = cuda_fail(e, "streamed CSR", __FILE__, __LINE__);
    else if (h.flags & 64u) { set_error("corrupt CSR offsets"); rc = IMX_EINVAL; }
    else if (h.flags & 32u) { set_error("adjacency entry outside 0..n-1"); rc = IMX_EINVAL; }
    g->symmetric = (h.flags & 8u) == 0 && h.symsum == 0 && (g->m2 % 2 == 0);
    g->max_prefix = (int64_t)h.maxp;
    g->me = g->m2 / 2;
    if (rc == IMX_OK) graph_nz_rows_done(g, h.nnz);
    if (rc == IMX_OK && !g->symmetric) { set_error("adjacency is not symmetric"); rc = IMX_EFORMAT; }
    if (rc == IMX_OK && g->me >= (int64_t(1) << 31)) {
        set_error("%lld undirected edges exceed 2^31 - 1", (long long)g->me);
        rc = IMX_ECONSTRAINT;
    }
    g->struct_rc = rc;
    return rc;
}

int graph_settle(imx_graph *g) {
    const int struct_rc = graph_settle_structure(g);
    if (!g->thr_pending) return struct_rc;
    g->thr_pending = false;
    if (g->wthread) {
        auto *t = static_cast<std::thread *>(g->wthread);
        t->join();
        delete t;
        g->wthread = nullptr;
    }
    int rc = g->wthread_rc;
    cudaError_t e = cudaEventSynchronize(g->wev);
    if (rc == IMX_OK && e != cudaSuccess) rc = cuda_fail(e, "weights", __FILE__, __LINE__);
    GStats h = *static_cast<GStats *>(g->wstats_h);
    cudaEventDestroy(g->wev);
    g->wev = nullptr;
    release_stream(g->dev, g->wst);
    g->wst = nullptr;
    pinned_put(g->wstats_h, sizeof(GStats));
    g->wstats_h = nullptr;
    cudaFreeAsync(g->wstats_d, g->stream);
    g->wstats_d = nullptr;
    if (struct_rc != IMX_OK) return struct_rc;
    if (rc != IMX_OK) return rc;
    if (g->m2 && !(h.flags & 256u)) {
        // every weight is weights[0]: the speculative threshold is the threshold
        // of every slot; the per-slot array is filled when something reads it
        h.flags = 0;
        h.tmin = h.tmax = g->thr_u;
        h.tsum = (unsigned long long)(uint32_t)g->thr_u * (unsigned long long)g->me;
        g->thr_ready = false;
    } else if (g->m2) {
        // per-slot thresholds: symmetrized through the reciprocal slots
        if (g->symmetric) IMX_TRY(ensure_recip(g));
        GStats *gs;
        IMX_CUDA(pool_alloc((void **)&gs, sizeof(GStats), g->stream));
        k_stats_init<<<1, 1, 0, g->stream>>>(gs);
        k_thresholds<<<grid_for(g->m2), 256, 0, g->stream>>>(g->w, g->symmetric ? g->recip : nullptr, g->src, g->adj,
                                                             g->hash, g->m2, g->thr, gs);
        note_launch(2);
        IMX_CHECK_LAUNCH();
        IMX_CUDA(cudaMemcpyAsync(&h, gs, sizeof h, cudaMemcpyDeviceToHost, g->stream));
        IMX_CUDA(cudaStreamSynchronize(g->stream));
        cudaFreeAsync(gs, g->stream);
    }
    g->hash_neg = (h.flags & 128u) != 0;
    g->uniform = g->m2 ? (h.tmin == h.tmax) : 1;
    g->thr_u = g->m2 ? h.tmin : 0;
    g->thr_mean = g->me ? (double)h.tsum / (double)g->me / 2147483647.0 : 0.0;
    g->index_ready = false;
    return IMX_OK;
}

int ensure_thr(imx_graph *g) {
    if (g->thr_ready) return IMX_OK;
    if (g->m2) {
        k_fill_i32<<<grid_for(g->m2), 256, 0, g->stream>>>(g->thr, g->m2, g->thr_u);
        note_launch();
        IMX_CHECK_LAUNCH();
        IMX_CUDA(cudaStreamSynchronize(g->stream));   // its readers run on other streams
    }
    g->thr_ready = true;
    return IMX_OK;
}

int ensure_recip(imx_graph *g) {
    if (g->recip_ready) return IMX_OK;
    cudaStream_t st = g->stream;
    const int64_t m2 = g->m2;
    GStats *gs;
    IMX_TRY(dalloc(g, &g->recip, m2));
    IMX_CUDA(pool_alloc((void **)&gs, sizeof(GStats), st));
    k_stats_init<<<1, 1, 0, st>>>(gs);
    if (m2) {
        IMX_CUDA(cudaMemsetAsync(g->recip, 0xff, sizeof(int64_t) * m2, st));     // -1
        k_reciprocal<<<grid_for(m2), 256, 0, st>>>(g->xadj, g->adj, g->src, nullptr, g->n, m2, g->recip,
                                                    g->thr, gs);
        k_recip_check<<<grid_for(m2), 256, 0, st>>>(g->xadj, g->adj, g->src, g->recip, m2, &gs->flags);
        note_launch(3);
        IMX_CHECK_LAUNCH();
    }
    GStats h;
    IMX_CUDA(cudaMemcpyAsync(&h, gs, sizeof h, cudaMemcpyDeviceToHost, st));
    IMX_CUDA(cudaStreamSynchronize(st));
    cudaFreeAsync(gs, st);
    if (h.flags & 8u) {
        g->symmetric = 0;
        set_error("adjacency is not symmetric");
        return IMX_EFORMAT;
    }
    g->recip_ready = true;
    return IMX_OK;
}

__global__ void k_nz_flags(const int64_t *__restrict__ xadj, int64_t n, uint8_t *__restrict__ flag) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        flag[v] = xadj[v + 1] > xadj[v];
}

// The rows the compression must stream: vertices with at least one slot,
// listed on the graph stream while the structure is analysed (the count
// rides on the analysis' one host sync: graph_nz_rows_done).
static int graph_nz_rows_async(imx_graph *g, GStats *gs) {
    cudaStream_t st = g->stream;
    const int64_t n = g->n;
    if (n == 0) return IMX_OK;
    uint8_t *flag = nullptr;
    void *tmp = nullptr;
    size_t tb = 0;
    if (g->nz_rows) { cudaFreeAsync(g->nz_rows, st); g->nz_rows = nullptr; }
    IMX_CUDA(pool_alloc((void **)&flag, n, st));
    IMX_CUDA(pool_alloc((void **)&g->nz_rows, sizeof(int32_t) * n, st));
    k_nz_flags<<<grid_for(n), 256, 0, st>>>(g->xadj, n, flag);
    note_launch();
    thrust::counting_iterator<int32_t> it(0);
    IMX_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, it, flag, g->nz_rows, &gs->nnz, n, st));
    IMX_CUDA(pool_alloc(&tmp, tb, st));
    IMX_CUDA(cub::DeviceSelect::Flagged(tmp, tb, it, flag, g->nz_rows, &gs->nnz, n, st));
    note_launch(2);
    cudaFreeAsync(flag, st);
    cudaFreeAsync(tmp, st);
    return IMX_OK;
}

// kept only when at least 1/8 of the vertices are isolated (C4: 44%)
static void graph_nz_rows_done(imx_graph *g, int64_t nnz) {
    if (g->nz_rows && g->n - nnz >= g->n / 8) {
        g->n_nz = nnz;
    } else {
        if (g->nz_rows) cudaFreeAsync(g->nz_rows, g->stream);
        g->nz_rows = nullptr;
        g->n_nz = g->n;
    }
}

int ensure_nz_rows(imx_graph *g) {
    if (g->n_nz >= 0) return IMX_OK;
    GStats *gs;
    IMX_CUDA(pool_alloc((void **)&gs, sizeof(GStats), g->stream));
    k_stats_init<<<1, 1, 0, g->stream>>>(gs);
    IMX_TRY(graph_nz_rows_async(g, gs));
    GStats h;
    IMX_CUDA(cudaMemcpyAsync(&h, gs, sizeof h, cudaMemcpyDeviceToHost, g->stream));
    IMX_CUDA(cudaStreamSynchronize(g->stream));
    cudaFreeAsync(gs, g->stream);
    graph_nz_rows_done(g, h.nnz);
    return IMX_OK;
}

// canonical slots (src < adj) in slot order, built on first use on large
// host CSRs (the enumeration index, evaluate_seeds and sampling_cdf need them)
int ensure_cslot(imx_graph *g) {
    if (g->cslot_ready) return IMX_OK;
    cudaStream_t st = g->stream;
    const int64_t m2 = g->m2;
    if (m2) {
        uint8_t *flag;
        int64_t *cnt;
        IMX_CUDA(pool_alloc((void **)&flag, m2, st));
        IMX_CUDA(pool_alloc((void **)&cnt, sizeof(int64_t), st));
        k_canon_flags<<<grid_for(m2), 256, 0, st>>>(g->src, g->adj, m2, flag); note_launch();
        size_t tmp_bytes = 0;
        thrust::counting_iterator<int64_t> it(0);
        IMX_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp_bytes, it, flag, g->cslot, cnt, m2, st));
        void *tmp;
        IMX_CUDA(pool_alloc(&tmp, tmp_bytes, st));
        IMX_CUDA(cub::DeviceSelect::Flagged(tmp, tmp_bytes, it, flag, g->cslot, cnt, m2, st));
        note_launch(2);
        int64_t me = 0;
        IMX_CUDA(cudaMemcpyAsync(&me, cnt, sizeof me, cudaMemcpyDeviceToHost, st));
        IMX_CUDA(cudaStreamSynchronize(st));
        cudaFreeAsync(tmp, st);
        cudaFreeAsync(flag, st);
        cudaFreeAsync(cnt, st);
        g->me = me;
    }
    g->cslot_ready = true;
    return IMX_OK;
}

int ensure_index(imx_graph *g) {
    IMX_TRY(graph_settle(g));
    if (g->index_ready) return IMX_OK;
    IMX_TRY(ensure_cslot(g));
    IMX_TRY(graph_build_index(g));
    // built on the graph stream; its users run on context streams
    IMX_CUDA(cudaStreamSynchronize(g->stream));
    g->index_ready = true;
    return IMX_OK;
}

static int graph_new(int32_t device, int64_t n, int64_t m2, imx_graph **out) {
    IMX_TRY(select_device(device));
    imx_graph *g = new imx_graph();
    g->dev = device;
    g->n = n;
    g->m2 = m2;
    if (acquire_stream(device, &g->stream) != cudaSuccess) {
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
    return graph_analyze(g, true);
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
            e = upload_h2d(dedges, edges, sizeof(int64_t) * 2 * k, st);
        if (e == cudaSuccess && w_edge) {
            if ((e = cudaMallocAsync((void **)&dw, sizeof(double) * k, st)) == cudaSuccess)
                e = upload_h2d(dw, w_edge, sizeof(double) * k, st);
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
    g_clock.start();
    // offsets are checked on the device (k_check_xadj) before anything uses them
    if (xadj[0] != 0 || xadj[n] != m2) { set_error("corrupt CSR offsets"); return IMX_EINVAL; }
    imx_graph *g;
    IMX_TRY(graph_new(device, n, m2, &g));
    cudaStream_t st = g->stream;
    g_clock.mark("validate+stream", st);
    auto fail = [&](int code) { graph_free(g); return code; };
    if (dalloc(g, &g->xadj, n + 1) || dalloc(g, &g->adj, m2) || dalloc(g, &g->w, m2)) return fail(IMX_ENOMEM);
    // large graphs: the weights (8 bytes per slot, the biggest array) go up on
    // a second stream and are not waited for (graph_analyze_deferred); very
    // large pinned ones also stream the adjacency (graph_analyze_streamed)
    const char *lw = getenv("IMX_LATE_WEIGHTS");
    const bool late = m2 > 0 && (lw ? atoi(lw) != 0 : m2 >= ((int64_t)1 << 22));
    const char *sc = getenv("IMX_STREAM_CSR");
    const bool streamed = late && n > 0 && (sc ? atoi(sc) != 0 : (m2 >= ((int64_t)1 << 24) && host_pinned_ptr(xadj) &&
                                                                   host_pinned_ptr(adj) && host_pinned_ptr(weights)));
    if (streamed) {
        const int rc = graph_analyze_streamed(g, xadj, adj, weights);
        if (rc != IMX_OK) {
            // chunk copies may still read the caller's arrays
            if (g->ust) cudaStreamSynchronize(g->ust);
            cudaStreamSynchronize(st);
            g->struct_pending = false;
            return fail(rc);
        }
        *out = g;
        return IMX_OK;
    }
    if (upload_h2d(g->xadj, xadj, sizeof(int64_t) * (n + 1), st) != cudaSuccess ||
        (m2 && upload_h2d(g->adj, adj, sizeof(int32_t) * m2, st) != cudaSuccess))
        return fail(cuda_fail(cudaGetLastError(), "upload csr", __FILE__, __LINE__));
    if (late) {
        g_clock.mark("upload csr", st);
        const int rc = graph_analyze_deferred(g, weights);
        if (rc != IMX_OK) return fail(rc);
        *out = g;
        return IMX_OK;
    }
    if (m2 && upload_h2d(g->w, weights, sizeof(double) * m2, st) != cudaSuccess)
        return fail(cuda_fail(cudaGetLastError(), "upload weights", __FILE__, __LINE__));
    g_clock.mark("upload csr", st);
    const int rc = graph_analyze(g, true);
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
    IMX_TRY(graph_settle(g));
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
    IMX_TRY(graph_settle(g));
    IMX_TRY(ensure_recip(g));
    if (g->m2) {
        IMX_CUDA(cudaMemcpyAsync(recip, g->recip, sizeof(int64_t) * g->m2, cudaMemcpyDeviceToHost, g->stream));
        IMX_CUDA(cudaStreamSynchronize(g->stream));
    }
    return IMX_OK;
}

extern "C" int imx_graph_set_weights(imx_graph *g, const double *weights) {
    if (!g || (!weights && g->m2)) { set_error("NULL argument"); return IMX_EINVAL; }
    IMX_CUDA(cudaSetDevice(g->dev));
    IMX_TRY(graph_settle(g));
    if (g->symmetric) IMX_TRY(ensure_recip(g));
    cudaStream_t st = g->stream;
    if (g->m2) {
        double *tmp;
        IMX_CUDA(cudaMallocAsync((void **)&tmp, sizeof(double) * g->m2, st));
        IMX_CUDA(upload_h2d(tmp, weights, sizeof(double) * g->m2, st));
        unsigned *dflags;
        IMX_CUDA(cudaMallocAsync((void **)&dflags, sizeof(unsigned), st));
        IMX_CUDA(cudaMemsetAsync(dflags, 0, sizeof(unsigned), st));
        k_weights_range<<<grid_for(g->m2), 256, 0, st>>>(tmp, g->m2, dflags); note_launch();
        IMX_CHECK_LAUNCH();
        unsigned flags = 0;
        IMX_CUDA(cudaMemcpyAsync(&flags, dflags, sizeof flags, cudaMemcpyDeviceToHost, st));
        IMX_CUDA(cudaStreamSynchronize(st));
        cudaFreeAsync(dflags, st);
        if (flags & 16u) {
            cudaFreeAsync(tmp, st);
            set_error("weights must lie in [0, 1]");
            return IMX_ECONSTRAINT;
        }
        IMX_CUDA(cudaMemcpyAsync(g->w, tmp, sizeof(double) * g->m2, cudaMemcpyDeviceToDevice, st));
        cudaFreeAsync(tmp, st);
    }
    return graph_analyze(g, false);
}

extern "C" int imx_graph_hashes(imx_graph *g, int32_t *out) {
    if (!g || (!out && g->m2)) { set_error("NULL argument"); return IMX_EINVAL; }
    IMX_CUDA(cudaSetDevice(g->dev));
    IMX_TRY(graph_settle_structure(g));
    if (g->m2) {
        IMX_CUDA(cudaMemcpyAsync(out, g->hash, sizeof(int32_t) * g->m2, cudaMemcpyDeviceToHost, g->stream));
        IMX_CUDA(cudaStreamSynchronize(g->stream));
    }
    return IMX_OK;
}

extern "C" int imx_graph_set_hashes(imx_graph *g, const int32_t *hashes) {
    if (!g) { set_error("NULL argument"); return IMX_EINVAL; }
    IMX_CUDA(cudaSetDevice(g->dev));
    IMX_TRY(graph_settle(g));
    if (g->symmetric) IMX_TRY(ensure_recip(g));
    if (g->m2) {
        if (hashes) {
            IMX_CUDA(cudaMemcpyAsync(g->hash, hashes, sizeof(int32_t) * g->m2, cudaMemcpyHostToDevice, g->stream));
        } else {
            k_slot_hashes<<<grid_for(g->m2), 256, 0, g->stream>>>(g->src, g->adj, g->m2, g->hash); note_launch();
            IMX_CHECK_LAUNCH();
        }
    }
    return graph_analyze(g, false);
}

extern "C" int imx_graph_thresholds(imx_graph *g, int32_t symmetrize, int32_t *thr_out,
                                    int32_t *uniform_out) {
    if (!g || (!thr_out && g->m2)) { set_error("NULL argument"); return IMX_EINVAL; }
    IMX_CUDA(cudaSetDevice(g->dev));
    IMX_TRY(graph_settle(g));
    cudaStream_t st = g->stream;
    if (symmetrize && !g->symmetric) { set_error("adjacency is not symmetric"); return IMX_EFORMAT; }
    if (g->m2) {
        if (symmetrize) {
            IMX_TRY(ensure_thr(g));
            IMX_CUDA(cudaMemcpyAsync(thr_out, g->thr, sizeof(int32_t) * g->m2, cudaMemcpyDeviceToHost, st));
        } else {
            int32_t *tmp;
            GStats *gs;
            IMX_CUDA(pool_alloc((void **)&tmp, sizeof(int32_t) * g->m2, st));
            IMX_CUDA(pool_alloc((void **)&gs, sizeof(GStats), st));
            k_stats_init<<<1, 1, 0, st>>>(gs);
            k_thresholds<<<grid_for(g->m2), 256, 0, st>>>(g->w, nullptr, g->src, g->adj, nullptr, g->m2, tmp, gs);
            note_launch(2);
            IMX_CHECK_LAUNCH();
            IMX_CUDA(cudaMemcpyAsync(thr_out, tmp, sizeof(int32_t) * g->m2, cudaMemcpyDeviceToHost, st));
            cudaFreeAsync(tmp, st);
            cudaFreeAsync(gs, st);
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
