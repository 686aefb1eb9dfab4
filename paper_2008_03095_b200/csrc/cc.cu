// cc.cu -- K3 fused sample + CC, K4/K5 memoization, K6-K8 CELF on sm_100a.
//
// Data layout in HBM (one context = one device, one lane window of width W):
//   L[n][ld]  uint32  labels, simulation-contiguous (propagation.py:1-8),
//                     ld = W rounded up to 4 so every row is 16-byte aligned.
//   C[n][ld]  uint32  per-root member count EXCLUDING the root; the component
//                     size of label l in lane r is C[l][r] + 1, and
//                     sizes[l][r] = C[l][r] + (L[l][r] == l) (propagation.py:349-356).
//   cov[n][cw] uint32 covered-component bitmap of the CELF state, cw = ceil(ns/32)
//                     (SeedState.owned, selection.py:36-60).
//
// Propagation is concurrent union-find over all W lanes at once, not
// min-label sweeps: the fixpoint the reference's sweeps reach (min vertex id
// of the component of every vertex in every lane) is unique, so
// any exact CC algorithm reproduces it.  Trees always hook the
// larger root under the smaller one, so a root is the minimum id of its tree.
//
//   k_init      L[v][r] = v                                    (streaming write)
//   k_hook      for every undirected edge {lo,hi} and lane r with
//               (X[r] ^ h) < thr:  union(lo, hi) in lane r      (sampler fused in)
//   k_compress  L[v][r] = root(v, r); C[root][r] += 1 for non-roots
//   k_verify    (optional) every live edge joins equal labels; every label is a root
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cub/cub.cuh>

#include "common.cuh"
#include "graph.cuh"

struct imx_ctx {
    imx_graph *g = nullptr;
    int dev = 0;
    cudaStream_t st = nullptr;
    int32_t W = 0, ns = 0, cw = 0;
    int64_t ld = 0;
    int vb = 0;                   // bits for vertex ids in packed CELF keys
    int32_t *X = nullptr;         // [ld]
    uint32_t *L = nullptr;        // [n*ld]
    uint32_t *C = nullptr;        // [n*ld]
    int64_t *gains = nullptr;     // [n]
    int64_t *prio = nullptr;      // [n]
    uint8_t *inS = nullptr;       // [n]
    uint32_t *cov = nullptr;      // [n*cw]
    int64_t *per_sim = nullptr;   // [W]
    int32_t *cand = nullptr;      // [n]
    int64_t *fresh = nullptr;     // [n]
    unsigned long long *scratch = nullptr;  // [16]; [8..12] = CELF round header
    int64_t ncand = 0;
    int32_t *cand2 = nullptr;     // [n] sort output
    unsigned long long *keys2 = nullptr;  // [n] sorted keys
    int64_t *eval_out = nullptr;  // [n]
    int32_t *d_one = nullptr;     // [1]
    void *sort_tmp = nullptr;
    size_t sort_tmp_bytes = 0;
    int32_t *h_ids = nullptr, *d_ids = nullptr;   // pinned staging for prio updates
    int64_t *h_vals = nullptr, *d_vals = nullptr;
    int64_t stage_cap = 0;
    int64_t evaluated = 0;
    int64_t *seg_a = nullptr, *seg_n = nullptr, *seg_off = nullptr;  // enumeration segments
    int64_t nseg_cap = 0;
    void *scan_tmp = nullptr;
    size_t scan_tmp_bytes = 0;
    bool labels_ready = false, memo_ready = false, celf_ready = false;
    int full_counts = 0;          // 1: C holds full sizes (host-loaded labels)
    cudaEvent_t ev[8];
    imx_timings tm{};
    std::vector<int64_t> trace;   // 5 per record
};

namespace imx {

// ---------------------------------------------------------------------------
// union-find primitives (per lane; every lane is an independent graph)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t *cell(uint32_t *L, int64_t ld, uint32_t v, int r) {
    return L + (int64_t)v * ld + r;
}

__device__ __forceinline__ uint32_t find_ro(const uint32_t *L, int64_t ld, uint32_t x, int r) {
    uint32_t p;
    while ((p = ld_relaxed(L + (int64_t)x * ld + r)) != x) x = p;
    return x;
}

// Two root searches advanced in lock step so their loads overlap.  Path
// splitting: every visited node is re-pointed at its grandparent (a benign
// race -- any value ever stored in a cell is an ancestor in the same tree).
// On entry pa = L[xa], pb = L[xb]; on exit xa, xb are roots.
__device__ __forceinline__ void find2(uint32_t *L, int64_t ld, int r, uint32_t &xa, uint32_t pa,
                                      uint32_t &xb, uint32_t pb) {
    for (;;) {
        const bool da = pa == xa, db = pb == xb;
        if (da && db) return;
        uint32_t ga = pa, gb = pb;
        if (!da) ga = ld_relaxed(cell(L, ld, pa, r));
        if (!db) gb = ld_relaxed(cell(L, ld, pb, r));
        if (!da) {
            if (ga == pa) xa = pa;
            else { st_relaxed(cell(L, ld, xa, r), ga); xa = pa; pa = ga; }
        }
        if (!db) {
            if (gb == pb) xb = pb;
            else { st_relaxed(cell(L, ld, xb, r), gb); xb = pb; pb = gb; }
        }
    }
}

// union of a and b in lane r: CAS-hook the larger root under the smaller.
__device__ __forceinline__ int unite(uint32_t *L, int64_t ld, uint32_t a, uint32_t b, int r) {
    uint32_t pa = ld_relaxed(cell(L, ld, a, r));
    uint32_t pb = ld_relaxed(cell(L, ld, b, r));
    find2(L, ld, r, a, pa, b, pb);
    while (a != b) {
        const uint32_t lo = a < b ? a : b, hi = a < b ? b : a;
        const uint32_t old = atomicCAS(cell(L, ld, hi, r), hi, lo);
        if (old == hi) return 1;
        a = lo;
        b = hi;
        find2(L, ld, r, a, ld_relaxed(cell(L, ld, lo, r)), b, old);
    }
    return 0;
}

// ---------------------------------------------------------------------------
// K3: init / hook / compress / verify
// ---------------------------------------------------------------------------
__global__ void k_init(uint32_t *__restrict__ L, int64_t n, int64_t ld) {
    const int64_t nq = ld >> 2;
    uint4 *L4 = reinterpret_cast<uint4 *>(L);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * nq;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t v = (uint32_t)(i / nq);
        L4[i] = make_uint4(v, v, v, v);
    }
}

// Sampler + hooking.  A warp takes tiles of 32 undirected edges (one edge per
// thread, coalesced loads of (lo, hi), hash and threshold), then walks the
// tile edge by edge: each thread tests 4 consecutive lanes of a 128-lane
// chunk against the edge ((X[r] ^ h) < t, X staged in shared memory once per
// CTA), and the live (edge, lane) pairs are appended to a per-warp queue in
// shared memory.  Whenever the queue holds 32 pairs the warp drains 32 at
// once -- one union per thread -- so the latency-bound root searches always
// run 32-wide instead of at the ~1% density of live lanes.  The adjacency and
// hash are read once per edge and reused across all W lanes.
constexpr int kHookWarps = 8;
constexpr int kQ = 32 + 128;  // drain threshold + one chunk's worth of appends

template <bool UNI>
__global__ void __launch_bounds__(kHookWarps * 32) k_hook(const int2 *__restrict__ E, const int32_t *__restrict__ EH,
                                                          const int32_t *__restrict__ ET, int32_t tu, int64_t me,
                                                          const int32_t *__restrict__ X, int32_t W, int64_t ld,
                                                          uint32_t *__restrict__ L,
                                                          unsigned long long *__restrict__ hooks) {
    extern __shared__ int4 smem4[];
    int32_t *sX = reinterpret_cast<int32_t *>(smem4);
    for (int i = threadIdx.x; i < ld; i += blockDim.x) sX[i] = (i < W) ? X[i] : 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t *qlo = reinterpret_cast<uint32_t *>(sX + ld) + warp * 3 * kQ;
    uint32_t *qhi = qlo + kQ;
    uint32_t *qr = qhi + kQ;
    __syncthreads();
    const int nq = (int)(ld >> 2);
    const unsigned FULL = 0xffffffffu;
    int qn = 0;  // warp-uniform queue length
    unsigned long long nh = 0;
    for (int64_t base = ((int64_t)blockIdx.x * kHookWarps + warp) * 32; base < me;
         base += (int64_t)gridDim.x * kHookWarps * 32) {
        const int64_t e = base + lane;
        int2 uv = make_int2(0, 0);
        int32_t h = 0, t = 0;  // t = 0: nothing is live
        if (e < me) {
            uv = __ldg(&E[e]);
            h = __ldg(&EH[e]);
            t = UNI ? tu : __ldg(&ET[e]);
        }
        const int cnt = (int)(me - base < 32 ? me - base : 32);
        for (int j = 0; j < cnt; ++j) {
            const int32_t hj = __shfl_sync(FULL, h, j), tj = __shfl_sync(FULL, t, j);
            const uint32_t lo = (uint32_t)__shfl_sync(FULL, uv.x, j);
            const uint32_t hi = (uint32_t)__shfl_sync(FULL, uv.y, j);
            for (int c0 = 0; c0 < nq; c0 += 32) {
                const int qd = c0 + lane;
                unsigned live = 0;
                if (qd < nq) {
                    const int4 x = smem4[qd];
                    live = ((unsigned)((x.x ^ hj) < tj)) | ((unsigned)((x.y ^ hj) < tj) << 1) |
                           ((unsigned)((x.z ^ hj) < tj) << 2) | ((unsigned)((x.w ^ hj) < tj) << 3);
                    const int r = qd << 2;
                    if (r + 4 > W) live &= (1u << (W > r ? W - r : 0)) - 1u;
                }
                if (!__any_sync(FULL, live != 0)) continue;
                const int k = __popc(live);
                int inc = k;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(FULL, inc, o);
                    if (lane >= o) inc += y;
                }
                int pos = qn + inc - k;
                while (live) {
                    const int b = __ffs(live) - 1;
                    live &= live - 1;
                    qlo[pos] = lo;
                    qhi[pos] = hi;
                    qr[pos] = (uint32_t)((qd << 2) + b);
                    ++pos;
                }
                qn += __shfl_sync(FULL, inc, 31);
                __syncwarp();
                while (qn >= 32) {
                    qn -= 32;
                    const uint32_t a = qlo[qn + lane], bb = qhi[qn + lane];
                    const int r = (int)qr[qn + lane];
                    __syncwarp();
                    nh += unite(L, ld, a, bb, r);
                }
            }
        }
    }
    __syncwarp();
    if (lane < qn) nh += unite(L, ld, qlo[lane], qhi[lane], (int)qr[lane]);
    if (hooks) {
        for (int o = 16; o; o >>= 1) nh += __shfl_xor_sync(FULL, nh, o);
        if (lane == 0 && nh) atomicAdd(hooks, nh);
    }
}

// ---------------------------------------------------------------------------
// Sampler by interval enumeration (default).  For a threshold t and a lane
// word x, {h : (x ^ h) < t} is the union over the set bits i of t of the
// aligned hash interval [((t ^ x) >> (i+1) << (i+1)) | (x & 2^i), +2^i)
// (the reference's _xor_below, propagation.py:104-118).  The undirected
// edges are sorted by (threshold bucket, hash) on the device (graph.cu), so a
// (lane, bucket, bit) segment is a contiguous range of edges found by two
// binary searches, and the live (edge, lane) pairs of all lanes form one
// flattened index space: no dead (edge, lane) pair is ever visited.  With
// per-edge thresholds a bucket's interval uses the bucket's max threshold
// and each enumerated edge is re-tested exactly ((x ^ h) < thr, strict).
// ---------------------------------------------------------------------------
__global__ void k_seg_count(const int32_t *__restrict__ X, int32_t W, int nb,
                            const int32_t *__restrict__ btmax, const int64_t *__restrict__ boff,
                            const int32_t *__restrict__ EH, int64_t *__restrict__ seg_a,
                            int64_t *__restrict__ seg_n) {
    const int64_t nseg = (int64_t)W * nb * 31;
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nseg;
         s += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(s / (nb * 31));
        const int rem = (int)(s - (int64_t)r * nb * 31);
        const int b = rem / 31, i = rem - b * 31;
        const uint32_t t = (uint32_t)btmax[b];
        int64_t a = boff[b], cnt = 0;
        if ((t >> i) & 1u) {
            const uint32_t x = (uint32_t)X[r];
            const uint64_t start = ((uint64_t)((t ^ x) >> (i + 1)) << (i + 1)) | (uint64_t)(x & (1u << i));
            const uint64_t end = start + (1ull << i);
            int64_t lo = boff[b], hi = boff[b + 1];
            while (lo < hi) {  // lower_bound(start)
                const int64_t mid = (lo + hi) >> 1;
                if ((uint64_t)(uint32_t)EH[mid] < start) lo = mid + 1; else hi = mid;
            }
            a = lo;
            hi = boff[b + 1];
            while (lo < hi) {  // lower_bound(end)
                const int64_t mid = (lo + hi) >> 1;
                if ((uint64_t)(uint32_t)EH[mid] < end) lo = mid + 1; else hi = mid;
            }
            cnt = lo - a;
        }
        seg_a[s] = a;
        seg_n[s] = cnt;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) seg_n[nseg] = 0;
}

// Every thread takes flattened live pairs j; a warp owns chunks of kEnumChunk
// consecutive j (one binary search over the segment offsets per chunk, then
// a forward walk), so consecutive threads read consecutive edges of the same
// hash interval (coalesced) and every thread runs one union per pair.
constexpr int kEnumChunk = 1024;
template <bool UNI>
__global__ void __launch_bounds__(256) k_hook_enum(const int64_t *__restrict__ off, const int64_t *__restrict__ seg_a,
                                                   int64_t nseg, int segs_per_lane,
                                                   const int2 *__restrict__ E, const int32_t *__restrict__ EH,
                                                   const int32_t *__restrict__ ET, const int32_t *__restrict__ X,
                                                   int64_t ld, uint32_t *__restrict__ L,
                                                   unsigned long long *__restrict__ hooks) {
    const int64_t total = off[nseg];
    const int lane = threadIdx.x & 31;
    const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long nh = 0;
    for (int64_t j0 = wg * kEnumChunk; j0 < total; j0 += nw * kEnumChunk) {
        int64_t s = 0;
        if (lane == 0) {
            int64_t lo = 0, hi = nseg;       // largest s with off[s] <= j0
            while (hi - lo > 1) {
                const int64_t mid = (lo + hi) >> 1;
                if (off[mid] <= j0) lo = mid; else hi = mid;
            }
            s = lo;
        }
        s = __shfl_sync(0xffffffffu, s, 0);
        const int64_t jend = (total - j0 < kEnumChunk) ? total : j0 + kEnumChunk;
        for (int64_t j = j0 + lane; j < jend; j += 32) {
            while (off[s + 1] <= j) ++s;
            const int64_t e = seg_a[s] + (j - off[s]);
            const int r = (int)(s / segs_per_lane);
            if (!UNI && !((X[r] ^ EH[e]) < ET[e])) continue;
            const int2 uv = E[e];
            nh += unite(L, ld, (uint32_t)uv.x, (uint32_t)uv.y, r);
        }
    }
    if (hooks) {
        for (int o = 16; o; o >>= 1) nh += __shfl_xor_sync(0xffffffffu, nh, o);
        if (lane == 0 && nh) atomicAdd(hooks, nh);
    }
}

// ---------------------------------------------------------------------------
// Pull sampler (dense live fraction).  Rows are sorted ascending, so the
// smaller neighbours of v are a prefix of its row.  Pass 1 writes, for every
// lane, L[v][r] = the smallest live smaller neighbour (or v) and C[v][r] = 0:
// a forest whose edges are live edges pointing to smaller ids, built with
// coalesced row writes and no random reads (it replaces the init kernel).
// Pass 2 rescans the same prefixes and unites only the live edges that are
// not a vertex's first live smaller neighbour -- 4-30% of the live pairs on
// the benchmark graphs -- through the per-warp queue of k_hook.
// ---------------------------------------------------------------------------
template <int PASS, bool UNI>
__global__ void __launch_bounds__(256) k_pull(const int64_t *__restrict__ xadj, const int32_t *__restrict__ adj,
                                              const int32_t *__restrict__ hash, const int32_t *__restrict__ thr,
                                              int32_t tu, int64_t n, const int32_t *__restrict__ X, int32_t W,
                                              int64_t ld, uint32_t *__restrict__ L, uint32_t *__restrict__ C,
                                              unsigned long long *__restrict__ hooks) {
    extern __shared__ int4 smem4[];
    int32_t *sX = reinterpret_cast<int32_t *>(smem4);
    for (int i = threadIdx.x; i < ld; i += blockDim.x) sX[i] = (i < W) ? X[i] : 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t *qlo = reinterpret_cast<uint32_t *>(sX + ld) + warp * 3 * kQ;
    uint32_t *qhi = qlo + kQ;
    uint32_t *qr = qhi + kQ;
    __syncthreads();
    const int nq = (int)(ld >> 2);
    const unsigned FULL = 0xffffffffu;
    int qn = 0;
    unsigned long long nh = 0;
    const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t v = wg; v < n; v += nw) {
        const int64_t s0 = xadj[v], s1 = xadj[v + 1];
        for (int c0 = 0; c0 < nq; c0 += 32) {
            const int qd = c0 + lane;
            const bool active = qd < nq;
            int4 x = make_int4(0, 0, 0, 0);
            if (active) x = smem4[qd];
            const int r = qd << 2;
            unsigned valid = 0xFu;
            if (r + 4 > W) valid = (1u << (W > r ? W - r : 0)) - 1u;
            if (!active) valid = 0;
            uint32_t best[4] = {(uint32_t)v, (uint32_t)v, (uint32_t)v, (uint32_t)v};
            unsigned seen = 0;
            for (int64_t sl = s0; sl < s1; ++sl) {
                const uint32_t u = (uint32_t)__ldg(adj + sl);
                if (u >= (uint32_t)v) break;
                const int32_t h = __ldg(hash + sl);
                const int32_t t = UNI ? tu : __ldg(thr + sl);
                unsigned live = ((unsigned)((x.x ^ h) < t)) | ((unsigned)((x.y ^ h) < t) << 1) |
                                ((unsigned)((x.z ^ h) < t) << 2) | ((unsigned)((x.w ^ h) < t) << 3);
                live &= valid;
                if (PASS == 1) {
                    unsigned fresh = live & ~seen;
                    while (fresh) {
                        const int j = __ffs(fresh) - 1;
                        fresh &= fresh - 1;
                        best[j] = u;
                    }
                    seen |= live;
                } else {
                    unsigned rest = live & seen;
                    seen |= live;
                    if (!__any_sync(FULL, rest != 0)) continue;
                    const int k = __popc(rest);
                    int inc = k;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int y = __shfl_up_sync(FULL, inc, o);
                        if (lane >= o) inc += y;
                    }
                    int pos = qn + inc - k;
                    while (rest) {
                        const int b = __ffs(rest) - 1;
                        rest &= rest - 1;
                        qlo[pos] = u;
                        qhi[pos] = (uint32_t)v;
                        qr[pos] = (uint32_t)(r + b);
                        ++pos;
                    }
                    qn += __shfl_sync(FULL, inc, 31);
                    __syncwarp();
                    while (qn >= 32) {
                        qn -= 32;
                        const uint32_t a = qlo[qn + lane], bb = qhi[qn + lane];
                        const int rr = (int)qr[qn + lane];
                        __syncwarp();
                        nh += unite(L, ld, a, bb, rr);
                    }
                }
            }
            if (PASS == 1 && active) {
                *(reinterpret_cast<uint4 *>(L + v * ld) + qd) = make_uint4(best[0], best[1], best[2], best[3]);
                *(reinterpret_cast<uint4 *>(C + v * ld) + qd) = make_uint4(0, 0, 0, 0);
            }
        }
    }
    if (PASS == 2) {
        __syncwarp();
        if (lane < qn) nh += unite(L, ld, qlo[lane], qhi[lane], (int)qr[lane]);
    }
    if (hooks) {
        for (int o = 16; o; o >>= 1) nh += __shfl_xor_sync(FULL, nh, o);
        if (lane == 0 && nh) atomicAdd(hooks, nh);
    }
}

// Full compression + component histogram, one thread per 16-byte quad of a
// label row (full occupancy; the latency of the root searches is hidden by
// thread-level parallelism).  The searches re-point every visited node at its
// grandparent with atomicMin (path splitting): concurrent owners store the
// final root, the smallest id of the tree, so min-updates can never undo a
// finished label.  Non-root cells add 1 to C[root][r].
__device__ __forceinline__ uint32_t find_split(uint32_t *L, int64_t ld, uint32_t x, uint32_t p, int r) {
    for (;;) {
        const uint32_t gp = ld_relaxed(cell(L, ld, p, r));
        if (gp == p) return p;
        atomicMin(cell(L, ld, x, r), gp);
        x = p;
        p = gp;
    }
}

__global__ void __launch_bounds__(256) k_compress(uint32_t *__restrict__ L, uint32_t *__restrict__ C,
                                                  int64_t n, int64_t ld, int32_t W,
                                                  unsigned long long *__restrict__ changed) {
    const int64_t nq = ld >> 2;
    unsigned long long nch = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * nq;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = i / nq;
        const int r = (int)(i - v * nq) << 2;
        uint4 *p4 = reinterpret_cast<uint4 *>(L) + i;
        const uint4 l = *p4;
        uint32_t lv[4] = {l.x, l.y, l.z, l.w};
        uint32_t par[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
            par[j] = (r + j < W && lv[j] != (uint32_t)v) ? ld_relaxed(cell(L, ld, lv[j], r + j)) : lv[j];
        bool any = false;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t x = lv[j];
            if (r + j >= W || x == (uint32_t)v) continue;
            const uint32_t root = (par[j] == x) ? x : find_split(L, ld, x, par[j], r + j);
            if (root != x) { lv[j] = root; any = true; }
            ++nch;   // non-root cell: its label moved off the identity
            atomicAdd(C + (int64_t)root * ld + r + j, 1u);
        }
        if (any) *p4 = make_uint4(lv[0], lv[1], lv[2], lv[3]);
    }
    if (changed) {
        for (int o = 16; o; o >>= 1) nch += __shfl_xor_sync(0xffffffffu, nch, o);
        if ((threadIdx.x & 31) == 0 && nch) atomicAdd(changed, nch);
    }
}

// Verification sweep: count live (edge, lane) pairs whose endpoint labels
// differ and labels that are not roots / exceed their vertex.
template <bool UNI>
__global__ void k_verify_edges(const int2 *__restrict__ E, const int32_t *__restrict__ EH,
                               const int32_t *__restrict__ ET, int32_t tu, int64_t me,
                               const int32_t *__restrict__ X, int32_t W, int64_t ld,
                               const uint32_t *__restrict__ L, unsigned long long *__restrict__ bad) {
    const int lane = threadIdx.x & 31;
    const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long nb = 0;
    for (int64_t e = wg; e < me; e += nw) {
        const int2 uv = E[e];
        const int32_t h = EH[e];
        const int32_t t = UNI ? tu : ET[e];
        for (int r = lane; r < W; r += 32)
            if ((X[r] ^ h) < t && L[(int64_t)uv.x * ld + r] != L[(int64_t)uv.y * ld + r]) ++nb;
    }
    for (int o = 16; o; o >>= 1) nb += __shfl_xor_sync(0xffffffffu, nb, o);
    if (lane == 0 && nb) atomicAdd(bad, nb);
}
__global__ void k_verify_roots(const uint32_t *__restrict__ L, int64_t n, int64_t ld, int32_t W,
                               unsigned long long *__restrict__ bad) {
    unsigned long long nb = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * (int64_t)W;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t v = i / W;
        int r = (int)(i - v * W);
        uint32_t l = L[v * ld + r];
        if (l > (uint32_t)v || L[(int64_t)l * ld + r] != l) ++nb;
    }
    for (int o = 16; o; o >>= 1) nb += __shfl_xor_sync(0xffffffffu, nb, o);
    if ((threadIdx.x & 31) == 0 && nb) atomicAdd(bad, nb);
}

__global__ void k_label_sum(const uint32_t *__restrict__ L, int64_t n, int64_t ld, int32_t W,
                            unsigned long long *__restrict__ out) {
    unsigned long long s = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * (int64_t)W;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t v = i / W;
        int r = (int)(i - v * W);
        s += L[v * ld + r];
    }
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

// ---------------------------------------------------------------------------
// K4/K5: gains[v] = sum_{r < ns} size(L[v][r], r)   (propagation.py:359-368)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_gains(const uint32_t *__restrict__ L, const uint32_t *__restrict__ C,
                                               int64_t n, int64_t ld, int32_t ns, uint32_t add1,
                                               int64_t *__restrict__ gains) {
    const int lane = threadIdx.x & 31;
    const int nqs = (ns + 3) >> 2;
    const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t v = wg; v < n; v += nw) {
        const uint4 *Lr = reinterpret_cast<const uint4 *>(L + v * ld);
        const uint4 *Cr = reinterpret_cast<const uint4 *>(C + v * ld);
        unsigned long long acc = 0;
        for (int q = lane; q < nqs; q += 32) {
            const uint4 l = __ldg(Lr + q), c = __ldg(Cr + q);
            const uint32_t lv[4] = {l.x, l.y, l.z, l.w}, cv[4] = {c.x, c.y, c.z, c.w};
            const int r = q << 2;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (r + j >= ns) break;
                uint32_t cnt = (lv[j] == (uint32_t)v) ? cv[j] : __ldg(C + (int64_t)lv[j] * ld + r + j);
                acc += cnt + add1;
            }
        }
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) gains[v] = (int64_t)acc;
    }
}

// sizes[v][r] for a lane window (C + own-root indicator)
__global__ void k_sizes_window(const uint32_t *__restrict__ L, const uint32_t *__restrict__ C,
                               int64_t v0, int64_t cnt, int64_t ld, int32_t r0, int32_t r1,
                               int full_counts, int32_t *__restrict__ out) {
    const int w = r1 - r0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt * (int64_t)w;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t v = v0 + i / w;
        int r = r0 + (int)(i % w);
        uint32_t c = C[v * ld + r];
        out[i] = (int32_t)(c + (!full_counts && L[v * ld + r] == (uint32_t)v ? 1u : 0u));
    }
}
__global__ void k_gather_i64(const int32_t *__restrict__ idx, int64_t cnt,
                             const int64_t *__restrict__ src, int64_t *__restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = src[idx[i]];
}
// Host-provided labels may be arbitrary (any int in 0..n-1), so C holds
// full counts for them (full_counts = 1: size = C[l][r], not C[l][r] + 1).
__global__ void k_hist_full(const uint32_t *__restrict__ L, uint32_t *__restrict__ C,
                            int64_t n, int64_t ld, int32_t W, unsigned *__restrict__ bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * (int64_t)W;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t v = i / W;
        int r = (int)(i - v * W);
        uint32_t l = L[v * ld + r];
        if (l >= (uint32_t)n) { atomicOr(bad, 1u); continue; }
        atomicAdd(C + (int64_t)l * ld + r, 1u);
    }
}

// ---------------------------------------------------------------------------
// K6-K8: CELF
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long pack_key(int64_t prio, uint32_t v, int vb) {
    const uint32_t vmask = (vb >= 32) ? 0xffffffffu : ((1u << vb) - 1u);
    return ((unsigned long long)prio << vb) | (unsigned long long)(vmask - v);
}

__global__ void k_top(const int64_t *__restrict__ prio, const uint8_t *__restrict__ inS, int64_t n,
                      int vb, unsigned long long *__restrict__ out) {
    unsigned long long best = 0;
    bool have = false;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        if (inS[v]) continue;
        unsigned long long k = pack_key(prio[v], (uint32_t)v, vb) + 1ull;  // +1: 0 = none
        if (!have || k > best) { best = k; have = true; }
    }
    for (int o = 16; o; o >>= 1) {
        unsigned long long x = __shfl_xor_sync(0xffffffffu, best, o);
        best = x > best ? x : best;
    }
    if ((threadIdx.x & 31) == 0 && best) atomicMax(out, best);
}

__global__ void k_collect(const int64_t *__restrict__ prio, const uint8_t *__restrict__ inS, int64_t n,
                          int vb, unsigned long long thr_key, int32_t exclude,
                          int32_t *__restrict__ cand, unsigned long long *__restrict__ count) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        bool take = !inS[v] && v != exclude && pack_key(prio[v], (uint32_t)v, vb) >= thr_key;
        unsigned m = __ballot_sync(__activemask(), take);
        if (!m) continue;
        int leader = __ffs(m) - 1;
        unsigned long long base = 0;
        if ((threadIdx.x & 31) == leader) base = atomicAdd(count, (unsigned long long)__popc(m));
        base = __shfl_sync(__activemask(), base, leader);
        if (take) cand[base + __popc(m & ((1u << (threadIdx.x & 31)) - 1u))] = (int32_t)v;
    }
}

// marginal_gain (selection.py:63-70): sum over scored lanes of the component
// size of L[u][r] when that component is not covered yet.  One CTA per
// candidate; each thread takes 16-byte quads of the label row so the label
// loads are coalesced and the dependent cov/size gathers of 4 lanes are in
// flight together.
constexpr int kEvalThreads = 128;
__global__ void __launch_bounds__(kEvalThreads) k_eval(const int32_t *__restrict__ cand, int64_t cnt,
                                                       const uint32_t *__restrict__ L, const uint32_t *__restrict__ C,
                                                       const uint32_t *__restrict__ cov, int64_t ld, int32_t ns,
                                                       int32_t cw, int full_counts,
                                                       int64_t *__restrict__ out) {
    __shared__ unsigned long long part[kEvalThreads / 32];
    const uint32_t add1 = full_counts ? 0u : 1u;
    const int nqs = (ns + 3) >> 2;
    for (int64_t i = blockIdx.x; i < cnt; i += gridDim.x) {
        const int64_t u = cand[i];
        if (u < 0) { if (threadIdx.x == 0) out[i] = 0; continue; }
        const uint4 *row = reinterpret_cast<const uint4 *>(L + u * ld);
        unsigned long long acc = 0;
        for (int q = threadIdx.x; q < nqs; q += kEvalThreads) {
            const uint4 l4 = row[q];
            const uint32_t lv[4] = {l4.x, l4.y, l4.z, l4.w};
            uint32_t w[4], s[4];
            const int r = q << 2;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const bool in = r + j < ns;
                w[j] = in ? cov[(int64_t)lv[j] * cw + ((r + j) >> 5)] : 0xffffffffu;
                s[j] = in ? C[(int64_t)lv[j] * ld + r + j] : 0u;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (!((w[j] >> ((r + j) & 31)) & 1u)) acc += s[j] + add1;
        }
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long t = 0;
            for (int k = 0; k < kEvalThreads / 32; ++k) t += part[k];
            out[i] = (int64_t)t;
        }
        __syncthreads();
    }
}

// commit_seed (selection.py:73-81)
__global__ void k_commit(int32_t u, const uint32_t *__restrict__ L, const uint32_t *__restrict__ C,
                         uint32_t *__restrict__ cov, int64_t ld, int32_t ns, int32_t cw,
                         int full_counts, int64_t *__restrict__ per_sim, uint8_t *__restrict__ inS,
                         unsigned long long *__restrict__ gain) {
    unsigned long long acc = 0;
    const uint32_t add1 = full_counts ? 0u : 1u;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < ns; r += gridDim.x * blockDim.x) {
        const uint32_t l = L[(int64_t)u * ld + r];
        const uint32_t bit = 1u << (r & 31);
        const uint32_t old = atomicOr(cov + (int64_t)l * cw + (r >> 5), bit);
        if (!(old & bit)) {
            const uint32_t s = C[(int64_t)l * ld + r] + add1;
            per_sim[r] += s;
            acc += s;
        }
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(gain, acc);
    if (blockIdx.x == 0 && threadIdx.x == 0) inS[u] = 1;
}

// CELF round header (scratch[8..12]): 0 top key+1, 1 fresh gain of the top,
// 2 collected count, 3 gain of the last commit, 4 collect threshold key.
enum { H_TOP = 0, H_F1 = 1, H_COUNT = 2, H_GAIN = 3, H_THR = 4 };

__global__ void k_round_decode(const unsigned long long *__restrict__ hdr, int vb, int32_t *__restrict__ one) {
    unsigned long long key = hdr[H_TOP];
    const uint32_t vmask = (vb >= 32) ? 0xffffffffu : ((1u << vb) - 1u);
    one[0] = key ? (int32_t)(vmask - (uint32_t)((key - 1) & vmask)) : -1;
}

__global__ void k_make_thr(unsigned long long *__restrict__ hdr, const int64_t *__restrict__ f1,
                           const int32_t *__restrict__ one, int vb) {
    const int32_t v = one[0];
    hdr[H_F1] = (unsigned long long)f1[0];
    hdr[H_THR] = v < 0 ? ~0ull : pack_key(f1[0], (uint32_t)v, vb);
}

// k_collect with the threshold key and the excluded vertex read from device memory
__global__ void k_collect_dev(const int64_t *__restrict__ prio, const uint8_t *__restrict__ inS, int64_t n,
                              int vb, const unsigned long long *__restrict__ hdr,
                              const int32_t *__restrict__ one, int32_t *__restrict__ cand,
                              unsigned long long *__restrict__ count) {
    const unsigned long long thr_key = hdr[H_THR];
    const int32_t exclude = one[0];
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        bool take = !inS[v] && v != exclude && pack_key(prio[v], (uint32_t)v, vb) >= thr_key;
        unsigned m = __ballot_sync(__activemask(), take);
        if (!m) continue;
        int leader = __ffs(m) - 1;
        unsigned long long base = 0;
        if ((threadIdx.x & 31) == leader) base = atomicAdd(count, (unsigned long long)__popc(m));
        base = __shfl_sync(__activemask(), base, leader);
        if (take) cand[base + __popc(m & ((1u << (threadIdx.x & 31)) - 1u))] = (int32_t)v;
    }
}

__global__ void k_keys_of(const int32_t *__restrict__ ids, int64_t cnt, const int64_t *__restrict__ prio,
                          int vb, unsigned long long *__restrict__ keys) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
         i += (int64_t)gridDim.x * blockDim.x)
        keys[i] = pack_key(prio[ids[i]], (uint32_t)ids[i], vb);
}

__global__ void k_set_prio(const int32_t *__restrict__ ids, const int64_t *__restrict__ vals,
                           int64_t cnt, int64_t *__restrict__ prio) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
         i += (int64_t)gridDim.x * blockDim.x)
        prio[ids[i]] = vals[i];
}

static int grid_for(int64_t work, int threads = 256) {
    int64_t b = ceil_div(work > 0 ? work : 1, threads);
    if (b > 148 * 16) b = 148 * 16;
    return (int)b;
}

}  // namespace imx

using namespace imx;

// ---------------------------------------------------------------------------
// context lifecycle
// ---------------------------------------------------------------------------
// The label/count matrices come from the device's stream-ordered pool with an
// unbounded release threshold, so back-to-back runs on the same graph reuse
// the memory instead of paying cudaMalloc/cudaFree every time.
static cudaError_t pool_alloc(void **p, size_t bytes, cudaStream_t st) {
    static bool configured[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64 && !configured[dev]) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        configured[dev] = true;
    }
    return cudaMallocAsync(p, bytes, st);
}

static void ctx_free(imx_ctx *c) {
    if (!c) return;
    cudaSetDevice(c->dev);
    if (c->st) cudaStreamSynchronize(c->st);
    if (c->L) cudaFreeAsync(c->L, c->st);
    if (c->C) cudaFreeAsync(c->C, c->st);
    c->L = c->C = nullptr;
    if (c->st) cudaStreamSynchronize(c->st);
    void *ptrs[] = {c->X, c->L, c->C, c->gains, c->prio, c->inS, c->cov, c->per_sim,
                    c->cand, c->fresh, c->scratch, c->cand2, c->keys2, c->eval_out, c->d_one,
                    c->sort_tmp, c->d_ids, c->d_vals, c->seg_a, c->seg_n, c->seg_off, c->scan_tmp};
    for (void *p : ptrs) if (p) cudaFree(p);
    if (c->h_ids) cudaFreeHost(c->h_ids);
    if (c->h_vals) cudaFreeHost(c->h_vals);
    for (auto &e : c->ev) if (e) cudaEventDestroy(e);
    if (c->st) cudaStreamDestroy(c->st);
    delete c;
}

#define CTX_CHECK(c)                                                       \
    do {                                                                   \
        if (!(c)) { set_error("context is NULL"); return IMX_EINVAL; }     \
        IMX_CUDA(cudaSetDevice((c)->dev));                                 \
    } while (0)

extern "C" int imx_create(imx_graph *g, const int32_t *X, int32_t width, int32_t num_scored,
                          imx_ctx **out) {
    if (!out) { set_error("out is NULL"); return IMX_EINVAL; }
    *out = nullptr;
    if (!g) { set_error("graph is NULL"); return IMX_EINVAL; }
    if (width < 1) { set_error("simulation width %d must be positive", width); return IMX_EINVAL; }
    if (num_scored < 0 || num_scored > width) {
        set_error("num_scored %d outside [0, %d]", num_scored, width);
        return IMX_EINVAL;
    }
    if (!X) { set_error("X is NULL"); return IMX_EINVAL; }
    for (int32_t r = 0; r < width; ++r)
        if (X[r] < 0) { set_error("simulation word %d is negative (must be 31-bit)", r); return IMX_EINVAL; }
    if (!g->symmetric) { set_error("adjacency is not symmetric"); return IMX_EFORMAT; }
    IMX_CUDA(cudaSetDevice(g->dev));
    imx_ctx *c = new imx_ctx();
    c->g = g;
    c->dev = g->dev;
    c->W = width;
    c->ns = num_scored;
    c->ld = (width + 3) & ~3;
    c->cw = (num_scored + 31) / 32;
    if (c->cw == 0) c->cw = 1;
    int vb = 1;
    while ((int64_t(1) << vb) < g->n + 1) ++vb;
    c->vb = vb;
    for (auto &e : c->ev) e = nullptr;
    const int64_t n = g->n;
    auto fail = [&](int code) { ctx_free(c); return code; };
    if (cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking) != cudaSuccess) return fail(IMX_ECUDA);
    for (auto &e : c->ev)
        if (cudaEventCreate(&e) != cudaSuccess) return fail(IMX_ECUDA);
    const size_t cells = (size_t)(n > 0 ? n : 1) * (size_t)c->ld;
    cudaError_t e = cudaSuccess;
    if ((e = cudaMalloc((void **)&c->X, sizeof(int32_t) * c->ld)) != cudaSuccess ||
        (e = pool_alloc((void **)&c->L, sizeof(uint32_t) * cells, c->st)) != cudaSuccess ||
        (e = pool_alloc((void **)&c->C, sizeof(uint32_t) * cells, c->st)) != cudaSuccess ||
        (e = cudaMalloc((void **)&c->gains, sizeof(int64_t) * (n + 1))) != cudaSuccess ||
        (e = cudaMalloc((void **)&c->scratch, sizeof(unsigned long long) * 16)) != cudaSuccess) {
        return fail(cuda_fail(e, "cudaMalloc(context)", __FILE__, __LINE__));
    }
    std::vector<int32_t> xpad(c->ld, 0);
    std::copy(X, X + width, xpad.begin());
    if ((e = cudaMemcpy(c->X, xpad.data(), sizeof(int32_t) * c->ld, cudaMemcpyHostToDevice)) != cudaSuccess)
        return fail(cuda_fail(e, "upload X", __FILE__, __LINE__));
    *out = c;
    return IMX_OK;
}

extern "C" void imx_destroy(imx_ctx *c) { ctx_free(c); }

static int ensure_celf_buffers(imx_ctx *c) {
    if (c->prio) return IMX_OK;
    const int64_t n = c->g->n > 0 ? c->g->n : 1;
    IMX_CUDA(cudaMalloc((void **)&c->prio, sizeof(int64_t) * n));
    IMX_CUDA(cudaMalloc((void **)&c->inS, n));
    IMX_CUDA(cudaMalloc((void **)&c->cov, sizeof(uint32_t) * (size_t)n * c->cw));
    IMX_CUDA(cudaMalloc((void **)&c->per_sim, sizeof(int64_t) * (c->W + 1)));
    IMX_CUDA(cudaMalloc((void **)&c->cand, sizeof(int32_t) * n));
    IMX_CUDA(cudaMalloc((void **)&c->fresh, sizeof(int64_t) * n));
    IMX_CUDA(cudaMalloc((void **)&c->cand2, sizeof(int32_t) * n));
    IMX_CUDA(cudaMalloc((void **)&c->keys2, sizeof(unsigned long long) * n));
    IMX_CUDA(cudaMalloc((void **)&c->eval_out, sizeof(int64_t) * n));
    IMX_CUDA(cudaMalloc((void **)&c->d_one, sizeof(int32_t) * 4));
    return IMX_OK;
}

static int ensure_pinned(imx_ctx *c, int64_t cnt) {
    if (cnt <= c->stage_cap) return IMX_OK;
    int64_t cap = std::max<int64_t>(cnt, 4096);
    if (c->h_ids) cudaFreeHost(c->h_ids);
    if (c->h_vals) cudaFreeHost(c->h_vals);
    if (c->d_ids) cudaFree(c->d_ids);
    if (c->d_vals) cudaFree(c->d_vals);
    c->h_ids = nullptr; c->h_vals = nullptr; c->d_ids = nullptr; c->d_vals = nullptr;
    c->stage_cap = 0;
    IMX_CUDA(cudaStreamSynchronize(c->st));
    IMX_CUDA(cudaMallocHost((void **)&c->h_ids, sizeof(int32_t) * cap));
    IMX_CUDA(cudaMallocHost((void **)&c->h_vals, sizeof(int64_t) * cap));
    IMX_CUDA(cudaMalloc((void **)&c->d_ids, sizeof(int32_t) * cap));
    IMX_CUDA(cudaMalloc((void **)&c->d_vals, sizeof(int64_t) * cap));
    c->stage_cap = cap;
    return IMX_OK;
}

static inline void count_launch(imx_ctx *c, int k = 1) { c->tm.kernel_launches += k; note_launch(k); }

// phases -----------------------------------------------------------------
static int run_init(imx_ctx *c) {
    const int64_t n = c->g->n;
    if (n == 0) return IMX_OK;
    k_init<<<grid_for(n * (c->ld >> 2)), 256, 0, c->st>>>(c->L, n, c->ld);
    IMX_CHECK_LAUNCH();
    IMX_CUDA(cudaMemsetAsync(c->C, 0, sizeof(uint32_t) * (size_t)n * c->ld, c->st));
    count_launch(c, 1);
    return IMX_OK;
}

static int run_hook_dense(imx_ctx *c, unsigned long long *hooks) {
    imx_graph *g = c->g;
    const size_t smem = sizeof(int32_t) * c->ld + sizeof(uint32_t) * 3 * kQ * kHookWarps;
    if (smem > 200 * 1024) { set_error("width %d too large for one context", c->W); return IMX_EINVAL; }
    const int64_t tiles = ceil_div(g->me, 32);
    int blocks = (int)std::min<int64_t>(ceil_div(tiles, kHookWarps), 148 * 8);
    auto kern = g->uniform ? k_hook<true> : k_hook<false>;
    if (smem > 48 * 1024) IMX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<blocks, kHookWarps * 32, smem, c->st>>>(g->E, g->EH, g->ET, g->thr_u, g->me, c->X, c->W,
                                                    c->ld, c->L, hooks);
    IMX_CHECK_LAUNCH();
    count_launch(c);
    return IMX_OK;
}

static int run_hook_enum(imx_ctx *c, unsigned long long *hooks) {
    imx_graph *g = c->g;
    const int64_t nseg = (int64_t)c->W * g->nb * 31;
    if (nseg + 1 > c->nseg_cap) {
        for (int64_t **p : {&c->seg_a, &c->seg_n, &c->seg_off}) { if (*p) cudaFree(*p); *p = nullptr; }
        c->nseg_cap = 0;
        IMX_CUDA(cudaMalloc((void **)&c->seg_a, sizeof(int64_t) * (nseg + 1)));
        IMX_CUDA(cudaMalloc((void **)&c->seg_n, sizeof(int64_t) * (nseg + 1)));
        IMX_CUDA(cudaMalloc((void **)&c->seg_off, sizeof(int64_t) * (nseg + 1)));
        c->nseg_cap = nseg + 1;
        size_t tb = 0;
        IMX_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, c->seg_n, c->seg_off, nseg + 1, c->st));
        if (tb > c->scan_tmp_bytes) {
            if (c->scan_tmp) cudaFree(c->scan_tmp);
            IMX_CUDA(cudaMalloc(&c->scan_tmp, tb));
            c->scan_tmp_bytes = tb;
        }
    }
    k_seg_count<<<grid_for(nseg), 256, 0, c->st>>>(c->X, c->W, g->nb, g->btmax, g->boff, g->EH,
                                                   c->seg_a, c->seg_n);
    IMX_CHECK_LAUNCH();
    size_t tb = c->scan_tmp_bytes;
    IMX_CUDA(cub::DeviceScan::ExclusiveSum(c->scan_tmp, tb, c->seg_n, c->seg_off, nseg + 1, c->st));
    const int blocks = 148 * 8;
    if (g->uniform)
        k_hook_enum<true><<<blocks, 256, 0, c->st>>>(c->seg_off, c->seg_a, nseg, g->nb * 31, g->E, g->EH,
                                                     g->ET, c->X, c->ld, c->L, hooks);
    else
        k_hook_enum<false><<<blocks, 256, 0, c->st>>>(c->seg_off, c->seg_a, nseg, g->nb * 31, g->E, g->EH,
                                                      g->ET, c->X, c->ld, c->L, hooks);
    IMX_CHECK_LAUNCH();
    count_launch(c, 3);
    return IMX_OK;
}

static int run_pull(imx_ctx *c, int pass, unsigned long long *hooks) {
    imx_graph *g = c->g;
    const int64_t n = g->n;
    if (n == 0) return IMX_OK;
    const size_t smem = sizeof(int32_t) * c->ld + sizeof(uint32_t) * 3 * kQ * 8;
    if (smem > 200 * 1024) { set_error("width %d too large for one context", c->W); return IMX_EINVAL; }
    const int blocks = (int)std::min<int64_t>(ceil_div(n, 8), 148 * 8);
    auto kern = pass == 1 ? (g->uniform ? k_pull<1, true> : k_pull<1, false>)
                          : (g->uniform ? k_pull<2, true> : k_pull<2, false>);
    if (smem > 48 * 1024) IMX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<blocks, 256, smem, c->st>>>(g->xadj, g->adj, g->hash, g->thr, g->thr_u, n, c->X, c->W, c->ld,
                                       c->L, c->C, hooks);
    IMX_CHECK_LAUNCH();
    count_launch(c);
    return IMX_OK;
}

// Sampler strategy.  Interval enumeration touches only live (edge, lane)
// pairs but each costs ~4 random label accesses; the pull passes cost two
// dense membership scans (ALU only) and random accesses for the non-forest
// live edges only.  Measured crossover on B200: live fraction ~2%.
enum { HOOK_ENUM = 0, HOOK_PULL = 1, HOOK_DENSE = 2 };
static int hook_mode(const imx_graph *g) {
    const char *m = getenv("IMX_HOOK");
    if (m && !strcmp(m, "dense")) return HOOK_DENSE;
    if (m && !strcmp(m, "enum")) return HOOK_ENUM;
    if (m && !strcmp(m, "pull")) return HOOK_PULL;
    const char *t = getenv("IMX_PULL_MIN_P");
    const double thr = t ? atof(t) : 0.02;
    return g->thr_mean >= thr ? HOOK_PULL : HOOK_ENUM;
}

// init + hook phases of one propagate (events 1 and 2 bracket them)
static int run_sample_cc(imx_ctx *c, unsigned long long *hooks, cudaEvent_t e_init, cudaEvent_t e_hook) {
    imx_graph *g = c->g;
    const int mode = g->me ? hook_mode(g) : HOOK_ENUM;
    if (mode == HOOK_PULL) {
        IMX_TRY(run_pull(c, 1, nullptr));
        if (e_init) IMX_CUDA(cudaEventRecord(e_init, c->st));
        IMX_TRY(run_pull(c, 2, hooks));
    } else {
        IMX_TRY(run_init(c));
        if (e_init) IMX_CUDA(cudaEventRecord(e_init, c->st));
        if (g->me) IMX_TRY(mode == HOOK_DENSE ? run_hook_dense(c, hooks) : run_hook_enum(c, hooks));
    }
    if (e_hook) IMX_CUDA(cudaEventRecord(e_hook, c->st));
    c->tm.hook_launches++;
    return IMX_OK;
}

static int run_compress(imx_ctx *c, unsigned long long *changed) {
    const int64_t n = c->g->n;
    if (n == 0) return IMX_OK;
    k_compress<<<grid_for(n * (c->ld >> 2)), 256, 0, c->st>>>(c->L, c->C, n, c->ld, c->W, changed);
    IMX_CHECK_LAUNCH();
    count_launch(c);
    return IMX_OK;
}

static int label_sum(imx_ctx *c, int64_t *out) {
    const int64_t n = c->g->n;
    IMX_CUDA(cudaMemsetAsync(c->scratch + 4, 0, sizeof(unsigned long long), c->st));
    if (n) {
        k_label_sum<<<grid_for(n * c->W), 256, 0, c->st>>>(c->L, n, c->ld, c->W, c->scratch + 4);
        IMX_CHECK_LAUNCH();
        count_launch(c);
    }
    unsigned long long s = 0;
    IMX_CUDA(cudaMemcpyAsync(&s, c->scratch + 4, sizeof s, cudaMemcpyDeviceToHost, c->st));
    IMX_CUDA(cudaStreamSynchronize(c->st));
    *out = (int64_t)s;
    return IMX_OK;
}

static void push_stat(imx_prop_stats *st, int mode, int64_t changed, int64_t lsum) {
    if (!st) return;
    int i = st->sweeps++;
    if (i < st->cap) {
        if (st->changed_pairs) st->changed_pairs[i] = changed;
        if (st->label_sums) st->label_sums[i] = lsum;
        if (st->modes) st->modes[i] = mode;
    }
}

extern "C" int imx_propagate(imx_ctx *c, int32_t verify, imx_prop_stats *st) {
    CTX_CHECK(c);
    imx_graph *g = c->g;
    const int64_t n = g->n;
    if (st) st->sweeps = 0;
    unsigned long long *sc = c->scratch;
    IMX_CUDA(cudaMemsetAsync(sc, 0, sizeof(unsigned long long) * 4, c->st));
    IMX_CUDA(cudaEventRecord(c->ev[0], c->st));
    if (g->m2 > 0) {
        IMX_TRY(run_sample_cc(c, st ? sc : nullptr, c->ev[1], c->ev[2]));
        IMX_TRY(run_compress(c, st ? sc + 1 : nullptr));
        IMX_CUDA(cudaEventRecord(c->ev[3], c->st));
    } else {
        IMX_TRY(run_init(c));
        IMX_CUDA(cudaEventRecord(c->ev[1], c->st));
        IMX_CUDA(cudaEventRecord(c->ev[2], c->st));
        IMX_CUDA(cudaEventRecord(c->ev[3], c->st));
    }
    IMX_CUDA(cudaEventSynchronize(c->ev[3]));
    cudaEventElapsedTime(&c->tm.init_ms, c->ev[0], c->ev[1]);
    cudaEventElapsedTime(&c->tm.hook_ms, c->ev[1], c->ev[2]);
    cudaEventElapsedTime(&c->tm.compress_ms, c->ev[2], c->ev[3]);
    cudaEventElapsedTime(&c->tm.propagate_ms, c->ev[0], c->ev[3]);
    c->labels_ready = true;
    c->memo_ready = false;
    c->celf_ready = false;
    c->full_counts = 0;
    if (g->m2 == 0) return IMX_OK;  // propagation.py:276-278: edgeless -> identity, no sweeps
    // One union-find pass reaches the fixpoint: it is reported as one sweep
    // whose changed count is the number of (vertex, lane) labels that moved
    // off the identity, followed (when asked) by the no-change sweep that
    // proves convergence, as the reference's loop does (propagation.py:304-320).
    int64_t changed = 0, lsum = 0;
    if (st) {
        unsigned long long hc[2];
        IMX_CUDA(cudaMemcpyAsync(hc, sc, sizeof hc, cudaMemcpyDeviceToHost, c->st));
        IMX_CUDA(cudaStreamSynchronize(c->st));
        IMX_TRY(label_sum(c, &lsum));
        changed = (int64_t)hc[1];  // non-root cells = labels moved off the identity
        push_stat(st, IMX_MODE_HOOK, changed, lsum);
    }
    if (verify || (st && changed > 0)) {
        IMX_CUDA(cudaMemsetAsync(sc + 2, 0, sizeof(unsigned long long), c->st));
        if (g->me) {
            if (g->uniform)
                k_verify_edges<true><<<grid_for(g->me * 32), 256, 0, c->st>>>(g->E, g->EH, g->ET, g->thr_u, g->me, c->X, c->W, c->ld, c->L, sc + 2);
            else
                k_verify_edges<false><<<grid_for(g->me * 32), 256, 0, c->st>>>(g->E, g->EH, g->ET, g->thr_u, g->me, c->X, c->W, c->ld, c->L, sc + 2);
            IMX_CHECK_LAUNCH();
        }
        k_verify_roots<<<grid_for(n * c->W), 256, 0, c->st>>>(c->L, n, c->ld, c->W, sc + 2);
        IMX_CHECK_LAUNCH();
        count_launch(c, 2);
        unsigned long long bad = 0;
        IMX_CUDA(cudaMemcpyAsync(&bad, sc + 2, sizeof bad, cudaMemcpyDeviceToHost, c->st));
        IMX_CUDA(cudaStreamSynchronize(c->st));
        if (bad) {
            set_error("propagation self-check failed: %llu violations", bad);
            return IMX_EINTERNAL;
        }
        if (st && changed > 0) push_stat(st, IMX_MODE_VERIFY, 0, lsum);
    }
    return IMX_OK;
}

extern "C" int imx_memoize(imx_ctx *c, int64_t *gains_out) {
    CTX_CHECK(c);
    if (!c->labels_ready) { set_error("labels not computed (call imx_propagate first)"); return IMX_EINVAL; }
    const int64_t n = c->g->n;
    IMX_CUDA(cudaEventRecord(c->ev[4], c->st));
    if (n) {
        k_gains<<<grid_for(n * 32), 256, 0, c->st>>>(c->L, c->C, n, c->ld, c->ns,
                                                     c->full_counts ? 0u : 1u, c->gains);
        IMX_CHECK_LAUNCH();
        count_launch(c);
    }
    IMX_CUDA(cudaEventRecord(c->ev[5], c->st));
    if (gains_out && n)
        IMX_CUDA(cudaMemcpyAsync(gains_out, c->gains, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, c->st));
    IMX_CUDA(cudaStreamSynchronize(c->st));
    cudaEventElapsedTime(&c->tm.memoize_ms, c->ev[4], c->ev[5]);
    c->memo_ready = true;
    return IMX_OK;
}

extern "C" int imx_load_labels(imx_ctx *c, const int32_t *labels, const int32_t *sizes, int64_t ldh) {
    CTX_CHECK(c);
    const int64_t n = c->g->n;
    if (!labels && n) { set_error("labels is NULL"); return IMX_EINVAL; }
    if (ldh < c->W) { set_error("row stride %lld < width %d", (long long)ldh, c->W); return IMX_EINVAL; }
    if (n) {
        IMX_CUDA(cudaMemsetAsync(c->L, 0, sizeof(uint32_t) * (size_t)n * c->ld, c->st));
        IMX_CUDA(cudaMemcpy2DAsync(c->L, sizeof(uint32_t) * c->ld, labels, sizeof(int32_t) * ldh,
                                   sizeof(int32_t) * c->W, n, cudaMemcpyHostToDevice, c->st));
        unsigned *bad = reinterpret_cast<unsigned *>(c->scratch + 6);
        IMX_CUDA(cudaMemsetAsync(bad, 0, sizeof(unsigned), c->st));
        if (sizes) {
            IMX_CUDA(cudaMemsetAsync(c->C, 0, sizeof(uint32_t) * (size_t)n * c->ld, c->st));
            IMX_CUDA(cudaMemcpy2DAsync(c->C, sizeof(uint32_t) * c->ld, sizes, sizeof(int32_t) * ldh,
                                       sizeof(int32_t) * c->W, n, cudaMemcpyHostToDevice, c->st));
        } else {
            IMX_CUDA(cudaMemsetAsync(c->C, 0, sizeof(uint32_t) * (size_t)n * c->ld, c->st));
            k_hist_full<<<grid_for(n * c->W), 256, 0, c->st>>>(c->L, c->C, n, c->ld, c->W, bad);
            IMX_CHECK_LAUNCH();
            count_launch(c);
        }
        unsigned hb = 0;
        IMX_CUDA(cudaMemcpyAsync(&hb, bad, sizeof hb, cudaMemcpyDeviceToHost, c->st));
        IMX_CUDA(cudaStreamSynchronize(c->st));
        if (hb) { set_error("label outside 0..n-1"); return IMX_EINVAL; }
    }
    c->labels_ready = true;
    c->memo_ready = false;
    c->celf_ready = false;
    c->full_counts = 1;
    return IMX_OK;
}

extern "C" int imx_copy_labels(imx_ctx *c, int32_t r0, int32_t r1, int32_t *out) {
    CTX_CHECK(c);
    if (r0 < 0 || r1 > c->W || r0 > r1) { set_error("lane window [%d, %d) invalid", r0, r1); return IMX_EINVAL; }
    if (!c->labels_ready) { set_error("labels not computed"); return IMX_EINVAL; }
    const int64_t n = c->g->n;
    if (n == 0 || r1 == r0) return IMX_OK;
    IMX_CUDA(cudaMemcpy2DAsync(out, sizeof(int32_t) * (r1 - r0), c->L + r0, sizeof(uint32_t) * c->ld,
                               sizeof(int32_t) * (r1 - r0), n, cudaMemcpyDeviceToHost, c->st));
    IMX_CUDA(cudaStreamSynchronize(c->st));
    return IMX_OK;
}

extern "C" int imx_copy_sizes(imx_ctx *c, int32_t r0, int32_t r1, int32_t *out) {
    CTX_CHECK(c);
    if (r0 < 0 || r1 > c->W || r0 > r1) { set_error("lane window [%d, %d) invalid", r0, r1); return IMX_EINVAL; }
    if (!c->labels_ready) { set_error("labels not computed"); return IMX_EINVAL; }
    const int64_t n = c->g->n;
    if (n == 0 || r1 == r0) return IMX_OK;
    const int w = r1 - r0;
    int64_t rows = std::max<int64_t>(1, (int64_t(256) << 20) / (4 * (int64_t)w));
    rows = std::min(rows, n);
    int32_t *tmp;
    IMX_CUDA(cudaMalloc((void **)&tmp, sizeof(int32_t) * rows * w));
    int rc = IMX_OK;
    for (int64_t v0 = 0; v0 < n && rc == IMX_OK; v0 += rows) {
        int64_t cnt = std::min(rows, n - v0);
        k_sizes_window<<<grid_for(cnt * w), 256, 0, c->st>>>(c->L, c->C, v0, cnt, c->ld, r0, r1,
                                                              c->full_counts, tmp);
        cudaError_t e = cudaGetLastError();
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(out + v0 * w, tmp, sizeof(int32_t) * cnt * w, cudaMemcpyDeviceToHost, c->st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(c->st);
        if (e != cudaSuccess) rc = cuda_fail(e, "copy sizes", __FILE__, __LINE__);
        count_launch(c);
    }
    cudaFree(tmp);
    return rc;
}

// ---------------------------------------------------------------------------
// CELF (selection.py:115-149) -- round-based exact formulation
// ---------------------------------------------------------------------------
extern "C" int imx_celf_reset(imx_ctx *c, const int64_t *prio) {
    CTX_CHECK(c);
    if (!c->labels_ready) { set_error("labels not computed"); return IMX_EINVAL; }
    IMX_TRY(ensure_celf_buffers(c));
    const int64_t n = c->g->n;
    if (n) {
        if (prio) {
            IMX_CUDA(cudaMemcpyAsync(c->prio, prio, sizeof(int64_t) * n, cudaMemcpyHostToDevice, c->st));
        } else {
            if (!c->memo_ready) { set_error("gains not computed (call imx_memoize first)"); return IMX_EINVAL; }
            IMX_CUDA(cudaMemcpyAsync(c->prio, c->gains, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, c->st));
        }
        IMX_CUDA(cudaMemsetAsync(c->inS, 0, n, c->st));
        IMX_CUDA(cudaMemsetAsync(c->cov, 0, sizeof(uint32_t) * (size_t)n * c->cw, c->st));
    }
    IMX_CUDA(cudaMemsetAsync(c->per_sim, 0, sizeof(int64_t) * (c->W + 1), c->st));
    IMX_CUDA(cudaStreamSynchronize(c->st));
    c->celf_ready = true;
    c->ncand = 0;
    c->trace.clear();
    return IMX_OK;
}

#define CELF_CHECK(c)                                                             \
    do {                                                                          \
        CTX_CHECK(c);                                                             \
        if (!(c)->celf_ready) { set_error("CELF state not initialised (imx_celf_reset)"); return IMX_EINVAL; } \
    } while (0)

static int celf_top(imx_ctx *c, int64_t *prio_out, int32_t *v_out) {
    const int64_t n = c->g->n;
    unsigned long long *sc = c->scratch + 5;
    IMX_CUDA(cudaMemsetAsync(sc, 0, sizeof(unsigned long long), c->st));
    if (n) {
        k_top<<<grid_for(n, 256), 256, 0, c->st>>>(c->prio, c->inS, n, c->vb, sc);
        IMX_CHECK_LAUNCH();
        count_launch(c);
    }
    unsigned long long key = 0;
    IMX_CUDA(cudaMemcpyAsync(&key, sc, sizeof key, cudaMemcpyDeviceToHost, c->st));
    IMX_CUDA(cudaStreamSynchronize(c->st));
    if (!key) { *v_out = -1; *prio_out = 0; return IMX_OK; }
    key -= 1;
    const uint64_t vmask = (c->vb >= 32) ? 0xffffffffull : ((1ull << c->vb) - 1);
    *v_out = (int32_t)(vmask - (key & vmask));
    *prio_out = (int64_t)(key >> c->vb);
    return IMX_OK;
}

extern "C" int imx_celf_top(imx_ctx *c, int64_t *prio_out, int32_t *v_out) {
    CELF_CHECK(c);
    if (!prio_out || !v_out) { set_error("NULL argument"); return IMX_EINVAL; }
    return celf_top(c, prio_out, v_out);
}

// Collect the non-seeds whose stale key (-prio, id) is <= (-g, u), sorted by
// that key on the device (descending packed key == ascending (-prio, id)).
// The sorted ids stay in c->cand for batch evaluation; ids/prio come back.
static int celf_collect(imx_ctx *c, int64_t g, int32_t u, int32_t exclude, std::vector<int32_t> *ids,
                        std::vector<int64_t> *pr) {
    const int64_t n = c->g->n;
    unsigned long long *sc = c->scratch + 6;
    IMX_CUDA(cudaMemsetAsync(sc, 0, sizeof(unsigned long long), c->st));
    const uint32_t vmask = (c->vb >= 32) ? 0xffffffffu : ((1u << c->vb) - 1u);
    const unsigned long long thr = ((unsigned long long)g << c->vb) | (unsigned long long)(vmask - (uint32_t)u);
    if (n) {
        k_collect<<<grid_for(n, 256), 256, 0, c->st>>>(c->prio, c->inS, n, c->vb, thr, exclude, c->cand, sc);
        IMX_CHECK_LAUNCH();
        count_launch(c);
    }
    unsigned long long cnt = 0;
    IMX_CUDA(cudaMemcpyAsync(&cnt, sc, sizeof cnt, cudaMemcpyDeviceToHost, c->st));
    IMX_CUDA(cudaStreamSynchronize(c->st));
    c->ncand = (int64_t)cnt;
    ids->resize(cnt);
    pr->resize(cnt);
    if (!cnt) return IMX_OK;
    // keys of the collected ids, then a device radix sort by key
    unsigned long long *keys = reinterpret_cast<unsigned long long *>(c->fresh);
    k_keys_of<<<grid_for((int64_t)cnt), 256, 0, c->st>>>(c->cand, (int64_t)cnt, c->prio, c->vb, keys);
    IMX_CHECK_LAUNCH();
    count_launch(c);
    const int end_bit = 64;
    size_t tmp_bytes = 0;
    IMX_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp_bytes, keys, c->keys2, c->cand,
                                                       c->cand2, (int64_t)cnt, 0, end_bit, c->st));
    if (tmp_bytes > c->sort_tmp_bytes) {
        if (c->sort_tmp) cudaFree(c->sort_tmp);
        c->sort_tmp = nullptr;
        c->sort_tmp_bytes = 0;
        IMX_CUDA(cudaMalloc(&c->sort_tmp, tmp_bytes));
        c->sort_tmp_bytes = tmp_bytes;
    }
    IMX_CUDA(cub::DeviceRadixSort::SortPairsDescending(c->sort_tmp, tmp_bytes, keys, c->keys2, c->cand,
                                                       c->cand2, (int64_t)cnt, 0, end_bit, c->st));
    std::swap(c->cand, c->cand2);
    std::vector<unsigned long long> hk(cnt);
    IMX_CUDA(cudaMemcpyAsync(ids->data(), c->cand, sizeof(int32_t) * cnt, cudaMemcpyDeviceToHost, c->st));
    IMX_CUDA(cudaMemcpyAsync(hk.data(), c->keys2, sizeof(unsigned long long) * cnt, cudaMemcpyDeviceToHost, c->st));
    IMX_CUDA(cudaStreamSynchronize(c->st));
    for (size_t i = 0; i < cnt; ++i) (*pr)[i] = (int64_t)(hk[i] >> c->vb);
    return IMX_OK;
}

extern "C" int imx_celf_collect(imx_ctx *c, int64_t g, int32_t u, int32_t exclude, int32_t *ids_out,
                                int64_t *prio_out, int64_t cap, int64_t *count) {
    CELF_CHECK(c);
    if (!count) { set_error("count is NULL"); return IMX_EINVAL; }
    if (g < 0) { set_error("gain bound must be non-negative"); return IMX_EINVAL; }
    std::vector<int32_t> ids;
    std::vector<int64_t> pr;
    IMX_TRY(celf_collect(c, g, u, exclude, &ids, &pr));
    *count = (int64_t)ids.size();
    const int64_t k = std::min<int64_t>(cap, *count);
    if (k > 0 && ids_out) std::copy(ids.begin(), ids.begin() + k, ids_out);
    if (k > 0 && prio_out) std::copy(pr.begin(), pr.begin() + k, prio_out);
    return IMX_OK;
}

static int celf_eval_dev(imx_ctx *c, const int32_t *dcand, int64_t cnt, int64_t *dout) {
    if (cnt <= 0) return IMX_OK;
    const int blocks = (int)std::min<int64_t>(cnt, 148 * 16);
    k_eval<<<blocks, kEvalThreads, 0, c->st>>>(dcand, cnt, c->L, c->C, c->cov, c->ld, c->ns, c->cw,
                                               c->full_counts, dout);
    IMX_CHECK_LAUNCH();
    count_launch(c);
    return IMX_OK;
}

// evaluate collected[lo, hi) -> fresh_out[hi - lo]
extern "C" int imx_celf_eval_collected(imx_ctx *c, int64_t lo, int64_t hi, int64_t *fresh_out) {
    CELF_CHECK(c);
    if (lo < 0 || hi > c->ncand || lo > hi) {
        set_error("collected range [%lld, %lld) outside [0, %lld)", (long long)lo, (long long)hi,
                  (long long)c->ncand);
        return IMX_EINVAL;
    }
    if (hi == lo) return IMX_OK;
    IMX_TRY(celf_eval_dev(c, c->cand + lo, hi - lo, c->eval_out));
    if (fresh_out)
        IMX_CUDA(cudaMemcpyAsync(fresh_out, c->eval_out, sizeof(int64_t) * (hi - lo), cudaMemcpyDeviceToHost, c->st));
    IMX_CUDA(cudaStreamSynchronize(c->st));
    return IMX_OK;
}

extern "C" int imx_eval_gains(imx_ctx *c, const int32_t *cand, int64_t cnt, int64_t *out) {
    CELF_CHECK(c);
    if (cnt < 0 || (cnt && (!cand || !out))) { set_error("bad arguments"); return IMX_EINVAL; }
    if (!cnt) return IMX_OK;
    for (int64_t i = 0; i < cnt; ++i)
        if (cand[i] < 0 || cand[i] >= c->g->n) { set_error("vertex %d outside vertex range", cand[i]); return IMX_EINVAL; }
    int32_t *dc;
    int64_t *dout;
    IMX_CUDA(cudaMallocAsync((void **)&dc, sizeof(int32_t) * cnt, c->st));
    IMX_CUDA(cudaMallocAsync((void **)&dout, sizeof(int64_t) * cnt, c->st));
    IMX_CUDA(cudaMemcpyAsync(dc, cand, sizeof(int32_t) * cnt, cudaMemcpyHostToDevice, c->st));
    int rc = celf_eval_dev(c, dc, cnt, dout);
    if (rc == IMX_OK)
        IMX_CUDA(cudaMemcpyAsync(out, dout, sizeof(int64_t) * cnt, cudaMemcpyDeviceToHost, c->st));
    cudaFreeAsync(dc, c->st);
    cudaFreeAsync(dout, c->st);
    IMX_CUDA(cudaStreamSynchronize(c->st));
    return rc;
}

static int celf_set_prio_async(imx_ctx *c, const int32_t *ids, const int64_t *vals, int64_t cnt) {
    if (cnt <= 0) return IMX_OK;
    // staged through the pinned host buffer
    IMX_TRY(ensure_pinned(c, cnt));
    std::copy(ids, ids + cnt, c->h_ids);
    std::copy(vals, vals + cnt, c->h_vals);
    IMX_CUDA(cudaMemcpyAsync(c->d_ids, c->h_ids, sizeof(int32_t) * cnt, cudaMemcpyHostToDevice, c->st));
    IMX_CUDA(cudaMemcpyAsync(c->d_vals, c->h_vals, sizeof(int64_t) * cnt, cudaMemcpyHostToDevice, c->st));
    k_set_prio<<<grid_for(cnt), 256, 0, c->st>>>(c->d_ids, c->d_vals, cnt, c->prio);
    IMX_CHECK_LAUNCH();
    count_launch(c);
    return IMX_OK;
}

extern "C" int imx_celf_set_prio(imx_ctx *c, const int32_t *ids, const int64_t *vals, int64_t cnt) {
    CELF_CHECK(c);
    IMX_TRY(celf_set_prio_async(c, ids, vals, cnt));
    IMX_CUDA(cudaStreamSynchronize(c->st));
    return IMX_OK;
}

static int celf_commit(imx_ctx *c, int32_t u, int64_t *gain_out) {
    unsigned long long *sc = c->scratch + 7;
    IMX_CUDA(cudaMemsetAsync(sc, 0, sizeof(unsigned long long), c->st));
    k_commit<<<grid_for(std::max(c->ns, 1)), 256, 0, c->st>>>(u, c->L, c->C, c->cov, c->ld, c->ns, c->cw,
                                                             c->full_counts, c->per_sim, c->inS, sc);
    IMX_CHECK_LAUNCH();
    count_launch(c);
    unsigned long long gsum = 0;
    IMX_CUDA(cudaMemcpyAsync(&gsum, sc, sizeof gsum, cudaMemcpyDeviceToHost, c->st));
    IMX_CUDA(cudaStreamSynchronize(c->st));
    if (gain_out) *gain_out = (int64_t)gsum;
    return IMX_OK;
}

extern "C" int imx_commit(imx_ctx *c, int32_t u, int64_t *gain_out) {
    CELF_CHECK(c);
    if (u < 0 || u >= c->g->n) { set_error("vertex %d outside vertex range", u); return IMX_EINVAL; }
    uint8_t in = 0;
    IMX_CUDA(cudaMemcpyAsync(&in, c->inS + u, 1, cudaMemcpyDeviceToHost, c->st));
    IMX_CUDA(cudaStreamSynchronize(c->st));
    if (in) { set_error("vertex %d committed twice", u); return IMX_EINTERNAL; }
    return celf_commit(c, u, gain_out);
}

static inline bool key_le(int64_t pa, int32_t va, int64_t pb, int32_t vb) {
    // (-pa, va) <= (-pb, vb)
    return pa > pb || (pa == pb && va <= vb);
}

// Whole CELF loop on one context.  Exactness argument: on a
// fixed sample set marginal gains are submodular, so the reference's lazy
// heap commits, at every round t, u* = argmin over V\S of (-fresh, id), after
// refreshing exactly R_t = {v : (-stale_v, v) <= (-fresh_u*, u*)} in
// (-stale, id) order.  Round t evaluates the top-priority vertex, collects
// the vertices whose stale key is at most that vertex's fresh key (nothing
// else can win), sorts them by stale key and evaluates them in doubling
// batches until the best fresh key found is below the next stale key -- so
// the evaluated set is R_t plus at most one batch.
//
// Launch pattern per round: top -> decode -> eval(top) -> threshold ->
// collect run back to back on the stream and end in ONE host sync that reads
// the round header (top key, its fresh gain, collected count, last commit's
// gain); the sort and the first batch end in a second sync; the priority
// update and the commit are left in flight for the next round.
extern "C" int imx_celf_select(imx_ctx *c, int32_t k, int32_t *seeds_out, int64_t *gains_out,
                               int64_t *trace_len) {
    CELF_CHECK(c);
    const int64_t n = c->g->n;
    if (k < 1 || k > n) { set_error("k=%d invalid for n=%lld", k, (long long)n); return IMX_ECONSTRAINT; }
    cudaEventRecord(c->ev[6], c->st);
    c->trace.clear();
    c->evaluated = 0;
    auto rec = [&](int64_t v, int64_t s, int64_t f, int64_t com, int64_t t) {
        c->trace.push_back(v); c->trace.push_back(s); c->trace.push_back(f);
        c->trace.push_back(com); c->trace.push_back(t);
    };
    unsigned long long *hdr = c->scratch + 8;
    const uint64_t vmask = (c->vb >= 32) ? 0xffffffffull : ((1ull << c->vb) - 1);
    IMX_TRY(ensure_pinned(c, 4096));
    unsigned long long *hh = reinterpret_cast<unsigned long long *>(c->h_vals);  // pinned header copy
    std::vector<int32_t> eids, ids;
    std::vector<int64_t> epr, efr, pr, fr;
    std::vector<unsigned long long> keys;
    int64_t batch0 = 64;
    int64_t pending_gain = -1;   // expected gain of the commit still in flight
    int32_t pending_v = -1;
    auto check_gain = [&](int64_t got) -> int {
        if (pending_gain >= 0 && got != pending_gain) {
            set_error("CELF self-check: committed gain %lld != evaluated %lld for vertex %d",
                      (long long)got, (long long)pending_gain, pending_v);
            return IMX_EINTERNAL;
        }
        return IMX_OK;
    };
    for (int32_t t = 0; t < k; ++t) {
        // ---- phase 1: top, its fresh gain, the collected candidates ----
        IMX_CUDA(cudaMemsetAsync(hdr + H_TOP, 0, sizeof(unsigned long long), c->st));
        IMX_CUDA(cudaMemsetAsync(hdr + H_COUNT, 0, sizeof(unsigned long long), c->st));
        k_top<<<grid_for(n, 256), 256, 0, c->st>>>(c->prio, c->inS, n, c->vb, hdr + H_TOP);
        k_round_decode<<<1, 1, 0, c->st>>>(hdr, c->vb, c->d_one);
        count_launch(c, 2);
        if (t > 0) {
            IMX_TRY(celf_eval_dev(c, c->d_one, 1, c->eval_out));
            k_make_thr<<<1, 1, 0, c->st>>>(hdr, c->eval_out, c->d_one, c->vb);
            k_collect_dev<<<grid_for(n, 256), 256, 0, c->st>>>(c->prio, c->inS, n, c->vb, hdr, c->d_one,
                                                               c->cand, hdr + H_COUNT);
            count_launch(c, 2);
        }
        IMX_CHECK_LAUNCH();
        IMX_CUDA(cudaMemcpyAsync(hh, hdr, sizeof(unsigned long long) * 4, cudaMemcpyDeviceToHost, c->st));
        IMX_CUDA(cudaStreamSynchronize(c->st));
        IMX_TRY(check_gain((int64_t)hh[H_GAIN]));
        if (!hh[H_TOP]) { set_error("no candidate left at round %d", t); return IMX_EINTERNAL; }
        const unsigned long long tk = hh[H_TOP] - 1;
        const int32_t vt = (int32_t)(vmask - (tk & vmask));
        const int64_t gt = (int64_t)(tk >> c->vb);
        int64_t best_f = gt;
        int32_t best_v = vt;
        if (t > 0) {
            const int64_t f1 = (int64_t)hh[H_F1];
            const int64_t cnt = (int64_t)hh[H_COUNT];
            c->evaluated += 1;
            best_f = f1;
            eids.assign(1, vt); epr.assign(1, gt); efr.assign(1, f1);
            c->ncand = cnt;
            if (cnt > 0) {
                // ---- phase 2: sort by stale key, first batch ----
                unsigned long long *dkeys = reinterpret_cast<unsigned long long *>(c->fresh);
                k_keys_of<<<grid_for(cnt), 256, 0, c->st>>>(c->cand, cnt, c->prio, c->vb, dkeys);
                IMX_CHECK_LAUNCH();
                count_launch(c);
                size_t tmp_bytes = 0;
                IMX_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp_bytes, dkeys, c->keys2, c->cand,
                                                                   c->cand2, cnt, 0, 64, c->st));
                if (tmp_bytes > c->sort_tmp_bytes) {
                    IMX_CUDA(cudaStreamSynchronize(c->st));
                    if (c->sort_tmp) cudaFree(c->sort_tmp);
                    c->sort_tmp = nullptr;
                    c->sort_tmp_bytes = 0;
                    IMX_CUDA(cudaMalloc(&c->sort_tmp, tmp_bytes * 2));
                    c->sort_tmp_bytes = tmp_bytes * 2;
                }
                IMX_CUDA(cub::DeviceRadixSort::SortPairsDescending(c->sort_tmp, tmp_bytes, dkeys, c->keys2, c->cand,
                                                                   c->cand2, cnt, 0, 64, c->st));
                std::swap(c->cand, c->cand2);
                ids.resize(cnt); pr.resize(cnt); fr.resize(cnt); keys.resize(cnt);
                int64_t lo = 0, b = batch0, fetched = 0;
                for (;;) {
                    const int64_t hi = std::min(cnt, lo + b);
                    const int64_t fetch_to = std::min(cnt, hi + 1);   // +1: next stale key
                    IMX_TRY(celf_eval_dev(c, c->cand + lo, hi - lo, c->eval_out));
                    if (fetch_to > fetched) {
                        IMX_CUDA(cudaMemcpyAsync(ids.data() + fetched, c->cand + fetched,
                                                 sizeof(int32_t) * (fetch_to - fetched), cudaMemcpyDeviceToHost, c->st));
                        IMX_CUDA(cudaMemcpyAsync(keys.data() + fetched, c->keys2 + fetched,
                                                 sizeof(unsigned long long) * (fetch_to - fetched),
                                                 cudaMemcpyDeviceToHost, c->st));
                    }
                    IMX_CUDA(cudaMemcpyAsync(fr.data() + lo, c->eval_out, sizeof(int64_t) * (hi - lo),
                                             cudaMemcpyDeviceToHost, c->st));
                    IMX_CUDA(cudaStreamSynchronize(c->st));
                    for (int64_t i = fetched; i < fetch_to; ++i) pr[i] = (int64_t)(keys[i] >> c->vb);
                    fetched = std::max(fetched, fetch_to);
                    for (int64_t i = lo; i < hi; ++i) {
                        if (key_le(fr[i], ids[i], best_f, best_v)) { best_f = fr[i]; best_v = ids[i]; }
                        eids.push_back(ids[i]); epr.push_back(pr[i]); efr.push_back(fr[i]);
                    }
                    c->evaluated += hi - lo;
                    lo = hi;
                    b *= 2;
                    if (lo >= cnt || key_le(best_f, best_v, pr[lo], ids[lo])) break;
                }
            }
            // ---- R_t in (-stale, id) order: refresh records, prio <- fresh ----
            std::vector<size_t> rt;
            for (size_t i = 0; i < eids.size(); ++i)
                if (key_le(epr[i], eids[i], best_f, best_v)) rt.push_back(i);
            std::sort(rt.begin(), rt.end(), [&](size_t a, size_t b2) {
                return epr[a] != epr[b2] ? epr[a] > epr[b2] : eids[a] < eids[b2];
            });
            IMX_TRY(ensure_pinned(c, (int64_t)rt.size() + 8));
            hh = reinterpret_cast<unsigned long long *>(c->h_vals);
            int64_t m = 0;
            for (size_t i : rt) {
                rec(eids[i], epr[i], efr[i], 0, t);
                c->h_ids[m] = eids[i];
                c->h_vals[8 + m] = efr[i];   // h_vals[0..7] hold the header copy
                ++m;
            }
            batch0 = std::max<int64_t>(64, m);
            if (m) {
                IMX_CUDA(cudaMemcpyAsync(c->d_ids, c->h_ids, sizeof(int32_t) * m, cudaMemcpyHostToDevice, c->st));
                IMX_CUDA(cudaMemcpyAsync(c->d_vals, c->h_vals + 8, sizeof(int64_t) * m, cudaMemcpyHostToDevice, c->st));
                k_set_prio<<<grid_for(m), 256, 0, c->st>>>(c->d_ids, c->d_vals, m, c->prio);
                IMX_CHECK_LAUNCH();
                count_launch(c);
            }
        }
        // ---- commit (in flight; its gain is checked at the next header read) ----
        IMX_CUDA(cudaMemsetAsync(hdr + H_GAIN, 0, sizeof(unsigned long long), c->st));
        k_commit<<<grid_for(std::max(c->ns, 1)), 256, 0, c->st>>>(best_v, c->L, c->C, c->cov, c->ld, c->ns, c->cw,
                                                                 c->full_counts, c->per_sim, c->inS, hdr + H_GAIN);
        IMX_CHECK_LAUNCH();
        count_launch(c);
        pending_gain = best_f;
        pending_v = best_v;
        rec(best_v, best_f, best_f, 1, t);
        if (seeds_out) seeds_out[t] = best_v;
        if (gains_out) gains_out[t] = best_f;
    }
    IMX_CUDA(cudaMemcpyAsync(hh, hdr, sizeof(unsigned long long) * 4, cudaMemcpyDeviceToHost, c->st));
    IMX_CUDA(cudaStreamSynchronize(c->st));
    IMX_TRY(check_gain((int64_t)hh[H_GAIN]));
    cudaEventRecord(c->ev[7], c->st);
    cudaEventSynchronize(c->ev[7]);
    cudaEventElapsedTime(&c->tm.select_ms, c->ev[6], c->ev[7]);
    c->tm.celf_evaluations = c->evaluated;
    c->ncand = 0;
    if (trace_len) *trace_len = (int64_t)(c->trace.size() / 5);
    return IMX_OK;
}

extern "C" int imx_celf_trace(imx_ctx *c, int64_t *out, int64_t cap) {
    CTX_CHECK(c);
    const int64_t len = (int64_t)(c->trace.size() / 5);
    const int64_t k = std::min(cap, len);
    if (k > 0 && out) std::copy(c->trace.begin(), c->trace.begin() + 5 * k, out);
    return IMX_OK;
}

extern "C" int imx_per_sim(imx_ctx *c, int64_t *out) {
    CELF_CHECK(c);
    if (!out) { set_error("out is NULL"); return IMX_EINVAL; }
    if (c->ns) {
        IMX_CUDA(cudaMemcpyAsync(out, c->per_sim, sizeof(int64_t) * c->ns, cudaMemcpyDeviceToHost, c->st));
        IMX_CUDA(cudaStreamSynchronize(c->st));
    }
    return IMX_OK;
}

extern "C" int imx_copy_owned(imx_ctx *c, uint32_t *bits_out) {
    CELF_CHECK(c);
    if (!bits_out) { set_error("out is NULL"); return IMX_EINVAL; }
    const int64_t n = c->g->n;
    if (n) {
        IMX_CUDA(cudaMemcpyAsync(bits_out, c->cov, sizeof(uint32_t) * (size_t)n * c->cw, cudaMemcpyDeviceToHost, c->st));
        IMX_CUDA(cudaStreamSynchronize(c->st));
    }
    return IMX_OK;
}

// ---------------------------------------------------------------------------
// measurement
// ---------------------------------------------------------------------------
extern "C" int imx_get_timings(imx_ctx *c, imx_timings *out) {
    CTX_CHECK(c);
    if (!out) { set_error("out is NULL"); return IMX_EINVAL; }
    *out = c->tm;
    return IMX_OK;
}

__global__ void k_flush(uint4 *buf, int64_t cnt, uint32_t salt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
         i += (int64_t)gridDim.x * blockDim.x)
        buf[i] = make_uint4(salt, (uint32_t)i, salt, (uint32_t)i);
}

extern "C" int imx_bench_propagate(imx_ctx *c, int32_t reps, int32_t flush_l2, float *avg_total_ms,
                                   float *avg_hook_ms, float *avg_compress_ms, float *avg_init_ms) {
    CTX_CHECK(c);
    if (reps < 1) { set_error("reps must be >= 1"); return IMX_EINVAL; }
    uint4 *fb = nullptr;
    const int64_t fcnt = (int64_t(256) << 20) / 16;  // 256 MB > 126 MB L2
    if (flush_l2) IMX_CUDA(cudaMalloc((void **)&fb, fcnt * 16));
    std::vector<cudaEvent_t> ev(4 * reps);
    for (auto &e : ev) IMX_CUDA(cudaEventCreate(&e));
    for (int i = 0; i < reps; ++i) {
        if (fb) k_flush<<<148 * 8, 256, 0, c->st>>>(fb, fcnt, (uint32_t)i);
        IMX_CUDA(cudaEventRecord(ev[4 * i], c->st));
        if (c->g->m2) {
            IMX_TRY(run_sample_cc(c, nullptr, ev[4 * i + 1], ev[4 * i + 2]));
            IMX_TRY(run_compress(c, nullptr));
        } else {
            IMX_TRY(run_init(c));
            IMX_CUDA(cudaEventRecord(ev[4 * i + 1], c->st));
            IMX_CUDA(cudaEventRecord(ev[4 * i + 2], c->st));
        }
        IMX_CUDA(cudaEventRecord(ev[4 * i + 3], c->st));
    }
    IMX_CUDA(cudaStreamSynchronize(c->st));
    double tot = 0, hk = 0, cp = 0, in = 0;
    for (int i = 0; i < reps; ++i) {
        float a, b, d, e;
        cudaEventElapsedTime(&a, ev[4 * i], ev[4 * i + 3]);
        cudaEventElapsedTime(&b, ev[4 * i + 1], ev[4 * i + 2]);
        cudaEventElapsedTime(&d, ev[4 * i + 2], ev[4 * i + 3]);
        cudaEventElapsedTime(&e, ev[4 * i], ev[4 * i + 1]);
        tot += a; hk += b; cp += d; in += e;
    }
    for (auto &e : ev) cudaEventDestroy(e);
    if (fb) cudaFree(fb);
    if (avg_total_ms) *avg_total_ms = (float)(tot / reps);
    if (avg_hook_ms) *avg_hook_ms = (float)(hk / reps);
    if (avg_compress_ms) *avg_compress_ms = (float)(cp / reps);
    if (avg_init_ms) *avg_init_ms = (float)(in / reps);
    c->labels_ready = true;
    c->memo_ready = false;
    c->celf_ready = false;
    c->full_counts = 0;
    return IMX_OK;
}
