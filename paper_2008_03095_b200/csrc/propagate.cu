// propagate.cu -- K2+K3: fused sample + connected components over all lanes
// of a context (reference propagate, propagation.py:260-321).
//
// The reference drives min-label sweeps to their unique fixpoint (min vertex
// id of every vertex's component in every sampled graph).  Any exact CC
// algorithm reaches the same fixpoint, so the device runs ONE
// concurrent union-find pass (uf.cuh) whose sampler is fused into it -- edge
// membership (X[r] ^ hash) < thr is decided where the edge is visited and
// never materialised -- followed by one compression pass:
//
//   sampler/hook  one of three strategies (hook_mode):
//     enum   sorted-hash interval enumeration: only live (edge, lane) pairs
//     pull   first-hop forest (every vertex points at its smallest live
//            smaller neighbour, written row by row) + unions of the rest
//     dense  edge-major scan of all lanes with a per-warp union queue
//   compress L[v][r] <- root; root cell counts its other members
//   verify   (optional) every live edge joins equal labels, labels are roots
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cub/cub.cuh>

#include "ctx.cuh"
#include "uf.cuh"

namespace imx {

// every cell starts as a root with no other members
__global__ void k_init(uint32_t *__restrict__ L, int64_t cells4) {
    uint4 *L4 = reinterpret_cast<uint4 *>(L);
    const uint4 r4 = make_uint4(ROOT, ROOT, ROOT, ROOT);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cells4;
         i += (int64_t)gridDim.x * blockDim.x)
        L4[i] = r4;
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
                                                          Lay y, uint32_t *__restrict__ L,
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
                    nh += unite(L, y, a, bb, r);
                }
            }
        }
    }
    __syncwarp();
    if (lane < qn) nh += unite(L, y, qlo[lane], qhi[lane], (int)qr[lane]);
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
// lower_bound of key (< 2^32) among bucket b's sorted hashes via the prefix LUT
__device__ __forceinline__ int64_t hash_lower_bound(const int32_t *__restrict__ EH, const int32_t *__restrict__ lut,
                                                    int bits, const int64_t *__restrict__ boff, int b,
                                                    uint64_t key) {
    if (key >= (1ull << 31)) return boff[b + 1];
    const int64_t per = ((int64_t)1 << bits) + 1;
    const int64_t k = (int64_t)(key >> (31 - bits));
    int64_t lo = lut[b * per + k], hi = lut[b * per + k + 1];
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((uint64_t)(uint32_t)EH[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// both bounds of a segment, the two searches advanced in lock step so their
// dependent loads overlap (the same result as two hash_lower_bound calls)
__device__ __forceinline__ void hash_lower_bound2(const int32_t *__restrict__ EH, const int32_t *__restrict__ lut,
                                                  int bits, const int64_t *__restrict__ boff, int b, uint64_t k1,
                                                  uint64_t k2, int64_t &r1, int64_t &r2) {
    const int64_t per = ((int64_t)1 << bits) + 1;
    const int64_t end = boff[b + 1];
    int64_t lo1 = end, hi1 = end, lo2 = end, hi2 = end;
    if (k1 < (1ull << 31)) {
        const int64_t q = (int64_t)(k1 >> (31 - bits));
        lo1 = lut[b * per + q]; hi1 = lut[b * per + q + 1];
    }
    if (k2 < (1ull << 31)) {
        const int64_t q = (int64_t)(k2 >> (31 - bits));
        lo2 = lut[b * per + q]; hi2 = lut[b * per + q + 1];
    }
    while (lo1 < hi1 || lo2 < hi2) {
        const int64_t m1 = (lo1 + hi1) >> 1, m2 = (lo2 + hi2) >> 1;
        const bool a1 = lo1 < hi1, a2 = lo2 < hi2;
        const uint32_t h1 = a1 ? (uint32_t)EH[m1] : 0u, h2 = a2 ? (uint32_t)EH[m2] : 0u;
        if (a1) { if ((uint64_t)h1 < k1) lo1 = m1 + 1; else hi1 = m1; }
        if (a2) { if ((uint64_t)h2 < k2) lo2 = m2 + 1; else hi2 = m2; }
    }
    r1 = lo1;
    r2 = lo2;
}

__global__ void k_seg_count(const int32_t *__restrict__ X, int32_t W, int nb,
                            const int32_t *__restrict__ btmax, const int64_t *__restrict__ boff,
                            const int32_t *__restrict__ EH, const int32_t *__restrict__ lut, int bits,
                            int64_t *__restrict__ seg_a, int64_t *__restrict__ seg_n) {
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
            int64_t e;
            hash_lower_bound2(EH, lut, bits, boff, b, start, end, a, e);
            cnt = e - a;
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
#ifndef IMX_ENUM_CHUNK
#define IMX_ENUM_CHUNK 128
#endif
constexpr int kEnumChunk = IMX_ENUM_CHUNK;

// largest s in [0, nseg) with off[s] <= j (off nondecreasing, off[0] = 0),
// by the whole warp: a 33-ary search -- 32 pivots per step, one load each,
// so ~log33(nseg) dependent loads instead of log2(nseg) on one lane
__device__ __forceinline__ int64_t seg_search(const int64_t *__restrict__ off, int64_t nseg, int64_t j, int lane) {
    int64_t lo = 0, hi = nseg;      // off[lo] <= j; hi == nseg or off[hi] > j
    while (hi - lo > 1) {
        const int64_t span = hi - lo;
        const int64_t piv = lo + span * (lane + 1) / 33;
        const unsigned b = __ballot_sync(0xffffffffu, __ldg(off + piv) <= j);
        const int c = __popc(b);    // pivots are nondecreasing: b is a prefix of ones
        const int64_t plo = __shfl_sync(0xffffffffu, piv, c > 0 ? c - 1 : 0);
        const int64_t phi = __shfl_sync(0xffffffffu, piv, c < 32 ? c : 31);
        if (c > 0) lo = plo;
        if (c < 32) hi = phi;
    }
    return lo;
}
// Segments [s_lo, s_hi) (whole lanes) only.
template <bool UNI, bool SKIP>
__global__ void __launch_bounds__(256) k_hook_enum(const int64_t *__restrict__ off, const int64_t *__restrict__ seg_a,
                                                   int64_t s_lo, int64_t s_hi, int segs_per_lane,
                                                   const int2 *__restrict__ E, const int32_t *__restrict__ EH,
                                                   const int32_t *__restrict__ ET, const int32_t *__restrict__ X,
                                                   Lay ld, uint32_t *__restrict__ L,
                                                   unsigned long long *__restrict__ hooks) {
    const int64_t jlo = off[s_lo], total = off[s_hi];
    const int lane = threadIdx.x & 31;
    const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long nh = 0;
    for (int64_t j0 = jlo + wg * kEnumChunk; j0 < total; j0 += nw * kEnumChunk) {
        int64_t s = s_lo + seg_search(off + s_lo, s_hi - s_lo, j0, lane);
        const int64_t jend = (total - j0 < kEnumChunk) ? total : j0 + kEnumChunk;
        if (!UNI) {
            // per-edge thresholds: the membership re-test gates the union
            for (int64_t j = j0 + lane; j < jend; j += 32) {
                while (off[s + 1] <= j) ++s;
                const int64_t e = seg_a[s] + (j - off[s]);
                const int r = (int)(s / segs_per_lane);
                if (!((X[r] ^ EH[e]) < ET[e])) continue;
                const int2 uv = E[e];
                if (SKIP && ld_relaxed(cell(L, ld, (uint32_t)uv.y, r)) == (uint32_t)uv.x) continue;
                nh += unite(L, ld, (uint32_t)uv.x, (uint32_t)uv.y, r);
            }
            continue;
        }
        // uniform threshold, two-stage pipeline: the next pair's segment
        // walk and edge load are issued before this pair's union, so the
        // edge fetch overlaps the root searches (C4 hook 23.5 -> 22.7 ms;
        // with per-edge thresholds the extra live state costs more than
        // it hides, C3 7.1 -> 8.0 ms)
        int64_t j = j0 + lane;
        int2 nuv = make_int2(0, 0);
        int32_t nhh = 0, ntt = 1, nxx = 0;
        int nr = 0;
        if (j < jend) {
            while (off[s + 1] <= j) ++s;
            const int64_t e = seg_a[s] + (j - off[s]);
            nr = (int)(s / segs_per_lane);
            nuv = E[e];
            if (!UNI) { nhh = EH[e]; ntt = ET[e]; nxx = X[nr]; }
        }
        for (; j < jend; j += 32) {
            const int2 uv = nuv;
            const int r = nr;
            const bool live = UNI || (nxx ^ nhh) < ntt;
            const int64_t jn = j + 32;
            if (jn < jend) {
                while (off[s + 1] <= jn) ++s;
                const int64_t e = seg_a[s] + (jn - off[s]);
                nr = (int)(s / segs_per_lane);
                nuv = E[e];
                if (!UNI) { nhh = EH[e]; ntt = ET[e]; nxx = X[nr]; }
            }
            if (!live) continue;
            // after the pull forest pass, a live edge that is its upper
            // endpoint's first live smaller neighbour is already a tree edge
            if (SKIP && ld_relaxed(cell(L, ld, (uint32_t)uv.y, r)) == (uint32_t)uv.x) continue;
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
//
// Heavy rows (HEAVY = true): a vertex whose smaller-neighbour prefix exceeds
// T slots would serialise one warp (C3: prefixes up to 3358 slots, 2048
// lanes, ~170 live smaller neighbours per lane to unite).  Its prefix is cut
// into slices of T slots, one warp per slice: pass 1 folds the slice's first
// live neighbour into the row with atomicMin (the light pass wrote the row
// as roots), pass 2 unites every live neighbour except the one the row
// points at (the forest edge; a pointer moved up by path splitting only
// makes the skipped or the extra union one between already-joined trees).
// The light passes skip heavy rows (heavy[v] != 0).
template <int PASS, bool UNI, int LPT, bool HEAVY>
__global__ void __launch_bounds__(256) k_pull(const int64_t *__restrict__ xadj, const int32_t *__restrict__ adj,
                                              const int32_t *__restrict__ hash, const int32_t *__restrict__ thr,
                                              int32_t tu, int64_t n, const int32_t *__restrict__ X, int32_t W,
                                              int64_t ld, Lay y, uint32_t *__restrict__ L,
                                              unsigned long long *__restrict__ hooks,
                                              const uint8_t *__restrict__ heavy, const int32_t *__restrict__ hs_v,
                                              const int64_t *__restrict__ hs_a, const int32_t *__restrict__ hs_len,
                                              int64_t nhs) {
    // LPT lanes per thread (4 or 8): each edge's loads and the loop overhead
    // are shared by LPT membership tests
    constexpr int Q = LPT / 4;                // 16-byte quads per thread
    extern __shared__ int4 smem4[];
    int32_t *sX = reinterpret_cast<int32_t *>(smem4);
    const int64_t ldp = (ld + LPT - 1) / LPT * LPT;   // staged X padded to whole thread groups
    for (int i = threadIdx.x; i < ldp; i += blockDim.x) sX[i] = (i < W) ? X[i] : 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int PQ = 32 + 32 * LPT;         // drain threshold + one edge's appends
    uint32_t *qlo = reinterpret_cast<uint32_t *>(sX + ldp) + warp * 3 * PQ;
    uint32_t *qhi = qlo + PQ;
    uint32_t *qr = qhi + PQ;
    __syncthreads();
    const int ng = (int)(ldp / LPT);          // lane groups per row
    const unsigned FULL = 0xffffffffu;
    int qn = 0;
    unsigned long long nh = 0;
    const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t items = HEAVY ? nhs : n;
    for (int64_t it = wg; it < items; it += nw) {
        int64_t v, s0, s1;
        if (HEAVY) {
            v = hs_v[it];
            s0 = hs_a[it];
            s1 = s0 + hs_len[it];
        } else {
            v = it;
            s0 = xadj[v];
            s1 = xadj[v + 1];
            if (heavy && heavy[v]) s1 = s0;      // heavy row: roots here, slices below
        }
        for (int c0 = 0; c0 < ng; c0 += 32) {
            const int gi = c0 + lane;
            const bool active = gi < ng;
            const int r = gi * LPT;
            int32_t x[LPT];
#pragma unroll
            for (int k = 0; k < Q; ++k) {
                const int4 q4 = active ? smem4[gi * Q + k] : make_int4(0, 0, 0, 0);
                x[4 * k] = q4.x; x[4 * k + 1] = q4.y; x[4 * k + 2] = q4.z; x[4 * k + 3] = q4.w;
            }
            unsigned valid = (1u << LPT) - 1u;
            if (r + LPT > W) valid = (1u << (W > r ? W - r : 0)) - 1u;
            if (!active) valid = 0;
            uint32_t best[LPT];
#pragma unroll
            for (int k = 0; k < LPT; ++k) best[k] = ROOT;
            unsigned seen = 0;
            uint32_t par[HEAVY && PASS == 2 ? LPT : 1];
            if (HEAVY && PASS == 2) {
#pragma unroll
                for (int k = 0; k < Q; ++k) {
                    const uint4 p4 = (active && r + 4 * k < ld)
                        ? *reinterpret_cast<const uint4 *>(L + y.off(v, r + 4 * k)) : make_uint4(ROOT, ROOT, ROOT, ROOT);
                    par[4 * k] = p4.x; par[4 * k + 1] = p4.y; par[4 * k + 2] = p4.z; par[4 * k + 3] = p4.w;
                }
            }
            // the prefix in batches of 32 slots: one coalesced load per
            // batch (lane i holds slot b0 + i), the slots then broadcast by
            // shuffles -- one memory round trip per 32 slots, not per slot
            for (int64_t b0 = s0; b0 < s1; b0 += 32) {
            const int64_t sb = b0 + lane;
            uint32_t bu = (uint32_t)v;
            int32_t bh = 0, bt = tu;
            if (sb < s1) {
                bu = (uint32_t)__ldg(adj + sb);
                bh = __ldg(hash + sb);
                if (!UNI) bt = __ldg(thr + sb);
            }
            // rows ascend, so the smaller neighbours are a prefix of the batch
            const int cnt = __popc(__ballot_sync(FULL, bu < (uint32_t)v));
            for (int j = 0; j < cnt; ++j) {
                const uint32_t u = __shfl_sync(FULL, bu, j);
                const int32_t h = __shfl_sync(FULL, bh, j);
                const int32_t t = UNI ? tu : __shfl_sync(FULL, bt, j);
                if (PASS == 1) {
                    // rows ascend, so the first live neighbour is the
                    // smallest: one predicated min per lane
#pragma unroll
                    for (int k = 0; k < LPT; ++k)
                        if ((x[k] ^ h) < t) best[k] = min(best[k], u);
                } else {
                    unsigned live = 0;
#pragma unroll
                    for (int k = 0; k < LPT; ++k) live |= (unsigned)((x[k] ^ h) < t) << k;
                    live &= valid;
                    unsigned rest;
                    if (HEAVY) {
                        unsigned fe = 0;     // lanes whose row points at u: the forest edge
#pragma unroll
                        for (int k = 0; k < LPT; ++k) fe |= (unsigned)(par[k] == u) << k;
                        rest = live & ~fe;
                    } else {
                        rest = live & seen;
                        seen |= live;
                    }
                    if (!__any_sync(FULL, rest != 0)) continue;
                    const int kk = __popc(rest);
                    int inc = kk;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int y = __shfl_up_sync(FULL, inc, o);
                        if (lane >= o) inc += y;
                    }
                    int pos = qn + inc - kk;
                    while (rest) {
                        const int bb = __ffs(rest) - 1;
                        rest &= rest - 1;
                        qlo[pos] = u;
                        qhi[pos] = (uint32_t)v;
                        qr[pos] = (uint32_t)(r + bb);
                        ++pos;
                    }
                    qn += __shfl_sync(FULL, inc, 31);
                    __syncwarp();
                    while (qn >= 32) {
                        qn -= 32;
                        const uint32_t a2 = qlo[qn + lane], b2 = qhi[qn + lane];
                        const int rr = (int)qr[qn + lane];
                        __syncwarp();
                        nh += unite(L, y, a2, b2, rr);
                    }
                }
            }
            if (cnt < 32) break;         // the prefix ended inside this batch
            }
            if (PASS == 1) {
#pragma unroll
                for (int k = 0; k < LPT; ++k)
                    if (!((valid >> k) & 1u)) best[k] = ROOT;   // padding lanes stay roots
            }
            if (PASS == 1 && active && HEAVY) {
#pragma unroll
                for (int k = 0; k < LPT; ++k)
                    if (best[k] != ROOT) atomicMin(L + y.off(v, r + k), best[k]);
            } else if (PASS == 1 && active) {
#pragma unroll
                for (int k = 0; k < Q; ++k)
                    if (r + 4 * k < ld)
                        *reinterpret_cast<uint4 *>(L + y.off(v, r + 4 * k)) =
                            make_uint4(best[4 * k], best[4 * k + 1], best[4 * k + 2], best[4 * k + 3]);
            }
        }
    }
    if (PASS == 2) {
        __syncwarp();
        if (lane < qn) nh += unite(L, y, qlo[lane], qhi[lane], (int)qr[lane]);
    }
    if (hooks) {
        for (int o = 16; o; o >>= 1) nh += __shfl_xor_sync(FULL, nh, o);
        if (lane == 0 && nh) atomicAdd(hooks, nh);
    }
}

// Full compression + component count, one thread per 16-byte quad of a label
// row; the grid stride is a multiple of the row length, so a thread keeps
// the same 4 lanes for all its vertices and the CTAs stream whole rows.
// Hub vertices (ids < kHot: the roots of the giant components of skewed
// graphs in nearly every lane) are read through L1 (ld.ca -- their root bit
// is final and a stale parent pointer is still an ancestor) and members of
// hub-rooted components are counted in registers, flushed once per thread,
// so the hub rows see neither hot L2 reads nor per-member atomics.  Other
// non-root cells walk to their root with min-safe path splitting, store it,
// and add 1 to the root cell's member count.  Root cells are never stored by
// their owner (their count is being incremented concurrently).
constexpr int kHot = 4;

__device__ __forceinline__ uint32_t ld_ca(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.global.ca.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// Walk one non-root cell (v, r) with parent p = w and parent word gw to its
// root, store the root, count the member.  Hub-rooted members are counted in
// the warp's shared-memory counters hc[kHot][128] (lane r - r0).
// slot of lane r in the warp's 128 hub counters: the warp's 32 quads cover
// lanes r0.. (wrapping around the row when the row is not a multiple of 128)
__device__ __forceinline__ int hub_slot(int r, int r0, int64_t ld) {
    return ld >= 128 ? (int)(((int64_t)r - r0 + ld) % ld) : r;
}

__device__ __forceinline__ void compress_cell(uint32_t *__restrict__ L, int64_t ld, int64_t lw, uint32_t v,
                                              uint32_t w, uint32_t gw, int r, int r0, uint32_t *hc) {
    uint32_t x = v, p = w;
    while (!is_root(gw)) {          // path splitting, min-safe
        atomicMin(cell(L, ld, x, r), gw);
        x = p;
        p = gw;
        gw = p < (uint32_t)kHot ? ld_ca(cell(L, ld, p, r)) : ld_relaxed(cell(L, ld, p, r));
    }
    if (p != w) L[(int64_t)v * ld + r] = p;
    if (p < (uint32_t)kHot) atomicAdd(hc + p * 128 + hub_slot(r, r0, lw), 1u);
    else atomicAdd(cell(L, ld, p, r), 1u);
}

// Streaming pass over the label rows: a warp reads 32 consecutive 16-byte
// quads (128 lanes) of two rows per step; the non-root cells of the step are
// compacted into a per-warp shared-memory queue and walked 32 at a time, so
// the walks (and their dependent loads) run warp-wide instead of diverging.
constexpr int kCRows = 2;                // label rows per thread per step
constexpr int kCQ = 32 + 32 * 4 * kCRows;  // drain threshold + one step's worth of appends
// rows (optional): the rows to stream (the graph's non-isolated vertices --
// an isolated vertex's row is all roots that nothing points to); n = their count
__global__ void __launch_bounds__(256) k_compress(uint32_t *__restrict__ L, int64_t n, int64_t ld, int32_t W,
                                                  int64_t nq, int64_t vstep,
                                                  unsigned long long *__restrict__ nonroot,
                                                  const int32_t *__restrict__ rows) {
    __shared__ uint32_t qv[8][kCQ], qw[8][kCQ], qr[8][kCQ];
    __shared__ uint32_t hcs[8][kHot * 128];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t *hc = hcs[warp];
    for (int i = lane; i < kHot * 128; i += 32) hc[i] = 0;
    __syncwarp();
    const int64_t lw = nq << 2;     // lanes per row of this pass (a window of the row)
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t q = t % nq;
    const int r = (int)(q << 2);
    const int r0 = (int)((t - lane) % nq) << 2;     // first lane of this warp's 128-lane chunk
    const unsigned FULL = 0xffffffffu;
    unsigned long long cnt = 0;
    int qn = 0;
    const bool live = t < vstep * nq;
    // every lane of the warp walks the same v sequence (vstep is a multiple of rows)
    // software-pipelined row stream: the next step's kCRows 16-byte loads are
    // issued before this step's cells are queued and walked (a stale word is
    // harmless: roots stay roots and any parent read is still an ancestor)
    uint4 nxt[kCRows];
    const int64_t v_first = live ? t / nq : n;
#pragma unroll
    for (int i = 0; i < kCRows; ++i) {
        const int64_t vi = v_first + i * vstep;
        nxt[i] = vi < n ? *(reinterpret_cast<const uint4 *>(L + (rows ? (int64_t)rows[vi] : vi) * ld) + q)
                        : make_uint4(ROOT, ROOT, ROOT, ROOT);
    }
    for (int64_t v = v_first; __any_sync(FULL, v < n); v += kCRows * vstep) {
        uint32_t w[4 * kCRows];
#pragma unroll
        for (int i = 0; i < kCRows; ++i) {
            w[4 * i] = nxt[i].x; w[4 * i + 1] = nxt[i].y; w[4 * i + 2] = nxt[i].z; w[4 * i + 3] = nxt[i].w;
            const int64_t vi = v + (kCRows + i) * vstep;
            nxt[i] = vi < n ? *(reinterpret_cast<const uint4 *>(L + (rows ? (int64_t)rows[vi] : vi) * ld) + q)
                            : make_uint4(ROOT, ROOT, ROOT, ROOT);
        }
        unsigned m = 0;
#pragma unroll
        for (int k = 0; k < 4 * kCRows; ++k)
            if (r + (k & 3) < W && !is_root(w[k])) m |= 1u << k;
        const int c = __popc(m);
        int inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULL, inc, o);
            if (lane >= o) inc += y;
        }
        int pos = qn + inc - c;
        // compile-time cell index: the row words stay in registers
#pragma unroll
        for (int k = 0; k < 4 * kCRows; ++k) {
            if ((m >> k) & 1u) {
                const int64_t vk = v + (k >> 2) * vstep;
                qv[warp][pos] = (uint32_t)(rows ? (int64_t)rows[vk] : vk);
                qw[warp][pos] = w[k];
                qr[warp][pos] = (uint32_t)(r + (k & 3));
                ++pos;
            }
        }
        qn += __shfl_sync(FULL, inc, 31);
        cnt += c;
        __syncwarp();
        // drain 128 / 64 at a time when possible: every parent word is loaded
        // before any walk starts
        while (qn >= 128) {
            qn -= 128;
            uint32_t xv[4], xw[4], xg[4];
            int xr[4];
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                xv[h] = qv[warp][qn + 32 * h + lane];
                xw[h] = qw[warp][qn + 32 * h + lane];
                xr[h] = (int)qr[warp][qn + 32 * h + lane];
            }
            __syncwarp();
#pragma unroll
            for (int h = 0; h < 4; ++h)
                xg[h] = xw[h] < (uint32_t)kHot ? ld_ca(cell(L, ld, xw[h], xr[h])) : ld_relaxed(cell(L, ld, xw[h], xr[h]));
#pragma unroll
            for (int h = 0; h < 4; ++h) compress_cell(L, ld, lw, xv[h], xw[h], xg[h], xr[h], r0, hc);
        }
        while (qn >= 64) {
            qn -= 64;
            const uint32_t cv = qv[warp][qn + lane], cw = qw[warp][qn + lane];
            const int cr = (int)qr[warp][qn + lane];
            const uint32_t dv = qv[warp][qn + 32 + lane], dw = qw[warp][qn + 32 + lane];
            const int dr = (int)qr[warp][qn + 32 + lane];
            __syncwarp();
            const uint32_t gw = cw < (uint32_t)kHot ? ld_ca(cell(L, ld, cw, cr)) : ld_relaxed(cell(L, ld, cw, cr));
            const uint32_t hw = dw < (uint32_t)kHot ? ld_ca(cell(L, ld, dw, dr)) : ld_relaxed(cell(L, ld, dw, dr));
            compress_cell(L, ld, lw, cv, cw, gw, cr, r0, hc);
            compress_cell(L, ld, lw, dv, dw, hw, dr, r0, hc);
        }
        while (qn >= 32) {
            qn -= 32;
            const uint32_t cv = qv[warp][qn + lane], cw = qw[warp][qn + lane];
            const int cr = (int)qr[warp][qn + lane];
            __syncwarp();
            const uint32_t gw = cw < (uint32_t)kHot ? ld_ca(cell(L, ld, cw, cr)) : ld_relaxed(cell(L, ld, cw, cr));
            compress_cell(L, ld, lw, cv, cw, gw, cr, r0, hc);
        }
    }
    __syncwarp();
    if (lane < qn) {
        const uint32_t cv = qv[warp][lane], cw = qw[warp][lane];
        const int cr = (int)qr[warp][lane];
        const uint32_t gw = cw < (uint32_t)kHot ? ld_ca(cell(L, ld, cw, cr)) : ld_relaxed(cell(L, ld, cw, cr));
        compress_cell(L, ld, lw, cv, cw, gw, cr, r0, hc);
    }
    __syncwarp();
    for (int i = lane; i < kHot * 128; i += 32) {
        if (!hc[i]) continue;
        const int rr = lw >= 128 ? (int)((r0 + (i & 127)) % lw) : (i & 127);
        atomicAdd(cell(L, ld, i >> 7, rr), hc[i]);
    }
    if (nonroot) {
        for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(FULL, cnt, o);
        if (lane == 0 && cnt) atomicAdd(nonroot, cnt);
    }
}

// Verification sweep: live (edge, lane) pairs whose endpoint labels differ,
// and non-root cells that do not point at a smaller root.
template <bool UNI>
__global__ void k_verify_edges(const int2 *__restrict__ E, const int32_t *__restrict__ EH,
                               const int32_t *__restrict__ ET, int32_t tu, int64_t me,
                               const int32_t *__restrict__ X, int32_t W, Lay y,
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
            if ((X[r] ^ h) < t &&
                label_of(uv.x, L[y.off(uv.x, r)]) != label_of(uv.y, L[y.off(uv.y, r)]))
                ++nb;
    }
    for (int o = 16; o; o >>= 1) nb += __shfl_xor_sync(0xffffffffu, nb, o);
    if (lane == 0 && nb) atomicAdd(bad, nb);
}
__global__ void k_verify_roots(const uint32_t *__restrict__ L, int64_t n, Lay y, int32_t W,
                               unsigned long long *__restrict__ bad) {
    unsigned long long nb = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * (int64_t)W;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = i / W;
        const int r = (int)(i - v * W);
        const uint32_t w = L[y.off(v, r)];
        if (!is_root(w) && (w >= (uint32_t)v || !is_root(L[y.off(w, r)]))) ++nb;
    }
    for (int o = 16; o; o >>= 1) nb += __shfl_xor_sync(0xffffffffu, nb, o);
    if ((threadIdx.x & 31) == 0 && nb) atomicAdd(bad, nb);
}

__global__ void k_label_sum(const uint32_t *__restrict__ L, int64_t n, Lay y, int32_t W,
                            unsigned long long *__restrict__ out) {
    unsigned long long s = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * (int64_t)W;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = i / W;
        const int r = (int)(i - v * W);
        s += label_of((uint32_t)v, L[y.off(v, r)]);
    }
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

__global__ void k_flush(uint4 *buf, int64_t cnt, uint32_t salt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
         i += (int64_t)gridDim.x * blockDim.x)
        buf[i] = make_uint4(salt, (uint32_t)i, salt, (uint32_t)i);
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
int launch_init(uint32_t *L, int64_t n, int64_t ld, cudaStream_t st) {
    if (n == 0) return IMX_OK;
    const int64_t cells4 = n * (ld >> 2);
    k_init<<<grid_for(cells4), 256, 0, st>>>(L, cells4);
    IMX_CHECK_LAUNCH();
    note_launch();
    return IMX_OK;
}

int run_init(imx_ctx *c) {
    if (c->g->n == 0) return IMX_OK;
    IMX_TRY(launch_init(c->L, c->g->n, c->ld, c->st));
    c->tm.kernel_launches++;
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
                                                    c->ld, c->lay, c->L, hooks);
    IMX_CHECK_LAUNCH();
    count_launch(c);
    return IMX_OK;
}

static int run_hook_enum(imx_ctx *c, unsigned long long *hooks, bool skip_forest = false) {
    imx_graph *g = c->g;
    const int64_t nseg = (int64_t)c->W * g->nb * 31;
    if (nseg + 1 > c->nseg_cap) {
        for (int64_t **p : {&c->seg_a, &c->seg_n, &c->seg_off}) { if (*p) cudaFreeAsync(*p, c->st); *p = nullptr; }
        c->nseg_cap = 0;
        IMX_CUDA(pool_alloc((void **)&c->seg_a, sizeof(int64_t) * (nseg + 1), c->st));
        IMX_CUDA(pool_alloc((void **)&c->seg_n, sizeof(int64_t) * (nseg + 1), c->st));
        IMX_CUDA(pool_alloc((void **)&c->seg_off, sizeof(int64_t) * (nseg + 1), c->st));
        c->nseg_cap = nseg + 1;
        size_t tb = 0;
        IMX_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, c->seg_n, c->seg_off, nseg + 1, c->st));
        if (tb > c->scan_tmp_bytes) {
            if (c->scan_tmp) cudaFreeAsync(c->scan_tmp, c->st);
            IMX_CUDA(pool_alloc(&c->scan_tmp, tb, c->st));
            c->scan_tmp_bytes = tb;
        }
    }
    // one segment per thread: the two lookups per segment are latency-bound
    const int sblocks = (int)std::min<int64_t>(ceil_div(nseg, 128), 148 * 64);
    k_seg_count<<<sblocks, 128, 0, c->st>>>(c->X, c->W, g->nb, g->btmax, g->boff, g->EH, g->lut,
                                            g->lut_bits, c->seg_a, c->seg_n);
    IMX_CHECK_LAUNCH();
    size_t tb = c->scan_tmp_bytes;
    IMX_CUDA(cub::DeviceScan::ExclusiveSum(c->scan_tmp, tb, c->seg_n, c->seg_off, nseg + 1, c->st));
    // blocks per SM: one resident wave, or two for huge enumerations (C4's
    // 307M live pairs: 22.4 -> 21.8 ms; C2's 1.8M pairs prefer one)
    const char *eb_env = getenv("IMX_ENUM_BPSM");
    const double pairs = (double)g->me * (double)c->W * g->thr_mean;
    const int blocks = 148 * (eb_env && atoi(eb_env) > 0 ? atoi(eb_env) : (pairs > 1e8 ? 16 : 8));
    auto kern = g->uniform ? (skip_forest ? k_hook_enum<true, true> : k_hook_enum<true, false>)
                           : (skip_forest ? k_hook_enum<false, true> : k_hook_enum<false, false>);
    // lanes per launch (IMX_ENUM_BLOCK, default all): launches run one after
    // the other.  Measured: narrower blocks are slower on every config (C3:
    // 7.2 ms at 2048 lanes, 8.5 ms at 256, 17.9 ms at 16) -- crowding the
    // warps onto few lanes' trees costs more than the L2 reuse gains.
    const char *eb = getenv("IMX_ENUM_BLOCK");
    const int lb = eb && atoi(eb) > 0 ? atoi(eb) : c->W;
    const int spl = g->nb * 31;
    for (int l0 = 0; l0 < c->W; l0 += lb) {
        const int l1 = std::min(c->W, l0 + lb);
        kern<<<blocks, 256, 0, c->st>>>(c->seg_off, c->seg_a, (int64_t)l0 * spl, (int64_t)l1 * spl, spl, g->E, g->EH,
                                        g->ET, c->X, c->lay, c->L, hooks);
        IMX_CHECK_LAUNCH();
        if (l1 < c->W) count_launch(c);
    }
    IMX_CHECK_LAUNCH();
    count_launch(c, 3);
    return IMX_OK;
}

// ---- heavy rows of the pull sampler ---------------------------------------
// rows [v0, v1); nsl[n] = 0 closes the exclusive scan
__global__ void k_heavy_count(const int64_t *__restrict__ xadj, const int32_t *__restrict__ adj, int64_t n, int T,
                              uint8_t *__restrict__ heavy, int32_t *__restrict__ pre, int64_t *__restrict__ nsl,
                              int64_t v0, int64_t v1) {
    for (int64_t v = v0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < v1; v += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = xadj[v], hi = xadj[v + 1];
        const int64_t s0 = lo;
        while (lo < hi) {                     // first slot with adj >= v (rows ascend)
            const int64_t mid = (lo + hi) >> 1;
            if (adj[mid] < (int32_t)v) lo = mid + 1; else hi = mid;
        }
        const int64_t p = lo - s0;
        const bool h = p > T;
        heavy[v] = h;
        pre[v] = (int32_t)p;
        nsl[v] = h ? (p + T - 1) / T : 0;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) nsl[n] = 0;
}

__global__ void k_heavy_fill(const int64_t *__restrict__ xadj, int64_t n, int T, const int32_t *__restrict__ pre,
                             const int64_t *__restrict__ nsl, const int64_t *__restrict__ off,
                             int32_t *__restrict__ hv, int64_t *__restrict__ ha, int32_t *__restrict__ hl) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = nsl[v];
        for (int64_t i = 0; i < k; ++i) {
            hv[off[v] + i] = (int32_t)v;
            ha[off[v] + i] = xadj[v] + i * T;
            hl[off[v] + i] = (int32_t)((pre[v] - i * T) < T ? (pre[v] - i * T) : T);
        }
    }
}

// A warp owns a whole smaller-neighbour prefix in the light pull passes; the
// graph is balanced when no prefix is long against the per-warp share of the
// edges.
static bool prefix_balanced(const imx_graph *g) {
    const double balanced_prefix = 8.0 * (double)g->me / (148.0 * 64.0);
    return (double)g->max_prefix <= std::max(64.0, balanced_prefix);
}

// slots per heavy slice: IMX_PULL_HEAVY (0 = no splitting), else 10 for
// unbalanced graphs (C3: 8.5 ms by enumeration; pulled with 4 / 6 / 8 / 10 /
// 12 / 16 / 24-slot slices 4.80 / 4.56 / 4.49 / 4.41 / 4.42 / 4.52 / 4.57 ms --
// pass 1 prefers long slices, pass 2 short ones) and no splitting for balanced ones, where
// the extra passes only add work (C2p1: 0.47 -> 0.58 ms at 32)
static int pull_heavy_T(const imx_graph *g) {
    if (const char *e = getenv("IMX_PULL_HEAVY")) return std::max(0, atoi(e));
    return prefix_balanced(g) ? 0 : 10;
}

static void heavy_drop(imx_ctx *c, imx_graph::HeavySlices &H) {
    for (void **p : {(void **)&H.heavy, (void **)&H.hs_v, (void **)&H.hs_a, (void **)&H.hs_len, (void **)&H.pre,
                     (void **)&H.nsl, (void **)&H.off}) {
        if (*p) cudaFreeAsync(*p, c->st);
        *p = nullptr;
    }
    H.nhs = 0;
    H.T = -1;
}

// start a table for slice length T (T > 0): flags and per-row counts to be
// filled by heavy_count_rows over every row, then heavy_finish
int heavy_begin(imx_ctx *c, int pass, int T) {
    imx_graph *g = c->g;
    auto &H = g->hv[pass - 1];
    heavy_drop(c, H);
    if (T <= 0) return IMX_OK;
    const int64_t n = g->n;
    IMX_CUDA(pool_alloc((void **)&H.heavy, n, c->st));
    IMX_CUDA(pool_alloc((void **)&H.pre, sizeof(int32_t) * n, c->st));
    IMX_CUDA(pool_alloc((void **)&H.nsl, sizeof(int64_t) * (n + 1), c->st));
    IMX_CUDA(pool_alloc((void **)&H.off, sizeof(int64_t) * (n + 1), c->st));
    return IMX_OK;
}

int heavy_count_rows(imx_ctx *c, int pass, int T, int64_t v0, int64_t v1) {
    imx_graph *g = c->g;
    auto &H = g->hv[pass - 1];
    if (T <= 0 || v1 <= v0) return IMX_OK;
    k_heavy_count<<<grid_for(v1 - v0), 256, 0, c->st>>>(g->xadj, g->adj, g->n, T, H.heavy, H.pre, H.nsl, v0, v1);
    IMX_CHECK_LAUNCH();
    note_launch(1);
    return IMX_OK;
}

// every row counted: the slices (one host sync for their number); a table
// without heavy rows keeps nothing
int heavy_finish(imx_ctx *c, int pass, int T) {
    imx_graph *g = c->g;
    auto &H = g->hv[pass - 1];
    if (T <= 0 || g->max_prefix <= T) {
        heavy_drop(c, H);
        H.T = T;
        return IMX_OK;
    }
    const int64_t n = g->n;
    size_t tb = 0;
    IMX_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, H.nsl, H.off, n + 1, c->st));
    void *tmp = nullptr;
    IMX_CUDA(pool_alloc(&tmp, tb, c->st));
    IMX_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, H.nsl, H.off, n + 1, c->st));
    int64_t total = 0;
    IMX_CUDA(cudaMemcpyAsync(&total, H.off + n, sizeof total, cudaMemcpyDeviceToHost, c->st));
    IMX_CUDA(cudaStreamSynchronize(c->st));
    if (total > 0) {
        IMX_CUDA(pool_alloc((void **)&H.hs_v, sizeof(int32_t) * total, c->st));
        IMX_CUDA(pool_alloc((void **)&H.hs_a, sizeof(int64_t) * total, c->st));
        IMX_CUDA(pool_alloc((void **)&H.hs_len, sizeof(int32_t) * total, c->st));
        k_heavy_fill<<<grid_for(n), 256, 0, c->st>>>(g->xadj, n, T, H.pre, H.nsl, H.off, H.hs_v, H.hs_a, H.hs_len);
        IMX_CHECK_LAUNCH();
    }
    note_launch(total > 0 ? 3 : 2);
    for (void **p : {(void **)&H.pre, (void **)&H.nsl, (void **)&H.off}) { cudaFreeAsync(*p, c->st); *p = nullptr; }
    cudaFreeAsync(tmp, c->st);
    IMX_CUDA(cudaStreamSynchronize(c->st));   // the slices are shared by every context of the graph
    H.nhs = total;
    H.T = T;
    return IMX_OK;
}

void heavy_abort(imx_ctx *c, int pass) { heavy_drop(c, c->g->hv[pass - 1]); }

// the heavy-row slices of the graph for slice length T, cached on the graph
int ensure_heavy(imx_ctx *c, int pass, int T) {
    imx_graph *g = c->g;
    auto &H = g->hv[pass - 1];
    if (H.T == T) return IMX_OK;
    if (T <= 0 || g->max_prefix <= T) {
        heavy_drop(c, H);
        H.T = T;
        return IMX_OK;
    }
    IMX_TRY(heavy_begin(c, pass, T));
    IMX_TRY(heavy_count_rows(c, pass, T, 0, g->n));
    return heavy_finish(c, pass, T);
}

// blocks per SM of the pull grids (IMX_PULL_BPSM, default 16): about three
// times what fits at once -- later waves of blocks measured faster than one
// resident wave (C3: 4.76 / 4.65 / 4.55 ms at one wave / 8 / 16 per SM;
// C2p1 0.487 / 0.464 / 0.443 ms; 32 per SM is slower on C2p1)
static int pull_bpsm() {
    const char *e = getenv("IMX_PULL_BPSM");
    return e && atoi(e) > 0 ? atoi(e) : 16;
}

static int run_pull(imx_ctx *c, int pass, unsigned long long *hooks) {
    imx_graph *g = c->g;
    const int64_t n = g->n;
    if (n == 0) return IMX_OK;
    IMX_TRY(ensure_thr(g));
    // pass 1 (atomicMin per slice and lane) prefers longer slices than
    // pass 2 (unions per slice): its table uses IMX_PULL_HEAVY1 (3) x T slots
    // (C3 pass 1 0.94 -> 0.83 ms)
    const int T2 = pull_heavy_T(g);
    const char *h1 = getenv("IMX_PULL_HEAVY1");
    const int T = pass == 1 && T2 > 0 ? T2 * (h1 && atoi(h1) > 0 ? atoi(h1) : 3) : T2;
    IMX_TRY(ensure_heavy(c, pass, T));
    const auto &H = g->hv[pass - 1];
    // 8 lanes per thread once a row spans several warp-widths of quads
    const char *wm = getenv("IMX_PULL_WIDE_MIN");
    const bool wide = c->W >= (wm && atoi(wm) > 0 ? atoi(wm) : 256);
    const int lpt = wide ? 8 : 4;
    const int64_t ldp = (c->ld + lpt - 1) / lpt * lpt;
    const size_t smem = sizeof(int32_t) * ldp + sizeof(uint32_t) * 3 * (32 + 32 * lpt) * 8;
    if (smem > 200 * 1024) { set_error("width %d too large for one context", c->W); return IMX_EINVAL; }
    const int blocks = (int)std::min<int64_t>(ceil_div(n, 8), 148 * pull_bpsm());
    using KF = void (*)(const int64_t *, const int32_t *, const int32_t *, const int32_t *, int32_t, int64_t,
                        const int32_t *, int32_t, int64_t, Lay, uint32_t *, unsigned long long *, const uint8_t *,
                        const int32_t *, const int64_t *, const int32_t *, int64_t);
    // [heavy][pass-1][uniform][wide]
    static const KF kerns[2][2][2][2] = {
        {{{k_pull<1, false, 4, false>, k_pull<1, false, 8, false>}, {k_pull<1, true, 4, false>, k_pull<1, true, 8, false>}},
         {{k_pull<2, false, 4, false>, k_pull<2, false, 8, false>}, {k_pull<2, true, 4, false>, k_pull<2, true, 8, false>}}},
        {{{k_pull<1, false, 4, true>, k_pull<1, false, 8, true>}, {k_pull<1, true, 4, true>, k_pull<1, true, 8, true>}},
         {{k_pull<2, false, 4, true>, k_pull<2, false, 8, true>}, {k_pull<2, true, 4, true>, k_pull<2, true, 8, true>}}}};
    const int hv = H.nhs > 0 ? 2 : 1;
    for (int h = 0; h < hv; ++h) {
        KF kern = kerns[h][pass - 1][g->uniform ? 1 : 0][wide ? 1 : 0];
        if (smem > 48 * 1024)
            IMX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const int hb = h ? (int)std::min<int64_t>(ceil_div(H.nhs, 8), 148 * pull_bpsm()) : blocks;
        kern<<<hb, 256, smem, c->st>>>(g->xadj, g->adj, g->hash, g->thr, g->thr_u, n, c->X, c->W, c->ld, c->lay, c->L, hooks,
                                       H.nhs > 0 ? H.heavy : nullptr, H.hs_v, H.hs_a, H.hs_len, H.nhs);
        IMX_CHECK_LAUNCH();
        count_launch(c);
    }
    return IMX_OK;
}

// Sampler strategy.  Interval enumeration touches only live (edge, lane)
// pairs but each costs ~4 random label accesses; the pull passes cost two
// dense membership scans (ALU only) plus random accesses for the non-forest
// live edges only, but a warp owns a whole row prefix, so a very long prefix
// (a high-degree vertex with many smaller neighbours) serialises.
enum { HOOK_ENUM = 0, HOOK_PULL = 1, HOOK_DENSE = 2, HOOK_HYBRID = 3, HOOK_SCAN = 4 };
static int hook_mode(const imx_graph *g, int32_t W) {
    const char *m = getenv("IMX_HOOK");
    if (m && !strcmp(m, "dense")) return HOOK_DENSE;
    // enumeration and the lane buckets assume 31-bit hashes ((x ^ h) >= 0);
    // the pull scans test exactly
    if (g->hash_neg) return HOOK_PULL;
    if (m && !strcmp(m, "enum")) return HOOK_ENUM;
    if (m && !strcmp(m, "pull")) return HOOK_PULL;
    if (m && !strcmp(m, "hybrid")) return HOOK_HYBRID;
    if (m && !strcmp(m, "scan")) return scan_eligible(g) ? HOOK_SCAN : HOOK_PULL;
    // uniform thresholds: the bucketed pull forest (scan.cu), except for
    // small dense work, where the plain pull passes win (C1: 0.039 vs 0.067 ms)
    if (scan_eligible(g) && (double)g->me * (double)W > 3.2e7) return HOOK_SCAN;
    const char *t = getenv("IMX_PULL_MIN_P");
    const double pmin = t ? atof(t) : 0.02;
    // long prefixes are split into slices (heavy rows), so they only
    // unbalance the pull passes when splitting is off
    const bool balanced = pull_heavy_T(g) > 0 || prefix_balanced(g);
    if (g->thr_mean >= pmin && balanced) return HOOK_PULL;
    // small dense work (C1: 31k edges x 128 lanes): two scans beat the
    // enumeration's segment count + scan + launch chain
    if (balanced && (double)g->me * (double)W <= 3.2e7) return HOOK_PULL;
    return HOOK_ENUM;
}

// init + hook phases of one propagate (events bracket them)
static bool needs_index(int mode) { return mode == HOOK_ENUM || mode == HOOK_DENSE || mode == HOOK_HYBRID; }

static int run_sample_cc(imx_ctx *c, unsigned long long *hooks, cudaEvent_t e_init, cudaEvent_t e_hook) {
    imx_graph *g = c->g;
    int mode = g->me ? hook_mode(g, c->W) : HOOK_ENUM;
    if (g->me && needs_index(mode)) {
        // the edge index needs the settled thresholds (ensure_index waits for
        // deferred weights), which may change the strategy
        IMX_TRY(ensure_index(g));
        mode = hook_mode(g, c->W);
        if (needs_index(mode)) IMX_TRY(ensure_index(g));
    }
    // a streamed CSR: only the scan's first pass can start on the chunks
    // that are up; everything else needs the settled structure
    if (g->struct_pending && mode != HOOK_SCAN) {
        IMX_TRY(graph_settle_structure(g));
        mode = g->me ? hook_mode(g, c->W) : HOOK_ENUM;
    }
    // scan / pull with a deferred graph run on the speculative threshold
    c->spec_used = g->thr_pending;
    if (mode == HOOK_SCAN) {
        if (g->struct_pending) IMX_TRY(run_scan_streamed(c));
        else IMX_TRY(run_scan(c, 1, nullptr));
        if (e_init) IMX_CUDA(cudaEventRecord(e_init, c->st));
        IMX_TRY(run_scan(c, 2, hooks));
    } else if (mode == HOOK_PULL || mode == HOOK_HYBRID) {
        IMX_TRY(run_pull(c, 1, nullptr));
        if (e_init) IMX_CUDA(cudaEventRecord(e_init, c->st));
        if (mode == HOOK_PULL) IMX_TRY(run_pull(c, 2, hooks));
        else IMX_TRY(run_hook_enum(c, hooks, true));
    } else {
        IMX_TRY(run_init(c));
        if (e_init) IMX_CUDA(cudaEventRecord(e_init, c->st));
        if (g->me) IMX_TRY(mode == HOOK_DENSE ? run_hook_dense(c, hooks) : run_hook_enum(c, hooks));
    }
    if (e_hook) IMX_CUDA(cudaEventRecord(e_hook, c->st));
    c->tm.hook_launches++;
    return IMX_OK;
}

// Lanes per compress pass: the whole row, or (IMX_COMPRESS_WINDOW / large
// label matrices) windows of lanes whose n*window*4 bytes stay L2-resident,
// so the dependent parent reads and root-count atomics hit L2.
static int64_t compress_window(int64_t n, int64_t ld) {
    if (const char *e = getenv("IMX_COMPRESS_WINDOW")) {
        const int64_t w = atoll(e);
        if (w > 0) return std::min<int64_t>(ld, std::max<int64_t>(4, w / 4 * 4));
    }
    return ld;
}

int launch_compress(uint32_t *L, int64_t n, int64_t ld, int32_t W, unsigned long long *nonroot,
                    cudaStream_t st, int *launches, int64_t window, const int32_t *rows, int64_t nrows) {
    if (rows) n = nrows;             // stream only these rows
    if (n == 0) return IMX_OK;
    const int64_t win = window > 0 ? window : compress_window(n, ld);
    if (launches) *launches = (int)ceil_div(W, win);
    for (int64_t l0 = 0; l0 < W; l0 += win) {
        const int32_t wl = (int32_t)std::min<int64_t>(win, W - l0);
        // grid stride = a whole number of rows, so every thread keeps its quad
        const int64_t nq = (wl + 3) >> 2;
        // threads: one resident wave (148 x 2048) for small matrices, more for
        // large ones (C2 77 -> 68 us at one wave instead of two; C3 1.06 ->
        // 0.98 ms at eight; C4 6.35 -> 5.46 ms at sixteen)
        const char *cw_env = getenv("IMX_COMPRESS_WAVES");
        const int64_t quads = n * nq;
        const int waves = cw_env && atoi(cw_env) > 0 ? atoi(cw_env)
                          : (quads < ((int64_t)1 << 26) ? 1 : (quads < ((int64_t)1 << 29) ? 8 : 16));
        const int64_t want = std::min<int64_t>(n * nq, (int64_t)148 * 2048 * waves);
        const int64_t prows = std::max<int64_t>(1, want / nq);
        const int64_t threads = prows * nq;
        const int blocks = (int)ceil_div(threads, 256);
        // threads beyond rows*nq would break the fixed-quad mapping: size the
        // stride from the launched thread count, rounded down to whole rows
        const int64_t vstep = ((int64_t)blocks * 256) / nq;
        k_compress<<<blocks, 256, 0, st>>>(L + l0, n, ld, wl, nq, vstep, nonroot, rows);
        IMX_CHECK_LAUNCH();
        note_launch();
    }
    return IMX_OK;
}

// Compression of the whole matrix.  Lane-tiled contexts (ctx.cu) compress
// tile by tile in place: a tile is a contiguous [n][tl] block, so its walks
// and root-count atomics stay in L2 (C5: 128 MB tiles of 32 lanes), and the
// memo fused into the propagate (imx_set_fuse_memo) sums each tile's gains
// while it is still on chip.
static int run_compress(imx_ctx *c, unsigned long long *nonroot) {
    const int64_t n = c->g->n;
    if (n == 0) return IMX_OK;
    IMX_TRY(ensure_nz_rows(c->g));
    const int32_t *rows = c->g->nz_rows;
    const int64_t nrows = c->g->n_nz;
    if (!c->lay.tiled()) {
        int k = 0;
        IMX_TRY(launch_compress(c->L, n, c->ld, c->W, nonroot, c->st, &k, 0, rows, nrows));
        c->tm.kernel_launches += k;
        return IMX_OK;
    }
    // each tile in windows of 32 lanes: a window is one 128-byte line per row,
    // so its walks stay in L2 (C5, 64-lane tiles: compress 40.1 -> 33.2 ms; the
    // tiles themselves are 64 lanes wide because the pass-1 row stores lose
    // DRAM locality at 128 bytes per tile: 10.8 vs 20.1 ms at 32)
    const int64_t tl = c->lay.ld, tiles = c->ld / tl;
    const int64_t win = std::min<int64_t>(tl, 32);
    const bool fuse = c->fuse_memo && !c->C;
    for (int64_t t = 0; t < tiles; ++t) {
        uint32_t *T = c->L + t * c->lay.tstride;
        for (int64_t w0 = 0; w0 < tl; w0 += win) {
            const int64_t l0 = t * tl + w0;
            if (l0 >= c->W) break;
            const int32_t wl = (int32_t)std::min<int64_t>(win, c->W - l0);
            int k = 0;
            IMX_TRY(launch_compress(T + w0, n, tl, wl, nonroot, c->st, &k, win, rows, nrows));
            c->tm.kernel_launches += k;
            if (fuse) {
                // the memo's gains over this window's scored lanes, while it is in L2
                const int32_t ns_w = (int32_t)std::max<int64_t>(0, std::min<int64_t>(wl, c->ns - l0));
                if (l0 == 0 || ns_w > 0) IMX_TRY(launch_gains_tile(T + w0, n, tl, ns_w, l0 == 0, c->gains, c->st));
                c->tm.kernel_launches++;
            }
        }
    }
    if (fuse) c->gains_fused = true;
    return IMX_OK;
}

static int label_sum(imx_ctx *c, int64_t *out) {
    const int64_t n = c->g->n;
    IMX_CUDA(cudaMemsetAsync(c->scratch + 4, 0, sizeof(unsigned long long), c->st));
    if (n) {
        k_label_sum<<<grid_for(n * c->W), 256, 0, c->st>>>(c->L, n, c->lay, c->W, c->scratch + 4);
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

}  // namespace imx

using namespace imx;

namespace imx {
int spec_settle(imx_ctx *c, int32_t *held) {
    *held = 1;
    if (!c->spec_used) return IMX_OK;
    imx_graph *g = c->g;
    IMX_TRY(graph_settle(g));
    c->spec_used = false;
    if (!g->uniform || g->thr_u != c->spec_thr || g->hash_neg) {
        *held = 0;
        c->labels_ready = false;
        c->memo_ready = false;
        c->celf_ready = false;
        c->gains_fused = false;
    }
    return IMX_OK;
}

int spec_guard(imx_ctx *c) {
    if (!c->spec_used) return IMX_OK;
    int32_t held = 1;
    IMX_TRY(spec_settle(c, &held));
    if (!held) {
        set_error("results stand on a speculative threshold that the uploaded weights do not confirm: propagate again");
        return IMX_EINVAL;
    }
    return IMX_OK;
}
}  // namespace imx

extern "C" int imx_spec_defer(imx_ctx *c, int32_t on) {
    CTX_CHECK(c);
    c->spec_defer = on != 0;
    return IMX_OK;
}

extern "C" int imx_spec_settle(imx_ctx *c, int32_t *held) {
    CTX_CHECK(c);
    if (!held) { set_error("NULL argument"); return IMX_EINVAL; }
    return spec_settle(c, held);
}

extern "C" int imx_set_fuse_memo(imx_ctx *c, int32_t on) {
    CTX_CHECK(c);
    c->fuse_memo = on != 0;
    return IMX_OK;
}

extern "C" int imx_propagate(imx_ctx *c, int32_t verify, imx_prop_stats *st) {
    CTX_CHECK(c);
    c->gains_fused = false;
    if (c->C) { cudaFreeAsync(c->C, c->st); c->C = nullptr; }   // back to encoded mode
    c->lay = c->lay_native;
    imx_graph *g = c->g;
    const int64_t n = g->n;
    if (st) st->sweeps = 0;
    unsigned long long *sc = c->scratch;
    IMX_CUDA(cudaMemsetAsync(sc, 0, sizeof(unsigned long long) * 4, c->st));
    IMX_CUDA(cudaEventRecord(c->ev[0], c->st));
    if (g->m2 > 0) {
        const int32_t t_spec = g->thr_u;
        IMX_TRY(run_sample_cc(c, st ? sc : nullptr, c->ev[1], c->ev[2]));
        IMX_TRY(run_compress(c, st ? sc + 1 : nullptr));
        if (c->spec_used && c->spec_defer) {
            c->spec_thr = t_spec;            // checked by imx_spec_settle / spec_guard
        } else if (c->spec_used) {
            // the propagate ran on the speculative uniform threshold while the
            // weights were still uploading: wait for them (the device is busy
            // meanwhile) and run again if the thresholds are not that one
            IMX_TRY(graph_settle(g));
            c->spec_used = false;
            if (!g->uniform || g->thr_u != t_spec || g->hash_neg) {
                c->gains_fused = false;
                IMX_CUDA(cudaMemsetAsync(sc, 0, sizeof(unsigned long long) * 4, c->st));
                IMX_CUDA(cudaEventRecord(c->ev[0], c->st));
                IMX_TRY(run_sample_cc(c, st ? sc : nullptr, c->ev[1], c->ev[2]));
                IMX_TRY(run_compress(c, st ? sc + 1 : nullptr));
            }
        }
    } else {
        IMX_TRY(run_init(c));
        IMX_CUDA(cudaEventRecord(c->ev[1], c->st));
        IMX_CUDA(cudaEventRecord(c->ev[2], c->st));
    }
    IMX_CUDA(cudaEventRecord(c->ev[3], c->st));
    // no host sync here: the caller's next calls (memo, CELF reset) are
    // enqueued while the device still propagates; the phase times are read
    // when asked for (imx_get_timings)
    c->tm_pending |= 1;
    c->labels_ready = true;
    c->memo_ready = false;
    c->celf_ready = false;
    if (c->C) { cudaFreeAsync(c->C, c->st); c->C = nullptr; }   // back to encoded mode
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
        changed = (int64_t)hc[1];
        push_stat(st, IMX_MODE_HOOK, changed, lsum);
    }
    if (verify || (st && changed > 0)) {
        if (g->me) IMX_TRY(ensure_index(g));
        IMX_CUDA(cudaMemsetAsync(sc + 2, 0, sizeof(unsigned long long), c->st));
        if (g->me) {
            if (g->uniform)
                k_verify_edges<true><<<grid_for(g->me * 32), 256, 0, c->st>>>(g->E, g->EH, g->ET, g->thr_u, g->me, c->X, c->W, c->lay, c->L, sc + 2);
            else
                k_verify_edges<false><<<grid_for(g->me * 32), 256, 0, c->st>>>(g->E, g->EH, g->ET, g->thr_u, g->me, c->X, c->W, c->lay, c->L, sc + 2);
            IMX_CHECK_LAUNCH();
        }
        k_verify_roots<<<grid_for(n * c->W), 256, 0, c->st>>>(c->L, n, c->lay, c->W, sc + 2);
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

extern "C" int imx_bench_propagate(imx_ctx *c, int32_t reps, int32_t flush_l2, float *avg_total_ms,
                                   float *avg_hook_ms, float *avg_compress_ms, float *avg_init_ms) {
    CTX_CHECK(c);
    c->gains_fused = false;
    if (reps < 1) { set_error("reps must be >= 1"); return IMX_EINVAL; }
    IMX_TRY(graph_settle(c->g));
    uint4 *fb = nullptr;
    const int64_t fcnt = (int64_t(256) << 20) / 16;  // 256 MB > 126 MB L2
    if (flush_l2) IMX_CUDA(pool_alloc((void **)&fb, fcnt * 16, c->st));
    std::vector<cudaEvent_t> ev(4 * reps);
    for (auto &e : ev) IMX_CUDA(cudaEventCreate(&e));
    if (c->C) { cudaFreeAsync(c->C, c->st); c->C = nullptr; }
    c->lay = c->lay_native;
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
    if (fb) cudaFreeAsync(fb, c->st);
    if (avg_total_ms) *avg_total_ms = (float)(tot / reps);
    if (avg_hook_ms) *avg_hook_ms = (float)(hk / reps);
    if (avg_compress_ms) *avg_compress_ms = (float)(cp / reps);
    if (avg_init_ms) *avg_init_ms = (float)(in / reps);
    c->labels_ready = true;
    c->memo_ready = false;
    c->celf_ready = false;
    return IMX_OK;
}
