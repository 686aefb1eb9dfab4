// celf.cu -- K6-K8: CELF seed selection on the device (reference
// select_seeds / marginal_gain / commit_seed, selection.py:63-149).
//
// Round-based exact formulation.  Gains are computed on one
// fixed sample family, so marginal gain is submodular and the reference's
// lazy heap commits, at every round, the lexicographic argmax of the fresh
// gains (max gain, then min id), after refreshing -- in (-stale, id) order --
// exactly the vertices whose stale key (-stale, id) does not exceed the
// winner's fresh key.  Those vertices are a PREFIX of the non-seeds sorted by
// stale key, so the device keeps that order as one sorted array of packed keys
// (prio << vb | ~id): a round evaluates prefix batches of doubling size until
// the best fresh key is below the next stale key, drops the refreshed prefix,
// commits the winner and merges the other refreshed vertices back with their
// fresh keys.  No per-round scan or sort of all n vertices; one or two host
// syncs per round; the dequeue trace is the evaluated prefix itself.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cub/cub.cuh>
#include <cooperative_groups.h>

namespace cg = cooperative_groups;

#include "ctx.cuh"
#include "uf.cuh"

namespace imx {

__device__ __forceinline__ unsigned long long pack_key(int64_t prio, uint32_t v, int vb) {
    const uint32_t vmask = (vb >= 32) ? 0xffffffffu : ((1u << vb) - 1u);
    return ((unsigned long long)prio << vb) | (unsigned long long)(vmask - v);
}

template <bool ENC>
__device__ __forceinline__ uint32_t cell_size(const uint32_t *__restrict__ L, const uint32_t *__restrict__ C,
                                              const Lay &ld, uint32_t u, uint32_t w, int r, uint32_t &label) {
    if (ENC) {
        if (is_root(w)) { label = u; return (w & COUNT) + 1u; }
        label = w;
        return (L[cell_off(ld, w, r)] & COUNT) + 1u;
    }
    label = w;
    return C[cell_off(ld, w, r)];
}

// marginal_gain (selection.py:63-70): sum over scored lanes of the component
// size of u's component when that component is not covered yet.  One CTA per
// candidate; each thread takes 16-byte quads of the label row so the label
// loads are coalesced and the dependent size / bitmap gathers of 4 lanes are
// in flight together.
constexpr int kEvalThreads = 128;
template <bool ENC>
__global__ void __launch_bounds__(kEvalThreads) k_eval(const int32_t *__restrict__ cand, int64_t cnt,
                                                       const uint32_t *__restrict__ L, const uint32_t *__restrict__ C,
                                                       const uint32_t *__restrict__ cov, Lay ld, int32_t ns,
                                                       int32_t cw, int64_t *__restrict__ out) {
    __shared__ unsigned long long part[kEvalThreads / 32];
    const int nqs = (ns + 3) >> 2;
    for (int64_t i = blockIdx.x; i < cnt; i += gridDim.x) {
        const int64_t u = cand[i];
        if (u < 0) { if (threadIdx.x == 0) out[i] = 0; continue; }
        const uint32_t *rowbase = L;   // quads via ld.off (rows or lane tiles)
        unsigned long long acc = 0;
        for (int q = threadIdx.x; q < nqs; q += kEvalThreads) {
            const uint4 l4 = row_quad(rowbase, ld, u, q);
            const uint32_t lv[4] = {l4.x, l4.y, l4.z, l4.w};
            uint32_t wd[4], s[4];
            const int r = q << 2;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const bool in = r + j < ns;
                uint32_t lab = 0;
                s[j] = in ? cell_size<ENC>(L, C, ld, (uint32_t)u, lv[j], r + j, lab) : 0u;
                wd[j] = in ? cov[(int64_t)lab * cw + ((r + j) >> 5)] : 0xffffffffu;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (!((wd[j] >> ((r + j) & 31)) & 1u)) acc += s[j];
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

// commit_seed (selection.py:73-81): own u's component in every scored lane;
// per_sim[r] += its size when newly owned (K8, SelectionResult.spread_se)
// seeds whose newly covered components are listed per lane (the seed table
// of the early CELF rounds, tab_covered)
constexpr int kTab = 4;

template <bool ENC>
__global__ void k_commit(int32_t u, const uint32_t *__restrict__ L, const uint32_t *__restrict__ C,
                         uint32_t *__restrict__ cov, Lay ld, int32_t ns, int32_t cw,
                         int64_t *__restrict__ per_sim, uint8_t *__restrict__ inS,
                         unsigned long long *__restrict__ gain, int2 *__restrict__ tab_row) {
    unsigned long long acc = 0;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < ns; r += gridDim.x * blockDim.x) {
        uint32_t lab;
        const uint32_t s = cell_size<ENC>(L, C, ld, (uint32_t)u, L[cell_off(ld, u, r)], r, lab);
        const uint32_t bit = 1u << (r & 31);
        const uint32_t old = atomicOr(cov + (int64_t)lab * cw + (r >> 5), bit);
        if (!(old & bit)) {
            per_sim[r] += s;
            acc += s;
        }
        if (tab_row) tab_row[r] = (old & bit) ? make_int2(-1, 0) : make_int2((int)lab, (int)s);
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(gain, acc);
    if (blockIdx.x == 0 && threadIdx.x == 0) inS[u] = 1;
}

__global__ void k_pack_keys(const int64_t *__restrict__ prio, int64_t n, int vb, int32_t *__restrict__ ids,
                            unsigned long long *__restrict__ keys, unsigned long long *__restrict__ maxp) {
    unsigned long long m = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = prio[v] < 0 ? 0 : prio[v];
        ids[v] = (int32_t)v;
        keys[v] = pack_key(p, (uint32_t)v, vb);
        m = (unsigned long long)p > m ? (unsigned long long)p : m;
    }
    for (int o = 16; o; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(0xffffffffu, m, o);
        m = y > m ? y : m;
    }
    if ((threadIdx.x & 31) == 0 && m) atomicMax(maxp, m);
}

// merge two key-descending lists (unique keys) into out
__global__ void k_merge(const int32_t *__restrict__ aid, const unsigned long long *__restrict__ akey, int64_t na,
                        const int32_t *__restrict__ bid, const unsigned long long *__restrict__ bkey, int64_t nb,
                        int32_t *__restrict__ oid, unsigned long long *__restrict__ okey) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < na + nb;
         i += (int64_t)gridDim.x * blockDim.x) {
        const bool in_a = i < na;
        const int64_t j = in_a ? i : i - na;
        const unsigned long long key = in_a ? akey[j] : bkey[j];
        const unsigned long long *other = in_a ? bkey : akey;
        int64_t lo = 0, hi = in_a ? nb : na;      // number of other keys > key
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (other[mid] > key) lo = mid + 1; else hi = mid;
        }
        const int64_t pos = j + lo;
        oid[pos] = in_a ? aid[j] : bid[j];
        okey[pos] = key;
    }
}

// t: the seed count before this commit when it is a round of the CELF loop
// (its seed-table row, kTab, is written too), -1 otherwise
static void launch_commit(imx_ctx *c, int32_t u, unsigned long long *gain, int32_t t = -1) {
    const int blocks = grid_for(std::max(c->ns, 1));
    int2 *row = (t >= 0 && t < kTab && c->stab && !c->C) ? c->stab + (int64_t)t * c->ld : nullptr;
    if (c->C) k_commit<false><<<blocks, 256, 0, c->st>>>(u, c->L, c->C, c->cov, c->lay, c->ns, c->cw, c->per_sim, c->inS, gain, nullptr);
    else k_commit<true><<<blocks, 256, 0, c->st>>>(u, c->L, nullptr, c->cov, c->lay, c->ns, c->cw, c->per_sim, c->inS, gain, row);
}

static int celf_eval_dev(imx_ctx *c, const int32_t *dcand, int64_t cnt, int64_t *dout) {
    if (cnt <= 0) return IMX_OK;
    const int blocks = (int)std::min<int64_t>(cnt, 148 * 16);
    if (c->C) k_eval<false><<<blocks, kEvalThreads, 0, c->st>>>(dcand, cnt, c->L, c->C, c->cov, c->lay, c->ns, c->cw, dout);
    else k_eval<true><<<blocks, kEvalThreads, 0, c->st>>>(dcand, cnt, c->L, nullptr, c->cov, c->lay, c->ns, c->cw, dout);
    IMX_CHECK_LAUNCH();
    count_launch(c);
    return IMX_OK;
}

static inline int64_t key_prio(const imx_ctx *c, unsigned long long k) { return (int64_t)(k >> c->vb); }
static inline unsigned long long host_key(const imx_ctx *c, int64_t prio, int32_t v) {
    const uint64_t vmask = (c->vb >= 32) ? 0xffffffffull : ((1ull << c->vb) - 1);
    return ((unsigned long long)prio << c->vb) | (vmask - (uint64_t)v);
}

// evaluate order[lo, hi) of the current order; ids/keys of order[lo, min(hi+1, len))
// and fresh gains of [lo, hi) land in the caller's host buffers.
// With a communicator (comm), the batch's partial gains -- and, when pend is
// given, one extra element: the previous commit's partial gain -- are summed
// over the ranks on the device before the copy; *pend then holds the sum.
static int celf_prefix(imx_ctx *c, int64_t lo, int64_t hi, int32_t *ids, unsigned long long *keys,
                       int64_t *fresh, imx_comm *comm = nullptr, int64_t *pend = nullptr) {
    const int64_t len = c->olen;
    hi = std::min(hi, len);
    if (lo >= hi) return IMX_OK;
    const int64_t base = c->ostart, cnt = hi - lo;
    IMX_TRY(celf_eval_dev(c, c->oid[c->ocur] + base + lo, cnt, c->eval_out));
    if (comm) {
        if (pend) IMX_CUDA(cudaMemcpyAsync(c->eval_out + cnt, pend, sizeof(int64_t), cudaMemcpyHostToDevice, c->st));
        IMX_TRY(comm_allreduce_i64(comm, c->eval_out, cnt + (pend ? 1 : 0), c->st));
        if (pend) IMX_CUDA(cudaMemcpyAsync(pend, c->eval_out + cnt, sizeof(int64_t), cudaMemcpyDeviceToHost, c->st));
    }
    const int64_t fetch = std::min(hi + 1, len) - lo;
    IMX_CUDA(cudaMemcpyAsync(ids, c->oid[c->ocur] + base + lo, sizeof(int32_t) * fetch, cudaMemcpyDeviceToHost, c->st));
    IMX_CUDA(cudaMemcpyAsync(keys, c->okey[c->ocur] + base + lo, sizeof(unsigned long long) * fetch,
                             cudaMemcpyDeviceToHost, c->st));
    IMX_CUDA(cudaMemcpyAsync(fresh, c->eval_out, sizeof(int64_t) * cnt, cudaMemcpyDeviceToHost, c->st));
    IMX_CUDA(cudaStreamSynchronize(c->st));
    c->evaluated += cnt;
    return IMX_OK;
}

// drop order[0, k), merge cnt (ids, keys) back (keys descending); async
static int celf_advance(imx_ctx *c, int64_t k, const int32_t *ids, const unsigned long long *keys, int64_t cnt) {
    if (k > c->olen) { set_error("advance past the end of the candidate order"); return IMX_EINVAL; }
    c->ostart += k;
    c->olen -= k;
    if (cnt <= 0) return IMX_OK;
    IMX_TRY(ensure_pinned(c, cnt + 8));
    std::copy(ids, ids + cnt, c->h_ids);
    std::copy(keys, keys + cnt, reinterpret_cast<unsigned long long *>(c->h_vals) + 8);
    IMX_CUDA(cudaMemcpyAsync(c->d_ids, c->h_ids, sizeof(int32_t) * cnt, cudaMemcpyHostToDevice, c->st));
    IMX_CUDA(cudaMemcpyAsync(c->d_vals, c->h_vals + 8, sizeof(int64_t) * cnt, cudaMemcpyHostToDevice, c->st));
    const int nxt = c->ocur ^ 1;
    k_merge<<<grid_for(c->olen + cnt), 256, 0, c->st>>>(
        c->oid[c->ocur] + c->ostart, c->okey[c->ocur] + c->ostart, c->olen, c->d_ids,
        reinterpret_cast<const unsigned long long *>(c->d_vals), cnt, c->oid[nxt], c->okey[nxt]);
    IMX_CHECK_LAUNCH();
    count_launch(c);
    c->ocur = nxt;
    c->ostart = 0;
    c->olen += cnt;
    // the staging buffers are reused next round: both callers read the commit
    // gain back and synchronise the stream before returning
    return IMX_OK;
}

// ---------------------------------------------------------------------------
// The whole CELF loop as ONE cooperative kernel (single-rank path).
//
// Every block keeps the same copy of the round state (order window, best
// candidate, trace length) and takes the same decisions from the same global
// data, so grid-wide barriers replace the host round trips of the
// host-driven loop.  A round: evaluate prefix batches (CTA per candidate),
// barrier, every block reduces the best fresh key and tests the stop rule;
// the refreshed prefix length kr is a binary search (keys are sorted); the
// prefix is written to the trace, the winner committed; the other kr-1
// refreshed vertices are ranked by their fresh keys (O(kr^2) compare-count,
// kr <= kMaxRank), scattered, and merged back into the order.  A round that
// does not fit (trace buffer full, kr too large) stops the kernel with the
// state saved; the host finishes that round and relaunches.
// ---------------------------------------------------------------------------
constexpr int64_t kMaxRank = 16384;
constexpr int64_t kSmemBack = 2048;     // refreshed keys staged in shared memory for the merge


template <bool ENC>
__device__ __forceinline__ int64_t block_eval(const uint32_t *__restrict__ L, const uint32_t *__restrict__ C,
                                              const uint32_t *__restrict__ cov, Lay ld, int32_t ns,
                                              int32_t cw, int64_t u, unsigned long long *red) {
    const int nqs = (ns + 3) >> 2;
    const uint32_t *rowbase = L;   // quads via ld.off (rows or lane tiles)
    unsigned long long acc = 0;
    for (int q = threadIdx.x; q < nqs; q += blockDim.x) {
        const uint4 l4 = row_quad(rowbase, ld, u, q);
        const uint32_t lv[4] = {l4.x, l4.y, l4.z, l4.w};
        uint32_t wd[4], sz[4];
        const int r = q << 2;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const bool in = r + j < ns;
            uint32_t lab = 0;
            sz[j] = in ? cell_size<ENC>(L, C, ld, (uint32_t)u, lv[j], r + j, lab) : 0u;
            wd[j] = in ? cov[(int64_t)lab * cw + ((r + j) >> 5)] : 0xffffffffu;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (!((wd[j] >> ((r + j) & 31)) & 1u)) acc += sz[j];
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    unsigned long long tot = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) tot += red[k];
    return (int64_t)tot;
}

// Number of leading entries of the descending array a[0, n) that are > key
// (GE: >= key), by one warp: a 33-ary search (32 pivots per step, one
// coalesced-free load per lane), so ~log33(n) dependent loads instead of
// log2(n).  Every lane returns the result.
template <bool GE>
__device__ __forceinline__ int64_t warp_count_above(const unsigned long long *a, int64_t n,
                                                    unsigned long long key) {
    const int lane = threadIdx.x & 31;
    int64_t lo = 0, hi = n;                 // answer in [lo, hi]
    while (hi - lo > 32) {
        const int64_t span = hi - lo;
        const int64_t p = lo + (span * (lane + 1)) / 33;
        const unsigned long long x = a[p];
        const int c = __popc(__ballot_sync(0xffffffffu, GE ? x >= key : x > key));
        const int64_t nlo = c == 0 ? lo : lo + (span * c) / 33 + 1;
        const int64_t nhi = c == 32 ? hi : lo + (span * (c + 1)) / 33;
        lo = nlo;
        hi = nhi;
    }
    bool in = false;
    if (lane < hi - lo) {
        const unsigned long long x = a[lo + lane];
        in = GE ? x >= key : x > key;
    }
    return lo + __popc(__ballot_sync(0xffffffffu, in));
}

__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Early rounds (t <= kTab seeds, encoded labels, one rank): the components
// covered so far are listed per lane in the seed table -- tab[i][r] = (label,
// size) of the component seed i newly covered in lane r, or (NONE, 0) -- so
// a candidate's fresh gain is its initial gain minus the sizes of its listed
// components: one row read per candidate, no root-cell or covered-bitmap
// gathers (C4's round 1 refreshes 2.3 M candidates after the hub seed).
__device__ __forceinline__ unsigned long long tab_covered(const uint32_t *__restrict__ L, const Lay &ld,
                                                          const int2 *__restrict__ tab, int64_t tld, int ntab,
                                                          int32_t ns, int64_t u, int q) {
    const uint4 l4 = row_quad(L, ld, u, q);
    const uint32_t lv[4] = {l4.x, l4.y, l4.z, l4.w};
    unsigned long long acc = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int r = (q << 2) + j;
        if (r >= ns) continue;
        const uint32_t lab = is_root(lv[j]) ? (uint32_t)u : lv[j];
        for (int i = 0; i < ntab; ++i) {
            const int2 e = __ldg(tab + i * tld + r);
            if ((uint32_t)e.x == lab) acc += (uint32_t)e.y;
        }
    }
    return acc;
}

// marginal gain of u (u < 0: none) by a group of gsz threads (tid in the
// group); per-warp partial sums meet in the group's shared accumulator.
// Every thread of the CTA must call it (it has a CTA barrier).
template <bool ENC>
__device__ __forceinline__ int64_t group_eval(const uint32_t *__restrict__ L, const uint32_t *__restrict__ C,
                                              const uint32_t *__restrict__ cov, Lay ld, int32_t ns,
                                              int32_t cw, int64_t u, int tid, int gsz,
                                              unsigned long long *acc_sh, const int2 *__restrict__ tab = nullptr,
                                              int64_t tld = 0, int ntab = 0) {
    unsigned long long acc = 0;
    if (u >= 0 && tab) {
        const int nqs = (ns + 3) >> 2;
        for (int q = tid; q < nqs; q += gsz) acc += tab_covered(L, ld, tab, tld, ntab, ns, u, q);
    } else if (u >= 0) {
        const int nqs = (ns + 3) >> 2;
        const uint32_t *rowbase = L;   // quads via ld.off (rows or lane tiles)
        for (int q = tid; q < nqs; q += gsz) {
            const uint4 l4 = row_quad(rowbase, ld, u, q);
            const uint32_t lv[4] = {l4.x, l4.y, l4.z, l4.w};
            uint32_t wd[4], sz[4];
            const int r = q << 2;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const bool in = r + j < ns;
                uint32_t lab = 0;
                sz[j] = in ? cell_size<ENC>(L, C, ld, (uint32_t)u, lv[j], r + j, lab) : 0u;
                wd[j] = in ? cov[(int64_t)lab * cw + ((r + j) >> 5)] : 0xffffffffu;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (!((wd[j] >> ((r + j) & 31)) & 1u)) acc += sz[j];
        }
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(acc_sh, acc);
    __syncthreads();
    return (int64_t)*acc_sh;
}

#ifndef IMX_CELF_STEP_PER_CTA
#define IMX_CELF_STEP_PER_CTA 256
#endif
constexpr int64_t kStepPerCta = IMX_CELF_STEP_PER_CTA;
#ifndef IMX_CELF_FIRST_CAP
#define IMX_CELF_FIRST_CAP 16384
#endif
constexpr int64_t kFirstBatchCap = IMX_CELF_FIRST_CAP;
#ifndef IMX_CELF_WIDE_OUT
#define IMX_CELF_WIDE_OUT 64
#endif
constexpr int64_t kWideOutPerCta = IMX_CELF_WIDE_OUT;   // seed-table batches above this many candidates per CTA leave the kernel

template <bool ENC, bool XM>
#ifndef IMX_CELF_MINB
#define IMX_CELF_MINB 4
#endif
__global__ void __launch_bounds__(256, IMX_CELF_MINB) k_celf_rounds(
    int32_t k, int vb, const uint32_t *__restrict__ L, const uint32_t *__restrict__ C, uint32_t *__restrict__ cov,
    Lay ld, int32_t ns, int32_t cw, int64_t *__restrict__ per_sim, uint8_t *__restrict__ inS,
    int32_t *oid0, int32_t *oid1, unsigned long long *okey0, unsigned long long *okey1,
    int64_t *__restrict__ fresh,
    unsigned long long *__restrict__ skey, int32_t *__restrict__ sid,
    int64_t *__restrict__ trace, int64_t trace_cap, int32_t *__restrict__ seeds,
    int64_t *__restrict__ sgains, unsigned long long *__restrict__ gain, CelfDev *__restrict__ st,
    int32_t bpct, int32_t ngroup, int64_t *__restrict__ xbuf, int64_t xcap, int2 *__restrict__ tab,
    int64_t tab_ld, const int64_t *__restrict__ gains0, int64_t wide_out, const int64_t *__restrict__ g1,
    const unsigned long long *__restrict__ hub) {
    cg::grid_group grid = cg::this_grid();
    constexpr bool xm = XM;                    // exchange mode (sharded run; xcap > 0)
    // a stop that waits for the host (done, trace full, error, big round)
    if (xm && st->status != 0 && st->status != 5) return;
    __shared__ unsigned long long sback[kSmemBack];
    __shared__ unsigned long long gacc[8];
    if (threadIdx.x < 8) gacc[threadIdx.x] = 0;
    __syncthreads();
    const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t gthreads = (int64_t)gridDim.x * blockDim.x;
    const uint32_t vmask = (vb >= 32) ? 0xffffffffu : ((1u << vb) - 1u);
    int64_t ostart = st->ostart, olen = st->olen, T = st->trace_len, batch0 = st->batch0;
    int ocur = st->ocur;
    int32_t t = st->t;
    int32_t status = 0;
    int32_t sstep = 0;                          // evaluation steps so far (uniform)
    const bool prof = gtid == 0;
    __shared__ unsigned long long pf[10];       // phase clock of block 0 (IMX_CELF_PROFILE)
    if (threadIdx.x < 10) pf[threadIdx.x] = 0;
    __syncthreads();
    unsigned long long tp = prof ? gtimer() : 0, ts = 0;
#define PROF_MARK(i)                                 \
    if (prof) {                                      \
        const unsigned long long _t = gtimer();      \
        pf[i] += _t - tp;                            \
        tp = _t;                                     \
    }
    while (t < k) {
        int32_t *oid = ocur ? oid1 : oid0;
        unsigned long long *okey = ocur ? okey1 : okey0;
        if (olen == 0) { status = 3; break; }
        // the previous round's gain was read by every block before its last barrier
        if (gtid == 0 && (t > st->t || (xm && t > 0))) *gain = 0;
        unsigned long long bestkey;
        int64_t kr;
        if (t == 0) {
            bestkey = okey[ostart];        // fresh_at == len(S) == 0: the first pop commits
            kr = 1;
        } else {
            int64_t lo = 0, hi = olen < batch0 ? olen : batch0;
            bestkey = 0;
            bool resume = false;
            if (xm && st->xphase == 1) {       // the exchanged batch of the paused launch
                lo = st->xlo;
                hi = st->xhi;
                bestkey = st->xbest;
                resume = true;
            } else if (xm && hi - lo > xcap) {
                hi = lo + xcap;
            }
            for (;;) {
                if (prof) ts = gtimer();
                unsigned long long m;
                if (resume) {
                    // the sums over the ranks: into fresh[lo, hi), their max key
                    resume = false;
                    unsigned long long lmax = 0;
                    for (int64_t i = lo + gtid; i < hi; i += gthreads) {
                        const int64_t f = xbuf[i - lo];
                        fresh[i] = f;
                        const unsigned long long fk = ((unsigned long long)f << vb) |
                                                      (unsigned long long)(vmask - (uint32_t)oid[ostart + i]);
                        lmax = fk > lmax ? fk : lmax;
                    }
                    for (int o = 16; o; o >>= 1) {
                        const unsigned long long y = __shfl_xor_sync(0xffffffffu, lmax, o);
                        lmax = y > lmax ? y : lmax;
                    }
                    if ((threadIdx.x & 31) == 0 && lmax) atomicMax(&st->smax[3], lmax);
                    bool bad = false;
                    if (st->xpend && xbuf[xcap] != st->xpend_want) bad = true;   // commit self-check
                    grid.sync();
                    m = ld_relaxed64(&st->smax[3]);
                    if (bad) {
                        if (gtid == 0) { st->bad_v = st->xpend_v; st->bad_want = st->xpend_want; st->bad_got = xbuf[xcap]; }
                        status = 3;
                        break;
                    }
                    grid.sync();                 // every block read smax[3] and xpend
                    if (gtid == 0) { st->smax[3] = 0; st->xpend = 0; st->xphase = 0; }
                } else {
                // slot (sstep+2)&3 was last read before the previous barrier
                if (gtid == 0) st->smax[(sstep + 2) & 3] = 0;
                // slot (sstep+2)&3 was last read before the previous barrier
                if (gtid == 0) st->smax[(sstep + 2) & 3] = 0;
                // huge batches (a round that refreshes most vertices): throughput
                // over latency -- a warp per candidate, per-warp max folded once
                const bool wide = hi - lo > (int64_t)gridDim.x * 8 && ns <= 4096;
                // the seed table instead of the covered bitmap (tab != NULL only for ENC, one rank)
                const int ntab = (tab && t <= kTab) ? t : 0;
                const int2 *etab = ntab ? tab : nullptr;
                // round 1 after the speculated first seed (memo.cu: the max-degree
                // vertex): the memo pass left every vertex's exact gain after that
                // seed in g1 -- one word per candidate, no row read
                const bool spec1 = !xm && g1 && ntab == 1 &&
                                   (unsigned long long)(uint32_t)(*(volatile int32_t *)seeds) == *hub;
                if (spec1) {
                    unsigned long long lmax = 0;
                    for (int64_t i = lo + gtid; i < hi; i += gthreads) {
                        const uint32_t u = (uint32_t)oid[ostart + i];
                        const int64_t f = g1[u];
                        fresh[i] = f;
                        const unsigned long long fk = ((unsigned long long)f << vb) | (unsigned long long)(vmask - u);
                        lmax = fk > lmax ? fk : lmax;
                    }
                    for (int o = 16; o; o >>= 1) {
                        const unsigned long long x = __shfl_xor_sync(0xffffffffu, lmax, o);
                        lmax = x > lmax ? x : lmax;
                    }
                    if ((threadIdx.x & 31) == 0 && lmax) atomicMax(&st->smax[sstep & 3], lmax);
                }
                // a huge batch through the seed table (C4's round 1 evaluates 2.4 M
                // candidates) is a streaming pass over rows: k_wide_tab_round does
                // it with the registers this kernel does not have
                if (!spec1 && !xm && etab && hi - lo > (int64_t)gridDim.x * wide_out) {
                    if (gtid == 0) { st->xlo = lo; st->xhi = hi; st->xbest = bestkey; }
                    status = 6;
                    break;
                }
                if (spec1) {
                } else if (wide && etab) {
                    unsigned long long wmax = 0;
                    const int wl = threadIdx.x & 31;
                    const int nqs = (ns + 3) >> 2;
                    for (int64_t i = lo + (gtid >> 5); i < hi; i += gthreads >> 5) {
                        const int64_t u = oid[ostart + i];
                        unsigned long long cov_sz = 0;
                        for (int q = wl; q < nqs; q += 32) cov_sz += tab_covered(L, ld, etab, tab_ld, ntab, ns, u, q);
                        for (int o = 16; o; o >>= 1) cov_sz += __shfl_xor_sync(0xffffffffu, cov_sz, o);
                        const unsigned long long acc = (unsigned long long)gains0[u] - cov_sz;
                        if (wl == 0) fresh[i] = (int64_t)acc;
                        const unsigned long long fk = (acc << vb) | (unsigned long long)(vmask - (uint32_t)u);
                        wmax = fk > wmax ? fk : wmax;
                    }
                    if (wl == 0 && wmax) atomicMax(&st->smax[sstep & 3], wmax);
                } else if (wide) {
                    unsigned long long wmax = 0;
                    const int wl = threadIdx.x & 31;
                    for (int64_t i = lo + (gtid >> 5); i < hi; i += gthreads >> 5) {
                        const int64_t u = oid[ostart + i];
                        const int nqs = (ns + 3) >> 2;
                        const uint32_t *rowbase = L;   // quads via ld.off (rows or lane tiles)
                        unsigned long long acc = 0;
                        for (int q = wl; q < nqs; q += 32) {
                            const uint4 l4 = row_quad(rowbase, ld, u, q);
                            const uint32_t lv[4] = {l4.x, l4.y, l4.z, l4.w};
                            uint32_t wd[4], sz[4];
                            const int r = q << 2;
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                const bool in = r + j < ns;
                                uint32_t lab = 0;
                                sz[j] = in ? cell_size<ENC>(L, C, ld, (uint32_t)u, lv[j], r + j, lab) : 0u;
                                wd[j] = in ? cov[(int64_t)lab * cw + ((r + j) >> 5)] : 0xffffffffu;
                            }
#pragma unroll
                            for (int j = 0; j < 4; ++j)
                                if (!((wd[j] >> ((r + j) & 31)) & 1u)) acc += sz[j];
                        }
                        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                        if (wl == 0) {
                            if (xm) xbuf[i - lo] = (int64_t)acc;
                            else fresh[i] = (int64_t)acc;
                        }
                        const unsigned long long fk = (acc << vb) | (unsigned long long)(vmask - (uint32_t)u);
                        wmax = fk > wmax ? fk : wmax;
                    }
                    if (!xm && wl == 0 && wmax) atomicMax(&st->smax[sstep & 3], wmax);
                }
                // otherwise ngroup candidates per CTA at a time, 256/ngroup threads each
                for (int64_t base = lo + (int64_t)blockIdx.x * ngroup; !wide && !spec1 && base < hi;
                     base += (int64_t)gridDim.x * ngroup) {
                    const int gsz = blockDim.x / ngroup, g = threadIdx.x / gsz;
                    const int64_t i = base + g;
                    const int64_t ui = i < hi ? (int64_t)oid[ostart + i] : -1;
                    int64_t f = group_eval<ENC>(L, C, cov, ld, ns, cw, ui, threadIdx.x - g * gsz, gsz, gacc + g,
                                                etab, tab_ld, ntab);
                    if (etab && ui >= 0) f = gains0[ui] - f;
                    if (threadIdx.x == g * gsz && i < hi) {
                        if (xm) {
                            xbuf[i - lo] = f;
                        } else {
                            fresh[i] = f;
                            atomicMax(&st->smax[sstep & 3], ((unsigned long long)f << vb) |
                                                            (unsigned long long)(vmask - (uint32_t)oid[ostart + i]));
                        }
                    }
                    __syncthreads();
                    if (threadIdx.x < ngroup) gacc[threadIdx.x] = 0;
                    __syncthreads();
                }
                if (xm) {
                    // pause: the host sums the partials over the ranks, relaunches
                    if (gtid == 0) {
                        st->xphase = 1; st->xlo = lo; st->xhi = hi; st->xbest = bestkey;
                        xbuf[xcap] = st->xpend ? st->xpend_got : 0;
                    }
                    status = 5;
                    break;
                }
                if (prof) { const unsigned long long x = gtimer(); pf[6] += x - ts; ts = x; }
                grid.sync();
                if (prof) { const unsigned long long x = gtimer(); pf[7] += x - ts; ts = x; pf[4]++; pf[5] += hi - lo; }
                m = ld_relaxed64(&st->smax[sstep & 3]);
                }
                ++sstep;
                bestkey = m > bestkey ? m : bestkey;
                const bool stop = hi >= olen || bestkey >= okey[ostart + hi];   // nothing unevaluated can win
                if (prof) pf[8] += gtimer() - ts;
                if (stop) break;
                lo = hi;
                // doubling batches, but at most ~256 candidates per CTA per
                // step: a round that refreshes millions of vertices (C4's
                // round 1 after the hub) would otherwise evaluate up to twice
                // its refreshed prefix in the last doubling
                int64_t step = batch0 > hi ? batch0 : hi;
                int64_t cap = (int64_t)gridDim.x * kStepPerCta;
                if (xm && cap > xcap) cap = xcap;          // a batch fits the exchange buffer
                if (step > cap) step = cap;
                hi = (olen - hi < step) ? olen : hi + step;
            }
            if (status) break;                            // paused for an exchange, or a failed check
            // refreshed prefix: stale key >= best fresh key (keys sorted descending)
            kr = warp_count_above<true>(okey + ostart, hi, bestkey);
        }
        PROF_MARK(0);
        const int32_t best_v = (int32_t)(vmask - (uint32_t)(bestkey & vmask));
        const int64_t best_f = (int64_t)(bestkey >> vb);
        const int64_t nrec = (t == 0 ? 0 : kr) + 1;
        if (T + nrec > trace_cap || kr > kMaxRank) {
            if (gtid == 0) { st->big_key = bestkey; st->big_kr = kr; }
            status = T + nrec > trace_cap ? 2 : 4;        // 2: host drains the trace and relaunches
            break;                                        // (or finishes an oversized round)
        }
        // phase 1: trace records; the refreshed vertices ranked by their fresh
        // keys (fresh[] / order ids of the evaluated prefix are complete since
        // the last evaluation barrier) and scattered sorted; commit
        const int64_t nback = t == 0 ? 0 : kr - 1;       // the winner is not re-inserted
        const int lane = threadIdx.x & 31;
        if (t > 0) {
            for (int64_t i = gtid; i < kr; i += gthreads) {
                const int32_t v = oid[ostart + i];
                const int64_t f = fresh[i];
                int64_t *rec = trace + 5 * (T + i);
                rec[0] = v; rec[1] = (int64_t)(okey[ostart + i] >> vb); rec[2] = f; rec[3] = 0; rec[4] = t;
            }
            // one warp per refreshed key; its rank = #fresh keys above it minus
            // the winner's (the unique maximum)
            for (int64_t j = gtid >> 5; j < kr; j += gthreads >> 5) {
                const int32_t vj = oid[ostart + j];
                if (vj == best_v) continue;
                const unsigned long long kj = ((unsigned long long)fresh[j] << vb) |
                                              (unsigned long long)(vmask - (uint32_t)vj);
                int64_t rk = 0;
                for (int64_t i = lane; i < kr; i += 32) {
                    const unsigned long long ki = ((unsigned long long)fresh[i] << vb) |
                                                  (unsigned long long)(vmask - (uint32_t)oid[ostart + i]);
                    rk += ki > kj;
                }
                for (int o = 16; o; o >>= 1) rk += __shfl_xor_sync(0xffffffffu, rk, o);
                rk -= 1;
                if (lane == 0) { skey[rk] = kj; sid[rk] = vj; }
            }
        }
        if (gtid == 0) {
            int64_t *rec = trace + 5 * (T + nrec - 1);
            rec[0] = best_v; rec[1] = best_f; rec[2] = best_f; rec[3] = 1; rec[4] = t;
            seeds[t] = best_v;
            sgains[t] = best_f;
            inS[best_v] = 1;
        }
        {
            unsigned long long acc = 0;
            for (int64_t r = gtid; r < ns; r += gthreads) {
                uint32_t lab;
                const uint32_t sz = cell_size<ENC>(L, C, ld, (uint32_t)best_v, L[cell_off(ld, best_v, r)], (int)r, lab);
                const uint32_t bit = 1u << (r & 31);
                const uint32_t old = atomicOr(cov + (int64_t)lab * cw + (r >> 5), bit);
                if (!(old & bit)) { per_sim[r] += sz; acc += sz; }
                if (tab && t < kTab)        // the seed table of the early rounds
                    tab[t * tab_ld + r] = (old & bit) ? make_int2(-1, 0) : make_int2((int)lab, (int)sz);
            }
            for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if ((threadIdx.x & 31) == 0 && acc) atomicAdd(gain, acc);
        }
        grid.sync();
        PROF_MARK(1);
        // phase 2: self-check of the commit, then merge order[kr, olen) with
        // the sorted refreshed vertices (exchange mode: the gain is this
        // rank's part; it is summed with the next batch and checked then)
        const unsigned long long got = *gain;
        if (xm) {
            if (gtid == 0) { st->xpend = 1; st->xpend_v = best_v; st->xpend_want = best_f; st->xpend_got = (int64_t)got; }
        } else if ((int64_t)got != best_f) {
            if (gtid == 0) { st->bad_v = best_v; st->bad_want = best_f; st->bad_got = (int64_t)got; }
            status = 3;
            break;
        }
        if (nback > 0) {
            int32_t *ob = ocur ? oid0 : oid1;
            unsigned long long *okb = ocur ? okey0 : okey1;
            const int64_t na = olen - kr;
            const unsigned long long *ak = okey + ostart + kr;
            const int32_t *ai = oid + ostart + kr;
            // order entries: shift by the refreshed keys above them (binary
            // search in a shared-memory copy of the sorted refreshed keys)
            const bool in_smem = nback <= kSmemBack;
            if (in_smem) {
                for (int64_t i = threadIdx.x; i < nback; i += blockDim.x) sback[i] = skey[i];
                __syncthreads();
            }
            const unsigned long long *sk = in_smem ? sback : skey;
            for (int64_t i = gtid; i < na; i += gthreads) {
                const unsigned long long key = ak[i];
                int64_t lo2 = 0, hi2 = nback;
                while (lo2 < hi2) {
                    const int64_t mid = (lo2 + hi2) >> 1;
                    if (sk[mid] > key) lo2 = mid + 1; else hi2 = mid;
                }
                ob[i + lo2] = ai[i];
                okb[i + lo2] = key;
            }
            // refreshed entries: shift by the order keys above them (warp search)
            for (int64_t j = gtid >> 5; j < nback; j += gthreads >> 5) {
                const unsigned long long key = sk[j];
                const int64_t pos = j + warp_count_above<false>(ak, na, key);
                if (lane == 0) { ob[pos] = sid[j]; okb[pos] = key; }
            }
            ocur ^= 1;
            ostart = 0;
            olen = na + nback;
        } else {
            ostart += kr;
            olen -= kr;
        }
        T += nrec;
        // next round's first batch: 1.5x this round's refreshed prefix, but at
        // most kFirstBatchCap -- one huge round (C4's round 1 refreshes 2.3M
        // vertices after the hub) must not make the next round evaluate
        // millions speculatively (C4: 4.66M -> ~2.5M evaluations)
        if (t > 0) batch0 = kr * bpct / 100 > 64 ? kr * bpct / 100 : 64;
        if (batch0 > kFirstBatchCap) batch0 = kFirstBatchCap;
        ++t;
        grid.sync();
        PROF_MARK(3);
    }
#undef PROF_MARK
    if (gtid == 0) {
        for (int i = 0; i < 10; ++i) st->prof[i] += pf[i];
        st->ostart = ostart; st->olen = olen; st->ocur = ocur; st->t = t;
        st->trace_len = T; st->batch0 = batch0;
        st->status = status ? status : 1;
        // done in exchange mode: the last commit's part goes out with one more exchange
        if (xm && !status) xbuf[xcap] = st->xpend ? st->xpend_got : 0;
    }
}

// tab_covered on a quad already in registers
__device__ __forceinline__ unsigned long long tab_covered_quad(const uint4 l4, const int2 *__restrict__ tab,
                                                               int64_t tld, int ntab, int32_t ns, int64_t u, int q) {
    const uint32_t lv[4] = {l4.x, l4.y, l4.z, l4.w};
    const int r0 = q << 2;
    unsigned long long acc = 0;
    if (r0 + 3 < ns) {
        for (int i = 0; i < ntab; ++i) {
            // four (label, size) entries as two 16-byte loads (tld and r0 are multiples of 4)
            const int4 e01 = __ldg(reinterpret_cast<const int4 *>(tab + i * tld + r0));
            const int4 e23 = __ldg(reinterpret_cast<const int4 *>(tab + i * tld + r0) + 1);
            const uint32_t el[4] = {(uint32_t)e01.x, (uint32_t)e01.z, (uint32_t)e23.x, (uint32_t)e23.z};
            const uint32_t es[4] = {(uint32_t)e01.y, (uint32_t)e01.w, (uint32_t)e23.y, (uint32_t)e23.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t lab = is_root(lv[j]) ? (uint32_t)u : lv[j];
                if (el[j] == lab) acc += es[j];
            }
        }
        return acc;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int r = r0 + j;
        if (r >= ns) continue;
        const uint32_t lab = is_root(lv[j]) ? (uint32_t)u : lv[j];
        for (int i = 0; i < ntab; ++i) {
            const int2 e = __ldg(tab + i * tld + r);
            if ((uint32_t)e.x == lab) acc += (uint32_t)e.y;
        }
    }
    return acc;
}

// A huge evaluation through the seed table (status 6 of k_celf_rounds: C4's
// round 1 refreshes 2.3 M candidates after the hub seed) as a streaming pass
// over the candidates' rows: fresh = initial gain - sizes of the listed
// components, one 4 KB row read per candidate and nothing else.  The same
// batch loop and stop rule as the persistent kernel (it continues that
// kernel's round from [xlo, xhi) with the best key so far), but a warp per
// candidate, its row staged in shared memory by cp.async one row ahead of the
// compares (no registers held by the loads in flight), candidates handed
// out kWideGrab at a time from a counter (with a static split the slowest of
// the warps held every step's barrier for ~40% of the step).  Ends with the
// round's best key and refreshed prefix length in big_key / big_kr (status
// 2): the host finishes the round with celf_big_round.
constexpr int kWideGrab = 16;           // candidates per counter grab
constexpr int kWideRowQuads = 256;      // quads per staged row segment (4 KB)
constexpr int kWideSmem = 8 * 2 * kWideRowQuads * (int)sizeof(uint4);   // 8 warps, double-buffered

__device__ __forceinline__ void cp_async16(void *smem, const void *gptr) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gptr) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// TAB1 (one listed seed, rows of <= 1024 lanes: C4's round 1): every thread
// keeps the table entries of its 32 cells in registers for the whole launch
// -- the compares then cost shared-memory reads only (with the entries read
// through L1, two 16-byte loads per quad, the L1 pipe bound the pass at 4 TB/s).
template <bool TAB1>
__global__ void __launch_bounds__(256, TAB1 ? 2 : 3) k_wide_tab_round(
    const uint32_t *__restrict__ L, Lay ld, int32_t ns, const int2 *__restrict__ tab, int64_t tab_ld, int ntab,
    const int64_t *__restrict__ gains0, const int32_t *__restrict__ cand, const unsigned long long *__restrict__ keys,
    int64_t olen, int64_t *__restrict__ fresh, int vb, CelfDev *__restrict__ st, int64_t batch0, int64_t cap) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ uint4 wide_rows[];
    const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const uint32_t vmask = (vb >= 32) ? 0xffffffffu : ((1u << vb) - 1u);
    const int wl = threadIdx.x & 31;
    const int nqs = (ns + 3) >> 2;
    const int nseg = (nqs + kWideRowQuads - 1) / kWideRowQuads;     // ns <= 1024: one
    uint4 *wbuf = wide_rows + (threadIdx.x >> 5) * 2 * kWideRowQuads;
    int64_t lo = st->xlo, hi = st->xhi;
    unsigned long long bestkey = st->xbest;
    unsigned long long evals = 0, steps = 0;
    uint32_t tl[TAB1 ? 32 : 1], tz[TAB1 ? 32 : 1];
    if (TAB1) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int q = wl + 32 * j;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int r = 4 * q + c;
                const int2 e = r < ns ? __ldg(tab + r) : make_int2(-1, 0);    // label -1 matches nothing
                tl[4 * j + c] = (uint32_t)e.x;
                tz[4 * j + c] = (uint32_t)e.y;
            }
        }
    }
    for (int s = 0;; ++s) {
        // slot (s+2)&3 was last used two barriers ago
        if (gtid == 0) { st->smax[(s + 2) & 3] = 0; st->wctr[(s + 2) & 3] = 0; }
        unsigned long long wmax = 0;
        for (;;) {
            unsigned long long b0 = 0;
            if (wl == 0) b0 = atomicAdd(&st->wctr[s & 3], (unsigned long long)kWideGrab);
            const int64_t ib = lo + (int64_t)__shfl_sync(0xffffffffu, b0, 0);
            if (ib >= hi) break;
            const int gcnt = (int)(hi - ib < kWideGrab ? hi - ib : kWideGrab);
            const int32_t uw = wl < gcnt ? cand[ib + wl] : 0;
            // unit j of the grab = segment j % nseg of candidate j / nseg; unit j + 1 is
            // copied into the other buffer while unit j is compared
            const int units = gcnt * nseg;
            auto issue = [&](int j) {
                const int64_t u = __shfl_sync(0xffffffffu, uw, j / nseg);
                const int qs = (j % nseg) * kWideRowQuads;
                const int qe = nqs - qs < kWideRowQuads ? nqs - qs : kWideRowQuads;
                uint4 *dst = wbuf + (j & 1) * kWideRowQuads;
                for (int q = wl; q < qe; q += 32) cp_async16(dst + q, L + cell_off(ld, u, (qs + q) << 2));
                cp_async_commit();
            };
            issue(0);
            const long long gw = wl < gcnt ? gains0[uw] : 0;
            unsigned long long cov_sz = 0;
            for (int j = 0; j < units; ++j) {
                if (j + 1 < units) {
                    issue(j + 1);
                    cp_async_wait<1>();
                } else {
                    cp_async_wait<0>();
                }
                __syncwarp();
                const int k2 = j / nseg;
                const int64_t u = __shfl_sync(0xffffffffu, uw, k2);
                const int qs = (j % nseg) * kWideRowQuads;
                const int qe = nqs - qs < kWideRowQuads ? nqs - qs : kWideRowQuads;
                const uint4 *src = wbuf + (j & 1) * kWideRowQuads;
                if (TAB1) {
#pragma unroll
                    for (int j2 = 0; j2 < 8; ++j2) {
                        if (wl + 32 * j2 < qe) {
                            const uint4 l4 = src[wl + 32 * j2];
                            const uint32_t lv[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                const uint32_t lab = is_root(lv[c]) ? (uint32_t)u : lv[c];
                                if (tl[4 * j2 + c] == lab) cov_sz += tz[4 * j2 + c];
                            }
                        }
                    }
                } else {
                    for (int q = wl; q < qe; q += 32)
                        cov_sz += tab_covered_quad(src[q], tab, tab_ld, ntab, ns, u, qs + q);
                }
                __syncwarp();                      // the buffer is refilled two units later
                if (j % nseg == nseg - 1) {
                    for (int o = 16; o; o >>= 1) cov_sz += __shfl_xor_sync(0xffffffffu, cov_sz, o);
                    const unsigned long long acc = (unsigned long long)__shfl_sync(0xffffffffu, gw, k2) - cov_sz;
                    if (wl == 0) fresh[ib + k2] = (int64_t)acc;
                    const unsigned long long fk = (acc << vb) | (unsigned long long)(vmask - (uint32_t)u);
                    wmax = fk > wmax ? fk : wmax;
                    cov_sz = 0;
                }
            }
        }
        if (wl == 0 && wmax) atomicMax(&st->smax[s & 3], wmax);
        grid.sync();
        const unsigned long long m = ld_relaxed64(&st->smax[s & 3]);
        bestkey = m > bestkey ? m : bestkey;
        evals += hi - lo;
        ++steps;
        if (hi >= olen || bestkey >= keys[hi]) break;            // nothing unevaluated can win
        lo = hi;
        int64_t step = batch0 > hi ? batch0 : hi;
        if (step > cap) step = cap;
        hi = (olen - hi < step) ? olen : hi + step;
    }
    // refreshed prefix: stale key >= best fresh key (keys sorted descending)
    const int64_t kr = warp_count_above<true>(keys, hi, bestkey);
    if (gtid == 0) {
        st->big_key = bestkey;
        st->big_kr = kr;
        st->status = 2;
        st->prof[4] += steps;
        st->prof[5] += evals;
    }
}

static inline bool key_le(int64_t pa, int32_t va, int64_t pb, int32_t vb) {
    // (-pa, va) <= (-pb, vb)
    return pa > pb || (pa == pb && va <= vb);
}

}  // namespace imx

using namespace imx;

// caller priorities below the memoized gains: the round-based CELF needs
// every stale priority to bound its vertex's fresh gain
__global__ void k_check_prio(const int64_t *__restrict__ prio, const int64_t *__restrict__ gains, int64_t n,
                             unsigned long long *__restrict__ bad) {
    unsigned long long b = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        b += prio[v] < gains[v];
    for (int o = 16; o; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(bad, b);
}

extern "C" int imx_celf_reset(imx_ctx *c, const int64_t *prio) {
    CTX_CHECK(c);
    if (!c->labels_ready) { set_error("labels not computed"); return IMX_EINVAL; }
    IMX_TRY(ensure_celf_buffers(c));
    const int64_t n = c->g->n;
    int64_t *dprio = c->gains;
    if (prio) {
        IMX_CUDA(cudaMemcpyAsync(c->eval_out, prio, sizeof(int64_t) * n, cudaMemcpyHostToDevice, c->st));
        dprio = c->eval_out;
    } else if (!c->memo_ready) {
        set_error("gains not computed (call imx_memoize first)");
        return IMX_EINVAL;
    }
    unsigned long long *maxp = c->scratch + 9;
    IMX_CUDA(cudaMemsetAsync(maxp, 0, sizeof(unsigned long long), c->st));
    if (prio && c->memo_ready && n) {
        // the round-based CELF (and its kernel) assume prio >= the fresh
        // gains; with the memo at hand, refuse caller priorities that are not
        unsigned long long *bad = c->scratch + 13, nb = 0;
        IMX_CUDA(cudaMemsetAsync(bad, 0, sizeof(unsigned long long), c->st));
        k_check_prio<<<grid_for(n), 256, 0, c->st>>>(dprio, c->gains, n, bad);
        IMX_CHECK_LAUNCH();
        count_launch(c);
        IMX_CUDA(cudaMemcpyAsync(&nb, bad, sizeof nb, cudaMemcpyDeviceToHost, c->st));
        IMX_CUDA(cudaStreamSynchronize(c->st));
        if (nb) {
            set_error("CELF priorities below the memoized gains for %llu vertices (they must be upper bounds)", nb);
            return IMX_EINVAL;
        }
    }
    if (n) {
        k_pack_keys<<<grid_for(n), 256, 0, c->st>>>(dprio, n, c->vb, c->oid[1], c->okey[1], maxp);
        IMX_CHECK_LAUNCH();
        count_launch(c);
    }
    unsigned long long mp = 0;
    IMX_CUDA(cudaMemcpyAsync(&mp, maxp, sizeof mp, cudaMemcpyDeviceToHost, c->st));
    IMX_CUDA(cudaStreamSynchronize(c->st));
    int pbits = 0;
    while (pbits < 64 && (mp >> pbits)) ++pbits;
    if (pbits + c->vb > 64) {
        set_error("gains need %d bits and vertex ids %d: packed CELF keys exceed 64 bits", pbits, c->vb);
        return IMX_ECONSTRAINT;
    }
    if (n) {
        const int end_bit = std::max(1, pbits + c->vb);
        size_t tb = 0;
        IMX_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, c->okey[1], c->okey[0], c->oid[1], c->oid[0],
                                                           n, 0, end_bit, c->st));
        if (tb > c->sort_tmp_bytes) {
            if (c->sort_tmp) cudaFreeAsync(c->sort_tmp, c->st);
            c->sort_tmp = nullptr;
            c->sort_tmp_bytes = 0;
            IMX_CUDA(pool_alloc(&c->sort_tmp, tb, c->st));
            c->sort_tmp_bytes = tb;
        }
        IMX_CUDA(cub::DeviceRadixSort::SortPairsDescending(c->sort_tmp, tb, c->okey[1], c->okey[0], c->oid[1],
                                                           c->oid[0], n, 0, end_bit, c->st));
        IMX_CUDA(cudaMemsetAsync(c->inS, 0, n, c->st));
        IMX_CUDA(cudaMemsetAsync(c->cov, 0, sizeof(uint32_t) * (size_t)n * c->cw, c->st));
    }
    IMX_CUDA(cudaMemsetAsync(c->per_sim, 0, sizeof(int64_t) * (c->W + 1), c->st));
    IMX_CUDA(cudaStreamSynchronize(c->st));
    c->ocur = 0;
    c->ostart = 0;
    c->olen = n;
    c->celf_ready = true;
    c->trace_n = 0;
    return IMX_OK;
}

extern "C" int imx_celf_top(imx_ctx *c, int64_t *prio_out, int32_t *v_out) {
    CELF_CHECK(c);
    IMX_TRY(spec_guard(c));
    if (!prio_out || !v_out) { set_error("NULL argument"); return IMX_EINVAL; }
    if (c->olen == 0) { *v_out = -1; *prio_out = 0; return IMX_OK; }
    int32_t id;
    unsigned long long key;
    IMX_CUDA(cudaMemcpyAsync(&id, c->oid[c->ocur] + c->ostart, sizeof id, cudaMemcpyDeviceToHost, c->st));
    IMX_CUDA(cudaMemcpyAsync(&key, c->okey[c->ocur] + c->ostart, sizeof key, cudaMemcpyDeviceToHost, c->st));
    IMX_CUDA(cudaStreamSynchronize(c->st));
    *v_out = id;
    *prio_out = key_prio(c, key);
    return IMX_OK;
}

extern "C" int imx_celf_prefix(imx_ctx *c, int64_t lo, int64_t hi, int32_t *ids_out, int64_t *prio_out,
                               int64_t *fresh_out, int64_t *len_out) {
    CELF_CHECK(c);
    IMX_TRY(spec_guard(c));
    if (lo < 0 || hi < lo) { set_error("prefix range [%lld, %lld) invalid", (long long)lo, (long long)hi); return IMX_EINVAL; }
    if (len_out) *len_out = c->olen;
    hi = std::min(hi, c->olen);
    if (lo >= hi) return IMX_OK;
    const int64_t fetch = std::min(hi + 1, c->olen) - lo;
    std::vector<unsigned long long> keys(fetch);
    std::vector<int32_t> ids(fetch);
    std::vector<int64_t> fr(hi - lo);
    IMX_TRY(celf_prefix(c, lo, hi, ids.data(), keys.data(), fr.data()));
    if (ids_out) std::copy(ids.begin(), ids.end(), ids_out);
    if (prio_out) for (int64_t i = 0; i < fetch; ++i) prio_out[i] = key_prio(c, keys[i]);
    if (fresh_out) std::copy(fr.begin(), fr.end(), fresh_out);
    return IMX_OK;
}

extern "C" int imx_celf_advance(imx_ctx *c, int64_t k, int32_t u, const int32_t *ids, const int64_t *prio,
                                int64_t cnt, int64_t *gain_out) {
    CELF_CHECK(c);
    IMX_TRY(spec_guard(c));
    if (k < 0 || cnt < 0 || (cnt && (!ids || !prio))) { set_error("bad arguments"); return IMX_EINVAL; }
    if (u < 0 || u >= c->g->n) { set_error("vertex %d outside vertex range", u); return IMX_EINVAL; }
    std::vector<unsigned long long> keys(cnt);
    for (int64_t i = 0; i < cnt; ++i) keys[i] = host_key(c, prio[i], ids[i]);
    for (int64_t i = 1; i < cnt; ++i)
        if (keys[i] >= keys[i - 1]) { set_error("re-inserted vertices must be sorted by (-prio, id)"); return IMX_EINVAL; }
    unsigned long long *sc = c->scratch + 7;
    IMX_CUDA(cudaMemsetAsync(sc, 0, sizeof(unsigned long long), c->st));
    launch_commit(c, u, sc);
    IMX_CHECK_LAUNCH();
    count_launch(c);
    IMX_TRY(celf_advance(c, k, ids, keys.data(), cnt));
    unsigned long long g = 0;
    IMX_CUDA(cudaMemcpyAsync(&g, sc, sizeof g, cudaMemcpyDeviceToHost, c->st));
    IMX_CUDA(cudaStreamSynchronize(c->st));
    if (gain_out) *gain_out = (int64_t)g;
    return IMX_OK;
}

extern "C" int imx_eval_gains(imx_ctx *c, const int32_t *cand, int64_t cnt, int64_t *out) {
    CELF_CHECK(c);
    IMX_TRY(spec_guard(c));
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

extern "C" int imx_commit(imx_ctx *c, int32_t u, int64_t *gain_out) {
    CELF_CHECK(c);
    IMX_TRY(spec_guard(c));
    if (u < 0 || u >= c->g->n) { set_error("vertex %d outside vertex range", u); return IMX_EINVAL; }
    uint8_t in = 0;
    IMX_CUDA(cudaMemcpyAsync(&in, c->inS + u, 1, cudaMemcpyDeviceToHost, c->st));
    IMX_CUDA(cudaStreamSynchronize(c->st));
    if (in) { set_error("vertex %d committed twice", u); return IMX_EINTERNAL; }
    unsigned long long *sc = c->scratch + 7;
    IMX_CUDA(cudaMemsetAsync(sc, 0, sizeof(unsigned long long), c->st));
    launch_commit(c, u, sc);
    IMX_CHECK_LAUNCH();
    count_launch(c);
    unsigned long long g = 0;
    IMX_CUDA(cudaMemcpyAsync(&g, sc, sizeof g, cudaMemcpyDeviceToHost, c->st));
    IMX_CUDA(cudaStreamSynchronize(c->st));
    if (gain_out) *gain_out = (int64_t)g;
    return IMX_OK;
}

// One round on the host-driven path (prefix batches + advance), synchronous.
// Sharded rounds (imx_celf_select_sharded): every evaluated batch's partial
// gains are summed over the ranks by the caller's allreduce before any
// decision, so all ranks take identical ones; the previous round's commit
// self-check rides along as one extra element of the next batch.
struct ShardReduce {
    imx_allreduce_fn fn = nullptr;    // host callback, or
    imx_comm *comm = nullptr;         // the device data plane (comm.cu)
    void *user = nullptr;
    bool pending = false;           // a commit gain waits for its check
    int64_t pending_got = 0, pending_want = 0;
    int32_t pending_v = -1;
    std::vector<int64_t> buf;
};

static int shard_check(const ShardReduce &sr, int64_t total) {
    if (total != sr.pending_want) {
        set_error("CELF self-check: committed gain %lld != evaluated %lld for vertex %d",
                  (long long)total, (long long)sr.pending_want, sr.pending_v);
        return IMX_EINTERNAL;
    }
    return IMX_OK;
}

// allreduce of fr[0, cnt) (+ the pending commit gain) in place
static int shard_reduce(ShardReduce &sr, int64_t *fr, int64_t cnt) {
    sr.buf.assign(fr, fr + cnt);
    if (sr.pending) sr.buf.push_back(sr.pending_got);
    if (sr.fn((int64_t *)sr.buf.data(), (int64_t)sr.buf.size(), sr.user) != 0) {
        set_error("allreduce callback failed");
        return IMX_EINTERNAL;
    }
    std::copy(sr.buf.begin(), sr.buf.begin() + cnt, fr);
    if (sr.pending) {
        IMX_TRY(shard_check(sr, sr.buf[cnt]));
        sr.pending = false;
    }
    return IMX_OK;
}

static int celf_host_round(imx_ctx *c, int32_t t, int64_t &batch0, int32_t *seeds_out, int64_t *gains_out,
                           ShardReduce *sr = nullptr) {
    auto rec = [&](int64_t v, int64_t s, int64_t f, int64_t com) {
        int64_t *o = c->trace + c->trace_n;
        o[0] = v; o[1] = s; o[2] = f; o[3] = com; o[4] = t;
        c->trace_n += 5;
    };
    if (c->olen == 0) { set_error("no candidate left at round %d", t); return IMX_EINTERNAL; }
    std::vector<int32_t> ids;
    std::vector<unsigned long long> keys;
    std::vector<int64_t> fr;
    std::vector<std::pair<unsigned long long, int32_t>> back;
    int64_t best_f = -1, kr = 1;
    int32_t best_v = -1;
    if (t == 0) {
        ids.resize(1);
        keys.resize(1);
        IMX_CUDA(cudaMemcpyAsync(ids.data(), c->oid[c->ocur] + c->ostart, sizeof(int32_t), cudaMemcpyDeviceToHost, c->st));
        IMX_CUDA(cudaMemcpyAsync(keys.data(), c->okey[c->ocur] + c->ostart, sizeof(unsigned long long),
                                 cudaMemcpyDeviceToHost, c->st));
        IMX_CUDA(cudaStreamSynchronize(c->st));
        best_v = ids[0];
        best_f = key_prio(c, keys[0]);
    } else {
        const int64_t len = c->olen;
        int64_t lo = 0, hi = std::min(len, batch0);
        for (;;) {
            if ((int64_t)ids.size() < hi + 1) { ids.resize(hi + 1); keys.resize(hi + 1); fr.resize(hi + 1); }
            if (sr && sr->comm) {
                // partial gains summed on the device, the pending commit check with them
                int64_t pend = sr->pending_got;
                IMX_TRY(celf_prefix(c, lo, hi, ids.data() + lo, keys.data() + lo, fr.data() + lo, sr->comm,
                                    sr->pending ? &pend : nullptr));
                if (sr->pending) {
                    IMX_TRY(shard_check(*sr, pend));
                    sr->pending = false;
                }
            } else {
                IMX_TRY(celf_prefix(c, lo, hi, ids.data() + lo, keys.data() + lo, fr.data() + lo));
                if (sr) IMX_TRY(shard_reduce(*sr, fr.data() + lo, hi - lo));
            }
            for (int64_t i = lo; i < hi; ++i)
                if (best_v < 0 || key_le(fr[i], ids[i], best_f, best_v)) { best_f = fr[i]; best_v = ids[i]; }
            if (hi >= len) break;
            if (key_le(best_f, best_v, key_prio(c, keys[hi]), ids[hi])) break;   // nothing unevaluated can win
            lo = hi;
            hi = std::min(len, hi + std::max<int64_t>(batch0, hi));
        }
        IMX_TRY(trace_reserve(c, c->trace_n + 5 * (hi + 1)));
        kr = 0;
        while (kr < hi && key_le(key_prio(c, keys[kr]), ids[kr], best_f, best_v)) {
            rec(ids[kr], key_prio(c, keys[kr]), fr[kr], 0);
            if (ids[kr] != best_v) back.emplace_back(host_key(c, fr[kr], ids[kr]), ids[kr]);
            ++kr;
        }
        batch0 = std::min<int64_t>(kFirstBatchCap, std::max<int64_t>(64, kr));
    }
    std::sort(back.begin(), back.end(), [](const auto &a, const auto &b) { return a.first > b.first; });
    std::vector<int32_t> bid(back.size());
    std::vector<unsigned long long> bkey(back.size());
    for (size_t i = 0; i < back.size(); ++i) { bkey[i] = back[i].first; bid[i] = back[i].second; }
    unsigned long long *gain = c->scratch + 7;
    IMX_CUDA(cudaMemsetAsync(gain, 0, sizeof(unsigned long long), c->st));
    launch_commit(c, best_v, gain, t);
    IMX_CHECK_LAUNCH();
    count_launch(c);
    IMX_TRY(celf_advance(c, kr, bid.data(), bkey.data(), (int64_t)back.size()));
    unsigned long long got = 0;
    IMX_CUDA(cudaMemcpyAsync(&got, gain, sizeof got, cudaMemcpyDeviceToHost, c->st));
    IMX_CUDA(cudaStreamSynchronize(c->st));
    if (sr) {                       // partial gain: checked after the next allreduce
        sr->pending = true;
        sr->pending_got = (int64_t)got;
        sr->pending_want = best_f;
        sr->pending_v = best_v;
    } else if ((int64_t)got != best_f) {
        set_error("CELF self-check: committed gain %lld != evaluated %lld for vertex %d",
                  (long long)got, (long long)best_f, best_v);
        return IMX_EINTERNAL;
    }
    IMX_TRY(trace_reserve(c, c->trace_n + 5));
    rec(best_v, best_f, best_f, 1);
    if (seeds_out) seeds_out[t] = best_v;
    if (gains_out) gains_out[t] = best_f;
    return IMX_OK;
}

// Persistent-kernel path: launch k_celf_rounds for rounds [t, k); returns
// the kernel's status (1 done, 2 trace full, 4 round too large).
static int celf_device_rounds(imx_ctx *c, int32_t t, int32_t k, int64_t batch0, int32_t *status_out,
                              int32_t *t_out, int64_t *batch0_out, std::vector<int32_t> &seeds,
                              std::vector<int64_t> &gains) {
    const int64_t n = c->g->n;
    if (!c->cdev) {
        IMX_CUDA(pool_alloc((void **)&c->cdev, sizeof(CelfDev), c->st));
        IMX_CUDA(pool_alloc((void **)&c->skey, sizeof(unsigned long long) * kMaxRank, c->st));
        IMX_CUDA(pool_alloc((void **)&c->sid, sizeof(int32_t) * kMaxRank, c->st));
        c->trace_cap = std::max<int64_t>(1 << 16, std::min<int64_t>(4 * n + 4096, 1 << 21));
        if (const char *tc = getenv("IMX_CELF_TRACE_CAP")) c->trace_cap = std::max<int64_t>(8, atoll(tc));
        IMX_CUDA(pool_alloc((void **)&c->dtrace, sizeof(int64_t) * 5 * c->trace_cap, c->st));
    }
    if (!c->dseeds || c->dseeds_cap < k) {
        if (c->dseeds) { cudaFreeAsync(c->dseeds, c->st); cudaFreeAsync(c->dsgains, c->st); }
        IMX_CUDA(pool_alloc((void **)&c->dseeds, sizeof(int32_t) * k, c->st));
        IMX_CUDA(pool_alloc((void **)&c->dsgains, sizeof(int64_t) * k, c->st));
        c->dseeds_cap = k;
    }
    CelfDev h{};
    h.ostart = c->ostart; h.olen = c->olen; h.ocur = c->ocur; h.t = t;
    h.trace_len = 0; h.batch0 = batch0; h.status = 0;
    IMX_CUDA(cudaMemcpyAsync(c->cdev, &h, sizeof h, cudaMemcpyHostToDevice, c->st));
    unsigned long long *gain = c->scratch + 7;
    IMX_CUDA(cudaMemsetAsync(gain, 0, sizeof(unsigned long long), c->st));
    int *grid_cache = c->celf_grid;
    const int enc = c->C ? 0 : 1;
    void *fn = enc ? (void *)k_celf_rounds<true, false> : (void *)k_celf_rounds<false, false>;
    if (!grid_cache[enc]) {
        // fewer CTAs make the grid barriers cheaper; the evaluation batches
        // still have one CTA per candidate in flight per SM slot
        int per_sm = 0, sms = 0;
        IMX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0));
        IMX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->dev));
        int want = 4;
        if (const char *b = getenv("IMX_CELF_BPSM")) want = std::max(1, atoi(b));
        grid_cache[enc] = std::max(1, std::min(per_sm, want)) * sms;
    }
    int32_t kk = k;
    int vb = c->vb;
    const uint32_t *L = c->L, *C = c->C;
    uint32_t *cov = c->cov;
    Lay ld = c->lay;
    int32_t ns = c->ns, cw = c->cw;
    int64_t *per_sim = c->per_sim, *fresh = c->eval_out, *trace = c->dtrace, *sg = c->dsgains;
    uint8_t *inS = c->inS;
    int32_t *o0 = c->oid[0], *o1 = c->oid[1], *sid = c->sid, *sd = c->dseeds;
    unsigned long long *k0 = c->okey[0], *k1 = c->okey[1], *skey = c->skey;
    int64_t cap = c->trace_cap;
    CelfDev *stp = c->cdev;
    // next round's first batch = bpct% of this round's refreshed prefix
    int32_t bpct = 150;
    if (const char *b = getenv("IMX_CELF_BATCH_PCT")) bpct = std::max(1, atoi(b));
    // candidates evaluated side by side per CTA (1, 2, 4 or 8)
    int32_t ngroup = 1;
    if (const char *gv = getenv("IMX_CELF_GROUPS")) ngroup = std::min(8, std::max(1, atoi(gv)));
    while (ngroup & (ngroup - 1)) --ngroup;
    int64_t *xbuf = nullptr, xcap = 0;
    // encoded labels with the memo's gains at hand: early rounds use the seed table
    if (!c->stab) IMX_CUDA(pool_alloc((void **)&c->stab, sizeof(int2) * kTab * c->ld, c->st));
    int2 *tab = (!c->C && c->memo_ready && !getenv("IMX_CELF_NO_TAB")) ? c->stab : nullptr;
    int64_t tab_ld = c->ld;
    const int64_t *gains0 = c->gains;
    // seed-table batches above this many candidates per CTA leave the kernel (k_wide_tab_round)
    int64_t wide_out = kWideOutPerCta;
    if (const char *wo = getenv("IMX_CELF_WIDE_OUT")) wide_out = std::max<int64_t>(0, atoll(wo));
    // the memo's first-seed speculation (round 1 from g1 when seed 0 is the max-degree vertex)
    const int64_t *g1 = (tab && c->g1_ready) ? c->g1 : nullptr;
    const unsigned long long *hubp = c->scratch + 15;
    void *args[] = {&kk, &vb, &L, &C, &cov, &ld, &ns, &cw, &per_sim, &inS, &o0, &o1, &k0, &k1, &fresh,
                    &skey, &sid, &trace, &cap, &sd, &sg, &gain, &stp, &bpct, &ngroup, &xbuf, &xcap, &tab,
                    &tab_ld, &gains0, &wide_out, &g1, &hubp};
    const bool hprof = getenv("IMX_CELF_PROFILE") != nullptr;
    auto hq0 = std::chrono::steady_clock::now();
    if (hprof) IMX_CUDA(cudaStreamSynchronize(c->st));
    auto hq1 = std::chrono::steady_clock::now();
    IMX_CUDA(cudaLaunchCooperativeKernel(fn, grid_cache[enc], 256, args, 0, c->st));
    count_launch(c);
    auto hq2 = std::chrono::steady_clock::now();
    IMX_CUDA(cudaMemcpyAsync(&h, c->cdev, sizeof h, cudaMemcpyDeviceToHost, c->st));
    IMX_CUDA(cudaStreamSynchronize(c->st));
    if (hprof)
        fprintf(stderr, "[celf host]   pre-launch wait %.3f ms, launch call %.3f ms, kernel+state %.3f ms\n",
                std::chrono::duration<double, std::milli>(hq1 - hq0).count(),
                std::chrono::duration<double, std::milli>(hq2 - hq1).count(),
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - hq2).count());
    c->big_key = h.big_key;
    c->big_kr = (h.status == 2 || h.status == 4) ? h.big_kr : 0;
    if (getenv("IMX_CELF_PROFILE"))
        fprintf(stderr, "[celf] rounds %d..%d grid %d: eval %.1f us, trace+rank+commit %.1f us, (unused) %.1f us, merge %.1f us; "
                "%llu eval steps, %llu evaluations (block 0 evals %.1f us, eval barrier %.1f us, batch max %.1f us)\n",
                t, h.t, grid_cache[enc], h.prof[0] * 1e-3, h.prof[1] * 1e-3,
                h.prof[2] * 1e-3, h.prof[3] * 1e-3, h.prof[4], h.prof[5], h.prof[6] * 1e-3, h.prof[7] * 1e-3,
                h.prof[8] * 1e-3);
    if (h.status == 3) {
        if (h.olen == 0) set_error("no candidate left at round %d", h.t);
        else set_error("CELF self-check: committed gain %lld != evaluated %lld for vertex %d",
                       (long long)h.bad_got, (long long)h.bad_want, h.bad_v);
        return IMX_EINTERNAL;
    }
    // collect the records and the seeds of the rounds this launch finished
    if (h.trace_len) {
        const int64_t base = c->trace_n;
        IMX_TRY(trace_reserve(c, base + 5 * h.trace_len));
        c->trace_n = base + 5 * h.trace_len;
        IMX_CUDA(cudaMemcpyAsync(c->trace + base, c->dtrace, sizeof(int64_t) * 5 * h.trace_len,
                                 cudaMemcpyDeviceToHost, c->st));
    }
    if (h.t > t) {
        IMX_CUDA(cudaMemcpyAsync(seeds.data() + t, c->dseeds + t, sizeof(int32_t) * (h.t - t), cudaMemcpyDeviceToHost, c->st));
        IMX_CUDA(cudaMemcpyAsync(gains.data() + t, c->dsgains + t, sizeof(int64_t) * (h.t - t), cudaMemcpyDeviceToHost, c->st));
    }
    IMX_CUDA(cudaStreamSynchronize(c->st));
    c->ostart = h.ostart; c->olen = h.olen; c->ocur = h.ocur;
    c->evaluated = -1;          // not tracked on the device path
    *status_out = h.status;
    *t_out = h.t;
    *batch0_out = h.batch0;
    return IMX_OK;
}

// An oversized round (refreshed prefix > kMaxRank, or more trace records than
// the kernel's buffer) finished with device-wide primitives: the persistent
// kernel stopped after evaluating the prefix (fresh[0, hi) and the best key
// are on the device), so nothing is re-evaluated; the refreshed vertices are
// radix-sorted by fresh key instead of ranked pairwise.
__global__ void k_big_round_prep(const int32_t *__restrict__ oid, const unsigned long long *__restrict__ okey,
                                 const int64_t *__restrict__ fresh, int64_t kr, int vb, int32_t best_v,
                                 int64_t best_f, int32_t t, int64_t *__restrict__ rec,
                                 unsigned long long *__restrict__ keys, int32_t *__restrict__ ids) {
    const uint32_t vmask = (vb >= 32) ? 0xffffffffu : ((1u << vb) - 1u);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= kr;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t *r = rec + 5 * i;
        if (i == kr) {          // the commit record follows the refresh records
            r[0] = best_v; r[1] = best_f; r[2] = best_f; r[3] = 1; r[4] = t;
            continue;
        }
        const int32_t v = oid[i];
        const int64_t f = fresh[i];
        r[0] = v; r[1] = (int64_t)(okey[i] >> vb); r[2] = f; r[3] = 0; r[4] = t;
        keys[i] = v == best_v ? 0ull : (((unsigned long long)f << vb) | (unsigned long long)(vmask - (uint32_t)v));
        ids[i] = v;
    }
}

static int celf_big_round(imx_ctx *c, int32_t t, int64_t &batch0, std::vector<int32_t> &seeds,
                          std::vector<int64_t> &gains, int64_t *partial_gain = nullptr) {
    const int64_t kr = c->big_kr;
    const unsigned long long bestkey = c->big_key;
    const uint64_t vmask = (c->vb >= 32) ? 0xffffffffull : ((1ull << c->vb) - 1);
    const int32_t best_v = (int32_t)(vmask - (bestkey & vmask));
    const int64_t best_f = (int64_t)(bestkey >> c->vb);
    cudaStream_t st = c->st;
    int32_t *oid = c->oid[c->ocur] + c->ostart;
    unsigned long long *okey = c->okey[c->ocur] + c->ostart;
    int64_t *rec = nullptr;
    unsigned long long *keys = nullptr, *skeys = nullptr;
    int32_t *ids = nullptr, *sids = nullptr;
    void *tmp = nullptr;
    size_t tb = 0;
    int rc = IMX_OK;
#define GB(call) do { cudaError_t _e = (call); if (_e != cudaSuccess) { rc = cuda_fail(_e, #call, __FILE__, __LINE__); goto done; } } while (0)
    GB(pool_alloc((void **)&rec, sizeof(int64_t) * 5 * (kr + 1), st));
    GB(pool_alloc((void **)&keys, sizeof(unsigned long long) * kr, st));
    GB(pool_alloc((void **)&skeys, sizeof(unsigned long long) * kr, st));
    GB(pool_alloc((void **)&ids, sizeof(int32_t) * kr, st));
    GB(pool_alloc((void **)&sids, sizeof(int32_t) * kr, st));
    k_big_round_prep<<<grid_for(kr + 1), 256, 0, st>>>(oid, okey, c->eval_out, kr, c->vb, best_v, best_f, t, rec,
                                                        keys, ids);
    GB(cudaGetLastError());
    GB(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, keys, skeys, ids, sids, kr, 0, 64, st));
    GB(pool_alloc(&tmp, tb, st));
    GB(cub::DeviceRadixSort::SortPairsDescending(tmp, tb, keys, skeys, ids, sids, kr, 0, 64, st));
    count_launch(c, 5);
    {
        unsigned long long *gain = c->scratch + 7;
        GB(cudaMemsetAsync(gain, 0, sizeof(unsigned long long), st));
        launch_commit(c, best_v, gain, t);
        GB(cudaGetLastError());
        count_launch(c);
        // merge order[kr, olen) with the kr-1 sorted refreshed vertices (the
        // winner's key 0 sorts last and is dropped)
        const int64_t na = c->olen - kr, nback = kr - 1;
        const int nxt = c->ocur ^ 1;
        k_merge<<<grid_for(na + nback), 256, 0, st>>>(oid + kr, okey + kr, na, sids, skeys, nback, c->oid[nxt],
                                                      c->okey[nxt]);
        GB(cudaGetLastError());
        count_launch(c);
        const int64_t base = c->trace_n;
        // room for the later rounds too (2^18 records): growing the host buffer
        // after this copy would wait for it and copy 91 MB on the host (C4: +6.6 ms)
        if ((rc = trace_reserve(c, base + 5 * (kr + 1) + 5 * ((int64_t)1 << 18))) != IMX_OK) goto done;
        // the records (C4 round 1: 2.3 M, 91 MB) go to the host on the side
        // stream while the next rounds run; rec is freed there after the copy
        if (!c->tst) GB(acquire_stream(c->dev, &c->tst));
        // the commit's gain is read back BEFORE the side stream is released: both copies
        // become ready behind k_merge, and when the 91 MB of records reached the one
        // device-to-host copy engine first, these 8 bytes (and the host) waited 1.7 ms
        // for them -- two runs in three on C4
        unsigned long long got = 0;
        GB(cudaMemcpyAsync(&got, gain, sizeof got, cudaMemcpyDeviceToHost, st));
        {
            cudaEvent_t ev;
            GB(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            GB(cudaEventRecord(ev, st));
            GB(cudaStreamWaitEvent(c->tst, ev, 0));
            cudaEventDestroy(ev);
        }
        GB(cudaMemcpyAsync(c->trace + base, rec, sizeof(int64_t) * 5 * (kr + 1), cudaMemcpyDeviceToHost, c->tst));
        GB(cudaFreeAsync(rec, c->tst));
        rec = nullptr;
        GB(cudaStreamSynchronize(st));
        if (partial_gain) {
            *partial_gain = (int64_t)got;       // one rank's part: checked after the next exchange
        } else if ((int64_t)got != best_f) {
            set_error("CELF self-check: committed gain %lld != evaluated %lld for vertex %d",
                      (long long)got, (long long)best_f, best_v);
            rc = IMX_EINTERNAL;
            goto done;
        }
        c->trace_n = base + 5 * (kr + 1);
        c->ocur = nxt;
        c->ostart = 0;
        c->olen = na + nback;
        seeds[t] = best_v;
        gains[t] = best_f;
        batch0 = std::min<int64_t>(kFirstBatchCap, std::max<int64_t>(64, kr));
    }
done:
    for (void *p : {(void *)rec, (void *)keys, (void *)skeys, (void *)ids, (void *)sids, tmp})
        if (p) cudaFreeAsync(p, st);
#undef GB
    return rc;
}

// status 6 of the persistent kernel: the huge seed-table batch it left
// (state in cdev: xlo, xhi, xbest) evaluated by k_wide_tab_round up to the
// round's stop; big_key / big_kr then feed celf_big_round
static int celf_wide_round(imx_ctx *c, int32_t t, int64_t batch0) {
    const bool tab1 = t == 1 && c->ns <= 4 * kWideRowQuads;
    int *grid = &c->wide_grid[tab1 ? 1 : 0];
    void *fn = tab1 ? (void *)k_wide_tab_round<true> : (void *)k_wide_tab_round<false>;
    if (!*grid) {
        int per_sm = 0, sms = 0;
        IMX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kWideSmem));
        IMX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, kWideSmem));
        IMX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->dev));
        *grid = std::max(1, std::min(per_sm, tab1 ? 2 : 3)) * sms;
    }
    IMX_CUDA(cudaMemsetAsync(c->cdev->smax, 0, sizeof(unsigned long long) * 8, c->st));   // smax[4], wctr[4]
    const uint32_t *L = c->L;
    Lay ld = c->lay;
    int32_t ns = c->ns;
    const int2 *tab = c->stab;
    int64_t tab_ld = c->ld;
    int ntab = t;
    const int64_t *gains0 = c->gains;
    const int32_t *cand = c->oid[c->ocur] + c->ostart;
    const unsigned long long *keys = c->okey[c->ocur] + c->ostart;
    int64_t olen = c->olen, *fresh = c->eval_out;
    int vb = c->vb;
    CelfDev *stp = c->cdev;
    int64_t cap = (int64_t)*grid * 512;
    void *args[] = {&L, &ld, &ns, &tab, &tab_ld, &ntab, &gains0, &cand, &keys, &olen, &fresh, &vb, &stp, &batch0, &cap};
    IMX_CUDA(cudaLaunchCooperativeKernel(fn, *grid, 256, args, kWideSmem, c->st));
    count_launch(c);
    CelfDev h;
    IMX_CUDA(cudaMemcpyAsync(&h, c->cdev, sizeof h, cudaMemcpyDeviceToHost, c->st));
    IMX_CUDA(cudaStreamSynchronize(c->st));
    c->big_key = h.big_key;
    c->big_kr = h.big_kr;
    if (getenv("IMX_CELF_PROFILE"))
        fprintf(stderr, "[celf] wide round %d grid %d: %llu eval steps, %llu evaluations, kr %lld\n", t, *grid,
                h.prof[4], h.prof[5], (long long)h.big_kr);
    return IMX_OK;
}

// The whole CELF loop on one context (single-rank path): the persistent
// cooperative kernel runs the rounds; a round it cannot hold (trace buffer
// full, refreshed prefix larger than kMaxRank) is finished on the host.
// Sharded CELF driven by the device (exchange mode).  The persistent kernel
// runs the rounds exactly as on one rank but pauses after every evaluated
// batch, leaving this rank's partial gains in the exchange buffer; the host
// only enqueues the sum over the ranks (comm_allreduce_i64: ncclAllReduce in
// place on the context stream) and the next launch, which resumes from the
// summed batch.  No host decision and no host copy of the data sit inside
// the loop: the host reads the kernel state with a lag of kXchgChunk
// launches, and since every rank reaches the same state at the same launch,
// all ranks enqueue the same collectives.  Launches after a stop are no-ops.
constexpr int64_t kXchgCap = 16384;     // candidates per exchanged batch
constexpr int kXchgChunk = 2;           // launches between state reads

static int celf_select_xchg(imx_ctx *c, int32_t k, std::vector<int32_t> &seeds, std::vector<int64_t> &gains) {
    const int64_t n = c->g->n;
    // the buffers of celf_device_rounds
    if (!c->cdev) {
        IMX_CUDA(pool_alloc((void **)&c->cdev, sizeof(CelfDev), c->st));
        IMX_CUDA(pool_alloc((void **)&c->skey, sizeof(unsigned long long) * kMaxRank, c->st));
        IMX_CUDA(pool_alloc((void **)&c->sid, sizeof(int32_t) * kMaxRank, c->st));
        c->trace_cap = std::max<int64_t>(1 << 16, std::min<int64_t>(4 * n + 4096, 1 << 21));
        if (const char *tc = getenv("IMX_CELF_TRACE_CAP")) c->trace_cap = std::max<int64_t>(8, atoll(tc));
        IMX_CUDA(pool_alloc((void **)&c->dtrace, sizeof(int64_t) * 5 * c->trace_cap, c->st));
    }
    if (!c->dseeds || c->dseeds_cap < k) {
        if (c->dseeds) { cudaFreeAsync(c->dseeds, c->st); cudaFreeAsync(c->dsgains, c->st); }
        IMX_CUDA(pool_alloc((void **)&c->dseeds, sizeof(int32_t) * k, c->st));
        IMX_CUDA(pool_alloc((void **)&c->dsgains, sizeof(int64_t) * k, c->st));
        c->dseeds_cap = k;
    }
    int64_t xcap = kXchgCap;
    if (const char *e = getenv("IMX_CELF_XCHG_CAP")) xcap = std::max<int64_t>(1, atoll(e));
    int64_t *xbuf = nullptr;
    IMX_CUDA(pool_alloc((void **)&xbuf, sizeof(int64_t) * (xcap + 1), c->st));
    IMX_CUDA(cudaMemsetAsync(xbuf, 0, sizeof(int64_t) * (xcap + 1), c->st));
    CelfDev h{};
    h.ostart = c->ostart; h.olen = c->olen; h.ocur = c->ocur; h.t = 0;
    h.batch0 = 64;
    IMX_CUDA(cudaMemcpyAsync(c->cdev, &h, sizeof h, cudaMemcpyHostToDevice, c->st));
    unsigned long long *gain = c->scratch + 7;
    IMX_CUDA(cudaMemsetAsync(gain, 0, sizeof(unsigned long long), c->st));
    const int enc = c->C ? 0 : 1;
    // the exchange-mode kernel may hold fewer CTAs per SM than the single-rank
    // one (its own grid cache slot)
    void *fn = enc ? (void *)k_celf_rounds<true, true> : (void *)k_celf_rounds<false, true>;
    if (!c->celf_grid[2 + enc]) {
        int per_sm = 0, sms = 0;
        IMX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0));
        IMX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->dev));
        int want = 4;
        if (const char *b = getenv("IMX_CELF_BPSM")) want = std::max(1, atoi(b));
        c->celf_grid[2 + enc] = std::max(1, std::min(per_sm, want)) * sms;
    }
    int32_t kk = k, bpct = 150, ngroup = 1;
    if (const char *b = getenv("IMX_CELF_BATCH_PCT")) bpct = std::max(1, atoi(b));
    int vb = c->vb;
    const uint32_t *L = c->L, *C = c->C;
    uint32_t *cov = c->cov;
    Lay ld = c->lay;
    int32_t ns = c->ns, cw = c->cw;
    int64_t *per_sim = c->per_sim, *fresh = c->eval_out, *trace = c->dtrace, *sg = c->dsgains;
    uint8_t *inS = c->inS;
    int32_t *o0 = c->oid[0], *o1 = c->oid[1], *sid = c->sid, *sd = c->dseeds;
    unsigned long long *k0 = c->okey[0], *k1 = c->okey[1], *skey = c->skey;
    int64_t cap = c->trace_cap;
    CelfDev *stp = c->cdev;
    int2 *tab = nullptr;             // partial gains per rank: the covered bitmap only
    int64_t tab_ld = 0, wide_out = 0;
    const int64_t *gains0 = nullptr, *g1 = nullptr;
    const unsigned long long *hubp = c->scratch + 15;
    void *args[] = {&kk, &vb, &L, &C, &cov, &ld, &ns, &cw, &per_sim, &inS, &o0, &o1, &k0, &k1, &fresh,
                    &skey, &sid, &trace, &cap, &sd, &sg, &gain, &stp, &bpct, &ngroup, &xbuf, &xcap, &tab,
                    &tab_ld, &gains0, &wide_out, &g1, &hubp};
    CelfDev *snap = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    int rc = IMX_OK;
    auto drain_trace = [&](CelfDev &s) -> int {
        if (s.trace_len) {
            const int64_t base = c->trace_n;
            IMX_TRY(trace_reserve(c, base + 5 * s.trace_len));
            IMX_CUDA(cudaMemcpyAsync(c->trace + base, c->dtrace, sizeof(int64_t) * 5 * s.trace_len,
                                     cudaMemcpyDeviceToHost, c->st));
            IMX_CUDA(cudaStreamSynchronize(c->st));
            c->trace_n = base + 5 * s.trace_len;
            s.trace_len = 0;
        }
        return IMX_OK;
    };
    auto body = [&]() -> int {
        IMX_CUDA(pinned_get((void **)&snap, sizeof(CelfDev) * 2));
        for (auto &e : ev) IMX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        int slot = 0, pending = -1;
        for (;;) {
            for (int j = 0; j < kXchgChunk; ++j) {
                IMX_CUDA(cudaLaunchCooperativeKernel(fn, c->celf_grid[2 + enc], 256, args, 0, c->st));
                count_launch(c);
                IMX_TRY(comm_allreduce_i64(c->comm, xbuf, xcap + 1, c->st));
            }
            IMX_CUDA(cudaMemcpyAsync(snap + slot, c->cdev, sizeof(CelfDev), cudaMemcpyDeviceToHost, c->st));
            IMX_CUDA(cudaEventRecord(ev[slot], c->st));
            const int look = pending;
            pending = slot;
            slot ^= 1;
            if (look < 0) continue;
            IMX_CUDA(cudaEventSynchronize(ev[look]));
            const int32_t status = snap[look].status;
            if (status == 0 || status == 5) continue;
            // a stop: everything enqueued after it was a no-op; act on the current state
            IMX_CUDA(cudaStreamSynchronize(c->st));
            IMX_CUDA(cudaMemcpy(&h, c->cdev, sizeof h, cudaMemcpyDeviceToHost));
            pending = -1;
            if (h.status == 3) {
                if (h.olen == 0) set_error("no candidate left at round %d", h.t);
                else set_error("CELF self-check: committed gain %lld != evaluated %lld for vertex %d",
                               (long long)h.bad_got, (long long)h.bad_want, h.bad_v);
                return IMX_EINTERNAL;
            }
            IMX_TRY(drain_trace(h));
            if (h.status == 1) return IMX_OK;
            // trace buffer full (2) or a round the kernel cannot hold (4)
            c->ostart = h.ostart; c->olen = h.olen; c->ocur = h.ocur;
            const bool oversized = h.big_kr > 0 && (h.status == 4 || h.big_kr + 1 > c->trace_cap);
            if (h.t > 0 && oversized) {
                c->big_key = h.big_key;
                c->big_kr = h.big_kr;
                int64_t b0 = h.batch0, part = 0;
                std::vector<int32_t> sdum(k);
                std::vector<int64_t> gdum(k);
                IMX_TRY(celf_big_round(c, h.t, b0, sdum, gdum, &part));
                IMX_CUDA(cudaMemcpyAsync(c->dseeds + h.t, &sdum[h.t], sizeof(int32_t), cudaMemcpyHostToDevice, c->st));
                IMX_CUDA(cudaMemcpyAsync(c->dsgains + h.t, &gdum[h.t], sizeof(int64_t), cudaMemcpyHostToDevice, c->st));
                h.xpend = 1; h.xpend_v = sdum[h.t]; h.xpend_want = gdum[h.t]; h.xpend_got = part;
                h.ostart = c->ostart; h.olen = c->olen; h.ocur = c->ocur;
                h.t += 1;
                h.batch0 = b0;
            }
            h.status = 0;
            h.xphase = 0;
            h.big_kr = 0;
            IMX_CUDA(cudaMemcpyAsync(c->cdev, &h, sizeof h, cudaMemcpyHostToDevice, c->st));
            IMX_CUDA(cudaMemsetAsync(gain, 0, sizeof(unsigned long long), c->st));
            IMX_CUDA(cudaStreamSynchronize(c->st));
            if (h.t >= k) {        // the big round was the last one: finish like a done kernel
                h.status = 1;
                return IMX_OK;
            }
        }
    };
    rc = body();
    if (rc == IMX_OK) {
        // the last commit's part goes out with one more exchange
        int64_t part = h.xpend ? h.xpend_got : 0;
        IMX_CUDA(cudaMemcpyAsync(xbuf + xcap, &part, sizeof part, cudaMemcpyHostToDevice, c->st));
        rc = comm_allreduce_i64(c->comm, xbuf + xcap, 1, c->st);
        int64_t tot = 0;
        if (rc == IMX_OK) {
            IMX_CUDA(cudaMemcpyAsync(&tot, xbuf + xcap, sizeof tot, cudaMemcpyDeviceToHost, c->st));
            IMX_CUDA(cudaMemcpyAsync(seeds.data(), c->dseeds, sizeof(int32_t) * k, cudaMemcpyDeviceToHost, c->st));
            IMX_CUDA(cudaMemcpyAsync(gains.data(), c->dsgains, sizeof(int64_t) * k, cudaMemcpyDeviceToHost, c->st));
            IMX_CUDA(cudaStreamSynchronize(c->st));
            if (h.xpend && tot != h.xpend_want) {
                set_error("CELF self-check: committed gain %lld != evaluated %lld for vertex %d",
                          (long long)tot, (long long)h.xpend_want, h.xpend_v);
                rc = IMX_EINTERNAL;
            }
            c->ostart = h.ostart; c->olen = h.olen; c->ocur = h.ocur;
        }
    }
    for (auto &e : ev) if (e) cudaEventDestroy(e);
    if (snap) pinned_put(snap, sizeof(CelfDev) * 2);
    cudaFreeAsync(xbuf, c->st);
    c->evaluated = -1;
    return rc;
}

extern "C" int imx_celf_select(imx_ctx *c, int32_t k, int32_t *seeds_out, int64_t *gains_out,
                               int64_t *trace_len) {
    CELF_CHECK(c);
    const int64_t n = c->g->n;
    if (k < 1 || k > n) { set_error("k=%d invalid for n=%lld", k, (long long)n); return IMX_ECONSTRAINT; }
    if (c->olen != n) { set_error("CELF state already advanced (call imx_celf_reset)"); return IMX_EINVAL; }
    cudaEventRecord(c->ev[6], c->st);
    c->trace_n = 0;
    c->evaluated = 0;
    std::vector<int32_t> seeds(k);
    std::vector<int64_t> gains(k);
    int64_t batch0 = 64;
    int32_t t = 0;
    const char *mode = getenv("IMX_CELF");
    const bool host_only = mode && !strcmp(mode, "host");
    int coop = 0;
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, c->dev);
    const bool hprof = getenv("IMX_CELF_PROFILE") != nullptr;
    auto hnow = [] { return std::chrono::steady_clock::now(); };
    auto hms = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
        return std::chrono::duration<double, std::milli>(b - a).count();
    };
    auto h0 = hnow();
    while (t < k) {
        if (!host_only && coop) {
            int32_t status = 0, t2 = t;
            auto h1 = hnow();
            IMX_TRY(celf_device_rounds(c, t, k, batch0, &status, &t2, &batch0, seeds, gains));
            if (hprof) fprintf(stderr, "[celf host] device rounds %d..%d: %.3f ms (status %d)\n", t, t2, hms(h1, hnow()), status);
            const bool progressed = t2 > t;
            t = t2;
            if (status == 1 || t >= k) break;
            // a round the kernel can never hold (refreshed prefix > kMaxRank, or
            // more records than the whole trace buffer) is finished right here
            // from its evaluated prefix; otherwise drain the trace and relaunch
            if (status == 6) {
                auto h2 = hnow();
                IMX_TRY(celf_wide_round(c, t, batch0));
                if (hprof) fprintf(stderr, "[celf host] wide round %d: %.3f ms\n", t, hms(h2, hnow()));
                status = 4;                   // evaluated: finished below from big_key / big_kr
            }
            const bool oversized = c->big_kr > 0 && (status == 4 || c->big_kr + 1 > c->trace_cap);
            if (t > 0 && oversized) {
                auto h2 = hnow();
                IMX_TRY(celf_big_round(c, t, batch0, seeds, gains));
                if (hprof) fprintf(stderr, "[celf host] big round %d (kr %lld): %.3f ms\n", t, (long long)c->big_kr, hms(h2, hnow()));
                ++t;
                continue;
            }
            if (status == 2 && progressed) continue;
        }
        IMX_TRY(celf_host_round(c, t, batch0, seeds.data(), gains.data()));   // status 4 or host mode
        ++t;
    }
    if (seeds_out) std::copy(seeds.begin(), seeds.end(), seeds_out);
    if (gains_out) std::copy(gains.begin(), gains.end(), gains_out);
    auto h3 = hnow();
    IMX_TRY(trace_flush(c));
    if (hprof) fprintf(stderr, "[celf host] trace flush %.3f ms, select total %.3f ms\n", hms(h3, hnow()), hms(h0, hnow()));
    cudaEventRecord(c->ev[7], c->st);
    cudaEventSynchronize(c->ev[7]);
    cudaEventElapsedTime(&c->tm.select_ms, c->ev[6], c->ev[7]);
    c->tm.celf_evaluations = c->evaluated;
    if (trace_len) *trace_len = c->trace_n / 5;
    return IMX_OK;
}

extern "C" int imx_celf_select_sharded(imx_ctx *c, int32_t k, imx_allreduce_fn allreduce, void *user,
                                       int32_t *seeds_out, int64_t *gains_out, int64_t *trace_len) {
    CELF_CHECK(c);
    const int64_t n = c->g->n;
    if (!allreduce) { set_error("allreduce callback is NULL"); return IMX_EINVAL; }
    if (k < 1 || k > n) { set_error("k=%d invalid for n=%lld", k, (long long)n); return IMX_ECONSTRAINT; }
    if (c->olen != n) { set_error("CELF state already advanced (call imx_celf_reset)"); return IMX_EINVAL; }
    cudaEventRecord(c->ev[6], c->st);
    c->trace_n = 0;
    c->evaluated = 0;
    std::vector<int32_t> seeds(k);
    std::vector<int64_t> gains(k);
    ShardReduce sr;
    sr.fn = allreduce;
    sr.user = user;
    int64_t batch0 = 64;
    for (int32_t t = 0; t < k; ++t) IMX_TRY(celf_host_round(c, t, batch0, seeds.data(), gains.data(), &sr));
    if (sr.pending) {               // the last commit has no later batch to ride on
        int64_t g = sr.pending_got;
        if (allreduce(&g, 1, user) != 0) { set_error("allreduce callback failed"); return IMX_EINTERNAL; }
        IMX_TRY(shard_check(sr, g));
    }
    if (seeds_out) std::copy(seeds.begin(), seeds.end(), seeds_out);
    if (gains_out) std::copy(gains.begin(), gains.end(), gains_out);
    cudaEventRecord(c->ev[7], c->st);
    cudaEventSynchronize(c->ev[7]);
    cudaEventElapsedTime(&c->tm.select_ms, c->ev[6], c->ev[7]);
    c->tm.celf_evaluations = c->evaluated;
    if (trace_len) *trace_len = c->trace_n / 5;
    return IMX_OK;
}

extern "C" int imx_celf_select_comm(imx_ctx *c, int32_t k, int32_t *seeds_out, int64_t *gains_out,
                                    int64_t *trace_len) {
    CELF_CHECK(c);
    const int64_t n = c->g->n;
    if (!c->comm) { set_error("no communicator attached (imx_ctx_attach_comm)"); return IMX_EINVAL; }
    if (k < 1 || k > n) { set_error("k=%d invalid for n=%lld", k, (long long)n); return IMX_ECONSTRAINT; }
    if (c->olen != n) { set_error("CELF state already advanced (call imx_celf_reset)"); return IMX_EINVAL; }
    cudaEventRecord(c->ev[6], c->st);
    c->trace_n = 0;
    c->evaluated = 0;
    std::vector<int32_t> seeds(k);
    std::vector<int64_t> gains(k);
    int coop = 0;
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, c->dev);
    const char *mode = getenv("IMX_CELF");
    if (coop && !(mode && !strcmp(mode, "host"))) {
        IMX_TRY(celf_select_xchg(c, k, seeds, gains));
        IMX_TRY(trace_flush(c));
        if (seeds_out) std::copy(seeds.begin(), seeds.end(), seeds_out);
        if (gains_out) std::copy(gains.begin(), gains.end(), gains_out);
        cudaEventRecord(c->ev[7], c->st);
        cudaEventSynchronize(c->ev[7]);
        cudaEventElapsedTime(&c->tm.select_ms, c->ev[6], c->ev[7]);
        c->tm.celf_evaluations = c->evaluated;
        if (trace_len) *trace_len = c->trace_n / 5;
        return IMX_OK;
    }
    ShardReduce sr;
    sr.comm = c->comm;
    int64_t batch0 = 64;
    for (int32_t t = 0; t < k; ++t) IMX_TRY(celf_host_round(c, t, batch0, seeds.data(), gains.data(), &sr));
    if (sr.pending) {               // the last commit has no later batch to ride on
        int64_t *d = c->eval_out;
        IMX_CUDA(cudaMemcpyAsync(d, &sr.pending_got, sizeof(int64_t), cudaMemcpyHostToDevice, c->st));
        IMX_TRY(comm_allreduce_i64(c->comm, d, 1, c->st));
        int64_t g = 0;
        IMX_CUDA(cudaMemcpyAsync(&g, d, sizeof g, cudaMemcpyDeviceToHost, c->st));
        IMX_CUDA(cudaStreamSynchronize(c->st));
        IMX_TRY(shard_check(sr, g));
    }
    if (seeds_out) std::copy(seeds.begin(), seeds.end(), seeds_out);
    if (gains_out) std::copy(gains.begin(), gains.end(), gains_out);
    cudaEventRecord(c->ev[7], c->st);
    cudaEventSynchronize(c->ev[7]);
    cudaEventElapsedTime(&c->tm.select_ms, c->ev[6], c->ev[7]);
    c->tm.celf_evaluations = c->evaluated;
    if (trace_len) *trace_len = c->trace_n / 5;
    return IMX_OK;
}

extern "C" int imx_celf_trace_take(imx_ctx *c, int64_t **out, int64_t *len) {
    CTX_CHECK(c);
    if (!out || !len) { set_error("NULL argument"); return IMX_EINVAL; }
    IMX_TRY(trace_flush(c));
    *len = c->trace_n / 5;
    *out = nullptr;
    if (*len == 0) return IMX_OK;
    *out = c->trace;
    pinned_lend(c->trace, sizeof(int64_t) * c->trace_hcap);
    c->trace = nullptr;
    c->trace_n = 0;
    c->trace_hcap = 0;
    return IMX_OK;
}

extern "C" int imx_celf_trace(imx_ctx *c, int64_t *out, int64_t cap) {
    CTX_CHECK(c);
    IMX_TRY(trace_flush(c));
    const int64_t len = c->trace_n / 5;
    const int64_t k = std::min(cap, len);
    if (k > 0 && out) memcpy(out, c->trace, sizeof(int64_t) * 5 * k);
    return IMX_OK;
}

extern "C" int imx_per_sim(imx_ctx *c, int64_t *out) {
    CELF_CHECK(c);
    IMX_TRY(spec_guard(c));
    if (!out) { set_error("out is NULL"); return IMX_EINVAL; }
    if (c->ns) {
        IMX_CUDA(cudaMemcpyAsync(out, c->per_sim, sizeof(int64_t) * c->ns, cudaMemcpyDeviceToHost, c->st));
        IMX_CUDA(cudaStreamSynchronize(c->st));
    }
    return IMX_OK;
}

extern "C" int imx_copy_owned(imx_ctx *c, uint32_t *bits_out) {
    CELF_CHECK(c);
    IMX_TRY(spec_guard(c));
    if (!bits_out) { set_error("out is NULL"); return IMX_EINVAL; }
    const int64_t n = c->g->n;
    if (n) {
        IMX_CUDA(cudaMemcpyAsync(bits_out, c->cov, sizeof(uint32_t) * (size_t)n * c->cw, cudaMemcpyDeviceToHost, c->st));
        IMX_CUDA(cudaStreamSynchronize(c->st));
    }
    return IMX_OK;
}

