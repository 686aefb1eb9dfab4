// celf.cu -- K6-K8: CELF seed selection on the device (reference
// select_seeds / marginal_gain / commit_seed, selection.py:63-149).
//
// Round-based exact formulation: gains are computed on one
// fixed sample family, so marginal gain is submodular and the reference's
// lazy heap commits, at every round, the lexicographic argmax (max fresh gain,
// then min id) after refreshing exactly the vertices whose stale key does not
// exceed the winner's fresh key.  The device keeps the stale priorities, the
// seed set, the per-lane covered-component bitmaps and per-lane covered
// totals; each round is a handful of kernels with one or two host syncs, and
// the dequeue trace is rebuilt exactly on the host.
#include <algorithm>
#include <vector>
#include <cub/cub.cuh>

#include "ctx.cuh"
#include "uf.cuh"

namespace imx {

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

// size and label of cell (u, r) (encoded labels, or caller labels + C)
template <bool ENC>
__device__ __forceinline__ uint32_t cell_size(const uint32_t *__restrict__ L, const uint32_t *__restrict__ C,
                                              int64_t ld, uint32_t u, uint32_t w, int r, uint32_t &label) {
    if (ENC) {
        if (is_root(w)) { label = u; return (w & COUNT) + 1u; }
        label = w;
        return (L[(int64_t)w * ld + r] & COUNT) + 1u;
    }
    label = w;
    return C[(int64_t)w * ld + r];
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
                                                       const uint32_t *__restrict__ cov, int64_t ld, int32_t ns,
                                                       int32_t cw, int64_t *__restrict__ out) {
    __shared__ unsigned long long part[kEvalThreads / 32];
    const int nqs = (ns + 3) >> 2;
    for (int64_t i = blockIdx.x; i < cnt; i += gridDim.x) {
        const int64_t u = cand[i];
        if (u < 0) { if (threadIdx.x == 0) out[i] = 0; continue; }
        const uint4 *row = reinterpret_cast<const uint4 *>(L + u * ld);
        unsigned long long acc = 0;
        for (int q = threadIdx.x; q < nqs; q += kEvalThreads) {
            const uint4 l4 = row[q];
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
template <bool ENC>
__global__ void k_commit(int32_t u, const uint32_t *__restrict__ L, const uint32_t *__restrict__ C,
                         uint32_t *__restrict__ cov, int64_t ld, int32_t ns, int32_t cw,
                         int64_t *__restrict__ per_sim, uint8_t *__restrict__ inS,
                         unsigned long long *__restrict__ gain) {
    unsigned long long acc = 0;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < ns; r += gridDim.x * blockDim.x) {
        uint32_t lab;
        const uint32_t s = cell_size<ENC>(L, C, ld, (uint32_t)u, L[(int64_t)u * ld + r], r, lab);
        const uint32_t bit = 1u << (r & 31);
        const uint32_t old = atomicOr(cov + (int64_t)lab * cw + (r >> 5), bit);
        if (!(old & bit)) {
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


static void launch_commit(imx_ctx *c, int32_t u, unsigned long long *gain) {
    const int blocks = grid_for(std::max(c->ns, 1));
    if (c->C) k_commit<false><<<blocks, 256, 0, c->st>>>(u, c->L, c->C, c->cov, c->ld, c->ns, c->cw, c->per_sim, c->inS, gain);
    else k_commit<true><<<blocks, 256, 0, c->st>>>(u, c->L, nullptr, c->cov, c->ld, c->ns, c->cw, c->per_sim, c->inS, gain);
}

}  // namespace imx

using namespace imx;

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
    if (c->C) k_eval<false><<<blocks, kEvalThreads, 0, c->st>>>(dcand, cnt, c->L, c->C, c->cov, c->ld, c->ns, c->cw, dout);
    else k_eval<true><<<blocks, kEvalThreads, 0, c->st>>>(dcand, cnt, c->L, nullptr, c->cov, c->ld, c->ns, c->cw, dout);
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
    launch_commit(c, u, sc);
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
        launch_commit(c, best_v, hdr + H_GAIN);
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

