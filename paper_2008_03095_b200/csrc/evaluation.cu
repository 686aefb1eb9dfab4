// evaluation.cu -- fresh-world Monte-Carlo scoring (evaluate_seeds) and the
// hash-sampling uniformity statistic (sampling_cdf), reference
// evaluation.py:101-136 and :157-183.
//
// evaluate_seeds.  The reference samples every world with numpy PCG64
// streams spawned per chunk of 4096 worlds (SeedSequence(rng_seed).spawn):
// world j of chunk c consumes draws [j*E, (j+1)*E) of stream c, edge e is
// live iff random() < p_e with p_e = max(w[slot], w[reciprocal]) over the
// canonical slots in slot order, and the world's score is the size of the
// union of the components that contain a seed.  The host passes each
// stream's 128-bit LCG state and increment; the device reproduces the same
// draws bit for bit by jumping the LCG ahead to a thread's first draw
// (O(log delta) 128-bit multiply-adds) and stepping it from there, so the
// per-world counts -- and the mean / standard error computed from them --
// are identical to the reference's.
//   random() = (next64 >> 11) * 2^-53, so random() < p  <=>
//   (next64 >> 11) < ceil(p * 2^53)   (an exact integer test, p in (0,1))
// A batch of up to 4096 worlds of one chunk is one label matrix
// L[n][ld] (lanes = worlds) fed through the same union-find / compress
// kernels as the hash-sampled lanes (uf.cuh, propagate.cu); the seed
// components are then summed once each through a root bitmap.
//
// sampling_cdf.  values = (hash[canon[i*stride]] ^ X[r]) / H_MAX for every
// strided canonical slot i and scored lane r; sorted on the device (cub
// radix sort of the int32 words -- order-preserving for the division), the
// exact KS distance is a max-reduction of the same f64 expressions the
// reference evaluates, and the histogram follows numpy's uniform-bin rule
// (x*bins truncated, then the +-1 corrections against the bin edges).
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <cub/cub.cuh>

#include "ctx.cuh"
#include "uf.cuh"

namespace imx {

typedef unsigned __int128 u128;

// PCG64 (XSL-RR 128/64) multiplier, numpy's pcg64.h
__host__ __device__ __forceinline__ u128 pcg_mult() {
    return ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
}

__device__ __forceinline__ uint64_t pcg_output(u128 s) {
    const unsigned rot = (unsigned)(s >> 122);
    const uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

// state after `delta` more LCG steps
__device__ __forceinline__ u128 pcg_advance(u128 state, u128 inc, uint64_t delta) {
    u128 am = 1, ap = 0, cm = pcg_mult(), cp = inc;
    while (delta) {
        if (delta & 1) {
            am *= cm;
            ap = ap * cm + cp;
        }
        cp = (cm + 1) * cp;
        cm *= cm;
        delta >>= 1;
    }
    return am * state + ap;
}

// canonical edge list with the integer form of the symmetrized probability
// (evaluation.py:40-44)
__global__ void k_eval_edges(const int64_t *__restrict__ cslot, int64_t me, const int32_t *__restrict__ src,
                             const int32_t *__restrict__ adj, const double *__restrict__ w,
                             const int64_t *__restrict__ recip, int2 *__restrict__ ce,
                             uint64_t *__restrict__ t53) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < me;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = cslot[e];
        const double a = w[s], b = w[recip[s]];
        const double p = a > b ? a : b;          // np.maximum (NaN: never live)
        uint64_t t;
        if (!(p > 0.0)) t = 0;
        else if (p >= 1.0) t = 1ull << 53;
        else t = (uint64_t)ceil(p * 9007199254740992.0);
        ce[e] = make_int2(src[s], adj[s]);
        t53[e] = t;
    }
}

// Jump tables.  The state of world w at edge e0 = j*kRun of its run is
//   S(w, e0) = A_j * S_w + C_j,   S_w = state at the world's first draw,
// with (A_j, C_j) the affine map of j*kRun LCG steps (same for every world
// of the chunk), so a hook thread starts with one 128-bit multiply-add
// instead of an O(log) jump.
constexpr int kRun = 512;
__global__ void k_eval_jumps(int64_t nruns, uint64_t i_hi, uint64_t i_lo, ulonglong2 *__restrict__ jt) {
    const u128 inc = ((u128)i_hi << 64) | i_lo;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nruns;
         j += (int64_t)gridDim.x * blockDim.x) {
        u128 am = 1, ap = 0, cm = pcg_mult(), cp = inc;
        for (uint64_t d = (uint64_t)j * kRun; d; d >>= 1) {
            if (d & 1) {
                am *= cm;
                ap = ap * cm + cp;
            }
            cp = (cm + 1) * cp;
            cm *= cm;
        }
        jt[2 * j] = make_ulonglong2((uint64_t)(am >> 64), (uint64_t)am);
        jt[2 * j + 1] = make_ulonglong2((uint64_t)(ap >> 64), (uint64_t)ap);
    }
}

__global__ void k_eval_worlds(uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo, int64_t pos0,
                              int32_t nw, int64_t me, ulonglong2 *__restrict__ ws) {
    const u128 S0 = ((u128)s_hi << 64) | s_lo, inc = ((u128)i_hi << 64) | i_lo;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nw; r += gridDim.x * blockDim.x) {
        const u128 s = pcg_advance(S0, inc, (uint64_t)(pos0 + r) * (uint64_t)me);
        ws[r] = make_ulonglong2((uint64_t)(s >> 64), (uint64_t)s);
    }
}

// One thread per (world lane, run of kRun edges); a CTA = 128 consecutive
// worlds of one run, so the run's edges are staged once in shared memory and
// the label cells of a vertex are touched by consecutive lanes.  Live
// (edge, world) pairs go to a per-warp queue and are united 32 at a time,
// so the root searches run warp-wide instead of at the live density.
constexpr int kGrp = 8;                   // draws per thread between warp-level enqueues
__global__ void __launch_bounds__(128) k_eval_hook(const int2 *__restrict__ ce, const uint64_t *__restrict__ t53,
                                                   int64_t me, const ulonglong2 *__restrict__ jt,
                                                   const ulonglong2 *__restrict__ ws, uint64_t i_hi,
                                                   uint64_t i_lo, int32_t nw, uint32_t *L, int64_t ld) {
    __shared__ int2 se[kRun];
    __shared__ uint64_t st[kRun + kGrp];
    __shared__ uint32_t qe[4][32 + 32 * kGrp];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned FULL = 0xffffffffu;
    const u128 inc = ((u128)i_hi << 64) | i_lo, M = pcg_mult();
    const int r = blockIdx.x * 128 + threadIdx.x;
    const bool act = r < nw;
    u128 Sw = 0;
    if (act) Sw = ((u128)ws[r].x << 64) | ws[r].y;
    const int64_t nruns = (me + kRun - 1) / kRun;
    uint32_t *q = qe[warp];
    const int rbase = blockIdx.x * 128;
    for (int64_t j = blockIdx.y; j < nruns; j += gridDim.y) {
        const int64_t e0 = j * kRun;
        const int cnt = (int)(me - e0 < kRun ? me - e0 : kRun);
        __syncthreads();
        for (int i = threadIdx.x; i < kRun + kGrp; i += 128) {
            if (i < cnt) {
                se[i] = ce[e0 + i];
                st[i] = t53[e0 + i];
            } else {
                st[i] = 0;                    // never live: draws past the run are discarded
            }
        }
        __syncthreads();
        const ulonglong2 a2 = jt[2 * j], c2 = jt[2 * j + 1];
        u128 s = (((u128)a2.x << 64) | a2.y) * Sw + (((u128)c2.x << 64) | c2.y);
        int qn = 0;
        for (int i0 = 0; i0 < cnt; i0 += kGrp) {
            // kGrp LCG steps, live edges as a bit mask (no per-draw warp vote)
            unsigned bits = 0;
#pragma unroll
            for (int k = 0; k < kGrp; ++k) {
                s = s * M + inc;
                bits |= (unsigned)((pcg_output(s) >> 11) < st[i0 + k]) << k;
            }
            if (!act) bits = 0;
            if (!__any_sync(FULL, bits)) continue;
            // warp prefix sum of the live counts -> queue slots
            const int c = __popc(bits);
            int incl = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += y;
            }
            int pos = qn + incl - c;
            while (bits) {
                const int k = __ffs(bits) - 1;
                bits &= bits - 1;
                q[pos++] = ((uint32_t)(i0 + k) << 8) | (uint32_t)threadIdx.x;
            }
            qn += __shfl_sync(FULL, incl, 31);
            __syncwarp();
            while (qn >= 32) {
                qn -= 32;
                const uint32_t x = q[qn + lane];
                __syncwarp();
                const int2 ed = se[x >> 8];
                unite(L, ld, (uint32_t)ed.x, (uint32_t)ed.y, rbase + (int)(x & 255));
            }
        }
        if (lane < qn) {
            const uint32_t x = q[lane];
            const int2 ed = se[x >> 8];
            unite(L, ld, (uint32_t)ed.x, (uint32_t)ed.y, rbase + (int)(x & 255));
        }
        __syncwarp();
    }
}

// counts[r] += size of each distinct component holding a seed (after the
// compress pass every non-root cell is its root)
__global__ void k_eval_reach(const int32_t *__restrict__ seeds, int32_t k, const uint32_t *__restrict__ L,
                             int64_t ld, int32_t nw, uint32_t *__restrict__ bm, int64_t bw,
                             unsigned long long *__restrict__ counts) {
    const int64_t total = (int64_t)k * nw;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(t / nw), r = (int)(t % nw);
        const uint32_t s = (uint32_t)seeds[i];
        const uint32_t c = L[(int64_t)s * ld + r];
        const uint32_t root = is_root(c) ? s : c;
        const uint32_t rc = is_root(c) ? c : L[(int64_t)root * ld + r];
        const uint32_t bit = 1u << (r & 31);
        const uint32_t old = atomicOr(bm + (int64_t)root * bw + (r >> 5), bit);
        if (!(old & bit)) atomicAdd(counts + r, (unsigned long long)(rc & COUNT) + 1ull);
    }
}

// ---- sampling_cdf ----------------------------------------------------------
__global__ void k_cdf_values(const int32_t *__restrict__ hash, const int64_t *__restrict__ cslot, int64_t stride,
                             const int32_t *__restrict__ X, int32_t scored, int64_t total,
                             int32_t *__restrict__ out) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / scored;
        const int r = (int)(t % scored);
        out[t] = hash[cslot[i * stride]] ^ X[r];
    }
}

// order-preserving map of doubles onto uint64 for atomicMax
__device__ __forceinline__ unsigned long long dkey(double x) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// KS distance over sorted values and the histogram, one pass
__global__ void __launch_bounds__(256) k_cdf_stats(const int32_t *__restrict__ sv, int64_t nv, int32_t bins,
                                                   const double *__restrict__ edges, int use_smem,
                                                   unsigned long long *__restrict__ counts,
                                                   unsigned long long *__restrict__ ksmax) {
    extern __shared__ unsigned int hs[];
    if (use_smem)
        for (int i = threadIdx.x; i < bins; i += blockDim.x) hs[i] = 0;
    __syncthreads();
    const double dn = (double)nv, db = (double)bins;
    double best = -INFINITY;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double x = __ddiv_rn((double)sv[i], 2147483647.0);
        const double above = __dsub_rn(__ddiv_rn((double)(i + 1), dn), x);
        const double below = __dsub_rn(x, __ddiv_rn((double)i, dn));
        best = fmax(best, fmax(above, below));
        if (x >= 0.0 && x <= 1.0) {          // numpy drops values outside the range
            int64_t idx = (int64_t)__dmul_rn(x, db);
            if (idx == bins) --idx;
            if (x < edges[idx]) --idx;
            if (x >= edges[idx + 1] && idx != bins - 1) ++idx;
            if (use_smem) atomicAdd(hs + idx, 1u);
            else atomicAdd(counts + idx, 1ull);
        }
    }
    typedef cub::BlockReduce<double, 256> BR;
    __shared__ typename BR::TempStorage tmp;
    const double bm = BR(tmp).Reduce(best, [](double a, double b) { return a > b ? a : b; });
    if (threadIdx.x == 0 && nv) atomicMax(ksmax, dkey(bm));
    if (use_smem) {
        __syncthreads();
        for (int i = threadIdx.x; i < bins; i += blockDim.x)
            if (hs[i]) atomicAdd(counts + i, (unsigned long long)hs[i]);
    }
}

}  // namespace imx

using namespace imx;

extern "C" int imx_evaluate_seeds(imx_graph *g, const int32_t *seeds, int32_t k, int64_t r_eval,
                                  const uint64_t *streams, int64_t chunk, int64_t *counts_out) {
    if (!g || !seeds || !streams || !counts_out) { set_error("NULL argument"); return IMX_EINVAL; }
    if (k < 1) { set_error("seed set must be nonempty"); return IMX_EINVAL; }
    if (r_eval < 1) { set_error("r_eval must be >= 1, got %lld", (long long)r_eval); return IMX_EINVAL; }
    if (chunk < 1) { set_error("chunk must be >= 1"); return IMX_EINVAL; }
    const int64_t n = g->n, me = g->me;
    for (int32_t i = 0; i < k; ++i)
        if (seeds[i] < 0 || seeds[i] >= n) { set_error("seed outside vertex range"); return IMX_EINVAL; }
    IMX_CUDA(cudaSetDevice(g->dev));
    IMX_TRY(graph_settle(g));          // weights of a deferred graph
    IMX_TRY(ensure_recip(g));          // p = max(w, w[reciprocal]) per canonical edge
    IMX_TRY(ensure_cslot(g));
    cudaStream_t st = g->stream;
    // worlds per batch: the label matrix stays under ~4 GiB
    int64_t B = std::min<int64_t>(chunk, 4096);
    B = std::min<int64_t>(B, std::max<int64_t>(32, ((int64_t)1 << 32) / (4 * std::max<int64_t>(n, 1)) / 32 * 32));
    if (const char *ev = getenv("IMX_EVAL_WORLDS"))   // batch-size override (tests)
        if (atoll(ev) > 0) B = std::min<int64_t>(B, atoll(ev));
    const int64_t ld = (B + 3) / 4 * 4, bw = (B + 31) / 32;
    int2 *ce = nullptr;
    uint64_t *t53 = nullptr;
    uint32_t *L = nullptr, *bm = nullptr;
    int32_t *dseeds = nullptr;
    unsigned long long *dcounts = nullptr;
    ulonglong2 *jt = nullptr, *ws = nullptr;
    int rc = IMX_OK;
    auto fail = [&](cudaError_t e, const char *what) { rc = cuda_fail(e, what, __FILE__, __LINE__); };
    do {
        cudaError_t e;
        if ((e = pool_alloc((void **)&ce, sizeof(int2) * std::max<int64_t>(me, 1), st))) { fail(e, "alloc"); break; }
        if ((e = pool_alloc((void **)&t53, sizeof(uint64_t) * std::max<int64_t>(me, 1), st))) { fail(e, "alloc"); break; }
        if ((e = pool_alloc((void **)&L, sizeof(uint32_t) * std::max<int64_t>(n, 1) * ld, st))) { fail(e, "alloc"); break; }
        if ((e = pool_alloc((void **)&bm, sizeof(uint32_t) * std::max<int64_t>(n, 1) * bw, st))) { fail(e, "alloc"); break; }
        if ((e = pool_alloc((void **)&dseeds, sizeof(int32_t) * k, st))) { fail(e, "alloc"); break; }
        if ((e = pool_alloc((void **)&jt, sizeof(ulonglong2) * 2 * std::max<int64_t>((me + kRun - 1) / kRun, 1), st))) { fail(e, "alloc"); break; }
        if ((e = pool_alloc((void **)&ws, sizeof(ulonglong2) * B, st))) { fail(e, "alloc"); break; }
        if ((e = pool_alloc((void **)&dcounts, sizeof(unsigned long long) * r_eval, st))) { fail(e, "alloc"); break; }
        if ((e = cudaMemcpyAsync(dseeds, seeds, sizeof(int32_t) * k, cudaMemcpyHostToDevice, st))) { fail(e, "copy"); break; }
        if ((e = cudaMemsetAsync(dcounts, 0, sizeof(unsigned long long) * r_eval, st))) { fail(e, "memset"); break; }
        if (me) {
            k_eval_edges<<<grid_for(me), 256, 0, st>>>(g->cslot, me, g->src, g->adj, g->w, g->recip, ce, t53);
            note_launch();
        }
        const int64_t nruns = (me + kRun - 1) / kRun;
        for (int64_t c0 = 0, ci = 0; c0 < r_eval && rc == IMX_OK; c0 += chunk, ++ci) {
            const int64_t cc = std::min<int64_t>(chunk, r_eval - c0);
            const uint64_t *sv = streams + 4 * ci;
            if (me) {
                k_eval_jumps<<<grid_for(nruns, 128), 128, 0, st>>>(nruns, sv[2], sv[3], jt);
                note_launch();
            }
            for (int64_t o = 0; o < cc; o += B) {
                const int32_t nw = (int32_t)std::min<int64_t>(B, cc - o);
                if ((rc = launch_init(L, n, ld, st))) break;
                if (me) {
                    k_eval_worlds<<<grid_for(nw, 128), 128, 0, st>>>(sv[0], sv[1], sv[2], sv[3], o, nw, me, ws);
                    note_launch();
                    const int gx = (int)((nw + 127) / 128);
                    const char *hb = getenv("IMX_EVAL_BPSM");
                    const int64_t bpsm = hb && atoi(hb) > 0 ? atoi(hb) : 64;   // C2 2.31M -> 2.42M worlds/s against 16
                    const int gy = (int)std::min<int64_t>(nruns, std::max<int64_t>(1, 148 * bpsm / gx));
                    k_eval_hook<<<dim3(gx, gy), 128, 0, st>>>(ce, t53, me, jt, ws, sv[2], sv[3], nw, L, ld);
                    note_launch();
                    if ((e = cudaGetLastError())) { fail(e, "k_eval_hook"); break; }
                    if ((rc = launch_compress(L, n, ld, nw, nullptr, st))) break;
                }
                if ((e = cudaMemsetAsync(bm, 0, sizeof(uint32_t) * n * bw, st))) { fail(e, "memset"); break; }
                k_eval_reach<<<grid_for((int64_t)k * nw), 256, 0, st>>>(dseeds, k, L, ld, nw, bm, bw, dcounts + c0 + o);
                note_launch();
                if ((e = cudaGetLastError())) { fail(e, "k_eval_reach"); break; }
            }
        }
        if (rc) break;
        if ((e = cudaMemcpyAsync(counts_out, dcounts, sizeof(int64_t) * r_eval, cudaMemcpyDeviceToHost, st))) { fail(e, "copy"); break; }
        if ((e = cudaStreamSynchronize(st))) { fail(e, "sync"); break; }
    } while (0);
    cudaFreeAsync(ce, st);
    cudaFreeAsync(t53, st);
    cudaFreeAsync(L, st);
    cudaFreeAsync(bm, st);
    cudaFreeAsync(dseeds, st);
    cudaFreeAsync(dcounts, st);
    cudaFreeAsync(jt, st);
    cudaFreeAsync(ws, st);
    return rc;
}

extern "C" int imx_sampling_cdf(imx_graph *g, const int32_t *X, int32_t scored, int64_t stride, int32_t bins,
                                const double *edges, int64_t *counts_out, double *ks_out, int64_t *nvals_out) {
    if (!g || !X || !edges || !counts_out || !ks_out || !nvals_out) { set_error("NULL argument"); return IMX_EINVAL; }
    if (bins < 1) { set_error("need at least 1 bin, got %d", bins); return IMX_EINVAL; }
    if (scored < 0 || stride < 1) { set_error("bad scored/stride"); return IMX_EINVAL; }
    IMX_CUDA(cudaSetDevice(g->dev));
    IMX_TRY(ensure_cslot(g));
    cudaStream_t st = g->stream;
    const int64_t nc = (g->me + stride - 1) / stride, nv = nc * scored;
    int32_t *dX = nullptr, *va = nullptr, *vb = nullptr;
    double *dedges = nullptr;
    unsigned long long *dc = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    int rc = IMX_OK;
    auto fail = [&](cudaError_t e, const char *what) { rc = cuda_fail(e, what, __FILE__, __LINE__); };
    do {
        cudaError_t e;
        const int64_t nva = std::max<int64_t>(nv, 1);
        if ((e = pool_alloc((void **)&dX, sizeof(int32_t) * std::max(scored, 1), st))) { fail(e, "alloc"); break; }
        if ((e = pool_alloc((void **)&va, sizeof(int32_t) * nva, st))) { fail(e, "alloc"); break; }
        if ((e = pool_alloc((void **)&vb, sizeof(int32_t) * nva, st))) { fail(e, "alloc"); break; }
        if ((e = pool_alloc((void **)&dedges, sizeof(double) * (bins + 1), st))) { fail(e, "alloc"); break; }
        if ((e = pool_alloc((void **)&dc, sizeof(unsigned long long) * (bins + 1), st))) { fail(e, "alloc"); break; }
        if ((e = cudaMemcpyAsync(dX, X, sizeof(int32_t) * scored, cudaMemcpyHostToDevice, st))) { fail(e, "copy"); break; }
        if ((e = cudaMemcpyAsync(dedges, edges, sizeof(double) * (bins + 1), cudaMemcpyHostToDevice, st))) { fail(e, "copy"); break; }
        if ((e = cudaMemsetAsync(dc, 0, sizeof(unsigned long long) * (bins + 1), st))) { fail(e, "memset"); break; }
        if (nv) {
            k_cdf_values<<<grid_for(nv), 256, 0, st>>>(g->hash, g->cslot, stride, dX, scored, nv, va);
            note_launch();
            if ((e = cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, va, vb, nv, 0, 32, st))) { fail(e, "sort"); break; }
            if ((e = pool_alloc(&tmp, tmp_bytes, st))) { fail(e, "alloc"); break; }
            if ((e = cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, va, vb, nv, 0, 32, st))) { fail(e, "sort"); break; }
            note_launch(4);
            const int use_smem = bins <= 12288;
            const size_t smem = use_smem ? sizeof(unsigned int) * bins : 0;
            k_cdf_stats<<<grid_for(nv), 256, smem, st>>>(vb, nv, bins, dedges, use_smem, dc, dc + bins);
            note_launch();
            if ((e = cudaGetLastError())) { fail(e, "k_cdf_stats"); break; }
        }
        unsigned long long hk = 0;
        if ((e = cudaMemcpyAsync(counts_out, dc, sizeof(int64_t) * bins, cudaMemcpyDeviceToHost, st))) { fail(e, "copy"); break; }
        if ((e = cudaMemcpyAsync(&hk, dc + bins, sizeof hk, cudaMemcpyDeviceToHost, st))) { fail(e, "copy"); break; }
        if ((e = cudaStreamSynchronize(st))) { fail(e, "sync"); break; }
        const unsigned long long b = (hk >> 63) ? (hk & 0x7FFFFFFFFFFFFFFFull) : ~hk;
        double ks;
        memcpy(&ks, &b, sizeof ks);
        *ks_out = nv ? ks : NAN;
        *nvals_out = nv;
    } while (0);
    cudaFreeAsync(dX, st);
    cudaFreeAsync(va, st);
    cudaFreeAsync(vb, st);
    cudaFreeAsync(dedges, st);
    cudaFreeAsync(dc, st);
    if (tmp) cudaFreeAsync(tmp, st);
    return rc;
}
