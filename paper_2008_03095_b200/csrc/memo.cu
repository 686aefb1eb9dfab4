// memo.cu -- K4/K5 memoization: component sizes and int64 gains
// (reference component_sizes_and_gains, propagation.py:349-390), plus label /
// size copies to the host and caller-provided label matrices.
//
// After propagate a root cell already holds its component's member count
// (uf.cuh), so the histogram is free: sizes[l][r] = (cell & COUNT) + 1 for a
// root cell, 0 otherwise, and the gain of v is the sum over the scored lanes
// of the size of v's root -- one coalesced row read plus one gather per
// non-root cell.  Caller labels (imx_load_labels) are arbitrary ids, so they
// get an explicit size array C[n][ld] (template ENC = false).
#include <algorithm>
#include <vector>

#include "ctx.cuh"
#include "uf.cuh"

namespace imx {

// gains[v] = sum_{r < ns} size(comp(v, r))   (propagation.py:359-368)
// Caller-label mode: warp per vertex, sizes from C.
__global__ void __launch_bounds__(256) k_gains_caller(const uint32_t *__restrict__ L, const uint32_t *__restrict__ C,
                                                      int64_t n, int64_t ld, int32_t ns,
                                                      int64_t *__restrict__ gains) {
    const int lane = threadIdx.x & 31;
    const int nqs = (ns + 3) >> 2;
    const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t v = wg; v < n; v += nw) {
        const uint4 *Lr = reinterpret_cast<const uint4 *>(L + v * ld);
        unsigned long long acc = 0;
        for (int q = lane; q < nqs; q += 32) {
            const uint4 l = __ldg(Lr + q);
            const uint32_t w[4] = {l.x, l.y, l.z, l.w};
            const int r = q << 2;
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (r + j < ns) acc += __ldg(C + (int64_t)w[j] * ld + r + j);
        }
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) gains[v] = (int64_t)acc;
    }
}

// Encoded labels: warp per vertex, 16-byte quads of its row; the size of a
// non-root cell's component is gathered from its root's cell through the
// read-only path (L is not written during memoization, so hub rows stay in
// L1/texture cache instead of hammering one L2 line).
// An isolated vertex (no slot in xadj) is its own component in every lane:
// its gain is ns without reading its row (C4: 44% of the rows).
//
// First-seed speculation (hublab != NULL): CELF's round 0 commits the vertex
// with the largest gain, and on skewed graphs that is the vertex with the
// most neighbours.  While v's row is here anyway, g1[v] = gains[v] - (sizes of
// v's components that contain that vertex) is v's exact marginal gain after
// that first seed, so round 1 -- which re-evaluates most candidates (C4:
// 2.3 M rows, 9.5 GB) -- reads one word per candidate instead of its row.  If
// the first seed turns out to be another vertex, g1 is not used.
template <bool G1>
__global__ void __launch_bounds__(256, G1 ? 5 : 1) k_gains_enc(const uint32_t *__restrict__ L, int64_t n, Lay y,
                                                   int32_t ns, int64_t *__restrict__ gains,
                                                   const int64_t *__restrict__ xadj,
                                                   const int32_t *__restrict__ hublab, int64_t *__restrict__ g1) {
    const int lane = threadIdx.x & 31;
    const int nqs = (ns + 3) >> 2;
    const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t v = wg; v < n; v += nw) {
        if (xadj && xadj[v + 1] == xadj[v]) {
            if (lane == 0) {
                gains[v] = ns;
                if (G1) g1[v] = ns;
            }
            continue;
        }
        unsigned long long acc = 0, acc1 = 0;
        // two quads per step, all eight root gathers issued before any is used
        for (int q0 = lane; q0 < nqs; q0 += 64) {
            uint32_t w[8];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int q = q0 + 32 * h;
                const uint4 l = q < nqs ? row_quad(L, y, v, q) : make_uint4(ROOT, ROOT, ROOT, ROOT);
                w[4 * h] = l.x; w[4 * h + 1] = l.y; w[4 * h + 2] = l.z; w[4 * h + 3] = l.w;
            }
            uint32_t rw[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int r = ((q0 + 32 * (k >> 2)) << 2) + (k & 3);
                rw[k] = is_root(w[k]) ? w[k] : __ldg(L + cell_off(y, w[k], r));
            }
            if (G1) {
                // the lanes' labels as 16-byte quads like the row (hublab has ld entries)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int q = q0 + 32 * h;
                    if (q < nqs) {
                        const int4 hq = __ldg(reinterpret_cast<const int4 *>(hublab) + q);
                        const uint32_t hl[4] = {(uint32_t)hq.x, (uint32_t)hq.y, (uint32_t)hq.z, (uint32_t)hq.w};
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const int k = 4 * h + j;
                            const uint32_t lab = is_root(w[k]) ? (uint32_t)v : w[k];
                            if (4 * q + j < ns && hl[j] == lab) acc1 += (rw[k] & COUNT) + 1u;
                        }
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int r = ((q0 + 32 * (k >> 2)) << 2) + (k & 3);
                if (r < ns) acc += (rw[k] & COUNT) + 1u;
            }
        }
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (G1)
            for (int o = 16; o; o >>= 1) acc1 += __shfl_xor_sync(0xffffffffu, acc1, o);
        if (lane == 0) {
            gains[v] = (int64_t)acc;
            if (G1) g1[v] = (int64_t)(acc - acc1);
        }
    }
}

// the vertex with the most slots (ties: the smallest id) as a packed key
__global__ void k_hub_degree(const int64_t *__restrict__ xadj, int64_t n, unsigned long long *__restrict__ key) {
    unsigned long long best = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long k = ((unsigned long long)(xadj[v + 1] - xadj[v]) << 32) | (0xffffffffull - (uint32_t)v);
        best = k > best ? k : best;
    }
    for (int o = 16; o; o >>= 1) {
        const unsigned long long x = __shfl_xor_sync(0xffffffffu, best, o);
        best = x > best ? x : best;
    }
    if ((threadIdx.x & 31) == 0 && best) atomicMax(key, best);
}
// its label in every lane (compressed matrix), the vertex itself in hub_out
__global__ void k_hub_labels(const uint32_t *__restrict__ L, Lay y, int64_t ld, const unsigned long long *__restrict__ key,
                             int32_t *__restrict__ hublab, unsigned long long *__restrict__ hub_out) {
    const uint32_t hub = 0xffffffffu - (uint32_t)(*key & 0xffffffffull);
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < ld; r += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t w = L[y.off(hub, (int)r)];
        hublab[r] = (int32_t)(is_root(w) ? hub : w);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *hub_out = hub;
}

// Gains of one compressed lane tile T[n][tld] (lanes l0.. of the matrix, the
// first ns_t of them scored), while the tile is still in L2 (the tiled
// compression of propagate.cu, when the caller fused the memo into it): 8
// threads per row, a thread per 16-byte quad, root gathers inside the tile;
// gains[v] = (first tile ? 0 : gains[v]) + the row's tile sum.
__global__ void __launch_bounds__(256) k_gains_tile(const uint32_t *__restrict__ T, int64_t n, int64_t tld,
                                                    int32_t ns_t, int first, int64_t *__restrict__ gains) {
    const int64_t nthreads = n * 8;
    const int nqr = (int)(tld >> 2);
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x; i0 < nthreads; i0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = i0 + threadIdx.x;
        const int64_t v = i >> 3;
        unsigned long long acc = 0;
        // 8 threads per row, each a quad of lanes every 8 quads
        for (int q = (int)(i & 7); i < nthreads && q < nqr && 4 * q < ns_t; q += 8) {
            const uint4 l = __ldg(reinterpret_cast<const uint4 *>(T + v * tld) + q);
            const uint32_t w[4] = {l.x, l.y, l.z, l.w};
            uint32_t rw[4];
#pragma unroll
            for (int k = 0; k < 4; ++k)
                rw[k] = (is_root(w[k]) || 4 * q + k >= ns_t) ? w[k] : __ldg(T + (int64_t)w[k] * tld + 4 * q + k);
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (4 * q + k < ns_t) acc += (rw[k] & COUNT) + 1u;
        }
#pragma unroll
        for (int o = 4; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (i < nthreads && (i & 7) == 0) gains[v] = (first ? 0 : gains[v]) + (int64_t)acc;
    }
}

int launch_gains_tile(const uint32_t *T, int64_t n, int64_t tld, int32_t ns_t, int first, int64_t *gains,
                      cudaStream_t st) {
    if (n == 0) return IMX_OK;
    const char *e = getenv("IMX_GAINS_TILE_BPSM");
    const int64_t bpsm = e && atoi(e) > 0 ? atoi(e) : 16;
    const int gb = (int)std::min<int64_t>(ceil_div(n * 8, 256), 148 * bpsm);
    k_gains_tile<<<gb, 256, 0, st>>>(T, n, tld, ns_t, first, gains);
    IMX_CHECK_LAUNCH();
    note_launch();
    return IMX_OK;
}

// decoded labels / sizes of rows [v0, v0+cnt), lanes [r0, r1) -> dense out
template <bool ENC>
__global__ void k_labels_window(const uint32_t *__restrict__ L, int64_t v0, int64_t cnt, Lay y,
                                int32_t r0, int32_t r1, int32_t *__restrict__ out) {
    const int w = r1 - r0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt * (int64_t)w;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = v0 + i / w;
        const int r = r0 + (int)(i % w);
        const uint32_t x = L[y.off(v, r)];
        out[i] = (int32_t)(ENC ? label_of((uint32_t)v, x) : x);
    }
}
template <bool ENC>
__global__ void k_sizes_window(const uint32_t *__restrict__ L, const uint32_t *__restrict__ C,
                               int64_t v0, int64_t cnt, Lay y, int32_t r0, int32_t r1,
                               int32_t *__restrict__ out) {
    const int w = r1 - r0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt * (int64_t)w;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = v0 + i / w;
        const int r = r0 + (int)(i % w);
        if (ENC) {
            const uint32_t x = L[y.off(v, r)];
            out[i] = is_root(x) ? (int32_t)((x & COUNT) + 1u) : 0;
        } else {
            out[i] = (int32_t)C[y.off(v, r)];
        }
    }
}

// full histogram of caller labels (component_sizes, propagation.py:349-356)
// sizes of caller labels: a thread per (32-row chunk, lane), the chunk's rows
// walked in order with a run-length count per lane, so a run of equal labels
// (hub components: label 0 in most rows of most lanes) costs one atomic
// instead of one per cell; loads stay coalesced (consecutive threads,
// consecutive lanes of the same row)
constexpr int kHistRows = 32;
__global__ void k_hist_full(const uint32_t *__restrict__ L, uint32_t *__restrict__ C, int64_t n, int64_t ld,
                            int32_t W, unsigned *__restrict__ bad) {
    const int64_t chunks = (n + kHistRows - 1) / kHistRows;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < chunks * (int64_t)W;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t ch = i / W;
        const int r = (int)(i - ch * W);
        const int64_t v1 = (ch + 1) * kHistRows < n ? (ch + 1) * kHistRows : n;
        uint32_t cur = 0, cnt = 0;
        for (int64_t v = ch * kHistRows; v < v1; ++v) {
            const uint32_t l = L[v * ld + r];
            if (l >= (uint32_t)n) { atomicOr(bad, 1u); continue; }
            if (l != cur && cnt) { atomicAdd(C + (int64_t)cur * ld + r, cnt); cnt = 0; }
            cur = l;
            ++cnt;
        }
        if (cnt) atomicAdd(C + (int64_t)cur * ld + r, cnt);
    }
}

// caller labels with caller sizes: every label in 0..n-1 and every size >= 0
// (the reference raises IndexError on a bad label, selection.py:63-81)
__global__ void k_check_loaded(const uint32_t *__restrict__ L, const uint32_t *__restrict__ C, int64_t n,
                               int64_t ld, int32_t W, unsigned *__restrict__ bad) {
    unsigned b = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * (int64_t)W;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = i / W;
        const int r = (int)(i - v * W);
        b |= L[v * ld + r] >= (uint32_t)n ? 1u : 0u;
        b |= (C[v * ld + r] & 0x80000000u) ? 2u : 0u;
    }
    if (b) atomicOr(bad, b);
}

// copy rows of a decoded window out through a device staging buffer
template <class Launch>
static int copy_window(imx_ctx *c, int32_t r0, int32_t r1, int32_t *out, Launch launch) {
    const int64_t n = c->g->n;
    const int w = r1 - r0;
    int64_t rows = std::max<int64_t>(1, (int64_t(256) << 20) / (4 * (int64_t)w));
    rows = std::min(rows, n);
    int32_t *tmp;
    IMX_CUDA(cudaMallocAsync((void **)&tmp, sizeof(int32_t) * rows * w, c->st));
    int rc = IMX_OK;
    for (int64_t v0 = 0; v0 < n && rc == IMX_OK; v0 += rows) {
        const int64_t cnt = std::min(rows, n - v0);
        launch(v0, cnt, tmp);
        cudaError_t e = cudaGetLastError();
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(out + v0 * w, tmp, sizeof(int32_t) * cnt * w, cudaMemcpyDeviceToHost, c->st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(c->st);
        if (e != cudaSuccess) rc = cuda_fail(e, "copy window", __FILE__, __LINE__);
        count_launch(c);
    }
    cudaFreeAsync(tmp, c->st);
    return rc;
}

}  // namespace imx

using namespace imx;

extern "C" int imx_memoize(imx_ctx *c, int64_t *gains_out) {
    CTX_CHECK(c);
    if (gains_out) IMX_TRY(spec_guard(c));
    if (!c->labels_ready) { set_error("labels not computed (call imx_propagate first)"); return IMX_EINVAL; }
    const int64_t n = c->g->n;
    c->g1_ready = false;
    IMX_CUDA(cudaEventRecord(c->ev[4], c->st));
    if (n && c->gains_fused && !c->C) {
        // already summed by the tiled compression of the last propagate
    } else if (n) {
        if (c->C) {
            k_gains_caller<<<grid_for(n * 32), 256, 0, c->st>>>(c->L, c->C, n, c->ld, c->ns, c->gains);
        } else {
            {
                // a warp per vertex, up to 64 blocks per SM (C4 3.83 -> 3.49 ms
                // against 16; C3 0.443 -> 0.430 ms)
                const char *mg = getenv("IMX_MEMO_BPSM");
                const int gb = (int)std::min<int64_t>(ceil_div(n * 32, 256), 148 * (mg && atoi(mg) > 0 ? atoi(mg) : 64));
                // first-seed speculation for the CELF loop of this rank alone
                const bool spec1 = c->g->m2 > 0 && !c->comm && !getenv("IMX_MEMO_NO_G1");
                if (spec1) {
                    if (!c->g1) {
                        IMX_CUDA(pool_alloc((void **)&c->g1, sizeof(int64_t) * n, c->st));
                        IMX_CUDA(pool_alloc((void **)&c->hublab, sizeof(int32_t) * c->ld, c->st));
                    }
                    IMX_CUDA(cudaMemsetAsync(c->scratch + 14, 0, sizeof(unsigned long long), c->st));
                    k_hub_degree<<<grid_for(n), 256, 0, c->st>>>(c->g->xadj, n, c->scratch + 14);
                    k_hub_labels<<<grid_for(c->ld), 256, 0, c->st>>>(c->L, c->lay, c->ld, c->scratch + 14, c->hublab,
                                                                   c->scratch + 15);
                    count_launch(c, 2);
                }
                if (spec1)
                    k_gains_enc<true><<<gb, 256, 0, c->st>>>(c->L, n, c->lay, c->ns, c->gains, c->g->xadj, c->hublab, c->g1);
                else
                    k_gains_enc<false><<<gb, 256, 0, c->st>>>(c->L, n, c->lay, c->ns, c->gains,
                                                              c->g->m2 ? c->g->xadj : nullptr, nullptr, nullptr);
                c->g1_ready = spec1;
            }
        }
        IMX_CHECK_LAUNCH();
        count_launch(c);
    }
    // ranks of a sharded run: the gains are sums over every rank's lanes
    if (c->comm && n) IMX_TRY(comm_allreduce_i64(c->comm, c->gains, n, c->st));
    IMX_CUDA(cudaEventRecord(c->ev[5], c->st));
    c->tm_pending |= 2;             // memoize_ms is read when the timings are asked for
    if (gains_out && n) {
        IMX_CUDA(cudaMemcpyAsync(gains_out, c->gains, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, c->st));
        IMX_CUDA(cudaStreamSynchronize(c->st));
    }
    c->memo_ready = true;
    return IMX_OK;
}

extern "C" int imx_load_labels(imx_ctx *c, const int32_t *labels, const int32_t *sizes, int64_t ldh) {
    CTX_CHECK(c);
    c->gains_fused = false;
    const int64_t n = c->g->n;
    if (!labels && n) { set_error("labels is NULL"); return IMX_EINVAL; }
    if (ldh < c->W) { set_error("row stride %lld < width %d", (long long)ldh, c->W); return IMX_EINVAL; }
    if (!c->C) IMX_CUDA(pool_alloc((void **)&c->C, sizeof(uint32_t) * (size_t)(n > 0 ? n : 1) * c->ld, c->st));
    c->lay = Lay(c->ld);             // caller labels and sizes: rows
    if (n) {
        const size_t bytes = sizeof(uint32_t) * (size_t)n * c->ld;
        IMX_CUDA(cudaMemsetAsync(c->L, 0, bytes, c->st));
        IMX_CUDA(cudaMemcpy2DAsync(c->L, sizeof(uint32_t) * c->ld, labels, sizeof(int32_t) * ldh,
                                   sizeof(int32_t) * c->W, n, cudaMemcpyHostToDevice, c->st));
        unsigned *bad = reinterpret_cast<unsigned *>(c->scratch + 6);
        IMX_CUDA(cudaMemsetAsync(bad, 0, sizeof(unsigned), c->st));
        IMX_CUDA(cudaMemsetAsync(c->C, 0, bytes, c->st));
        if (sizes) {
            IMX_CUDA(cudaMemcpy2DAsync(c->C, sizeof(uint32_t) * c->ld, sizes, sizeof(int32_t) * ldh,
                                       sizeof(int32_t) * c->W, n, cudaMemcpyHostToDevice, c->st));
            k_check_loaded<<<grid_for(n * c->W), 256, 0, c->st>>>(c->L, c->C, n, c->ld, c->W, bad);
            IMX_CHECK_LAUNCH();
            count_launch(c);
        } else {
            k_hist_full<<<grid_for(ceil_div(n, kHistRows) * c->W), 256, 0, c->st>>>(c->L, c->C, n, c->ld, c->W, bad);
            IMX_CHECK_LAUNCH();
            count_launch(c);
        }
        unsigned hb = 0;
        IMX_CUDA(cudaMemcpyAsync(&hb, bad, sizeof hb, cudaMemcpyDeviceToHost, c->st));
        IMX_CUDA(cudaStreamSynchronize(c->st));
        if (hb) {
            c->labels_ready = false;
            set_error(hb & 1u ? "label outside 0..n-1" : "negative component size");
            return IMX_EINVAL;
        }
    }
    c->labels_ready = true;
    c->memo_ready = false;
    c->celf_ready = false;
    return IMX_OK;
}

extern "C" int imx_copy_labels(imx_ctx *c, int32_t r0, int32_t r1, int32_t *out) {
    CTX_CHECK(c);
    IMX_TRY(spec_guard(c));
    if (r0 < 0 || r1 > c->W || r0 > r1) { set_error("lane window [%d, %d) invalid", r0, r1); return IMX_EINVAL; }
    if (!c->labels_ready) { set_error("labels not computed"); return IMX_EINVAL; }
    if (c->g->n == 0 || r1 == r0) return IMX_OK;
    const bool enc = c->C == nullptr;
    return copy_window(c, r0, r1, out, [&](int64_t v0, int64_t cnt, int32_t *tmp) {
        if (enc) k_labels_window<true><<<grid_for(cnt * (r1 - r0)), 256, 0, c->st>>>(c->L, v0, cnt, c->lay, r0, r1, tmp);
        else k_labels_window<false><<<grid_for(cnt * (r1 - r0)), 256, 0, c->st>>>(c->L, v0, cnt, c->lay, r0, r1, tmp);
    });
}

extern "C" int imx_copy_sizes(imx_ctx *c, int32_t r0, int32_t r1, int32_t *out) {
    CTX_CHECK(c);
    IMX_TRY(spec_guard(c));
    if (r0 < 0 || r1 > c->W || r0 > r1) { set_error("lane window [%d, %d) invalid", r0, r1); return IMX_EINVAL; }
    if (!c->labels_ready) { set_error("labels not computed"); return IMX_EINVAL; }
    if (c->g->n == 0 || r1 == r0) return IMX_OK;
    const bool enc = c->C == nullptr;
    return copy_window(c, r0, r1, out, [&](int64_t v0, int64_t cnt, int32_t *tmp) {
        if (enc) k_sizes_window<true><<<grid_for(cnt * (r1 - r0)), 256, 0, c->st>>>(c->L, nullptr, v0, cnt, c->lay, r0, r1, tmp);
        else k_sizes_window<false><<<grid_for(cnt * (r1 - r0)), 256, 0, c->st>>>(c->L, c->C, v0, cnt, c->lay, r0, r1, tmp);
    });
}
