// ctx.cu -- context lifecycle (imx_create / imx_destroy / imx_get_timings)
// and buffer management shared by propagate.cu, memo.cu and celf.cu.
#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "ctx.cuh"

namespace imx {

// Pinned host staging buffers are recycled process-wide: cudaMallocHost is a
// millisecond-scale call, and every run_fused creates a fresh context.
static std::mutex g_pin_mu;
static std::vector<std::pair<void *, size_t>> g_pin_free;

cudaError_t pinned_get(void **p, size_t bytes) {
    {
        // best fit, so small requests do not take the large staging buffers
        std::lock_guard<std::mutex> lk(g_pin_mu);
        size_t best = g_pin_free.size();
        for (size_t i = 0; i < g_pin_free.size(); ++i)
            if (g_pin_free[i].second >= bytes &&
                (best == g_pin_free.size() || g_pin_free[i].second < g_pin_free[best].second))
                best = i;
        if (best < g_pin_free.size()) {
            *p = g_pin_free[best].first;
            g_pin_free.erase(g_pin_free.begin() + best);
            return cudaSuccess;
        }
    }
    return cudaMallocHost(p, bytes);
}

void pinned_put(void *p, size_t bytes) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_pin_mu);
    g_pin_free.emplace_back(p, bytes);
}

// pinned buffers handed to the caller (imx_celf_trace_take) and their sizes
static std::vector<std::pair<void *, size_t>> g_pin_lent;

void pinned_lend(void *p, size_t bytes) {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    g_pin_lent.emplace_back(p, bytes);
}

// The label/count matrices come from the device's stream-ordered pool with an
// unbounded release threshold, so back-to-back runs on the same graph reuse
// the memory instead of paying cudaMalloc/cudaFree every time.
cudaError_t pool_alloc(void **p, size_t bytes, cudaStream_t st) {
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

// Label matrices are the only multi-GB buffers (C4 17 GB, C5 33 GB).  Back-
// to-back runs release one and ask for another of the same size, often on a
// different recycled stream; the stream-ordered pool then sometimes maps
// fresh memory (up to ~0.8 s at 33 GB) instead of reusing the block.  A
// released matrix is kept (one per device) and handed to the next context
// that fits it.
static std::mutex g_lbuf_mu;
struct LBuf { int dev; void *p; size_t bytes; };
static std::vector<LBuf> g_lbuf;

static cudaError_t label_alloc(int dev, void **p, size_t bytes, cudaStream_t st) {
    {
        std::lock_guard<std::mutex> lk(g_lbuf_mu);
        for (size_t i = 0; i < g_lbuf.size(); ++i)
            if (g_lbuf[i].dev == dev && g_lbuf[i].bytes >= bytes && g_lbuf[i].bytes <= 2 * bytes + (64 << 20)) {
                *p = g_lbuf[i].p;
                g_lbuf.erase(g_lbuf.begin() + i);
                return cudaSuccess;
            }
    }
    return pool_alloc(p, bytes, st);
}

static void label_release(int dev, void *p, size_t bytes, cudaStream_t st) {
    if (!p) return;
    if (bytes < ((size_t)256 << 20)) { cudaFreeAsync(p, st); return; }
    cudaStreamSynchronize(st);       // the matrix is idle before anyone else gets it
    std::lock_guard<std::mutex> lk(g_lbuf_mu);
    for (size_t i = 0; i < g_lbuf.size(); ++i)
        if (g_lbuf[i].dev == dev) {   // one kept per device: the newest
            cudaFreeAsync(g_lbuf[i].p, st);
            g_lbuf.erase(g_lbuf.begin() + i);
            break;
        }
    g_lbuf.push_back({dev, p, bytes});
}

void ctx_free(imx_ctx *c) {
    if (!c) return;
    cudaSetDevice(c->dev);
    if (c->st) cudaStreamSynchronize(c->st);
    if (c->L) label_release(c->dev, c->L, c->L_bytes, c->st);
    if (c->C) cudaFreeAsync(c->C, c->st);
    c->L = c->C = nullptr;
    if (c->st) cudaStreamSynchronize(c->st);
    void *ptrs[] = {c->X, c->L, c->C, c->gains, c->inS, c->cov, c->per_sim, c->oid[0], c->oid[1],
                    c->okey[0], c->okey[1], c->scratch, c->eval_out, c->d_one,
                    c->sort_tmp, c->d_ids, c->d_vals, c->seg_a, c->seg_n, c->seg_off, c->scan_tmp,
                    c->scan_xs, c->scan_perm, c->scan_boff, c->scan_ctr,
                    c->cdev, c->skey, c->sid, c->dtrace, c->dseeds, c->dsgains, c->stab, c->hublab, c->g1};
    for (void *p : ptrs) if (p) cudaFreeAsync(p, c->st);
    if (c->st) cudaStreamSynchronize(c->st);
    pinned_put(c->h_ids, sizeof(int32_t) * c->stage_cap);
    pinned_put(c->h_vals, sizeof(int64_t) * c->stage_cap);
    pinned_put(c->trace, sizeof(int64_t) * c->trace_hcap);
    for (auto &e : c->ev) if (e) cudaEventDestroy(e);
    if (c->tst) { cudaStreamSynchronize(c->tst); release_stream(c->dev, c->tst); }
    release_stream(c->dev, c->st);
    delete c;
}

int ensure_celf_buffers(imx_ctx *c) {
    if (c->inS) return IMX_OK;
    const int64_t n = c->g->n > 0 ? c->g->n : 1;
    IMX_CUDA(pool_alloc((void **)&c->inS, n, c->st));
    IMX_CUDA(pool_alloc((void **)&c->cov, sizeof(uint32_t) * (size_t)n * c->cw, c->st));
    IMX_CUDA(pool_alloc((void **)&c->per_sim, sizeof(int64_t) * (c->W + 1), c->st));
    for (int b = 0; b < 2; ++b) {
        IMX_CUDA(pool_alloc((void **)&c->oid[b], sizeof(int32_t) * n, c->st));
        IMX_CUDA(pool_alloc((void **)&c->okey[b], sizeof(unsigned long long) * n, c->st));
    }
    IMX_CUDA(pool_alloc((void **)&c->eval_out, sizeof(int64_t) * (n + 1), c->st));   // + a commit check (celf_prefix)
    IMX_CUDA(pool_alloc((void **)&c->d_one, sizeof(int32_t) * 4, c->st));
    return IMX_OK;
}

int ensure_pinned(imx_ctx *c, int64_t cnt) {
    if (cnt <= c->stage_cap) return IMX_OK;
    int64_t cap = std::max<int64_t>(cnt, 4096);
    IMX_CUDA(cudaStreamSynchronize(c->st));
    pinned_put(c->h_ids, sizeof(int32_t) * c->stage_cap);
    pinned_put(c->h_vals, sizeof(int64_t) * c->stage_cap);
    if (c->d_ids) cudaFreeAsync(c->d_ids, c->st);
    if (c->d_vals) cudaFreeAsync(c->d_vals, c->st);
    c->h_ids = nullptr; c->h_vals = nullptr; c->d_ids = nullptr; c->d_vals = nullptr;
    c->stage_cap = 0;
    IMX_CUDA(cudaStreamSynchronize(c->st));
    IMX_CUDA(pinned_get((void **)&c->h_ids, sizeof(int32_t) * cap));
    IMX_CUDA(pinned_get((void **)&c->h_vals, sizeof(int64_t) * cap));
    IMX_CUDA(pool_alloc((void **)&c->d_ids, sizeof(int32_t) * cap, c->st));
    IMX_CUDA(pool_alloc((void **)&c->d_vals, sizeof(int64_t) * cap, c->st));
    c->stage_cap = cap;
    return IMX_OK;
}


}  // namespace imx

using namespace imx;

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
    // lane tiles (uf.cuh Lay): a very wide label matrix of a graph whose
    // 32-lane slice is L2-sized is stored as [W/64][n][64], so each tile's
    // compression walks (32 lanes at a time) stay in L2 with no copy (C5:
    // n = 1M, 8192 lanes: propagate 84.4 -> 60.2 ms against the copied
    // 32-lane tiles of round 1); IMX_TILE_LANES forces a tile width (power of
    // 2 >= 4; 0 = rows)
    int tsh = 0;
    {
        int tl = 0;
        if (const char *e = getenv("IMX_TILE_LANES")) tl = atoi(e);
        else if (g->n <= ((int64_t)1 << 20) && (double)g->n * c->ld * 4 >= 8e9) tl = 64;
        if (tl >= 4) {
            while ((1 << (tsh + 1)) <= tl) ++tsh;
            const int64_t t = (int64_t)1 << tsh;
            c->ld = (width + t - 1) / t * t;
        }
    }
    c->lay_native = tsh ? imx::Lay::tiles(g->n, tsh) : imx::Lay(c->ld);
    c->lay = c->lay_native;
    c->cw = (num_scored + 31) / 32;
    if (c->cw == 0) c->cw = 1;
    int vb = 1;
    while ((int64_t(1) << vb) < g->n + 1) ++vb;
    c->vb = vb;
    for (auto &e : c->ev) e = nullptr;
    const int64_t n = g->n;
    auto fail = [&](int code) { ctx_free(c); return code; };
    if (acquire_stream(c->dev, &c->st) != cudaSuccess) return fail(IMX_ECUDA);
    for (auto &e : c->ev)
        if (cudaEventCreate(&e) != cudaSuccess) return fail(IMX_ECUDA);
    const size_t cells = (size_t)(n > 0 ? n : 1) * (size_t)c->ld;
    c->L_bytes = sizeof(uint32_t) * cells;
    cudaError_t e = cudaSuccess;
    if ((e = pool_alloc((void **)&c->X, sizeof(int32_t) * c->ld, c->st)) != cudaSuccess ||
        (e = label_alloc(c->dev, (void **)&c->L, sizeof(uint32_t) * cells, c->st)) != cudaSuccess ||
        (e = pool_alloc((void **)&c->gains, sizeof(int64_t) * (n + 1), c->st)) != cudaSuccess ||
        (e = pool_alloc((void **)&c->scratch, sizeof(unsigned long long) * 16, c->st)) != cudaSuccess ||
        (e = cudaMemsetAsync(c->scratch, 0, sizeof(unsigned long long) * 16, c->st)) != cudaSuccess) {
        return fail(cuda_fail(e, "cudaMalloc(context)", __FILE__, __LINE__));
    }
    std::vector<int32_t> xpad(c->ld, 0);
    std::copy(X, X + width, xpad.begin());
    c->hX.assign(X, X + width);
    if ((e = cudaMemcpyAsync(c->X, xpad.data(), sizeof(int32_t) * c->ld, cudaMemcpyHostToDevice, c->st)) != cudaSuccess ||
        (e = cudaStreamSynchronize(c->st)) != cudaSuccess)
        return fail(cuda_fail(e, "upload X", __FILE__, __LINE__));
    *out = c;
    return IMX_OK;
}

extern "C" void imx_destroy(imx_ctx *c) { ctx_free(c); }


extern "C" int imx_get_timings(imx_ctx *c, imx_timings *out) {
    CTX_CHECK(c);
    if (!out) { set_error("out is NULL"); return IMX_EINVAL; }
    settle_timings(c);
    *out = c->tm;
    return IMX_OK;
}

namespace imx {
// grow the pinned host trace buffer to hold at least cnt int64 (keeps content)
// the host trace buffer is complete (an asynchronous big-round copy landed)
int trace_flush(imx_ctx *c) {
    if (c->tst) IMX_CUDA(cudaStreamSynchronize(c->tst));
    return IMX_OK;
}

int trace_reserve(imx_ctx *c, int64_t cnt) {
    if (cnt <= c->trace_hcap) return IMX_OK;
    IMX_TRY(trace_flush(c));         // no copy may still be landing in the old buffer
    const int64_t cap = std::max<int64_t>(cnt, std::max<int64_t>(2 * c->trace_hcap, 1 << 16));
    int64_t *p = nullptr;
    IMX_CUDA(pinned_get((void **)&p, sizeof(int64_t) * cap));
    if (c->trace_n) memcpy(p, c->trace, sizeof(int64_t) * c->trace_n);
    pinned_put(c->trace, sizeof(int64_t) * c->trace_hcap);
    c->trace = p;
    c->trace_hcap = cap;
    return IMX_OK;
}
}  // namespace imx

using namespace imx;

// return a buffer lent by imx_celf_trace_take to the pinned cache
extern "C" void imx_host_free(void *p) {
    if (!p) return;
    size_t bytes = 0;
    {
        std::lock_guard<std::mutex> lk(g_pin_mu);
        for (size_t i = 0; i < g_pin_lent.size(); ++i)
            if (g_pin_lent[i].first == p) {
                bytes = g_pin_lent[i].second;
                g_pin_lent.erase(g_pin_lent.begin() + i);
                break;
            }
    }
    if (bytes) pinned_put(p, bytes);
}
