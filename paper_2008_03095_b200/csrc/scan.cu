// scan.cu -- sampler "scan": the pull forest with lanes bucketed by the top
// bits of their simulation word (uniform thresholds).
//
// Membership of edge slot s in lane r is (X[r] ^ h_s) < t (hashing.py:141-150,
// strict, 31-bit words).  With t <= 2^k, (x ^ h) < t forces x >> k == h >> k,
// so for a slot with hash h only the lanes whose word shares h's top 31-k
// bits can be live: C4 (t = 0.005 * 2^31 < 2^24) keeps 1 lane in 128, C5
// (p = 0.05) 1 in 16.  At context setup the lanes of every chunk of <= 1024
// lanes are sorted by x >> kb (kb >= k) into buckets; a slot then tests only
// its bucket's lanes instead of all of them -- the reference's _xor_below
// interval idea (propagation.py:104-118) applied to the lane side, so the
// adjacency is still read once per row and reused across every lane.
//
// Pass 1 (replaces k_init): a warp owns a vertex row.  It stages the row of
// the chunk in shared memory (all ROOT), walks v's smaller-neighbour prefix
// in ascending order (rows are sorted, graph.py:149), and for every live
// (slot, lane) keeps the first -- i.e. smallest -- live smaller neighbour:
// L[v][r] = that neighbour (a parent pointer to a smaller id) or ROOT.  The
// row is then written with 16-byte coalesced stores: a forest of live edges,
// no random access.
// Pass 2: the same walk; every live pair that is not its lane's first live
// neighbour (the forest edge) is united through a per-warp shared-memory
// queue (uf.cuh unite), 32 unions at a time.
// Heavy rows (prefix > T slots) are cut into slices of T slots, one warp
// each.  Pass 1 leaves them all ROOT (the light pass writes the row) and pass 2
// unites every live neighbour; optionally (IMX_SCAN_HEAVY_P1) pass 1 folds the
// slices' first live neighbours into the row with atomicMin and pass 2 skips
// the neighbour the row points at.
//
// Correctness does not depend on the buckets: a bucket is a superset of the
// live lanes and every candidate is re-tested exactly.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "ctx.cuh"
#include "uf.cuh"

namespace imx {

constexpr int kScanCW = 1024;        // lanes per chunk: a 4 KB shared row per warp
constexpr int kScanWarps = 8;
constexpr int kScanQ = 64;           // per-warp union queue: drain at 32, one step adds <= 32
constexpr int kScanMaxBucketBits = 10;

template <int PASS, bool HEAVY>
__global__ void __launch_bounds__(kScanWarps * 32)
k_scan(const int64_t *__restrict__ xadj, const int32_t *__restrict__ adj, const int32_t *__restrict__ hash,
       int32_t t, int kb, int nb, int cw, int nchunks, const int32_t *__restrict__ xs_all,
       const uint16_t *__restrict__ perm_all, const int32_t *__restrict__ boff_all, int64_t n, int32_t W,
       int64_t ld, Lay y, uint32_t *__restrict__ L, unsigned long long *__restrict__ hooks,
       const uint8_t *__restrict__ heavy, const int32_t *__restrict__ hs_v, const int64_t *__restrict__ hs_a,
       const int32_t *__restrict__ hs_len, int64_t nhs, unsigned long long *__restrict__ ctr, int grab,
       int64_t row0, int iso_pass, int heavy_forest) {
    extern __shared__ int4 smem4[];
    // 16-byte aligned sections (run_scan sizes them): per-warp first-live
    // flags, per-warp union queues (pass 2), the chunk's lane tables
    uint8_t *flags_all = reinterpret_cast<uint8_t *>(smem4);                   // [warps][cw]
    uint32_t *queues = reinterpret_cast<uint32_t *>(flags_all + kScanWarps * cw);   // [warps][3][kScanQ]
    // the chunk's lanes sorted by bucket as (word, lane) pairs, and every
    // bucket's [lo, hi): one 8-byte shared load each
    int2 *sx2 = reinterpret_cast<int2 *>(queues + (PASS == 2 ? kScanWarps * 3 * kScanQ : 0));   // [cw]
    int2 *sbb = sx2 + cw;                                                        // [nb]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t *flag = flags_all + warp * cw;
    uint32_t *qlo = queues + warp * 3 * kScanQ, *qhi = qlo + kScanQ, *qr = qhi + kScanQ;
    const unsigned FULL = 0xffffffffu;
    const unsigned lt_mask = (1u << lane) - 1u;
    int qn = 0;
    unsigned long long nh = 0;
    // light rows: [row0, row0 + n) (a chunk of a streamed CSR; otherwise row0 = 0)
    const int64_t items = HEAVY ? nhs : n;
    for (int c = 0; c < nchunks; ++c) {
        const int r0 = c * cw;
        // row cells of this chunk; the last chunk also covers the row padding
        const int rwc = (int)(c == nchunks - 1 ? ld - r0 : min((int64_t)cw, ld - r0));
        __syncthreads();
        for (int i = threadIdx.x; i < cw; i += blockDim.x)
            sx2[i] = make_int2(xs_all[(int64_t)c * cw + i], (int)perm_all[(int64_t)c * cw + i]);
        for (int i = threadIdx.x; i < nb; i += blockDim.x)
            sbb[i] = make_int2(boff_all[(int64_t)c * (nb + 1) + i], boff_all[(int64_t)c * (nb + 1) + i + 1]);
        __syncthreads();
        for (;;) {
            // dynamic distribution: rows differ by orders of magnitude in
            // prefix length, so warps take small batches from a counter
            unsigned long long base = 0;
            if (lane == 0) base = atomicAdd(ctr + c, (unsigned long long)grab);
            base = __shfl_sync(FULL, base, 0);
            if ((int64_t)base >= items) break;
            const int cntv = (int)(min((int64_t)base + grab, items) - (int64_t)base);
            // the grab's row bounds in one coalesced load (light rows); the
            // next row's first slot batch is loaded while this row is worked
            int64_t xa = 0;
            bool hv_l = false;
            if (!HEAVY) {
                if (lane <= cntv) xa = __ldg(xadj + row0 + base + lane);
                if (heavy && lane < cntv) hv_l = heavy[row0 + base + lane] != 0;
            }
            const unsigned hmask = __ballot_sync(FULL, hv_l);
            // isolated rows (no slot at all: 44% of C4's) are all ROOT and nothing
            // reads them before the compression, so either pass can write them
            // (iso_pass): pass 2's light launch is latency-bound with HBM bandwidth
            // to spare while pass 1 is bound by its row stores (C4: 19.5 GB, of which
            // 7.5 GB isolated) -- unless pass 1 runs hidden behind the upload of a
            // streamed CSR, where the stores cost nothing
            const int64_t xa_next = __shfl_down_sync(FULL, xa, 1);      // every lane takes part
            const unsigned imask = HEAVY ? 0u : __ballot_sync(FULL, lane < cntv && xa == xa_next);
            auto bounds = [&](int k, int64_t &v, int64_t &s0, int64_t &s1) {
                if (HEAVY) {
                    v = hs_v[base + k];
                    s0 = hs_a[base + k];
                    s1 = s0 + hs_len[base + k];
                } else {
                    v = row0 + (int64_t)base + k;
                    s0 = __shfl_sync(FULL, xa, k);
                    s1 = __shfl_sync(FULL, xa, k + 1);
                    if ((hmask >> k) & 1u) s1 = s0;        // heavy row: ROOT here, slices below
                }
            };
            auto batch = [&](int64_t b0, int64_t s1, int64_t v, uint32_t &bu, int32_t &bh) {
                const int64_t sb = b0 + lane;
                bu = (uint32_t)v;
                bh = 0;
                if (sb < s1) {
                    bu = (uint32_t)__ldg(adj + sb);
                    bh = __ldg(hash + sb);
                }
            };
            int64_t v, s0, s1;
            uint32_t bu0;
            int32_t bh0;
            bounds(0, v, s0, s1);
            batch(s0, s1, v, bu0, bh0);
            for (int k = 0; k < cntv; ++k) {
                int64_t nv = 0, ns0 = 0, ns1 = 0;
                uint32_t nbu = 0;
                int32_t nbh = 0;
                // pass 1 prefetches the next row's first batch; pass 2 keeps
                // its registers for the unions (prefetching there measured
                // slower: C5 pass 2 15.8 -> 21.3 ms)
                if (PASS == 1 && k + 1 < cntv) {
                    bounds(k + 1, nv, ns0, ns1);
                    batch(ns0, ns1, nv, nbu, nbh);
                }
                if (PASS == 2 && k > 0) {
                    bounds(k, v, s0, s1);
                    batch(s0, s1, v, bu0, bh0);
                }
                // the row starts as all roots (an isolated one: in pass 2)
                if (!HEAVY && (((imask >> k) & 1u) ? PASS == iso_pass : PASS == 1)) {
                    for (int q = lane; q < (rwc >> 2); q += 32)
                        *reinterpret_cast<uint4 *>(L + y.off(v, r0 + 4 * q)) = make_uint4(ROOT, ROOT, ROOT, ROOT);
                }
                // any smaller neighbour (rows ascend: the first slot says)
                const bool has = s0 < s1 && __shfl_sync(FULL, bu0, 0) < (uint32_t)v;
                if (has) {
                if (PASS == 1 || !HEAVY) {
                    uint4 *f4 = reinterpret_cast<uint4 *>(flag);
                    for (int q = lane; q < (cw >> 4); q += 32) f4[q] = make_uint4(0, 0, 0, 0);
                }
                __syncwarp();
                for (int64_t b0 = s0; b0 < s1; b0 += 32) {
                    uint32_t bu = bu0;
                    int32_t bh = bh0;
                    if (b0 != s0) batch(b0, s1, v, bu, bh);
                    // rows ascend: the smaller neighbours are a prefix of the batch
                    const int cnt = __popc(__ballot_sync(FULL, bu < (uint32_t)v));
                    if (HEAVY) {
                        // heavy slices: both passes are order-free (atomicMin into the
                        // row; "all but the forest edge"), so four slots go at once,
                        // eight threads each (buckets hold ~8 lanes: C4)
                        const int sg = lane >> 3, sl = lane & 7;
                        for (int j0 = 0; j0 < cnt; j0 += 4) {
                            const int j = j0 + sg;
                            const bool has = j < cnt;
                            const uint32_t u = __shfl_sync(FULL, bu, has ? j : 0);
                            const int32_t h = __shfl_sync(FULL, bh, has ? j : 0);
                            int lo = 0, hi = 0;
                            if (has) {
                                const int2 bb = sbb[(uint32_t)h >> kb];
                                lo = bb.x;
                                hi = bb.y;
                            }
                            const int its = __reduce_max_sync(FULL, (unsigned)((hi - lo + 7) >> 3));
                            for (int it = 0; it < its; ++it) {
                                const int i = lo + (it << 3) + sl;
                                const int2 xp = i < hi ? sx2[i] : make_int2(0x7fffffff, 0);
                                const bool live = i < hi && (xp.x ^ h) < t;
                                const int p = live ? xp.y : 0;
                                if (PASS == 1) {
                                    if (live && !flag[p]) {       // a racing duplicate only repeats the min
                                        flag[p] = 1;
                                        atomicMin(L + y.off(v, r0 + p), u);
                                    }
                                } else {
                                    // all but the forest edge of heavy pass 1 -- or all, when that pass was skipped
                                    const bool un = live && (!heavy_forest || ld_relaxed(L + y.off(v, r0 + p)) != u);
                                    const unsigned b = __ballot_sync(FULL, un);
                                    if (b) {
                                        if (un) {
                                            const int pos = qn + __popc(b & lt_mask);
                                            qlo[pos] = u;
                                            qhi[pos] = (uint32_t)v;
                                            qr[pos] = (uint32_t)(r0 + p);
                                        }
                                        qn += __popc(b);
                                        __syncwarp();
                                        if (qn >= 32) {
                                            qn -= 32;
                                            const uint32_t a2 = qlo[qn + lane], b2 = qhi[qn + lane];
                                            const int rr = (int)qr[qn + lane];
                                            __syncwarp();
                                            nh += unite(L, y, a2, b2, rr);
                                        }
                                    }
                                }
                            }
                            __syncwarp();
                        }
                        if (cnt < 32) break;
                        continue;
                    }
                    for (int j = 0; j < cnt; ++j) {
                        const uint32_t u = __shfl_sync(FULL, bu, j);
                        const int32_t h = __shfl_sync(FULL, bh, j);
                        const int bk = (int)((uint32_t)h >> kb);
                        const int2 bb = sbb[bk];
                        const int lo = bb.x, hi = bb.y;
                        for (int i0 = lo; i0 < hi; i0 += 32) {
                            const int i = i0 + lane;
                            const int2 xp = i < hi ? sx2[i] : make_int2(0x7fffffff, 0);
                            const bool live = i < hi && (xp.x ^ h) < t;
                            const int p = live ? xp.y : 0;
                            if (PASS == 1) {
                                // ascending slots: the first live neighbour is the smallest
                                if (live && !flag[p]) {
                                    flag[p] = 1;
                                    if (HEAVY) atomicMin(L + y.off(v, r0 + p), u);
                                    else L[y.off(v, r0 + p)] = u;
                                }
                            } else {
                                bool un = false;
                                if (live) {
                                    if (HEAVY) {
                                        un = !heavy_forest || ld_relaxed(L + y.off(v, r0 + p)) != u;   // all but the forest edge
                                    } else {
                                        un = flag[p] != 0;              // all but the first live neighbour
                                        flag[p] = 1;
                                    }
                                }
                                const unsigned b = __ballot_sync(FULL, un);
                                if (b) {                            // most live pairs are forest edges
                                    if (un) {
                                        const int pos = qn + __popc(b & lt_mask);
                                        qlo[pos] = u;
                                        qhi[pos] = (uint32_t)v;
                                        qr[pos] = (uint32_t)(r0 + p);
                                    }
                                    qn += __popc(b);
                                    __syncwarp();
                                    if (qn >= 32) {
                                        qn -= 32;
                                        const uint32_t a2 = qlo[qn + lane], b2 = qhi[qn + lane];
                                        const int rr = (int)qr[qn + lane];
                                        __syncwarp();
                                        nh += unite(L, y, a2, b2, rr);
                                    }
                                }
                            }
                        }
                        __syncwarp();
                    }
                    if (cnt < 32) break;                   // the prefix ended inside this batch
                }
                }
                if (PASS == 1) { v = nv; s0 = ns0; s1 = ns1; bu0 = nbu; bh0 = nbh; }
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

// ---- host side ---------------------------------------------------------------

// bucket shift for threshold t: smallest k with t <= 2^k, raised so that
// there are at most 2^kScanMaxBucketBits buckets
static int scan_kb(int32_t t) {
    int k = 0;
    while (k < 31 && ((int64_t)1 << k) < (int64_t)t) ++k;
    return std::max(k, 31 - kScanMaxBucketBits);
}

bool scan_eligible(const imx_graph *g) {
    if (const char *e = getenv("IMX_SCAN")) if (!atoi(e)) return false;
    return g->uniform && !g->hash_neg && g->thr_u > 0;
}

// the per-chunk lane tables for this context's X and the graph's threshold
static int ensure_scan_tables(imx_ctx *c) {
    const int kb = scan_kb(c->g->thr_u);
    if (c->scan_xs && c->scan_kb == kb) return IMX_OK;
    for (void **p : {(void **)&c->scan_xs, (void **)&c->scan_perm, (void **)&c->scan_boff}) {
        if (*p) cudaFreeAsync(*p, c->st);
        *p = nullptr;
    }
    const int cw = std::min<int>(kScanCW, (c->W + 15) & ~15);
    const int nchunks = (c->W + cw - 1) / cw;
    const int nb = 1 << (31 - kb);
    std::vector<int32_t> xs((size_t)nchunks * cw, 0), boff((size_t)nchunks * (nb + 1), 0);
    std::vector<uint16_t> perm((size_t)nchunks * cw, 0);
    for (int ch = 0; ch < nchunks; ++ch) {
        const int r0 = ch * cw, cnt = std::min(cw, c->W - r0);
        std::vector<int> idx(cnt);
        for (int i = 0; i < cnt; ++i) idx[i] = i;
        std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) {
            return ((uint32_t)c->hX[r0 + a] >> kb) < ((uint32_t)c->hX[r0 + b] >> kb);
        });
        int32_t *bo = boff.data() + (size_t)ch * (nb + 1);
        for (int i = 0; i < cnt; ++i) {
            xs[(size_t)ch * cw + i] = c->hX[r0 + idx[i]];
            perm[(size_t)ch * cw + i] = (uint16_t)idx[i];
            ++bo[((uint32_t)c->hX[r0 + idx[i]] >> kb) + 1];
        }
        for (int b = 0; b < nb; ++b) bo[b + 1] += bo[b];
    }
    IMX_CUDA(pool_alloc((void **)&c->scan_xs, sizeof(int32_t) * xs.size(), c->st));
    IMX_CUDA(pool_alloc((void **)&c->scan_perm, sizeof(uint16_t) * perm.size(), c->st));
    IMX_CUDA(pool_alloc((void **)&c->scan_boff, sizeof(int32_t) * boff.size(), c->st));
    if (c->scan_ctr) cudaFreeAsync(c->scan_ctr, c->st);
    IMX_CUDA(pool_alloc((void **)&c->scan_ctr, sizeof(unsigned long long) * nchunks, c->st));
    IMX_CUDA(cudaMemcpyAsync(c->scan_xs, xs.data(), sizeof(int32_t) * xs.size(), cudaMemcpyHostToDevice, c->st));
    IMX_CUDA(cudaMemcpyAsync(c->scan_perm, perm.data(), sizeof(uint16_t) * perm.size(), cudaMemcpyHostToDevice, c->st));
    IMX_CUDA(cudaMemcpyAsync(c->scan_boff, boff.data(), sizeof(int32_t) * boff.size(), cudaMemcpyHostToDevice, c->st));
    IMX_CUDA(cudaStreamSynchronize(c->st));     // the host vectors go out of scope
    c->scan_kb = kb;
    c->scan_nb = nb;
    c->scan_cw = cw;
    c->scan_nchunks = nchunks;
    return IMX_OK;
}

// slice length of heavy rows (IMX_SCAN_HEAVY, default 64 slots).  With the
// forest edge of heavy rows (pass 1 over the slices): C4 18.7 / 18.0 / 18.7 /
// 21.7 ms at 128 / 256 / 512 / 1024.  Without it (the default now) shorter
// slices win -- the order-free slice walk (four slots per warp step) beats the
// light rows' slot-by-slot walk with its first-live flags: C4 21.0 / 17.0 /
// 15.9 / 15.5 / 15.7 / 16.3 / 17.6 ms at 16 / 32 / 48 / 64 / 128 / 256 / 512;
// C2 0.221 / 0.181 ms at 32 / 64 (no heavy row at 64); C5 unchanged.
static int scan_heavy_T() {
    const char *e = getenv("IMX_SCAN_HEAVY");
    return e ? std::max(0, atoi(e)) : 64;
}

// the pass that writes the isolated rows of a resident graph (IMX_SCAN_ISO_PASS, default 2)
static int scan_iso_pass() {
    const char *e = getenv("IMX_SCAN_ISO_PASS");
    return e && atoi(e) == 1 ? 1 : 2;
}

// Heavy rows' pass 1 (the slices' first live neighbours folded into the row
// by atomicMin, so that pass 2 can skip one union per row and lane) is off by
// default: a heavy row has many live neighbours per lane (C4's hubs: ~250),
// so the forest edge spares pass 2 well under 1% of its unions while the
// slices' pass 1 costs a full walk of every heavy prefix (C4: 0.92 ms;
// propagate 17.3 -> 16.25 ms without it).  Pass 2 then unites every live pair
// of a heavy row.  IMX_SCAN_HEAVY_P1=1 brings it back.
static int scan_heavy_forest() {
    const char *e = getenv("IMX_SCAN_HEAVY_P1");
    return e ? (atoi(e) != 0) : 0;
}

static int scan_bpsm() {
    const char *e = getenv("IMX_SCAN_BPSM");
    return e && atoi(e) > 0 ? atoi(e) : 8;
}

using ScanKernel = void (*)(const int64_t *, const int32_t *, const int32_t *, int32_t, int, int, int, int,
                            const int32_t *, const uint16_t *, const int32_t *, int64_t, int32_t, int64_t, Lay, uint32_t *,
                            unsigned long long *, const uint8_t *, const int32_t *, const int64_t *, const int32_t *,
                            int64_t, unsigned long long *, int, int64_t, int, int);
static const ScanKernel kScanKernels[2][2] = {{k_scan<1, false>, k_scan<1, true>}, {k_scan<2, false>, k_scan<2, true>}};

// one launch: the light rows [row0, row0 + rows) (heavy = false), or all heavy slices
static int launch_scan(imx_ctx *c, int pass, bool heavy, int64_t row0, int64_t rows, unsigned long long *hooks) {
    imx_graph *g = c->g;
    const auto &H = g->hv[0];            // both passes cut heavy rows alike: one table
    const int cw = c->scan_cw, nb = c->scan_nb;
    // cw is a multiple of 16, so every section keeps 16-byte alignment
    const size_t smem = (size_t)kScanWarps * cw + (pass == 2 ? sizeof(uint32_t) * kScanWarps * 3 * kScanQ : 0) +
                        sizeof(int2) * cw + sizeof(int2) * nb;
    ScanKernel kern = kScanKernels[pass - 1][heavy ? 1 : 0];
    IMX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t items = heavy ? H.nhs : rows;
    if (items <= 0) return IMX_OK;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(items, kScanWarps), 148 * scan_bpsm()));
    // items per counter grab: up to 16 rows, fewer when that would leave
    // warps idle (C2: 37k rows over ~9.5k warps)
    const int64_t warps = (int64_t)blocks * kScanWarps;
    const int grab = heavy ? 1 : (int)std::max<int64_t>(1, std::min<int64_t>(16, items / (warps * 8)));
    IMX_CUDA(cudaMemsetAsync(c->scan_ctr, 0, sizeof(unsigned long long) * c->scan_nchunks, c->st));
    kern<<<blocks, kScanWarps * 32, smem, c->st>>>(g->xadj, g->adj, g->hash, g->thr_u, c->scan_kb, nb, cw,
                                                   c->scan_nchunks, c->scan_xs, c->scan_perm, c->scan_boff, rows,
                                                   c->W, c->ld, c->lay, c->L, pass == 2 ? hooks : nullptr,
                                                   H.heavy, H.hs_v, H.hs_a, H.hs_len, H.nhs, c->scan_ctr, grab, row0,
                                                   c->scan_iso_pass, c->scan_heavy_forest);
    IMX_CHECK_LAUNCH();
    count_launch(c);
    return IMX_OK;
}

int run_scan(imx_ctx *c, int pass, unsigned long long *hooks) {
    imx_graph *g = c->g;
    const int64_t n = g->n;
    if (n == 0) return IMX_OK;
    IMX_TRY(ensure_scan_tables(c));
    const int T = scan_heavy_T();
    IMX_TRY(ensure_heavy(c, 1, T));
    if (pass == 1) {
        c->scan_iso_pass = scan_iso_pass();
        c->scan_heavy_forest = scan_heavy_forest();
    }
    IMX_TRY(launch_scan(c, pass, false, 0, n, hooks));
    if (g->hv[0].nhs > 0 && (pass == 2 || c->scan_heavy_forest)) IMX_TRY(launch_scan(c, pass, true, 0, n, hooks));
    return IMX_OK;
}

// Pass 1 on a streamed CSR (graph.cuh, struct_pending): the light rows of
// every chunk as soon as its adjacency, sources and hashes are on the device
// (the chunk's event), while the later chunks are still on the link; the
// heavy flags of a chunk's rows are computed right before.  Then the
// structure is settled (the host waits for the last chunk here; its
// statistics can fail the call) and the heavy slices follow as usual.
int run_scan_streamed(imx_ctx *c) {
    imx_graph *g = c->g;
    const int64_t n = g->n;
    IMX_TRY(ensure_scan_tables(c));
    const int T = scan_heavy_T();
    c->scan_iso_pass = 1;            // hidden behind the upload
    c->scan_heavy_forest = scan_heavy_forest();
    IMX_TRY(heavy_begin(c, 1, T));
    for (int ch = 0; ch < g->nchunk; ++ch) {
        const int64_t v0 = g->chunk_lo[ch], v1 = g->chunk_hi[ch];
        IMX_CUDA(cudaStreamWaitEvent(c->st, g->chunk_ev[ch], 0));
        if (v1 <= v0) continue;
        IMX_TRY(heavy_count_rows(c, 1, T, v0, v1));
        IMX_TRY(launch_scan(c, 1, false, v0, v1 - v0, nullptr));
    }
    const int rc = graph_settle_structure(g);
    if (rc != IMX_OK) { heavy_abort(c, 1); return rc; }
    IMX_TRY(heavy_finish(c, 1, T));
    if (g->hv[0].nhs > 0 && c->scan_heavy_forest) IMX_TRY(launch_scan(c, 1, true, 0, n, nullptr));
    (void)n;
    return IMX_OK;
}

}  // namespace imx
