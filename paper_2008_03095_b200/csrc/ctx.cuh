// ctx.cuh -- the per-device, per-lane-window context shared by the K3-K8
// translation units (propagate.cu, memo.cu, celf.cu, ctx.cu).
//
// Data layout in HBM (one context = one device, one lane window of width W):
//   L[n][ld] uint32  the label matrix, simulation-contiguous (propagation.py:1-8),
//                    ld = W rounded up to 4 so every row is 16-byte aligned.
//                    Cell encoding (see uf.cuh):
//                      bit 31 set   -> v is the root (= min id) of its component
//                                      in lane r; bits 0-30 = number of OTHER
//                                      members (filled by the compress pass)
//                      bit 31 clear -> parent pointer; after compress, the root
//                    so label(v, r) = root ? v : cell, and the component size of
//                    a root cell is (cell & 0x7FFFFFFF) + 1: labels and sizes
//                    (propagation.py:349-390) live in ONE n*W*4-byte array.
//   C[n][ld] uint32  only for contexts fed with caller labels (imx_load_labels):
//                    L then holds plain labels and C their full component sizes.
//   cov[n][cw]       covered-component bitmap of the CELF state, cw = ceil(ns/32)
//                    (SeedState.owned, selection.py:36-60).
#pragma once
#include <vector>

#include "common.cuh"
#include "graph.cuh"
#include "uf.cuh"

// device-resident state of the persistent CELF kernel (celf.cu)
struct CelfDev {
    // order window
    int64_t ostart, olen;
    int32_t ocur, t;
    int64_t trace_len, batch0;
    int32_t status;        // 1 done, 2 trace buffer full, 3 self-check failed, 4 round too large,
                           // 5 paused for an exchange, 6 a huge seed-table batch [xlo, xhi) is left to k_wide_tab_round
    int32_t bad_v;
    int64_t bad_want, bad_got;
    // phase times (ns, %globaltimer on block 0): eval, commit, rank, merge;
    // [4] eval batch steps, [5] evaluations; eval step split: [6] block 0's
    // own evaluations, [7] barrier wait, [8] batch max + stop test
    // (IMX_CELF_PROFILE prints them)
    unsigned long long prof[10];
    // per-step maximum fresh key of the evaluated batch, 4 rotating slots
    unsigned long long smax[4];
    // work counters of k_wide_tab_round's dynamic candidate grabs, rotating like smax
    unsigned long long wctr[4];
    // a round the kernel cannot hold (status 2/4): its best fresh key and
    // refreshed prefix length (fresh[] holds the evaluated prefix)
    unsigned long long big_key;
    int64_t big_kr;
    // exchange mode (sharded runs, celf_select_xchg): the kernel pauses with
    // status 5 after writing an evaluated batch's partial gains to the
    // exchange buffer; the host sums them over the ranks (NCCL) and
    // relaunches, which resumes at xphase 1 with batch [xlo, xhi) and the
    // round's best key so far.  A commit's partial gain rides in the
    // exchange buffer's last slot and is checked at the next resume.
    int32_t xphase, xpend, xpend_v, xpad;
    int64_t xlo, xhi;
    unsigned long long xbest;
    int64_t xpend_want, xpend_got;
};

struct imx_ctx {
    imx_graph *g = nullptr;
    int dev = 0;
    cudaStream_t st = nullptr;
    int32_t W = 0, ns = 0, cw = 0;
    int64_t ld = 0;               // cells per vertex: W rounded up to 4 (rows) or to the tile width
    // layout of L (uf.cuh): rows, or lane tiles for very wide contexts
    // (lay_native); caller labels (imx_load_labels) always use rows
    imx::Lay lay, lay_native;
    int vb = 0;                   // bits for vertex ids in packed CELF keys
    int32_t *X = nullptr;         // [ld]
    uint32_t *L = nullptr;        // [n*ld]
    size_t L_bytes = 0;
    uint32_t *C = nullptr;        // [n*ld] caller-label mode only
    int64_t *gains = nullptr;     // [n]
    // CELF state
    uint8_t *inS = nullptr;       // [n]
    uint32_t *cov = nullptr;      // [n*cw]
    int64_t *per_sim = nullptr;   // [W]
    int64_t *eval_out = nullptr;  // [n]
    int32_t *d_one = nullptr;     // [4]
    // candidate order: non-seeds sorted by packed stale key, double-buffered
    int32_t *oid[2] = {nullptr, nullptr};
    unsigned long long *okey[2] = {nullptr, nullptr};
    int ocur = 0;
    int64_t ostart = 0, olen = 0;
    void *sort_tmp = nullptr;
    size_t sort_tmp_bytes = 0;
    int32_t *h_ids = nullptr, *d_ids = nullptr;   // pinned staging for prio updates
    int64_t *h_vals = nullptr, *d_vals = nullptr;
    int64_t stage_cap = 0;
    int64_t evaluated = 0;
    // dequeue trace, 5 int64 per record, in pinned host memory (the device
    // trace is copied straight into it)
    int64_t *trace = nullptr;
    int64_t trace_n = 0, trace_hcap = 0;
    // persistent CELF kernel state and buffers
    CelfDev *cdev = nullptr;
    unsigned long long *skey = nullptr;   // refreshed keys ranked by fresh gain
    int32_t *sid = nullptr;
    int64_t *dtrace = nullptr;
    int64_t trace_cap = 0;
    unsigned long long big_key = 0;   // last kernel stop on an oversized round
    int64_t big_kr = 0;
    int32_t *dseeds = nullptr;
    int64_t *dsgains = nullptr;
    int32_t dseeds_cap = 0;
    int2 *stab = nullptr;             // [kTab][ld] seed table of the early CELF rounds
    // first-seed speculation (memo.cu): labels of the max-degree vertex's components per lane and
    // g1[v] = gain of v once that vertex is the first seed; scratch[15] = that vertex
    int32_t *hublab = nullptr;        // [ld]
    int64_t *g1 = nullptr;            // [n]
    bool g1_ready = false;
    int celf_grid[4] = {0, 0, 0, 0};  // cooperative grids of k_celf_rounds<ENC, XM> on this context's device
    int wide_grid[2] = {0, 0};        // and of k_wide_tab_round<TAB1>
    // interval-enumeration sampler
    int64_t *seg_a = nullptr, *seg_n = nullptr, *seg_off = nullptr;
    int64_t nseg_cap = 0;
    void *scan_tmp = nullptr;
    size_t scan_tmp_bytes = 0;
    // scan sampler (scan.cu): lanes of every chunk of scan_cw lanes sorted by
    // X >> scan_kb; scan_boff = bucket offsets per chunk
    std::vector<int32_t> hX;          // the context's words on the host
    int32_t *scan_xs = nullptr;
    uint16_t *scan_perm = nullptr;
    int32_t *scan_boff = nullptr;
    unsigned long long *scan_ctr = nullptr;   // [scan_nchunks] work counters of one launch
    int scan_kb = -1, scan_nb = 0, scan_cw = 0, scan_nchunks = 0;
    int scan_heavy_forest = 1;        // heavy rows got their forest edge in pass 1 (pass 2 skips it)
    int scan_iso_pass = 2;            // the pass of the current propagate that writes the isolated rows
    // misc
    unsigned long long *scratch = nullptr;  // [16]: per-call counters (4 label sum, 6 bad labels, 7 commit gain, 9 max prio, 13 bad prio, 14 hub degree key, 15 hub)
    bool labels_ready = false, memo_ready = false, celf_ready = false;
    cudaEvent_t ev[8];
    // phase timings not read back yet: 1 = propagate (ev 0-3), 2 = memo (ev 4-5)
    int tm_pending = 0;
    // memoisation fused into the tiled compression (imx_set_fuse_memo): the
    // last propagate left the gains in `gains` (gains_fused)
    bool fuse_memo = false, gains_fused = false;
    // ranks of a sharded run (comm.cu); NULL = single rank
    imx_comm *comm = nullptr;
    // a big CELF round's trace records travel to the host on this side stream
    // while the later rounds run (celf_big_round); trace_flush waits for it
    cudaStream_t tst = nullptr;
    // the last sampler launch used a deferred graph's speculative threshold
    bool spec_used = false;
    // imx_spec_defer: imx_propagate does not wait for the weights; the caller
    // checks with imx_spec_settle before it trusts any result (run_fused does,
    // after the CELF loop); spec_thr = the threshold the results stand on
    bool spec_defer = false;
    int32_t spec_thr = 0;
    imx_timings tm{};
};

namespace imx {

inline int grid_for(int64_t work, int threads = 256) {
    int64_t b = ceil_div(work > 0 ? work : 1, threads);
    if (b > 148 * 16) b = 148 * 16;
    return (int)b;
}

// read the pending phase times (waits for their end events)
inline void settle_timings(imx_ctx *c) {
    if (c->tm_pending & 1) {
        if (cudaEventSynchronize(c->ev[3]) == cudaSuccess) {
            cudaEventElapsedTime(&c->tm.init_ms, c->ev[0], c->ev[1]);
            cudaEventElapsedTime(&c->tm.hook_ms, c->ev[1], c->ev[2]);
            cudaEventElapsedTime(&c->tm.compress_ms, c->ev[2], c->ev[3]);
            cudaEventElapsedTime(&c->tm.propagate_ms, c->ev[0], c->ev[3]);
        }
    }
    if (c->tm_pending & 2) {
        if (cudaEventSynchronize(c->ev[5]) == cudaSuccess) cudaEventElapsedTime(&c->tm.memoize_ms, c->ev[4], c->ev[5]);
    }
    c->tm_pending = 0;
}

inline void count_launch(imx_ctx *c, int k = 1) {
    c->tm.kernel_launches += k;
    note_launch(k);
}

int ensure_celf_buffers(imx_ctx *c);
int trace_reserve(imx_ctx *c, int64_t cnt);
int trace_flush(imx_ctx *c);
void pinned_lend(void *p, size_t bytes);   // handed to the caller; imx_host_free returns it
int ensure_pinned(imx_ctx *c, int64_t cnt);
int run_init(imx_ctx *c);
// heavy-row slices of the graph for slice length T, cached on the graph (propagate.cu)
int ensure_heavy(imx_ctx *c, int pass, int T);
// the same in steps, for row ranges that become available one after the other (streamed CSR)
int heavy_begin(imx_ctx *c, int pass, int T);
int heavy_count_rows(imx_ctx *c, int pass, int T, int64_t v0, int64_t v1);
int heavy_finish(imx_ctx *c, int pass, int T);
void heavy_abort(imx_ctx *c, int pass);
// buf[0, n) on the device <- its sum over the communicator's ranks (comm.cu)
int comm_allreduce_i64(imx_comm *cm, int64_t *dbuf, int64_t n, cudaStream_t st);
// the scan sampler (scan.cu)
bool scan_eligible(const imx_graph *g);
int run_scan(imx_ctx *c, int pass, unsigned long long *hooks);
int run_scan_streamed(imx_ctx *c);
// results computed on a speculative threshold (spec_used): wait for the
// weights; held = the speculation was right.  spec_guard: the same before a
// result leaves the device, failing when it did not hold.
int spec_settle(imx_ctx *c, int32_t *held);
int spec_guard(imx_ctx *c);
// raw label-matrix passes shared with the evaluation worlds (evaluation.cu)
int launch_init(uint32_t *L, int64_t n, int64_t ld, cudaStream_t st);
int launch_gains_tile(const uint32_t *T, int64_t n, int64_t tld, int32_t ns_t, int first, int64_t *gains,
                      cudaStream_t st);
int launch_compress(uint32_t *L, int64_t n, int64_t ld, int32_t W, unsigned long long *nonroot,
                    cudaStream_t st, int *launches = nullptr, int64_t window = 0,
                    const int32_t *rows = nullptr, int64_t nrows = 0);

}  // namespace imx

#define CTX_CHECK(c)                                                       \
    do {                                                                   \
        if (!(c)) { ::imx::set_error("context is NULL"); return IMX_EINVAL; } \
        IMX_CUDA(cudaSetDevice((c)->dev));                                 \
    } while (0)

#define CELF_CHECK(c)                                                             \
    do {                                                                          \
        CTX_CHECK(c);                                                             \
        if (!(c)->celf_ready) { ::imx::set_error("CELF state not initialised (imx_celf_reset)"); return IMX_EINVAL; } \
    } while (0)
