// graph.cuh -- device-resident CSR shared by the CC / memo / CELF kernels.
#pragma once
#include "common.cuh"

struct imx_graph {
    int dev = 0;
    cudaStream_t stream = nullptr;
    int64_t n = 0;           // vertices
    int64_t m2 = 0;          // directed slots (Graph.m in the reference)
    int64_t me = 0;          // canonical (lo < hi) slots = undirected edges
    int64_t *xadj = nullptr; // [n+1]
    int32_t *adj = nullptr;  // [m2]  rows sorted ascending
    double *w = nullptr;     // [m2]  per-slot weight
    int32_t *src = nullptr;  // [m2]  row of each slot
    int32_t *hash = nullptr; // [m2]  31-bit edge hash (hashing.py:97-101)
    int32_t *thr = nullptr;  // [m2]  symmetrized threshold (hashing.py:153-165)
    int64_t *recip = nullptr;// [m2]  reciprocal slot
    int64_t *cslot = nullptr;// [me]  canonical slot ids in slot order
    // Undirected edges (lo < hi) sorted by (threshold bucket, hash): the
    // sampler enumerates the live edges of a lane as hash intervals of a
    // bucket (see cc.cu, k_hook_enum).  With a uniform threshold there is one
    // bucket; otherwise nb quantile buckets of the threshold.
    int2 *E = nullptr;       // [me]  (lo, hi) of each undirected edge
    int32_t *EH = nullptr;   // [me]  its hash (ascending within a bucket)
    int32_t *ET = nullptr;   // [me]  its threshold
    int nb = 1;              // threshold buckets
    int32_t *btmax = nullptr;// [nb]  max threshold of each bucket
    int64_t *boff = nullptr; // [nb+1] bucket offsets into E/EH/ET
    // hash-prefix lookup: lut[b*(2^lut_bits+1) + k] = first edge of bucket b
    // whose hash >> (31 - lut_bits) >= k, so a lower_bound over a bucket is
    // one lookup + a short binary search
    int32_t *lut = nullptr;
    int lut_bits = 0;
    int32_t thr_u = 0;       // the threshold when uniform
    int64_t max_prefix = 0;  // max over v of #neighbours smaller than v
    double thr_mean = 0;     // mean canonical-edge threshold / H_MAX = mean live fraction
    int uniform = 1;         // all thresholds equal
    int hash_neg = 0;        // some hash has bit 31 set (caller table): no interval enumeration
    int symmetric = 1;
    // pull sampler, one table per pass: vertices whose smaller-neighbour
    // prefix exceeds hv[p].T slots (heavy[v] = 1) and their prefix slices
    // (vertex, first slot, length), built on first use (propagate.cu,
    // ensure_heavy)
    // Large host CSRs (imx_graph_from_csr): the weights -- the biggest
    // array, 8 bytes per slot -- go up on a second stream and their per-slot
    // thresholds are computed there, while the caller already propagates with
    // the speculative uniform threshold thr_u = threshold(weights[0]);
    // graph_settle() waits for them and says whether the speculation held.
    // The reciprocal slots and the enumeration index are built on first use.
    bool thr_pending = false;
    cudaStream_t wst = nullptr;
    cudaEvent_t wev = nullptr;
    void *wstats_d = nullptr, *wstats_h = nullptr;   // GStats (device, pinned host)
    void *wthread = nullptr;                           // std::thread of a pageable upload
    int wthread_rc = 0;
    // Streamed structure (imx_graph_from_csr on large pinned host CSRs): the
    // adjacency goes up in row-aligned chunks on its own stream `ust`, the
    // per-slot structure (sources, hashes, symmetry sums, prefix maxima) of a
    // chunk is computed on `stream` as soon as it lands (chunk_ev[c] marks
    // it), and imx_graph_from_csr returns once the offsets are checked --
    // before the adjacency is up.  The scan sampler's first pass starts on the
    // chunks as they arrive (scan.cu, run_scan_streamed); everything else waits
    // in graph_settle_structure(), which reads the statistics and reports
    // what imx_graph_from_csr would have (bad entries, asymmetry).
    bool struct_pending = false;
    int struct_rc = 0;                  // sticky result of the settled structure
    cudaStream_t ust = nullptr;
    static constexpr int kMaxChunks = 32;
    int nchunk = 0;
    int64_t chunk_row[kMaxChunks + 1] = {0};       // row cuts, ascending
    int64_t chunk_lo[kMaxChunks] = {0}, chunk_hi[kMaxChunks] = {0};   // rows of chunk c in upload order
    cudaEvent_t chunk_ev[kMaxChunks] = {nullptr};
    cudaEvent_t sev_done = nullptr;
    void *sstats_d = nullptr, *sstats_h = nullptr;   // GStats (device, pinned host)
    bool recip_ready = true;
    bool index_ready = false;
    // false: the thresholds are uniform (thr_u) and the per-slot array is filled on first use
    // (ensure_thr): a deferred graph only checks that every weight equals weights[0]
    bool thr_ready = true;
    bool cslot_ready = true;     // false: cslot built on first use (ensure_cslot)
    // non-isolated vertices (built on first use, ensure_nz_rows); NULL when
    // isolated vertices are too few to be worth skipping
    int32_t *nz_rows = nullptr;
    int64_t n_nz = -1;
    struct HeavySlices {
        int T = -1;
        uint8_t *heavy = nullptr;
        int32_t *hs_v = nullptr;
        int64_t *hs_a = nullptr;
        int32_t *hs_len = nullptr;
        int64_t nhs = 0;
        // scratch of a table under construction (heavy_begin .. heavy_finish)
        int32_t *pre = nullptr;
        int64_t *nsl = nullptr, *off = nullptr;
    } hv[2];
};

namespace imx {
int select_device(int32_t device);
void graph_free(imx_graph *g);
int graph_create(int32_t device, int64_t n, int64_t m2, imx_graph **out);
int graph_build_from_device_edges(imx_graph *g, const int64_t *dedges, int64_t k, const double *dw,
                                  double w_scalar);
// the deferred weights/thresholds are in (waits for them); the lazily built
// reciprocal slots and sampler index
int graph_settle(imx_graph *g);
// the streamed structure is complete and valid (waits for the chunk uploads)
int graph_settle_structure(imx_graph *g);
int ensure_recip(imx_graph *g);
int ensure_thr(imx_graph *g);
int ensure_index(imx_graph *g);
int ensure_nz_rows(imx_graph *g);
int ensure_cslot(imx_graph *g);
}
