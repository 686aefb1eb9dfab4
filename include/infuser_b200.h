/*
 * infuser_b200.h -- C ABI of libinfuser_b200.so, the sm_100a hot path of
 * InFuseR-MG (fused hash-sampled IC simulation -> per-simulation connected
 * components -> memoized component-size gains -> CELF seed selection).
 *
 * The reference (`infmax`, pure Python/numpy, /root/reference/pkg/src/infmax)
 * has no FFI.  Each entry point below replaces one reference routine; the
 * citation after each declaration names the routine (file:line, relative to
 * pkg/src/infmax/) whose semantics it reproduces bit for bit.  The Python
 * package paper_2008_03095_b200 binds these symbols with ctypes
 * (see INTEGRATION.md for the binding a reference maintainer would add).
 *
 * Conventions
 *   - Plain pointers and sizes only.  Every pointer argument is HOST memory,
 *     borrowed for the duration of the call, unless the name ends in _dev.
 *   - Return 0 on success, a negative IMX_E* code on failure; the message is
 *     available from imx_last_error() (thread-local).
 *   - Vertex ids and labels are int32 (ids < 2^31, graph.py:22); labels and
 *     sizes are [n][width] int32, simulation-contiguous (propagation.py:1-8).
 *   - One context owns one device and one lane window [lane0, lane0+width)
 *     of the simulation set; multi-GPU runs create one context per rank and
 *     combine the int64 partial sums (gains, CELF gains) with an allreduce.
 *   - Every call is synchronous with respect to the host unless noted.
 */
#ifndef INFUSER_B200_H
#define INFUSER_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IMX_OK          0
#define IMX_EINVAL     -1   /* bad argument            -> ValueError          */
#define IMX_ENOMEM     -2   /* device allocation failed -> MemoryError        */
#define IMX_ECUDA      -3   /* CUDA runtime error       -> RuntimeError       */
#define IMX_ENODEV     -4   /* no usable sm_100 device  -> RuntimeError       */
#define IMX_ECONSTRAINT -5  /* documented limit violated -> ConstraintError   */
#define IMX_EFORMAT    -6   /* malformed graph          -> GraphFormatError   */
#define IMX_EINTERNAL  -7   /* failed self-check        -> AssertionError     */
#define IMX_ENCCL      -8   /* NCCL error               -> RuntimeError       */

typedef struct imx_graph imx_graph;   /* device-resident symmetric CSR        */
typedef struct imx_ctx   imx_ctx;     /* device-resident labels/sizes/CELF    */
typedef struct imx_comm  imx_comm;    /* int64 sums over the ranks of a run   */

/* ---- library ----------------------------------------------------------- */
const char *imx_last_error(void);
int  imx_version(void);                                   /* 10000*maj+100*min */
/* number of visible CUDA devices with compute capability 10.x (0 on a CPU box) */
int  imx_device_count(void);
/* kernels this library has launched in this process (all contexts)        */
int64_t imx_launch_count(void);

/* ---- K1: CSR builder ----------------------------------------------------
 * Graph.from_edges (graph.py:124-155): k distinct undirected edges
 * (edges[2i], edges[2i+1]) on 0..n-1 -> rows sorted by (src, dst), both
 * directions share weight w_edge[i] (or w_scalar when w_edge == NULL).
 * Validation order and messages follow graph.py:134-146.  The graph stays on
 * the device; imx_graph_get_csr copies xadj/adj/weights back.             */
int  imx_graph_from_edges(int32_t device, int64_t n, const int64_t *edges,
                          int64_t k, const double *w_edge, double w_scalar,
                          imx_graph **out);
/* Upload an existing CSR (Graph(xadj, adj, weights, orig_ids), graph.py:37).
 * Large graphs (>= 4 M slots) leave the weights on the link when the call
 * returns, very large ones in pinned host memory (>= 16 M slots) also the
 * adjacency: the caller's arrays must stay valid and unchanged until the
 * first result of the graph has been read back (or the graph is destroyed).
 * What the eager build reports for a bad CSR ("corrupt CSR offsets",
 * "adjacency entry outside 0..n-1", "adjacency is not symmetric") then
 * surfaces from the first call that needs the structure (imx_propagate,
 * imx_graph_get_csr, ...); the offsets are always checked before return.    */
int  imx_graph_from_csr(int32_t device, int64_t n, int64_t m2,
                        const int64_t *xadj, const int32_t *adj,
                        const double *weights, imx_graph **out);
/* Seeded synthetic graph generated and built on the device (SURVEY 8(f)
 * rank 1; the reference's generate_er / generate_rmat, graph.py:444-491, are
 * host numpy).  kind 0 Erdos-Renyi, 1 R-MAT (params = probs[4], n = 2^scale),
 * 2 Chung-Lu (cdf = n normalised cumulative expected degrees).  Counter-based
 * SplitMix64 streams (gen.cu); m > 0: first m distinct non-loop pairs in draw
 * order (draws = initial candidate count, 0 = auto), m == 0: every distinct
 * non-loop pair among `draws` candidates.  Unit weights.                    */
int  imx_graph_generate(int32_t device, int32_t kind, int64_t n, int64_t m,
                        int64_t draws, uint64_t seed, const double *params,
                        const double *cdf, imx_graph **out);
void imx_graph_destroy(imx_graph *g);
int  imx_graph_dims(const imx_graph *g, int64_t *n, int64_t *m2);
int  imx_graph_get_csr(imx_graph *g, int64_t *xadj, int32_t *adj, double *weights);
/* Graph.reciprocal_slots (graph.py:85-99); IMX_EFORMAT if not symmetric.  */
int  imx_graph_reciprocal(imx_graph *g, int64_t *recip);
/* Graph.with_weights (graph.py:112-119): replace per-slot weights, then
 * refresh thresholds.  IMX_ECONSTRAINT if a weight is outside [0, 1].     */
int  imx_graph_set_weights(imx_graph *g, const double *weights);

/* ---- K2: sampler tables -------------------------------------------------
 * build_hash_table (hashing.py:97-101): per-slot
 * murmur3_x86_32(LE32(min) || LE32(max), seed 0) & 0x7FFFFFFF.            */
int  imx_graph_hashes(imx_graph *g, int32_t *hashes_out);
/* Use caller-provided per-slot hashes (EdgeHashTable.hashes) instead;
 * hashes == NULL restores the computed table.                              */
int  imx_graph_set_hashes(imx_graph *g, const int32_t *hashes);
/* slot_thresholds (hashing.py:153-165): int32(int64(w * (2^31-1))),
 * max-symmetrized over reciprocal slots when symmetrize != 0.
 * *uniform_out (nullable) = 1 when all symmetrized thresholds are equal.  */
int  imx_graph_thresholds(imx_graph *g, int32_t symmetrize, int32_t *thr_out,
                          int32_t *uniform_out);
/* Vectorized murmur3 over (lo[i], hi[i]) 8-byte keys, unmasked
 * (_murmur3_pair_array, hashing.py:65-86).                                 */
int  imx_murmur3_pairs(int32_t device, const uint32_t *lo, const uint32_t *hi,
                       int64_t count, uint32_t *out);

/* ---- context: one lane window on one device ----------------------------- */
typedef struct {
    int32_t  sweeps;           /* phases executed (init, hook, compress[, verify]) */
    int32_t  cap;              /* capacity of the arrays below             */
    int64_t *changed_pairs;    /* per phase: (vertex, lane) labels changed */
    int64_t *label_sums;       /* per phase: sum of all labels (int64)     */
    int32_t *modes;            /* per phase: IMX_MODE_*                    */
} imx_prop_stats;              /* PropagateStats (propagation.py:49-56)   */

#define IMX_MODE_INIT     0
#define IMX_MODE_HOOK     1
#define IMX_MODE_COMPRESS 2
#define IMX_MODE_VERIFY   3

/* X: the 31-bit per-simulation words of lanes [lane0, lane0+width)
 * (SimulationRandoms.values, hashing.py:111-119); num_scored: how many of
 * this window's lanes are scored (the rest are padding).                  */
int  imx_create(imx_graph *g, const int32_t *X, int32_t width,
                int32_t num_scored, imx_ctx **out);
void imx_destroy(imx_ctx *c);

/* K3: fused sample + CC (propagate, propagation.py:260-321): converged
 * min-id labels of every lane.  verify != 0 adds a checking pass (every live
 * edge joins equal labels, every label is its own root) whose changed count
 * must be 0 (otherwise IMX_EINTERNAL).  st may be NULL.                    */
int  imx_propagate(imx_ctx *c, int32_t verify, imx_prop_stats *st);

/* K4+K5: component_sizes_and_gains (propagation.py:371-390): component
 * histogram over all lanes, int64 gains over the scored lanes.
 * gains_out may be NULL (gains stay on the device for CELF).              */
int  imx_memoize(imx_ctx *c, int64_t *gains_out);
/* Fuse the memo into propagation where the labels are compressed in lane
 * tiles (very wide label matrices): the gains are summed from each tile
 * while it is on chip, and the next imx_memoize only copies them out.      */
int  imx_set_fuse_memo(imx_ctx *c, int32_t on);

/* Large host CSRs: imx_graph_from_csr leaves the 8-byte-per-slot weights on
 * the link and imx_propagate starts on the speculative uniform threshold of
 * weights[0].  By default imx_propagate waits for the weights before it
 * returns results (and runs again if they differ).  imx_spec_defer(c, 1)
 * hands that check to the caller: memoisation and the CELF loop then also run
 * while the weights upload, and imx_spec_settle says afterwards whether the
 * speculation held (held = 0: call imx_propagate again and redo what followed;
 * the thresholds are settled then).  Getters of labels, sizes, gains and the
 * seed state check by themselves and fail rather than return unconfirmed
 * results.  The reference has no counterpart: Graph.weights is a host array
 * (graph.py:37-60) and thresholds are computed eagerly (hashing.py:153-165). */
int  imx_spec_defer(imx_ctx *c, int32_t on);
int  imx_spec_settle(imx_ctx *c, int32_t *held);

/* Load labels (and optionally sizes; NULL -> recomputed from labels) from
 * the host instead of propagating: select_seeds / initial_marginal_gains on
 * caller arrays (selection.py:115, propagation.py:349-368).  ld = row
 * stride of the host arrays in elements (>= width).                        */
int  imx_load_labels(imx_ctx *c, const int32_t *labels, const int32_t *sizes,
                     int64_t ld);

/* D2H copies of lanes [r0, r1) of this window into dense [n][r1-r0].      */
int  imx_copy_labels(imx_ctx *c, int32_t r0, int32_t r1, int32_t *out);
int  imx_copy_sizes (imx_ctx *c, int32_t r0, int32_t r1, int32_t *out);

/* ---- K6-K8: CELF (selection.py:115-149) ---------------------------------
 * Round-based exact CELF.  The device keeps the non-seeds sorted by stale
 * key (-prio, id), the per-lane covered-component bitmaps and the per-lane
 * covered totals.  The vertices the reference's lazy heap refreshes in a
 * round are a prefix of that order.                      */
/* prio: n int64 initial priorities (NULL -> this context's own gains).    */
int  imx_celf_reset(imx_ctx *c, const int64_t *prio);
/* first vertex of the order (max prio, min id); *v = -1 when none remain. */
int  imx_celf_top(imx_ctx *c, int64_t *prio_out, int32_t *v_out);
/* marginal_gain (selection.py:63-70), partial over this window's scored
 * lanes, of order[lo, hi): fresh_out[hi-lo]; ids_out/prio_out receive
 * order[lo, min(hi+1, len)) (one extra entry: the next stale key); *len_out
 * = current order length.  Identical ids/prio on every rank.              */
int  imx_celf_prefix(imx_ctx *c, int64_t lo, int64_t hi, int32_t *ids_out,
                     int64_t *prio_out, int64_t *fresh_out, int64_t *len_out);
/* End of a round: commit_seed(u) (selection.py:73-81; *gain_out = partial
 * newly covered total), drop order[0, k) and merge back the cnt refreshed
 * vertices ids[] with their fresh gains prio[] (sorted by (-prio, id)).    */
int  imx_celf_advance(imx_ctx *c, int64_t k, int32_t u, const int32_t *ids,
                      const int64_t *prio, int64_t cnt, int64_t *gain_out);
/* marginal_gain of an explicit candidate list.                            */
int  imx_eval_gains(imx_ctx *c, const int32_t *cand, int64_t cnt, int64_t *out);
/* commit_seed of u without touching the order (per-vertex API).           */
int  imx_commit(imx_ctx *c, int32_t u, int64_t *gain_out);
/* Whole CELF loop on one context (single-rank fast path): k seeds and their
 * gains; *trace_len = number of dequeues recorded (fetch with
 * imx_celf_trace).  Requires a fresh imx_celf_reset.                       */
int  imx_celf_select(imx_ctx *c, int32_t k, int32_t *seeds_out,
                     int64_t *gains_out, int64_t *trace_len);
/* The same loop over a lane shard of a multi-rank run (select_rounds,
 * celf.py): allreduce(buf, n, user) must replace buf[0, n) by its int64 sum
 * over the ranks (every rank calls it in the same order); partial gains of
 * each evaluated batch and the commit self-check go through it.  Requires a
 * fresh imx_celf_reset with the GLOBAL initial gains.                       */
typedef int (*imx_allreduce_fn)(int64_t *buf, int64_t n, void *user);
int  imx_celf_select_sharded(imx_ctx *c, int32_t k, imx_allreduce_fn allreduce,
                             void *user, int32_t *seeds_out, int64_t *gains_out,
                             int64_t *trace_len);
/* ---- multi-rank data plane ----------------------------------
 * Replaces the reference's thread-pool split of the lanes
 * (propagation.py:209-216, 244-251) by ranks holding lane windows; their
 * int64 partial sums (memo gains, CELF batch gains, commit self-checks) are
 * added on the device, in place, on the context's stream.
 *   NCCL:  rank 0 gets an id (imx_comm_unique_id), the launcher sends it to
 *          every rank, each rank calls imx_comm_create (ncclCommInitRank;
 *          libnccl.so.2 is opened at first use).
 *   LOCAL: ranks as threads of one process (one GPU; tests): one group,
 *          one imx_comm_create_local per rank.
 * A context with an attached communicator (imx_ctx_attach_comm) allreduces
 * the gains inside imx_memoize and runs imx_celf_select_comm.              */
#define IMX_COMM_ID_BYTES 128
int  imx_comm_unique_id(uint8_t *id_out /* IMX_COMM_ID_BYTES */);
int  imx_comm_create(int32_t device, int32_t nranks, int32_t rank, const uint8_t *id,
                     imx_comm **out);
int  imx_local_group_create(int32_t nranks, void **group_out);
void imx_local_group_destroy(void *group);
int  imx_comm_create_local(void *group, int32_t rank, int32_t device, imx_comm **out);
void imx_comm_destroy(imx_comm *comm);
/* host buf[0, n) <- its sum over the ranks (through device memory)         */
int  imx_comm_allreduce(imx_comm *comm, int64_t *buf, int64_t n);
int  imx_ctx_attach_comm(imx_ctx *c, imx_comm *comm /* NULL detaches */);
/* select_seeds over the lane shards of an attached communicator: the
 * round-based CELF of imx_celf_select_sharded with every batch's partial
 * gains and the commit self-check summed on the device (no host bounce of
 * the data); every rank calls it.  Requires imx_memoize (which allreduced
 * the gains) and imx_celf_reset(c, NULL).  selection.py:115-149.           */
int  imx_celf_select_comm(imx_ctx *c, int32_t k, int32_t *seeds_out, int64_t *gains_out,
                          int64_t *trace_len);
/* The trace of the last imx_celf_select: records of 5 int64
 * (vertex, stale_gain, fresh_gain, committed, seeds_before) -- TraceRecord,
 * selection.py:25-33 -- up to cap records.                                 */
int  imx_celf_trace(imx_ctx *c, int64_t *out, int64_t cap);
/* The same trace without a copy: *out = the context's pinned host buffer of
 * *len records (NULL when empty), now owned by the caller -- release it with
 * imx_host_free.  The context starts a new buffer for its next select.     */
int  imx_celf_trace_take(imx_ctx *c, int64_t **out, int64_t *len);
void imx_host_free(void *p);
/* per_sim[r] = covered vertices of lane r (SelectionResult.spread_se,
 * selection.py:105-112), for this window's scored lanes.                  */
int  imx_per_sim(imx_ctx *c, int64_t *out);
/* owned bitmap rows: [n][ceil(num_scored/32)] uint32 (SeedState.owned).  */
int  imx_copy_owned(imx_ctx *c, uint32_t *bits_out);

/* ---- evaluation (evaluation.py) -----------------------------------------
 * evaluate_seeds (evaluation.py:101-136) on fresh rng-sampled worlds: world j
 * of chunk c (c = j / chunk) consumes draws [(j mod chunk)*E, ..+E) of numpy
 * PCG64 stream c, given as 4 uint64 per chunk {state_hi, state_lo, inc_hi,
 * inc_lo} (default_rng(SeedSequence(seed).spawn(..)[c]).bit_generator.state);
 * edge e (canonical slots, slot order) is live iff random() < max(w, w_recip).
 * counts_out[j] = reached-set size of world j (seeds: k distinct ids).     */
int  imx_evaluate_seeds(imx_graph *g, const int32_t *seeds, int32_t k, int64_t r_eval,
                        const uint64_t *streams, int64_t chunk, int64_t *counts_out);
/* sampling_cdf (evaluation.py:157-183): values (hash[canon[i*stride]] ^
 * X[r]) / H_MAX over strided canonical slots and r < scored; outputs the
 * numpy-rule histogram over `edges` (bins+1 ascending f64), the exact KS
 * distance to U(0,1) and the number of values.                            */
int  imx_sampling_cdf(imx_graph *g, const int32_t *X, int32_t scored, int64_t stride,
                      int32_t bins, const double *edges, int64_t *counts_out,
                      double *ks_out, int64_t *nvals_out);

/* ---- graph files (graph.py:269-437) --------------------------------------
 * Native parser of a whitespace-separated "u v [w]" text edge list
 * (load_edge_list, graph.py:273-330): comments / blank lines skipped, ids
 * compacted in order of first appearance, self-loops dropped, duplicate
 * undirected edges collapse to the first occurrence.  On IMX_EFORMAT,
 * *err_kind: 1 field count (*err_aux = fields), 2 non-numeric field,
 * 3 weight outside [0, 1] (err_text = the weight field), 4 no edges,
 * 5 cannot open (*err_aux = errno), 6 id beyond int64, 7 id space full;
 * *err_line = 1-based line, err_text = the stripped line (kinds 1, 2, 6).  */
typedef struct imx_edge_list imx_edge_list;
int  imx_edge_list_parse(const char *path, imx_edge_list **out, int64_t *err_line,
                         int32_t *err_kind, int64_t *err_aux, char *err_text,
                         int64_t err_text_cap);
int  imx_edge_list_dims(const imx_edge_list *e, int64_t *n_vertices, int64_t *n_edges);
/* edges: 2 int64 per edge (compact ids), weights: f64 per edge,
 * orig_ids: int64 per compact id.                                          */
int  imx_edge_list_copy(const imx_edge_list *e, int64_t *edges, double *weights,
                        int64_t *orig_ids);
void imx_edge_list_free(imx_edge_list *e);

/* ---- measurement --------------------------------------------------------
 * Device time (CUDA events on the context stream) of the last call of each
 * phase and the number of kernels this context launched so far.           */
typedef struct {
    float   propagate_ms, memoize_ms, select_ms;
    float   init_ms, hook_ms, compress_ms;
    int64_t kernel_launches;
    int64_t hook_launches;
    int64_t celf_evaluations;  /* marginal-gain evaluations of the last select */
} imx_timings;
int  imx_get_timings(imx_ctx *c, imx_timings *out);
/* Run propagate `reps` times back to back (inputs resident) and report the
 * average device time of the whole propagate and of its dominant kernel.  */
int  imx_bench_propagate(imx_ctx *c, int32_t reps, int32_t flush_l2,
                         float *avg_total_ms, float *avg_hook_ms,
                         float *avg_compress_ms, float *avg_init_ms);

#ifdef __cplusplus
}
#endif
#endif /* INFUSER_B200_H */
