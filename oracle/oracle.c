/*
 * oracle.c -- CPU restatement of the reference's fused hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in paper_2008_03095_b200/ links, loads
 * or calls this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs use it, as the checker and as the
 * timed CPU baseline.
 *
 * Every function restates one routine of the reference package
 * /root/reference/pkg/src/infmax (cited file:line) in plain C, with the
 * reference's exact integer semantics:
 *   - murmur3 pair hash, 31-bit mask      hashing.py:65-86, 97-101
 *   - membership (X[r] ^ h) < thr, strict hashing.py:141-150, propagation.py:170
 *   - min-label propagation to fixpoint   propagation.py:166-221 (dense pull
 *     sweeps; the reference's index/sparse sweeps reach the same fixpoint)
 *   - component sizes and int64 gains     propagation.py:371-390
 *   - CELF with a (-gain, id) min-heap    selection.py:115-149
 *   - config-scale checker: union-find labels per lane (oracles.py:112-133),
 *     lane-chunked sizes + fresh-gain tables, and the same CELF heap driven
 *     by the fresh-gain table (selection.py:63-70, 115-149)
 *
 * Threads: the lanes are independent samples, so lane blocks are split over
 * OpenMP threads; each thread runs its own lanes to their fixpoint in place
 * (Gauss-Seidel order inside a block, like the reference's in-place block
 * updates).  Results do not depend on the thread count.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline uint32_t rotl32(uint32_t x, int r) { return (x << r) | (x >> (32 - r)); }

/* murmur3_x86_32 of LE32(lo) || LE32(hi), seed 0 (hashing.py:65-86) */
uint32_t oracle_murmur3_pair(uint32_t lo, uint32_t hi) {
    const uint32_t c1 = 0xCC9E2D51u, c2 = 0x1B873593u;
    uint32_t h = 0, blocks[2] = {lo, hi};
    for (int i = 0; i < 2; ++i) {
        uint32_t k = blocks[i] * c1;
        k = rotl32(k, 15) * c2;
        h = rotl32(h ^ k, 13) * 5u + 0xE6546B64u;
    }
    h ^= 8u;
    h ^= h >> 16; h *= 0x85EBCA6Bu;
    h ^= h >> 13; h *= 0xC2B2AE35u;
    return h ^ (h >> 16);
}

/* build_hash_table (hashing.py:97-101): per slot hash of (min, max) & H_MAX */
void oracle_hash_table(int64_t n, const int64_t *xadj, const int32_t *adj, int32_t *out) {
    for (int64_t u = 0; u < n; ++u)
        for (int64_t s = xadj[u]; s < xadj[u + 1]; ++s) {
            uint32_t a = (uint32_t)u, b = (uint32_t)adj[s];
            out[s] = (int32_t)(oracle_murmur3_pair(a < b ? a : b, a < b ? b : a) & 0x7FFFFFFFu);
        }
}

/* One lane block [r0, r1) of the dense pull propagation, to its fixpoint.
 * labels is the full (n, W) matrix; returns the number of sweeps run
 * (including the final no-change sweep). */
static int propagate_block(int64_t n, const int64_t *xadj, const int32_t *adj,
                           const int32_t *hashes, const int32_t *thr, int32_t thr_uniform,
                           int uniform, const int32_t *X, int64_t W, int r0, int r1,
                           int32_t *labels, int64_t *changed_total) {
    const int B = r1 - r0;
    int32_t *best = (int32_t *)malloc(sizeof(int32_t) * (size_t)B);
    int sweeps = 0;
    int64_t changed;
    do {
        changed = 0;
        for (int64_t v = 0; v < n; ++v) {
            const int64_t s0 = xadj[v], s1 = xadj[v + 1];
            if (s0 == s1) continue;
            int32_t *lv = labels + v * W + r0;
            for (int j = 0; j < B; ++j) best[j] = lv[j];
            for (int64_t s = s0; s < s1; ++s) {
                const int32_t h = hashes[s];
                const int32_t t = uniform ? thr_uniform : thr[s];
                const int32_t *lu = labels + (int64_t)adj[s] * W + r0;
                const int32_t *x = X + r0;
                for (int j = 0; j < B; ++j) {
                    const int live = (x[j] ^ h) < t;            /* strict, signed */
                    const int32_t c = live ? lu[j] : INT32_MAX;
                    best[j] = c < best[j] ? c : best[j];
                }
            }
            for (int j = 0; j < B; ++j)
                if (best[j] < lv[j]) { lv[j] = best[j]; ++changed; }
        }
        *changed_total += changed;
        ++sweeps;
    } while (changed);
    free(best);
    return sweeps;
}

/* propagate (propagation.py:260-321): labels (n, W) int32 min-id labels.
 * thr may be NULL when uniform (thr_uniform used).  Returns the max sweep
 * count over lane blocks; *changed = total label decreases. */
int oracle_propagate(int64_t n, const int64_t *xadj, const int32_t *adj,
                     const int32_t *hashes, const int32_t *thr, int32_t thr_uniform,
                     const int32_t *X, int64_t W, int32_t *labels, int nthreads,
                     int lane_block, int64_t *changed) {
    for (int64_t v = 0; v < n; ++v)
        for (int64_t r = 0; r < W; ++r) labels[v * W + r] = (int32_t)v;
    if (changed) *changed = 0;
    if (xadj[n] == 0) return 0;
    if (lane_block <= 0) lane_block = 64;
    const int nblocks = (int)((W + lane_block - 1) / lane_block);
    int max_sweeps = 0;
    int64_t total = 0;
    const int uniform = thr == NULL;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1) reduction(max : max_sweeps) reduction(+ : total)
#endif
    for (int b = 0; b < nblocks; ++b) {
        int r0 = b * lane_block;
        int r1 = r0 + lane_block < W ? r0 + lane_block : (int)W;
        int64_t ch = 0;
        int sw = propagate_block(n, xadj, adj, hashes, thr, thr_uniform, uniform, X, W, r0, r1,
                                 labels, &ch);
        if (sw > max_sweeps) max_sweeps = sw;
        total += ch;
    }
    if (changed) *changed = total;
    return max_sweeps;
}

/* component_sizes_and_gains (propagation.py:371-390): sizes (n, W) int32
 * histogram per lane over all W lanes; gains over lanes < num_scored. */
void oracle_sizes_gains(int64_t n, int64_t W, const int32_t *labels, int64_t num_scored,
                        int32_t *sizes, int64_t *gains, int nthreads) {
    memset(sizes, 0, sizeof(int32_t) * (size_t)(n * W));
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#endif
    for (int64_t r = 0; r < W; ++r)
        for (int64_t v = 0; v < n; ++v) sizes[(int64_t)labels[v * W + r] * W + r] += 1;
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
    for (int64_t v = 0; v < n; ++v) {
        int64_t acc = 0;
        for (int64_t r = 0; r < num_scored; ++r) acc += sizes[(int64_t)labels[v * W + r] * W + r];
        gains[v] = acc;
    }
}

/* ---- CELF (selection.py:115-149) --------------------------------------- */
typedef struct { int64_t neg; int32_t v; } hkey;

static inline int hless(hkey a, hkey b) { return a.neg < b.neg || (a.neg == b.neg && a.v < b.v); }

static void sift_down(hkey *h, int64_t len, int64_t i) {
    for (;;) {
        int64_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < len && hless(h[l], h[m])) m = l;
        if (r < len && hless(h[r], h[m])) m = r;
        if (m == i) return;
        hkey t = h[i]; h[i] = h[m]; h[m] = t;
        i = m;
    }
}
static void sift_up(hkey *h, int64_t i) {
    while (i > 0) {
        int64_t p = (i - 1) / 2;
        if (!hless(h[i], h[p])) return;
        hkey t = h[i]; h[i] = h[p]; h[p] = t;
        i = p;
    }
}

/* marginal_gain (selection.py:63-70) */
static int64_t celf_gain(int32_t u, int64_t W, const int32_t *labels, const int32_t *sizes,
                         const uint8_t *owned, int64_t ns) {
    int64_t acc = 0;
    for (int64_t r = 0; r < ns; ++r) {
        int64_t l = labels[(int64_t)u * W + r];
        if (!owned[l * ns + r]) acc += sizes[l * W + r];
    }
    return acc;
}

/* select_seeds: writes k seeds and gains, the trace (5 int64 per dequeue,
 * up to trace_cap records), per_sim[ns] covered totals; returns the number of
 * dequeues, or -1 on bad arguments. */
int64_t oracle_celf(int64_t n, int64_t W, const int32_t *labels, const int32_t *sizes,
                    const int64_t *init_gains, int64_t ns, int32_t k, int32_t *seeds_out,
                    int64_t *gains_out, int64_t *trace, int64_t trace_cap, int64_t *per_sim) {
    if (k < 1 || k > n || ns > W) return -1;
    hkey *heap = (hkey *)malloc(sizeof(hkey) * (size_t)n);
    int64_t *fresh_at = (int64_t *)calloc((size_t)n, sizeof(int64_t));
    uint8_t *owned = (uint8_t *)calloc((size_t)(n * ns), 1);
    for (int64_t v = 0; v < n; ++v) { heap[v].neg = -init_gains[v]; heap[v].v = (int32_t)v; }
    int64_t len = n;
    for (int64_t i = n / 2 - 1; i >= 0; --i) sift_down(heap, len, i);
    int32_t nseeds = 0;
    int64_t ntrace = 0;
    if (per_sim) memset(per_sim, 0, sizeof(int64_t) * (size_t)ns);
    while (nseeds < k) {
        hkey top = heap[0];
        heap[0] = heap[--len];
        sift_down(heap, len, 0);
        const int32_t u = top.v;
        const int64_t stale = -top.neg;
        int64_t rec[5];
        if (fresh_at[u] == nseeds) {
            for (int64_t r = 0; r < ns; ++r) {          /* commit_seed, :73-81 */
                int64_t l = labels[(int64_t)u * W + r];
                if (!owned[l * ns + r]) {
                    owned[l * ns + r] = 1;
                    if (per_sim) per_sim[r] += sizes[l * W + r];
                }
            }
            seeds_out[nseeds] = u;
            gains_out[nseeds] = stale;
            rec[0] = u; rec[1] = stale; rec[2] = stale; rec[3] = 1; rec[4] = nseeds;
            ++nseeds;
        } else {
            int64_t f = celf_gain(u, W, labels, sizes, owned, ns);
            fresh_at[u] = nseeds;
            heap[len].neg = -f; heap[len].v = u;
            sift_up(heap, len++);
            rec[0] = u; rec[1] = stale; rec[2] = f; rec[3] = 0; rec[4] = nseeds;
        }
        if (trace && ntrace < trace_cap) memcpy(trace + 5 * ntrace, rec, sizeof rec);
        ++ntrace;
    }
    free(heap); free(fresh_at); free(owned);
    return ntrace;
}

/* ------------------------------------------------------------------------
 * Config-scale checker: the same fixpoint and the same
 * selection as above, restated so that they run lane chunk by lane chunk on
 * graphs whose full (n, R) matrices do not fit the dense restatement's time
 * budget (C4: 4.19M x 1024, C5: 1M x 8192).
 * ------------------------------------------------------------------------ */

/* Component labels by union-find over the live edges of each lane -- the
 * reference's own independent label oracle is a per-lane BFS
 * (oracles.py:112-133, bfs_component_labels); any exact CC algorithm reaches
 * the unique fixpoint of propagate (propagation.py:1-8: every vertex gets
 * the minimum id of its component).  Roots are kept minimal (the larger root
 * is linked under the smaller), so find(v) is that minimum.  Membership is
 * the reference's strict signed (X[r] ^ h) < thr (hashing.py:141-150), each
 * undirected edge tested once from its lower endpoint's row.  Lanes are
 * processed 8 at a time per thread (one parent array per lane). */
static inline int32_t uf_find(int32_t *p, int32_t x) {
    while (p[x] != x) { p[x] = p[p[x]]; x = p[x]; }
    return x;
}

void oracle_uf_labels(int64_t n, const int64_t *xadj, const int32_t *adj, const int32_t *hashes,
                      const int32_t *thr, int32_t thr_uniform, const int32_t *X, int64_t W,
                      int32_t *labels, int nthreads) {
    enum { B = 8 };
    const int64_t nblocks = (W + B - 1) / B;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel
    {
        int32_t *par = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n ? n : 1) * B);
#pragma omp for schedule(dynamic, 1)
        for (int64_t b = 0; b < nblocks; ++b) {
            const int64_t r0 = b * B, nb = (W - r0) < B ? (W - r0) : B;
            int32_t x[B];
            for (int j = 0; j < B; ++j) x[j] = j < nb ? X[r0 + j] : 0;
            for (int j = 0; j < nb; ++j)
                for (int64_t v = 0; v < n; ++v) par[j * n + v] = (int32_t)v;
            for (int64_t v = 0; v < n; ++v) {
                for (int64_t s = xadj[v]; s < xadj[v + 1]; ++s) {
                    const int32_t u = adj[s];
                    if (u <= v) continue;                 /* each undirected edge once */
                    const int32_t h = hashes[s], t = thr ? thr[s] : thr_uniform;
                    unsigned live = 0;
                    for (int j = 0; j < B; ++j) live |= (unsigned)((x[j] ^ h) < t) << j;
                    live &= (1u << nb) - 1u;
                    while (live) {
                        const int j = __builtin_ctz(live);
                        live &= live - 1;
                        int32_t *p = par + j * n;
                        int32_t a = uf_find(p, (int32_t)v), c = uf_find(p, u);
                        if (a == c) continue;
                        if (a < c) p[c] = a; else p[a] = c;
                    }
                }
            }
            for (int j = 0; j < nb; ++j) {
                int32_t *p = par + j * n;
                for (int64_t v = 0; v < n; ++v) labels[v * W + r0 + j] = uf_find(p, (int32_t)v);
            }
        }
        free(par);
    }
}

/* One lane chunk of the selection check.  labels / sizes are this chunk's
 * (n, W) columns, lanes [0, ns) of it scored.  Given the claimed seed
 * sequence seeds[0..K), component c of lane r is covered from step
 * cs(c, r) = min{t : labels[seeds[t]][r] == c} on (K if never).  The
 * reference's marginal_gain (selection.py:63-70) of v at step t -- given
 * S_<t = seeds[0..t) -- sums size(comp(v, r)) over the lanes where
 * t <= cs(comp(v, r), r); it is accumulated as a difference table
 * D[(K+1) x n] (D[0][v] += size, D[cs+1][v] -= size), so the prefix sums
 * over t of all chunks' D give every fresh gain of every step.  sizes_out
 * is component_sizes (propagation.py:349-356) of the chunk; per_sim[r]
 * (lanes < ns) counts the vertices covered after all K seeds
 * (SelectionResult.spread_se, selection.py:106-112). */
void oracle_chunk_cover(int64_t n, int64_t W, const int32_t *labels, int64_t ns, const int32_t *seeds,
                        int32_t K, int32_t *sizes_out, int64_t *D, int64_t *per_sim, int nthreads) {
    int32_t *cs = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n * W > 0 ? n * W : 1));
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n * W; ++i) { sizes_out[i] = 0; cs[i] = K; }
    /* rows in order (each label row read once, contiguous); the histogram
     * scatters into row labels[v][r] <= v */
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < n; ++v)
        for (int64_t r = 0; r < W; ++r) {
#pragma omp atomic
            sizes_out[(int64_t)labels[v * W + r] * W + r] += 1;
        }
    for (int32_t t = K - 1; t >= 0; --t)
        for (int64_t r = 0; r < W; ++r) cs[(int64_t)labels[(int64_t)seeds[t] * W + r] * W + r] = t;
    for (int64_t r = 0; r < ns; ++r) per_sim[r] = 0;
#pragma omp parallel
    {
        int64_t *cov = (int64_t *)calloc((size_t)(ns > 0 ? ns : 1), sizeof(int64_t));
#pragma omp for schedule(static)
        for (int64_t v = 0; v < n; ++v) {
            for (int64_t r = 0; r < ns; ++r) {
                const int64_t l = labels[v * W + r];
                const int64_t sz = sizes_out[l * W + r];
                const int32_t c = cs[l * W + r];
                D[v] += sz;
                if (c < K) { D[(int64_t)(c + 1) * n + v] -= sz; cov[r] += 1; }
            }
        }
#pragma omp critical
        for (int64_t r = 0; r < ns; ++r) per_sim[r] += cov[r];
        free(cov);
    }
    free(cs);
}

/* select_seeds (selection.py:115-149) driven by a table of fresh gains:
 * F[t][v] = marginal_gain(v) given the first t seeds (t < K).  The heap,
 * fresh_at rule and trace are exactly oracle_celf's; only marginal_gain is a
 * table lookup.  Returns the number of dequeues (trace records). */
int64_t oracle_celf_fresh(int64_t n, int32_t k, const int64_t *F, int32_t *seeds_out, int64_t *gains_out,
                          int64_t *trace, int64_t trace_cap) {
    if (k < 1 || k > n) return -1;
    hkey *heap = (hkey *)malloc(sizeof(hkey) * (size_t)n);
    int64_t *fresh_at = (int64_t *)calloc((size_t)n, sizeof(int64_t));
    for (int64_t v = 0; v < n; ++v) { heap[v].neg = -F[v]; heap[v].v = (int32_t)v; }
    int64_t len = n;
    for (int64_t i = n / 2 - 1; i >= 0; --i) sift_down(heap, len, i);
    int32_t nseeds = 0;
    int64_t ntrace = 0;
    while (nseeds < k) {
        hkey top = heap[0];
        heap[0] = heap[--len];
        sift_down(heap, len, 0);
        const int32_t u = top.v;
        const int64_t stale = -top.neg;
        int64_t rec[5];
        if (fresh_at[u] == nseeds) {
            seeds_out[nseeds] = u;
            gains_out[nseeds] = stale;
            rec[0] = u; rec[1] = stale; rec[2] = stale; rec[3] = 1; rec[4] = nseeds;
            ++nseeds;
        } else {
            const int64_t f = F[(int64_t)nseeds * n + u];
            fresh_at[u] = nseeds;
            heap[len].neg = -f; heap[len].v = u;
            sift_up(heap, len++);
            rec[0] = u; rec[1] = stale; rec[2] = f; rec[3] = 0; rec[4] = nseeds;
        }
        if (trace && ntrace < trace_cap) memcpy(trace + 5 * ntrace, rec, sizeof rec);
        ++ntrace;
    }
    free(heap); free(fresh_at);
    return ntrace;
}

/* ------------------------------------------------------------------------
 * Config graphs on the host at C4 scale (the CPU reference arm's setup and
 * the tests' host CSR): the repo's counter-based generator
 * (paper_2008_03095_b200/generators.py, restated here in C) and
 * Graph.from_edges (graph.py:124-155) for a sorted unique edge-key list.
 * ------------------------------------------------------------------------ */
static inline uint64_t g_mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static inline double g_unit(uint64_t r) { return (double)(r >> 11) * (1.0 / 9007199254740992.0); }
static inline uint64_t g_below(uint64_t r, uint64_t n) {
    return ((r >> 32) * n + (((r & 0xFFFFFFFFull) * n) >> 32)) >> 32;
}

/* candidate keys lo * n + hi (UINT64_MAX for self-loops) of draws
 * [first, first + count): kind 0 ER, 1 R-MAT (probs a, b, c, d), 2 Chung-Lu
 * (cdf[n]) -- generators.py _candidates */
void oracle_gen_candidates(int kind, int64_t n, uint64_t seed, int64_t first, int64_t count,
                           const double *probs, const double *cdf, uint64_t *out, int nthreads) {
    const uint64_t ms = g_mix64(seed), nn = (uint64_t)n;
    int scale = 0;
    while ((2ll << scale) <= n) ++scale;
    double ca = 0, cb = 0, cc = 0;
    if (kind == 1) {
        const double tot = probs[0] + probs[1] + probs[2] + probs[3];
        ca = probs[0] / tot; cb = (probs[0] + probs[1]) / tot; cc = (probs[0] + probs[1] + probs[2]) / tot;
    }
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#endif
    for (int64_t j = 0; j < count; ++j) {
        const uint64_t i = (uint64_t)(first + j);
        uint64_t u = 0, v = 0;
        if (kind == 0) {
            u = g_below(g_mix64(ms ^ (2 * i)), nn);
            v = g_below(g_mix64(ms ^ (2 * i + 1)), nn);
        } else if (kind == 1) {
            for (int l = 0; l < scale; ++l) {
                const double x = g_unit(g_mix64(ms ^ (64 * i + (uint64_t)l)));
                const uint64_t down = x >= cb, right = (x >= ca && x < cb) || x >= cc;
                u = (u << 1) | down;
                v = (v << 1) | right;
            }
        } else {
            const double x1 = g_unit(g_mix64(ms ^ (2 * i))), x2 = g_unit(g_mix64(ms ^ (2 * i + 1)));
            int64_t lo = 0, hi = n;                    /* searchsorted(cdf, x, 'right') */
            while (lo < hi) { int64_t m = (lo + hi) >> 1; if (cdf[m] <= x1) lo = m + 1; else hi = m; }
            u = (uint64_t)(lo < n - 1 ? lo : n - 1);
            lo = 0; hi = n;
            while (lo < hi) { int64_t m = (lo + hi) >> 1; if (cdf[m] <= x2) lo = m + 1; else hi = m; }
            v = (uint64_t)(lo < n - 1 ? lo : n - 1);
        }
        out[j] = u == v ? UINT64_MAX : (u < v ? u : v) * nn + (u < v ? v : u);
    }
}

/* Graph.from_edges (graph.py:124-155) of m unique undirected edges given as
 * keys lo * n + hi in ascending order: rows sorted by (src, dst).  In key
 * order every edge (l, v) with l < v precedes every edge (v, h), so one pass
 * appending to per-row cursors writes each row already sorted. */
void oracle_csr_from_sorted_keys(int64_t n, int64_t m, const uint64_t *keys, int64_t *xadj, int32_t *adj) {
    memset(xadj, 0, sizeof(int64_t) * (size_t)(n + 1));
    for (int64_t e = 0; e < m; ++e) {
        ++xadj[keys[e] / (uint64_t)n + 1];
        ++xadj[keys[e] % (uint64_t)n + 1];
    }
    for (int64_t v = 0; v < n; ++v) xadj[v + 1] += xadj[v];
    int64_t *cur = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    memcpy(cur, xadj, sizeof(int64_t) * (size_t)n);
    for (int64_t e = 0; e < m; ++e) {
        const int64_t lo = (int64_t)(keys[e] / (uint64_t)n), hi = (int64_t)(keys[e] % (uint64_t)n);
        adj[cur[lo]++] = (int32_t)hi;
        adj[cur[hi]++] = (int32_t)lo;
    }
    free(cur);
}

/* ------------------------------------------------------------------------
 * evaluate_seeds worker (evaluation.py:70-98, 101-136): world j of chunk c
 * draws E doubles from numpy PCG64 stream c (state/inc given by the caller,
 * taken from default_rng(SeedSequence(seed).spawn(..)[c])), starting at
 * draw (j mod chunk) * E; edge e is live iff random() < probs[e]; the count
 * is the size of the union of the seed components.  random() is numpy's
 * next_double: (next64 >> 11) * 2^-53; next64 is the XSL-RR output of the
 * 128-bit LCG state after the step (pcg64.h).
 * ------------------------------------------------------------------------ */
typedef unsigned __int128 o_u128;
static inline o_u128 o_pcg_mult(void) {
    return ((o_u128)0x2360ED051FC65DA4ULL << 64) | (o_u128)0x4385DF649FCCF645ULL;
}
static inline uint64_t o_pcg_out(o_u128 s) {
    unsigned rot = (unsigned)(s >> 122);
    uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
    return (x >> rot) | (x << ((64u - rot) & 63u));
}
static o_u128 o_pcg_advance(o_u128 s, o_u128 inc, uint64_t d) {
    o_u128 am = 1, ap = 0, cm = o_pcg_mult(), cp = inc;
    while (d) {
        if (d & 1) { am *= cm; ap = ap * cm + cp; }
        cp = (cm + 1) * cp; cm *= cm; d >>= 1;
    }
    return am * s + ap;
}
static int32_t o_find(int32_t *par, int32_t x) {
    while (par[x] != x) { par[x] = par[par[x]]; x = par[x]; }
    return x;
}

void oracle_evaluate(int64_t n, int64_t E, const int32_t *cu, const int32_t *cv, const double *probs,
                     const int32_t *seeds, int32_t k, int64_t r_eval, const uint64_t *streams,
                     int64_t chunk, int64_t *counts, int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
    const o_u128 M = o_pcg_mult();
#pragma omp parallel
    {
        int32_t *par = (int32_t *)malloc(sizeof(int32_t) * (n ? n : 1));
        int64_t *sz = (int64_t *)malloc(sizeof(int64_t) * (n ? n : 1));
        int64_t *stamp = (int64_t *)malloc(sizeof(int64_t) * (n ? n : 1));
        for (int64_t v = 0; v < n; ++v) stamp[v] = -1;
#pragma omp for schedule(dynamic, 16)
        for (int64_t j = 0; j < r_eval; ++j) {
            const uint64_t *sv = streams + 4 * (j / chunk);
            const o_u128 inc = ((o_u128)sv[2] << 64) | sv[3];
            o_u128 s = o_pcg_advance(((o_u128)sv[0] << 64) | sv[1], inc, (uint64_t)(j % chunk) * (uint64_t)E);
            for (int64_t v = 0; v < n; ++v) { par[v] = (int32_t)v; sz[v] = 1; }
            for (int64_t e = 0; e < E; ++e) {
                s = s * M + inc;
                const double u = (double)(o_pcg_out(s) >> 11) * (1.0 / 9007199254740992.0);
                if (!(u < probs[e])) continue;
                int32_t a = o_find(par, cu[e]), b = o_find(par, cv[e]);
                if (a == b) continue;
                if (sz[a] < sz[b]) { int32_t t = a; a = b; b = t; }
                par[b] = a;
                sz[a] += sz[b];
            }
            int64_t tot = 0;
            for (int32_t i = 0; i < k; ++i) {
                const int32_t r = o_find(par, seeds[i]);
                if (stamp[r] != j) { stamp[r] = j; tot += sz[r]; }
            }
            counts[j] = tot;
        }
        free(par); free(sz); free(stamp);
    }
}
