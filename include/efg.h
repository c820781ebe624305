/*
 * efg.h -- C ABI of the B200-native Expected Force engine (libefg.so).
 *
 * Plain pointers and sizes only; no torch or CUDA types except an opaque
 * `void*` stream.  Status codes: 0 ok, 1 invalid argument (-> ValueError),
 * 2 CUDA error, 3 NCCL error, 4 out of memory.  efg_last_error() returns the
 * calling thread's last message.  Caller owns every input and output buffer
 * (outputs pre-allocated, e.g. np.empty); the library owns device memory
 * through the opaque context.  Calls on one context are serialised by an
 * internal mutex.
 *
 * Each entry point cites the reference interface it replaces
 * (paths relative to /root/reference/pkg/src/efgraph/).
 */
#ifndef EFG_H
#define EFG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EFG_ABI_VERSION 1

#if defined(__GNUC__)
#define EFG_API __attribute__((visibility("default")))
#else
#define EFG_API
#endif

typedef struct efg_ctx efg_ctx;

/* mode: expected_force.py:114-120 (`ef(g, mode=...)`) */
enum { EFG_MODE_CLUSTER_CENTRIC = 0, EFG_MODE_VERTEX_CENTRIC = 1 };

/* engine: which device algorithm evaluates the per-seed cluster sums.
 *  FACTORIZED -- degree-histogram factorisation + triangle corrections (default)
 *  DIRECT     -- per-seed enumeration of every star and chain (original formulation)
 *  ALG1       -- Algorithm-1 middle-triplet scatter, an independent
 *                cross-check (fp64 W summed by atomics: EF may vary in the last bits) */
enum { EFG_ENGINE_AUTO = 0, EFG_ENGINE_FACTORIZED = 1, EFG_ENGINE_DIRECT = 2, EFG_ENGINE_ALG1 = 3 };

typedef struct efg_stats {
    double ms_device;            /* device time of the whole call (CUDA events) */
    double ms_prepare;           /* degrees, neighbour degrees, F table, orientation */
    double ms_enumerate;         /* cluster sums (the hot kernels) */
    double ms_h2d;               /* host->device copies (host-buffer entry points) */
    double ms_d2h;               /* device->host copies */
    int64_t clusters_processed;  /* reference semantics: sum C(d,2), x3 in vertex mode */
    int64_t cluster_visits;      /* clusters represented: 3 * sum C(d,2) */
    int64_t terms;               /* pair terms evaluated by the engine */
    int64_t bytes_alg;           /* 16*sumC + 64*m + 33*n */
    int64_t launches;            /* kernels launched by the library in this call */
    int64_t h2d_bytes, d2h_bytes;
    int32_t engine;
    int32_t dmax;
} efg_stats;

EFG_API int efg_abi_version(void);
EFG_API const char *efg_last_error(void);

/* Context on CUDA device `device` with a library-owned non-blocking stream. */
EFG_API int efg_create(int device, efg_ctx **out);
EFG_API int efg_destroy(efg_ctx *ctx);
/* Use a caller-provided cudaStream_t (NULL restores the library's own). */
EFG_API int efg_set_stream(efg_ctx *ctx, void *stream);
EFG_API int efg_synchronize(efg_ctx *ctx);

/* K1: replaces graph.py:147-190 `build_graph(edges)`.  `edges` is k host
 * (u, v) int64 pairs.  The CSR stays resident in the context; sizes out. */
EFG_API int efg_build_graph(efg_ctx *ctx, const int64_t *edges, int64_t k, int64_t *n_out, int64_t *m_out);
/* Copy the resident CSR out: offsets[n+1], neighbors[2m], orig_ids[n]
 * (the Graph fields of graph.py:34-57). */
EFG_API int efg_fetch_graph(efg_ctx *ctx, int64_t *offsets, int32_t *neighbors, int64_t *orig_ids);
/* Device R-MAT sampler, bit-identical to graph.py:204-246 `generate_rmat`
 * (numpy PCG64 double stream, first-`target`-distinct-code semantics, attempt
 * cap 20*target).  probs[4] are the quadrant probabilities; pcg_state and
 * pcg_inc are the 128-bit PCG64 state/increment of np.random.default_rng(seed)
 * as {low 64 bits, high 64 bits}.  The CSR stays resident like
 * efg_build_graph's; *truncated = 1 when the cap was hit. */
EFG_API int efg_rmat_build(efg_ctx *ctx, int32_t scale, int64_t avg_degree, const double *probs,
                           const uint64_t *pcg_state, const uint64_t *pcg_inc, int32_t *truncated,
                           int64_t *n_out, int64_t *m_out);

/* Device pointers of the resident CSR (valid until the next build). */
EFG_API int efg_graph_device(efg_ctx *ctx, const int64_t **d_offsets, const int32_t **d_neighbors,
                     int64_t *n_out, int64_t *m_out);

/* Replaces expected_force.py:114-120 `ef`, :138-174 `ef_cluster_centric` and
 * :345-418 `ef_vertex_centric` for a host CSR (offsets[n+1], neighbors[2m]).
 * Outputs (host, length n): ef f64, cluster_total i64, flags u8;
 * *clusters_processed per the reference mode semantics.  T_out (exact
 * int64 sum w*d) and W_out (f64 sum w*d*ln d) are optional (NULL). */
EFG_API int efg_expected_force(efg_ctx *ctx, const int64_t *offsets, const int32_t *neighbors, int64_t n,
                       int32_t mode, int32_t engine, double *ef, int64_t *cluster_total,
                       uint8_t *flags, int64_t *clusters_processed, int64_t *T_out, double *W_out,
                       efg_stats *stats);

/* Device-resident variant: every pointer is device memory; computes seeds
 * [seed_lo, seed_hi) of the graph and writes outputs at index seed - seed_lo.
 * Asynchronous on the context stream when stats == NULL. */
EFG_API int efg_expected_force_device(efg_ctx *ctx, const int64_t *d_offsets, const int32_t *d_neighbors,
                              int64_t n, int64_t seed_lo, int64_t seed_hi, int32_t engine,
                              double *d_ef, int64_t *d_cluster_total, uint8_t *d_flags,
                              int64_t *d_T, double *d_W, efg_stats *stats);

/* K2: balanced contiguous seed shards for `parts` devices by the engine's
 * per-seed work prefix (bounds_out[parts+1], host).  Independent of which
 * device runs which shard, so results are identical for any device count. */
EFG_API int efg_shard_bounds(efg_ctx *ctx, const int64_t *d_offsets, const int32_t *d_neighbors, int64_t n,
                     int32_t engine, int32_t parts, int64_t *bounds_out);

/* Distributed whole-graph pass (factorized engine, one part per device; no
 * reference counterpart -- it replaces the reference's thread-pool merge,
 * expected_force.py:158-172).  Part p owns the contiguous
 * node range [bounds[p], bounds[p+1]) of efg_part_bounds (balanced by row
 * work; identical on every rank): its rows' neighbour degrees, S1/S2,
 * label-sorted Adj+ rows, chain tables and pushes.  The triangle listing is
 * split by work unit (every nparts-th).  Every part writes EFG_DIST_WORDS
 * uint64 words per node (d_words[EFG_DIST_WORDS * n]: exact integer sums, own
 * rows / own units only) and f64 stars terms (d_ws[n], own rows only); the
 * caller sums both over all parts (one all-reduce: integer addition and
 * disjoint supports, so exact and order-free), then efg_ef_finish produces
 * the outputs of seeds [seed_lo, seed_hi).  Bitwise equal to
 * efg_expected_force_device for any nparts.
 *
 * Row-partitioned form (per-rank work ~ 1/nparts of the whole pass), three
 * calls on one context:
 *   efg_ef_partial_rows -- the part's rows: neighbour degrees, S1/S2, its
 *     label-sorted Adj+ rows into the caller's slot-space buffer d_adjp[2m]
 *     (row v at [offsets[v], offsets[v] + dplus[v])) and |Adj+(v)| into
 *     d_dplus[n]; clears the words;
 *   (caller: every part broadcasts its slot range [offsets[bounds[p]],
 *    offsets[bounds[p+1]]) of d_adjp and node range of d_dplus, so that every
 *    rank holds all rows -- asynchronously, while the next call runs)
 *   efg_ef_partial_tables -- the part's histograms, chain tables and pushes;
 *   efg_ef_partial_list -- the part's listing units on the exchanged rows.
 * The tables and listing calls add into the words the rows call cleared.
 * Self-contained form: efg_ef_partial runs both with every row's orientation
 * prepared locally (no exchange; more work per rank). */
#define EFG_DIST_WORDS 9
EFG_API int efg_part_bounds(efg_ctx *ctx, const int64_t *d_offsets, const int32_t *d_neighbors, int64_t n,
                            int32_t nparts, int64_t *bounds_out);
EFG_API int efg_ef_partial(efg_ctx *ctx, const int64_t *d_offsets, const int32_t *d_neighbors, int64_t n,
                           int32_t part, int32_t nparts, uint64_t *d_words, double *d_ws, efg_stats *stats);
EFG_API int efg_ef_partial_rows(efg_ctx *ctx, const int64_t *d_offsets, const int32_t *d_neighbors, int64_t n,
                                int32_t part, int32_t nparts, const int64_t *bounds, int32_t *d_adjp,
                                int32_t *d_dplus, uint64_t *d_words, double *d_ws, efg_stats *stats);
EFG_API int efg_ef_partial_tables(efg_ctx *ctx, const int64_t *d_offsets, const int32_t *d_neighbors, int64_t n,
                                  int32_t part, int32_t nparts, const int64_t *bounds, uint64_t *d_words,
                                  double *d_ws, efg_stats *stats);
EFG_API int efg_ef_partial_list(efg_ctx *ctx, const int64_t *d_offsets, const int32_t *d_neighbors, int64_t n,
                                int32_t part, int32_t nparts, const int64_t *bounds, int32_t *d_adjp,
                                int32_t *d_dplus, uint64_t *d_words, double *d_ws, efg_stats *stats);
EFG_API int efg_ef_finish(efg_ctx *ctx, const int64_t *d_offsets, const int32_t *d_neighbors, int64_t n,
                          int64_t seed_lo, int64_t seed_hi, const uint64_t *d_words, const double *d_ws,
                          double *d_ef, int64_t *d_cluster_total, uint8_t *d_flags, int64_t *d_T, double *d_W);

/* K5: key-node ranking -- the k largest EF values, ties to the smaller id,
 * i.e. np.lexsort((ids, -ef))[:k] (cf. analysis.py:101, :240).  ids_out is
 * host int64[k].  The _device form reads a device ef array. */
EFG_API int efg_topk(efg_ctx *ctx, const double *ef, int64_t n, int64_t k, int64_t *ids_out);
EFG_API int efg_topk_device(efg_ctx *ctx, const double *d_ef, int64_t n, int64_t k, int64_t *ids_out);

/* Ranking consumers of K5.
 * efg_rank_ascending: order_out (host int64[n]) = np.argsort(ef, kind="stable"),
 *   the ranking analysis.py:240 (immunization_experiment) cuts windows from.
 * efg_ef_bins: analysis.py:84-103 ef_bins -- k targets equally spaced over
 *   [min ef, max ef] (same IEEE operation order), and per target the node
 *   nearest to it, ties to the lowest id.  Status 1 (ValueError) when k < 1 or
 *   when there are fewer than k distinct values (message names the count). */
EFG_API int efg_rank_ascending(efg_ctx *ctx, const double *ef, int64_t n, int64_t *order_out);
EFG_API int efg_ef_bins(efg_ctx *ctx, const double *ef, int64_t n, int64_t k, double *target_out, int64_t *rep_out);

/* Live per-kernel device timing: when enabled, every kernel launch (and each
 * CUB call) records a CUDA event pair on the launching stream; the report is
 * JSON {"kernel": [total_ms, launches], ...} accumulated since the last reset. */
EFG_API int efg_profile_enable(efg_ctx *ctx, int32_t on);
EFG_API int efg_profile_reset(efg_ctx *ctx);
EFG_API int efg_profile_report(efg_ctx *ctx, char *buf, int64_t cap);
/* The last profiled call's records in issue order as JSON
 * [["name", start_ms, ms], ...], start relative to the call's first record
 * (host->device copies of efg_expected_force appear as "h2d"). */
EFG_API int efg_profile_timeline(efg_ctx *ctx, char *buf, int64_t cap);

/* Host-side row formatter of write_ef_csv (expected_force.py:123-130): for
 * i in [0, n) appends "<orig_ids[i]>,<ef[i] as %.9g>,<cluster_total[i]>\n"
 * (the reference's f-string format: C's %.9g and Python's format(x, ".9g")
 * agree -- both correctly rounded) into buf (capacity cap >= 64 n bytes),
 * rows split over `threads` host threads; *len_out = bytes written.  No
 * device work; loads and runs without a GPU. */
EFG_API int efg_format_ef_csv(const int64_t *orig_ids, const double *ef, const int64_t *cluster_total, int64_t n,
                              int32_t threads, char *buf, int64_t cap, int64_t *len_out);

/* Pinned (page-locked) host memory for zero-staging copies; the Python layer
 * allocates Graph arrays and EF outputs here. */
EFG_API int efg_host_alloc(int64_t bytes, void **out);
EFG_API int efg_host_free(void *p);

#ifdef __cplusplus
}
#endif

#endif /* EFG_H */
