/*
 * mcfunm_cuda.h -- C ABI of the B200 walk-sampling estimator (libmcfunm_cuda.so).
 *
 * Drop-in boundary for the hot path of the reference package `mcfunm`
 * (arXiv 2308.01037).  The reference has no native code and no FFI: its hot
 * path is the per-column Python loop of the (SPEC-only) estimators around
 * walker.run_walks_batch (/root/reference/pkg/src/mcfunm/walker.py:245-290) with
 * a per-step Python callback `on_step(k, states, weights, ids)` that cannot
 * cross a device boundary.  Each entry point below replaces one piece of that
 * path; the replaced reference interface is cited per function.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Array arguments marked [dev] are CUDA
 *    device pointers owned by the caller (e.g. torch.Tensor.data_ptr());
 *    [host] pointers are ordinary host memory.
 *  - `stream` is a cudaStream_t passed as void*; 0 = legacy default stream.
 *    Every call is stream-ordered; calls that must return a host-visible
 *    value synchronise that stream and say so.
 *  - Return value: MCF_OK or an error code that maps 1:1 onto the reference
 *    exception hierarchy (errors.py:8-47); mcf_last_error() gives the message
 *    (thread-local).
 *  - Node ids fit int32 (n < 2^31); nnz < 2^31 (int32 entry indices in replay
 *    streams).  All arithmetic is fp64.
 */
#ifndef MCFUNM_CUDA_H
#define MCFUNM_CUDA_H

#include <stdint.h>

#if defined(__GNUC__)
#define MCF_API __attribute__((visibility("default")))
#else
#define MCF_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes (errors.py:8-47; CLI exit codes SPEC.md:623). */
#define MCF_OK 0
#define MCF_ERR_ARGUMENT 1    /* errors.ArgumentError: bad parameters (walker.py:60-67) */
#define MCF_ERR_DEGENERATE 2  /* errors.DegenerateInputError: nnz == 0 (walker.py:100-103) */
#define MCF_ERR_CONVERGENCE 3 /* errors.ConvergenceError */
#define MCF_ERR_RESOURCE 4    /* errors.ResourceError: device out of memory */
#define MCF_ERR_CUDA 5        /* any other CUDA failure (kernel fault, no device) */

/* mcf_walk_params.flags */
#define MCF_FLAG_NONE 0
#define MCF_FLAG_TIME_KERNELS 1 /* bracket the walk / Q-build kernels with CUDA events
                                   (read with mcf_graph_kernel_times) */
#define MCF_FLAG_RETURN_ONLY 2  /* action walks accumulate zeta W only at emissions where the walk is
                                   back at its start node (classic MC diagonal, Alg. 1) */

/* Run only the walks w (index inside their column) with w = g mod G, every
 * other walk contributing nothing (W0 stays 1/N_c): the G group estimates of
 * a diag or action pass sum to the full estimate, and their spread gives the
 * standard error (batch means; SPEC.md:410 asks for a per-walk SE).  G in
 * [1, 256] and g < G are packed with MCF_GROUP_FLAGS.  Device-RNG walks only. */
#define MCF_FLAG_WALK_GROUP 4
#define MCF_GROUP_FLAGS(G, g) (MCF_FLAG_WALK_GROUP | ((((G) - 1) & 0xff) << 8) | (((g) & 0xff) << 16))
#define MCF_GROUP_COUNT(flags) ((((flags) >> 8) & 0xff) + 1)
#define MCF_GROUP_INDEX(flags) (((flags) >> 16) & 0xff)
typedef struct mcf_graph mcf_graph;

/* Square sparse matrix in both CSR and CSC form, already scaled by gamma
 * (sparsemat.py:29-100, scale() sparsemat.py:338-352).  Column ids inside each
 * row (row ids inside each column) must be sorted.  For a symmetric matrix the
 * csc_* pointers may alias the csr ones. */
typedef struct {
    int64_t n;
    int64_t nnz;
    const int64_t *row_ptr;  /* [dev] n+1 */
    const int32_t *col_ids;  /* [dev] nnz */
    const double *vals;      /* [dev] nnz */
    const int64_t *csc_ptr;  /* [dev] n+1 */
    const int32_t *csc_rows; /* [dev] nnz */
    const double *csc_vals;  /* [dev] nnz */
} mcf_csr;

/* Host-visible facts about a built graph. */
typedef struct {
    int64_t n;
    int64_t nnz;
    int64_t n_uniform_rows;   /* rows whose |a_ij| are all equal (index sampling) */
    int64_t n_empty_rows;     /* absorbing rows (walker.py:274-278) */
    int64_t n_negative;       /* stored entries with a < 0 */
    int64_t max_degree;
    double max_row_abs_sum;   /* sqrt(alpha_diagnostic) (walker.py:293-302) */
    double col_norm_total;    /* sum_j ||C_j||_2 (walker.py:128) */
    int64_t walk_layout;      /* 0: compact (entry id, then the target's 32-B header: two random
                                 sectors per step); 1: fat (target header copied into every
                                 entry: one random sector per step, 32 B x nnz) */
} mcf_graph_info;

/* Walk termination and RNG (WalkConfig, walker.py:44-67) plus the series. */
typedef struct {
    int64_t max_steps;       /* hard cap m_max >= 1 */
    double weight_cutoff;    /* W_c in (0,1): walk stops once |W| <= W_c * W0 */
    uint64_t seed;           /* Philox key; stream per (seed, column, walk, step) */
    const double *zeta;      /* [dev] max_steps + 2 coefficients zeta_0.. (series.py:69-80) */
    int64_t walk_capacity;   /* upper bound on the walks of the column range (e.g. N_s);
                                0 = read the exact count (synchronises the stream) */
    int32_t flags;
} mcf_walk_params;

/* Device-side counters, int64[4], accumulated (never reset) by walk calls:
 * [0] walks run, [1] emissions (= reference WalkOutcome.steps), [2] walks
 * truncated by max_steps, [3] walks absorbed in an empty row. */
#define MCF_STATS_LEN 4

MCF_API const char *mcf_version(void);
MCF_API const char *mcf_last_error(void);

/* Cumulative number of kernels this library has launched in the process
 * (benchmark accounting; no reference counterpart). */
MCF_API int64_t mcf_kernel_launches(void);

/* Build the device transition tables for `csr` (replaces
 * walker.build_transition_model, walker.py:97-145): per-row |a| sums in CSR
 * order, uniform-row flags, within-row CDFs for weighted rows, column norms
 * ||C_j||_2 and the start distribution p_j (walker.py:127-129, reproduced
 * bit-for-bit).  Keeps the caller's arrays by pointer: they must outlive the
 * handle.  Synchronises `stream`.  nnz == 0 -> MCF_ERR_DEGENERATE. */
MCF_API int mcf_graph_create(const mcf_csr *csr, void *stream, mcf_graph **out);
MCF_API int mcf_graph_destroy(mcf_graph *g);
MCF_API int mcf_graph_get_info(const mcf_graph *g, mcf_graph_info *info);

/* Copy derived tables out ([dev] n each; any pointer may be NULL):
 * row |a| sums (sparsemat.row_abs_sums), column norms, start probabilities. */
MCF_API int mcf_graph_tables(const mcf_graph *g, double *row_abs_sum, double *col_norms,
                     double *init_prob, void *stream);

/* Per-column walk budgets N_i = floor(p_i N_s) + largest-remainder correction,
 * ties by ascending index, p_i = 0 -> 0 (replaces walker.allocate_walks /
 * largest_remainder, walker.py:148-170; identical output).  Writes ni[n] and
 * walk_pre[n+1] = exclusive prefix sum of ni ([dev] int64). */
MCF_API int mcf_allocate_walks(mcf_graph *g, int64_t n_walks, int64_t *ni, int64_t *walk_pre, void *stream);

/* y = alpha * v + beta * r + A x over rows [row_begin, row_end) ([dev] n; v, r
 * may be NULL).  With alpha = beta = 0 this is r = A v; with
 * (zeta_0, zeta_1, q) it is the Alg. 3 combine y = z0 v + z1 r + A q
 * (PAPER.md:362).  x = NULL means x = 1 with alpha = beta = 0: y = A 1 as
 * row sums in CSR order, bit-identical to the reference's A @ ones (what
 * mcf_funm_action uses for v = 1; the general x path sums long rows
 * warp-parallel). */
MCF_API int mcf_spmv(mcf_graph *g, double alpha, const double *v, double beta, const double *r,
             const double *x, double *y, int64_t row_begin, int64_t row_end, void *stream);

/* Multi-GPU Alg. 3 combine with the exchange folded in (one process per GPU,
 * one node; replaces all-gather(q) + SpMV + all-gather(y), PAPER.md:362 and
 * SURVEY.md 8(e)): y = alpha v + beta r + A x over rows [row_begin, row_end),
 * gathering x[j] from x_parts[k] for part_bounds[k] <= j < part_bounds[k+1]
 * (each rank's q buffer, mapped with mcf_peer_open) and storing every row to
 * all n_outs buffers y_outs[k] (every rank's y).  1 <= n_parts, n_outs <= 8;
 * pointer arrays are host memory, the buffers device (local or peer). */
MCF_API int mcf_spmv_peer(mcf_graph *g, double alpha, const double *v, double beta, const double *r,
                          const double *const *x_parts, const int64_t *part_bounds, int n_parts,
                          double *const *y_outs, int n_outs, int64_t row_begin, int64_t row_end, void *stream);

/* Peer buffers: cudaMalloc'd, zero-filled, exported as a 64-byte CUDA IPC
 * handle (mcf_peer_alloc); another process on the node maps it with
 * mcf_peer_open and unmaps with mcf_peer_close; the owner frees it with
 * mcf_peer_free. */
MCF_API int mcf_peer_alloc(int64_t bytes, void **ptr, void *ipc_handle);
MCF_API int mcf_peer_open(const void *ipc_handle, void **ptr);
MCF_API int mcf_peer_close(void *ptr);
MCF_API int mcf_peer_free(void *ptr);

/* Action walks (Alg. 3 inner loops): for
 * every column c in [col_begin, col_end) run N_c = walk_pre[c+1]-walk_pre[c]
 * walks with W0 = 1/N_c and write
 *     q[c] = sum_walks sum_k zeta_{k+2} W_k r[l_k]
 * and, if q_var != NULL, the estimated variance of q[c] from the per-walk
 * contributions.  Replaces the estimator's per-column loop around
 * run_walks_batch (walker.py:245-290) with its on_step accumulation.
 * Counter-based Philox-4x32-10 keyed by (seed, column, walk, step). */
MCF_API int mcf_walk_action(mcf_graph *g, const mcf_walk_params *p, const int64_t *walk_pre,
                    int64_t col_begin, int64_t col_end, const double *r, double *q,
                    double *q_var, int64_t *stats, void *stream);

/* The whole RandFunmAction estimate in one call (Alg. 3, PAPER.md:337-367,
 * SPEC.md:369-377): the budgets for n_walks (-> walk_pre[n+1] and, unless
 * ni is NULL, ni[n], as mcf_allocate_walks), the walks of every column, q,
 * optional q_var, and y = zeta0 v + zeta1 r + A q ([dev] n each).  v may be NULL for v = 1 (total
 * communicability): r is then the row sums of A, bit-identical
 * to the reference's A @ ones.  q, q_var, y and stats[4] are overwritten
 * (unlike mcf_walk_action, stats need not be zeroed).  Single process (the
 * multi-GPU path composes mcf_spmv / mcf_walk_action with an exchange of q).
 * No host synchronisation: capturable in a CUDA graph. */
MCF_API int mcf_funm_action(mcf_graph *g, const mcf_walk_params *p, int64_t n_walks, int64_t *ni,
                            int64_t *walk_pre, const double *v, double zeta0, double zeta1, double *r, double *q,
                            double *q_var, double *y, int64_t *stats, void *stream);

/* Same as mcf_walk_action, but every draw is taken from a recorded entry stream instead of the
 * RNG: walk g = walk_pre[c] + w consumes entries[walk_off[g] .. walk_off[g+1])
 * (global CSR entry indices, step order), exactly the entries the reference
 * batch driver picked (walker.py:280-283).  The device re-derives weights and
 * termination and checks the stream is consumed exactly; synchronises
 * `stream`; a mismatch -> MCF_ERR_ARGUMENT. */
MCF_API int mcf_replay_action(mcf_graph *g, const mcf_walk_params *p, const int64_t *walk_pre,
                      int64_t col_begin, int64_t col_end, const int64_t *walk_off,
                      const int32_t *entries, const double *r, double *q, int64_t *stats,
                      void *stream);

/* Diagonal walks + Eq. 20 partials (Alg. 2):
 * for every column c in [col_begin, col_end) builds Q_c (sum of zeta_{k+2} W_k
 * per visited state, W0 = 1/N_c) and writes, for every stored entry (i, c) of
 * column c, pcol[csc_ptr[c] + t] = a_ic <Q_c, C_i>.  Entries of columns outside
 * the range or with N_c = 0 are left untouched (caller zeroes pcol).
 * Deterministic: Q_c is accumulated in a fixed order. */
MCF_API int mcf_walk_diag(mcf_graph *g, const mcf_walk_params *p, const int64_t *walk_pre,
                  int64_t col_begin, int64_t col_end, double *pcol, int64_t *stats, void *stream);

/* Replay variant of mcf_walk_diag (see mcf_replay_action). Synchronises. */
MCF_API int mcf_replay_diag(mcf_graph *g, const mcf_walk_params *p, const int64_t *walk_pre,
                    int64_t col_begin, int64_t col_end, const int64_t *walk_off,
                    const int32_t *entries, double *pcol, int64_t *stats, void *stream);

/* Dense rows of Q for the full estimator (Alg. 2,
 * Eq. 18-19): Q[(c - col_begin) * ldq + j] = sum over visits of j by the walks
 * from column c of zeta_{k+2} W_k, for c in [col_begin, col_end).  The caller
 * forms f(A) ~ zeta_0 I + zeta_1 A + A Q A block by block (dense GEMMs).
 * Needs n <= 16384 (else MCF_ERR_RESOURCE); synchronises `stream`. */
MCF_API int mcf_walk_qdense(mcf_graph *g, const mcf_walk_params *p, const int64_t *walk_pre, int64_t col_begin,
                            int64_t col_end, double *Q, int64_t ldq, int64_t *stats, void *stream);

/* The full estimate F = zeta_0 I + zeta_1 A + A Q A (Alg. 2 / Eq. 19,
 * SPEC.md:347-356) into the dense row-major F ([dev] n x ldf), Q in blocks of
 * `block` walked columns ("row blocks", default 1024): per block
 * the dense Q rows (as mcf_walk_qdense, transposed), R^T = A^T Q_b^T and
 * F += A[:, block] R, both products over the sparse A (CSC / CSR), fixed
 * summation orders.  walk_pre from mcf_allocate_walks.  n <= 16384 (dense
 * output), else MCF_ERR_RESOURCE; synchronises `stream`. */
MCF_API int mcf_funm_full(mcf_graph *g, const mcf_walk_params *p, const int64_t *walk_pre, double zeta0,
                          double zeta1, double *F, int64_t ldf, int64_t block, int64_t *stats, void *stream);

/* d_i = zeta_0 + zeta_1 a_ii + sum_{c} pcol[(i,c)] for rows [row_begin, row_end)
 * (Eq. 20 final sum), fixed summation order. */
MCF_API int mcf_diag_combine(mcf_graph *g, double zeta0, double zeta1, const double *pcol, double *d,
                     int64_t row_begin, int64_t row_end, void *stream);

/* Estimated variance of d_i for rows [row_begin, row_end) from G >= 2 walk-
 * group passes of mcf_walk_diag (MCF_GROUP_FLAGS(G, g), g = 0..G-1):
 * pcol_groups holds the G partial vectors back to back (G x nnz, CSC order).
 * Per entry (i, c) the between-group spread of the per-walk mean estimates
 * Var(pcol[(i, c)]) (batch means, G' = min(G, N_c) - 1 degrees of freedom);
 * columns are independent, so var_i = sum_c Var(pcol[(i, c)]).  The standard
 * error SPEC.md:410 attaches to every result (there from a 1% walk subsample). */
MCF_API int mcf_diag_variance(mcf_graph *g, const double *pcol_groups, int groups, const int64_t *walk_pre,
                              double *var, int64_t row_begin, int64_t row_end, void *stream);

/* Multi-GPU diag combine with the exchange folded in (as mcf_spmv_peer):
 * d over rows [row_begin, row_end), reading pcol[(i, c)] from
 * pcol_parts[k] for the part k whose column range [col_bounds[k],
 * col_bounds[k+1]) holds c, and storing every d_i to all n_outs buffers. */
MCF_API int mcf_diag_combine_peer(mcf_graph *g, double zeta0, double zeta1, const double *const *pcol_parts,
                                  const int64_t *col_bounds, int n_parts, double *const *d_outs, int n_outs,
                                  int64_t row_begin, int64_t row_end, void *stream);

/* Work estimate per column for cost-balanced column shards (multi-GPU,
 * SURVEY 8(e)): cost[c] (int64, [dev] n) = N_c for mode 0 (action walks);
 * for mode 1 (diag) the emissions 3 N_c (max_steps + 1) plus the Eq. 20
 * combine's probes sum_{i in C_c} min(deg i, N_c (max_steps + 1))
 * (PAPER.md:303).  No counterpart in the reference (single process); the
 * paper balances by OpenMP dynamic scheduling. */
MCF_API int mcf_column_costs(mcf_graph *g, const int64_t *walk_pre, int64_t max_steps, int mode, int64_t *cost,
                             void *stream);

/* Device time of the kernels launched with MCF_FLAG_TIME_KERNELS since the
 * last reset: the walk kernels (action walks or diag emission walks) and, in
 * q_ms, the diag Q-build/combine kernel -- or, for mcf_funm_action, the span
 * before the walks (budgets and r) -- in ms, plus the number of timed walk
 * launches.
 * Synchronises on the recorded events.  reset != 0 destroys them; reset == 0
 * keeps them, so events captured into a CUDA graph can be re-read after every
 * replay. */
MCF_API int mcf_graph_kernel_times(mcf_graph *g, double *walk_ms, double *q_ms, int64_t *walk_launches,
                                   int reset);

/* ---- graph generation and ingest on the device ----------
 * Edges are 64-bit keys (u << 32) | v. */

/* R-MAT: `draws` edges, each `scale` levels of the reference's quadrant rule
 * (graphgen.py:138-143: row bit r >= a + b; column bit a <= r < a + b or
 * r >= a + b + c), Philox-4x32-10 uniforms keyed by seed. */
MCF_API int mcf_gen_rmat_keys(int scale, int64_t draws, double a, double b, double c, uint64_t seed, uint64_t *keys,
                              void *stream);

/* Chung-Lu: m edges, both endpoints drawn from the cumulative expected-degree
 * distribution cdf[n] (normalised, increasing). */
MCF_API int mcf_gen_chung_lu_keys(const double *cdf, int64_t n, int64_t m, uint64_t seed, uint64_t *keys,
                                  void *stream);

#define MCF_EDGES_DROP_LOOPS 1          /* remove (u, u) (sparsemat.py:258-260) */
#define MCF_EDGES_ADD_REVERSE 2         /* undirected: add (v, u) for every (u, v) (sparsemat.py:262-264) */
#define MCF_EDGES_FAIL_ON_DUPLICATES 4  /* duplicates -> MCF_ERR_ARGUMENT instead of being merged */

/* Edge keys -> CSR with n rows (the cleanup filters of simple_graph_from_edges,
 * sparsemat.py:243-290, in the reference's order: loops, undirected
 * expansion, duplicates): row_ptr[n+1] and col_ids (capacity col_cap >= the
 * resulting nnz, e.g. 2 m), columns sorted within every row.  *nnz receives
 * the edge count.  Synchronises `stream`. */
MCF_API int mcf_edges_to_csr(const uint64_t *keys, int64_t m, int64_t n, int flags, int64_t *row_ptr,
                             int32_t *col_ids, int64_t col_cap, int64_t *nnz, void *stream);

/* Isolated-node compaction (sparsemat.py:271-278): the nodes with an incident
 * edge are renumbered in order; new_row_ptr[n_out+1] (caller capacity n+1),
 * old_ids[n_out] (their original ids), col_ids remapped in place.
 * Synchronises `stream`. */
MCF_API int mcf_csr_compact(int64_t n, const int64_t *row_ptr, int32_t *col_ids, int64_t nnz, int64_t *new_row_ptr,
                            int64_t *old_ids, int64_t *n_out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* MCFUNM_CUDA_H */
