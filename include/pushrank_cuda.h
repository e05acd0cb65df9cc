/*
 * pushrank_cuda.h -- C-ABI of the B200-native IFP1/IFP2 push-round library
 * (libpushrank_cuda.so, sm_100a).
 *
 * The drop-in boundary.  The reference (pushrank 0.1.0) has one native
 * seam: the Cython kernel module resolved by _backend.resolve_backend
 * (/root/reference/pkg/src/pushrank/_backend.py:31-45) exposing
 * worker_loop/probe (_kernels.pyx:66-137).  That per-CPU-thread protocol
 * (K free-running loops + a polling monitor) has no GPU meaning, so this
 * library replaces the layer one level up: the engine entry points
 * (engines.py ifp1_run/ifp2_run/sync_simulate, solvers.py power_method)
 * and the graph core they consume (graph.py from_edges/classify/
 * dangling_target_counts/preprocess_ifp2).  Each entry point below cites
 * the reference interface it replaces.
 *
 * Conventions
 *  - plain pointers and sizes only; host arrays are caller-owned (the
 *    reference allocates every array in Python and kernels borrow them,
 *    engines.py:128-129); device state lives in opaque handles.
 *  - index arrays crossing the boundary are int64 (the reference's dtype,
 *    graph.py:141-142); the device keeps int32 column indices + int64
 *    offsets.
 *  - every call returns 0 on success or a negative PR_ERR_* code; the
 *    message is available from pr_last_error() (thread-local).  Argument
 *    validation with the reference's ValueError texts stays in the Python
 *    host layer; the library re-checks and fails with PR_ERR_ARG.
 *  - calls are synchronous on return and stream-ordered on the context's
 *    stream; one host thread per context.
 */
#ifndef PUSHRANK_CUDA_H
#define PUSHRANK_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PR_OK 0
#define PR_ERR_ARG (-1)         /* invalid argument (reference: ValueError) */
#define PR_ERR_CUDA (-2)        /* CUDA runtime / launch failure */
#define PR_ERR_STATE (-3)       /* missing prerequisite (e.g. preprocess before IFP2) */
#define PR_ERR_NOT_SETTLED (-4) /* max_rounds exhausted (engines.py:455-456 RuntimeError) */
#define PR_ERR_NOMEM (-5)       /* device allocation failed */
#define PR_ERR_FORMAT (-6)      /* edge-list text the device parser does not accept (graph.py:180-233) */

#define PR_ABI_VERSION 3

typedef struct pr_ctx pr_ctx;       /* one device + stream + workspace */
typedef struct pr_graph pr_graph;   /* device-resident CSR+CSC and derived data */

/* Per-round trace row; mirrors TraceSample (trace.py:12-38).  Field order
 * also matches oracle.ROW_DTYPE so rows compare column-for-column. */
typedef struct pr_round_stats {
    double h_l1;               /* sum of pending mass over all vertices */
    double alpha;              /* non-dangling share of above-threshold mass */
    double active_mass;        /* sum of pending mass above threshold */
    double carry_mass;         /* h_l1 - active_mass */
    int64_t converged;         /* #(h <= xi): scan set (engines) or all vertices (sync) */
    int64_t work;              /* sum(out_degree + 1) over active vertices */
    int64_t push_ops;          /* cumulative edge pushes before this state */
    int64_t push_ops_dangling; /* cumulative pushes into dangling vertices */
    uint64_t digest;           /* exact mode: position-weighted bit digest of (reserved, h) */
    double wall_ms;            /* device globaltimer since the run started */
} pr_round_stats;

typedef struct pr_class_counts {    /* VertexClassification (graph.py:68-89) */
    int64_t dangling, unreferenced, weak_dangling, weak_unreferenced;
    int64_t dangling_edge_count;    /* m_d */
    int64_t peel_rounds;
} pr_class_counts;

typedef struct pr_ifp2_counts {     /* IFP2Graph (graph.py:92-110) */
    int64_t live_edges, dangling, source_edges;
} pr_ifp2_counts;

enum pr_algorithm { PR_ALGO_IFP1 = 0, PR_ALGO_IFP2 = 1, PR_ALGO_FPFULL = 2 };
enum pr_mode {
    PR_MODE_AUTO = 0,   /* pull (CSC gather) in dense rounds, push (frontier scatter) in sparse ones */
    PR_MODE_PULL = 1,   /* every round as a deterministic CSC pull */
    PR_MODE_PUSH = 2,   /* every round (after the first) as a frontier scatter */
    PR_MODE_EXACT = 3   /* sync_simulate bit-exact: sequential ascending-source sums */
};
enum pr_converged_scope { PR_CONV_SCAN = 0, PR_CONV_ALL = 1 };

typedef struct pr_run_params {
    int32_t algorithm;        /* pr_algorithm */
    int32_t mode;             /* pr_mode */
    double damping;           /* c, SolverConfig.damping (solvers.py:39) */
    double threshold;         /* xi, SolverConfig.threshold (solvers.py:41) */
    int64_t max_rounds;       /* RuntimeError guard (engines.py:420,455) */
    double push_switch;       /* AUTO: push when active work < push_switch * pull work; <=0 -> default */
    int32_t converged_scope;  /* pr_converged_scope */
    int32_t host_loop;        /* 0: device-side loop (CUDA graph WHILE node); 1: host-driven rounds */
    /* Optional per-round observer (sync_simulate's on_iteration(t, reserved,
     * pushing), engines.py:453-454).  EXACT mode only.  The device loop runs
     * in batches: every state is snapshotted into a device ring (up to 64
     * states, 256 MiB) that the host drains into page-locked memory with one
     * copy per batch and then
     * calls on_round for each state in order (host_loop = 1: round by round).
     * The host arrays are valid for the duration of the call. */
    void (*on_round)(void *user, int64_t t, const double *reserved, const double *pending);
    void *user;
} pr_run_params;

typedef struct pr_run_result {
    int64_t rounds;           /* push rounds executed (sync_simulate "iterations") */
    int64_t rows;             /* trace rows produced (may exceed row_cap; extra rows dropped) */
    int64_t push_ops;         /* final cumulative push count (incl. IFP2 settle) */
    int64_t push_ops_dangling;
    int64_t settled;          /* IFP2 settle pushes (= m_d) */
    int64_t pull_rounds, push_rounds;
    double mass_total;        /* PageRankVector.mass_total */
    double push_ms;           /* device time: first round .. normalised output (CUDA events) */
    double round_ms;          /* device time of the round loop alone */
    double bytes_moved;       /* algorithmic bytes of the round loop (DESIGN.md roofline) */
    double pull_ms;           /* device time inside the dense-round kernels (globaltimer, first block
                                 start .. last block finalise), summed over pull rounds */
    double pull_bytes;        /* algorithmic bytes of those pull rounds */
    double sparse_ms;         /* same for the sparse rounds (push + scan kernels) */
    int64_t launches;         /* kernels launched by the solve (device-counted; unrolled graph
                                 slots that exit at once included) -- ABI 3 */
} pr_run_result;

/* ---- library / context ------------------------------------------------ */
int pr_abi_version(void);
const char *pr_last_error(void);
int pr_device_count(int *count);
int pr_ctx_create(int device, pr_ctx **out);
int pr_ctx_destroy(pr_ctx *ctx);
int pr_ctx_synchronize(pr_ctx *ctx);

/* ---- graph core ---------------------------------------------------------
 * graph.py:133-177 from_edges: dedup (src,dst) pairs, keep self-loops,
 * CSR sorted by (src,dst), CSC ascending source within a target. */
int pr_graph_from_edges(pr_ctx *ctx, int64_t n, const int64_t *src, const int64_t *dst,
                        int64_t m_raw, pr_graph **out);
/* Same from device-resident int64 edge arrays (e.g. pr_rmat_generate output). */
int pr_graph_from_device_edges(pr_ctx *ctx, int64_t n, const int64_t *d_src,
                               const int64_t *d_dst, int64_t m_raw, pr_graph **out);
/* Upload an already-built reference Graph (graph.py:21-42 arrays).
 * out_targets may be NULL: the fast engines (pr_run, modes auto/pull/push)
 * and pr_power only need the in-adjacency and out_offsets (they rebuild the
 * out-adjacency of their own layout on the device); classify, the
 * original-layout IFP2 arrays, exact mode and exporting out_targets then
 * fail with PR_ERR_STATE until pr_graph_attach_out_targets is called. */
int pr_graph_upload(pr_ctx *ctx, int64_t n, int64_t m, const int64_t *out_offsets,
                    const int64_t *out_targets, const int64_t *in_offsets,
                    const int64_t *in_sources, pr_graph **out);
int pr_graph_attach_out_targets(pr_graph *g, const int64_t *out_targets);
/* graph.py:201-259 load_edge_list, on the device: `text` is the raw bytes of
 * a whitespace-separated "src dst" edge list ('#' comments, blank lines).
 * Ids are remapped densely in order of first appearance (interleaved
 * src/dst), duplicates dropped, self-loops kept.  Returns PR_ERR_FORMAT for
 * text outside that grammar (a third column, a non-digit, a negative id, an
 * int64 overflow, no edges): the caller re-parses it on the host to report
 * the reference's line-numbered error, then calls pr_graph_from_raw_ids. */
int pr_graph_load_edge_list(pr_ctx *ctx, const char *text, int64_t len, pr_graph **out,
                            int64_t *raw_edges);
/* graph.py:243-257 on already-parsed raw ids (int64[m] each, non-negative). */
int pr_graph_from_raw_ids(pr_ctx *ctx, const int64_t *src, const int64_t *dst, int64_t m,
                          pr_graph **out);
/* Graph.original_ids -> int64[n] (identity for graphs not built from raw ids). */
int pr_graph_original_ids(pr_graph *g, int64_t *out);

/* ---- output formats (serialize.py) ----------------------------------------
 * serialize.py:16 ranking order: indices of `values` by score descending,
 * ties by original id ascending (np.lexsort((original_ids, -values))); the
 * first k of them.  original_ids NULL = identity. */
int pr_rank_order(pr_ctx *ctx, const double *values, const int64_t *original_ids, int64_t n, int64_t k,
                  int64_t *order);
/* serialize.py:14-21 write_ranking_csv: byte-identical to the reference's
 * csv.writer output (scores formatted as Python repr(float)). */
int pr_write_ranking_csv(pr_ctx *ctx, const double *values, const int64_t *original_ids, int64_t n,
                         const char *path);
/* repr(float) of one finite double into out[32]; returns the length. */
int pr_format_score(double value, char *out);
int pr_graph_destroy(pr_graph *g);
int pr_graph_info(const pr_graph *g, int64_t *n, int64_t *m);
/* Bytes pr_graph_upload / pr_graph_attach_out_targets copied host -> device
 * (the int64 index arrays travel partly narrowed to int32 on host threads). */
int pr_graph_h2d_bytes(const pr_graph *g, int64_t *bytes);
/* Graph arrays back to the host (int64, reference layout); NULL skips one. */
int pr_graph_export(pr_graph *g, int64_t *out_offsets, int64_t *out_targets,
                    int64_t *in_offsets, int64_t *in_sources);

/* graph.py:274-318 classify: base sets + joint weak peel; result stays on
 * the device, counts returned. */
int pr_classify(pr_graph *g, pr_class_counts *counts);
/* ascending id arrays sized by pr_classify's counts; NULL skips one */
int pr_classify_export(pr_graph *g, int64_t *dangling, int64_t *unreferenced,
                       int64_t *weak_dangling, int64_t *weak_unreferenced);
/* graph.py:334-340 dangling_target_counts -> int64[n] */
int pr_dangling_target_counts(pr_graph *g, int64_t *out);
/* graph.py:343-378 preprocess_ifp2: live CSR + dangling-source CSR on device */
int pr_preprocess_ifp2(pr_graph *g, pr_ifp2_counts *counts);
int pr_ifp2_export(pr_graph *g, int64_t *live_offsets, int64_t *live_targets,
                   int64_t *live_degree, int64_t *dangling_ids, int64_t *source_offsets,
                   int64_t *source_ids);

/* ---- engines ------------------------------------------------------------
 * engines.py:225-266 ifp1_run, engines.py:292-343 ifp2_run (+ settle
 * engines.py:269-289) and engines.py:349-485 sync_simulate.
 * Host outputs (values/reserved/pending, n doubles each; NULL skips one),
 * rows: up to row_cap trace rows. */
int pr_run(pr_graph *g, const pr_run_params *params, double *values, double *reserved,
           double *pending, pr_round_stats *rows, int64_t row_cap, pr_run_result *result);
/* Same with device output pointers (values may be NULL): no host copies. */
int pr_run_device(pr_graph *g, const pr_run_params *params, double *d_values,
                  double *d_reserved, double *d_pending, pr_round_stats *rows,
                  int64_t row_cap, pr_run_result *result);

/* solvers.py:186-243 power_method: pi (n doubles); per iteration k:
 * deltas[k] = L1 change (trace.h_l1) and converged[k] = #(|pi_k - pi_{k-1}| <=
 * threshold) (solvers.py:225-231); either may be NULL.  personalization may
 * be NULL (uniform 1/n).  result->rounds = iterations executed (early stop
 * when tolerance > 0 and delta < tolerance, solvers.py:234). */
int pr_power(pr_graph *g, double damping, int64_t iterations, double tolerance, double threshold,
             const double *personalization, double *pi, double *deltas, int64_t *converged,
             pr_run_result *result);
/* Same with on_iterate(k, pi) (solvers.py:232-233): called after every
 * iteration with the host copy of the iterate; a non-zero return stops. */
int pr_power_observed(pr_graph *g, double damping, int64_t iterations, double tolerance,
                      double threshold, const double *personalization, double *pi, double *deltas,
                      int64_t *converged, int (*on_iterate)(void *user, int64_t k, const double *pi),
                      void *user, pr_run_result *result);

/* ---- ERR harness (bench.py:90-112, 255-275) ------
 * max_relative_error: ERR = max_v |est_v - ref_v| / ref_v, its first argmax
 * (worst vertex), the L1 error, and the number of ref_v <= 0 (the reference
 * raises ValueError on any; the caller does).  d_est / d_ref are device
 * vectors of n doubles. */
int pr_error_report(pr_ctx *ctx, const double *d_est, const double *d_ref, int64_t n,
                    double *max_rel, double *l1, int64_t *worst, int64_t *nonpositive);
/* _power_iterations_to_target (bench.py:255-275): power iterations (limit at
 * most) with the ERR of every iterate against d_ref checked on the device;
 * *hit = the first k+1 whose iterate has ERR < target_err, or 0 if none. */
int pr_power_to_target(pr_graph *g, double damping, int64_t limit, const double *personalization,
                       const double *d_ref, double target_err, int64_t *hit);

/* ---- synthetic inputs ---------------------------------------------------
 * Device R-MAT sampler, bit-identical to synthetic.rmat_edges (counter
 * based splitmix64): samples first..first+count into device int64 arrays. */
int pr_rmat_generate(pr_ctx *ctx, int scale, int64_t edge_factor, double a, double b,
                     double c, uint64_t seed, int64_t first, int64_t count,
                     int64_t *d_src, int64_t *d_dst);
/* Build C2/C3/C5-shaped graphs entirely on the device: R-MAT samples, self
 * loops removed, optional seeded out-edge drop handled by the caller. */
int pr_graph_rmat(pr_ctx *ctx, int scale, int64_t edge_factor, double a, double b, double c,
                  uint64_t seed, pr_graph **out);

/* ---- vertex-range partitions (multi-GPU) ---------------
 * Local step of the bulk-synchronous partitioned rounds driven by
 * paper_2302_03245_b200/distributed.py: the rank owns `owned` vertices and
 * their in-edge rows, with source ids in a padded global space (rank r at
 * [r*slot, r*slot + owned_r)).  Shares are exchanged by the caller (NCCL
 * all-gather) between calls; d_* pointers are device memory.  Statistics:
 * ints = {active, work, push_ops, push_ops_dangling, converged_all,
 * converged_scan}, floats = {h_l1, active_mass, nd_active_mass} -- the
 * caller all-reduces them into the TraceSample row (engines.py:421-435). */
typedef struct pr_part pr_part;
int pr_part_create(pr_ctx *ctx, int64_t owned, int64_t slot, const int64_t *in_offsets,
                   const int64_t *in_sources, int64_t edges, const int64_t *out_degree,
                   const int64_t *row_len, const int64_t *dangling_target_counts,
                   const uint8_t *dangling, const uint8_t *receives, int32_t algorithm,
                   double damping, double threshold, pr_part **out);
int pr_part_init(pr_part *p, double *d_shares_mine, int64_t *ints, double *floats);
int pr_part_round(pr_part *p, const double *d_shares_full, double *d_shares_mine, int64_t *ints,
                  double *floats);
/* Device-resident forms for a queued round loop (no host synchronisation):
 * d_stats receives the 9 statistics as doubles {h_l1, active_mass,
 * nd_active_mass, active, work, push_ops, push_ops_dangling, converged_all,
 * converged_scan}, ready for an in-place device all-reduce.  fast = 1 runs
 * the single-GPU dense-round gather (degree-binned schedule of the
 * receiving rows, deterministic but not ascending-source order); fast = 0
 * the exact ascending-source sums of pr_part_round.  kind (fast form):
 * 0 Jacobi, 1 transition, 2 Gauss-Seidel -- the sweep kinds of rank-local
 * sections on large IFP2 partitions (round 0 after init is Jacobi, round 1
 * the transition, later rounds GS; without sections kind is ignored).
 * Work is queued on the
 * library stream (pr_part_stream), which the caller orders its collectives
 * on. */
/* The partition's rank among `parts` (its padded slot rank*slot): needed by
 * the fast form before the first round (rank-local Gauss-Seidel sections);
 * the fused-exchange setup sets it too. */
int pr_part_set_rank(pr_part *p, int32_t parts, int32_t rank);
/* Rank `rank`'s partition built on the device from a device graph, with no
 * host arrays: vertex ranges of the engines' run layout
 * (graph.cu; distributed.run_order) with edge-balanced bounds (in-degree + 8
 * per row, distributed.edge_balanced_ranges), padded source ids, global
 * out-degrees, push-row lengths (IFP2: live degree), dangling-target counts
 * and flags -- the content of distributed.partition_graph(g, parts, rank,
 * algorithm, order=run_order(...)).  bounds (parts+1 int64, run ids) may be
 * NULL.  The partition lives on the graph's device and stays valid after
 * the graph is destroyed.  The rank is set (pr_part_set_rank). */
int pr_part_from_graph(pr_graph *g, int32_t parts, int32_t rank, int32_t algorithm, double damping,
                       double threshold, int64_t *bounds, pr_part **out);
/* A partition's sizes (owned rows, padded slot, edges) and its rows as host
 * arrays in pr_part_create's layout (int64 offsets[owned+1], padded
 * sources[edges], degrees / row lengths / dangling-target counts[owned],
 * uint8 flags[owned]); any output pointer may be NULL. */
int pr_part_sizes(pr_part *p, int64_t *owned, int64_t *slot, int64_t *edges);
/* The next fast round (pr_part_round_device fast = 1 / pr_part_round_fused)
 * reads d_prev_stats9, the previous round's all-reduced statistics row, on
 * the device and skips its sweep when it shows no active vertex (the state
 * is final): rounds queued past termination cost a launch, not a sweep.
 * Applies to one round; NULL clears it. */
int pr_part_skip_if_done(pr_part *p, const double *d_prev_stats9);
/* Shares the fused exchange sends per dense round at most: the sum over
 * owned vertices of the ranks reading each (a partition built by
 * pr_part_from_graph with parts > 1 stores a vertex's share only into the
 * replicas of ranks that have one of its out-edges -- the sparse boundary
 * exchange, PUSHRANK_SPARSE_EXCHANGE=0 disables it); owned * parts otherwise. */
int pr_part_exchange_entries(pr_part *p, int64_t *entries);
int pr_part_export_rows(pr_part *p, int64_t *in_offsets, int64_t *in_sources, int64_t *out_degree,
                        int64_t *row_len, int64_t *dangling_target_counts, uint8_t *dangling, uint8_t *receives);
/* Kernel launches of one fast round (one per Gauss-Seidel section; the
 * last section's launch also reduces the statistics). */
int pr_part_launches_per_round(pr_part *p, int32_t *launches);
int pr_part_init_device(pr_part *p, double *d_shares_mine, double *d_stats);
int pr_part_round_device(pr_part *p, const double *d_shares_full, double *d_shares_mine, int32_t fast,
                         int32_t kind, double *d_stats);
int pr_part_stream(pr_part *p, void **stream);
/* Fused exchange (one process per GPU over NVLink/NVSwitch): the round
 * kernel stores every drained share straight into every rank's replica of
 * the full share vector, so no all-gather follows it; the caller's
 * statistics all-reduce is the round's barrier.
 *   pr_part_share_buffers: allocates this rank's two replicas (parity 0/1,
 *     slot*parts doubles, cudaMalloc) -> d_full[2] and their CUDA IPC
 *     handles (2 x 64 bytes at ipc_handles, may be NULL);
 *   pr_part_set_peers: opens the other ranks' handles (parts x 2 x 64 bytes,
 *     rank-major, as gathered from every rank);
 *   pr_part_set_peer_ptrs: the same from device pointers (2 per rank) -- the
 *     ranks emulated in one process on one device (tests);
 *   pr_part_init_fused / pr_part_round_fused(parity): state 0 into replicas
 *     0; a round reading replica `parity`, writing replicas 1-parity. */
int pr_part_share_buffers(pr_part *p, int32_t parts, int32_t rank, void **d_full, void *ipc_handles);
int pr_part_set_peers(pr_part *p, const void *ipc_handles);
int pr_part_set_peer_ptrs(pr_part *p, int32_t parts, int32_t rank, void *const *d_full);
int pr_part_init_fused(pr_part *p, double *d_stats);
/* Unmap the other ranks' replicas; call on every rank, then a barrier,
 * before destroying the partitions (an exporter must not free a replica
 * another rank still maps). */
int pr_part_close_peers(pr_part *p);
int pr_part_round_fused(pr_part *p, int32_t parity, int32_t kind, double *d_stats);
int pr_part_settle_shares(pr_part *p, double *d_x_mine);
int pr_part_settle(pr_part *p, const double *d_x_full, int64_t *settled, int64_t *ints, double *floats);
int pr_part_total(pr_part *p, int32_t include_pending, double *total);
int pr_part_export(pr_part *p, double *reserved, double *pending);
int pr_part_destroy(pr_part *p);

/* ---- device buffers (for torch-free hosts and tests) ---------------------- */
int pr_device_alloc(pr_ctx *ctx, int64_t bytes, void **d_ptr);
int pr_device_free(pr_ctx *ctx, void *d_ptr);
int pr_memcpy_h2d(pr_ctx *ctx, void *d_dst, const void *h_src, int64_t bytes);
int pr_memcpy_d2h(pr_ctx *ctx, void *h_dst, const void *d_src, int64_t bytes);
/* Page-locked host blocks from a process-wide cache (a freed block is reused
 * by the next request of the same size): output buffers that pr_run copies
 * into at full link speed instead of through pageable staging. */
int pr_host_alloc(int64_t bytes, void **h_ptr);
int pr_host_free(void *h_ptr);

#ifdef __cplusplus
}
#endif
#endif /* PUSHRANK_CUDA_H */
