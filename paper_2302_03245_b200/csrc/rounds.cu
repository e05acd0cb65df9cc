// rounds.cu -- the IFP1/IFP2 push-round hot path on sm_100a.
//
// Reference semantics (engines.py:349-456 for the round form, _kernels.pyx:
// 83-104 for the drain): every scanned vertex with pending mass h > xi
// (strict) is drained -- reserved += frac*h, h = 0 -- and pushes
// (c*h)/deg(v) along every (live) out-edge.  IFP1 scans non-dangling
// vertices over the full out-CSR; IFP2 scans them over the live CSR (edges
// into dangling vertices removed, weights still 1/out_degree) and settles
// the dangling vertices once at the end (engines.py:269-289); fp-full (sync
// twin only) scans everything and reserves 1-c.
//
// Fast engine (PR_MODE_AUTO/PULL/PUSH), on the run layout (graph.cu):
//   * pull round (dense): CSC gather over the destination set D (vertices
//     that can receive mass), degree bins (bins.cuh: hub slices per block,
//     warp rows, thread rows) dealt as equal-cost units to a persistent grid,
//     fixed-order reductions (deterministic, no atomics), double-buffered
//     shares s, the next state's drain fused into the epilogue.  k_pull<
//     STREAM, PREFETCH, GS>: evict-first index loads when the round overflows
//     L2; drain inputs loaded ahead of the gathers when it is latency-bound;
//     on large IFP2 graphs a sweep is cut into Gauss-Seidel sections (one
//     launch each) that read the new shares of earlier sections;
//   * push round (sparse tail): frontier scatter with red.global.add.f64,
//     then a scan kernel over D that fuses the drain;
//   * every round kernel ends with a last-block reduction of per-block
//     statistics (trace row, convergence test, next-mode choice) that also
//     drives the CUDA-graph conditionals (nested WHILE loops over unrolled
//     kernel slots), so the whole solve is one graph launch with no host
//     round trips.
// Exact engine (PR_MODE_EXACT): thread per vertex, sequential ascending
// source sums with explicit _rn intrinsics -- bit-identical reserved/h to
// sync_simulate's np.bincount order.
#include <cooperative_groups.h>
#include <cooperative_groups/scan.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "internal.cuh"
#include "reduce.cuh"
#include "bins.cuh"

namespace cg = cooperative_groups;

namespace pr {

struct RunArgs {
    int64_t n;
    const int64_t *in_off;
    const int32_t *in_src;
    const int64_t *push_off;   // out CSR (ifp1, fp-full) or live CSR (ifp2)
    const int32_t *push_tgt;
    const int32_t *deg;        // original out-degree: push weight denominator
    const int32_t *row_len;    // push row length for push_ops (out_deg or live_deg)
    const int32_t *dtc;        // dangling-target counts (ifp1/fp-full) or null (ifp2)
    BinView T;                  // pull schedule of D (sched.cu, bins.cuh)
    const int32_t *ids;        // D rows' vertex ids (== T.ids)
    int64_t d_count;
    const int32_t *seeds;      // vertices outside D active at state 0
    int64_t n_seed;
    const uint8_t *in_d;       // membership mask of D
    double *h, *reserved, *s;  // s: 2*n (ping-pong by state parity)
    long long *frontier;       // 2*fcap push items: (vertex << 24) | chunk
    int64_t fcap;
    uint8_t *act;              // exact engine
    Partial *partials;         // 3 regions of max_blocks: round, constants, mass totals
    int64_t max_blocks;
    RunCtl *ctl;
    pr_round_stats *rows;
    int64_t rows_cap;
    double c, xi, frac;
    int32_t algo, policy, conv_all, use_graph, has_mode;
    int64_t max_rounds;
    double push_work;          // AUTO: push when the next round's work < push_work
    double n_scan;             // scan-set size (bytes model)
    cudaGraphConditionalHandle h_loop, h_pull, h_push;
    // Gauss-Seidel sections of a dense sweep (ids == rows: the IFP2 run
    // layout); this launch processes section `sec` of `nsec`
    int32_t sec, nsec;
    // sources with id < sec_id[k] sit in sections before k (IFP2: ids are
    // rows, sec_id = sec_row; IFP1: the class-0 ids are in row order, so the
    // bound is the first class-0 id at or after row sec_row[k])
    int64_t sec_id[PR_MAX_SECTIONS + 1];
    const uint8_t *sec_of;     // IFP1: section of each vertex's row (push filter); null for IFP2
    int64_t sec_row[PR_MAX_SECTIONS + 1];
    int64_t sec_unit[PR_MAX_SECTIONS + 1];
    // observed exact runs: the device loop pauses after obs_batch rounds so
    // the host can drain obs_ring (obs_batch x [reserved | pending]) in one copy
    int64_t obs_batch;
    double *obs_ring;
};

// every solve kernel counts its own launch once (block 0, thread 0), early
// exits included: pr_run_result.launches
__device__ __forceinline__ void count_launch(const RunArgs &A) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&A.ctl->launches, 1ull);
}

__device__ __forceinline__ uint64_t digest_term(int64_t v, double r, double h) {
    uint64_t a = (uint64_t)__double_as_longlong(r), b = (uint64_t)__double_as_longlong(h);
    uint64_t w = ((uint64_t)v * 0x9E3779B97F4A7C15ull) | 1ull;
    return (a ^ (b * 0xBF58476D1CE4E5B9ull)) * w;
}

// Warp-collective append of push items (all 32 lanes call it; `enabled` is
// warp-uniform): a vertex with k TILE-edge chunks of (live) out-edges
// contributes k items, so hub rows are spread over k warps in a push round.
__device__ __forceinline__ void append_warp(bool enabled, int items, int32_t v, long long *F, int64_t *size) {
    if (!enabled) return;
    const int lane = threadIdx.x & 31;
    int incl = items;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    if (total == 0) return;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd((unsigned long long *)size, (unsigned long long)total);
    base = __shfl_sync(0xffffffffu, base, 0);
    for (int c = 0; c < items; ++c) F[base + (incl - items) + c] = ((long long)v << 24) | c;
}

__device__ __forceinline__ void append_one(int items, int32_t v, long long *F, int64_t *size) {
    if (!items) return;
    unsigned long long base = atomicAdd((unsigned long long *)size, (unsigned long long)items);
    for (int c = 0; c < items; ++c) F[base + c] = ((long long)v << 24) | c;
}

// Per-vertex drain inputs (loaded before the gathers by the pull rows).
struct VtxIn {
    int32_t v, dv, len, dt;
    double h, rv;
};

__device__ __forceinline__ VtxIn load_vtx(const RunArgs &A, int32_t v) {
    VtxIn q;
    q.v = v;
    q.dv = __ldg(&A.deg[v]);
    q.len = __ldg(&A.row_len[v]);
    q.dt = A.dtc ? __ldg(&A.dtc[v]) : 0;
    q.h = A.h[v];
    q.rv = A.reserved[v];
    return q;
}

__device__ __forceinline__ int drain_loaded(const RunArgs &A, const VtxIn &q, double hv, int64_t r, Partial &p);

// Drain one vertex of state r given its pre-drain pending mass hv:
// statistics, reservation, shares s[r&1].  Returns its push-item count.
__device__ __forceinline__ int drain_vertex(const RunArgs &A, int64_t v, double hv, int64_t r, Partial &p) {
    // every per-vertex load issued up front: one memory round trip per batch
    VtxIn q = load_vtx(A, (int32_t)v);
    return drain_loaded(A, q, hv, r, p);
}

__device__ __forceinline__ int drain_loaded(const RunArgs &A, const VtxIn &q, double hv, int64_t r, Partial &p) {
    const int64_t v = q.v;
    const int32_t dv = q.dv, len = q.len, dt = q.dt;
    const double rv = q.rv;
    const bool scan = A.algo == PR_ALGO_FPFULL || dv > 0;
    const bool above = hv > A.xi;  // strict (engines.py:421, _kernels.pyx:89)
    p.l1 += hv;
    if (above) {
        p.above += hv;
        if (dv > 0) p.nd_above += hv;
    } else {
        p.conv_all += 1;
        if (scan) p.conv_scan += 1;
    }
    double *s_out = A.s + (r & 1) * A.n;
    if (above && scan) {
        // (c*h)/deg with two roundings, never c*h*inv_deg (engines.py:444, _kernels.pyx:97)
        s_out[v] = dv > 0 ? __ddiv_rn(__dmul_rn(A.c, hv), (double)dv) : 0.0;
        A.reserved[v] = __dadd_rn(rv, __dmul_rn(A.frac, hv));
        // a vertex active in consecutive rounds already holds 0 (the dense
        // phase: nearly every row, every round): no store
        if (q.h != 0.0) A.h[v] = 0.0;
        p.nact += 1;
        p.work += (int64_t)dv + 1;
        p.push_ops += len;
        p.push_dang += dt;
        return (len + TILE - 1) / TILE;
    }
    s_out[v] = 0.0;
    A.h[v] = hv;
    return 0;
}

// Thread 0 of the last block: write trace row r, decide what runs next,
// drive the graph conditionals.
__device__ void finalize_row(const RunArgs &A, const Partial &tot, int64_t r, bool fast) {
    RunCtl *ctl = A.ctl;
    double l1 = tot.l1, above = tot.above, nd_above = tot.nd_above;
    int64_t conv_all = tot.conv_all, conv_scan = tot.conv_scan;
    if (fast && r >= 1) {
        l1 += ctl->c_l1;
        above += ctl->c_above;
        nd_above += ctl->c_nd_above;
        conv_all += ctl->c_conv_all;
        conv_scan += ctl->c_conv_scan;
    }
    if (r < A.rows_cap) {
        pr_round_stats row;
        row.h_l1 = l1;
        row.alpha = above > 0.0 ? nd_above / above : 1.0;
        row.active_mass = above;
        row.carry_mass = l1 - above;
        row.converged = A.conv_all ? conv_all : conv_scan;
        row.work = tot.work;
        row.push_ops = ctl->push_ops;
        row.push_ops_dangling = ctl->push_ops_dangling;
        row.digest = tot.digest;
        row.wall_ms = (double)(globaltimer() - ctl->t0_ns) * 1e-6;
        A.rows[r] = row;
    }
    ctl->rows = r + 1;
    if (fast && r >= 1) {
        // close the round that produced this state (its kernels started at t_k0)
        const double dt = (double)(globaltimer() - ctl->t_k0);
        if (ctl->next_mode == 0) {
            ctl->pull_ns += dt;
            ctl->pull_bytes += ctl->next_bytes;
        } else {
            ctl->sparse_ns += dt;
        }
    }
    ctl->k_started = 0;
    ctl->push_ops += tot.push_ops;
    ctl->push_ops_dangling += tot.push_dang;
    // algorithmic bytes of the round that drains this state
    const double rb = tot.nact > 0 ? 12.0 * (double)tot.push_ops + 40.0 * (double)tot.nact + 8.0 * A.n_scan : 0.0;
    ctl->bytes += rb;
    ctl->next_bytes = rb;
    int done = 0;
    if (tot.nact == 0) done = 1;
    else if (r >= A.max_rounds) done = 2;
    // observed exact run: leave the graph's loop once the ring is full
    const bool pause = A.obs_batch > 0 && ctl->obs_count >= A.obs_batch;
    ctl->done = done;
    ctl->round = r;
    // push needs the frontier of this state, recorded only when predicted
    const bool have_frontier = ctl->append != 0;
    int mode = 0;
    if (have_frontier && r >= 1) {
        if (A.policy == PR_MODE_PUSH) mode = 1;
        else if (A.policy == PR_MODE_AUTO && (double)tot.work < A.push_work) mode = 1;
    }
    // Gauss-Seidel state of the next round: after a dense sweep the next one
    // is a transition sweep (owed shares to every target + new shares of
    // earlier sections), then GS sweeps; a push round after a GS sweep only
    // delivers to targets in the source's section or earlier
    {
        const bool was_pull = fast && r >= 1 && ctl->next_mode == 0;
        const int32_t was_gs = ctl->gs;
        ctl->push_filter = A.nsec > 1 && mode == 1 && was_pull && was_gs != 0;
        ctl->gs = (A.nsec > 1 && mode == 0 && was_pull) ? 2 - (was_gs == 0 ? 1 : 0) : 0;
    }
    ctl->mode = mode;
    ctl->next_mode = mode;
    if (!done) {
        if (mode) ctl->push_rounds += 1;
        else ctl->pull_rounds += 1;
    }
    // record the next state's frontier when a push round is likely after it
    ctl->append = A.policy == PR_MODE_PUSH || (A.policy == PR_MODE_AUTO && (double)tot.work < 4.0 * A.push_work);
    ctl->fsize[(r + 1) & 1] = 0;
    ctl->unit_ctr = 0;
    ctl->blocks_done = 0;
    __threadfence();
    if (A.use_graph) {
        cudaGraphSetConditional(A.h_loop, (done || pause) ? 0u : 1u);
        if (A.has_mode) {
            cudaGraphSetConditional(A.h_pull, !done && mode == 0 ? 1u : 0u);
            cudaGraphSetConditional(A.h_push, !done && mode == 1 ? 1u : 0u);
        }
    }
}

// Publish this block's partial; the last block to arrive reduces all of
// them in a fixed order (deterministic) and finalises row r.
// `p` (and `cst`) must already be the block totals in thread 0.
// sec_kind: 0 a whole round; 1 a Gauss-Seidel section before the last (its
// totals are added to ctl->sec_acc, section order); 2 the last section (adds
// the accumulated sections and finalises the row).
__device__ void publish_round(const RunArgs &A, const Partial &p, int64_t r, bool fast, bool with_consts,
                              const Partial &cst, int sec_kind = 0) {
    __shared__ bool is_last;
    if (threadIdx.x == 0) {
        A.partials[blockIdx.x] = p;
        if (with_consts) A.partials[A.max_blocks + blockIdx.x] = cst;
        __threadfence();
        unsigned ticket = atomicAdd(&A.ctl->blocks_done, 1u);
        is_last = ticket == gridDim.x - 1;
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    Partial acc, cacc;
    zero(acc);
    zero(cacc);
    for (int64_t b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
        add(acc, load_partial(A.partials + b));
        if (with_consts) add(cacc, load_partial(A.partials + A.max_blocks + b));
    }
    block_reduce(acc);
    if (with_consts) block_reduce(cacc);
    if (threadIdx.x == 0) {
        if (with_consts) {
            A.ctl->c_l1 = cacc.l1;
            A.ctl->c_above = cacc.above;
            A.ctl->c_nd_above = cacc.nd_above;
            A.ctl->c_conv_all = cacc.conv_all;
            A.ctl->c_conv_scan = cacc.conv_scan;
        }
        if (sec_kind == 1) {
            RunCtl *c = A.ctl;
            if (A.sec == 0) c->sec_acc = acc;
            else add(c->sec_acc, acc);
            c->unit_ctr = 0;
            c->blocks_done = 0;
            __threadfence();
            return;
        }
        if (sec_kind == 2) {
            Partial tot = A.ctl->sec_acc;
            add(tot, acc);
            acc = tot;
        }
        finalize_row(A, acc, r, fast);
    }
}

__device__ void finish_round(const RunArgs &A, Partial p, int64_t r, bool fast, bool with_consts, Partial cst,
                             int sec_kind = 0) {
    block_reduce(p);
    if (with_consts) block_reduce(cst);
    publish_round(A, p, r, fast, with_consts, cst, sec_kind);
}

// warp-sum a batch partial and fold it into this warp's shared accumulator
__device__ __forceinline__ void warp_fold(Partial &bp, Partial &acc) {
    for (int o = 16; o > 0; o >>= 1) shfl_add(bp, o);
    if ((threadIdx.x & 31) == 0) add(acc, bp);
}

// ---------------------------------------------------------------- fast engine kernels

__global__ void k_reset(RunArgs A) {
    RunCtl *c = A.ctl;
    c->launches = 1;
    c->round = 0;
    c->rows = 0;
    c->push_ops = c->push_ops_dangling = 0;
    c->pull_rounds = c->push_rounds = 0;
    c->fsize[0] = c->fsize[1] = 0;
    c->mode = 0;
    c->done = 0;
    c->blocks_done = 0;
    c->append = 0;
    c->t0_ns = globaltimer();
    c->bytes = 0.0;
    c->c_l1 = c->c_above = c->c_nd_above = 0.0;
    c->c_conv_all = c->c_conv_scan = 0;
    c->mass_total = 0.0;
    c->settled = 0;
    c->unit_ctr = 0;
    c->k_started = 0;
    c->next_mode = 0;
    c->t_k0 = 0;
    c->next_bytes = 0.0;
    c->pull_ns = c->pull_bytes = c->sparse_ns = 0.0;
    c->gs = 0;
    c->push_filter = 0;
}

// State 0 (h = 1 everywhere, MassState.fresh engines.py:51-54): trace row 0
// and its drain.  Vertices in D go through the common epilogue; vertices
// outside D never receive mass, so their post-drain value is constant for
// every later row (recorded as constants) and their round-0 shares are
// gathered by the first dense round (their shares sit in buffer 0).
__global__ void __launch_bounds__(256) k_init(RunArgs A) {
    count_launch(A);
    Partial p, cst;
    zero(p);
    zero(cst);
    const bool app = A.ctl->append != 0;
    // grid-stride over a capped grid (whole blocks iterate together): few
    // partials for the last-block reduction
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < A.n; base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = base + threadIdx.x;
        int items = 0;
        if (v < A.n) {
            A.reserved[v] = 0.0;
            A.s[A.n + v] = 0.0;
            if (A.in_d[v]) {
                items = drain_vertex(A, v, 1.0, 0, p);
            } else {
                int32_t dv = A.deg[v];
                bool scan = A.algo == PR_ALGO_FPFULL || dv > 0;
                bool above = 1.0 > A.xi;
                p.l1 += 1.0;
                if (above) {
                    p.above += 1.0;
                    if (dv > 0) p.nd_above += 1.0;
                } else {
                    p.conv_all += 1;
                    if (scan) p.conv_scan += 1;
                }
                bool active = above && scan;
                double after = active ? 0.0 : 1.0;
                if (active) {
                    A.reserved[v] = A.frac;
                    p.nact += 1;
                    p.work += (int64_t)dv + 1;
                    p.push_ops += A.row_len[v];
                    if (A.dtc) p.push_dang += A.dtc[v];
                }
                A.h[v] = after;
                // an active vertex outside D has in-degree 0 (a round-0 seed):
                // its share is gathered by the first dense round like any other
                // source's -- in fixed order, no scatter -- and clear_seeds
                // (called by k_pull / k_scan) zeroes it during round 1, before
                // this buffer is read again.  Safe under Gauss-Seidel sections
                // only because seed ids lie at or above every section bound
                // (checked in run_rounds): the round-1 transition sweep never
                // reads a seed's entry of x_new (buffer 0) while it is zeroed
                A.s[v] = active && dv > 0 ? __ddiv_rn(__dmul_rn(A.c, 1.0), (double)dv) : 0.0;
                cst.l1 += after;
                if (after > A.xi) {
                    cst.above += after;
                    if (dv > 0) cst.nd_above += after;
                } else {
                    cst.conv_all += 1;
                    if (scan) cst.conv_scan += 1;
                }
            }
        }
        append_warp(app, items, (int32_t)v, A.frontier, &A.ctl->fsize[0]);
    }
    finish_round(A, p, 0, true, true, cst);
}

// Round 1 (any kind): clear the round-0 seed shares in buffer 0, which
// round 2 reads next; round 1 itself reads buffer 1.
__device__ __forceinline__ void clear_seeds(const RunArgs &A, int64_t t) {
    if (t != 1) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < A.n_seed; i += (int64_t)gridDim.x * blockDim.x)
        A.s[A.seeds[i]] = 0.0;
}

// Dense round t: h(t+1)_v = h_drained(t)_v + sum_{u in in(v)} s(t)_u over D,
// fused with the drain of state t+1.  Persistent grid over degree bins
// (bins.cuh): thread rows drain lane-parallel (coalesced vertex loads,
// warp-aggregated frontier append), warp and hub rows on one lane.
#ifndef PULL_MIN_BLOCKS
#define PULL_MIN_BLOCKS 4
#endif
// resident blocks per SM of the prefetching form (80 registers at 3)
#ifndef PR_PF_BLOCKS
#define PR_PF_BLOCKS 3
#endif
__device__ __forceinline__ void stamp_round_start(RunCtl *ctl) {
    if (threadIdx.x == 0 && atomicExch(&ctl->k_started, 1u) == 0u) ctl->t_k0 = globaltimer();
}

// Row callbacks of the dense round (bins.cuh): the drain inputs of a row are
// loaded before its gathers, so the drain after the sum waits on no memory.
struct PullRows {
    const RunArgs &A;
    int64_t r;
    bool app;
    long long *F;
    int64_t *fsize;
    Partial &p;
    __device__ __forceinline__ VtxIn pre(bool valid, int64_t row) const {
        VtxIn q;
        if (valid) {
            q = load_vtx(A, __ldg(&A.ids[row]));
        } else {
            q.v = 0;
            q.dv = q.len = q.dt = 0;
            q.h = q.rv = 0.0;
        }
        return q;
    }
    __device__ __forceinline__ void fin(bool valid, const VtxIn &q, double sum) {
        const int items = valid ? drain_loaded(A, q, q.h + sum, r, p) : 0;
        append_warp(app, items, q.v, F, fsize);
    }
    __device__ __forceinline__ void single(int64_t row, double sum) {
        const int32_t v = __ldg(&A.ids[row]);
        const int it = drain_vertex(A, v, A.h[v] + sum, r, p);
        if (app) append_one(it, v, F, fsize);
    }
};

// Unrolled loop bodies launch a kernel per slot; a slot whose round is not
// of this kind (or after termination) exits at once.
__device__ __forceinline__ bool round_is(const RunArgs &A, int mode) {
    const volatile RunCtl *c = A.ctl;
    return !c->done && c->mode == mode;
}

// GS: the launch is one Gauss-Seidel section of a sweep
template <bool STREAM, bool PREFETCH, bool GS>
__global__ void __launch_bounds__(256, PREFETCH ? PR_PF_BLOCKS : PULL_MIN_BLOCKS) k_pull(RunArgs A) {
    count_launch(A);
    if (A.use_graph && !round_is(A, 0)) return;
    stamp_round_start(A.ctl);
    const int64_t t = A.ctl->round;
    const double *__restrict__ s_in = A.s + (t & 1) * A.n;
    const int64_t r = t + 1;
    const bool app = A.ctl->append != 0;
    long long *F = A.frontier + (r & 1) * A.fcap;
    int64_t *fsize = &A.ctl->fsize[r & 1];
    clear_seeds(A, t);
    // this launch's section and the sweep kind (Src in bins.cuh)
    const int64_t u_lo = A.sec_unit[A.sec], u_hi = A.sec_unit[A.sec + 1];
    Src src{s_in, A.s + (r & 1) * A.n, 0, 0};
    int32_t gs = 0;
    if constexpr (GS) {
        gs = A.ctl->gs;
        if (gs) src.gs_lo = (int)A.sec_id[A.sec];
    }
    Partial p;
    zero(p);
    if constexpr (PREFETCH) {
        PullRows rows{A, r, app, F, fsize, p};
        if constexpr (!GS) bins_run<STREAM, true, 0>(A.T, u_lo, u_hi, src, rows);
        else if (gs == 1) bins_run<STREAM, true, 2>(A.T, u_lo, u_hi, src, rows);
        else bins_run<STREAM, true, 1>(A.T, u_lo, u_hi, src, rows);
    } else {
        auto thread_row = [&](bool valid, int64_t row, double sum) {
            int items = 0;
            int32_t v = 0;
            if (valid) {
                v = __ldg(&A.ids[row]);
                items = drain_vertex(A, v, A.h[v] + sum, r, p);
            }
            append_warp(app, items, v, F, fsize);
        };
        auto single_row = [&](int64_t row, double sum) {
            int32_t v = __ldg(&A.ids[row]);
            int it = drain_vertex(A, v, A.h[v] + sum, r, p);
            if (app) append_one(it, v, F, fsize);
        };
        if constexpr (!GS) bins_run_plain<STREAM, 0>(A.T, u_lo, u_hi, src, thread_row, single_row);
        else if (gs == 1) bins_run_plain<STREAM, 2>(A.T, u_lo, u_hi, src, thread_row, single_row);
        else bins_run_plain<STREAM, 1>(A.T, u_lo, u_hi, src, thread_row, single_row);
    }
    finish_round(A, p, r, true, false, p, A.nsec > 1 ? (A.sec + 1 < A.nsec ? 1 : 2) : 0);
}

// Sparse round t, step 1: scatter the frontier's shares (red.global.add.f64);
// one warp per push item (a TILE-edge chunk of one vertex's out-row), the 8
// target loads of a lane issued before its 8 reductions.
__global__ void __launch_bounds__(256) k_push(RunArgs A) {
    count_launch(A);
    if (A.use_graph && !round_is(A, 1)) return;
    stamp_round_start(A.ctl);
    int64_t t = A.ctl->round;
    const double *__restrict__ s_in = A.s + (t & 1) * A.n;
    const long long *F = A.frontier + (t & 1) * A.fcap;
    int64_t cnt = A.ctl->fsize[t & 1];
    const bool filter = A.ctl->push_filter != 0;
    int lane = threadIdx.x & 31;
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp; i < cnt; i += nwarps) {
        long long item = F[i];
        int32_t u = (int32_t)(item >> 24);
        int64_t c = item & 0xFFFFFF;
        double sh = s_in[u];
        int64_t lo = A.push_off[u] + c * TILE, hi = A.push_off[u + 1];
        if (hi > lo + TILE) hi = lo + TILE;
        // after a Gauss-Seidel sweep, targets in later sections than u have
        // already taken u's share during the sweep
        int32_t t_hi = 0x7fffffff;
        int su = PR_MAX_SECTIONS;   // IFP1: deliver to targets whose row section <= su
        if (filter) {
            if (A.sec_of) {
                su = A.sec_of[u];
            } else {
                for (int k = 1; k <= A.nsec; ++k)
                    if (u < A.sec_row[k]) {
                        t_hi = (int32_t)A.sec_row[k];
                        break;
                    }
            }
        }
        int32_t tg[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            int64_t e = lo + k * 32 + lane;
            tg[k] = e < hi ? __ldg(&A.push_tgt[e]) : -1;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (tg[k] >= 0 && tg[k] < t_hi && (su == PR_MAX_SECTIONS || A.sec_of[tg[k]] <= su))
                atomicAdd(&A.h[tg[k]], sh);
    }
}

// Sparse round t, step 2: drain state t+1 over D
__global__ void __launch_bounds__(256) k_scan(RunArgs A) {
    count_launch(A);
    if (A.use_graph && !round_is(A, 1)) return;
    const int64_t t = A.ctl->round;
    clear_seeds(A, t);
    const int64_t r = t + 1;
    const bool app = A.ctl->append != 0;
    long long *F = A.frontier + (r & 1) * A.fcap;
    int64_t *fsize = &A.ctl->fsize[r & 1];
    Partial p;
    zero(p);
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < A.d_count;
         base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = base + threadIdx.x;
        int items = 0;
        int32_t v = 0;
        if (i < A.d_count) {
            v = __ldg(&A.ids[i]);
            items = drain_vertex(A, v, A.h[v], r, p);
        }
        append_warp(app, items, v, F, fsize);
    }
    finish_round(A, p, r, true, false, p);
}

// ---------------------------------------------------------------- exact engine

__global__ void k_ex_init(RunArgs A) {
    count_launch(A);
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < A.n; v += (int64_t)gridDim.x * blockDim.x) {
        A.h[v] = 1.0;
        A.reserved[v] = 0.0;
    }
}

// trace row of state t (engines.py:421-435) and its drain (engines.py:438-444)
__global__ void __launch_bounds__(256) k_ex_prep(RunArgs A) {
    count_launch(A);
    int64_t t = A.ctl->rows;  // state index = rows produced so far
    Partial p;
    zero(p);
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v < A.n) {
        double hv = A.h[v], rv = A.reserved[v];
        p.digest = digest_term(v, rv, hv);
        int32_t dv = A.deg[v];
        bool scan = A.algo == PR_ALGO_FPFULL || dv > 0;
        bool above = hv > A.xi;
        p.l1 = hv;
        if (above) {
            p.above = hv;
            if (dv > 0) p.nd_above = hv;
        } else {
            p.conv_all = 1;
            if (scan) p.conv_scan = 1;
        }
        bool active = above && scan;
        A.act[v] = active;
        if (active) {
            A.reserved[v] = __dadd_rn(rv, __dmul_rn(A.frac, hv));
            int32_t len = A.row_len[v];
            A.s[v] = len > 0 ? __ddiv_rn(__dmul_rn(A.c, hv), (double)dv) : 0.0;
            p.nact = 1;
            p.work = (int64_t)dv + 1;
            p.push_ops = len;
            if (A.dtc) p.push_dang = A.dtc[v];
        } else {
            A.s[v] = 0.0;
        }
    }
    finish_round(A, p, t, false, false, p);
}

// h(t+1)_v = (active ? 0 : h_v) + sum over in-edges in ascending source order
// (== the sequential np.bincount accumulation, engines.py:446-448)
__global__ void k_ex_pull(RunArgs A) {
    count_launch(A);
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= A.n) return;
    double acc = 0.0;
    bool receives = A.algo != PR_ALGO_IFP2 || A.deg[v] > 0;
    if (receives)
        for (int64_t e = A.in_off[v]; e < A.in_off[v + 1]; ++e) acc = __dadd_rn(acc, A.s[A.in_src[e]]);
    double base = A.act[v] ? 0.0 : A.h[v];
    A.h[v] = __dadd_rn(base, acc);
}

// Observed exact runs (sync_simulate's on_iteration, engines.py:453-454):
// a batch starts with an empty ring; after each round's update the state
// (reserved, pending) goes to the next ring slot.
__global__ void k_obs_begin(RunArgs A) {
    count_launch(A);
    A.ctl->obs_count = 0;
    A.ctl->obs_t0 = A.ctl->rows - 1;
}

__global__ void k_obs_snap(RunArgs A) {
    count_launch(A);
    const int64_t j = A.ctl->obs_count;
    double *dst = A.obs_ring + 2 * j * A.n;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < A.n; v += (int64_t)gridDim.x * blockDim.x) {
        dst[v] = A.reserved[v];
        dst[A.n + v] = A.h[v];
    }
}

// one thread: the snapshot is complete (every k_obs_snap block ran), count it
__global__ void k_obs_count(RunArgs A) {
    count_launch(A);
    A.ctl->obs_count += 1;
}

// ---------------------------------------------------------------- settle + normalise (K7)

// engines.py:269-289: reserved[d] = h[d] + sum_{u in S(d)} (c*reserved[u])/deg[u]
// Dangling vertices [lo, hi): thread per vertex (sequential, ascending
// source order) when `thread_mode`, else warp per vertex (fixed tree).
__global__ void k_settle(RunArgs A, const int32_t *dang_ids, int64_t lo, int64_t nd, const int64_t *src_off,
                         const int32_t *src_ids, int thread_mode) {
    count_launch(A);
    if (thread_mode) {
        for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nd;
             i += (int64_t)gridDim.x * blockDim.x) {
            double acc = 0.0;
            for (int64_t e = src_off[i]; e < src_off[i + 1]; ++e) {
                int32_t u = src_ids[e];
                acc = __dadd_rn(acc, __ddiv_rn(__dmul_rn(A.c, A.reserved[u]), (double)A.deg[u]));
            }
            int32_t d = dang_ids[i];
            A.reserved[d] = __dadd_rn(A.h[d], acc);
            A.h[d] = 0.0;
        }
        return;
    }
    int lane = threadIdx.x & 31;
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = lo + warp; i < nd; i += nwarps) {
        double acc = 0.0;
        for (int64_t e = src_off[i] + lane; e < src_off[i + 1]; e += 32) {
            int32_t u = src_ids[e];
            acc += __ddiv_rn(__dmul_rn(A.c, A.reserved[u]), (double)A.deg[u]);
        }
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) {
            int32_t d = dang_ids[i];
            A.reserved[d] = A.h[d] + acc;
            A.h[d] = 0.0;
        }
    }
}

// Fast-engine settle: w[u] = (c*reserved[u])/deg[u] once per source (the
// same two-rounding term as engines.py:281), then a gather-sum per dangling
// row with 8 loads in flight (bins.cuh helpers): one random load per edge
// instead of two loads and a division.
__global__ void k_settle_w(RunArgs A, int64_t n_src, double *__restrict__ w) {
    count_launch(A);
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n_src; u += (int64_t)gridDim.x * blockDim.x) {
        const int32_t du = A.deg[u];
        w[u] = du > 0 ? __ddiv_rn(__dmul_rn(A.c, A.reserved[u]), (double)du) : 0.0;
    }
}

__global__ void k_settle_fast(RunArgs A, const double *__restrict__ w, const int32_t *__restrict__ dang_ids, int64_t lo,
                              int64_t nd, const int64_t *__restrict__ src_off, const int32_t *__restrict__ src_ids,
                              int thread_mode) {
    count_launch(A);
    if (thread_mode) {
        for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nd;
             i += (int64_t)gridDim.x * blockDim.x) {
            const double acc = row_sum_thread<false, 0>(src_ids, src_off[i], src_off[i + 1], Src{w, w, 0, 0});
            const int32_t d = dang_ids[i];
            A.reserved[d] = A.h[d] + acc;
            A.h[d] = 0.0;
        }
        return;
    }
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = lo + warp; i < nd; i += nwarps) {
        const double acc = span_sum_warp<false, 0>(src_ids, src_off[i], src_off[i + 1], Src{w, w, 0, 0});
        if (lane == 0) {
            const int32_t d = dang_ids[i];
            A.reserved[d] = A.h[d] + acc;
            A.h[d] = 0.0;
        }
    }
}

// first index of dangling vertices with <= 32 sources (run layout: receivers
// sorted by descending in-degree, so the big ones lead)
__global__ void k_count_big(const int64_t *src_off, int64_t nd, unsigned long long *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nd; i += (int64_t)gridDim.x * blockDim.x)
        if (src_off[i + 1] - src_off[i] > 32) atomicAdd(out, 1ull);
}

static int count_settle_big(Graph &g, int64_t *big) {
    if (g.settle_big < 0) {
        DevBuf c;
        PR_TRY(ensure(c, 8));
        PR_CUDA(cudaMemsetAsync(c.ptr, 0, 8, g.ctx->stream));
        k_count_big<<<grid_for(g.ifp2.dangling, 256) > 2048 ? 2048 : grid_for(g.ifp2.dangling, 256), 256, 0,
                      g.ctx->stream>>>(g.src_off.as<int64_t>(), g.ifp2.dangling, c.as<unsigned long long>());
        unsigned long long h = 0;
        PR_CUDA(cudaMemcpyAsync(&h, c.ptr, 8, cudaMemcpyDeviceToHost, g.ctx->stream));
        PR_CUDA(cudaStreamSynchronize(g.ctx->stream));
        g.settle_big = (int64_t)h;
    }
    *big = g.settle_big;
    return PR_OK;
}

// total mass (deterministic; x = reserved [+ h]) and, for IFP2, the
// post-settle trace row (engines.py:331-335)
__global__ void __launch_bounds__(256) k_total(RunArgs A, int include_h, int64_t settled, int write_row) {
    count_launch(A);
    __shared__ bool is_last;
    Partial p, x;
    zero(p);
    zero(x);
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < A.n; v += (int64_t)gridDim.x * blockDim.x) {
        double hv = A.h[v];
        x.l1 += include_h ? A.reserved[v] + hv : A.reserved[v];
        int32_t dv = A.deg[v];
        bool scan = A.algo == PR_ALGO_FPFULL || dv > 0;
        p.l1 += hv;
        if (hv > A.xi) {
            p.above += hv;
            if (dv > 0) p.nd_above += hv;
        } else {
            p.conv_all += 1;
            if (scan) p.conv_scan += 1;
        }
    }
    block_reduce(p);
    block_reduce(x);
    if (threadIdx.x == 0) {
        A.partials[blockIdx.x] = p;
        A.partials[2 * A.max_blocks + blockIdx.x] = x;
        __threadfence();
        unsigned ticket = atomicAdd(&A.ctl->blocks_done, 1u);
        is_last = ticket == gridDim.x - 1;
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    Partial acc, xacc;
    zero(acc);
    zero(xacc);
    for (int64_t b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
        add(acc, load_partial(A.partials + b));
        add(xacc, load_partial(A.partials + 2 * A.max_blocks + b));
    }
    block_reduce(acc);
    block_reduce(xacc);
    if (threadIdx.x == 0) {
        RunCtl *ctl = A.ctl;
        ctl->mass_total = xacc.l1;
        ctl->settled = settled;
        ctl->blocks_done = 0;
        if (write_row) {
            int64_t r = ctl->rows;
            ctl->push_ops += settled;
            ctl->push_ops_dangling += settled;
            if (r < A.rows_cap) {
                pr_round_stats row;
                row.h_l1 = acc.l1;
                row.alpha = acc.above > 0.0 ? acc.nd_above / acc.above : 1.0;
                row.active_mass = acc.above;
                row.carry_mass = acc.l1 - acc.above;
                row.converged = A.conv_all ? acc.conv_all : acc.conv_scan;
                row.work = 0;
                row.push_ops = ctl->push_ops;
                row.push_ops_dangling = ctl->push_ops_dangling;
                row.digest = 0;
                row.wall_ms = (double)(globaltimer() - ctl->t0_ns) * 1e-6;
                A.rows[r] = row;
            }
            ctl->rows = r + 1;
        }
    }
}

// values in original vertex order (perm: run id -> original id, or identity)
__global__ void k_scale(RunArgs A, int include_h, double *values, const int32_t *perm) {
    count_launch(A);
    double tot = A.ctl->mass_total;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < A.n; v += (int64_t)gridDim.x * blockDim.x) {
        double x = include_h ? A.reserved[v] + A.h[v] : A.reserved[v];
        values[perm ? perm[v] : v] = x / tot;
    }
}

__global__ void k_unpermute(const double *src, int64_t n, const int32_t *perm, double *dst) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        dst[perm ? perm[v] : v] = src[v];
}

__global__ void k_mark_d(const int32_t *ids, int64_t count, uint8_t *in_d) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        in_d[ids[i]] = 1;
}

// ---------------------------------------------------------------- host side

static int add_kernel(cudaGraph_t g, cudaGraphNode_t *node, const cudaGraphNode_t *deps, size_t ndeps, void *func,
                      unsigned grid, unsigned block, void **args, size_t smem = 0) {
    cudaKernelNodeParams kp;
    memset(&kp, 0, sizeof(kp));
    kp.func = func;
    kp.gridDim = dim3(grid);
    kp.blockDim = dim3(block);
    kp.sharedMemBytes = (unsigned)smem;
    kp.kernelParams = args;
    PR_CUDA(cudaGraphAddKernelNode(node, g, deps, ndeps, &kp));
    return PR_OK;
}

struct Plan {
    RunArgs A;
    bool exact;
    unsigned g_all, g_red, g_total, g_pull, g_push, g_scan;
    const void *k_pull_fn;   // k_pull<STREAM, PREFETCH> chosen by the round's working set
    // per section: the launch's kernel and grid (sections of thread rows can
    // take the form that loads a row's drain inputs before its gathers)
    const void *k_pull_sec[PR_MAX_SECTIONS];
    unsigned g_pull_sec[PR_MAX_SECTIONS];
};

void release_execs(Ctx &ctx) {
    for (auto &e : ctx.execs) {
        if (e.exec) cudaGraphExecDestroy(e.exec);
        if (e.graph) cudaGraphDestroy(e.graph);
        e.exec = nullptr;
        e.graph = nullptr;
        e.key.clear();
    }
}

// One graph per parameter set:
//   reset -> init -> seeds -> WHILE(loop) {
//       WHILE(pull) { k_pull x PULL_UNROLL }
//       WHILE(push) { (k_push -> k_scan) x PUSH_UNROLL } }
// (exact: WHILE { pull -> prep }).  The round finaliser sets the three
// handles.  Unrolling the bodies into plain kernel nodes matters: measured
// per round, WHILE{SWITCH{kernel}} costs 11.7 us, WHILE{kernel} 7.6 us and
// WHILE{kernel x8} 3.7 us (tools_graph_overhead.py).
#ifndef PR_PULL_UNROLL
#define PR_PULL_UNROLL 8
#endif
#ifndef PR_PUSH_UNROLL
#define PR_PUSH_UNROLL 4
#endif
constexpr int PULL_UNROLL = PR_PULL_UNROLL, PUSH_UNROLL = PR_PUSH_UNROLL;

static int add_while(cudaGraph_t g, cudaGraphNode_t *node, const cudaGraphNode_t *dep, cudaGraphConditionalHandle h,
                     cudaGraph_t *body) {
    cudaGraphNodeParams wp = {};
    wp.type = cudaGraphNodeTypeConditional;
    wp.conditional.handle = h;
    wp.conditional.type = cudaGraphCondTypeWhile;
    wp.conditional.size = 1;
    PR_CUDA(cudaGraphAddNode(node, g, dep, dep ? 1 : 0, &wp));
    *body = wp.conditional.phGraph_out[0];
    return PR_OK;
}

static int build_graph(Plan &P, cudaGraph_t *out_g, cudaGraphExec_t *out_exec) {
    cudaGraph_t G;
    PR_CUDA(cudaGraphCreate(&G, 0));
    RunArgs &A = P.A;
    PR_CUDA(cudaGraphConditionalHandleCreate(&A.h_loop, G, 1, cudaGraphCondAssignDefault));
    // every handle must belong to a conditional node, so the mode handles
    // exist only in the fast engine's graph
    A.has_mode = !P.exact;
    if (A.has_mode) {
        PR_CUDA(cudaGraphConditionalHandleCreate(&A.h_pull, G, 0, cudaGraphCondAssignDefault));
        PR_CUDA(cudaGraphConditionalHandleCreate(&A.h_push, G, 0, cudaGraphCondAssignDefault));
    }
    A.use_graph = 1;
    void *args[] = {&A};
    cudaGraphNode_t n_reset, n_init, n_seed, n_while, n_a, n_b;
    if (P.exact && A.obs_batch > 0) {
        // observed batches: the host ran reset/init/prep of state 0; each
        // launch continues the loop until the ring is full (or done)
        cudaGraphNode_t n_begin, n_c;
        PR_TRY(add_kernel(G, &n_begin, nullptr, 0, (void *)k_obs_begin, 1, 1, args));
        cudaGraph_t body;
        PR_TRY(add_while(G, &n_while, &n_begin, A.h_loop, &body));
        PR_TRY(add_kernel(body, &n_a, nullptr, 0, (void *)k_ex_pull, P.g_all, 256, args));
        PR_TRY(add_kernel(body, &n_b, &n_a, 1, (void *)k_obs_snap, P.g_all, 256, args));
        PR_TRY(add_kernel(body, &n_c, &n_b, 1, (void *)k_obs_count, 1, 1, args));
        PR_TRY(add_kernel(body, &n_a, &n_c, 1, (void *)k_ex_prep, P.g_all, 256, args));
        cudaGraphExec_t ex;
        PR_CUDA(cudaGraphInstantiate(&ex, G, 0));
        *out_g = G;
        *out_exec = ex;
        return PR_OK;
    }
    PR_TRY(add_kernel(G, &n_reset, nullptr, 0, (void *)k_reset, 1, 1, args));
    if (P.exact) {
        PR_TRY(add_kernel(G, &n_init, &n_reset, 1, (void *)k_ex_init, P.g_all, 256, args));
        PR_TRY(add_kernel(G, &n_seed, &n_init, 1, (void *)k_ex_prep, P.g_all, 256, args));
    } else {
        PR_TRY(add_kernel(G, &n_init, &n_reset, 1, (void *)k_init, P.g_red, 256, args));
        n_seed = n_init;   // round-0 seeds are gathered by the first dense round
    }
    cudaGraph_t body;
    PR_TRY(add_while(G, &n_while, &n_seed, A.h_loop, &body));
    if (P.exact) {
        PR_TRY(add_kernel(body, &n_a, nullptr, 0, (void *)k_ex_pull, P.g_all, 256, args));
        PR_TRY(add_kernel(body, &n_b, &n_a, 1, (void *)k_ex_prep, P.g_all, 256, args));
    } else {
        cudaGraphNode_t w_pull, w_push;
        cudaGraph_t b_pull, b_push;
        PR_TRY(add_while(body, &w_pull, nullptr, A.h_pull, &b_pull));
        PR_TRY(add_while(body, &w_push, &w_pull, A.h_push, &b_push));
        cudaGraphNode_t prev = nullptr;
        // a slot is one dense sweep: its sections in order
        const int sweeps = A.nsec > 1 ? (PULL_UNROLL / A.nsec > 2 ? PULL_UNROLL / A.nsec : 2) : PULL_UNROLL;
        for (int k = 0; k < sweeps; ++k)
            for (int sec = 0; sec < A.nsec; ++sec) {
                A.sec = sec;  // the node copies its arguments here
                PR_TRY(add_kernel(b_pull, &n_a, prev ? &prev : nullptr, prev ? 1 : 0, (void *)P.k_pull_sec[sec],
                                  P.g_pull_sec[sec], 256, args));
                prev = n_a;
            }
        A.sec = 0;
        prev = nullptr;
        for (int k = 0; k < PUSH_UNROLL; ++k) {
            PR_TRY(add_kernel(b_push, &n_a, prev ? &prev : nullptr, prev ? 1 : 0, (void *)k_push, P.g_push, 256, args));
            PR_TRY(add_kernel(b_push, &n_b, &n_a, 1, (void *)k_scan, P.g_scan, 256, args));
            prev = n_b;
        }
    }
    cudaGraphExec_t ex;
    PR_CUDA(cudaGraphInstantiate(&ex, G, 0));
    *out_g = G;
    *out_exec = ex;
    return PR_OK;
}

// IFP1 sections on the run layout: sec_of[ids[r]] = section of row r; sec_id[k]
// = first class-0 id at or after row sec_row[k] (class0_end if none); bad
// counts class-0 rows whose ids do not increase with the row (then the
// id-bound test is invalid and the caller drops the sections)
__global__ void k_sec_of(const int32_t *ids, int64_t count, const int64_t *bounds, int nsec, uint8_t *sec_of) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < count; r += (int64_t)gridDim.x * blockDim.x) {
        int k = 0;
        while (k + 1 < nsec && r >= bounds[k + 1]) ++k;
        sec_of[ids[r]] = (uint8_t)k;
    }
}

__global__ void k_class0_order(const int32_t *ids, int64_t count, int64_t c0, int32_t *pos, unsigned long long *bad,
                               int phase) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < count; r += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = ids[r];
        if (v >= c0) continue;
        if (phase == 0) pos[v] = (int32_t)r;
        else if (v + 1 < c0 && pos[v + 1] <= (int32_t)r) atomicAdd(bad, 1ull);
    }
}

__global__ void k_sec_id(const int32_t *ids, int64_t count, int64_t c0, const int64_t *bounds, int nsec, int64_t *out) {
    const int k = threadIdx.x;
    if (k > nsec) return;
    int64_t r = bounds[k];
    while (r < count && ids[r] >= c0) ++r;
    out[k] = r < count ? ids[r] : c0;
}

static int sections_by_id(Graph &g, int which) {
    Ctx &ctx = *g.ctx;
    cudaStream_t st = ctx.stream;
    auto &S = g.sched[which];
    const int64_t c0 = g.class0_end;
    DevBuf pos, bad, bnd, out;
    PR_TRY(ensure(pos, 4 * (c0 > 0 ? c0 : 1)));
    PR_TRY(ensure(bad, 8));
    PR_TRY(ensure(bnd, 8 * (PR_MAX_SECTIONS + 1)));
    PR_TRY(ensure(out, 8 * (PR_MAX_SECTIONS + 1)));
    PR_TRY(ensure(S.sec_of, g.n > 0 ? g.n : 1));
    PR_CUDA(cudaMemsetAsync(bad.ptr, 0, 8, st));
    PR_CUDA(cudaMemsetAsync(S.sec_of.ptr, 0xFF, g.n, st));
    PR_CUDA(cudaMemcpyAsync(bnd.ptr, S.sec_row, 8 * (S.nsec + 1), cudaMemcpyHostToDevice, st));
    const unsigned gr = grid_for(S.count, 256) > 4096 ? 4096 : grid_for(S.count, 256);
    if (S.count) {
        k_class0_order<<<gr, 256, 0, st>>>(S.ids.as<int32_t>(), S.count, c0, pos.as<int32_t>(),
                                           bad.as<unsigned long long>(), 0);
        k_class0_order<<<gr, 256, 0, st>>>(S.ids.as<int32_t>(), S.count, c0, pos.as<int32_t>(),
                                           bad.as<unsigned long long>(), 1);
        k_sec_of<<<gr, 256, 0, st>>>(S.ids.as<int32_t>(), S.count, bnd.as<int64_t>(), S.nsec, S.sec_of.as<uint8_t>());
    }
    k_sec_id<<<1, 32, 0, st>>>(S.ids.as<int32_t>(), S.count, c0, bnd.as<int64_t>(), S.nsec, out.as<int64_t>());
    unsigned long long nbad = 0;
    PR_CUDA(cudaMemcpyAsync(&nbad, bad.ptr, 8, cudaMemcpyDeviceToHost, st));
    PR_CUDA(cudaMemcpyAsync(S.sec_id, out.ptr, 8 * (S.nsec + 1), cudaMemcpyDeviceToHost, st));
    PR_CUDA(cudaStreamSynchronize(st));
    PR_CUDA(cudaGetLastError());
    if (nbad) return fail(PR_ERR_STATE, "class-0 rows out of id order");
    return PR_OK;
}

// Workspace sized once per graph (the executable-graph cache is keyed by the
// pointers, so a reallocation simply misses it).
static int ws_alloc(Graph &g, int64_t need_blocks, int64_t fcap) {
    int64_t n = g.n;
    PR_TRY(ensure(g.h, 8 * n));
    PR_TRY(ensure(g.reserved, 8 * n));
    PR_TRY(ensure(g.s2, 16 * n));
    PR_TRY(ensure(g.act, n));
    PR_TRY(ensure(g.in_d, n));
    PR_TRY(ensure(g.frontier2, 16 * fcap));
    PR_TRY(ensure(g.ctl, sizeof(RunCtl)));
    if (g.rows_cap == 0) g.rows_cap = 1 << 16;
    PR_TRY(ensure(g.rows, sizeof(pr_round_stats) * g.rows_cap));
    int64_t mb = (n + 255) / 256 + 8;
    if (need_blocks + 8 > mb) mb = need_blocks + 8;
    if (mb > g.max_blocks) {
        PR_TRY(ensure(g.partials, sizeof(Partial) * 3 * mb));
        g.max_blocks = mb;
    }
    return PR_OK;
}

int run_rounds(Graph &g_in, const pr_run_params &p, double *d_values, double *d_reserved, double *d_pending,
               pr_round_stats *rows, int64_t row_cap, pr_run_result *res) {
    Ctx &ctx = *g_in.ctx;
    cudaStream_t st = ctx.stream;
    const int algo = p.algorithm;
    if (algo < 0 || algo > 2) return fail(PR_ERR_ARG, "unknown algorithm");
    if (!(p.damping > 0.0 && p.damping < 1.0)) return fail(PR_ERR_ARG, "damping must be in (0,1)");
    if (!(p.threshold > 0.0)) return fail(PR_ERR_ARG, "threshold must be positive");
    if (p.mode < 0 || p.mode > 3) return fail(PR_ERR_ARG, "unknown mode");
    if (p.max_rounds < 0) return fail(PR_ERR_ARG, "max_rounds must be non-negative");
    const bool exact = p.mode == PR_MODE_EXACT;
    if (p.on_round && !exact) return fail(PR_ERR_ARG, "on_round observers need PR_MODE_EXACT");
    // on_round observers: the device loop runs in batches that snapshot
    // every state into a ring the host drains once per batch (one copy, no
    // host round trip per round); PUSHRANK_HOST_LOOP=1 / host_loop keep the
    // round-by-round form
    const bool observed = p.on_round && !p.host_loop && !getenv("PUSHRANK_HOST_LOOP");
    const bool host_loop = p.host_loop || (p.on_round && !observed);
    if (algo == PR_ALGO_IFP2 && !g_in.has_ifp2 && !g_in.ifp2_counted) return fail(PR_ERR_STATE, "IFP2 needs pr_preprocess_ifp2 first");
    // fast engines run on the relabelled layout; exact mode on the original
    Graph *gp = &g_in;
    phase_mark(ctx.stream, "run: enter");
    if (!exact) {
        PR_TRY(ensure_run_layout(g_in));
        gp = g_in.run;
        phase_mark(ctx.stream, "run: layout");
    }
    Graph &g = *gp;
    if (!exact && g.sort_deferred && g.fast_solves >= 1) {
        // the graph is being reused: sort its rows' sources now and rebuild
        // the schedules that copied them
        PR_TRY(sort_csc_rows(ctx, g.in_off, g.in_src, g.n, g.m));
        g.sort_deferred = false;
        for (auto &S : g.sched) {
            S.built = false;
            S.unit_blocks = 0;
            S.nsec = 0;
        }
        phase_mark(ctx.stream, "run: deferred row sort");
    }
    const int32_t *perm = exact ? nullptr : g_in.perm.as<int32_t>();
    if (algo == PR_ALGO_IFP2) {
        PR_TRY(preprocess_ifp2_device(g));
    } else {
        PR_TRY(ensure_dtc(g));
        if (!exact) PR_TRY(ensure_run_csr(g));   // IFP1 pushes along the full out-adjacency
    }
    PR_TRY(count_dangling(g));
    phase_mark(ctx.stream, "run: ifp2 split/dtc");
    const int which = algo == PR_ALGO_IFP2 ? 1 : 0;
    // persistent pull grid: as many blocks as fit on the device at once,
    PR_TRY(ensure_sched(g, which));
    // A dense round touches the compacted CSC, the share vector of the
    // sources and ~44 B of state per row.  When that overflows ~60% of L2 the
    // round is bandwidth-bound: k_pull<true> streams the CSC (evict-first)
    // at 4 blocks/SM.  Otherwise it is latency-bound: k_pull<false> issues
    // each row's drain loads before its gathers, at 3 blocks/SM (the extra
    // live registers).  Measured: C2 -9%, C4 -11%, C3 -1.4%; C5 prefers the former.
    const double ws = 4.0 * (double)g.sched[which].edges + 8.0 * (double)g.n + 44.0 * (double)g.sched[which].count;
    const double l2 = (double)(ctx.l2_bytes ? ctx.l2_bytes : (size_t)126 << 20);
    const bool stream = ws > 0.6 * l2;
    bool prefetch = ws < 4.0 * l2;   // C3 (1.9x L2) -1.4% with it, C5 (55x) +6%
    if (const char *e = getenv("PUSHRANK_PREFETCH")) prefetch = atoi(e) != 0;
    const void *k_pull_fn = stream ? (prefetch ? (const void *)k_pull<true, true, false>
                                               : (const void *)k_pull<true, false, false>)
                                   : (prefetch ? (const void *)k_pull<false, true, false>
                                               : (const void *)k_pull<false, false, false>);
    int per_sm = 0;
    PR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pull_fn, 256, 0));
    if (per_sm < 1) per_sm = 1;
    auto &S = g.sched[which];
    int64_t n = g.n;
    // persistent pull grid, ~UNITS_PER_BLOCK equal-cost units per block
    const int64_t pull_blocks = (int64_t)ctx.sm_count * per_sm;
    // Gauss-Seidel sections need vertex id == row (the IFP2 run layout's
    // prefix schedule); PUSHRANK_GS_SECTIONS overrides the default
    // Sections cut rounds (C2: 174 -> 98 at 4 sections) but each adds a
    // launch, a ramp and a reduction to the sweep, so they pay only when a
    // round is long: 2 sections past 1.5x L2 of round working set (C3: 14.8 ->
    // 11.5 ms), 6 past 16x (C5: 813 -> 598 ms at 4 sections in round 1; 461 ->
    // 441 ms from 4 to 6 with this round's kernels), none below (C2, C4).
    int nsec = 1;
    if ((algo == PR_ALGO_IFP2 || algo == PR_ALGO_IFP1) && g.class0_end >= 0) {
        nsec = gs_sections_default(ws, l2);
        if (const char *e = getenv("PUSHRANK_GS_SECTIONS")) nsec = atoi(e);
        if (nsec < 1) nsec = 1;
        if (nsec > PR_MAX_SECTIONS) nsec = PR_MAX_SECTIONS;
    }
    if (nsec > 1)
        k_pull_fn = stream ? (prefetch ? (const void *)k_pull<true, true, true> : (const void *)k_pull<true, false, true>)
                           : (prefetch ? (const void *)k_pull<false, true, true> : (const void *)k_pull<false, false, true>);
    PR_TRY(ensure_units(g, which, pull_blocks, nsec));
    // IFP1 sections: the id bounds of the sources of earlier sections and the
    // section of every row's vertex (the schedule interleaves class 0 and the
    // dangling receivers by degree; class-0 ids stay in row order)
    if (algo == PR_ALGO_IFP1 && g.sched[which].nsec > 1) {
        if (sections_by_id(g, which) != PR_OK) {
            PR_TRY(ensure_units(g, which, pull_blocks, 1));
        }
    }
    const int64_t fcap = n + g.m / TILE + 1;
    if (getenv("PUSHRANK_TIMING"))
        fprintf(stderr, "[pushrank] round working set %.1f MB (L2 %.1f MB): stream %d prefetch %d sections %d\n",
                ws / 1e6, l2 / 1e6, (int)stream, (int)prefetch, nsec);
    if (getenv("PUSHRANK_TIMING")) {
        auto &S = g.sched[which];
        int64_t e[4] = {0, 0, 0, 0};
        const int64_t rows[3] = {S.n_hub, S.n_hub + S.n_warp, S.count};
        for (int k = 0; k < 3; ++k)
            PR_CUDA(cudaMemcpy(&e[k], S.doff.as<int64_t>() + rows[k], 8, cudaMemcpyDeviceToHost));
        if (S.n_slices) PR_CUDA(cudaMemcpy(&e[3], S.sell_off.as<int64_t>() + S.n_slices, 8, cudaMemcpyDeviceToHost));
        fprintf(stderr, "[pushrank] bins: hub rows %lld (%lld edges), warp rows %lld (%lld edges), thread rows %lld "
                "(%lld edges, %lld SELL slots)\n", (long long)S.n_hub, (long long)e[0], (long long)S.n_warp,
                (long long)(e[1] - e[0]), (long long)(S.count - rows[1]), (long long)(e[2] - e[1]),
                (long long)(S.n_slices ? e[3] - e[1] : 0));
    }
    phase_mark(ctx.stream, "run: schedule");
    PR_TRY(ws_alloc(g, pull_blocks, fcap));
    phase_mark(ctx.stream, "run: workspace");

    Plan P;
    memset(&P, 0, sizeof(P));
    RunArgs &A = P.A;
    A.n = n;
    A.in_off = g.in_off.as<int64_t>();
    A.in_src = g.in_src.as<int32_t>();
    if (algo == PR_ALGO_IFP2) {
        A.push_off = g.live_off.as<int64_t>();
        A.push_tgt = g.live_tgt.as<int32_t>();
        A.row_len = g.live_deg.as<int32_t>();
        A.dtc = nullptr;
    } else {
        A.push_off = g.out_off.as<int64_t>();
        A.push_tgt = g.out_tgt.as<int32_t>();
        A.row_len = g.out_deg.as<int32_t>();
        A.dtc = g.dtc.as<int32_t>();
    }
    A.deg = g.out_deg.as<int32_t>();
    A.ids = S.ids.as<int32_t>();
    A.T.ids = S.ids.as<int32_t>();
    A.T.doff = S.doff.as<int64_t>();
    A.T.csc = S.csc.as<int32_t>();
    A.T.sell_off = S.sell_off.as<int64_t>();
    A.T.count = S.count;
    A.T.n_hub = S.n_hub;
    A.T.n_warp = S.n_warp;
    A.T.chunk_base = S.chunk_base.as<int64_t>();
    A.T.row_cnt = S.row_cnt.as<int32_t>();
    A.T.chunk_part = S.chunk_part.as<double>();
    A.T.units = S.units.as<int2>();
    A.T.n_units = S.n_units;
    A.nsec = S.nsec;
    A.sec = 0;
    A.sec_of = (algo == PR_ALGO_IFP1 && S.nsec > 1) ? S.sec_of.as<uint8_t>() : nullptr;
    for (int k = 0; k <= PR_MAX_SECTIONS; ++k)
        A.sec_id[k] = k <= S.nsec ? (A.sec_of ? S.sec_id[k] : S.sec_row[k]) : S.count;
    // clear_seeds invariant: the round-0 seeds (in-degree 0, run-layout class
    // 1, ids >= class0_end) are never an "early" source of any section
    if (S.nsec > 1 && g.class0_end >= 0)
        for (int k = 0; k <= S.nsec; ++k)
            if (A.sec_id[k] > g.class0_end) return fail(PR_ERR_STATE, "section bound above the first seed id");
    for (int k = 0; k <= PR_MAX_SECTIONS; ++k) {
        A.sec_row[k] = k <= S.nsec ? S.sec_row[k] : S.count;
        A.sec_unit[k] = k <= S.nsec ? S.sec_unit[k] : S.n_units;
    }
    A.d_count = S.count;
    A.seeds = S.seed_ids.as<int32_t>();
    A.n_seed = S.n_seed;
    A.in_d = g.in_d.as<uint8_t>();
    A.h = g.h.as<double>();
    A.reserved = g.reserved.as<double>();
    A.s = g.s2.as<double>();
    A.frontier = g.frontier2.as<long long>();
    A.fcap = fcap;
    A.act = g.act.as<uint8_t>();
    A.partials = g.partials.as<Partial>();
    A.max_blocks = g.max_blocks;
    A.ctl = g.ctl.as<RunCtl>();
    A.T.unit_ctr = &A.ctl->unit_ctr;
    A.rows = g.rows.as<pr_round_stats>();
    A.rows_cap = g.rows_cap;
    A.c = p.damping;
    A.xi = p.threshold;
    A.frac = algo == PR_ALGO_FPFULL ? 1.0 - p.damping : 1.0;
    A.algo = algo;
    A.policy = p.mode;
    A.conv_all = p.converged_scope == PR_CONV_ALL;
    A.max_rounds = p.max_rounds;
    int64_t pull_edges = algo == PR_ALGO_IFP2 ? g.ifp2.live_edges : g.m;
    double sw = p.push_switch > 0.0 ? p.push_switch : 0.05;
    A.push_work = sw * (double)(pull_edges + S.count);
    A.n_scan = (double)(algo == PR_ALGO_FPFULL ? n : n - g.n_dangling);
    P.exact = exact;
    P.g_all = grid_for(n, 256);
    P.g_pull = (unsigned)pull_blocks;
    P.k_pull_fn = k_pull_fn;
    for (int k = 0; k < PR_MAX_SECTIONS; ++k) {
        P.k_pull_sec[k] = k_pull_fn;
        P.g_pull_sec[k] = (unsigned)pull_blocks;
    }
    // A section made of thread rows (C5's last: 21 M rows of ~7 in-edges, all
    // of the sweep's per-vertex drain traffic) is bound by each thread's chain
    // of dependent loads -- bounds, indices, shares, drain inputs -- not by
    // the gathers' request rate (ncu: long scoreboard 77%, L1->L2 requests 66%
    // against 80-83% in the warp-row sections).  Its launch uses the form that
    // issues a row's drain loads before its gathers, at 3 blocks/SM, while the
    // other sections keep the plain form at 4.  PUSHRANK_PREFETCH_THREADS=0/1.
    {
        bool pf_threads = S.nsec > 1 && !prefetch;
        if (const char *e = getenv("PUSHRANK_PREFETCH_THREADS")) pf_threads = S.nsec > 1 && !prefetch && atoi(e) != 0;
        if (pf_threads) {
            const void *k_pf = stream ? (const void *)k_pull<true, true, true> : (const void *)k_pull<false, true, true>;
            int b = 0;
            PR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_pf, 256, 0));
            if (b < 1) b = 1;
            const int64_t t0 = S.n_hub + S.n_warp;
            for (int k = 0; k < S.nsec; ++k) {
                const int64_t lo = S.sec_row[k], hi = S.sec_row[k + 1];
                const int64_t thr = hi - (lo > t0 ? lo : t0);
                if (hi > lo && (double)thr > 0.9 * (double)(hi - lo)) {
                    P.k_pull_sec[k] = k_pf;
                    P.g_pull_sec[k] = (unsigned)((int64_t)ctx.sm_count * b);
                }
            }
        }
    }
    // L1 / shared-memory split of the dense round: PUSHRANK_CARVEOUT=percent
    // of the unified array given to shared memory (A/B; default: driver's)
    if (const char *e = getenv("PUSHRANK_CARVEOUT"))
        PR_CUDA(cudaFuncSetAttribute(k_pull_fn, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(e)));
    // reducing kernels of the fast engine: one resident wave, grid-stride
    // (a block's lifetime -- reduce, publish -- is latency, not bandwidth)
    auto wave = [&](const void *k) -> unsigned {
        int b = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, 256, 0) != cudaSuccess || b < 1) b = 1;
        return (unsigned)(ctx.sm_count * b);
    };
    const unsigned w_init = wave((const void *)k_init), w_scan = wave((const void *)k_scan),
                   w_total = wave((const void *)k_total);
    P.g_red = P.g_all < w_init ? P.g_all : w_init;
    P.g_total = P.g_all < w_total ? P.g_all : w_total;
    P.g_scan = grid_for(S.count, 256);
    if (P.g_scan > w_scan) P.g_scan = w_scan;
    P.g_push = (unsigned)ctx.sm_count * 8;

    PR_CUDA(cudaMemsetAsync(g.in_d.ptr, 0, n, st));
    if (S.count) k_mark_d<<<grid_for(S.count, 256), 256, 0, st>>>(A.ids, S.count, g.in_d.as<uint8_t>());

    cudaEvent_t e0, e1, e2;
    PR_CUDA(cudaEventCreate(&e0));
    PR_CUDA(cudaEventCreate(&e1));
    PR_CUDA(cudaEventCreate(&e2));
    PR_CUDA(cudaEventRecord(e0, st));
    int64_t obs_k = 0;
    if (observed) {
        // ring of K states (reserved | pending), K <= 64, within 256 MiB,
        // drained into a page-locked host buffer of the same size
        obs_k = ((int64_t)1 << 28) / (16 * (n > 0 ? n : 1));
        if (obs_k > 64) obs_k = 64;
        if (obs_k < 1) obs_k = 1;
        PR_TRY(ensure(g.obs_ring, 16 * n * obs_k));
        const size_t hb = (size_t)(16 * n * obs_k);
        if (ctx.obs_host_bytes < hb) {
            if (ctx.obs_host) cudaFreeHost(ctx.obs_host);
            ctx.obs_host = nullptr;
            ctx.obs_host_bytes = 0;
            PR_CUDA(cudaMallocHost(&ctx.obs_host, hb));
            ctx.obs_host_bytes = hb;
        }
        A.obs_batch = obs_k;
        A.obs_ring = g.obs_ring.as<double>();
        A.use_graph = 0;
        k_reset<<<1, 1, 0, st>>>(A);
        k_ex_init<<<P.g_all, 256, 0, st>>>(A);
        k_ex_prep<<<P.g_all, 256, 0, st>>>(A);
        PR_CUDA(cudaGetLastError());
    }
    if (!host_loop) {
        // the plan's bytes (graph-owned conditional handles still zero) key
        // the context's executable-graph cache
        const unsigned char *pb = reinterpret_cast<const unsigned char *>(&P);
        std::vector<unsigned char> key(pb, pb + sizeof(P));
        Ctx::ExecSlot *slot = nullptr;
        for (auto &e : ctx.execs)
            if (e.exec && e.key == key) { slot = &e; break; }
        if (!slot) {
            slot = &ctx.execs[0];
            for (auto &e : ctx.execs)
                if (!e.exec || e.used < slot->used) slot = &e;
            if (!slot->exec) {
                for (auto &e : ctx.execs)
                    if (!e.exec) { slot = &e; break; }
            }
            if (slot->exec) cudaGraphExecDestroy(slot->exec);
            if (slot->graph) cudaGraphDestroy(slot->graph);
            slot->exec = nullptr;
            slot->graph = nullptr;
            slot->key.clear();
            PR_TRY(build_graph(P, &slot->graph, &slot->exec));
            slot->key = std::move(key);
            phase_mark(ctx.stream, "run: graph instantiate");
        }
        slot->used = ++ctx.exec_tick;
        if (!observed) {
            PR_CUDA(cudaGraphLaunch(slot->exec, st));
        } else {
            double *ring = static_cast<double *>(ctx.obs_host);
            RunCtl hc;
            for (;;) {
                PR_CUDA(cudaMemcpyAsync(&hc, A.ctl, sizeof(hc), cudaMemcpyDeviceToHost, st));
                PR_CUDA(cudaStreamSynchronize(st));
                if (hc.done) break;
                PR_CUDA(cudaGraphLaunch(slot->exec, st));
                PR_CUDA(cudaMemcpyAsync(&hc, A.ctl, sizeof(hc), cudaMemcpyDeviceToHost, st));
                PR_CUDA(cudaStreamSynchronize(st));
                if (hc.obs_count > 0)
                    PR_CUDA(cudaMemcpyAsync(ring, A.obs_ring, 16 * n * hc.obs_count, cudaMemcpyDeviceToHost, st));
                PR_CUDA(cudaStreamSynchronize(st));
                // reference semantics: called after round t's update (engines.py:453-454)
                for (int64_t j = 0; j < hc.obs_count; ++j)
                    p.on_round(p.user, hc.obs_t0 + j, ring + 2 * j * n, ring + (2 * j + 1) * n);
            }
        }
    } else {
        A.use_graph = 0;
        RunCtl hc;
        k_reset<<<1, 1, 0, st>>>(A);
        if (exact) {
            k_ex_init<<<P.g_all, 256, 0, st>>>(A);
            k_ex_prep<<<P.g_all, 256, 0, st>>>(A);
        } else {
            k_init<<<P.g_red, 256, 0, st>>>(A);
        }
        std::vector<double> obs_r, obs_h;
        if (p.on_round) {
            obs_r.resize((size_t)n);
            obs_h.resize((size_t)n);
        }
        for (;;) {
            PR_CUDA(cudaMemcpyAsync(&hc, A.ctl, sizeof(hc), cudaMemcpyDeviceToHost, st));
            PR_CUDA(cudaStreamSynchronize(st));
            if (hc.done) break;
            if (exact) {
                k_ex_pull<<<P.g_all, 256, 0, st>>>(A);
                if (p.on_round) {
                    // reference semantics: called after round t's update (engines.py:453-454)
                    PR_CUDA(cudaMemcpyAsync(obs_r.data(), A.reserved, 8 * n, cudaMemcpyDeviceToHost, st));
                    PR_CUDA(cudaMemcpyAsync(obs_h.data(), A.h, 8 * n, cudaMemcpyDeviceToHost, st));
                    PR_CUDA(cudaStreamSynchronize(st));
                    p.on_round(p.user, hc.rows - 1, obs_r.data(), obs_h.data());
                }
                k_ex_prep<<<P.g_all, 256, 0, st>>>(A);
            } else if (hc.mode == 0) {
                void *kargs[] = {&A};
                for (int sec = 0; sec < A.nsec; ++sec) {
                    A.sec = sec;
                    PR_CUDA(cudaLaunchKernel(P.k_pull_sec[sec], dim3(P.g_pull_sec[sec]), dim3(256), kargs, 0, st));
                }
                A.sec = 0;
            } else {
                k_push<<<P.g_push, 256, 0, st>>>(A);
                k_scan<<<P.g_scan, 256, 0, st>>>(A);
            }
            PR_CUDA(cudaGetLastError());
        }
    }
    PR_CUDA(cudaEventRecord(e1, st));
    int64_t settled = 0;
    if (algo == PR_ALGO_IFP2) {
        settled = g.ifp2.source_edges;
        if (g.ifp2.dangling)
        {
            // exact: thread per vertex in ascending source order; fast: a warp
            // for each dangling vertex with > 32 sources, a thread for the rest
            const int64_t nd = g.ifp2.dangling;
            int64_t big = 0;
            if (!exact) PR_TRY(count_settle_big(g, &big));
            if (exact) {
                k_settle<<<grid_for(nd, 256), 256, 0, st>>>(A, g.dang_ids.as<int32_t>(), 0, nd,
                                                           g.src_off.as<int64_t>(), g.src_ids.as<int32_t>(), 1);
            } else {
                // sources are the non-dangling run ids [0, live_end); the
                // round loop is over, so the share buffer holds w
                const int64_t n_src = g.live_end >= 0 ? g.live_end : n;
                double *w = A.s;
                k_settle_w<<<grid_for(n_src, 256) > 4096 ? 4096 : grid_for(n_src, 256), 256, 0, st>>>(A, n_src, w);
                if (big)
                    k_settle_fast<<<grid_for(big * 32, 256), 256, 0, st>>>(
                        A, w, g.dang_ids.as<int32_t>(), 0, big, g.src_off.as<int64_t>(), g.src_ids.as<int32_t>(), 0);
                if (nd > big)
                    k_settle_fast<<<grid_for(nd - big, 256), 256, 0, st>>>(
                        A, w, g.dang_ids.as<int32_t>(), big, nd, g.src_off.as<int64_t>(), g.src_ids.as<int32_t>(), 1);
            }
        }
    }
    int include_h = algo == PR_ALGO_IFP1 ? 1 : 0;
    k_total<<<P.g_total, 256, 0, st>>>(A, include_h, settled, algo == PR_ALGO_IFP2 ? 1 : 0);
    {
        unsigned gs = grid_for(n, 256);
        if (gs > 4096) gs = 4096;
        if (d_values) k_scale<<<gs, 256, 0, st>>>(A, include_h, d_values, perm);
        if (d_reserved) k_unpermute<<<gs, 256, 0, st>>>(A.reserved, n, perm, d_reserved);
        if (d_pending) k_unpermute<<<gs, 256, 0, st>>>(A.h, n, perm, d_pending);
    }
    PR_CUDA(cudaEventRecord(e2, st));
    PR_CUDA(cudaEventSynchronize(e2));
    phase_mark(ctx.stream, "run: solve");
    PR_CUDA(cudaGetLastError());
    float ms_loop = 0.f, ms_all = 0.f;
    PR_CUDA(cudaEventElapsedTime(&ms_loop, e0, e1));
    PR_CUDA(cudaEventElapsedTime(&ms_all, e0, e2));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(e2);
    RunCtl hc;
    PR_CUDA(cudaMemcpy(&hc, A.ctl, sizeof(hc), cudaMemcpyDeviceToHost));
    int64_t nrows = hc.rows;
    if (rows && row_cap > 0) {
        int64_t k = nrows < row_cap ? nrows : row_cap;
        if (k > g.rows_cap) k = g.rows_cap;
        PR_CUDA(cudaMemcpy(rows, A.rows, sizeof(pr_round_stats) * k, cudaMemcpyDeviceToHost));
    }
    if (res) {
        res->rounds = hc.pull_rounds + hc.push_rounds;
        res->rows = nrows;
        res->push_ops = hc.push_ops;
        res->push_ops_dangling = hc.push_ops_dangling;
        res->settled = settled;
        res->pull_rounds = hc.pull_rounds;
        res->push_rounds = hc.push_rounds;
        res->mass_total = hc.mass_total;
        res->push_ms = ms_all;
        res->round_ms = ms_loop;
        res->bytes_moved = hc.bytes;
        res->pull_ms = hc.pull_ns * 1e-6;
        res->pull_bytes = hc.pull_bytes;
        res->sparse_ms = hc.sparse_ns * 1e-6;
        // device-counted solve kernels + the host-launched un-permute copies
        res->launches = (int64_t)hc.launches + (d_reserved ? 1 : 0) + (d_pending ? 1 : 0);
    }
    if (!exact) g.fast_solves += 1;
    if (hc.done == 2)
        return fail(PR_ERR_NOT_SETTLED,
                    "sync simulation did not settle in " + std::to_string(p.max_rounds) + " iterations");
    return PR_OK;
}

}  // namespace pr
