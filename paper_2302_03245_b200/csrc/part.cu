// part.cu -- local step of the vertex-range partitioned rounds (multi-GPU,
// SURVEY.md §8(e); host orchestration in distributed.py).
//
// A partition owns `owned` vertices and the in-edge rows of them, with
// source ids in the padded global space (rank r's vertices at [r*slot, ...)).
// Each call is one bulk-synchronous step on the context stream:
//   init   -- state 0 (h = 1): drain, shares of the owned slice, statistics
//   round  -- h_v = (active ? 0 : h_v) + sum_{u in in(v)} s_full[u] for owned
//             v (sequential ascending-source sums: the same order as the
//             single-GPU exact engine and np.bincount), then the drain
//   settle -- IFP2: reserved_d = h_d + sum x_full[u] over d's sources
// Statistics are reduced per block and then by one block in fixed order
// (deterministic) and returned to the host, which all-reduces them.
//
// Two forms of the round:
//   exact -- thread per owned vertex, sequential ascending-source sums: the
//            summation order of the single-GPU exact engine and np.bincount,
//            so partitions are bit-identical to sync_simulate (tests);
//   fast  -- the single-GPU dense-round gather (bins.cuh) over a pull
//            schedule of the partition's receiving rows (sched.cu: rows by
//            descending in-degree, hub chunks / warp rows / thread rows,
//            equal-cost units for a persistent grid), then the owned
//            vertices outside it.  Summation order is fixed by the schedule
//            (deterministic run to run), not ascending.
// The *_device entry points leave the statistics on the device (9 doubles:
// l1, above, nd_above, nact, work, push_ops, push_dang, conv_all,
// conv_scan) and never synchronise, so the caller can queue rounds and
// their collectives back to back on the library stream.
#include <cstring>
#include <vector>

#include <type_traits>

#include "internal.cuh"
#include "reduce.cuh"
#include "bins.cuh"
#include "cubutil.cuh"

#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

namespace pr {

// resident blocks per SM of the plain k_part_pull form (registers: 64 at 4, 85 at 3)
#ifndef PR_PART_BLOCKS
#define PR_PART_BLOCKS 4
#endif
constexpr int64_t PART_ROW_COST = 8;   // default per-row weight of the partition bounds

#define PR_MAX_PEERS 8   // fused exchange: ranks whose replicas a round stores into

// an owned vertex that is not a row of the pull schedule
struct OutsideRow {
    const int64_t *in_off;
    const uint8_t *recv;
    __host__ __device__ bool operator()(int32_t v) const { return !(recv[v] && in_off[v + 1] > in_off[v]); }
};

struct Part {
    Ctx *ctx;
    int64_t owned, slot, edges;
    int algorithm;
    double c, xi;
    DevBuf in_off, in_src, deg, row_len, dtc, dang, recv;   // int64 offsets, int32 ids/degrees, uint8 flags
    DevBuf h, reserved, act, partials, stats;
    // fast form: the partition as a Graph of `owned` rows (local ids) whose
    // sources are padded global ids, and its pull schedule
    Graph *sg = nullptr;
    int which = 0;            // schedule: 0 in-degree > 0 (IFP1), 1 and non-dangling (IFP2)
    int64_t blocks = 0;       // persistent pull grid
    bool stream_csc = false;  // evict-first index loads (round working set > 0.6 L2)
    bool prefetch = false;    // drain inputs ahead of the gathers (round working set < 4 L2)
    int nsec = 1;             // rank-local Gauss-Seidel sections
    int64_t sec_id[PR_MAX_SECTIONS + 1] = {};   // local-id bound of earlier sections' sources
    DevBuf outside;           // int32: owned vertices outside the schedule
    int64_t n_outside = 0;
    // fused exchange: replicas of the full share vector (parity 0/1) of
    // every rank; own ones allocated here, peers' opened through CUDA IPC
    int parts = 0, rank = 0;
    void *own_full[2] = {nullptr, nullptr};
    double *peer[2][PR_MAX_PEERS] = {};
    std::vector<void *> opened;
    // the replicas of every rank are mapped (set_peers / set_peer_ptrs) and
    // not yet closed: the fused entry points refuse to run otherwise
    bool fused_ready = false;
    const double *prev9 = nullptr;   // next fast round: skip it if this row shows no active vertex
    DevBuf cst;               // Partial: statistics of the outside vertices from round 1 on
    DevBuf dmask;             // uint8 [owned]: destination ranks of each vertex's out-edges (empty: all)
    int64_t exch_entries = -1;   // sum over owned vertices of popcount(dmask): shares sent per dense round
    DevBuf big_dang;          // int32: dangling rows with > 32 sources (fast settle: a warp each)
    int64_t n_big = -1;
    unsigned long long *unit_ctr = nullptr;
    unsigned *done = nullptr;   // last-block counter of the fast round's last section
    ~Part() {
        delete sg;
        for (void *p : opened) cudaIpcCloseMemHandle(p);
        for (void *p : own_full)
            if (p) cudaFree(p);
    }
};

struct PartArgs {
    int64_t owned;
    const int64_t *in_off;
    const int32_t *in_src;
    const int32_t *deg, *row_len, *dtc;
    const uint8_t *dang, *recv;
    // sparse boundary exchange: bit k set iff the vertex has an out-edge into
    // rank k's range (only those ranks' replicas receive its share); null = all
    const uint8_t *dmask;
    double *h, *reserved;
    uint8_t *act;
    Partial *partials;
    double c, xi;
};

// Where a drained share goes.  peers.n == 0: this rank's slice `mine` (the
// caller all-gathers it).  peers.n > 0: the fused exchange -- the share is
// stored straight into every rank's replica of the full share vector at
// this rank's slot (peer pointers mapped over NVLink through CUDA IPC; own
// replica included), so the all-gather happens inside the round kernel,
// overlapped with the gathers of the rows still running.
struct ShareOut {
    double *mine;
    double *peer[PR_MAX_PEERS];
    int n;
    int64_t off;   // rank * slot
    __device__ __forceinline__ void store(int64_t v, double x, unsigned mask) const {
        if (n == 0) {
            mine[v] = x;
            return;
        }
#pragma unroll
        for (int k = 0; k < PR_MAX_PEERS; ++k)
            if (k < n && (mask >> k & 1u)) peer[k][off + v] = x;
    }
};

// per-block statistics of the drain (ints: nact, work, push_ops, push_dang,
// conv_all, conv_scan; floats in l1/above/nd_above)
// per-vertex inputs of the drain, loadable ahead of a row's gathers
struct PartIn {
    int32_t v, dv;
    double h, rv;
    bool act, dang;
    unsigned mask;   // replicas that receive this vertex's share
};

__device__ __forceinline__ PartIn part_load(const PartArgs &A, int32_t v) {
    PartIn q;
    q.v = v;
    q.dv = __ldg(&A.deg[v]);
    q.h = A.h[v];
    q.rv = A.reserved[v];
    q.act = A.act[v] != 0;
    q.dang = __ldg(&A.dang[v]) != 0;
    q.mask = A.dmask ? (unsigned)__ldg(&A.dmask[v]) : 0xFFu;
    return q;
}

// h_v = (drained last state ? 0 : h_v) + inflow, then the drain
__device__ __forceinline__ void part_finish(const PartArgs &A, const PartIn &q, double sum, const ShareOut &out,
                                            Partial &p) {
    const int64_t v = q.v;
    const double hv = __dadd_rn(q.act ? 0.0 : q.h, sum);
    const bool scan = !q.dang;
    const bool above = hv > A.xi;
    p.l1 += hv;
    if (above) {
        p.above += hv;
        if (scan) p.nd_above += hv;
    } else {
        p.conv_all += 1;
        if (scan) p.conv_scan += 1;
    }
    const bool active = above && scan;
    A.act[v] = active;
    if (active) {
        const int32_t len = __ldg(&A.row_len[v]);
        A.reserved[v] = __dadd_rn(q.rv, hv);
        A.h[v] = hv;
        out.store(v, len > 0 ? __ddiv_rn(__dmul_rn(A.c, hv), (double)q.dv) : 0.0, q.mask);
        p.nact += 1;
        p.work += (int64_t)q.dv + 1;
        p.push_ops += len;
        p.push_dang += __ldg(&A.dtc[v]);
    } else {
        A.h[v] = hv;
        out.store(v, 0.0, q.mask);
    }
}

__device__ __forceinline__ void part_drain(const PartArgs &A, int64_t v, double *s_mine, Partial &p) {
    const double hv = A.h[v];
    const int32_t dv = A.deg[v];
    const bool scan = !A.dang[v];
    const bool above = hv > A.xi;
    p.l1 += hv;
    if (above) {
        p.above += hv;
        if (scan) p.nd_above += hv;
    } else {
        p.conv_all += 1;
        if (scan) p.conv_scan += 1;
    }
    const bool active = above && scan;
    A.act[v] = active;
    if (active) {
        const int32_t len = A.row_len[v];
        A.reserved[v] = __dadd_rn(A.reserved[v], hv);
        s_mine[v] = len > 0 ? __ddiv_rn(__dmul_rn(A.c, hv), (double)dv) : 0.0;
        p.nact += 1;
        p.work += (int64_t)dv + 1;
        p.push_ops += len;
        p.push_dang += A.dtc[v];
    } else {
        s_mine[v] = 0.0;
    }
}

__global__ void __launch_bounds__(256) k_part_init(PartArgs A, double *s_mine) {
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    Partial p;
    zero(p);
    if (v < A.owned) {
        A.h[v] = 1.0;
        A.reserved[v] = 0.0;
        part_drain(A, v, s_mine, p);
    }
    block_reduce(p);
    if (threadIdx.x == 0) A.partials[blockIdx.x] = p;
}

__global__ void __launch_bounds__(256) k_part_round(PartArgs A, const double *__restrict__ s_full, double *s_mine) {
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    Partial p;
    zero(p);
    if (v < A.owned) {
        double acc = 0.0;
        if (A.recv[v])
            for (int64_t e = A.in_off[v]; e < A.in_off[v + 1]; ++e) acc = __dadd_rn(acc, __ldg(&s_full[A.in_src[e]]));
        A.h[v] = __dadd_rn(A.act[v] ? 0.0 : A.h[v], acc);
        part_drain(A, v, s_mine, p);
    }
    block_reduce(p);
    if (threadIdx.x == 0) A.partials[blockIdx.x] = p;
}

// fast round: binned gather over the receiving rows (drain inputs loaded
// before each row's gathers when the round is L2-resident), then the owned
// vertices outside the schedule (no inflow)
struct PartRows {
    const PartArgs &A;
    const int32_t *ids;
    const ShareOut &s_mine;
    Partial &p;
    __device__ __forceinline__ PartIn pre(bool valid, int64_t row) const {
        if (valid) return part_load(A, __ldg(&ids[row]));
        PartIn q;
        q.v = 0;
        q.dv = 0;
        q.h = q.rv = 0.0;
        q.act = q.dang = false;
        return q;
    }
    __device__ __forceinline__ void fin(bool valid, const PartIn &q, double sum) {
        if (valid) part_finish(A, q, sum, s_mine, p);
    }
    __device__ __forceinline__ void single(int64_t row, double sum) {
        part_finish(A, part_load(A, __ldg(&ids[row])), sum, s_mine, p);
    }
};

// One launch of a round: the units [u_lo, u_hi) of one Gauss-Seidel section
// (all of them without sections).  kind: 0 Jacobi, 1 transition, 2 GS
// (bins.cuh Src: sections are rank-local, early(u) tests this rank's padded
// slot); the last section also drains the vertices outside the schedule.
// Each section writes its block partials to its own region.
struct PullSec {
    int64_t u_lo, u_hi;
    Src src;
    int kind, last, region;
    // the last section's last block reduces every section's partials (fixed
    // order) into the statistics, so a round needs no separate reduction
    unsigned *done;          // block arrival counter of the last section
    Partial *stats;          // the reduced statistics
    double *out9;            // and as 9 doubles (may be null)
    unsigned long long *ctr; // unit counters to reset (PR_MAX_SECTIONS)
    // the previous round's all-reduced statistics (may be null): with no
    // active vertex anywhere the state is final and this queued round is a
    // no-op -- skip its sweep (rounds queued past termination in a batch)
    const double *prev9;
    // the round's sweep kind regardless of sections (distributed.sweep_kind:
    // 0 round 0, 1 round 1, 2 later): the owned vertices outside the
    // schedule (no inflow) are drained in rounds 0 and 1 only -- round 1
    // clears their round-0 shares -- and their statistics, constant from
    // then on, are recorded in round 1 (*cst) and added in later rounds
    int round_kind;
    Partial *cst;
};

template <bool STREAM, bool PREFETCH, int SRC>
__device__ __forceinline__ void part_bins(const PartArgs &A, const BinView &T, const PullSec &S, const ShareOut &s_mine,
                                          Partial &p) {
    PartRows rows{A, T.ids, s_mine, p};
    if constexpr (PREFETCH) {
        bins_run<STREAM, true, SRC>(T, S.u_lo, S.u_hi, S.src, rows);
    } else {
        auto thread_row = [&](bool valid, int64_t row, double sum) {
            if (valid) part_finish(A, part_load(A, __ldg(&T.ids[row])), sum, s_mine, p);
        };
        auto single_row = [&](int64_t row, double sum) { rows.single(row, sum); };
        bins_run_plain<STREAM, SRC>(T, S.u_lo, S.u_hi, S.src, thread_row, single_row);
    }
}

template <bool STREAM, bool PREFETCH>
__global__ void __launch_bounds__(256, PREFETCH ? 3 : PR_PART_BLOCKS) k_part_pull(PartArgs A, BinView T, const int32_t *outside,
                                                                    int64_t n_outside, const PullSec S,
                                                                    const ShareOut s_mine) {
    if (S.prev9 && S.prev9[3] == 0.0) {
        // terminated: leave the state as it is; a zero statistics row (never
        // read: the host stops at the previous one)
        if (S.last && blockIdx.x == 0 && threadIdx.x < 9 && S.out9) S.out9[threadIdx.x] = 0.0;
        return;
    }
    Partial p;
    zero(p);
    if (S.kind == 0) part_bins<STREAM, PREFETCH, 0>(A, T, S, s_mine, p);
    else if (S.kind == 1) part_bins<STREAM, PREFETCH, 2>(A, T, S, s_mine, p);
    else part_bins<STREAM, PREFETCH, 1>(A, T, S, s_mine, p);
    Partial q;   // the outside vertices' share of the statistics
    zero(q);
    if (S.last && S.round_kind < 2)
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_outside;
             i += (int64_t)gridDim.x * blockDim.x)
            part_finish(A, part_load(A, __ldg(&outside[i])), 0.0, s_mine, q);
    add(p, q);
    if (s_mine.n) __threadfence_system();   // peer stores performed before the round's barrier
    block_reduce(p);
    if (threadIdx.x == 0) A.partials[(int64_t)S.region * gridDim.x + blockIdx.x] = p;
    if (!S.last) return;
    if (S.round_kind == 1) {
        block_reduce(q);
        if (threadIdx.x == 0) A.partials[(int64_t)PR_MAX_SECTIONS * gridDim.x + blockIdx.x] = q;
    }
    __shared__ bool is_last;
    if (threadIdx.x == 0) {
        __threadfence();
        is_last = atomicAdd(S.done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    Partial acc;
    zero(acc);
    const int64_t total = (int64_t)(S.region + 1) * gridDim.x;
    for (int64_t b = threadIdx.x; b < total; b += blockDim.x) add(acc, load_partial(A.partials + b));
    block_reduce(acc);
    if (S.round_kind == 1) {
        Partial c;
        zero(c);
        for (int64_t b = threadIdx.x; b < gridDim.x; b += blockDim.x)
            add(c, load_partial(A.partials + (int64_t)PR_MAX_SECTIONS * gridDim.x + b));
        block_reduce(c);
        if (threadIdx.x == 0) *S.cst = c;
    }
    if (threadIdx.x == 0) {
        if (S.round_kind >= 2) add(acc, *S.cst);
        *S.stats = acc;
        if (S.out9) {
            S.out9[0] = acc.l1;
            S.out9[1] = acc.above;
            S.out9[2] = acc.nd_above;
            S.out9[3] = (double)acc.nact;
            S.out9[4] = (double)acc.work;
            S.out9[5] = (double)acc.push_ops;
            S.out9[6] = (double)acc.push_dang;
            S.out9[7] = (double)acc.conv_all;
            S.out9[8] = (double)acc.conv_scan;
        }
        for (int k = 0; k < PR_MAX_SECTIONS; ++k) S.ctr[k] = 0;
        *S.done = 0;
    }
}

// state 0 (h = 1) of the fast form: shares through the ShareOut
__global__ void __launch_bounds__(256) k_part_init_fast(PartArgs A, const ShareOut out) {
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    Partial p;
    zero(p);
    if (v < A.owned) {
        A.reserved[v] = 0.0;
        PartIn q = part_load(A, (int32_t)v);
        q.h = 1.0;
        q.rv = 0.0;
        q.act = false;
        A.h[v] = 1.0;
        part_finish(A, q, 0.0, out, p);
    }
    if (out.n) __threadfence_system();
    block_reduce(p);
    if (threadIdx.x == 0) A.partials[blockIdx.x] = p;
}

__global__ void k_part_shares(PartArgs A, double *x_mine) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < A.owned; v += (int64_t)gridDim.x * blockDim.x)
        x_mine[v] = A.deg[v] > 0 ? __ddiv_rn(__dmul_rn(A.c, A.reserved[v]), (double)A.deg[v]) : 0.0;
}

__global__ void __launch_bounds__(256) k_part_settle(PartArgs A, const double *__restrict__ x_full) {
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    Partial p;
    zero(p);
    if (v < A.owned) {
        if (A.dang[v]) {
            double acc = 0.0;
            for (int64_t e = A.in_off[v]; e < A.in_off[v + 1]; ++e) acc = __dadd_rn(acc, x_full[A.in_src[e]]);
            p.push_ops = A.in_off[v + 1] - A.in_off[v];
            A.reserved[v] = __dadd_rn(A.h[v], acc);
            A.h[v] = 0.0;
        }
        const double hv = A.h[v];
        const bool above = hv > A.xi, scan = !A.dang[v];
        p.l1 = hv;
        if (above) {
            p.above = hv;
            if (scan) p.nd_above = hv;
        } else {
            p.conv_all = 1;
            if (scan) p.conv_scan = 1;
        }
    }
    block_reduce(p);
    if (threadIdx.x == 0) A.partials[blockIdx.x] = p;
}

// The settle of the fast local step, as the engine's (rounds.cu
// k_settle_fast): every dangling row with more than 32 sources gets a warp of
// its own (8 gathers in flight per lane, fixed shuffle tree), launched first
// over the list of those rows; then a thread per owned vertex sums the short
// rows (8 in flight, ascending) and reduces the statistics.  Deterministic;
// k_part_settle keeps the sequential ascending-source sums of the exact form.
struct BigDang {
    const int64_t *in_off;
    const uint8_t *dang;
    __host__ __device__ bool operator()(int32_t v) const { return dang[v] && in_off[v + 1] - in_off[v] > 32; }
};

__global__ void __launch_bounds__(256) k_part_settle_big(PartArgs A, const double *__restrict__ x_full,
                                                         const int32_t *__restrict__ big, int64_t n_big) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp; i < n_big; i += nwarps) {
        const int32_t v = big[i];
        const double acc = span_sum_warp<false, 0>(A.in_src, A.in_off[v], A.in_off[v + 1], Src{x_full, x_full, 0, 0});
        if (lane == 0) {
            A.reserved[v] = __dadd_rn(A.h[v], acc);
            A.h[v] = 0.0;
        }
    }
}

__global__ void __launch_bounds__(256) k_part_settle_fast(PartArgs A, const double *__restrict__ x_full) {
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    Partial p;
    zero(p);
    if (v < A.owned) {
        if (A.dang[v]) {
            const int64_t lo = A.in_off[v], hi = A.in_off[v + 1];
            p.push_ops = hi - lo;
            if (hi - lo <= 32) {   // longer rows: k_part_settle_big
                const double acc = row_sum_thread<false, 0>(A.in_src, lo, hi, Src{x_full, x_full, 0, 0});
                A.reserved[v] = __dadd_rn(A.h[v], acc);
                A.h[v] = 0.0;
            }
        }
        const double hv = A.h[v];
        const bool above = hv > A.xi, scan = !A.dang[v];
        p.l1 = hv;
        if (above) {
            p.above = hv;
            if (scan) p.nd_above = hv;
        } else {
            p.conv_all = 1;
            if (scan) p.conv_scan = 1;
        }
    }
    block_reduce(p);
    if (threadIdx.x == 0) A.partials[blockIdx.x] = p;
}

__global__ void __launch_bounds__(256) k_part_total(PartArgs A, int include_h) {
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    Partial p;
    zero(p);
    if (v < A.owned) p.l1 = include_h ? A.reserved[v] + A.h[v] : A.reserved[v];
    block_reduce(p);
    if (threadIdx.x == 0) A.partials[blockIdx.x] = p;
}

// one block: fixed-order reduction of the block partials; optionally the 9
// statistics as doubles for a device all-reduce, and the unit counter reset
__global__ void k_part_reduce(const Partial *partials, int64_t blocks, Partial *out, double *out9,
                              unsigned long long *unit_ctr, int nctr = 1) {
    Partial acc;
    zero(acc);
    for (int64_t b = threadIdx.x; b < blocks; b += blockDim.x) add(acc, partials[b]);
    block_reduce(acc);
    if (threadIdx.x == 0) {
        *out = acc;
        if (out9) {
            out9[0] = acc.l1;
            out9[1] = acc.above;
            out9[2] = acc.nd_above;
            out9[3] = (double)acc.nact;
            out9[4] = (double)acc.work;
            out9[5] = (double)acc.push_ops;
            out9[6] = (double)acc.push_dang;
            out9[7] = (double)acc.conv_all;
            out9[8] = (double)acc.conv_scan;
        }
        if (unit_ctr)
            for (int k = 0; k < nctr; ++k) unit_ctr[k] = 0;
    }
}

static PartArgs args_of(Part &P) {
    PartArgs A;
    A.owned = P.owned;
    A.in_off = P.in_off.as<int64_t>();
    A.in_src = P.in_src.as<int32_t>();
    A.deg = P.deg.as<int32_t>();
    A.row_len = P.row_len.as<int32_t>();
    A.dtc = P.dtc.as<int32_t>();
    A.dang = P.dang.as<uint8_t>();
    A.recv = P.recv.as<uint8_t>();
    A.dmask = P.dmask.ptr ? P.dmask.as<uint8_t>() : nullptr;
    A.h = P.h.as<double>();
    A.reserved = P.reserved.as<double>();
    A.act = P.act.as<uint8_t>();
    A.partials = P.partials.as<Partial>();
    A.c = P.c;
    A.xi = P.xi;
    return A;
}

static int finish_stats(Part &P, unsigned blocks, int64_t *ints, double *floats) {
    cudaStream_t st = P.ctx->stream;
    k_part_reduce<<<1, 256, 0, st>>>(P.partials.as<Partial>(), blocks, P.stats.as<Partial>(), nullptr, P.unit_ctr);
    Partial h;
    PR_CUDA(cudaMemcpyAsync(&h, P.stats.ptr, sizeof(h), cudaMemcpyDeviceToHost, st));
    PR_CUDA(cudaStreamSynchronize(st));
    PR_CUDA(cudaGetLastError());
    if (ints) {
        ints[0] = h.nact;
        ints[1] = h.work;
        ints[2] = h.push_ops;
        ints[3] = h.push_dang;
        ints[4] = h.conv_all;
        ints[5] = h.conv_scan;
    }
    if (floats) {
        floats[0] = h.l1;
        floats[1] = h.above;
        floats[2] = h.nd_above;
    }
    return PR_OK;
}

template <class T>
static int upload_as(Ctx &ctx, DevBuf &dst, const int64_t *src, int64_t count) {
    if constexpr (std::is_same<T, int32_t>::value) {
        // host-thread narrowing into page-locked staging (hostio.cu)
        PR_TRY(ensure(dst, 4 * (count > 0 ? count : 1)));
        PR_TRY(upload_narrow(ctx, src, count, dst.as<int32_t>(), nullptr));
        PR_CUDA(cudaStreamSynchronize(ctx.stream));
        return PR_OK;
    }
    std::vector<T> tmp((size_t)(count > 0 ? count : 1));
    for (int64_t i = 0; i < count; ++i) tmp[(size_t)i] = (T)src[i];
    PR_TRY(ensure(dst, sizeof(T) * (count > 0 ? count : 1)));
    if (count) PR_CUDA(cudaMemcpyAsync(dst.ptr, tmp.data(), sizeof(T) * count, cudaMemcpyHostToDevice, ctx.stream));
    PR_CUDA(cudaStreamSynchronize(ctx.stream));
    return PR_OK;
}

int part_create(Ctx &ctx, int64_t owned, int64_t slot, const int64_t *in_off, const int64_t *in_src, int64_t edges,
                const int64_t *deg, const int64_t *row_len, const int64_t *dtc, const uint8_t *dang,
                const uint8_t *recv, int algorithm, double c, double xi, Part **out) {
    if (owned < 0 || slot < owned) return fail(PR_ERR_ARG, "partition: need 0 <= owned <= slot");
    if (!(c > 0.0 && c < 1.0)) return fail(PR_ERR_ARG, "damping must be in (0,1)");
    if (!(xi > 0.0)) return fail(PR_ERR_ARG, "threshold must be positive");
    Part *P = new Part();
    P->ctx = &ctx;
    P->owned = owned;
    P->slot = slot;
    P->edges = edges;
    P->algorithm = algorithm;
    P->c = c;
    P->xi = xi;
    int rc = PR_OK;
    do {
        if ((rc = ensure(P->in_off, 8 * (owned + 1)))) break;
        if (cudaMemcpyAsync(P->in_off.ptr, in_off, 8 * (owned + 1), cudaMemcpyHostToDevice, ctx.stream) != cudaSuccess) {
            rc = fail(PR_ERR_CUDA, "partition upload");
            break;
        }
        if ((rc = upload_as<int32_t>(ctx, P->in_src, in_src, edges))) break;
        if ((rc = upload_as<int32_t>(ctx, P->deg, deg, owned))) break;
        if ((rc = upload_as<int32_t>(ctx, P->row_len, row_len, owned))) break;
        if ((rc = upload_as<int32_t>(ctx, P->dtc, dtc, owned))) break;
        if ((rc = ensure(P->dang, owned ? owned : 1))) break;
        if ((rc = ensure(P->recv, owned ? owned : 1))) break;
        if (owned) {
            cudaMemcpyAsync(P->dang.ptr, dang, owned, cudaMemcpyHostToDevice, ctx.stream);
            cudaMemcpyAsync(P->recv.ptr, recv, owned, cudaMemcpyHostToDevice, ctx.stream);
        }
        if ((rc = ensure(P->h, 8 * (owned ? owned : 1)))) break;
        if ((rc = ensure(P->reserved, 8 * (owned ? owned : 1)))) break;
        if ((rc = ensure(P->act, owned ? owned : 1))) break;
        if ((rc = ensure(P->partials, sizeof(Partial) * (grid_for(owned, 256) +
                                                         (int64_t)ctx.sm_count * 4 * (PR_MAX_SECTIONS + 1) + 1))))
            break;
        if ((rc = ensure(P->stats, sizeof(Partial) + 32 + 8 * PR_MAX_SECTIONS + 16))) break;
        if ((rc = ensure(P->cst, sizeof(Partial)))) break;
        P->unit_ctr = (unsigned long long *)(P->stats.as<char>() + sizeof(Partial) + 32);
        P->done = (unsigned *)(P->unit_ctr + PR_MAX_SECTIONS);
        cudaMemsetAsync(P->unit_ctr, 0, 8 * PR_MAX_SECTIONS + 16, ctx.stream);
        if (cudaStreamSynchronize(ctx.stream) != cudaSuccess) rc = fail(PR_ERR_CUDA, "partition upload");
    } while (0);
    if (rc) { delete P; return rc; }
    *out = P;
    return PR_OK;
}

// ---------------------------------------------------------------- partitions built on the device
// A rank's partition of a device graph's run layout (graph.cu
// ensure_run_layout), without host arrays: the same content as
// distributed.partition_graph(g, parts, rank, order=run_order(...)) -- the
// bounds bit-identical (edge_balanced_ranges), each row's sources the same
// set in the run layout's row order (the fast local step's schedule does not
// depend on it).

// per-row weight of a receiving vertex, in edge units (distributed.ROW_COST reads the same variable)
static int64_t part_row_cost() {
    const char *e = getenv("PUSHRANK_PART_ROW_COST");
    const int64_t v = e && *e ? atoll(e) : PART_ROW_COST;
    return v > 0 ? v : PART_ROW_COST;
}

// w[v] = in_degree(v) + ROW_COST for the vertices a round gathers into
// (in-degree > 0; IFP2: and out-degree > 0), 0 for the others, which are
// drained in rounds 0-1 only (distributed.receiving_rows); w[n] = 0
// (exclusive scan -> cum[0..n])
__global__ void k_part_weights(const int64_t *__restrict__ in_off, const int32_t *__restrict__ out_deg, int ifp2,
                               int64_t row_cost, int64_t n, int64_t *__restrict__ w) {
    GRID_STRIDE(v, n + 1) {
        int64_t x = 0;
        if (v < n) {
            const int64_t d = in_off[v + 1] - in_off[v];
            if (d > 0 && (!ifp2 || out_deg[v] > 0)) x = d + row_cost;
        }
        w[v] = x;
    }
}

// b[k] = first v with cum[v] >= floor(cum[n] * k / parts) (np.searchsorted
// side="left"), b[0] = 0, b[parts] = n, then a running maximum
__global__ void k_part_bounds(const int64_t *__restrict__ cum, int64_t n, int parts, int64_t *__restrict__ b) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int64_t prev = 0;
    for (int k = 0; k <= parts; ++k) {
        int64_t x;
        if (k == 0) x = 0;
        else if (k == parts) x = n;
        else {
            const int64_t target = (int64_t)((__int128)cum[n] * k / parts);
            int64_t lo = 0, hi = n + 1;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (cum[mid] >= target) hi = mid;
                else lo = mid + 1;
            }
            x = lo;
        }
        prev = x > prev ? x : prev;
        b[k] = prev;
    }
}

struct PadMap {
    int64_t b[PR_MAX_PEERS + 1];
    int parts;
    int64_t slot;
    __device__ __forceinline__ int32_t operator()(int32_t u) const {
        int r = 0;
        while (r + 1 < parts && u >= b[r + 1]) ++r;
        return (int32_t)(r * slot + (u - b[r]));
    }
};

__global__ void k_part_rows(const int64_t *__restrict__ in_off, int64_t lo, int64_t owned, int64_t *__restrict__ out) {
    GRID_STRIDE(i, owned + 1) out[i] = in_off[lo + i] - in_off[lo];
}

__global__ void k_part_sources(const int32_t *__restrict__ in_src, int64_t e0, int64_t edges, PadMap map,
                               int32_t *__restrict__ out) {
    GRID_STRIDE(e, edges) out[e] = map(in_src[e0 + e]);
}

__global__ void k_part_vertex(const int32_t *__restrict__ out_deg, const int32_t *__restrict__ dtc, int64_t lo,
                              int64_t owned, int ifp2, int32_t *__restrict__ deg, int32_t *__restrict__ row_len,
                              int32_t *__restrict__ pdtc, uint8_t *__restrict__ dang, uint8_t *__restrict__ recv) {
    GRID_STRIDE(i, owned) {
        const int32_t d = out_deg[lo + i], t = dtc ? dtc[lo + i] : 0;
        deg[i] = d;
        row_len[i] = ifp2 ? d - t : d;           // live degree (graph.py:353-356) / out-degree
        pdtc[i] = ifp2 ? 0 : t;
        dang[i] = d == 0;
        recv[i] = ifp2 ? d > 0 : 1;
    }
}

// dmask[u - lo] |= 1 << rank(t) for every edge u -> t with u owned (one pass
// over the run layout's CSC: row t, source u)
__global__ void k_part_dmask(const int64_t *__restrict__ in_off, const int32_t *__restrict__ in_src, int64_t n,
                             int64_t m, PadMap map, int64_t lo, int64_t hi, unsigned *__restrict__ mask32) {
    // edge-parallel (hub rows hold up to ~1e6 edges): an edge whose source
    // is owned finds its row -- and so the target's rank -- by binary search
    GRID_STRIDE(e, m) {
        const int64_t u = in_src[e];
        if (u < lo || u >= hi) continue;
        int64_t a = 0, b = n;   // last row t with in_off[t] <= e
        while (b - a > 1) {
            const int64_t mid = (a + b) >> 1;
            if (in_off[mid] <= e) a = mid;
            else b = mid;
        }
        int r = 0;
        while (r + 1 < map.parts && a >= map.b[r + 1]) ++r;
        atomicOr(&mask32[u - lo], 1u << r);
    }
}

__global__ void k_part_mask8(const unsigned *__restrict__ m32, int64_t owned, uint8_t *__restrict__ m8,
                             unsigned long long *__restrict__ pop) {
    GRID_STRIDE(i, owned) {
        m8[i] = (uint8_t)m32[i];
        atomicAdd(pop, (unsigned long long)__popc(m32[i]));
    }
}

int part_from_graph(Graph &g_in, int parts, int rank, int algorithm, double c, double xi, int64_t *bounds_out,
                    Part **out) {
    if (parts < 1 || parts > PR_MAX_PEERS || rank < 0 || rank >= parts)
        return fail(PR_ERR_ARG, "partition: need 1 <= parts <= " + std::to_string(PR_MAX_PEERS) +
                                    " and 0 <= rank < parts");
    if (algorithm != PR_ALGO_IFP1 && algorithm != PR_ALGO_IFP2)
        return fail(PR_ERR_ARG, "partition: algorithm must be ifp1 or ifp2");
    if (!(c > 0.0 && c < 1.0)) return fail(PR_ERR_ARG, "damping must be in (0,1)");
    if (!(xi > 0.0)) return fail(PR_ERR_ARG, "threshold must be positive");
    PR_TRY(ensure_run_layout(g_in));
    Graph &r = *g_in.run;
    Ctx &ctx = *r.ctx;
    cudaStream_t st = ctx.stream;
    const int64_t n = r.n;
    PR_TRY(ensure_dtc(r));
    int64_t b[PR_MAX_PEERS + 1];
    {
        DevBuf w, cum, db;
        PR_TRY(ensure(w, 8 * (n + 1)));
        PR_TRY(ensure(cum, 8 * (n + 1)));
        PR_TRY(ensure(db, 8 * (PR_MAX_PEERS + 1)));
        k_part_weights<<<grid_for(n + 1, 256) > 4096 ? 4096 : grid_for(n + 1, 256), 256, 0, st>>>(
            r.in_off.as<int64_t>(), r.out_deg.as<int32_t>(), algorithm == PR_ALGO_IFP2 ? 1 : 0, part_row_cost(), n,
            w.as<int64_t>());
        PR_TRY(cub_run(ctx, [&](void *t, size_t &bytes) {
            return cub::DeviceScan::ExclusiveSum(t, bytes, w.as<int64_t>(), cum.as<int64_t>(), (int)(n + 1), st);
        }));
        k_part_bounds<<<1, 32, 0, st>>>(cum.as<int64_t>(), n, parts, db.as<int64_t>());
        PR_CUDA(cudaMemcpyAsync(b, db.ptr, 8 * (parts + 1), cudaMemcpyDeviceToHost, st));
        PR_CUDA(cudaStreamSynchronize(st));
    }
    int64_t slot = 1;
    for (int k = 0; k < parts; ++k) slot = b[k + 1] - b[k] > slot ? b[k + 1] - b[k] : slot;
    const int64_t lo = b[rank], hi = b[rank + 1], owned = hi - lo;
    int64_t e_lo = 0, e_hi = 0;
    PR_CUDA(cudaMemcpyAsync(&e_lo, r.in_off.as<int64_t>() + lo, 8, cudaMemcpyDeviceToHost, st));
    PR_CUDA(cudaMemcpyAsync(&e_hi, r.in_off.as<int64_t>() + hi, 8, cudaMemcpyDeviceToHost, st));
    PR_CUDA(cudaStreamSynchronize(st));
    const int64_t edges = e_hi - e_lo;
    Part *P = new Part();
    P->ctx = &ctx;
    P->owned = owned;
    P->slot = slot;
    P->edges = edges;
    P->algorithm = algorithm;
    P->c = c;
    P->xi = xi;
    int rc = PR_OK;
    do {
        const int64_t k1 = owned ? owned : 1;
        if ((rc = ensure(P->in_off, 8 * (owned + 1)))) break;
        if ((rc = ensure(P->in_src, 4 * (edges ? edges : 1)))) break;
        if ((rc = ensure(P->deg, 4 * k1)) || (rc = ensure(P->row_len, 4 * k1)) || (rc = ensure(P->dtc, 4 * k1)) ||
            (rc = ensure(P->dang, k1)) || (rc = ensure(P->recv, k1)))
            break;
        const unsigned gv = grid_for(owned + 1, 256) > 4096 ? 4096 : grid_for(owned + 1, 256);
        k_part_rows<<<gv, 256, 0, st>>>(r.in_off.as<int64_t>(), lo, owned, P->in_off.as<int64_t>());
        PadMap map;
        for (int k = 0; k <= PR_MAX_PEERS; ++k) map.b[k] = k <= parts ? b[k] : n;
        map.parts = parts;
        map.slot = slot;
        if (edges)
            k_part_sources<<<grid_for(edges, 256) > 65535 ? 65535 : grid_for(edges, 256), 256, 0, st>>>(
                r.in_src.as<int32_t>(), e_lo, edges, map, P->in_src.as<int32_t>());
        if (owned)
            k_part_vertex<<<gv, 256, 0, st>>>(r.out_deg.as<int32_t>(), r.dtc.as<int32_t>(), lo, owned,
                                              algorithm == PR_ALGO_IFP2, P->deg.as<int32_t>(),
                                              P->row_len.as<int32_t>(), P->dtc.as<int32_t>(), P->dang.as<uint8_t>(),
                                              P->recv.as<uint8_t>());
        // sparse boundary exchange: each vertex's share
        // goes only to the ranks that read it (PUSHRANK_SPARSE_EXCHANGE=0: all)
        const char *se = getenv("PUSHRANK_SPARSE_EXCHANGE");
        if (parts > 1 && !(se && atoi(se) == 0) && owned) {
            DevBuf m32, pop;
            if ((rc = ensure(m32, 4 * owned)) || (rc = ensure(pop, 8)) || (rc = ensure(P->dmask, owned))) break;
            cudaMemsetAsync(m32.ptr, 0, 4 * owned, st);
            cudaMemsetAsync(pop.ptr, 0, 8, st);
            k_part_dmask<<<grid_for(r.m, 256) > 65535 ? 65535 : grid_for(r.m, 256), 256, 0, st>>>(
                r.in_off.as<int64_t>(), r.in_src.as<int32_t>(), n, r.m, map, lo, hi, m32.as<unsigned>());
            k_part_mask8<<<gv, 256, 0, st>>>(m32.as<unsigned>(), owned, P->dmask.as<uint8_t>(),
                                             pop.as<unsigned long long>());
            unsigned long long np = 0;
            cudaMemcpyAsync(&np, pop.ptr, 8, cudaMemcpyDeviceToHost, st);
            if (cudaStreamSynchronize(st) != cudaSuccess) { rc = fail(PR_ERR_CUDA, "partition exchange mask"); break; }
            P->exch_entries = (int64_t)np;
        }
        if ((rc = ensure(P->h, 8 * k1)) || (rc = ensure(P->reserved, 8 * k1)) || (rc = ensure(P->act, k1))) break;
        if ((rc = ensure(P->partials, sizeof(Partial) * (grid_for(owned, 256) +
                                                         (int64_t)ctx.sm_count * 4 * (PR_MAX_SECTIONS + 1) + 1))))
            break;
        if ((rc = ensure(P->stats, sizeof(Partial) + 32 + 8 * PR_MAX_SECTIONS + 16))) break;
        if ((rc = ensure(P->cst, sizeof(Partial)))) break;
        P->unit_ctr = (unsigned long long *)(P->stats.as<char>() + sizeof(Partial) + 32);
        P->done = (unsigned *)(P->unit_ctr + PR_MAX_SECTIONS);
        cudaMemsetAsync(P->unit_ctr, 0, 8 * PR_MAX_SECTIONS + 16, st);
        if (cudaStreamSynchronize(st) != cudaSuccess || cudaGetLastError() != cudaSuccess)
            rc = fail(PR_ERR_CUDA, "partition build");
    } while (0);
    if (rc) {
        delete P;
        return rc;
    }
    P->parts = parts;
    P->rank = rank;
    if (bounds_out)
        for (int k = 0; k <= parts; ++k) bounds_out[k] = b[k];
    *out = P;
    return PR_OK;
}

__global__ void k_part_widen(const int32_t *__restrict__ a, int64_t count, int64_t *__restrict__ out) {
    GRID_STRIDE(i, count) out[i] = a[i];
}

// the partition's rows as host arrays in partition_graph's layout (int64
// offsets / padded sources / degrees, uint8 flags); any pointer may be NULL
int part_export_rows(Part &P, int64_t *in_off, int64_t *in_src, int64_t *deg, int64_t *row_len, int64_t *dtc,
                     uint8_t *dang, uint8_t *recv) {
    Ctx &ctx = *P.ctx;
    cudaStream_t st = ctx.stream;
    const int64_t k = P.owned, m = P.edges;
    DevBuf wide;
    PR_TRY(ensure(wide, 8 * ((m > k ? m : k) + 1)));
    if (in_off) PR_CUDA(cudaMemcpyAsync(in_off, P.in_off.ptr, 8 * (k + 1), cudaMemcpyDeviceToHost, st));
    auto widen = [&](const DevBuf &src, int64_t count, int64_t *dst) -> int {
        if (!dst || !count) return PR_OK;
        k_part_widen<<<grid_for(count, 256) > 65535 ? 65535 : grid_for(count, 256), 256, 0, st>>>(src.as<int32_t>(), count,
                                                                                         wide.as<int64_t>());
        PR_CUDA(cudaMemcpyAsync(dst, wide.ptr, 8 * count, cudaMemcpyDeviceToHost, st));
        PR_CUDA(cudaStreamSynchronize(st));
        return PR_OK;
    };
    PR_TRY(widen(P.in_src, m, in_src));
    PR_TRY(widen(P.deg, k, deg));
    PR_TRY(widen(P.row_len, k, row_len));
    PR_TRY(widen(P.dtc, k, dtc));
    if (dang && k) PR_CUDA(cudaMemcpyAsync(dang, P.dang.ptr, k, cudaMemcpyDeviceToHost, st));
    if (recv && k) PR_CUDA(cudaMemcpyAsync(recv, P.recv.ptr, k, cudaMemcpyDeviceToHost, st));
    PR_CUDA(cudaStreamSynchronize(st));
    return PR_OK;
}

int part_exchange_entries(Part &P, int64_t *entries) {
    *entries = P.exch_entries >= 0 ? P.exch_entries : (int64_t)P.owned * (P.parts > 0 ? P.parts : 1);
    return PR_OK;
}

int part_sizes(Part &P, int64_t *owned, int64_t *slot, int64_t *edges) {
    if (owned) *owned = P.owned;
    if (slot) *slot = P.slot;
    if (edges) *edges = P.edges;
    return PR_OK;
}

__global__ void k_ids_identity(const int32_t *ids, int64_t count, unsigned long long *bad) {
    GRID_STRIDE(i, count) if (ids[i] != (int32_t)i) atomicAdd(bad, 1ull);
}

// IFP1 partitions: the schedule interleaves class-0 rows (in > 0, out > 0)
// with dangling receivers by degree.  In a run-layout partition the class-0
// vertices are the local ids [0, c0), and the stable degree sort keeps them
// in id order, so the sources of sections before k are the local ids below
// the first class-0 id at or after row sec_row[k] (as the engine's IFP1
// sections, rounds.cu).  Both properties are checked; on failure the caller
// keeps one section.
__global__ void k_part_c0(const int64_t *in_off, const int32_t *deg, int64_t owned, unsigned long long *cnt) {
    GRID_STRIDE(v, owned) if (deg[v] > 0 && in_off[v + 1] > in_off[v]) atomicAdd(cnt, 1ull);
}

__global__ void k_part_c0_check(const int64_t *in_off, const int32_t *deg, int64_t owned, int64_t c0,
                                const int32_t *ids, int64_t count, int32_t *pos, unsigned long long *bad, int phase) {
    if (phase == 0) {
        GRID_STRIDE(v, owned) {
            const bool c = deg[v] > 0 && in_off[v + 1] > in_off[v];
            if (c != (v < c0)) atomicAdd(bad, 1ull);
        }
        GRID_STRIDE(r, count) if (ids[r] < c0) pos[ids[r]] = (int32_t)r;
    } else {
        GRID_STRIDE(r, count) {
            const int32_t v = ids[r];
            if (v < c0 && v + 1 < c0 && pos[v + 1] <= (int32_t)r) atomicAdd(bad, 1ull);
        }
    }
}

__global__ void k_part_sec_id(const int32_t *ids, int64_t count, int64_t c0, const int64_t *bounds, int nsec,
                              int64_t *out) {
    const int k = threadIdx.x;
    if (k > nsec) return;
    int64_t r = bounds[k];
    while (r < count && ids[r] >= c0) ++r;
    out[k] = r < count ? ids[r] : c0;
}

static int part_sections_by_id(Part &P, Graph &g) {
    Ctx &ctx = *P.ctx;
    cudaStream_t st = ctx.stream;
    auto &S = g.sched[P.which];
    DevBuf cnt, pos, bnd, out;
    PR_TRY(ensure(cnt, 16));
    PR_TRY(ensure(pos, 4 * (P.owned > 0 ? P.owned : 1)));
    PR_TRY(ensure(bnd, 8 * (PR_MAX_SECTIONS + 1)));
    PR_TRY(ensure(out, 8 * (PR_MAX_SECTIONS + 1)));
    PR_CUDA(cudaMemsetAsync(cnt.ptr, 0, 16, st));
    const unsigned gr = grid_for(P.owned > S.count ? P.owned : S.count, 256) > 4096
                            ? 4096 : grid_for(P.owned > S.count ? P.owned : S.count, 256);
    unsigned long long *c = cnt.as<unsigned long long>();
    if (P.owned) k_part_c0<<<gr, 256, 0, st>>>(P.in_off.as<int64_t>(), P.deg.as<int32_t>(), P.owned, c);
    unsigned long long c0 = 0;
    PR_CUDA(cudaMemcpyAsync(&c0, c, 8, cudaMemcpyDeviceToHost, st));
    PR_CUDA(cudaStreamSynchronize(st));
    for (int phase = 0; phase < 2; ++phase)
        k_part_c0_check<<<gr, 256, 0, st>>>(P.in_off.as<int64_t>(), P.deg.as<int32_t>(), P.owned, (int64_t)c0,
                                            S.ids.as<int32_t>(), S.count, pos.as<int32_t>(), c + 1, phase);
    PR_CUDA(cudaMemcpyAsync(bnd.ptr, S.sec_row, 8 * (S.nsec + 1), cudaMemcpyHostToDevice, st));
    k_part_sec_id<<<1, 32, 0, st>>>(S.ids.as<int32_t>(), S.count, (int64_t)c0, bnd.as<int64_t>(), S.nsec,
                                    out.as<int64_t>());
    unsigned long long nbad = 0;
    PR_CUDA(cudaMemcpyAsync(&nbad, c + 1, 8, cudaMemcpyDeviceToHost, st));
    PR_CUDA(cudaMemcpyAsync(P.sec_id, out.ptr, 8 * (S.nsec + 1), cudaMemcpyDeviceToHost, st));
    PR_CUDA(cudaStreamSynchronize(st));
    PR_CUDA(cudaGetLastError());
    if (nbad) return fail(PR_ERR_STATE, "partition: class-0 rows out of id order");
    return PR_OK;
}

// the fast form's pull schedule, built on first use
static int ensure_part_sched(Part &P) {
    if (P.sg) return PR_OK;
    Ctx &ctx = *P.ctx;
    cudaStream_t st = ctx.stream;
    Graph *g = new Graph();
    g->ctx = &ctx;
    g->n = P.owned;
    g->m = P.edges;
    int rc = PR_OK;
    do {
        if ((rc = ensure(g->in_off, 8 * (P.owned + 1)))) break;
        if ((rc = ensure(g->in_src, 4 * (P.edges > 0 ? P.edges : 1)))) break;
        if ((rc = ensure(g->out_deg, 4 * (P.owned > 0 ? P.owned : 1)))) break;
        cudaMemcpyAsync(g->in_off.ptr, P.in_off.ptr, 8 * (P.owned + 1), cudaMemcpyDeviceToDevice, st);
        if (P.edges) cudaMemcpyAsync(g->in_src.ptr, P.in_src.ptr, 4 * P.edges, cudaMemcpyDeviceToDevice, st);
        if (P.owned) cudaMemcpyAsync(g->out_deg.ptr, P.deg.ptr, 4 * P.owned, cudaMemcpyDeviceToDevice, st);
        // rows' sources ascending on HBM-bound partitions, as the engine's run
        // layout (graph.cu): past 16x L2 of round working set
        {
            const double l2b = (double)(ctx.l2_bytes ? ctx.l2_bytes : (size_t)126 << 20);
            bool sort_rows = 4.0 * (double)P.edges + 8.0 * (double)P.slot > 16.0 * l2b;
            if (const char *e = getenv("PUSHRANK_SORT_ROWS")) sort_rows = atoi(e) != 0;
            if (sort_rows && (rc = sort_csc_rows(ctx, g->in_off, g->in_src, P.owned, P.edges))) break;
        }
        // IFP2 pulls into non-dangling rows only (receives = !dangling), IFP1 into all
        P.which = P.algorithm == PR_ALGO_IFP2 ? 1 : 0;
        if ((rc = ensure_sched(*g, P.which))) break;
        // the same working-set rules as the engine's k_pull (rounds.cu)
        // (44 B per scheduled row, as there: the owned vertices outside the schedule are not swept)
        const double ws = 4.0 * (double)g->sched[P.which].edges + 8.0 * (double)P.slot +
                          44.0 * (double)g->sched[P.which].count;
        const double l2 = (double)(ctx.l2_bytes ? ctx.l2_bytes : (size_t)126 << 20);
        P.stream_csc = ws > 0.6 * l2;
        P.prefetch = ws < 4.0 * l2;
        P.blocks = (int64_t)ctx.sm_count * (P.prefetch ? 3 : PR_PART_BLOCKS);
        // rank-local Gauss-Seidel sections, as the engine chooses them
        // (rounds.cu): IFP2 on rows that are the local ids in order (a
        // run-layout partition), 2 past 1.5x L2 of round working set, 4 past 16x
        P.nsec = gs_sections_default(ws, l2);
        if (const char *e = getenv("PUSHRANK_GS_SECTIONS")) P.nsec = atoi(e);
        if (P.nsec < 1) P.nsec = 1;
        if (P.nsec > PR_MAX_SECTIONS) P.nsec = PR_MAX_SECTIONS;
        auto &Sc = g->sched[P.which];
        if (P.nsec > 1 && P.which == 1) {
            // IFP2: the rows must be the local ids in order
            DevBuf bad;
            if ((rc = ensure(bad, 8))) break;
            cudaMemsetAsync(bad.ptr, 0, 8, st);
            if (Sc.count) k_ids_identity<<<grid_for(Sc.count, 256), 256, 0, st>>>(Sc.ids.as<int32_t>(), Sc.count,
                                                                                bad.as<unsigned long long>());
            unsigned long long nbad = 0;
            cudaMemcpyAsync(&nbad, bad.ptr, 8, cudaMemcpyDeviceToHost, st);
            cudaStreamSynchronize(st);
            if (nbad) P.nsec = 1;
        }
        if ((rc = ensure_units(*g, P.which, P.blocks, P.nsec))) break;
        for (int k = 0; k <= PR_MAX_SECTIONS; ++k) P.sec_id[k] = k <= Sc.nsec ? Sc.sec_row[k] : Sc.count;
        if (P.nsec > 1 && P.which == 0 && part_sections_by_id(P, *g) != PR_OK) {
            P.nsec = 1;
            if ((rc = ensure_units(*g, P.which, P.blocks, 1))) break;
        }
        // owned vertices outside the schedule: no inflow, drained alone
        {
            DevBuf cnt;
            if ((rc = ensure(cnt, 8))) break;
            if ((rc = ensure(P.outside, 4 * (P.owned > 0 ? P.owned : 1)))) break;
            auto first = thrust::make_counting_iterator<int32_t>(0);
            OutsideRow pred{P.in_off.as<int64_t>(), P.recv.as<uint8_t>()};
            if ((rc = cub_run(ctx, [&](void *t, size_t &b) {
                     return cub::DeviceSelect::If(t, b, first, P.outside.as<int32_t>(), cnt.as<int64_t>(),
                                                  (int)P.owned, pred, st);
                 })))
                break;
            cudaMemcpyAsync(&P.n_outside, cnt.ptr, 8, cudaMemcpyDeviceToHost, st);
        }
        if (cudaStreamSynchronize(st) != cudaSuccess) rc = fail(PR_ERR_CUDA, "partition schedule");
    } while (0);
    if (rc) {
        delete g;
        return rc;
    }
    P.sg = g;
    return PR_OK;
}

static BinView part_view(Part &P) {
    auto &S = P.sg->sched[P.which];
    BinView T;
    T.ids = S.ids.as<int32_t>();
    T.doff = S.doff.as<int64_t>();
    T.csc = S.csc.as<int32_t>();
    T.sell_off = S.sell_off.as<int64_t>();
    T.count = S.count;
    T.n_hub = S.n_hub;
    T.n_warp = S.n_warp;
    T.chunk_base = S.chunk_base.as<int64_t>();
    T.units = S.units.as<int2>();
    T.n_units = S.n_units;
    T.row_cnt = S.row_cnt.as<int32_t>();
    T.chunk_part = S.chunk_part.as<double>();
    T.unit_ctr = P.unit_ctr;
    return T;
}

// one round: a launch per section; x = shares of the previous round (all
// ranks), x_new = this round's full vector (own slot written by the earlier
// sections); kind 0 Jacobi / 1 transition / 2 GS (ignored without sections)
static void launch_part_pull(Part &P, const double *s_full, const double *x_new, int kind, const ShareOut &so,
                             double *out9) {
    cudaStream_t st = P.ctx->stream;
    const unsigned g = (unsigned)P.blocks;
    const int32_t *out = P.outside.as<int32_t>();
    const int64_t no = P.n_outside;
    auto &Sc = P.sg->sched[P.which];
    const int nsec = P.nsec > 1 ? P.nsec : 1;
    for (int k = 0; k < nsec; ++k) {
        PullSec S;
        S.u_lo = nsec > 1 ? Sc.sec_unit[k] : 0;
        S.u_hi = nsec > 1 ? Sc.sec_unit[k + 1] : Sc.n_units;
        S.kind = nsec > 1 ? kind : 0;
        S.src = Src{s_full, x_new, S.kind ? (int)P.sec_id[k] : 0, (int)((int64_t)P.rank * P.slot)};
        S.last = k == nsec - 1;
        S.region = k;
        S.done = P.done;
        S.stats = P.stats.as<Partial>();
        S.out9 = out9;
        S.ctr = P.unit_ctr;
        S.prev9 = P.prev9;
        S.round_kind = kind;
        S.cst = P.cst.as<Partial>();
        BinView T = part_view(P);
        T.unit_ctr = P.unit_ctr + k;
        if (P.stream_csc) {
            if (P.prefetch) k_part_pull<true, true><<<g, 256, 0, st>>>(args_of(P), T, out, no, S, so);
            else k_part_pull<true, false><<<g, 256, 0, st>>>(args_of(P), T, out, no, S, so);
        } else {
            if (P.prefetch) k_part_pull<false, true><<<g, 256, 0, st>>>(args_of(P), T, out, no, S, so);
            else k_part_pull<false, false><<<g, 256, 0, st>>>(args_of(P), T, out, no, S, so);
        }
    }
    P.prev9 = nullptr;   // one round only
}

// ---- fused exchange: share replicas in peer memory ----------------------

int part_share_buffers(Part &P, int parts, int rank, void **d_full, void *ipc) {
    if (parts < 1 || parts > PR_MAX_PEERS || rank < 0 || rank >= parts)
        return fail(PR_ERR_ARG, "fused exchange: need 1 <= parts <= 8 and 0 <= rank < parts");
    P.parts = parts;
    P.rank = rank;
    const size_t bytes = 8 * (size_t)P.slot * (size_t)parts;
    for (int k = 0; k < 2; ++k) {
        if (!P.own_full[k]) {
            // plain cudaMalloc: IPC handles need it (pool allocations are not exportable this way)
            PR_CUDA(cudaMalloc(&P.own_full[k], bytes));
            PR_CUDA(cudaMemset(P.own_full[k], 0, bytes));
        }
        d_full[k] = P.own_full[k];
        if (ipc) PR_CUDA(cudaIpcGetMemHandle((cudaIpcMemHandle_t *)ipc + k, P.own_full[k]));
    }
    for (int r = 0; r < PR_MAX_PEERS; ++r) P.peer[0][r] = P.peer[1][r] = nullptr;
    P.peer[0][rank] = (double *)P.own_full[0];
    P.peer[1][rank] = (double *)P.own_full[1];
    P.fused_ready = false;   // until set_peers has mapped the other ranks' replicas
    return PR_OK;
}

int part_set_peers(Part &P, const void *handles) {
    if (!P.own_full[0]) return fail(PR_ERR_STATE, "fused exchange: call pr_part_share_buffers first");
    const cudaIpcMemHandle_t *h = (const cudaIpcMemHandle_t *)handles;
    for (int r = 0; r < P.parts; ++r) {
        if (r == P.rank) continue;
        for (int k = 0; k < 2; ++k) {
            void *ptr = nullptr;
            PR_CUDA(cudaIpcOpenMemHandle(&ptr, h[2 * r + k], cudaIpcMemLazyEnablePeerAccess));
            P.peer[k][r] = (double *)ptr;
            P.opened.push_back(ptr);
        }
    }
    P.fused_ready = true;
    return PR_OK;
}

// launches per fast round (one per Gauss-Seidel section + the statistics
// reduction); builds the schedule if needed
int part_launches_per_round(Part &P, int *out) {
    PR_TRY(ensure_part_sched(P));
    *out = P.nsec > 1 ? P.nsec : 1;   // the last section's launch also reduces the statistics
    return PR_OK;
}

// this partition's place among the ranks (the padded slot it owns: the
// rank-local Gauss-Seidel test and the fused exchange's store offset)
int part_skip_if_done(Part &P, const double *d_prev9) {
    P.prev9 = d_prev9;
    return PR_OK;
}

int part_set_rank(Part &P, int parts, int rank) {
    if (parts < 1 || parts > PR_MAX_PEERS || rank < 0 || rank >= parts)
        return fail(PR_ERR_ARG, "partition: need 1 <= parts <= 8 and 0 <= rank < parts");
    P.parts = parts;
    P.rank = rank;
    return PR_OK;
}

// unmap the other ranks' replicas (before any rank frees its own: the
// caller puts a barrier between this and the destruction)
int part_close_peers(Part &P) {
    cudaStreamSynchronize(P.ctx->stream);
    for (void *p : P.opened) cudaIpcCloseMemHandle(p);
    P.opened.clear();
    for (int r = 0; r < PR_MAX_PEERS; ++r)
        if (r != P.rank) P.peer[0][r] = P.peer[1][r] = nullptr;
    P.fused_ready = false;
    return PR_OK;
}

// same-process emulation (tests): the ranks' replicas are device pointers
int part_set_peer_ptrs(Part &P, int parts, int rank, void *const *ptrs) {
    if (parts < 1 || parts > PR_MAX_PEERS || rank < 0 || rank >= parts)
        return fail(PR_ERR_ARG, "fused exchange: need 1 <= parts <= 8 and 0 <= rank < parts");
    P.parts = parts;
    P.rank = rank;
    for (int r = 0; r < parts; ++r) {
        P.peer[0][r] = (double *)ptrs[2 * r];
        P.peer[1][r] = (double *)ptrs[2 * r + 1];
    }
    P.fused_ready = true;
    for (int r = 0; r < parts; ++r) P.fused_ready = P.fused_ready && P.peer[0][r] && P.peer[1][r];
    return PR_OK;
}

static ShareOut fused_out(Part &P, int parity) {
    ShareOut so;
    memset(&so, 0, sizeof(so));
    so.n = P.parts;
    so.off = (int64_t)P.rank * P.slot;
    for (int r = 0; r < P.parts; ++r) so.peer[r] = P.peer[parity][r];
    return so;
}

int part_init_fused(Part &P, double *d_stats9) {
    if (P.parts < 1 || !P.fused_ready) return fail(PR_ERR_STATE, "fused exchange not set up (or closed)");
    PR_TRY(ensure_part_sched(P));
    cudaStream_t st = P.ctx->stream;
    const unsigned g = grid_for(P.owned, 256);
    k_part_init_fast<<<g, 256, 0, st>>>(args_of(P), fused_out(P, 0));
    k_part_reduce<<<1, 256, 0, st>>>(P.partials.as<Partial>(), g, P.stats.as<Partial>(), d_stats9, P.unit_ctr);
    PR_CUDA(cudaGetLastError());
    return PR_OK;
}

// round reading this rank's replica `parity`, writing every replica 1-parity
int part_round_fused(Part &P, int parity, int kind, double *d_stats9) {
    if (P.parts < 1 || !P.fused_ready) return fail(PR_ERR_STATE, "fused exchange not set up (or closed)");
    PR_TRY(ensure_part_sched(P));
    launch_part_pull(P, P.peer[parity & 1][P.rank], P.peer[1 - (parity & 1)][P.rank], kind,
                     fused_out(P, 1 - (parity & 1)), d_stats9);
    PR_CUDA(cudaGetLastError());
    return PR_OK;
}

int part_init_device(Part &P, double *d_s_mine, double *d_stats9) {
    unsigned g = grid_for(P.owned, 256);
    cudaStream_t st = P.ctx->stream;
    k_part_init<<<g, 256, 0, st>>>(args_of(P), d_s_mine);
    k_part_reduce<<<1, 256, 0, st>>>(P.partials.as<Partial>(), g, P.stats.as<Partial>(), d_stats9, P.unit_ctr);
    PR_CUDA(cudaGetLastError());
    return PR_OK;
}

int part_round_device(Part &P, const double *d_s_full, double *d_s_mine, int fast, int kind, double *d_stats9) {
    cudaStream_t st = P.ctx->stream;
    unsigned g;
    if (fast) {
        PR_TRY(ensure_part_sched(P));
        g = (unsigned)P.blocks;
        ShareOut so;
        memset(&so, 0, sizeof(so));
        so.mine = d_s_mine;
        // d_s_mine is this rank's slot of the next round's full vector
        launch_part_pull(P, d_s_full, d_s_mine - (int64_t)P.rank * P.slot, kind, so, d_stats9);
    } else {
        g = grid_for(P.owned, 256);
        k_part_round<<<g, 256, 0, st>>>(args_of(P), d_s_full, d_s_mine);
        k_part_reduce<<<1, 256, 0, st>>>(P.partials.as<Partial>(), g, P.stats.as<Partial>(), d_stats9, P.unit_ctr,
                                         PR_MAX_SECTIONS);
    }
    PR_CUDA(cudaGetLastError());
    return PR_OK;
}

int part_init(Part &P, double *d_s_mine, int64_t *ints, double *floats) {
    unsigned g = grid_for(P.owned, 256);
    k_part_init<<<g, 256, 0, P.ctx->stream>>>(args_of(P), d_s_mine);
    return finish_stats(P, g, ints, floats);
}

int part_round(Part &P, const double *d_s_full, double *d_s_mine, int64_t *ints, double *floats) {
    unsigned g = grid_for(P.owned, 256);
    k_part_round<<<g, 256, 0, P.ctx->stream>>>(args_of(P), d_s_full, d_s_mine);
    return finish_stats(P, g, ints, floats);
}

int part_settle_shares(Part &P, double *d_x_mine) {
    k_part_shares<<<grid_for(P.owned, 256), 256, 0, P.ctx->stream>>>(args_of(P), d_x_mine);
    PR_CUDA(cudaStreamSynchronize(P.ctx->stream));
    return PR_OK;
}

int part_settle(Part &P, const double *d_x_full, int64_t *settled, int64_t *ints, double *floats) {
    unsigned g = grid_for(P.owned, 256);
    cudaStream_t st = P.ctx->stream;
    if (P.sg) {
        if (P.n_big < 0) {
            DevBuf cnt;
            PR_TRY(ensure(cnt, 8));
            PR_TRY(ensure(P.big_dang, 4 * (P.owned > 0 ? P.owned : 1)));
            auto first = thrust::make_counting_iterator<int32_t>(0);
            PR_TRY(cub_run(*P.ctx, [&](void *t, size_t &b) {
                return cub::DeviceSelect::If(t, b, first, P.big_dang.as<int32_t>(), cnt.as<int64_t>(), (int)P.owned,
                                             BigDang{P.in_off.as<int64_t>(), P.dang.as<uint8_t>()}, st);
            }));
            PR_CUDA(cudaMemcpyAsync(&P.n_big, cnt.ptr, 8, cudaMemcpyDeviceToHost, st));
            PR_CUDA(cudaStreamSynchronize(st));
        }
        if (P.n_big > 0)
            k_part_settle_big<<<grid_for(P.n_big * 32, 256) > 4096 ? 4096 : grid_for(P.n_big * 32, 256), 256, 0, st>>>(
                args_of(P), d_x_full, P.big_dang.as<int32_t>(), P.n_big);
        k_part_settle_fast<<<g, 256, 0, st>>>(args_of(P), d_x_full);
    } else {
        k_part_settle<<<g, 256, 0, st>>>(args_of(P), d_x_full);
    }
    int64_t tmp[6];
    PR_TRY(finish_stats(P, g, tmp, floats));
    if (settled) *settled = tmp[2];
    if (ints) memcpy(ints, tmp, sizeof(tmp));
    return PR_OK;
}

int part_total(Part &P, int include_h, double *total) {
    unsigned g = grid_for(P.owned, 256);
    k_part_total<<<g, 256, 0, P.ctx->stream>>>(args_of(P), include_h);
    double f[3];
    PR_TRY(finish_stats(P, g, nullptr, f));
    *total = f[0];
    return PR_OK;
}

int part_export(Part &P, double *reserved, double *pending) {
    cudaStream_t st = P.ctx->stream;
    if (reserved && P.owned)
        PR_CUDA(cudaMemcpyAsync(reserved, P.reserved.ptr, 8 * P.owned, cudaMemcpyDeviceToHost, st));
    if (pending && P.owned) PR_CUDA(cudaMemcpyAsync(pending, P.h.ptr, 8 * P.owned, cudaMemcpyDeviceToHost, st));
    PR_CUDA(cudaStreamSynchronize(st));
    return PR_OK;
}

void part_destroy(Part *P) {
    if (!P) return;
    cudaStreamSynchronize(P->ctx->stream);
    delete P;
}

Ctx &part_ctx(Part &P) { return *P.ctx; }
void *part_stream(Part &P) { return (void *)P.ctx->stream; }

}  // namespace pr
