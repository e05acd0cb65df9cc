// bins.cuh -- degree-binned CSC gather over the pull schedule (sched.cu).
//
// Rows are sorted by descending in-degree and cut into block work units of
// near-equal cost (edges + ROW_COST * rows); a unit never mixes bins:
//   * hub unit    -- HUB_CHUNK edges of one row with > HUB_DEG edges, summed
//                    HUB_STEP at a time (16 coalesced gathers per thread in
//                    flight) with one block reduction per unit; the last chunk
//                    of a row to arrive adds the chunk sums in chunk order;
//   * warp unit   -- rows with THREAD_DEG < d <= HUB_DEG; warp w takes rows
//                    w, w+8, ...; lanes stride a row with 8 gathers in flight;
//   * thread unit -- rows with d <= THREAD_DEG; thread t takes rows t, t+256,
//                    ... (coalesced drains), 8 index loads then 8 gathers;
//                    the bin is stored SELL-32 (column-major 32-row slices)
//                    so each warp index load is one 128-byte line.
// Rows of a unit have near-equal degree (sorted), so warps carry uniform
// work.  Blocks of a persistent grid claim units dynamically (an atomic per
// unit, issued at the start of the previous one); a launch covers the unit
// range of one Gauss-Seidel section.  Every summation order is fixed by the
// schedule (row sums do not depend on which block claims a unit), so a pull
// round is run-to-run deterministic; the engine's sparse push rounds add with
// atomics (rounds.cu).
#pragma once

#include "internal.cuh"

namespace pr {

// Cache policy of the index stream (compacted CSC, read once per round):
// when a round's working set overflows L2 (C3, C5) it is loaded with
// ld.global.cs (evict-first) so that it does not push the share vector out
// of L2; when everything fits (C1, C2) the CSC stays L2-resident across
// rounds with plain loads.  Measured: C3 -5%, C5 -1%, C2 +4% if streamed.
#ifndef PR_IDXP
#define PR_IDXP 0
#endif
template <bool STREAM>
__device__ __forceinline__ int ld_idx(const int32_t *p) {
    if constexpr (STREAM) {
#if PR_IDXP == 1
        int v;
        asm("{ .reg .b64 pol; createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
            "  ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], pol; }"
            : "=r"(v) : "l"(p));
        return v;
#else
        return __ldcs(p);
#endif
    } else {
        return __ldg(p);
    }
}
// Share gathers (random 8-byte loads; A/B builds): 0 ld.global.nc; 1 without
// L1 allocation; 2 ld.global.cg (L2 only); 3-5 split by source id (hot =
// id < PR_HOT, the run layout's most-gathered sources): 3 hot L1::evict_last,
// cold L1::no_allocate; 4 hot evict_last, cold plain; 5 hot plain, cold
// no_allocate
#ifndef PR_GATHER
#define PR_GATHER 0
#endif
#ifndef PR_HOT
#define PR_HOT 32768
#endif
#define PR_LDSPLIT(A, B)                                                                      \
    asm("{ .reg .pred p; setp.ne.u32 p, %2, 0;\n"                                             \
        "  @p ld.global.nc" A ".f64 %0, [%1];\n"                                               \
        "  @!p ld.global.nc" B ".f64 %0, [%1]; }"                                               \
        : "=d"(v) : "l"(p), "r"((unsigned)hot))
__device__ __forceinline__ double ld_share(const double *p, int idx) {
#if PR_GATHER == 1
    double v;
    asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
#elif PR_GATHER == 2
    return __ldcg(p);
#elif PR_GATHER >= 3
    const bool hot = (unsigned)idx < (unsigned)PR_HOT;
    double v;
#if PR_GATHER == 3
    PR_LDSPLIT(".L1::evict_last", ".L1::no_allocate");
#elif PR_GATHER == 4
    PR_LDSPLIT(".L1::evict_last", "");
#else
    PR_LDSPLIT("", ".L1::no_allocate");
#endif
    return v;
#else
    return __ldg(p);
#endif
}

// Share sources of a dense round (rounds.cu, Gauss-Seidel sections):
//   Jacobi      gs_lo = 0:              x[u]
//   GS sweep    gs_lo = section start:  early(u) ? x_new[u] : x[u]
//   transition                          x[u] + (early(u) ? x_new[u] : 0)
// x holds the shares still owed to this row, x_new the shares drained
// earlier in the same sweep (sources of earlier sections):
// early(u) = base <= u < base + gs_lo, with base = 0 on one GPU and the
// rank's first padded id in a partition (part.cu: sections are rank-local,
// other ranks' sources always read x).
struct Src {
    const double *x, *x_new;
    int gs_lo, base;
};

__device__ __forceinline__ bool early(const Src &S, int idx) { return (unsigned)(idx - S.base) < (unsigned)S.gs_lo; }

// SRC: 0 Jacobi only (plain x), 1 section sweep (select), 2 transition
template <int SRC>
__device__ __forceinline__ double ld_src(const Src S, int idx) {
    if constexpr (SRC == 0) {
        return ld_share(S.x + idx, idx);
    } else if constexpr (SRC == 1) {
        return ld_share((early(S, idx) ? S.x_new : S.x) + idx, idx);
    } else {
        return ld_share(S.x + idx, idx) + (early(S, idx) ? ld_share(S.x_new + idx, idx) : 0.0);
    }
}

struct BinView {
    const int32_t *ids;      // row -> vertex id
    const int64_t *doff;     // row offsets in csc
    const int32_t *csc;      // compacted sources (padded); thread rows in SELL-32 slices
    const int64_t *sell_off; // csc offset of each 32-row slice of the thread bin (sched.cu sell_layout)
    int64_t count, n_hub, n_warp;
    const int64_t *chunk_base;   // first chunk unit of each hub row
    const int2 *units;           // (row_begin, row_end) or hub chunk (row, -(chunk+1))
    int64_t n_units;
    int32_t *row_cnt;
    double *chunk_part;          // per hub chunk unit
    unsigned long long *unit_ctr;  // dynamic dispatch counter (0 at kernel start)
};

template <bool STREAM, int SRC>
__device__ __forceinline__ double row_sum_thread(const int32_t *__restrict__ csc, int64_t lo, int64_t hi,
                                                 const Src x) {
    double acc = 0.0;
    for (int64_t e = lo; e < hi; e += 8) {
        int idx[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) idx[q] = e + q < hi ? ld_idx<STREAM>(&csc[e + q]) : -1;
        double t[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) t[q] = idx[q] >= 0 ? ld_src<SRC>(x, idx[q]) : 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) acc += t[q];
    }
    return acc;
}

// A thread row in its SELL-32 slice: the k-th source at p[32 k].  Same
// summation order as row_sum_thread (ascending position, 8 at a time), so a
// row's sum is bit-identical to the CSR form; the warp's loads of position k
// are one 128-byte line.
template <bool STREAM, int SRC>
__device__ __forceinline__ double row_sum_sell(const int32_t *__restrict__ p, int deg, const Src x) {
    double acc = 0.0;
    for (int k = 0; k < deg; k += 8) {
        int idx[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) idx[q] = k + q < deg ? ld_idx<STREAM>(&p[32 * (k + q)]) : -1;
        double t[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) t[q] = idx[q] >= 0 ? ld_src<SRC>(x, idx[q]) : 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) acc += t[q];
    }
    return acc;
}

// Sum of thread row `row` (rows of a warp are one slice: base aligned to 32
// rows past the bin start t0)
template <bool STREAM, int SRC>
__device__ __forceinline__ double thread_row_sum(const BinView &B, int64_t t0, int64_t row, const Src x) {
#if PR_SELL
    const int64_t i = row - t0;
    const int deg = (int)(B.doff[row + 1] - B.doff[row]);
    return row_sum_sell<STREAM, SRC>(B.csc + B.sell_off[i >> 5] + (i & 31), deg, x);
#else
    return row_sum_thread<STREAM, SRC>(B.csc, B.doff[row], B.doff[row + 1], x);
#endif
}

// lanes stride [lo, hi) with 8 gathers in flight; warp-reduced (fixed tree)
template <bool STREAM, int SRC>
__device__ __forceinline__ double span_sum_warp(const int32_t *__restrict__ csc, int64_t lo, int64_t hi,
                                                const Src x) {
    const int lane = threadIdx.x & 31;
    double acc = 0.0;
    for (int64_t e = lo + lane; e < hi; e += 256) {
        int idx[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) idx[q] = e + 32 * q < hi ? ld_idx<STREAM>(&csc[e + 32 * q]) : -1;
        double t[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) t[q] = idx[q] >= 0 ? ld_src<SRC>(x, idx[q]) : 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) acc += t[q];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    return acc;
}

// Sub-warp rows: warp-bin rows of at most PR_SUB_MAX edges are summed by
// groups of PR_SUB_LANES lanes, 32 / PR_SUB_LANES rows at a time (each lane
// 8 gathers in flight at stride 8 * PR_SUB_LANES); longer rows by the whole
// warp.  PR_SUB_LANES = 32 keeps one row per warp throughout.  16 lanes
// measured C5 -2.6% (-6% with sorted rows), C2 -0.7%, C3 +0.4%, C4 0.
#ifndef PR_SUB_LANES
#define PR_SUB_LANES 16
#endif
#ifndef PR_SUB_MAX
#define PR_SUB_MAX 512
#endif

template <bool STREAM, int SRC, int L>
__device__ __forceinline__ double span_sum_sub(const int32_t *__restrict__ csc, int64_t lo, int64_t hi, const Src x) {
    const int sl = threadIdx.x & (L - 1);
    double acc = 0.0;
    for (int64_t e = lo + sl; e < hi; e += 8 * L) {
        int idx[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) idx[q] = e + L * q < hi ? ld_idx<STREAM>(&csc[e + L * q]) : -1;
        double t[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) t[q] = idx[q] >= 0 ? ld_src<SRC>(x, idx[q]) : 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) acc += t[q];
    }
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    return acc;
}

// Sums of the cnt rows of a warp batch (row j's bounds in lane j's
// my_lo/my_hi, rows in descending degree): lane j returns row j's sum.
// Every lane must call it.  The order of each row's sum is fixed (lane and
// q order, then the shuffle tree), so results stay run-to-run identical.
template <bool STREAM, int SRC>
__device__ __forceinline__ double warp_batch_sums(const BinView &B, const Src x, int64_t my_lo, int64_t my_hi,
                                                  int cnt) {
    const int lane = threadIdx.x & 31;
    double mine = 0.0;
    int j = 0;
    for (; j < cnt; ++j) {
        const int64_t lo = __shfl_sync(0xffffffffu, my_lo, j), hi = __shfl_sync(0xffffffffu, my_hi, j);
        if (PR_SUB_LANES < 32 && hi - lo <= PR_SUB_MAX) break;
        const double s = span_sum_warp<STREAM, SRC>(B.csc, lo, hi, x);
        if (lane == j) mine = s;
    }
    if constexpr (PR_SUB_LANES < 32) {
        constexpr int L = PR_SUB_LANES, G = 32 / L;
        for (; j < cnt; j += G) {
            const int jj = j + lane / L;
            const int src = jj < 31 ? jj : 31;
            int64_t lo = __shfl_sync(0xffffffffu, my_lo, src), hi = __shfl_sync(0xffffffffu, my_hi, src);
            if (jj >= cnt) hi = lo;
            const double s = span_sum_sub<STREAM, SRC, L>(B.csc, lo, hi, x);
            const int k = lane - j;   // this lane's row is summed by group k
            const double v = __shfl_sync(0xffffffffu, s, (k >= 0 && k < G ? k : 0) * L);
            if (k >= 0 && k < G) mine = v;
        }
    }
    return mine;
}

#ifndef PR_UNIT_RING
#define PR_UNIT_RING 1
#endif

// Row callbacks R (a functor):
//   R::Pre pre(bool valid, int64_t row)   per-row loads that do not depend on
//                                         the sum (issued before the gathers)
//   void fin(bool valid, const Pre&, double sum)   all 32 lanes of a warp
//   void single(int64_t row, double sum)           one thread (hub rows)
// PREFETCH: load a row's bounds and drain inputs before its gathers (more
// live registers; pays when the round is latency-bound, i.e. L2-resident)
template <bool STREAM, bool PREFETCH, int SRC, class R>
__device__ __forceinline__ void bins_run(const BinView &B, const int64_t u_lo, const int64_t u_hi, const Src x,
                                         R &rows) {
    __shared__ double red[8];
    __shared__ int64_t next_unit[2];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int64_t warp_rows = B.n_hub + B.n_warp;
    // dynamic unit dispatch: first unit = blockIdx.x, then one atomic per unit
    // (units are ordered heaviest first); the round finaliser resets the counter
    int ring = 0;
    for (int64_t u = u_lo + blockIdx.x; u < u_hi;) {
#if PR_DYNAMIC_UNITS
        // claim the following unit now; the atomic's latency hides behind this unit
        unsigned long long claim = 0;
        if (tid == 0) claim = atomicAdd(B.unit_ctr, 1ull);
#endif
        const int2 d = B.units[u];
        if (d.y < 0) {
            // ---- HUB_CHUNK edges of one hub row, whole block
            const int64_t r = d.x, c = -(int64_t)d.y - 1;
            const int64_t rb = B.doff[r], re = B.doff[r + 1];
            const int64_t c0 = rb + c * HUB_CHUNK;
            const int64_t c1 = c0 + HUB_CHUNK < re ? c0 + HUB_CHUNK : re;
            // HUB_STEP edges at a time (16 gathers per thread in flight), no
            // barrier until the whole chunk is summed
            double acc = 0.0;
            for (int64_t s0 = c0; s0 < c1; s0 += HUB_STEP) {
                int idx[HUB_STEP / 256];
#pragma unroll
                for (int q = 0; q < HUB_STEP / 256; ++q) {
                    const int64_t e = s0 + tid + 256 * q;
                    idx[q] = e < c1 ? ld_idx<STREAM>(&B.csc[e]) : -1;
                }
#pragma unroll
                for (int q = 0; q < HUB_STEP / 256; ++q) acc += idx[q] >= 0 ? ld_src<SRC>(x, idx[q]) : 0.0;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            __syncthreads();
            if (lane == 0) red[wid] = acc;
            __syncthreads();
            if (tid == 0) {
                double s = 0.0;
                for (int k = 0; k < 8; ++k) s += red[k];
                const int nch = (int)((re - rb + HUB_CHUNK - 1) / HUB_CHUNK);
                B.chunk_part[B.chunk_base[r] + c] = s;
                __threadfence();
                if (atomicAdd(&B.row_cnt[r], 1) == nch - 1) {
                    __threadfence();
                    const int64_t first = B.chunk_base[r];
                    double tot = 0.0;
                    for (int k = 0; k < nch; ++k) tot += __ldcg(&B.chunk_part[first + k]);
                    B.row_cnt[r] = 0;
                    rows.single(r, tot);
                }
            }
        } else if (d.x < warp_rows) {
            // ---- warp rows: warp w takes rows w, w+8, ...; lane j loads the
            // bounds and drain inputs of row j of the batch up front, then the
            // warp sums the rows one by one and drains them lane-parallel
            for (int64_t base = d.x + wid; base < d.y; base += 8 * 32) {
                const int64_t my_row = base + 8 * lane;
                const bool my_valid = my_row < d.y;
                const int cnt = __popc(__ballot_sync(0xffffffffu, my_valid));
                double mine = 0.0;
                if constexpr (PREFETCH) {
                    int64_t my_lo = 0, my_hi = 0;
                    if (my_valid) {
                        my_lo = B.doff[my_row];
                        my_hi = B.doff[my_row + 1];
                    }
                    const auto pre = rows.pre(my_valid, my_row);
                    mine = warp_batch_sums<STREAM, SRC>(B, x, my_lo, my_hi, cnt);
                    rows.fin(my_valid, pre, mine);
                } else {
                    int64_t my_lo = 0, my_hi = 0;
                    if (my_valid) {
                        my_lo = B.doff[my_row];
                        my_hi = B.doff[my_row + 1];
                    }
                    mine = warp_batch_sums<STREAM, SRC>(B, x, my_lo, my_hi, cnt);
                    rows.fin(my_valid, rows.pre(my_valid, my_row), mine);
                }
            }
        } else {
            // ---- thread rows: thread t takes rows t, t+256, ... from the
            // 32-row slice boundary at or before the unit start (a warp walks
            // whole SELL slices; rows outside the unit idle)
            for (int64_t base = warp_rows + ((d.x - warp_rows) & ~(int64_t)31); base < d.y; base += 256) {
                const int64_t row = base + tid;
                const bool valid = row >= d.x && row < d.y;
                if constexpr (PREFETCH) {
                    const auto pre = rows.pre(valid, row);
                    const double s = valid ? thread_row_sum<STREAM, SRC>(B, warp_rows, row, x) : 0.0;
                    rows.fin(valid, pre, s);
                } else {
                    const double s = valid ? thread_row_sum<STREAM, SRC>(B, warp_rows, row, x) : 0.0;
                    rows.fin(valid, rows.pre(valid, row), s);
                }
            }
        }
#if PR_DYNAMIC_UNITS
#if PR_UNIT_RING
        // two-slot ring: one barrier per unit
        if (tid == 0) next_unit[ring] = u_lo + (int64_t)gridDim.x + (int64_t)claim;
        __syncthreads();
        u = next_unit[ring];
        ring ^= 1;
#else
        if (tid == 0) next_unit[0] = (int64_t)gridDim.x + (int64_t)claim;
        __syncthreads();
        u = next_unit[0];
        __syncthreads();
#endif
#else
        u += gridDim.x;
#endif
    }
}

// The same schedule with lambda callbacks and no prefetch (the streamed,
// bandwidth-bound rounds and the power gather; this form measured ~3% faster
// there than the functor form above with PREFETCH = false, same SASS mix).
// thread_row(valid, row, sum): all 32 lanes of a warp (warp-collective safe)
// single_row(row, sum): one thread
template <bool STREAM, int SRC, class ThreadRow, class SingleRow>
__device__ __forceinline__ void bins_run_plain(const BinView &B, const int64_t u_lo, const int64_t u_hi, const Src x,
                                               ThreadRow &thread_row, SingleRow &single_row) {
    __shared__ double red[8];
    __shared__ int64_t next_unit[2];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int64_t warp_rows = B.n_hub + B.n_warp;
    // dynamic unit dispatch: first unit = blockIdx.x, then one atomic per unit
    // (units are ordered heaviest first); the round finaliser resets the counter
    int ring = 0;
    for (int64_t u = u_lo + blockIdx.x; u < u_hi;) {
#if PR_DYNAMIC_UNITS
        // claim the following unit now; the atomic's latency hides behind this unit
        unsigned long long claim = 0;
        if (tid == 0) claim = atomicAdd(B.unit_ctr, 1ull);
#endif
        const int2 d = B.units[u];
        if (d.y < 0) {
            // ---- HUB_CHUNK edges of one hub row, whole block
            const int64_t r = d.x, c = -(int64_t)d.y - 1;
            const int64_t rb = B.doff[r], re = B.doff[r + 1];
            const int64_t c0 = rb + c * HUB_CHUNK;
            const int64_t c1 = c0 + HUB_CHUNK < re ? c0 + HUB_CHUNK : re;
            // HUB_STEP edges at a time (16 gathers per thread in flight), no
            // barrier until the whole chunk is summed
            double acc = 0.0;
            for (int64_t s0 = c0; s0 < c1; s0 += HUB_STEP) {
                int idx[HUB_STEP / 256];
#pragma unroll
                for (int q = 0; q < HUB_STEP / 256; ++q) {
                    const int64_t e = s0 + tid + 256 * q;
                    idx[q] = e < c1 ? ld_idx<STREAM>(&B.csc[e]) : -1;
                }
#pragma unroll
                for (int q = 0; q < HUB_STEP / 256; ++q) acc += idx[q] >= 0 ? ld_src<SRC>(x, idx[q]) : 0.0;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            __syncthreads();
            if (lane == 0) red[wid] = acc;
            __syncthreads();
            if (tid == 0) {
                double s = 0.0;
                for (int k = 0; k < 8; ++k) s += red[k];
                const int nch = (int)((re - rb + HUB_CHUNK - 1) / HUB_CHUNK);
                B.chunk_part[B.chunk_base[r] + c] = s;
                __threadfence();
                if (atomicAdd(&B.row_cnt[r], 1) == nch - 1) {
                    __threadfence();
                    const int64_t first = B.chunk_base[r];
                    double tot = 0.0;
                    for (int k = 0; k < nch; ++k) tot += __ldcg(&B.chunk_part[first + k]);
                    B.row_cnt[r] = 0;
                    single_row(r, tot);
                }
            }
        } else if (d.x < warp_rows) {
            // ---- warp rows: warp w takes rows w, w+8, ...; sums of 32 rows
            // collected (lane j holds row j's) and drained lane-parallel
            for (int64_t base = d.x + wid; base < d.y; base += 8 * 32) {
                const int64_t row = base + 8 * lane;
                const bool valid = row < d.y;
                const int cnt = __popc(__ballot_sync(0xffffffffu, valid));
                int64_t my_lo = 0, my_hi = 0;
                if (valid) {
                    my_lo = B.doff[row];
                    my_hi = B.doff[row + 1];
                }
                const double mine = warp_batch_sums<STREAM, SRC>(B, x, my_lo, my_hi, cnt);
                thread_row(valid, row, mine);
            }
        } else {
            // ---- thread rows: whole SELL slices per warp (see bins_run)
            for (int64_t base = warp_rows + ((d.x - warp_rows) & ~(int64_t)31); base < d.y; base += 256) {
                const int64_t row = base + tid;
                const bool valid = row >= d.x && row < d.y;
                const double s = valid ? thread_row_sum<STREAM, SRC>(B, warp_rows, row, x) : 0.0;
                thread_row(valid, row, s);
            }
        }
#if PR_DYNAMIC_UNITS
        // two-slot ring: one barrier per unit
        if (tid == 0) next_unit[ring] = u_lo + (int64_t)gridDim.x + (int64_t)claim;
        __syncthreads();
        u = next_unit[ring];
        ring ^= 1;
#else
        u += gridDim.x;
#endif
    }
}

}  // namespace pr
