// tiles.cuh -- warp-streamed segmented CSC gather (merge-path style).
//
// The compacted CSC of the destination set D is cut into merge-path ranges
// of equal weight (edges + ALPHA * rows, range starts aligned to 8 edges),
// ~4 per warp of the persistent grid, assigned round-robin.  A warp streams its range in 256-edge windows: lane j owns edges
// [w + 8j, w + 8j + 8), loads their sources with two 16-byte loads and
// issues the 8 gathers x[src] back to back; the next window's indices and
// row-start bits are fetched before the current window is reduced, so index
// latency hides behind the gathers.  Row boundaries come from a 1-bit-per-
// edge row-start bitmap.  In-lane rows are summed sequentially; rows
// crossing lanes are joined by a segmented warp scan (fixed shuffle tree),
// rows crossing windows by a carry.  Completed rows are staged in a per-warp
// shared buffer and drained in lane-parallel batches (coalesced vertex
// loads) by the caller's drain_batch.
//
// Rows cut by a range boundary ("split rows") are finished by the last of
// their ranges to arrive: the range where the row starts publishes its
// trailing partial T[k], every later range its leading partial L[k]; the
// last arrival (per-row counter) adds T[k1] + L[k1+1] + ... + L[k2] in range
// order.  All summation orders are fixed by the schedule, so results are
// run-to-run deterministic.
#pragma once

#include "internal.cuh"

namespace pr {

constexpr int RS_CAP = 512;  // staged row sums per warp (doubles)

struct RangeView {
    const int32_t *ids;      // D row -> vertex id
    const int64_t *doff;     // row offsets in csc
    const int32_t *csc;      // compacted sources (padded)
    const uint8_t *flags8;   // row-start bitmap (LSB first)
    const int64_t *rstart;   // range k = edges [rstart[k], rstart[k+1]), multiples of 8
    const int32_t *rrow;     // range k -> row containing its first edge
    const int2 *rsplit;      // range k -> (range where rrow[k] starts, range where the row open at
                             //             the range end finishes)
    int64_t edges, n_ranges;
    int32_t *row_cnt;        // split-row arrival counters
    double *lead, *trail;    // per-range partials of split rows
};

__device__ __forceinline__ void load_window(const RangeView &R, int64_t w, int (&idx)[8], unsigned &fl) {
    const int lane = threadIdx.x & 31;
    const int64_t eb = w + 8 * lane;
    const int4 *p = reinterpret_cast<const int4 *>(R.csc + eb);
    int4 a = __ldg(p), b = __ldg(p + 1);
    idx[0] = a.x; idx[1] = a.y; idx[2] = a.z; idx[3] = a.w;
    idx[4] = b.x; idx[5] = b.y; idx[6] = b.z; idx[7] = b.w;
    fl = __ldg(R.flags8 + (eb >> 3));
}

// Split row `row` gets contribution `part` from range k (trail if it starts
// in k, else lead); the last of its ranges to arrive finishes it.
// Ranges k1..k2 cover the row (precomputed by the schedule).
template <class SplitFn>
__device__ __forceinline__ void split_arrive(const RangeView &R, int64_t row, int64_t k, int64_t k1, int64_t k2,
                                             double part, bool is_trail, SplitFn &finish) {
    if (is_trail) R.trail[k] = part;
    else R.lead[k] = part;
    __threadfence();
    if (atomicAdd(&R.row_cnt[row], 1) == (int)(k2 - k1)) {
        __threadfence();
        double tot = __ldcg(&R.trail[k1]);
        for (int64_t q = k1 + 1; q <= k2; ++q) tot += __ldcg(&R.lead[q]);
        R.row_cnt[row] = 0;
        finish(row, tot);
    }
}

// drain_batch(row0, count, rs): rows row0 .. row0+count-1 complete with sums
// rs[0..count) (warp-collective).  finish(row, sum): one split row (lane 0).
template <class DrainFn, class SplitFn>
__device__ __forceinline__ void warp_range(const RangeView &R, int64_t k, const double *__restrict__ x, double *rs,
                                           DrainFn &drain_batch, SplitFn &finish) {
    const int lane = threadIdx.x & 31;
    const int64_t b0 = R.rstart[k];
    const int64_t b1 = R.rstart[k + 1];
    const int64_t r_first = R.rrow[k];
    const bool starts_at_b0 = R.doff[r_first] == b0;
    const int2 ks = R.rsplit[k];  // .x: start range of r_first, .y: end range of the row open at b1
    // local row index of the open segment (0 = r_first); -1 before any row
    int64_t open = starts_at_b0 ? -1 : 0;
    int64_t pend_row = r_first + (starts_at_b0 ? 0 : 1);  // first full row not yet drained
    int pend = 0;
    double carry = 0.0;
    int idx[8];
    unsigned fl;
    load_window(R, b0, idx, fl);
    for (int64_t w = b0; w < b1; w += 256) {
        const int64_t eb = w + 8 * lane;
        double v[8];
        unsigned starts = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const bool valid = eb + q < b1;
            v[q] = valid ? __ldg(&x[idx[q]]) : 0.0;
            if (valid && ((fl >> q) & 1u)) starts |= 1u << q;
        }
        if (w + 256 < b1) load_window(R, w + 256, idx, fl);  // prefetch behind the gathers
        const int ns = __popc(starts);
        int incl = ns;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const int win_starts = __shfl_sync(0xffffffffu, incl, 31);
        // local row of the segment open before this lane's first start
        const int64_t lane_open = open + (incl - ns);
        // the drain buffer must hold every row completing in this window
        if (pend + win_starts >= RS_CAP) {
            __syncwarp();
            drain_batch(pend_row, pend, rs);
            __syncwarp();
            pend_row += pend;
            pend = 0;
        }
        const int64_t rs_base = pend_row - r_first;  // local row held in rs[0]
        double acc = 0.0, lead = 0.0;
        int64_t row = lane_open;
        bool seen = false;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if ((starts >> q) & 1u) {
                if (seen) rs[row - rs_base] = acc;  // a row started and ended inside this lane
                else lead = acc;
                seen = true;
                acc = 0.0;
                ++row;
            }
            acc += v[q];
        }
        double S = acc;
        bool H = seen;
        if (lane == 0 && !H) S = carry + S;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            double S2 = __shfl_up_sync(0xffffffffu, S, o);
            bool H2 = __shfl_up_sync(0xffffffffu, H, o);
            if (lane >= o && !H) S = S2 + S;
            if (lane >= o) H = H || H2;
        }
        double cin = __shfl_up_sync(0xffffffffu, S, 1);
        if (lane == 0) cin = carry;
        if (seen && lane_open >= 0) {
            const double sum = cin + lead;
            if (lane_open == 0 && !starts_at_b0)
                split_arrive(R, r_first, k, ks.x, k, sum, false, finish);  // lead of a split row ending here
            else rs[lane_open - rs_base] = sum;
        }
        carry = __shfl_sync(0xffffffffu, S, 31);
        open += win_starts;
        // rows finished in this window: every row before the open one
        const int64_t done_to = r_first + open;  // exclusive (global row of the open segment)
        pend = (int)(done_to - pend_row);
        if (pend < 0) pend = 0;
        __syncwarp();
    }
    // the segment still open at the range end
    if (lane == 0 && open >= 0) {
        const int64_t row = r_first + open;
        if (open == 0 && !starts_at_b0) {
            split_arrive(R, row, k, ks.x, ks.y, carry, false, finish);  // whole range inside one row
        } else if (R.doff[row + 1] > b1) {
            split_arrive(R, row, k, k, ks.y, carry, true, finish);      // continues into the next range
        } else {
            rs[row - pend_row] = carry;                     // ends exactly at the range end
        }
    }
    __syncwarp();
    if (open >= 0) {
        const int64_t row = r_first + open;
        const bool last_full = !(open == 0 && !starts_at_b0) && !(R.doff[row + 1] > b1);
        const int64_t end = last_full ? row + 1 : row;
        const int cnt = (int)(end - pend_row);
        if (cnt > 0) drain_batch(pend_row, cnt, rs);
    }
    __syncwarp();
}

}  // namespace pr
