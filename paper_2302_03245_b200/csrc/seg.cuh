// seg.cuh -- load-balanced segmented row gather (preprocessing).
//
// Output row i (edges [noff[i], noff[i+1])) is a copy of input row map[i]
// (edges from off[map[i]]), optionally renamed through rank.  Work is cut by
// OUTPUT EDGES, not rows: a block takes a tile of SEG_TILE edges, finds the
// tile's row range with two binary searches, and every thread finds the row
// of its edge by a binary search inside that range (L1-resident).  Power-law
// hub rows therefore cost the same per edge as short rows -- a warp- or
// lane-per-row copy leaves one warp walking a 10^5-edge hub alone.
#pragma once

#include "internal.cuh"

namespace pr {

constexpr int SEG_TILE = 2048;

// first r in [lo, hi) with off[r] > e (hi if none)
__device__ __forceinline__ int64_t seg_upper(const int64_t *__restrict__ off, int64_t lo, int64_t hi, int64_t e) {
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(&off[mid]) > e) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

template <bool RENAME>
__global__ void __launch_bounds__(256) k_seg_gather(const int64_t *__restrict__ noff, int64_t rows,
                                                    const int32_t *__restrict__ map, const int64_t *__restrict__ off,
                                                    const int32_t *__restrict__ col, const int32_t *__restrict__ rank,
                                                    int32_t *__restrict__ out, int64_t m_out) {
    __shared__ int64_t s_r0, s_r1;
    for (int64_t base = blockIdx.x * (int64_t)SEG_TILE; base < m_out; base += (int64_t)gridDim.x * SEG_TILE) {
        const int64_t end = base + SEG_TILE < m_out ? base + SEG_TILE : m_out;
        if (threadIdx.x == 0) s_r0 = seg_upper(noff, 0, rows + 1, base) - 1;  // row holding edge base
        if (threadIdx.x == 32) s_r1 = seg_upper(noff, 0, rows + 1, end - 1);  // one past the row holding end-1
        __syncthreads();
        const int64_t r0 = s_r0, r1 = s_r1;
        for (int64_t e = base + threadIdx.x; e < end; e += blockDim.x) {
            const int64_t i = seg_upper(noff, r0, r1 + 1, e) - 1;
            const int64_t v = map ? (int64_t)__ldg(&map[i]) : i;
            const int32_t c = __ldg(&col[__ldg(&off[v]) + (e - __ldg(&noff[i]))]);
            out[e] = RENAME ? __ldg(&rank[c]) : c;
        }
        __syncthreads();
    }
}

inline unsigned seg_grid(const Ctx &ctx, int64_t m_out) {
    int64_t b = (m_out + SEG_TILE - 1) / SEG_TILE;
    const int64_t cap = (int64_t)ctx.sm_count * 8;
    if (b > cap) b = cap;
    return (unsigned)(b < 1 ? 1 : b);
}

}  // namespace pr
