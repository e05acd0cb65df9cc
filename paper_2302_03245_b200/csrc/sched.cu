// sched.cu -- pull schedules: the destination set D, its compacted CSC and
// the row-aligned warp tiles the gather kernels walk.
//
// Layout (built once per graph and engine, all on the device):
//   ids[i]     vertex id of row i (ascending)
//   doff[i]    offsets of row i's sources in csc (in-edges, ascending source)
//   flags      1 bit per edge: set on the first edge of every row
//   ranges     equal runs of ew edges (ew a multiple of 256), one per warp of
//              the persistent gather grid; rrow[k] = row holding edge k*ew
//              (tiles.cuh streams them and fixes up rows cut by a boundary)
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "cubutil.cuh"
#include "internal.cuh"

namespace pr {

struct RowMember {
    const int64_t *in_off;
    const int32_t *out_deg;
    int which;
    __host__ __device__ bool operator()(int32_t v) const {
        int64_t d = in_off[v + 1] - in_off[v];
        return d > 0 && (which != 1 || out_deg[v] > 0);
    }
};
struct ZeroIn {
    const int64_t *in_off;
    __host__ __device__ bool operator()(int32_t v) const { return in_off[v + 1] == in_off[v]; }
};
struct SeedPred {
    const int64_t *in_off;
    const int32_t *out_deg;
    __host__ __device__ bool operator()(int32_t v) const { return in_off[v + 1] == in_off[v] && out_deg[v] > 0; }
};

__global__ void k_row_len(const int32_t *__restrict__ ids, int64_t cnt, const int64_t *__restrict__ in_off,
                          int64_t *__restrict__ len) {
    GRID_STRIDE(i, cnt) {
        int32_t v = ids[i];
        len[i] = in_off[v + 1] - in_off[v];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) len[cnt] = 0;
}

// warp per row: copy the row's sources and set its start bit
__global__ void k_fill_csc(const int32_t *__restrict__ ids, int64_t cnt, const int64_t *__restrict__ in_off,
                           const int32_t *__restrict__ in_src, const int64_t *__restrict__ doff,
                           int32_t *__restrict__ csc, unsigned *__restrict__ flags) {
    int lane = threadIdx.x & 31;
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp; i < cnt; i += nw) {
        int32_t v = ids[i];
        int64_t lo = in_off[v], len = in_off[v + 1] - lo, o = doff[i];
        for (int64_t k = lane; k < len; k += 32) csc[o + k] = in_src[lo + k];
        if (lane == 0) atomicOr(&flags[o >> 5], 1u << (o & 31));
    }
}

// Merge-path split: range k starts at weight k*W on the axis where row i
// occupies ALPHA units (its drain) followed by its edges.  The start is
// snapped down to a multiple of 8 edges; rrow[k] = row holding that edge.
__global__ void k_range_split(const int64_t *__restrict__ doff, int64_t cnt, int64_t edges, int64_t W,
                              int64_t n_ranges, int64_t *__restrict__ rstart, int32_t *__restrict__ rrow) {
    GRID_STRIDE(k, n_ranges + 1) {
        if (k == n_ranges) { rstart[k] = edges; continue; }
        const int64_t p = k * W;
        int64_t lo = 0, hi = cnt - 1;  // last row i with doff[i] + ALPHA*i <= p
        while (lo < hi) {
            int64_t mid = (lo + hi + 1) >> 1;
            if (doff[mid] + RANGE_ALPHA * mid <= p) lo = mid;
            else hi = mid - 1;
        }
        int64_t e = p - RANGE_ALPHA * lo;
        if (e < doff[lo]) e = doff[lo];
        if (e > doff[lo + 1]) e = doff[lo + 1];
        e &= ~7ll;
        if (k == 0) e = 0;
        rstart[k] = e;
        // row holding edge e (doff strictly increasing: every D row has an edge)
        int64_t a = 0, b = cnt - 1;
        while (a < b) {
            int64_t mid = (a + b + 1) >> 1;
            if (doff[mid] <= e) a = mid;
            else b = mid - 1;
        }
        rrow[k] = (int32_t)a;
    }
}

__device__ __forceinline__ int64_t range_holding(const int64_t *rstart, int64_t n_ranges, int64_t e) {
    int64_t lo = 0, hi = n_ranges - 1;
    while (lo < hi) {
        int64_t mid = (lo + hi + 1) >> 1;
        if (rstart[mid] <= e) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// per range: (range where its first row starts, range where the row holding
// its last edge ends) -- the split-row fix-up bounds used by tiles.cuh
__global__ void k_range_bounds(const int64_t *__restrict__ doff, const int64_t *__restrict__ rstart,
                               const int32_t *__restrict__ rrow, int64_t cnt, int64_t n_ranges,
                               int2 *__restrict__ rsplit) {
    GRID_STRIDE(k, n_ranges) {
        int64_t r0 = rrow[k];
        int64_t b1 = rstart[k + 1];
        int64_t lo = 0, hi = cnt - 1;  // row holding edge b1-1
        while (lo < hi) {
            int64_t mid = (lo + hi + 1) >> 1;
            if (doff[mid] <= b1 - 1) lo = mid;
            else hi = mid - 1;
        }
        int64_t k1 = range_holding(rstart, n_ranges, doff[r0]);
        int64_t k2 = range_holding(rstart, n_ranges, doff[lo + 1] - 1);
        rsplit[k] = make_int2((int)k1, (int)k2);
    }
}

int ensure_sched(Graph &g, int which, int64_t target_warps) {
    auto &S = g.sched[which];
    if (S.built) return PR_OK;
    Ctx &ctx = *g.ctx;
    cudaStream_t st = ctx.stream;
    int64_t n = g.n;
    DevBuf dcount, len;
    PR_TRY(ensure(dcount, 8));
    PR_TRY(ensure(S.ids, 4 * n));
    auto first = thrust::make_counting_iterator<int32_t>(0);
    int mode = which;
    PR_TRY(cub_run(ctx, [&](void *t, size_t &b) {
        return cub::DeviceSelect::If(t, b, first, S.ids.as<int32_t>(), dcount.as<int64_t>(), (int)n,
                                     RowMember{g.in_off.as<int64_t>(), g.out_deg.as<int32_t>(), mode}, st);
    }));
    int64_t cnt = 0;
    PR_CUDA(cudaMemcpyAsync(&cnt, dcount.ptr, 8, cudaMemcpyDeviceToHost, st));
    PR_CUDA(cudaStreamSynchronize(st));
    S.count = cnt;
    // compacted CSC offsets
    PR_TRY(ensure(len, 8 * (cnt + 1)));
    PR_TRY(ensure(S.doff, 8 * (cnt + 1)));
    k_row_len<<<grid_for(cnt + 1, 256) > 4096 ? 4096 : grid_for(cnt + 1, 256), 256, 0, st>>>(
        S.ids.as<int32_t>(), cnt, g.in_off.as<int64_t>(), len.as<int64_t>());
    PR_TRY(cub_run(ctx, [&](void *t, size_t &b) {
        return cub::DeviceScan::ExclusiveSum(t, b, len.as<int64_t>(), S.doff.as<int64_t>(), (int)(cnt + 1), st);
    }));
    int64_t edges = 0;
    PR_CUDA(cudaMemcpyAsync(&edges, S.doff.as<int64_t>() + cnt, 8, cudaMemcpyDeviceToHost, st));
    PR_CUDA(cudaStreamSynchronize(st));
    S.edges = edges;
    PR_TRY(ensure(S.csc, 4 * (edges + CSC_PAD)));
    size_t flag_words = (size_t)((edges + CSC_PAD) / 32 + 2);
    PR_TRY(ensure(S.flags, 4 * flag_words));
    PR_CUDA(cudaMemsetAsync(S.csc.ptr, 0, 4 * (edges + CSC_PAD), st));
    PR_CUDA(cudaMemsetAsync(S.flags.ptr, 0, 4 * flag_words, st));
    if (cnt) {
        unsigned gr = grid_for(cnt * 32, 256);
        if (gr > (unsigned)ctx.sm_count * 32) gr = ctx.sm_count * 32;
        k_fill_csc<<<gr, 256, 0, st>>>(S.ids.as<int32_t>(), cnt, g.in_off.as<int64_t>(), g.in_src.as<int32_t>(),
                                       S.doff.as<int64_t>(), S.csc.as<int32_t>(), S.flags.as<unsigned>());
    }
    // merge-path ranges of equal weight, ~RANGES_PER_WARP per warp of the gather grid
    int64_t target = (target_warps > 0 ? target_warps : (int64_t)ctx.sm_count * 24) * RANGES_PER_WARP;
    const int64_t weight = edges + RANGE_ALPHA * cnt;
    int64_t W = (weight + target - 1) / target;
    if (W < 64 * (RANGE_ALPHA + 1)) W = 64 * (RANGE_ALPHA + 1);
    S.ew = W;
    S.n_ranges = edges ? (weight + W - 1) / W : 0;
    PR_TRY(ensure(S.rrow, 4 * (S.n_ranges + 1)));
    PR_TRY(ensure(S.rstart, 8 * (S.n_ranges + 1)));
    if (cnt) {
        unsigned gc = grid_for(S.n_ranges + 1, 256);
        k_range_split<<<gc, 256, 0, st>>>(S.doff.as<int64_t>(), cnt, edges, W, S.n_ranges, S.rstart.as<int64_t>(),
                                          S.rrow.as<int32_t>());
    }
    PR_TRY(ensure(S.rsplit, 8 * (S.n_ranges + 1)));
    if (cnt && S.n_ranges)
        k_range_bounds<<<grid_for(S.n_ranges, 256), 256, 0, st>>>(S.doff.as<int64_t>(), S.rstart.as<int64_t>(),
                                                                   S.rrow.as<int32_t>(), cnt, S.n_ranges,
                                                                   S.rsplit.as<int2>());
    PR_TRY(ensure(S.row_cnt, 4 * (cnt ? cnt : 1)));
    PR_CUDA(cudaMemsetAsync(S.row_cnt.ptr, 0, 4 * (cnt ? cnt : 1), st));
    PR_TRY(ensure(S.lead, 8 * (S.n_ranges ? S.n_ranges : 1)));
    PR_TRY(ensure(S.trail, 8 * (S.n_ranges ? S.n_ranges : 1)));
    // power: in-degree-0 vertices; engines: round-0 scatter seeds
    PR_TRY(ensure(S.zero_ids, 4 * n));
    if (which == 2) {
        PR_TRY(cub_run(ctx, [&](void *t, size_t &b) {
            return cub::DeviceSelect::If(t, b, first, S.zero_ids.as<int32_t>(), dcount.as<int64_t>(), (int)n,
                                         ZeroIn{g.in_off.as<int64_t>()}, st);
        }));
        PR_CUDA(cudaMemcpyAsync(&S.n_zero, dcount.ptr, 8, cudaMemcpyDeviceToHost, st));
        PR_CUDA(cudaStreamSynchronize(st));
    }
    PR_TRY(ensure(S.seed_ids, 4 * n));
    PR_TRY(cub_run(ctx, [&](void *t, size_t &b) {
        return cub::DeviceSelect::If(t, b, first, S.seed_ids.as<int32_t>(), dcount.as<int64_t>(), (int)n,
                                     SeedPred{g.in_off.as<int64_t>(), g.out_deg.as<int32_t>()}, st);
    }));
    PR_CUDA(cudaMemcpyAsync(&S.n_seed, dcount.ptr, 8, cudaMemcpyDeviceToHost, st));
    PR_CUDA(cudaStreamSynchronize(st));
    PR_CUDA(cudaGetLastError());
    S.built = true;
    return PR_OK;
}

}  // namespace pr
