// sched.cu -- pull schedules: the destination set D, its compacted CSC and
// the degree bins the gather kernels walk.
//
// Layout (built once per graph and engine, all on the device):
//   ids[i]     vertex id of row i; rows sorted by descending in-degree
//              (stable, so ties keep ascending id)
//   doff[i]    offsets of row i's sources in csc (in-edges, ascending source)
//   bins       rows [0, n_hub): > HUB_DEG edges; [n_hub, n_hub + n_warp):
//              > THREAD_DEG edges (warp per row); the rest thread per row
//   units      per grid size: hub rows cut into HUB_CHUNK-edge block units
//              (combined by the last arriving chunk in chunk order); each
//              other bin cut into contiguous row ranges of near-equal cost
//              (edges + ROW_COST * rows, by a prefix sum), ~UNITS_PER_BLOCK
//              per block of the persistent grid.
#include <cub/cub.cuh>
#include <utility>
#include <thrust/iterator/counting_iterator.h>

#include "cubutil.cuh"
#include "internal.cuh"
#include "seg.cuh"

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

__global__ void k_iota(int32_t *__restrict__ out, int64_t start, int64_t count) {
    GRID_STRIDE(i, count) out[i] = (int32_t)(start + i);
}

// descending-degree sort key (ascending radix sort of ~degree)
__global__ void k_deg_keys(const int32_t *__restrict__ ids, int64_t cnt, const int64_t *__restrict__ in_off,
                           unsigned *__restrict__ keys) {
    GRID_STRIDE(i, cnt) {
        int32_t v = ids[i];
        keys[i] = ~(unsigned)(in_off[v + 1] - in_off[v]);
    }
}

__global__ void k_row_len(const int32_t *__restrict__ ids, int64_t cnt, const int64_t *__restrict__ in_off,
                          int64_t *__restrict__ len) {
    GRID_STRIDE(i, cnt + 1) {
        if (i == cnt) { len[cnt] = 0; continue; }
        int32_t v = ids[i];
        len[i] = in_off[v + 1] - in_off[v];
    }
}

// numbers of rows with degree > t1 and > t2 (rows sorted by descending degree)
__global__ void k_count_above(const int64_t *__restrict__ doff, int64_t cnt, int64_t t1, int64_t t2,
                              unsigned long long *__restrict__ out) {
    GRID_STRIDE(i, cnt) {
        int64_t d = doff[i + 1] - doff[i];
        if (d > t1) atomicAdd(&out[0], 1ull);
        if (d > t2) atomicAdd(&out[1], 1ull);
    }
}

__global__ void k_chunks_of(const int64_t *__restrict__ doff, int64_t n_hub, int64_t *__restrict__ nch) {
    GRID_STRIDE(i, n_hub + 1) { nch[i] = i < n_hub ? (doff[i + 1] - doff[i] + HUB_CHUNK - 1) / HUB_CHUNK : 0; }
}


__global__ void k_row_cost(const int64_t *__restrict__ doff, int64_t cnt, int64_t *__restrict__ cost) {
    GRID_STRIDE(i, cnt + 1) { cost[i] = i < cnt ? doff[i + 1] - doff[i] + ROW_COST : 0; }
}

// SELL-32 slices of the thread-row bin (rows [t0, count), 32 per slice):
// width[s] = 32 * (largest degree in the slice); width[n_slices] = 0
__global__ void k_slice_width(const int64_t *__restrict__ doff, int64_t t0, int64_t count, int64_t n_slices,
                              int64_t *__restrict__ width) {
    GRID_STRIDE(s, n_slices + 1) {
        int64_t w = 0;
        if (s < n_slices) {
            const int64_t r0 = t0 + 32 * s, r1 = r0 + 32 < count ? r0 + 32 : count;
            for (int64_t r = r0; r < r1; ++r) {
                const int64_t d = doff[r + 1] - doff[r];
                w = d > w ? d : w;
            }
        }
        width[s] = 32 * w;
    }
}

__global__ void k_add_i64(int64_t *__restrict__ a, int64_t count, int64_t v) {
    GRID_STRIDE(i, count) a[i] += v;
}

// thread row r = t0 + 32 s + j: its k-th source goes to sell_off[s] + 32 k + j,
// so lane j's k-th index load of a warp over slice s is one 128-byte line
__global__ void k_sell_scatter(const int64_t *__restrict__ doff, int64_t t0, int64_t count,
                               const int32_t *__restrict__ csr, const int64_t *__restrict__ sell_off,
                               int32_t *__restrict__ out) {
    GRID_STRIDE(i, count - t0) {
        const int64_t r = t0 + i;
        const int64_t lo = doff[r], d = doff[r + 1] - lo;
        int32_t *dst = out + sell_off[i >> 5] + (i & 31);
        for (int64_t k = 0; k < d; ++k) dst[32 * k] = csr[lo + k];
    }
}

// hub chunk units (row, -(chunk+1)) in row/chunk order
// units of the hub rows [h0, h1), written from `out` on: one per HUB_CHUNK
// slice, (row, -(slice+1))
__global__ void k_hub_units(const int64_t *__restrict__ base, int64_t h0, int64_t h1, int2 *__restrict__ out) {
    GRID_STRIDE(j, h1 - h0) {
        const int64_t i = h0 + j;
        for (int64_t c = base[i]; c < base[i + 1]; ++c) out[c - base[h0]] = make_int2((int)i, (int)(-(c - base[i] + 1)));
    }
}

// section row bounds: b[k] = first row whose CSC offset reaches k*E/K
__global__ void k_section_bounds(const int64_t *__restrict__ doff, int64_t count, int nsec, int64_t *__restrict__ b) {
    const int k = threadIdx.x;
    if (k > nsec) return;
    if (k == 0) { b[0] = 0; return; }
    if (k == nsec) { b[k] = count; return; }
    const int64_t E = doff[count], target = (int64_t)((__int128)E * k / nsec);
    int64_t lo = 0, hi = count;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (doff[mid] >= target) hi = mid;
        else lo = mid + 1;
    }
    b[k] = lo;
}

// k equal-cost row ranges over rows [r0, r1): unit j = [first row with
// cum >= j*C/k, first row with cum >= (j+1)*C/k)
__global__ void k_range_units(const int64_t *__restrict__ cum, int64_t r0, int64_t r1, int64_t k,
                              int2 *__restrict__ units) {
    GRID_STRIDE(j, k) {
        const int64_t base = cum[r0], total = cum[r1] - base;
        auto find = [&](int64_t target) {
            int64_t lo = r0, hi = r1;
            while (lo < hi) {
                int64_t mid = (lo + hi) >> 1;
                if (cum[mid] - base >= target) hi = mid;
                else lo = mid + 1;
            }
            return lo;
        };
        const int64_t a = j == 0 ? r0 : find((int64_t)((__int128)total * j / k));
        const int64_t b = j == k - 1 ? r1 : find((int64_t)((__int128)total * (j + 1) / k));
        units[j] = make_int2((int)a, (int)b);
    }
}

// Work units of a schedule for a persistent grid of `blocks` blocks, cut into
// `nsec` Gauss-Seidel sections of equal edge count (rounds.cu).  Units are
// laid out section by section, each section hub slices, then warp-row ranges,
// then thread-row ranges, so a section's units are the contiguous range
// [sec_unit[k], sec_unit[k+1]).
int ensure_units(Graph &g, int which, int64_t blocks, int nsec) {
    auto &S = g.sched[which];
    if (nsec < 1) nsec = 1;
    if (nsec > PR_MAX_SECTIONS) nsec = PR_MAX_SECTIONS;
    if (S.unit_blocks == blocks && S.nsec == nsec) return PR_OK;
    Ctx &ctx = *g.ctx;
    cudaStream_t st = ctx.stream;
    // section row bounds
    int64_t b[PR_MAX_SECTIONS + 1];
    {
        DevBuf db;
        PR_TRY(ensure(db, 8 * (PR_MAX_SECTIONS + 1)));
        k_section_bounds<<<1, 32, 0, st>>>(S.doff.as<int64_t>(), S.count, nsec, db.as<int64_t>());
        PR_CUDA(cudaMemcpyAsync(b, db.ptr, 8 * (nsec + 1), cudaMemcpyDeviceToHost, st));
        PR_CUDA(cudaStreamSynchronize(st));
    }
    // segments (section x bin) and the prefix values they need
    const int64_t bin_lo[3] = {0, S.n_hub, S.n_hub + S.n_warp};
    const int64_t bin_hi[3] = {S.n_hub, S.n_hub + S.n_warp, S.count};
    int64_t seg_lo[PR_MAX_SECTIONS][3], seg_hi[PR_MAX_SECTIONS][3];
    int64_t cum_lo[PR_MAX_SECTIONS][3], cum_hi[PR_MAX_SECTIONS][3], hb_lo[PR_MAX_SECTIONS], hb_hi[PR_MAX_SECTIONS];
    for (int k = 0; k < nsec; ++k)
        for (int j = 0; j < 3; ++j) {
            // section k's rows of bin j, clamped inside the bin
            int64_t lo = b[k] > bin_lo[j] ? b[k] : bin_lo[j];
            int64_t hi = b[k + 1] < bin_hi[j] ? b[k + 1] : bin_hi[j];
            if (lo > bin_hi[j]) lo = bin_hi[j];
            if (hi < lo) hi = lo;
            seg_lo[k][j] = lo;
            seg_hi[k][j] = hi;
            PR_CUDA(cudaMemcpyAsync(&cum_lo[k][j], S.row_cum.as<int64_t>() + seg_lo[k][j], 8, cudaMemcpyDeviceToHost, st));
            PR_CUDA(cudaMemcpyAsync(&cum_hi[k][j], S.row_cum.as<int64_t>() + seg_hi[k][j], 8, cudaMemcpyDeviceToHost, st));
            if (j == 0) {
                PR_CUDA(cudaMemcpyAsync(&hb_lo[k], S.chunk_base.as<int64_t>() + seg_lo[k][0], 8, cudaMemcpyDeviceToHost,
                                        st));
                PR_CUDA(cudaMemcpyAsync(&hb_hi[k], S.chunk_base.as<int64_t>() + seg_hi[k][0], 8, cudaMemcpyDeviceToHost,
                                        st));
            }
        }
    PR_CUDA(cudaStreamSynchronize(st));
    int64_t total = 0;
    for (int k = 0; k < nsec; ++k) total += (cum_hi[k][1] - cum_lo[k][1]) + (cum_hi[k][2] - cum_lo[k][2]);
    int64_t T = total / (blocks * UNITS_PER_BLOCK);
    // very long sweeps (C5: ~220K edge-units per unit): ~UNITS_PER_BLOCK units
    // per block in every section, not over the whole sweep, so that the tail
    // of each section launch is short (C5 4896 -> 4538 us per sweep; C3's
    // short units lose with more of them: 9.9 -> 11.0 ms at 2x)
    if (nsec > 1 && T > LONG_UNIT) T = total / (blocks * UNITS_PER_BLOCK * nsec);
    // smallest unit, in edge-units: each unit costs a dispatch barrier, so
    // L2-resident sweeps want fewer, larger ones (measured against 3200:
    // 8K C2 -7%, 16K C4 -7%; C3 and C5 units are larger anyway)
    if (T < PR_MIN_UNIT) T = PR_MIN_UNIT;
    int64_t cnt[PR_MAX_SECTIONS][3];
    int64_t n_units = 0;
    for (int k = 0; k < nsec; ++k) {
        S.sec_row[k] = b[k];
        S.sec_unit[k] = n_units;
        cnt[k][0] = hb_hi[k] - hb_lo[k];
        for (int j = 1; j < 3; ++j) {
            const int64_t c = cum_hi[k][j] - cum_lo[k][j];
            cnt[k][j] = seg_hi[k][j] > seg_lo[k][j] ? (c + T - 1) / T : 0;
        }
        n_units += cnt[k][0] + cnt[k][1] + cnt[k][2];
    }
    S.sec_row[nsec] = b[nsec];
    S.sec_unit[nsec] = n_units;
    S.n_units = n_units;
    PR_TRY(ensure(S.units, 8 * (n_units + 1)));
    int2 *U = S.units.as<int2>();
    for (int k = 0; k < nsec; ++k) {
        int64_t off = S.sec_unit[k];
        if (cnt[k][0]) {
            const int64_t nh = seg_hi[k][0] - seg_lo[k][0];
            k_hub_units<<<grid_for(nh, 256), 256, 0, st>>>(S.chunk_base.as<int64_t>(), seg_lo[k][0], seg_hi[k][0],
                                                          U + off);
        }
        off += cnt[k][0];
        for (int j = 1; j < 3; ++j) {
            if (cnt[k][j])
                k_range_units<<<grid_for(cnt[k][j], 256), 256, 0, st>>>(S.row_cum.as<int64_t>(), seg_lo[k][j],
                                                                       seg_hi[k][j], cnt[k][j], U + off);
            off += cnt[k][j];
        }
    }
    PR_CUDA(cudaGetLastError());
    S.unit_blocks = blocks;
    S.nsec = nsec;
    return PR_OK;
}

// Thread rows (<= THREAD_DEG in-edges, one thread each) in SELL-32 order:
// a row-major CSR makes each warp index load touch 32 lines (one per lane's
// row), as many L1TEX wavefronts as the gathers themselves; column-major
// slices of 32 degree-sorted rows make it one line per load with almost no
// padding (rows of a slice have near-equal degree).  The per-row summation
// order is unchanged (ascending position, bins.cuh row_sum_sell).
static int sell_layout(Ctx &ctx, Graph::Sched &S) {
    cudaStream_t st = ctx.stream;
    const int64_t t0 = S.n_hub + S.n_warp, nt = S.count - t0;
    S.n_slices = (nt + 31) / 32;
    PR_TRY(ensure(S.sell_off, 8 * (S.n_slices + 1)));
    int64_t e0 = 0, sell = 0;
    PR_CUDA(cudaMemcpyAsync(&e0, S.doff.as<int64_t>() + t0, 8, cudaMemcpyDeviceToHost, st));
    if (nt <= 0 || !PR_SELL) {
        PR_CUDA(cudaMemcpyAsync(S.sell_off.ptr, S.doff.as<int64_t>() + t0, 8, cudaMemcpyDeviceToDevice, st));
        PR_CUDA(cudaStreamSynchronize(st));
        return PR_OK;
    }
    DevBuf width;
    PR_TRY(ensure(width, 8 * (S.n_slices + 1)));
    const unsigned gs = grid_for(S.n_slices + 1, 256) > 4096 ? 4096 : grid_for(S.n_slices + 1, 256);
    k_slice_width<<<gs, 256, 0, st>>>(S.doff.as<int64_t>(), t0, S.count, S.n_slices, width.as<int64_t>());
    PR_TRY(cub_run(ctx, [&](void *t, size_t &b) {
        return cub::DeviceScan::ExclusiveSum(t, b, width.as<int64_t>(), S.sell_off.as<int64_t>(), (int)(S.n_slices + 1),
                                             st);
    }));
    PR_CUDA(cudaMemcpyAsync(&sell, S.sell_off.as<int64_t>() + S.n_slices, 8, cudaMemcpyDeviceToHost, st));
    PR_CUDA(cudaStreamSynchronize(st));
    k_add_i64<<<gs, 256, 0, st>>>(S.sell_off.as<int64_t>(), S.n_slices + 1, e0);
    DevBuf out;
    PR_TRY(ensure(out, 4 * (e0 + sell + CSC_PAD)));
    if (e0) PR_CUDA(cudaMemcpyAsync(out.ptr, S.csc.ptr, 4 * e0, cudaMemcpyDeviceToDevice, st));
    PR_CUDA(cudaMemsetAsync(out.as<int32_t>() + e0, 0, 4 * (sell + CSC_PAD), st));
    const unsigned gt = grid_for(nt, 256) > 65535 ? 65535 : grid_for(nt, 256);
    k_sell_scatter<<<gt, 256, 0, st>>>(S.doff.as<int64_t>(), t0, S.count, S.csc.as<int32_t>(), S.sell_off.as<int64_t>(),
                                      out.as<int32_t>());
    PR_CUDA(cudaGetLastError());
    std::swap(S.csc.ptr, out.ptr);
    std::swap(S.csc.bytes, out.bytes);
    return PR_OK;
}

int ensure_sched(Graph &g, int which) {
    auto &S = g.sched[which];
    if (S.built) return PR_OK;
    Ctx &ctx = *g.ctx;
    cudaStream_t st = ctx.stream;
    int64_t n = g.n;
    DevBuf dcount, len, unsorted, keys, keys2;
    PR_TRY(ensure(dcount, 16));
    PR_TRY(ensure(unsorted, 4 * n));
    PR_TRY(ensure(S.ids, 4 * n));
    auto first = thrust::make_counting_iterator<int32_t>(0);
    int mode = which;
    // run layout, IFP2: D = class 0, already the id prefix [0, class0_end) in
    // descending in-degree order (ties by id, as the stable sort below would
    // leave them) -- its rows are the CSC prefix
    const bool prefix = which == 1 && g.class0_end >= 0;
    int64_t cnt = 0;
    if (prefix) {
        cnt = g.class0_end;
        S.count = cnt;
        PR_TRY(ensure(S.doff, 8 * (cnt + 1)));
        int64_t edges = 0;
        PR_CUDA(cudaMemcpyAsync(&edges, g.in_off.as<int64_t>() + cnt, 8, cudaMemcpyDeviceToHost, st));
        PR_CUDA(cudaMemcpyAsync(S.doff.ptr, g.in_off.ptr, 8 * (cnt + 1), cudaMemcpyDeviceToDevice, st));
        if (cnt) k_iota<<<grid_for(cnt, 256) > 4096 ? 4096 : grid_for(cnt, 256), 256, 0, st>>>(S.ids.as<int32_t>(), 0, cnt);
        PR_CUDA(cudaStreamSynchronize(st));
        S.edges = edges;
        PR_TRY(ensure(S.csc, 4 * (edges + CSC_PAD)));
        PR_CUDA(cudaMemsetAsync(S.csc.as<int32_t>() + edges, 0, 4 * CSC_PAD, st));
        if (edges) PR_CUDA(cudaMemcpyAsync(S.csc.ptr, g.in_src.ptr, 4 * edges, cudaMemcpyDeviceToDevice, st));
    } else {
        PR_TRY(cub_run(ctx, [&](void *t, size_t &b) {
            return cub::DeviceSelect::If(t, b, first, unsorted.as<int32_t>(), dcount.as<int64_t>(), (int)n,
                                         RowMember{g.in_off.as<int64_t>(), g.out_deg.as<int32_t>(), mode}, st);
        }));
        PR_CUDA(cudaMemcpyAsync(&cnt, dcount.ptr, 8, cudaMemcpyDeviceToHost, st));
        PR_CUDA(cudaStreamSynchronize(st));
        S.count = cnt;
        // rows by descending in-degree (stable)
        PR_TRY(ensure(keys, 4 * (cnt ? cnt : 1)));
        PR_TRY(ensure(keys2, 4 * (cnt ? cnt : 1)));
        if (cnt) {
            k_deg_keys<<<grid_for(cnt, 256) > 4096 ? 4096 : grid_for(cnt, 256), 256, 0, st>>>(
                unsorted.as<int32_t>(), cnt, g.in_off.as<int64_t>(), keys.as<unsigned>());
            PR_TRY(cub_run(ctx, [&](void *t, size_t &b) {
                return cub::DeviceRadixSort::SortPairs(t, b, keys.as<unsigned>(), keys2.as<unsigned>(),
                                                       unsorted.as<int32_t>(), S.ids.as<int32_t>(), (int)cnt, 0, 32, st);
            }));
        }
        // compacted CSC in row order
        PR_TRY(ensure(len, 8 * (cnt + 1)));
        PR_TRY(ensure(S.doff, 8 * (cnt + 1)));
        k_row_len<<<grid_for(cnt + 1, 256) > 4096 ? 4096 : grid_for(cnt + 1, 256), 256, 0, st>>>(S.ids.as<int32_t>(), cnt, g.in_off.as<int64_t>(), len.as<int64_t>());
        PR_TRY(cub_run(ctx, [&](void *t, size_t &b) {
            return cub::DeviceScan::ExclusiveSum(t, b, len.as<int64_t>(), S.doff.as<int64_t>(), (int)(cnt + 1), st);
        }));
        int64_t edges = 0;
        PR_CUDA(cudaMemcpyAsync(&edges, S.doff.as<int64_t>() + cnt, 8, cudaMemcpyDeviceToHost, st));
        PR_CUDA(cudaStreamSynchronize(st));
        S.edges = edges;
        PR_TRY(ensure(S.csc, 4 * (edges + CSC_PAD)));
        PR_CUDA(cudaMemsetAsync(S.csc.ptr, 0, 4 * (edges + CSC_PAD), st));
        if (cnt) {
            if (edges)
                k_seg_gather<false><<<seg_grid(ctx, edges), 256, 0, st>>>(S.doff.as<int64_t>(), cnt, S.ids.as<int32_t>(),
                                                                      g.in_off.as<int64_t>(), g.in_src.as<int32_t>(),
                                                                      nullptr, S.csc.as<int32_t>(), edges);
        }
    }
    const unsigned gc = grid_for(cnt + 1, 256) > 4096 ? 4096 : grid_for(cnt + 1, 256);
    // bins
    PR_CUDA(cudaMemsetAsync(dcount.ptr, 0, 16, st));
    if (cnt)
        k_count_above<<<gc, 256, 0, st>>>(S.doff.as<int64_t>(), cnt, THREAD_DEG, HUB_DEG,
                                          dcount.as<unsigned long long>());
    unsigned long long above[2] = {0, 0};
    PR_CUDA(cudaMemcpyAsync(above, dcount.ptr, 16, cudaMemcpyDeviceToHost, st));
    PR_CUDA(cudaStreamSynchronize(st));
    S.n_hub = (int64_t)above[1];
    S.n_warp = (int64_t)above[0] - S.n_hub;
    DevBuf nch;
    DevBuf &cbase = S.chunk_base;
    PR_TRY(ensure(nch, 8 * (S.n_hub + 1)));
    PR_TRY(ensure(cbase, 8 * (S.n_hub + 1)));
    k_chunks_of<<<grid_for(S.n_hub + 1, 256), 256, 0, st>>>(S.doff.as<int64_t>(), S.n_hub, nch.as<int64_t>());
    PR_TRY(cub_run(ctx, [&](void *t, size_t &b) {
        return cub::DeviceScan::ExclusiveSum(t, b, nch.as<int64_t>(), cbase.as<int64_t>(), (int)(S.n_hub + 1), st);
    }));
    PR_CUDA(cudaMemcpyAsync(&S.n_chunks, cbase.as<int64_t>() + S.n_hub, 8, cudaMemcpyDeviceToHost, st));
    PR_CUDA(cudaStreamSynchronize(st));
    PR_TRY(ensure(S.chunk_part, 8 * (S.n_chunks + 1)));
    PR_TRY(ensure(S.row_cnt, 4 * (S.n_hub + 1)));
    PR_CUDA(cudaMemsetAsync(S.row_cnt.ptr, 0, 4 * (S.n_hub + 1), st));
    PR_TRY(sell_layout(ctx, S));
    // row cost prefix (unit sizing, ensure_units)
    DevBuf rcost;
    PR_TRY(ensure(rcost, 8 * (cnt + 1)));
    PR_TRY(ensure(S.row_cum, 8 * (cnt + 1)));
    k_row_cost<<<gc, 256, 0, st>>>(S.doff.as<int64_t>(), cnt, rcost.as<int64_t>());
    PR_TRY(cub_run(ctx, [&](void *t, size_t &b) {
        return cub::DeviceScan::ExclusiveSum(t, b, rcost.as<int64_t>(), S.row_cum.as<int64_t>(), (int)(cnt + 1), st);
    }));
    S.unit_blocks = 0;
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
    if (g.class0_end >= 0) {
        // run layout: seeds (in = 0, out > 0) are class 1, [class0_end, live_end)
        S.n_seed = g.live_end - g.class0_end;
        if (S.n_seed)
            k_iota<<<grid_for(S.n_seed, 256) > 4096 ? 4096 : grid_for(S.n_seed, 256), 256, 0, st>>>(
                S.seed_ids.as<int32_t>(), g.class0_end, S.n_seed);
        PR_CUDA(cudaStreamSynchronize(st));
    } else {
        PR_TRY(cub_run(ctx, [&](void *t, size_t &b) {
            return cub::DeviceSelect::If(t, b, first, S.seed_ids.as<int32_t>(), dcount.as<int64_t>(), (int)n,
                                         SeedPred{g.in_off.as<int64_t>(), g.out_deg.as<int32_t>()}, st);
        }));
        PR_CUDA(cudaMemcpyAsync(&S.n_seed, dcount.ptr, 8, cudaMemcpyDeviceToHost, st));
        PR_CUDA(cudaStreamSynchronize(st));
    }
    PR_CUDA(cudaGetLastError());
    S.built = true;
    return PR_OK;
}

}  // namespace pr
