// graph.cu -- device graph core: K1 (from_edges), K2 (classify + joint
// peel), K3 (dangling_target_counts, preprocess_ifp2), pull schedules and
// the R-MAT sampler.  Integer-only, bit-exact with the reference
// (graph.py:133-177, 274-318, 334-340, 343-378).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <cstring>

#include "internal.cuh"
#include "seg.cuh"
#include "cubutil.cuh"

namespace pr {

cudaStream_t &alloc_stream() {
    static thread_local cudaStream_t s = nullptr;
    return s;
}

int ensure(DevBuf &b, size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (b.bytes >= bytes) return PR_OK;
    b.release();
    cudaError_t e = cudaMallocAsync(&b.ptr, bytes, alloc_stream());
    if (e != cudaSuccess) {
        b.ptr = nullptr;
        cudaGetLastError();
        return fail(PR_ERR_NOMEM, "cudaMallocAsync(" + std::to_string(bytes) + " B) failed: " +
                                      cudaGetErrorString(e));
    }
    b.bytes = bytes;
    return PR_OK;
}

Graph::~Graph() { delete run; }


static int bit_width_u64(unsigned long long x) {
    int b = 0;
    while (x) { ++b; x >>= 1; }
    return b;
}


// ---------------------------------------------------------------- elementwise helpers

__global__ void k_degree(const int64_t *__restrict__ off, int64_t n, int32_t *__restrict__ deg) {
    GRID_STRIDE(v, n) deg[v] = (int32_t)(off[v + 1] - off[v]);
}

__global__ void k_narrow(const int64_t *__restrict__ in, int64_t count, int32_t *__restrict__ out) {
    GRID_STRIDE(i, count) out[i] = (int32_t)in[i];
}

__global__ void k_widen(const int32_t *__restrict__ in, int64_t count, int64_t *__restrict__ out) {
    GRID_STRIDE(i, count) out[i] = in[i];
}

__global__ void k_gather_i32(const int32_t *__restrict__ src, const int64_t *__restrict__ idx, int64_t count,
                             int32_t *__restrict__ out) {
    GRID_STRIDE(i, count) out[i] = src[idx[i]];
}

__global__ void k_gather_i64_pair(const int64_t *__restrict__ a, const int64_t *__restrict__ b,
                                  const int64_t *__restrict__ idx, int64_t count, int64_t *__restrict__ oa,
                                  int64_t *__restrict__ ob) {
    GRID_STRIDE(i, count) {
        int64_t j = idx[i];
        oa[i] = a[j];
        ob[i] = b[j];
    }
}

static unsigned gs_grid(Ctx &ctx, int64_t items) {
    int64_t b = (items + 255) / 256;
    int64_t cap = (int64_t)ctx.sm_count * 16;
    if (b > cap) b = cap;
    return (unsigned)(b < 1 ? 1 : b);
}

// ---------------------------------------------------------------- K1: from_edges

__global__ void k_edge_keys(const int64_t *__restrict__ src, const int64_t *__restrict__ dst, int64_t m, int64_t n,
                            unsigned long long *__restrict__ keys, int *__restrict__ bad) {
    GRID_STRIDE(i, m) {
        int64_t s = src[i], t = dst[i];
        if (s < 0 || t < 0 || s >= n || t >= n) { *bad = 1; s = 0; t = 0; }
        keys[i] = (unsigned long long)s * (unsigned long long)n + (unsigned long long)t;
    }
}

// sorted unique keys (row-major) -> column index + row offsets by boundary
// detection: off[v] = first position whose row >= v (no atomics, O(n+m)).
__global__ void k_split_keys(const unsigned long long *__restrict__ keys, int64_t m, int64_t n,
                             int32_t *__restrict__ col, int64_t *__restrict__ off) {
    GRID_STRIDE(e, m + 1) {
        int64_t row = e < m ? (int64_t)(keys[e] / (unsigned long long)n) : n;
        int64_t prev = e > 0 ? (int64_t)(keys[e - 1] / (unsigned long long)n) : -1;
        if (e < m) col[e] = (int32_t)(keys[e] % (unsigned long long)n);
        for (int64_t v = prev + 1; v <= row; ++v) off[v] = e;
    }
}

__global__ void k_transpose_keys(const unsigned long long *__restrict__ keys, int64_t m, int64_t n,
                                 unsigned long long *__restrict__ out) {
    GRID_STRIDE(e, m) {
        unsigned long long k = keys[e];
        unsigned long long s = k / (unsigned long long)n, t = k % (unsigned long long)n;
        out[e] = t * (unsigned long long)n + s;
    }
}

static int alloc_graph_arrays(Graph &g) {
    PR_TRY(ensure(g.out_off, sizeof(int64_t) * (g.n + 1)));
    PR_TRY(ensure(g.in_off, sizeof(int64_t) * (g.n + 1)));
    PR_TRY(ensure(g.out_deg, sizeof(int32_t) * g.n));
    if (g.has_csr) PR_TRY(ensure(g.out_tgt, sizeof(int32_t) * g.m));
    PR_TRY(ensure(g.in_src, sizeof(int32_t) * g.m));
    return PR_OK;
}

static int build_body(Ctx &ctx, Graph &g, const int64_t *d_src, const int64_t *d_dst, int64_t m_raw) {
    cudaStream_t st = ctx.stream;
    int64_t n = g.n;
    DevBuf keys, alt, flag, cnt;
    PR_TRY(ensure(keys, sizeof(unsigned long long) * m_raw));
    PR_TRY(ensure(alt, sizeof(unsigned long long) * m_raw));
    PR_TRY(ensure(flag, sizeof(int)));
    PR_TRY(ensure(cnt, sizeof(int64_t)));
    PR_CUDA(cudaMemsetAsync(flag.ptr, 0, sizeof(int), st));
    int64_t m = 0;
    int bits = bit_width_u64((unsigned long long)n * (unsigned long long)n - 1ull);
    if (bits < 1) bits = 1;
    unsigned long long *K = keys.as<unsigned long long>(), *A = alt.as<unsigned long long>();
    if (m_raw > 0) {
        k_edge_keys<<<gs_grid(ctx, m_raw), 256, 0, st>>>(d_src, d_dst, m_raw, n, K, flag.as<int>());
        int bad = 0;
        PR_CUDA(cudaMemcpyAsync(&bad, flag.ptr, sizeof(int), cudaMemcpyDeviceToHost, st));
        PR_CUDA(cudaStreamSynchronize(st));
        if (bad) return fail(PR_ERR_ARG, "vertex id out of range");
        // (src,dst) order + dedup == np.unique(src*n+dst) (graph.py:151-152)
        PR_TRY(cub_run(ctx, [&](void *t, size_t &b) {
            return cub::DeviceRadixSort::SortKeys(t, b, K, A, (int)m_raw, 0, bits, st);
        }));
        PR_TRY(cub_run(ctx, [&](void *t, size_t &b) {
            return cub::DeviceSelect::Unique(t, b, A, K, cnt.as<int64_t>(), (int)m_raw, st);
        }));
        PR_CUDA(cudaMemcpyAsync(&m, cnt.ptr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        PR_CUDA(cudaStreamSynchronize(st));
    }
    g.m = m;
    PR_TRY(alloc_graph_arrays(g));
    k_split_keys<<<gs_grid(ctx, m + 1), 256, 0, st>>>(K, m, n, g.out_tgt.as<int32_t>(), g.out_off.as<int64_t>());
    k_degree<<<gs_grid(ctx, n), 256, 0, st>>>(g.out_off.as<int64_t>(), n, g.out_deg.as<int32_t>());
    if (m > 0) {
        // CSC: full sort on (dst,src) == stable argsort(dst) of the (src,dst) order (graph.py:164)
        k_transpose_keys<<<gs_grid(ctx, m), 256, 0, st>>>(K, m, n, A);
        PR_TRY(cub_run(ctx, [&](void *t, size_t &b) {
            return cub::DeviceRadixSort::SortKeys(t, b, A, K, (int)m, 0, bits, st);
        }));
    }
    k_split_keys<<<gs_grid(ctx, m + 1), 256, 0, st>>>(K, m, n, g.in_src.as<int32_t>(), g.in_off.as<int64_t>());
    PR_CUDA(cudaStreamSynchronize(st));
    PR_CUDA(cudaGetLastError());
    return PR_OK;
}

int build_from_device_edges(Ctx &ctx, int64_t n, const int64_t *d_src, const int64_t *d_dst, int64_t m_raw,
                            Graph **out) {
    if (n < 1) return fail(PR_ERR_ARG, "graph must have at least one vertex");
    if (n > INT32_MAX - 1) return fail(PR_ERR_ARG, "n exceeds the int32 column-index range");
    if (m_raw > INT32_MAX) return fail(PR_ERR_ARG, "edge sample count exceeds 2^31-1");
    Graph *g = new Graph();
    g->ctx = &ctx;
    g->n = n;
    g->raw = m_raw;
    int rc = build_body(ctx, *g, d_src, d_dst, m_raw);
    if (rc) { delete g; return rc; }
    *out = g;
    return PR_OK;
}

// ---------------------------------------------------------------- K2: classify

__global__ void k_classify_init(const int32_t *__restrict__ out_deg, const int64_t *__restrict__ in_off, int64_t n,
                                uint8_t *__restrict__ flags, int32_t *__restrict__ cur_out,
                                int32_t *__restrict__ cur_in, uint8_t *__restrict__ alive,
                                int32_t *__restrict__ mark, int32_t *__restrict__ frontier,
                                unsigned long long *__restrict__ fsize, unsigned long long *__restrict__ m_d) {
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    unsigned long long md = 0;
    bool doomed = false;
    if (v < n) {
        int32_t od = out_deg[v];
        int32_t id = (int32_t)(in_off[v + 1] - in_off[v]);
        flags[v] = (uint8_t)((od == 0 ? 1 : 0) | (id == 0 ? 2 : 0));
        cur_out[v] = od;
        cur_in[v] = id;
        alive[v] = 1;
        mark[v] = 0;
        if (od == 0) md = (unsigned long long)id;  // graph.py:285
        doomed = od == 0 || id == 0;              // graph.py:293
    }
    // warp-aggregated frontier append
    unsigned ballot = __ballot_sync(0xffffffffu, doomed);
    int lane = threadIdx.x & 31;
    unsigned long long base = 0;
    if (lane == 0 && ballot) base = atomicAdd(fsize, (unsigned long long)__popc(ballot));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (doomed) frontier[base + __popc(ballot & ((1u << lane) - 1u))] = (int32_t)v;
    for (int o = 16; o > 0; o >>= 1) md += __shfl_down_sync(0xffffffffu, md, o);
    if (lane == 0 && md) atomicAdd(m_d, md);
}

__global__ void k_peel_kill(const int32_t *__restrict__ frontier, int64_t count, uint8_t *__restrict__ alive) {
    GRID_STRIDE(i, count) alive[frontier[i]] = 0;  // graph.py:296
}

__device__ __forceinline__ void peel_candidate(int32_t v, int32_t round, int32_t *mark, int32_t *next,
                                               unsigned long long *nsize) {
    if (atomicCAS(&mark[v], 0, round) == 0) next[atomicAdd(nsize, 1ull)] = v;
}

// warp per victim: decrement live neighbours' counters (graph.py:298-304);
// a counter reaching zero makes that vertex a candidate of the next round
__global__ void k_peel_decrement(const int32_t *__restrict__ frontier, int64_t count,
                                 const int64_t *__restrict__ out_off, const int32_t *__restrict__ out_tgt,
                                 const int64_t *__restrict__ in_off, const int32_t *__restrict__ in_src,
                                 const uint8_t *__restrict__ alive, int32_t *__restrict__ cur_out,
                                 int32_t *__restrict__ cur_in, int32_t *__restrict__ mark, int32_t round,
                                 int32_t *__restrict__ next, unsigned long long *__restrict__ nsize) {
    int lane = threadIdx.x & 31;
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp; i < count; i += nwarps) {
        int32_t v = frontier[i];
        for (int64_t e = out_off[v] + lane; e < out_off[v + 1]; e += 32) {
            int32_t t = out_tgt[e];
            if (alive[t] && atomicSub(&cur_in[t], 1) == 1) peel_candidate(t, round, mark, next, nsize);
        }
        for (int64_t e = in_off[v] + lane; e < in_off[v + 1]; e += 32) {
            int32_t s = in_src[e];
            if (alive[s] && atomicSub(&cur_out[s], 1) == 1) peel_candidate(s, round, mark, next, nsize);
        }
    }
}

// newly exposed vertices become weak (graph.py:306-310)
__global__ void k_peel_flag(const int32_t *__restrict__ next, int64_t count, const int32_t *__restrict__ cur_out,
                            const int32_t *__restrict__ cur_in, uint8_t *__restrict__ flags) {
    GRID_STRIDE(i, count) {
        int32_t v = next[i];
        uint8_t f = flags[v];
        if (cur_out[v] == 0 && !(f & 1)) f |= 4;
        if (cur_in[v] == 0 && !(f & 2)) f |= 8;
        flags[v] = f;
    }
}

struct BitSet {
    const uint8_t *flags;
    uint8_t bit;
    __host__ __device__ bool operator()(int32_t v) const { return (flags[v] & bit) != 0; }
};

// ascending id list of vertices whose flag has `bit` (np.flatnonzero order)
static int compact_flag(Ctx &ctx, const uint8_t *flags, uint8_t bit, int64_t n, int32_t *out, int64_t *d_count,
                        int64_t *h_count) {
    auto first = thrust::make_counting_iterator<int32_t>(0);
    PR_TRY(cub_run(ctx, [&](void *t, size_t &b) {
        return cub::DeviceSelect::If(t, b, first, out, d_count, (int)n, BitSet{flags, bit}, ctx.stream);
    }));
    if (h_count) {
        PR_CUDA(cudaMemcpyAsync(h_count, d_count, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx.stream));
        PR_CUDA(cudaStreamSynchronize(ctx.stream));
    }
    return PR_OK;
}

int classify_device(Graph &g) {
    if (g.classified) return PR_OK;
    PR_TRY(need_csr(g, "classify"));
    Ctx &ctx = *g.ctx;
    cudaStream_t st = ctx.stream;
    int64_t n = g.n;
    DevBuf cur_out, cur_in, alive, mark, fr0, fr1, sizes;
    PR_TRY(ensure(g.cls_flags, n));
    PR_TRY(ensure(cur_out, 4 * n));
    PR_TRY(ensure(cur_in, 4 * n));
    PR_TRY(ensure(alive, n));
    PR_TRY(ensure(mark, 4 * n));
    PR_TRY(ensure(fr0, 4 * n));
    PR_TRY(ensure(fr1, 4 * n));
    PR_TRY(ensure(sizes, 4 * sizeof(unsigned long long)));
    unsigned long long *dsz = sizes.as<unsigned long long>();
    PR_CUDA(cudaMemsetAsync(dsz, 0, 4 * sizeof(unsigned long long), st));
    k_classify_init<<<grid_for(n, 256), 256, 0, st>>>(g.out_deg.as<int32_t>(), g.in_off.as<int64_t>(), n,
                                                      g.cls_flags.as<uint8_t>(), cur_out.as<int32_t>(),
                                                      cur_in.as<int32_t>(), alive.as<uint8_t>(), mark.as<int32_t>(),
                                                      fr0.as<int32_t>(), dsz + 0, dsz + 2);
    unsigned long long hs[4];
    PR_CUDA(cudaMemcpyAsync(hs, dsz, sizeof(hs), cudaMemcpyDeviceToHost, st));
    PR_CUDA(cudaStreamSynchronize(st));
    int64_t count = (int64_t)hs[0];
    int64_t m_d = (int64_t)hs[2];
    int32_t *cur = fr0.as<int32_t>(), *nxt = fr1.as<int32_t>();
    int64_t rounds = 0;
    while (count > 0) {
        ++rounds;
        PR_CUDA(cudaMemsetAsync(dsz + 1, 0, sizeof(unsigned long long), st));
        k_peel_kill<<<gs_grid(ctx, count), 256, 0, st>>>(cur, count, alive.as<uint8_t>());
        k_peel_decrement<<<gs_grid(ctx, count * 32), 256, 0, st>>>(
            cur, count, g.out_off.as<int64_t>(), g.out_tgt.as<int32_t>(), g.in_off.as<int64_t>(),
            g.in_src.as<int32_t>(), alive.as<uint8_t>(), cur_out.as<int32_t>(), cur_in.as<int32_t>(),
            mark.as<int32_t>(), (int32_t)rounds, nxt, dsz + 1);
        unsigned long long nc = 0;
        PR_CUDA(cudaMemcpyAsync(&nc, dsz + 1, sizeof(nc), cudaMemcpyDeviceToHost, st));
        PR_CUDA(cudaStreamSynchronize(st));
        count = (int64_t)nc;
        if (count)
            k_peel_flag<<<gs_grid(ctx, count), 256, 0, st>>>(nxt, count, cur_out.as<int32_t>(), cur_in.as<int32_t>(),
                                                              g.cls_flags.as<uint8_t>());
        std::swap(cur, nxt);
    }
    PR_CUDA(cudaGetLastError());
    DevBuf tmp, dcount;
    PR_TRY(ensure(tmp, 4 * n));
    PR_TRY(ensure(dcount, sizeof(int64_t)));
    int64_t c[4];
    for (int k = 0; k < 4; ++k)
        PR_TRY(compact_flag(ctx, g.cls_flags.as<uint8_t>(), (uint8_t)(1 << k), n, tmp.as<int32_t>(),
                            dcount.as<int64_t>(), &c[k]));
    g.counts.dangling = c[0];
    g.counts.unreferenced = c[1];
    g.counts.weak_dangling = c[2];
    g.counts.weak_unreferenced = c[3];
    g.counts.dangling_edge_count = m_d;
    g.counts.peel_rounds = rounds;
    g.classified = true;
    return PR_OK;
}

int classify_export(Graph &g, int64_t *outs[4]) {
    PR_TRY(classify_device(g));
    Ctx &ctx = *g.ctx;
    DevBuf tmp, wide, dcount;
    PR_TRY(ensure(tmp, 4 * g.n));
    PR_TRY(ensure(wide, 8 * g.n));
    PR_TRY(ensure(dcount, sizeof(int64_t)));
    for (int k = 0; k < 4; ++k) {
        if (!outs[k]) continue;
        int64_t cnt = 0;
        PR_TRY(compact_flag(ctx, g.cls_flags.as<uint8_t>(), (uint8_t)(1 << k), g.n, tmp.as<int32_t>(),
                            dcount.as<int64_t>(), &cnt));
        if (cnt) {
            k_widen<<<gs_grid(ctx, cnt), 256, 0, ctx.stream>>>(tmp.as<int32_t>(), cnt, wide.as<int64_t>());
            PR_CUDA(cudaMemcpyAsync(outs[k], wide.ptr, 8 * cnt, cudaMemcpyDeviceToHost, ctx.stream));
            PR_CUDA(cudaStreamSynchronize(ctx.stream));
        }
    }
    return PR_OK;
}

// ---------------------------------------------------------------- K3

// graph.py:334-340: per-row count of dangling targets
// dtc[u] = #(out-neighbours of u with out-degree 0), counted from the CSC:
// every in-edge (u -> v) of a dangling v adds one to dtc[u].  Edge-parallel
// and load-balanced (the row of an edge by binary search inside the block's
// tile, as in k_seg_gather), so hub rows cost what short rows cost, and the
// out-adjacency is not needed.
__global__ void __launch_bounds__(256) k_dtc_csc(const int64_t *__restrict__ in_off, const int32_t *__restrict__ in_src,
                                                 const int32_t *__restrict__ out_deg, int64_t n, int64_t m,
                                                 int32_t *__restrict__ dtc) {
    __shared__ int64_t s_r0, s_r1;
    for (int64_t base = blockIdx.x * (int64_t)SEG_TILE; base < m; base += (int64_t)gridDim.x * SEG_TILE) {
        const int64_t end = base + SEG_TILE < m ? base + SEG_TILE : m;
        if (threadIdx.x == 0) s_r0 = seg_upper(in_off, 0, n + 1, base) - 1;
        if (threadIdx.x == 32) s_r1 = seg_upper(in_off, 0, n + 1, end - 1);
        __syncthreads();
        const int64_t r0 = s_r0, r1 = s_r1;
        for (int64_t e = base + threadIdx.x; e < end; e += blockDim.x) {
            const int64_t v = seg_upper(in_off, r0, r1 + 1, e) - 1;
            if (__ldg(&out_deg[v]) == 0) atomicAdd(&dtc[__ldg(&in_src[e])], 1);
        }
        __syncthreads();
    }
}

// run layout: the in-edges of the dangling tail [live_end, n) are the CSC
// suffix, so dtc is a histogram of their sources (edge-parallel, balanced)
__global__ void k_dtc_tail(const int64_t *__restrict__ in_off, const int32_t *__restrict__ in_src, int64_t live_end,
                           int64_t n, int32_t *__restrict__ dtc) {
    const int64_t lo = in_off[live_end], hi = in_off[n];
    for (int64_t e = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < hi; e += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&dtc[__ldg(&in_src[e])], 1);
}

int ensure_dtc(Graph &g) {
    if (g.has_dtc) return PR_OK;
    PR_TRY(ensure(g.dtc, 4 * g.n));
    if (g.live_end >= 0) {
        PR_CUDA(cudaMemsetAsync(g.dtc.ptr, 0, 4 * g.n, g.ctx->stream));
        if (g.live_end < g.n)
            k_dtc_tail<<<gs_grid(*g.ctx, g.m), 256, 0, g.ctx->stream>>>(g.in_off.as<int64_t>(), g.in_src.as<int32_t>(),
                                                                      g.live_end, g.n, g.dtc.as<int32_t>());
        PR_CUDA(cudaGetLastError());
        g.has_dtc = true;
        return PR_OK;
    }
    PR_CUDA(cudaMemsetAsync(g.dtc.ptr, 0, 4 * g.n, g.ctx->stream));
    if (g.m)
        k_dtc_csc<<<seg_grid(*g.ctx, g.m), 256, 0, g.ctx->stream>>>(g.in_off.as<int64_t>(), g.in_src.as<int32_t>(),
                                                                   g.out_deg.as<int32_t>(), g.n, g.m,
                                                                   g.dtc.as<int32_t>());
    PR_CUDA(cudaGetLastError());
    g.has_dtc = true;
    return PR_OK;
}

struct LiveEdge {
    const int32_t *tgt, *deg;
    __host__ __device__ bool operator()(int64_t e) const { return deg[tgt[e]] > 0; }
};
struct IsDangling {
    const int32_t *deg;
    __host__ __device__ bool operator()(int32_t v) const { return deg[v] == 0; }
};

__global__ void k_live_degree(const int32_t *__restrict__ out_deg, const int32_t *__restrict__ dtc, int64_t n,
                              int64_t *__restrict__ live_deg64, int32_t *__restrict__ live_deg) {
    GRID_STRIDE(v, n) {
        int32_t d = out_deg[v] - dtc[v];
        live_deg[v] = d;
        live_deg64[v] = d;
    }
}

__global__ void k_gather_count(const int32_t *__restrict__ ids, int64_t count, const int64_t *__restrict__ in_off,
                               int64_t *__restrict__ cnt) {
    GRID_STRIDE(i, count) {
        int32_t d = ids[i];
        cnt[i] = in_off[d + 1] - in_off[d];
    }
}

// _gather_rows(in_offsets, in_sources, dangling_ids) (graph.py:262-271, 367): k_seg_gather<false>

__global__ void k_tail_rows(const int64_t *__restrict__ in_off, int64_t live_end, int64_t nd,
                            int32_t *__restrict__ ids, int64_t *__restrict__ off) {
    GRID_STRIDE(i, nd + 1) {
        if (i < nd) ids[i] = (int32_t)(live_end + i);
        off[i] = in_off[live_end + i] - in_off[live_end];
    }
}

static int sort_by_source(Ctx &ctx, const DevBuf &in_off, const DevBuf &in_src, int64_t rows, int64_t m_e,
                          int64_t n, DevBuf &out_tgt);

int preprocess_ifp2_device(Graph &g) {
    if (g.has_ifp2) return PR_OK;
    if (g.live_end < 0) PR_TRY(need_csr(g, "the IFP2 live CSR"));
    Ctx &ctx = *g.ctx;
    cudaStream_t st = ctx.stream;
    int64_t n = g.n, m = g.m;
    PR_TRY(ensure_dtc(g));
    DevBuf deg64, dcount;
    PR_TRY(ensure(deg64, 8 * (n + 1)));
    PR_TRY(ensure(dcount, sizeof(int64_t)));
    PR_TRY(ensure(g.live_deg, 4 * n));
    PR_TRY(ensure(g.live_off, 8 * (n + 1)));
    k_live_degree<<<gs_grid(ctx, n), 256, 0, st>>>(g.out_deg.as<int32_t>(), g.dtc.as<int32_t>(), n,
                                                   deg64.as<int64_t>(), g.live_deg.as<int32_t>());
    PR_CUDA(cudaMemsetAsync(deg64.as<int64_t>() + n, 0, 8, st));
    PR_TRY(cub_run(ctx, [&](void *t, size_t &b) {
        return cub::DeviceScan::ExclusiveSum(t, b, deg64.as<int64_t>(), g.live_off.as<int64_t>(), (int)(n + 1), st);
    }));
    // live_targets: stable compaction keeps each row's target order (graph.py:353-354)
    int64_t live_m = 0;
    if (g.live_end >= 0) {
        // run layout: the live edges are the CSC rows of the non-dangling
        // prefix [0, live_end); sorted by source they are the live CSR
        PR_CUDA(cudaMemcpyAsync(&live_m, g.in_off.as<int64_t>() + g.live_end, 8, cudaMemcpyDeviceToHost, st));
        PR_CUDA(cudaStreamSynchronize(st));
        PR_TRY(sort_by_source(ctx, g.in_off, g.in_src, g.live_end, live_m, n, g.live_tgt));
    } else if (m) {
        PR_TRY(ensure(g.live_tgt, 4 * m));
        auto first = thrust::make_counting_iterator<int64_t>(0);
        DevBuf eids;
        PR_TRY(ensure(eids, 8 * m));
        PR_TRY(cub_run(ctx, [&](void *t, size_t &b) {
            return cub::DeviceSelect::If(t, b, first, eids.as<int64_t>(), dcount.as<int64_t>(), m,
                                         LiveEdge{g.out_tgt.as<int32_t>(), g.out_deg.as<int32_t>()}, st);
        }));
        PR_CUDA(cudaMemcpyAsync(&live_m, dcount.ptr, 8, cudaMemcpyDeviceToHost, st));
        PR_CUDA(cudaStreamSynchronize(st));
        if (live_m)
            k_gather_i32<<<gs_grid(ctx, live_m), 256, 0, st>>>(g.out_tgt.as<int32_t>(), eids.as<int64_t>(), live_m,
                                                               g.live_tgt.as<int32_t>());
    }
    if (!g.live_tgt.ptr) PR_TRY(ensure(g.live_tgt, 4));
    // dangling ids (ascending) and their source CSR (graph.py:363-367)
    int64_t nd = 0, md = 0;
    if (g.live_end >= 0) {
        // run layout: the dangling vertices are the id tail and their
        // source rows the CSC suffix -- slices, no selection or gather
        nd = n - g.live_end;
        int64_t base = m;
        if (nd) {
            PR_CUDA(cudaMemcpyAsync(&base, g.in_off.as<int64_t>() + g.live_end, 8, cudaMemcpyDeviceToHost, st));
            PR_CUDA(cudaStreamSynchronize(st));
        }
        md = m - base;
        PR_TRY(ensure(g.dang_ids, 4 * (nd ? nd : 1)));
        PR_TRY(ensure(g.src_off, 8 * (nd + 1)));
        PR_TRY(ensure(g.src_ids, 4 * (md ? md : 1)));
        k_tail_rows<<<gs_grid(ctx, nd + 1), 256, 0, st>>>(g.in_off.as<int64_t>(), g.live_end, nd,
                                                          g.dang_ids.as<int32_t>(), g.src_off.as<int64_t>());
        if (md)
            PR_CUDA(cudaMemcpyAsync(g.src_ids.ptr, g.in_src.as<int32_t>() + base, 4 * md, cudaMemcpyDeviceToDevice,
                                    st));
    } else {
        PR_TRY(ensure(g.dang_ids, 4 * n));
        auto vfirst = thrust::make_counting_iterator<int32_t>(0);
        PR_TRY(cub_run(ctx, [&](void *t, size_t &b) {
            return cub::DeviceSelect::If(t, b, vfirst, g.dang_ids.as<int32_t>(), dcount.as<int64_t>(), (int)n,
                                         IsDangling{g.out_deg.as<int32_t>()}, st);
        }));
        PR_CUDA(cudaMemcpyAsync(&nd, dcount.ptr, 8, cudaMemcpyDeviceToHost, st));
        PR_CUDA(cudaStreamSynchronize(st));
        PR_TRY(ensure(g.src_off, 8 * (nd + 1)));
        DevBuf cnt;
        PR_TRY(ensure(cnt, 8 * (nd + 1)));
        PR_CUDA(cudaMemsetAsync(cnt.ptr, 0, 8 * (nd + 1), st));
        if (nd)
            k_gather_count<<<gs_grid(ctx, nd), 256, 0, st>>>(g.dang_ids.as<int32_t>(), nd, g.in_off.as<int64_t>(),
                                                             cnt.as<int64_t>());
        PR_TRY(cub_run(ctx, [&](void *t, size_t &b) {
            return cub::DeviceScan::ExclusiveSum(t, b, cnt.as<int64_t>(), g.src_off.as<int64_t>(), (int)(nd + 1), st);
        }));
        PR_CUDA(cudaMemcpyAsync(&md, g.src_off.as<int64_t>() + nd, 8, cudaMemcpyDeviceToHost, st));
        PR_CUDA(cudaStreamSynchronize(st));
        PR_TRY(ensure(g.src_ids, 4 * (md ? md : 1)));
        if (md)
            k_seg_gather<false><<<seg_grid(ctx, md), 256, 0, st>>>(g.src_off.as<int64_t>(), nd,
                                                                   g.dang_ids.as<int32_t>(), g.in_off.as<int64_t>(),
                                                                   g.in_src.as<int32_t>(), nullptr,
                                                                   g.src_ids.as<int32_t>(), md);
        PR_CUDA(cudaStreamSynchronize(st));
        PR_CUDA(cudaGetLastError());
    }
    g.ifp2.live_edges = live_m;
    g.ifp2.dangling = nd;
    g.ifp2.source_edges = md;
    g.has_ifp2 = true;
    return PR_OK;
}

// IFP2Graph's three counts without building the split (graph.py:343-378):
// dangling = #(deg == 0), source_edges = m_d = the dangling vertices'
// in-degree sum, live_edges = m - m_d (every edge into a dangling vertex is
// dead).  The fast engines build their split on the run layout; the
// original-layout arrays are built only when exported or run in exact mode.
__global__ void k_ifp2_counts(const int32_t *__restrict__ out_deg, const int64_t *__restrict__ in_off, int64_t n,
                              unsigned long long *acc) {
    unsigned long long nd = 0, md = 0;
    GRID_STRIDE(v, n) {
        if (out_deg[v] == 0) {
            nd += 1;
            md += (unsigned long long)(in_off[v + 1] - in_off[v]);
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        nd += __shfl_xor_sync(0xffffffffu, nd, o);
        md += __shfl_xor_sync(0xffffffffu, md, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (nd) atomicAdd(acc, nd);
        if (md) atomicAdd(acc + 1, md);
    }
}

int ifp2_counts_device(Graph &g) {
    if (g.has_ifp2 || g.ifp2_counted) return PR_OK;
    Ctx &ctx = *g.ctx;
    cudaStream_t st = ctx.stream;
    DevBuf acc;
    PR_TRY(ensure(acc, 2 * sizeof(unsigned long long)));
    PR_CUDA(cudaMemsetAsync(acc.ptr, 0, 2 * sizeof(unsigned long long), st));
    if (g.n)
        k_ifp2_counts<<<gs_grid(ctx, g.n), 256, 0, st>>>(g.out_deg.as<int32_t>(), g.in_off.as<int64_t>(), g.n,
                                                         acc.as<unsigned long long>());
    unsigned long long h[2] = {0, 0};
    PR_CUDA(cudaMemcpyAsync(h, acc.ptr, sizeof(h), cudaMemcpyDeviceToHost, st));
    PR_CUDA(cudaStreamSynchronize(st));
    g.ifp2.dangling = (int64_t)h[0];
    g.ifp2.source_edges = (int64_t)h[1];
    g.ifp2.live_edges = g.m - (int64_t)h[1];
    g.n_dangling = (int64_t)h[0];
    g.ifp2_counted = true;
    return PR_OK;
}

// ---------------------------------------------------------------- run layout

// sort key: class (2 bits) | descending in-degree (clipped to 30 bits)
// inside the receiving classes 0 and 2; a stable sort of (key, id) pairs
// keeps ascending ids inside equal keys
__global__ void k_relabel_keys(const int64_t *__restrict__ out_off, const int64_t *__restrict__ in_off, int64_t n,
                               uint32_t *__restrict__ keys, int32_t *__restrict__ ids) {
    GRID_STRIDE(v, n) {
        int64_t od = out_off[v + 1] - out_off[v], id = in_off[v + 1] - in_off[v];
        uint32_t cls = od > 0 ? (id > 0 ? 0u : 1u) : (id > 0 ? 2u : 3u);
        if (id > 0x3FFFFFFF) id = 0x3FFFFFFF;
        uint32_t dk = (cls == 0 || cls == 2) ? (uint32_t)(0x3FFFFFFF - id) : 0u;
        keys[v] = (cls << 30) | dk;
        ids[v] = (int32_t)v;
    }
}

// rank = inverse permutation; bounds[k] = first run id of class > k
// (bounds[0] = end of class 0, bounds[1] = live_end, the dangling tail)
__global__ void k_rank_from_perm(const uint32_t *__restrict__ keys, const int32_t *__restrict__ perm, int64_t n,
                                 int32_t *__restrict__ rank, int64_t *__restrict__ bounds) {
    GRID_STRIDE(i, n) {
        rank[perm[i]] = (int32_t)i;
        const uint32_t c = keys[i] >> 30, p = i > 0 ? keys[i - 1] >> 30 : 0u;
        if (c >= 1 && (i == 0 || p < 1)) bounds[0] = i;
        if (c >= 2 && (i == 0 || p < 2)) bounds[1] = i;
    }
}

// degree of new row i = degree of old row perm[i]
__global__ void k_perm_len(const int64_t *__restrict__ off, const int32_t *__restrict__ perm, int64_t n,
                           int64_t *__restrict__ len) {
    GRID_STRIDE(i, n + 1) {
        if (i == n) { len[n] = 0; continue; }
        int32_t v = perm[i];
        len[i] = off[v + 1] - off[v];
    }
}

// Permuted copy of one adjacency direction (no sort: a relabelling only
// moves rows and renames columns; row-internal order is irrelevant to the
// fast engines, whose summation order is fixed by their own schedule).
static int permute_adjacency(Ctx &ctx, const DevBuf &off, const DevBuf &col, const DevBuf &perm, const DevBuf &rank,
                             int64_t n, int64_t m, DevBuf &noff, DevBuf &ncol) {
    cudaStream_t st = ctx.stream;
    DevBuf len;
    PR_TRY(ensure(len, 8 * (n + 1)));
    PR_TRY(ensure(noff, 8 * (n + 1)));
    PR_TRY(ensure(ncol, 4 * (m ? m : 1)));
    k_perm_len<<<gs_grid(ctx, n + 1), 256, 0, st>>>(off.as<int64_t>(), perm.as<int32_t>(), n, len.as<int64_t>());
    PR_TRY(cub_run(ctx, [&](void *t, size_t &b) {
        return cub::DeviceScan::ExclusiveSum(t, b, len.as<int64_t>(), noff.as<int64_t>(), (int)(n + 1), st);
    }));
    if (m)
        k_seg_gather<true><<<seg_grid(ctx, m), 256, 0, st>>>(noff.as<int64_t>(), n, perm.as<int32_t>(),
                                                             off.as<int64_t>(), col.as<int32_t>(), rank.as<int32_t>(),
                                                             ncol.as<int32_t>(), m);
    return PR_OK;
}

// row id of every edge of a CSR/CSC (load-balanced, as k_seg_gather)
__global__ void __launch_bounds__(256) k_edge_rows(const int64_t *__restrict__ off, int64_t rows, int64_t m,
                                                   int32_t *__restrict__ row_of) {
    __shared__ int64_t s_r0, s_r1;
    for (int64_t base = blockIdx.x * (int64_t)SEG_TILE; base < m; base += (int64_t)gridDim.x * SEG_TILE) {
        const int64_t end = base + SEG_TILE < m ? base + SEG_TILE : m;
        if (threadIdx.x == 0) s_r0 = seg_upper(off, 0, rows + 1, base) - 1;
        if (threadIdx.x == 32) s_r1 = seg_upper(off, 0, rows + 1, end - 1);
        __syncthreads();
        const int64_t r0 = s_r0, r1 = s_r1;
        for (int64_t e = base + threadIdx.x; e < end; e += blockDim.x)
            row_of[e] = (int32_t)(seg_upper(off, r0, r1 + 1, e) - 1);
        __syncthreads();
    }
}

// Out-adjacency from in-adjacency: a stable sort of the (source, destination)
// pairs of the first m_e CSC edges (rows [0, rows)) by source.  Destinations
// come out ascending inside every row, so the result is deterministic.  The
// caller provides the out-offsets (the per-source counts of those edges).
static int sort_by_source(Ctx &ctx, const DevBuf &in_off, const DevBuf &in_src, int64_t rows, int64_t m_e,
                          int64_t n, DevBuf &out_tgt) {
    cudaStream_t st = ctx.stream;
    PR_TRY(ensure(out_tgt, 4 * (m_e ? m_e : 1)));
    if (!m_e) return PR_OK;
    DevBuf keys_out, row_of;
    PR_TRY(ensure(keys_out, 4 * m_e));
    PR_TRY(ensure(row_of, 4 * m_e));
    k_edge_rows<<<seg_grid(ctx, m_e), 256, 0, st>>>(in_off.as<int64_t>(), rows, m_e, row_of.as<int32_t>());
    int bits = 1;
    while (bits < 31 && ((int64_t)1 << bits) < n) ++bits;
    PR_TRY(cub_run(ctx, [&](void *t, size_t &b) {
        return cub::DeviceRadixSort::SortPairs(t, b, (const uint32_t *)in_src.ptr, keys_out.as<uint32_t>(),
                                               row_of.as<int32_t>(), out_tgt.as<int32_t>(), m_e, 0, bits, st);
    }));
    return PR_OK;
}

// The run layout's full out-adjacency, built on first use (IFP1's push
// rounds): permuted from the original when that has one, else sorted out of
// the run layout's CSC.  IFP2 never needs it (its live CSR comes from the
// CSC prefix, preprocess_ifp2_device).
int ensure_run_csr(Graph &r) {
    if (r.has_csr) return PR_OK;
    Ctx &ctx = *r.ctx;
    Graph &g = *r.orig;
    if (g.has_csr)
        PR_TRY(permute_adjacency(ctx, g.out_off, g.out_tgt, g.perm, g.rank, r.n, r.m, r.out_off, r.out_tgt));
    else
        PR_TRY(sort_by_source(ctx, r.in_off, r.in_src, r.n, r.m, r.n, r.out_tgt));
    PR_CUDA(cudaGetLastError());
    r.has_csr = true;
    return PR_OK;
}

int need_csr(const Graph &g, const char *what) {
    if (g.has_csr) return PR_OK;
    return fail(PR_ERR_STATE, std::string(what) +
                                  " needs the out-adjacency; the graph was uploaded without out_targets "
                                  "(pr_graph_attach_out_targets)");
}

int attach_out_targets(Graph &g, const int64_t *out_tgt) {
    if (g.has_csr) return PR_OK;
    Ctx &ctx = *g.ctx;
    cudaStream_t st = ctx.stream;
    PR_TRY(ensure(g.out_tgt, 4 * (g.m ? g.m : 1)));
    if (g.m) {
        PR_TRY(upload_narrow(ctx, out_tgt, g.m, g.out_tgt.as<int32_t>(), &g.h2d_bytes));
        PR_CUDA(cudaStreamSynchronize(st));
        PR_CUDA(cudaGetLastError());
    }
    g.has_csr = true;
    return PR_OK;
}

int ensure_run_layout(Graph &g) {
    if (g.run) return PR_OK;
    Ctx &ctx = *g.ctx;
    cudaStream_t st = ctx.stream;
    int64_t n = g.n, m = g.m;
    DevBuf keys, sorted, ids, dl;
    PR_TRY(ensure(keys, 4 * n));
    PR_TRY(ensure(sorted, 4 * n));
    PR_TRY(ensure(ids, 4 * n));
    PR_TRY(ensure(dl, 16));
    PR_TRY(ensure(g.perm, 4 * n));
    PR_TRY(ensure(g.rank, 4 * n));
    k_relabel_keys<<<gs_grid(ctx, n), 256, 0, st>>>(g.out_off.as<int64_t>(), g.in_off.as<int64_t>(), n,
                                                   keys.as<uint32_t>(), ids.as<int32_t>());
    PR_TRY(cub_run(ctx, [&](void *t, size_t &b) {
        return cub::DeviceRadixSort::SortPairs(t, b, keys.as<uint32_t>(), sorted.as<uint32_t>(), ids.as<int32_t>(),
                                               g.perm.as<int32_t>(), (int)n, 0, 32, st);
    }));
    const int64_t none[2] = {n, n};
    PR_CUDA(cudaMemcpyAsync(dl.ptr, none, 16, cudaMemcpyHostToDevice, st));
    k_rank_from_perm<<<gs_grid(ctx, n), 256, 0, st>>>(sorted.as<uint32_t>(), g.perm.as<int32_t>(), n,
                                                      g.rank.as<int32_t>(), dl.as<int64_t>());
    Graph *r = new Graph();
    r->ctx = &ctx;
    r->n = n;
    r->m = m;
    r->raw = g.raw;
    r->orig = &g;
    r->has_csr = false;       // out_tgt on demand (ensure_run_csr)
    int rc = permute_adjacency(ctx, g.in_off, g.in_src, g.perm, g.rank, n, m, r->in_off, r->in_src);
    // Sources of every row ascending in run ids, so the hot (low-id) sources
    // of a warp or hub row sit next to each other and neighbouring lanes
    // share 128-byte lines.  Measured: solve C5 -4% (-6% with 16-lane
    // sub-warp rows), C2 -0.9%, C3/C4 0; the segmented sort adds 0.7 ms (C2)
    // / 7.5 ms (C3) to a fresh graph's preprocessing.  So it runs only where
    // the rounds are HBM-bound: a round working set past 16x L2 (C5), as for
    // 4 Gauss-Seidel sections.  PUSHRANK_SORT_ROWS=0/1 forces it.
    {
        const double l2 = (double)(ctx.l2_bytes ? ctx.l2_bytes : (size_t)126 << 20);
        bool sort_rows = 4.0 * (double)m + 8.0 * (double)n > 16.0 * l2;
        // PUSHRANK_SORT_ROWS=0/1 forces it off / on now; by default it waits
        // for the graph's second fast solve (run_rounds)
        if (const char *e = getenv("PUSHRANK_SORT_ROWS")) {
            if (!rc && atoi(e) != 0) rc = sort_csc_rows(ctx, r->in_off, r->in_src, n, m);
        } else {
            r->sort_deferred = sort_rows;
        }
    }
    DevBuf len;
    if (!rc) rc = ensure(len, 8 * (n + 1));
    if (!rc) rc = ensure(r->out_off, 8 * (n + 1));
    if (!rc) {
        k_perm_len<<<gs_grid(ctx, n + 1), 256, 0, st>>>(g.out_off.as<int64_t>(), g.perm.as<int32_t>(), n,
                                                        len.as<int64_t>());
        rc = cub_run(ctx, [&](void *t, size_t &b) {
            return cub::DeviceScan::ExclusiveSum(t, b, len.as<int64_t>(), r->out_off.as<int64_t>(), (int)(n + 1), st);
        });
    }
    if (!rc) rc = ensure(r->out_deg, 4 * n);
    if (!rc) k_degree<<<gs_grid(ctx, n), 256, 0, st>>>(r->out_off.as<int64_t>(), n, r->out_deg.as<int32_t>());
    int64_t bounds[2] = {n, n};
    if (!rc && cudaMemcpyAsync(bounds, dl.ptr, 16, cudaMemcpyDeviceToHost, st) != cudaSuccess)
        rc = fail(PR_ERR_CUDA, "run layout build failed");
    if (!rc && (cudaStreamSynchronize(st) != cudaSuccess || cudaGetLastError() != cudaSuccess))
        rc = fail(PR_ERR_CUDA, "run layout build failed");
    if (rc) { delete r; return rc; }
    r->class0_end = bounds[0];
    r->live_end = bounds[1];
    r->n_dangling = n - bounds[1];
    g.run = r;
    return PR_OK;
}

int sort_csc_rows(Ctx &ctx, const DevBuf &in_off, DevBuf &in_src, int64_t n, int64_t m) {
    if (m <= 0 || n <= 0) return PR_OK;
    cudaStream_t st = ctx.stream;
    DevBuf alt;
    PR_TRY(ensure(alt, 4 * m));
    cub::DoubleBuffer<int32_t> keys(in_src.as<int32_t>(), alt.as<int32_t>());
    const int64_t *off = in_off.as<int64_t>();
    PR_TRY(cub_run(ctx, [&](void *t, size_t &b) {
        return cub::DeviceSegmentedSort::SortKeys(t, b, keys, (int)m, (int)n, off, off + 1, st);
    }));
    if (keys.Current() != in_src.as<int32_t>())
        PR_CUDA(cudaMemcpyAsync(in_src.ptr, keys.Current(), 4 * m, cudaMemcpyDeviceToDevice, st));
    PR_CUDA(cudaStreamSynchronize(st));
    return PR_OK;
}

int count_dangling(Graph &g) {
    if (g.n_dangling >= 0) return PR_OK;
    Ctx &ctx = *g.ctx;
    DevBuf tmp, dcount;
    PR_TRY(ensure(tmp, 4 * g.n));
    PR_TRY(ensure(dcount, 8));
    auto first = thrust::make_counting_iterator<int32_t>(0);
    PR_TRY(cub_run(ctx, [&](void *t, size_t &b) {
        return cub::DeviceSelect::If(t, b, first, tmp.as<int32_t>(), dcount.as<int64_t>(), (int)g.n,
                                     IsDangling{g.out_deg.as<int32_t>()}, ctx.stream);
    }));
    int64_t c = 0;
    PR_CUDA(cudaMemcpyAsync(&c, dcount.ptr, 8, cudaMemcpyDeviceToHost, ctx.stream));
    PR_CUDA(cudaStreamSynchronize(ctx.stream));
    g.n_dangling = c;
    return PR_OK;
}

// ---------------------------------------------------------------- R-MAT sampler

__host__ __device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// identical integer arithmetic to synthetic.rmat_edges
__global__ void k_rmat(int scale, unsigned long long key0, unsigned long long ta, unsigned long long tb,
                       unsigned long long tc, int64_t first, int64_t count, int64_t *__restrict__ src,
                       int64_t *__restrict__ dst) {
    const unsigned long long G = 0x9E3779B97F4A7C15ull;
    GRID_STRIDE(i, count) {
        unsigned long long base = key0 + (unsigned long long)(first + i) * 64ull * G;
        unsigned long long s = 0, d = 0;
        for (int l = 0; l < scale; ++l) {
            unsigned long long u = mix64(base + (unsigned long long)l * G) >> 32;
            unsigned long long sb = u >= tb;
            unsigned long long db = (u >= ta && u < tb) || u >= tc;
            s = (s << 1) | sb;
            d = (d << 1) | db;
        }
        src[i] = (int64_t)s;
        dst[i] = (int64_t)d;
    }
}

int rmat_generate(Ctx &ctx, int scale, double a, double b, double c, uint64_t seed, int64_t first, int64_t count,
                  int64_t *d_src, int64_t *d_dst) {
    if (scale < 1 || scale > 30) return fail(PR_ERR_ARG, "rmat scale must be in [1, 30]");
    const double S = 4294967296.0;
    unsigned long long ta = (unsigned long long)(a * S), tb = (unsigned long long)((a + b) * S),
                       tc = (unsigned long long)((a + b + c) * S);
    unsigned long long key0 = mix64((unsigned long long)seed);
    if (count > 0)
        k_rmat<<<gs_grid(ctx, count), 256, 0, ctx.stream>>>(scale, key0, ta, tb, tc, first, count, d_src, d_dst);
    PR_CUDA(cudaGetLastError());
    return PR_OK;
}

struct NotLoop {
    const int64_t *s, *d;
    __host__ __device__ bool operator()(int64_t i) const { return s[i] != d[i]; }
};

int graph_rmat(Ctx &ctx, int scale, int64_t ef, double a, double b, double c, uint64_t seed, Graph **out) {
    if (scale < 1 || scale > 30) return fail(PR_ERR_ARG, "rmat scale must be in [1, 30]");
    int64_t n = 1ll << scale, count = ef * n;
    DevBuf src, dst, keep, cnt, s2, d2;
    PR_TRY(ensure(src, 8 * count));
    PR_TRY(ensure(dst, 8 * count));
    PR_TRY(rmat_generate(ctx, scale, a, b, c, seed, 0, count, src.as<int64_t>(), dst.as<int64_t>()));
    // drop self-loops (BASELINE configs: "duplicates and self-loops removed")
    PR_TRY(ensure(keep, 8 * count));
    PR_TRY(ensure(cnt, 8));
    auto first = thrust::make_counting_iterator<int64_t>(0);
    PR_TRY(cub_run(ctx, [&](void *t, size_t &bb) {
        return cub::DeviceSelect::If(t, bb, first, keep.as<int64_t>(), cnt.as<int64_t>(), count,
                                     NotLoop{src.as<int64_t>(), dst.as<int64_t>()}, ctx.stream);
    }));
    int64_t kept = 0;
    PR_CUDA(cudaMemcpyAsync(&kept, cnt.ptr, 8, cudaMemcpyDeviceToHost, ctx.stream));
    PR_CUDA(cudaStreamSynchronize(ctx.stream));
    PR_TRY(ensure(s2, 8 * kept));
    PR_TRY(ensure(d2, 8 * kept));
    k_gather_i64_pair<<<gs_grid(ctx, kept), 256, 0, ctx.stream>>>(src.as<int64_t>(), dst.as<int64_t>(),
                                                                  keep.as<int64_t>(), kept, s2.as<int64_t>(),
                                                                  d2.as<int64_t>());
    PR_CUDA(cudaStreamSynchronize(ctx.stream));
    src.release();
    dst.release();
    keep.release();
    return build_from_device_edges(ctx, n, s2.as<int64_t>(), d2.as<int64_t>(), kept, out);
}

// ---------------------------------------------------------------- upload / export

int upload_graph(Ctx &ctx, int64_t n, int64_t m, const int64_t *out_off, const int64_t *out_tgt,
                 const int64_t *in_off, const int64_t *in_src, Graph **out) {
    if (n < 1) return fail(PR_ERR_ARG, "graph must have at least one vertex");
    if (n > INT32_MAX - 1) return fail(PR_ERR_ARG, "n exceeds the int32 column-index range");
    if (out_off[0] != 0 || out_off[n] != m || in_off[0] != 0 || in_off[n] != m)
        return fail(PR_ERR_ARG, "offsets inconsistent with n/m");
    cudaStream_t st = ctx.stream;
    Graph *g = new Graph();
    g->ctx = &ctx;
    g->n = n;
    g->m = m;
    g->raw = m;
    g->has_csr = out_tgt != nullptr || m == 0;
    int rc = alloc_graph_arrays(*g);
    if (!rc) {
        // the offsets travel on the copy lane of the index upload (hostio.cu)
        // while the host threads narrow the indices
        const RawCopy offs[2] = {{g->out_off.ptr, out_off, (size_t)(8 * (n + 1))},
                                 {g->in_off.ptr, in_off, (size_t)(8 * (n + 1))}};
        g->h2d_bytes = 16 * (n + 1);
        if (m && out_tgt) rc = upload_narrow(ctx, out_tgt, m, g->out_tgt.as<int32_t>(), &g->h2d_bytes);
        if (!rc) rc = upload_narrow(ctx, in_src, m, g->in_src.as<int32_t>(), &g->h2d_bytes, offs, 2);
        if (!rc) {
            k_degree<<<gs_grid(ctx, n), 256, 0, st>>>(g->out_off.as<int64_t>(), n, g->out_deg.as<int32_t>());
            cudaError_t e = cudaStreamSynchronize(st);
            if (e == cudaSuccess) e = cudaGetLastError();
            if (e != cudaSuccess) rc = fail(PR_ERR_CUDA, std::string("graph upload: ") + cudaGetErrorString(e));
        }
    }
    if (rc) { delete g; return rc; }
    *out = g;
    return PR_OK;
}

int export_graph(Graph &g, int64_t *out_off, int64_t *out_tgt, int64_t *in_off, int64_t *in_src) {
    Ctx &ctx = *g.ctx;
    cudaStream_t st = ctx.stream;
    DevBuf wide;
    PR_TRY(ensure(wide, 8 * (g.m ? g.m : 1)));
    if (out_off) PR_CUDA(cudaMemcpyAsync(out_off, g.out_off.ptr, 8 * (g.n + 1), cudaMemcpyDeviceToHost, st));
    if (in_off) PR_CUDA(cudaMemcpyAsync(in_off, g.in_off.ptr, 8 * (g.n + 1), cudaMemcpyDeviceToHost, st));
    if (out_tgt && g.m) {
        PR_TRY(need_csr(g, "exporting out_targets"));
        k_widen<<<gs_grid(ctx, g.m), 256, 0, st>>>(g.out_tgt.as<int32_t>(), g.m, wide.as<int64_t>());
        PR_CUDA(cudaMemcpyAsync(out_tgt, wide.ptr, 8 * g.m, cudaMemcpyDeviceToHost, st));
        PR_CUDA(cudaStreamSynchronize(st));
    }
    if (in_src && g.m) {
        k_widen<<<gs_grid(ctx, g.m), 256, 0, st>>>(g.in_src.as<int32_t>(), g.m, wide.as<int64_t>());
        PR_CUDA(cudaMemcpyAsync(in_src, wide.ptr, 8 * g.m, cudaMemcpyDeviceToHost, st));
    }
    PR_CUDA(cudaStreamSynchronize(st));
    return PR_OK;
}

int export_i32(Ctx &ctx, const DevBuf &src, int64_t count, int64_t *host) {
    if (!host || count <= 0) return PR_OK;
    DevBuf wide;
    PR_TRY(ensure(wide, 8 * count));
    k_widen<<<gs_grid(ctx, count), 256, 0, ctx.stream>>>(src.as<int32_t>(), count, wide.as<int64_t>());
    PR_CUDA(cudaMemcpyAsync(host, wide.ptr, 8 * count, cudaMemcpyDeviceToHost, ctx.stream));
    PR_CUDA(cudaStreamSynchronize(ctx.stream));
    return PR_OK;
}

int export_i64(Ctx &ctx, const DevBuf &src, int64_t count, int64_t *host) {
    if (!host || count <= 0) return PR_OK;
    PR_CUDA(cudaMemcpyAsync(host, src.ptr, 8 * count, cudaMemcpyDeviceToHost, ctx.stream));
    PR_CUDA(cudaStreamSynchronize(ctx.stream));
    return PR_OK;
}

}  // namespace pr
