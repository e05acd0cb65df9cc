// ingest.cu -- edge-list ingest on the device: load_edge_list (graph.py:201-259).
//
// Text -> (raw src, raw dst): every line is parsed by one thread (lines are
// found with a scan over the bytes).  The accepted grammar is what the
// reference's pandas call reads (sep=\s+, comment='#', two int64 columns):
// blank and comment-only lines are skipped, text after '#' is ignored, ids
// are non-negative decimal integers with an optional '+'.  Anything else
// (a third column, a non-digit, a negative id, an overflow, no edges at all)
// returns PR_ERR_FORMAT, and the Python side re-parses the text on the host
// to raise the reference's line-numbered GraphFormatError.
//
// Raw ids -> dense ids in order of first appearance over the interleaved
// (src0, dst0, src1, dst1, ...) sequence (graph.py:243-251): a stable radix
// sort of (id, position) pairs gives every distinct id with its first
// position at the head of its run; sorting the heads by first position gives
// the appearance order.  Bit-exact integer work; the graph is then built by
// the device from_edges (K1) and keeps original_ids on the device.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <utility>

#include "cubutil.cuh"
#include "internal.cuh"

namespace pr {

__device__ __forceinline__ bool is_ws(unsigned char c) {
    return c == ' ' || c == '\t' || c == '\r' || c == '\f' || c == '\v';
}

struct LineStart {
    const unsigned char *b;
    __host__ __device__ bool operator()(int64_t i) const { return i == 0 || b[i - 1] == '\n'; }
};

// kind: 0 blank/comment, 1 edge, 2 malformed
__global__ void k_parse_lines(const unsigned char *__restrict__ b, int64_t len, const int64_t *__restrict__ starts,
                              int64_t n_lines, int8_t *__restrict__ kind, int64_t *__restrict__ va,
                              int64_t *__restrict__ vb) {
    GRID_STRIDE(l, n_lines) {
        int64_t p = starts[l];
        const int64_t end = l + 1 < n_lines ? starts[l + 1] : len;  // one past the '\n' (or len)
        int8_t k = 0;
        int64_t vals[2] = {0, 0};
        int cols = 0;
        bool bad = false;
        while (p < end) {
            const unsigned char c = b[p];
            if (c == '\n' || c == '#') break;
            if (is_ws(c)) { ++p; continue; }
            // a token: [+]digits
            if (cols == 2) { bad = true; break; }
            if (c == '+') ++p;
            unsigned long long v = 0;
            int digits = 0;
            while (p < end && b[p] >= '0' && b[p] <= '9') {
                const unsigned d = b[p] - '0';
                if (v > (0x7fffffffffffffffull - d) / 10ull) { bad = true; break; }
                v = v * 10ull + d;
                ++digits;
                ++p;
            }
            if (bad) break;
            if (!digits) { bad = true; break; }
            if (p < end && !(is_ws(b[p]) || b[p] == '\n' || b[p] == '#')) { bad = true; break; }
            vals[cols++] = (int64_t)v;
        }
        if (bad || cols == 1) k = 2;
        else if (cols == 2) k = 1;
        kind[l] = k;
        va[l] = vals[0];
        vb[l] = vals[1];
    }
}

struct IsEdge {
    const int8_t *kind;
    __host__ __device__ bool operator()(int64_t l) const { return kind[l] == 1; }
};

__global__ void k_any_bad(const int8_t *__restrict__ kind, int64_t n, int *__restrict__ flag) {
    GRID_STRIDE(l, n) if (kind[l] == 2) *flag = 1;
}

__global__ void k_gather_pairs(const int64_t *__restrict__ lines, int64_t m, const int64_t *__restrict__ va,
                               const int64_t *__restrict__ vb, int64_t *__restrict__ flat) {
    GRID_STRIDE(i, m) {
        const int64_t l = lines[i];
        flat[2 * i] = va[l];
        flat[2 * i + 1] = vb[l];
    }
}

__global__ void k_interleave(const int64_t *__restrict__ s, const int64_t *__restrict__ d, int64_t m,
                             int64_t *__restrict__ flat, int *__restrict__ neg) {
    GRID_STRIDE(i, m) {
        flat[2 * i] = s[i];
        flat[2 * i + 1] = d[i];
        if (s[i] < 0 || d[i] < 0) *neg = 1;
    }
}

__global__ void k_iota64(int64_t *__restrict__ out, int64_t count) { GRID_STRIDE(i, count) out[i] = i; }

__global__ void k_heads(const unsigned long long *__restrict__ keys, int64_t count, int64_t *__restrict__ head) {
    GRID_STRIDE(j, count) head[j] = (j == 0 || keys[j] != keys[j - 1]) ? 1 : 0;
}

// for every run head: its id and first position (the stable sort keeps
// positions ascending inside a run)
__global__ void k_run_heads(const unsigned long long *__restrict__ keys, const int64_t *__restrict__ pos,
                            const int64_t *__restrict__ seg_incl, int64_t count, int64_t *__restrict__ uid,
                            unsigned long long *__restrict__ first) {
    GRID_STRIDE(j, count) {
        if (j == 0 || keys[j] != keys[j - 1]) {
            const int64_t s = seg_incl[j] - 1;
            uid[s] = (int64_t)keys[j];
            first[s] = (unsigned long long)pos[j];
        }
    }
}

__global__ void k_rank_of(const int64_t *__restrict__ app, int64_t n, const int64_t *__restrict__ uid,
                          int64_t *__restrict__ rank, int64_t *__restrict__ orig) {
    GRID_STRIDE(k, n) {
        rank[app[k]] = k;
        orig[k] = uid[app[k]];
    }
}

__global__ void k_dense(const int64_t *__restrict__ pos, const int64_t *__restrict__ seg_incl, int64_t count,
                        const int64_t *__restrict__ rank, int64_t *__restrict__ dense_src,
                        int64_t *__restrict__ dense_dst) {
    GRID_STRIDE(j, count) {
        const int64_t p = pos[j], r = rank[seg_incl[j] - 1];
        if (p & 1) dense_dst[p >> 1] = r;
        else dense_src[p >> 1] = r;
    }
}

static unsigned ig_grid(Ctx &ctx, int64_t items) {
    int64_t b = (items + 255) / 256, cap = (int64_t)ctx.sm_count * 16;
    if (b > cap) b = cap;
    return (unsigned)(b < 1 ? 1 : b);
}

// raw ids (device, int64, m edges, interleaved in `flat`) -> graph
static int remap_and_build(Ctx &ctx, DevBuf &flat, int64_t m, Graph **out) {
    cudaStream_t st = ctx.stream;
    const int64_t cnt = 2 * m;
    DevBuf pos, keys2, pos2, head, seg, uid, first, first2, app, app_in, rank, orig, ds, dd;
    PR_TRY(ensure(pos, 8 * cnt));
    PR_TRY(ensure(keys2, 8 * cnt));
    PR_TRY(ensure(pos2, 8 * cnt));
    k_iota64<<<ig_grid(ctx, cnt), 256, 0, st>>>(pos.as<int64_t>(), cnt);
    PR_TRY(cub_run(ctx, [&](void *t, size_t &b) {
        return cub::DeviceRadixSort::SortPairs(t, b, flat.as<unsigned long long>(), keys2.as<unsigned long long>(),
                                               pos.as<int64_t>(), pos2.as<int64_t>(), cnt, 0, 63, st);
    }));
    PR_TRY(ensure(head, 8 * cnt));
    PR_TRY(ensure(seg, 8 * cnt));
    k_heads<<<ig_grid(ctx, cnt), 256, 0, st>>>(keys2.as<unsigned long long>(), cnt, head.as<int64_t>());
    PR_TRY(cub_run(ctx, [&](void *t, size_t &b) {
        return cub::DeviceScan::InclusiveSum(t, b, head.as<int64_t>(), seg.as<int64_t>(), cnt, st);
    }));
    int64_t n = 0;
    PR_CUDA(cudaMemcpyAsync(&n, seg.as<int64_t>() + cnt - 1, 8, cudaMemcpyDeviceToHost, st));
    PR_CUDA(cudaStreamSynchronize(st));
    if (n > INT32_MAX - 1) return fail(PR_ERR_ARG, "more distinct vertex ids than the int32 column-index range");
    PR_TRY(ensure(uid, 8 * n));
    PR_TRY(ensure(first, 8 * n));
    PR_TRY(ensure(first2, 8 * n));
    PR_TRY(ensure(app_in, 8 * n));
    PR_TRY(ensure(app, 8 * n));
    PR_TRY(ensure(rank, 8 * n));
    PR_TRY(ensure(orig, 8 * n));
    k_run_heads<<<ig_grid(ctx, cnt), 256, 0, st>>>(keys2.as<unsigned long long>(), pos2.as<int64_t>(),
                                                   seg.as<int64_t>(), cnt, uid.as<int64_t>(),
                                                   first.as<unsigned long long>());
    // appearance order: runs sorted by first position (distinct keys)
    k_iota64<<<ig_grid(ctx, n), 256, 0, st>>>(app_in.as<int64_t>(), n);
    PR_TRY(cub_run(ctx, [&](void *t, size_t &b) {
        return cub::DeviceRadixSort::SortPairs(t, b, first.as<unsigned long long>(), first2.as<unsigned long long>(),
                                               app_in.as<int64_t>(), app.as<int64_t>(), n, 0, 63, st);
    }));
    k_rank_of<<<ig_grid(ctx, n), 256, 0, st>>>(app.as<int64_t>(), n, uid.as<int64_t>(), rank.as<int64_t>(),
                                               orig.as<int64_t>());
    PR_TRY(ensure(ds, 8 * m));
    PR_TRY(ensure(dd, 8 * m));
    k_dense<<<ig_grid(ctx, cnt), 256, 0, st>>>(pos2.as<int64_t>(), seg.as<int64_t>(), cnt, rank.as<int64_t>(),
                                               ds.as<int64_t>(), dd.as<int64_t>());
    PR_CUDA(cudaGetLastError());
    Graph *g = nullptr;
    PR_TRY(build_from_device_edges(ctx, n, ds.as<int64_t>(), dd.as<int64_t>(), m, &g));
    // keep the first-appearance id table with the graph
    std::swap(g->orig_ids.ptr, orig.ptr);
    std::swap(g->orig_ids.bytes, orig.bytes);
    *out = g;
    return PR_OK;
}

int load_edge_list_device(Ctx &ctx, const char *text, int64_t len, Graph **out) {
    cudaStream_t st = ctx.stream;
    if (len <= 0) return fail(PR_ERR_FORMAT, "empty graph: no edges found");
    DevBuf bytes, starts, cnt, kind, va, vb, lines, flag, flat;
    PR_TRY(ensure(bytes, (size_t)len));
    PR_CUDA(cudaMemcpyAsync(bytes.ptr, text, (size_t)len, cudaMemcpyHostToDevice, st));
    PR_TRY(ensure(starts, 8 * (len + 1)));
    PR_TRY(ensure(cnt, 8));
    auto first = thrust::make_counting_iterator<int64_t>(0);
    PR_TRY(cub_run(ctx, [&](void *t, size_t &b) {
        return cub::DeviceSelect::If(t, b, first, starts.as<int64_t>(), cnt.as<int64_t>(), len,
                                     LineStart{bytes.as<unsigned char>()}, st);
    }));
    int64_t n_lines = 0;
    PR_CUDA(cudaMemcpyAsync(&n_lines, cnt.ptr, 8, cudaMemcpyDeviceToHost, st));
    PR_CUDA(cudaStreamSynchronize(st));
    PR_TRY(ensure(kind, n_lines ? n_lines : 1));
    PR_TRY(ensure(va, 8 * (n_lines ? n_lines : 1)));
    PR_TRY(ensure(vb, 8 * (n_lines ? n_lines : 1)));
    PR_TRY(ensure(flag, 4));
    PR_CUDA(cudaMemsetAsync(flag.ptr, 0, 4, st));
    if (n_lines) {
        k_parse_lines<<<ig_grid(ctx, n_lines), 256, 0, st>>>(bytes.as<unsigned char>(), len, starts.as<int64_t>(),
                                                            n_lines, kind.as<int8_t>(), va.as<int64_t>(),
                                                            vb.as<int64_t>());
        k_any_bad<<<ig_grid(ctx, n_lines), 256, 0, st>>>(kind.as<int8_t>(), n_lines, flag.as<int>());
    }
    int bad = 0;
    PR_CUDA(cudaMemcpyAsync(&bad, flag.ptr, 4, cudaMemcpyDeviceToHost, st));
    PR_CUDA(cudaStreamSynchronize(st));
    if (bad) return fail(PR_ERR_FORMAT, "edge list needs the host parser (malformed or unusual line)");
    PR_TRY(ensure(lines, 8 * (n_lines ? n_lines : 1)));
    PR_TRY(cub_run(ctx, [&](void *t, size_t &b) {
        return cub::DeviceSelect::If(t, b, first, lines.as<int64_t>(), cnt.as<int64_t>(), n_lines,
                                     IsEdge{kind.as<int8_t>()}, st);
    }));
    int64_t m = 0;
    PR_CUDA(cudaMemcpyAsync(&m, cnt.ptr, 8, cudaMemcpyDeviceToHost, st));
    PR_CUDA(cudaStreamSynchronize(st));
    if (m == 0) return fail(PR_ERR_FORMAT, "empty graph: no edges found");
    PR_TRY(ensure(flat, 16 * m));
    k_gather_pairs<<<ig_grid(ctx, m), 256, 0, st>>>(lines.as<int64_t>(), m, va.as<int64_t>(), vb.as<int64_t>(),
                                                   flat.as<int64_t>());
    bytes.release();
    starts.release();
    return remap_and_build(ctx, flat, m, out);
}

int graph_from_raw_ids(Ctx &ctx, const int64_t *src, const int64_t *dst, int64_t m, Graph **out) {
    cudaStream_t st = ctx.stream;
    if (m <= 0) return fail(PR_ERR_FORMAT, "empty graph: no edges found");
    DevBuf hs, hd, flat, neg;
    PR_TRY(ensure(hs, 8 * m));
    PR_TRY(ensure(hd, 8 * m));
    PR_TRY(ensure(flat, 16 * m));
    PR_TRY(ensure(neg, 4));
    PR_CUDA(cudaMemcpyAsync(hs.ptr, src, 8 * m, cudaMemcpyHostToDevice, st));
    PR_CUDA(cudaMemcpyAsync(hd.ptr, dst, 8 * m, cudaMemcpyHostToDevice, st));
    PR_CUDA(cudaMemsetAsync(neg.ptr, 0, 4, st));
    k_interleave<<<ig_grid(ctx, m), 256, 0, st>>>(hs.as<int64_t>(), hd.as<int64_t>(), m, flat.as<int64_t>(),
                                                  neg.as<int>());
    int bad = 0;
    PR_CUDA(cudaMemcpyAsync(&bad, neg.ptr, 4, cudaMemcpyDeviceToHost, st));
    PR_CUDA(cudaStreamSynchronize(st));
    if (bad) return fail(PR_ERR_ARG, "negative vertex id");
    return remap_and_build(ctx, flat, m, out);
}

}  // namespace pr
