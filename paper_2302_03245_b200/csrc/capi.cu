// capi.cu -- extern "C" boundary of libpushrank_cuda (include/pushrank_cuda.h).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>

#include "internal.cuh"

namespace pr {

static thread_local std::string g_last_error;

void phase_mark(cudaStream_t st, const char *what) {
    static const bool on = [] {
        const char *e = getenv("PUSHRANK_TIMING");
        return e && e[0] == '1';
    }();
    if (!on) return;
    static thread_local std::chrono::steady_clock::time_point last = std::chrono::steady_clock::now();
    cudaStreamSynchronize(st);
    auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[pushrank] %-28s %9.3f ms\n", what,
            std::chrono::duration<double, std::milli>(now - last).count());
    last = now;
}

void set_error(const std::string &msg) { g_last_error = msg; }

int fail(int code, const std::string &msg) {
    set_error(msg);
    return code;
}

int classify_export(Graph &g, int64_t *outs[4]);
int rmat_generate(Ctx &ctx, int scale, double a, double b, double c, uint64_t seed, int64_t first, int64_t count,
                  int64_t *d_src, int64_t *d_dst);
int graph_rmat(Ctx &ctx, int scale, int64_t ef, double a, double b, double c, uint64_t seed, Graph **out);
int upload_graph(Ctx &ctx, int64_t n, int64_t m, const int64_t *out_off, const int64_t *out_tgt,
                 const int64_t *in_off, const int64_t *in_src, Graph **out);
int export_graph(Graph &g, int64_t *out_off, int64_t *out_tgt, int64_t *in_off, int64_t *in_src);
int export_i32(Ctx &ctx, const DevBuf &src, int64_t count, int64_t *host);
int export_i64(Ctx &ctx, const DevBuf &src, int64_t count, int64_t *host);
#ifdef PR_UBENCH
int debug_gather(Graph &g0, int variant, int iters, int blocks_per_sm, double *ms_out);
int debug_graph(Ctx &ctx, int variant, int64_t iters, int blocks, double *us_out);
#endif
struct Part;
int part_create(Ctx &ctx, int64_t owned, int64_t slot, const int64_t *in_off, const int64_t *in_src, int64_t edges,
                const int64_t *deg, const int64_t *row_len, const int64_t *dtc, const uint8_t *dang,
                const uint8_t *recv, int algorithm, double c, double xi, Part **out);
int part_init(Part &P, double *d_s_mine, int64_t *ints, double *floats);
int part_round(Part &P, const double *d_s_full, double *d_s_mine, int64_t *ints, double *floats);
int part_settle_shares(Part &P, double *d_x_mine);
int part_settle(Part &P, const double *d_x_full, int64_t *settled, int64_t *ints, double *floats);
int part_total(Part &P, int include_h, double *total);
int part_export(Part &P, double *reserved, double *pending);
void part_destroy(Part *P);
Ctx &part_ctx(Part &P);
void *part_stream(Part &P);
int part_init_device(Part &P, double *d_s_mine, double *d_stats9);
int part_round_device(Part &P, const double *d_s_full, double *d_s_mine, int fast, int kind, double *d_stats9);
int part_share_buffers(Part &P, int parts, int rank, void **d_full, void *ipc);
int part_set_peers(Part &P, const void *handles);
int part_set_peer_ptrs(Part &P, int parts, int rank, void *const *ptrs);
int part_set_rank(Part &P, int parts, int rank);
int part_from_graph(Graph &g, int parts, int rank, int algorithm, double c, double xi, int64_t *bounds, Part **out);
int part_export_rows(Part &P, int64_t *in_off, int64_t *in_src, int64_t *deg, int64_t *row_len, int64_t *dtc,
                     uint8_t *dang, uint8_t *recv);
int part_sizes(Part &P, int64_t *owned, int64_t *slot, int64_t *edges);
int part_skip_if_done(Part &P, const double *d_prev9);
int part_exchange_entries(Part &P, int64_t *entries);
int part_launches_per_round(Part &P, int *out);
int part_close_peers(Part &P);
int part_init_fused(Part &P, double *d_stats9);
int part_round_fused(Part &P, int parity, int kind, double *d_stats9);

static int set_device(Ctx &ctx) {
    PR_CUDA(cudaSetDevice(ctx.device));
    alloc_stream() = ctx.stream;
    return PR_OK;
}

}  // namespace pr

using namespace pr;

struct pr_ctx {
    Ctx c;
};
struct pr_graph {
    Graph *g;
};

#define CHECK_PTR(p, name) \
    if (!(p)) return fail(PR_ERR_ARG, std::string(name) + " is NULL")

extern "C" {

int pr_abi_version(void) { return PR_ABI_VERSION; }

const char *pr_last_error(void) { return g_last_error.c_str(); }

int pr_device_count(int *count) {
    CHECK_PTR(count, "count");
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *count = 0;
        return fail(PR_ERR_CUDA, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
    }
    *count = c;
    return PR_OK;
}

int pr_ctx_create(int device, pr_ctx **out) {
    CHECK_PTR(out, "out");
    *out = nullptr;
    int count = 0;
    PR_TRY(pr_device_count(&count));
    if (device < 0 || device >= count)
        return fail(PR_ERR_ARG, "device " + std::to_string(device) + " not present (" + std::to_string(count) +
                                    " CUDA devices)");
    pr_ctx *c = new pr_ctx();
    c->c.device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->c.stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) {
        // keep freed pool memory cached: graph builds reuse it without driver calls
        cudaMemPool_t pool;
        e = cudaDeviceGetDefaultMemPool(&pool, device);
        uint64_t keep = UINT64_MAX;
        if (e == cudaSuccess) e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    alloc_stream() = c->c.stream;
    if (e == cudaSuccess) {
        cudaDeviceProp prop;
        e = cudaGetDeviceProperties(&prop, device);
        if (e == cudaSuccess) {
            c->c.sm_count = prop.multiProcessorCount;
            c->c.l2_bytes = (size_t)prop.l2CacheSize;
            if (prop.major < 10) {
                cudaStreamDestroy(c->c.stream);
                delete c;
                return fail(PR_ERR_STATE, std::string("device ") + prop.name + " is sm_" +
                                              std::to_string(prop.major * 10 + prop.minor) +
                                              "; this library is built for sm_100a (B200)");
            }
        }
    }
    if (e != cudaSuccess) {
        delete c;
        return fail(PR_ERR_CUDA, std::string("context init: ") + cudaGetErrorString(e));
    }
    *out = c;
    return PR_OK;
}

int pr_ctx_destroy(pr_ctx *ctx) {
    if (!ctx) return PR_OK;
    cudaSetDevice(ctx->c.device);
    alloc_stream() = ctx->c.stream;
    cudaStreamSynchronize(ctx->c.stream);
    release_execs(ctx->c);
    ctx->c.scratch.release();
    ctx->c.flush.release();
    if (ctx->c.obs_host) cudaFreeHost(ctx->c.obs_host);
    uploader_destroy(ctx->c);
    cudaStreamDestroy(ctx->c.stream);
    delete ctx;
    return PR_OK;
}

int pr_ctx_synchronize(pr_ctx *ctx) {
    CHECK_PTR(ctx, "ctx");
    PR_CUDA(cudaStreamSynchronize(ctx->c.stream));
    return PR_OK;
}

int pr_graph_from_edges(pr_ctx *ctx, int64_t n, const int64_t *src, const int64_t *dst, int64_t m_raw,
                        pr_graph **out) {
    CHECK_PTR(ctx, "ctx");
    CHECK_PTR(out, "out");
    if (m_raw < 0) return fail(PR_ERR_ARG, "negative edge count");
    if (m_raw > 0) {
        CHECK_PTR(src, "src");
        CHECK_PTR(dst, "dst");
    }
    PR_TRY(set_device(ctx->c));
    DevBuf ds, dd;
    PR_TRY(ensure(ds, 8 * (m_raw ? m_raw : 1)));
    PR_TRY(ensure(dd, 8 * (m_raw ? m_raw : 1)));
    if (m_raw) {
        PR_CUDA(cudaMemcpyAsync(ds.ptr, src, 8 * m_raw, cudaMemcpyHostToDevice, ctx->c.stream));
        PR_CUDA(cudaMemcpyAsync(dd.ptr, dst, 8 * m_raw, cudaMemcpyHostToDevice, ctx->c.stream));
    }
    Graph *g = nullptr;
    PR_TRY(build_from_device_edges(ctx->c, n, ds.as<int64_t>(), dd.as<int64_t>(), m_raw, &g));
    *out = new pr_graph{g};
    return PR_OK;
}

int pr_graph_from_device_edges(pr_ctx *ctx, int64_t n, const int64_t *d_src, const int64_t *d_dst, int64_t m_raw,
                               pr_graph **out) {
    CHECK_PTR(ctx, "ctx");
    CHECK_PTR(out, "out");
    PR_TRY(set_device(ctx->c));
    Graph *g = nullptr;
    PR_TRY(build_from_device_edges(ctx->c, n, d_src, d_dst, m_raw, &g));
    *out = new pr_graph{g};
    return PR_OK;
}

int pr_graph_load_edge_list(pr_ctx *ctx, const char *text, int64_t len, pr_graph **out, int64_t *raw_edges) {
    CHECK_PTR(ctx, "ctx");
    CHECK_PTR(out, "out");
    if (len > 0) CHECK_PTR(text, "text");
    PR_TRY(set_device(ctx->c));
    Graph *g = nullptr;
    PR_TRY(load_edge_list_device(ctx->c, text, len, &g));
    if (raw_edges) *raw_edges = g->raw;
    *out = new pr_graph{g};
    return PR_OK;
}

int pr_graph_from_raw_ids(pr_ctx *ctx, const int64_t *src, const int64_t *dst, int64_t m, pr_graph **out) {
    CHECK_PTR(ctx, "ctx");
    CHECK_PTR(out, "out");
    if (m > 0) {
        CHECK_PTR(src, "src");
        CHECK_PTR(dst, "dst");
    }
    PR_TRY(set_device(ctx->c));
    Graph *g = nullptr;
    PR_TRY(graph_from_raw_ids(ctx->c, src, dst, m, &g));
    *out = new pr_graph{g};
    return PR_OK;
}

int pr_graph_original_ids(pr_graph *g, int64_t *out) {
    CHECK_PTR(g, "graph");
    CHECK_PTR(out, "out");
    Graph &G = *g->g;
    PR_TRY(set_device(*G.ctx));
    if (G.orig_ids.ptr) {
        PR_CUDA(cudaMemcpy(out, G.orig_ids.ptr, 8 * G.n, cudaMemcpyDeviceToHost));
    } else {
        for (int64_t i = 0; i < G.n; ++i) out[i] = i;
    }
    return PR_OK;
}

int pr_rank_order(pr_ctx *ctx, const double *values, const int64_t *original_ids, int64_t n, int64_t k,
                  int64_t *order) {
    CHECK_PTR(ctx, "ctx");
    if (n > 0) {
        CHECK_PTR(values, "values");
        CHECK_PTR(order, "order");
    }
    if (n < 0 || k < 0) return fail(PR_ERR_ARG, "n and k must be non-negative");
    PR_TRY(set_device(ctx->c));
    return rank_order(ctx->c, values, original_ids, n, k, order);
}

int pr_write_ranking_csv(pr_ctx *ctx, const double *values, const int64_t *original_ids, int64_t n,
                         const char *path) {
    CHECK_PTR(ctx, "ctx");
    CHECK_PTR(path, "path");
    if (n > 0) CHECK_PTR(values, "values");
    PR_TRY(set_device(ctx->c));
    return write_ranking_csv(ctx->c, values, original_ids, n, path);
}

int pr_format_score(double value, char *out) {
    CHECK_PTR(out, "out");
    return format_score(value, out);
}

int pr_graph_upload(pr_ctx *ctx, int64_t n, int64_t m, const int64_t *out_offsets, const int64_t *out_targets,
                    const int64_t *in_offsets, const int64_t *in_sources, pr_graph **out) {
    CHECK_PTR(ctx, "ctx");
    CHECK_PTR(out, "out");
    CHECK_PTR(out_offsets, "out_offsets");
    CHECK_PTR(in_offsets, "in_offsets");
    if (m > 0) CHECK_PTR(in_sources, "in_sources");
    PR_TRY(set_device(ctx->c));
    Graph *g = nullptr;
    PR_TRY(upload_graph(ctx->c, n, m, out_offsets, out_targets, in_offsets, in_sources, &g));
    *out = new pr_graph{g};
    return PR_OK;
}

int pr_graph_attach_out_targets(pr_graph *g, const int64_t *out_targets) {
    CHECK_PTR(g, "graph");
    if (g->g->m > 0) CHECK_PTR(out_targets, "out_targets");
    PR_TRY(set_device(*g->g->ctx));
    return attach_out_targets(*g->g, out_targets);
}

int pr_graph_destroy(pr_graph *g) {
    if (!g) return PR_OK;
    cudaSetDevice(g->g->ctx->device);
    alloc_stream() = g->g->ctx->stream;
    cudaStreamSynchronize(g->g->ctx->stream);
    phase_mark(g->g->ctx->stream, "destroy: sync");
    cudaStream_t st = g->g->ctx->stream;
    delete g->g;
    phase_mark(st, "destroy: free");
    delete g;
    return PR_OK;
}

int pr_graph_info(const pr_graph *g, int64_t *n, int64_t *m) {
    CHECK_PTR(g, "graph");
    if (n) *n = g->g->n;
    if (m) *m = g->g->m;
    return PR_OK;
}

int pr_graph_h2d_bytes(const pr_graph *g, int64_t *bytes) {
    CHECK_PTR(g, "graph");
    CHECK_PTR(bytes, "bytes");
    *bytes = g->g->h2d_bytes;
    return PR_OK;
}

int pr_graph_export(pr_graph *g, int64_t *out_offsets, int64_t *out_targets, int64_t *in_offsets,
                    int64_t *in_sources) {
    CHECK_PTR(g, "graph");
    PR_TRY(set_device(*g->g->ctx));
    return export_graph(*g->g, out_offsets, out_targets, in_offsets, in_sources);
}

int pr_classify(pr_graph *g, pr_class_counts *counts) {
    CHECK_PTR(g, "graph");
    PR_TRY(set_device(*g->g->ctx));
    PR_TRY(classify_device(*g->g));
    if (counts) *counts = g->g->counts;
    return PR_OK;
}

int pr_classify_export(pr_graph *g, int64_t *dangling, int64_t *unreferenced, int64_t *weak_dangling,
                       int64_t *weak_unreferenced) {
    CHECK_PTR(g, "graph");
    PR_TRY(set_device(*g->g->ctx));
    int64_t *outs[4] = {dangling, unreferenced, weak_dangling, weak_unreferenced};
    return classify_export(*g->g, outs);
}

int pr_dangling_target_counts(pr_graph *g, int64_t *out) {
    CHECK_PTR(g, "graph");
    CHECK_PTR(out, "out");
    PR_TRY(set_device(*g->g->ctx));
    PR_TRY(ensure_dtc(*g->g));
    return export_i32(*g->g->ctx, g->g->dtc, g->g->n, out);
}

int pr_preprocess_ifp2(pr_graph *g, pr_ifp2_counts *counts) {
    CHECK_PTR(g, "graph");
    PR_TRY(set_device(*g->g->ctx));
    PR_TRY(ifp2_counts_device(*g->g));
    if (counts) *counts = g->g->ifp2;
    return PR_OK;
}

int pr_ifp2_export(pr_graph *g, int64_t *live_offsets, int64_t *live_targets, int64_t *live_degree,
                   int64_t *dangling_ids, int64_t *source_offsets, int64_t *source_ids) {
    CHECK_PTR(g, "graph");
    Graph &G = *g->g;
    if (!G.has_ifp2 && !G.ifp2_counted) return fail(PR_ERR_STATE, "pr_preprocess_ifp2 has not run");
    PR_TRY(set_device(*G.ctx));
    PR_TRY(preprocess_ifp2_device(G));
    Ctx &c = *G.ctx;
    PR_TRY(export_i64(c, G.live_off, G.n + 1, live_offsets));
    PR_TRY(export_i32(c, G.live_tgt, G.ifp2.live_edges, live_targets));
    PR_TRY(export_i32(c, G.live_deg, G.n, live_degree));
    PR_TRY(export_i32(c, G.dang_ids, G.ifp2.dangling, dangling_ids));
    PR_TRY(export_i64(c, G.src_off, G.ifp2.dangling + 1, source_offsets));
    PR_TRY(export_i32(c, G.src_ids, G.ifp2.source_edges, source_ids));
    return PR_OK;
}

static int run_common(pr_graph *g, const pr_run_params *params, double *values, double *reserved, double *pending,
                      pr_round_stats *rows, int64_t row_cap, pr_run_result *result, bool host_out) {
    CHECK_PTR(g, "graph");
    CHECK_PTR(params, "params");
    Graph &G = *g->g;
    PR_TRY(set_device(*G.ctx));
    cudaStream_t st = G.ctx->stream;
    DevBuf dv, dr, dp;
    double *d_values = values, *d_reserved = reserved, *d_pending = pending;
    if (host_out) {
        if (values) { PR_TRY(ensure(dv, 8 * G.n)); d_values = dv.as<double>(); }
        if (reserved) { PR_TRY(ensure(dr, 8 * G.n)); d_reserved = dr.as<double>(); }
        if (pending) { PR_TRY(ensure(dp, 8 * G.n)); d_pending = dp.as<double>(); }
    }
    pr_run_result local;
    memset(&local, 0, sizeof(local));
    int rc = run_rounds(G, *params, d_values, d_reserved, d_pending, rows, row_cap, &local);
    if (result) *result = local;
    if (rc != PR_OK && rc != PR_ERR_NOT_SETTLED) return rc;
    if (host_out) {
        if (values) PR_CUDA(cudaMemcpyAsync(values, d_values, 8 * G.n, cudaMemcpyDeviceToHost, st));
        if (reserved) PR_CUDA(cudaMemcpyAsync(reserved, d_reserved, 8 * G.n, cudaMemcpyDeviceToHost, st));
        if (pending) PR_CUDA(cudaMemcpyAsync(pending, d_pending, 8 * G.n, cudaMemcpyDeviceToHost, st));
    }
    PR_CUDA(cudaStreamSynchronize(st));
    return rc;
}

int pr_run(pr_graph *g, const pr_run_params *params, double *values, double *reserved, double *pending,
           pr_round_stats *rows, int64_t row_cap, pr_run_result *result) {
    return run_common(g, params, values, reserved, pending, rows, row_cap, result, true);
}

int pr_run_device(pr_graph *g, const pr_run_params *params, double *d_values, double *d_reserved,
                  double *d_pending, pr_round_stats *rows, int64_t row_cap, pr_run_result *result) {
    return run_common(g, params, d_values, d_reserved, d_pending, rows, row_cap, result, false);
}

int pr_power(pr_graph *g, double damping, int64_t iterations, double tolerance, double threshold,
             const double *personalization, double *pi, double *deltas, int64_t *converged,
             pr_run_result *result) {
    CHECK_PTR(g, "graph");
    PR_TRY(set_device(*g->g->ctx));
    return power_device(*g->g, damping, iterations, tolerance, threshold, personalization, pi, deltas, converged,
                        nullptr, nullptr, result);
}

int pr_power_observed(pr_graph *g, double damping, int64_t iterations, double tolerance, double threshold,
                      const double *personalization, double *pi, double *deltas, int64_t *converged,
                      int (*on_iterate)(void *user, int64_t k, const double *pi), void *user,
                      pr_run_result *result) {
    CHECK_PTR(g, "graph");
    PR_TRY(set_device(*g->g->ctx));
    return power_device(*g->g, damping, iterations, tolerance, threshold, personalization, pi, deltas, converged,
                        on_iterate, user, result);
}

int pr_error_report(pr_ctx *ctx, const double *d_est, const double *d_ref, int64_t n, double *max_rel, double *l1,
                    int64_t *worst, int64_t *nonpositive) {
    CHECK_PTR(ctx, "ctx");
    CHECK_PTR(d_est, "est");
    CHECK_PTR(d_ref, "ref");
    PR_TRY(set_device(ctx->c));
    return error_report(ctx->c, d_est, d_ref, n, max_rel, l1, worst, nonpositive);
}

int pr_power_to_target(pr_graph *g, double damping, int64_t limit, const double *personalization,
                       const double *d_ref, double target_err, int64_t *hit) {
    CHECK_PTR(g, "graph");
    CHECK_PTR(d_ref, "ref");
    CHECK_PTR(hit, "hit");
    PR_TRY(set_device(*g->g->ctx));
    *hit = 0;
    if (limit <= 0) return PR_OK;
    return power_device(*g->g, damping, limit, 0.0, 1e-10, personalization, nullptr, nullptr, nullptr, nullptr,
                        nullptr, nullptr, d_ref, target_err, hit);
}

int pr_rmat_generate(pr_ctx *ctx, int scale, int64_t edge_factor, double a, double b, double c, uint64_t seed,
                     int64_t first, int64_t count, int64_t *d_src, int64_t *d_dst) {
    CHECK_PTR(ctx, "ctx");
    (void)edge_factor;
    PR_TRY(set_device(ctx->c));
    PR_TRY(rmat_generate(ctx->c, scale, a, b, c, seed, first, count, d_src, d_dst));
    PR_CUDA(cudaStreamSynchronize(ctx->c.stream));
    return PR_OK;
}

int pr_graph_rmat(pr_ctx *ctx, int scale, int64_t edge_factor, double a, double b, double c, uint64_t seed,
                  pr_graph **out) {
    CHECK_PTR(ctx, "ctx");
    CHECK_PTR(out, "out");
    PR_TRY(set_device(ctx->c));
    Graph *g = nullptr;
    PR_TRY(graph_rmat(ctx->c, scale, edge_factor, a, b, c, seed, &g));
    *out = new pr_graph{g};
    return PR_OK;
}

int pr_device_alloc(pr_ctx *ctx, int64_t bytes, void **d_ptr) {
    CHECK_PTR(ctx, "ctx");
    CHECK_PTR(d_ptr, "d_ptr");
    PR_TRY(set_device(ctx->c));
    PR_CUDA(cudaMalloc(d_ptr, bytes > 0 ? (size_t)bytes : 16));
    return PR_OK;
}

int pr_device_free(pr_ctx *ctx, void *d_ptr) {
    CHECK_PTR(ctx, "ctx");
    PR_TRY(set_device(ctx->c));
    PR_CUDA(cudaFree(d_ptr));
    return PR_OK;
}

static std::mutex g_host_mu;
static std::unordered_map<void *, size_t> g_host_size;          // live + cached blocks
static std::unordered_multimap<size_t, void *> g_host_free;     // cached blocks by size

int pr_host_alloc(int64_t bytes, void **h_ptr) {
    CHECK_PTR(h_ptr, "h_ptr");
    const size_t sz = bytes > 0 ? (size_t)bytes : 16;
    {
        std::lock_guard<std::mutex> lk(g_host_mu);
        auto it = g_host_free.find(sz);
        if (it != g_host_free.end()) {
            *h_ptr = it->second;
            g_host_free.erase(it);
            return PR_OK;
        }
    }
    void *p = nullptr;
    PR_CUDA(cudaHostAlloc(&p, sz, cudaHostAllocPortable));
    std::lock_guard<std::mutex> lk(g_host_mu);
    g_host_size[p] = sz;
    *h_ptr = p;
    return PR_OK;
}

int pr_host_free(void *h_ptr) {
    if (!h_ptr) return PR_OK;
    std::lock_guard<std::mutex> lk(g_host_mu);
    auto it = g_host_size.find(h_ptr);
    if (it == g_host_size.end()) return fail(PR_ERR_ARG, "pr_host_free: not a pr_host_alloc block");
    g_host_free.emplace(it->second, h_ptr);
    return PR_OK;
}

int pr_memcpy_h2d(pr_ctx *ctx, void *d_dst, const void *h_src, int64_t bytes) {
    CHECK_PTR(ctx, "ctx");
    PR_TRY(set_device(ctx->c));
    PR_CUDA(cudaMemcpyAsync(d_dst, h_src, bytes, cudaMemcpyHostToDevice, ctx->c.stream));
    PR_CUDA(cudaStreamSynchronize(ctx->c.stream));
    return PR_OK;
}

int pr_memcpy_d2h(pr_ctx *ctx, void *h_dst, const void *d_src, int64_t bytes) {
    CHECK_PTR(ctx, "ctx");
    PR_TRY(set_device(ctx->c));
    PR_CUDA(cudaMemcpyAsync(h_dst, d_src, bytes, cudaMemcpyDeviceToHost, ctx->c.stream));
    PR_CUDA(cudaStreamSynchronize(ctx->c.stream));
    return PR_OK;
}

struct pr_part {
    Part *p;
};

int pr_part_create(pr_ctx *ctx, int64_t owned, int64_t slot, const int64_t *in_offsets, const int64_t *in_sources,
                   int64_t edges, const int64_t *out_degree, const int64_t *row_len,
                   const int64_t *dangling_target_counts, const uint8_t *dangling, const uint8_t *receives,
                   int32_t algorithm, double damping, double threshold, pr_part **out) {
    CHECK_PTR(ctx, "ctx");
    CHECK_PTR(out, "out");
    CHECK_PTR(in_offsets, "in_offsets");
    PR_TRY(set_device(ctx->c));
    Part *P = nullptr;
    PR_TRY(part_create(ctx->c, owned, slot, in_offsets, in_sources, edges, out_degree, row_len,
                       dangling_target_counts, dangling, receives, algorithm, damping, threshold, &P));
    *out = new pr_part{P};
    return PR_OK;
}

int pr_part_from_graph(pr_graph *g, int32_t parts, int32_t rank, int32_t algorithm, double damping,
                       double threshold, int64_t *bounds, pr_part **out) {
    CHECK_PTR(g, "graph");
    CHECK_PTR(out, "out");
    PR_TRY(set_device(*g->g->ctx));
    Part *P = nullptr;
    PR_TRY(part_from_graph(*g->g, parts, rank, algorithm, damping, threshold, bounds, &P));
    *out = new pr_part{P};
    return PR_OK;
}

#define PART_ENTER(p)            \
    CHECK_PTR(p, "partition");   \
    PR_TRY(set_device(part_ctx(*(p)->p)))

int pr_part_skip_if_done(pr_part *p, const double *d_prev_stats9) {
    PART_ENTER(p);
    return part_skip_if_done(*p->p, d_prev_stats9);
}

int pr_part_exchange_entries(pr_part *p, int64_t *entries) {
    PART_ENTER(p);
    CHECK_PTR(entries, "entries");
    return part_exchange_entries(*p->p, entries);
}

int pr_part_sizes(pr_part *p, int64_t *owned, int64_t *slot, int64_t *edges) {
    PART_ENTER(p);
    return part_sizes(*p->p, owned, slot, edges);
}

int pr_part_export_rows(pr_part *p, int64_t *in_offsets, int64_t *in_sources, int64_t *out_degree,
                        int64_t *row_len, int64_t *dangling_target_counts, uint8_t *dangling, uint8_t *receives) {
    PART_ENTER(p);
    return part_export_rows(*p->p, in_offsets, in_sources, out_degree, row_len, dangling_target_counts, dangling,
                            receives);
}

int pr_part_init(pr_part *p, double *d_shares_mine, int64_t *ints, double *floats) {
    PART_ENTER(p);
    return part_init(*p->p, d_shares_mine, ints, floats);
}
int pr_part_round(pr_part *p, const double *d_shares_full, double *d_shares_mine, int64_t *ints, double *floats) {
    PART_ENTER(p);
    return part_round(*p->p, d_shares_full, d_shares_mine, ints, floats);
}
int pr_part_init_device(pr_part *p, double *d_shares_mine, double *d_stats) {
    PART_ENTER(p);
    CHECK_PTR(d_stats, "stats");
    return part_init_device(*p->p, d_shares_mine, d_stats);
}
int pr_part_round_device(pr_part *p, const double *d_shares_full, double *d_shares_mine, int32_t fast,
                         int32_t kind, double *d_stats) {
    PART_ENTER(p);
    CHECK_PTR(d_stats, "stats");
    return part_round_device(*p->p, d_shares_full, d_shares_mine, fast, kind, d_stats);
}
int pr_part_share_buffers(pr_part *p, int32_t parts, int32_t rank, void **d_full, void *ipc_handles) {
    PART_ENTER(p);
    CHECK_PTR(d_full, "d_full");
    return part_share_buffers(*p->p, parts, rank, d_full, ipc_handles);
}
int pr_part_set_peers(pr_part *p, const void *ipc_handles) {
    PART_ENTER(p);
    CHECK_PTR(ipc_handles, "ipc_handles");
    return part_set_peers(*p->p, ipc_handles);
}
int pr_part_close_peers(pr_part *p) {
    PART_ENTER(p);
    return part_close_peers(*p->p);
}
int pr_part_launches_per_round(pr_part *p, int32_t *launches) {
    PART_ENTER(p);
    CHECK_PTR(launches, "launches");
    int v = 0;
    PR_TRY(part_launches_per_round(*p->p, &v));
    *launches = v;
    return PR_OK;
}
int pr_part_set_rank(pr_part *p, int32_t parts, int32_t rank) {
    PART_ENTER(p);
    return part_set_rank(*p->p, parts, rank);
}
int pr_part_set_peer_ptrs(pr_part *p, int32_t parts, int32_t rank, void *const *d_full) {
    PART_ENTER(p);
    CHECK_PTR(d_full, "d_full");
    return part_set_peer_ptrs(*p->p, parts, rank, d_full);
}
int pr_part_init_fused(pr_part *p, double *d_stats) {
    PART_ENTER(p);
    CHECK_PTR(d_stats, "stats");
    return part_init_fused(*p->p, d_stats);
}
int pr_part_round_fused(pr_part *p, int32_t parity, int32_t kind, double *d_stats) {
    PART_ENTER(p);
    CHECK_PTR(d_stats, "stats");
    return part_round_fused(*p->p, parity, kind, d_stats);
}
int pr_part_stream(pr_part *p, void **stream) {
    PART_ENTER(p);
    CHECK_PTR(stream, "stream");
    *stream = part_stream(*p->p);
    return PR_OK;
}
int pr_part_settle_shares(pr_part *p, double *d_x_mine) {
    PART_ENTER(p);
    return part_settle_shares(*p->p, d_x_mine);
}
int pr_part_settle(pr_part *p, const double *d_x_full, int64_t *settled, int64_t *ints, double *floats) {
    PART_ENTER(p);
    return part_settle(*p->p, d_x_full, settled, ints, floats);
}
int pr_part_total(pr_part *p, int32_t include_pending, double *total) {
    PART_ENTER(p);
    return part_total(*p->p, include_pending, total);
}
int pr_part_export(pr_part *p, double *reserved, double *pending) {
    PART_ENTER(p);
    return part_export(*p->p, reserved, pending);
}
int pr_part_destroy(pr_part *p) {
    if (!p) return PR_OK;
    set_device(part_ctx(*p->p));
    part_destroy(p->p);
    delete p;
    return PR_OK;
}

#ifdef PR_UBENCH  // tools/ubench.cu, variant libraries only (tools/ubench.py)
// diagnostics (not part of the documented ABI): gather microbenchmarks
int pr_debug_gather(pr_graph *g, int variant, int iters, int blocks_per_sm, double *ms_out) {
    CHECK_PTR(g, "graph");
    PR_TRY(set_device(*g->g->ctx));
    return debug_gather(*g->g, variant, iters, blocks_per_sm, ms_out);
}

int pr_debug_graph(pr_ctx *ctx, int variant, int64_t iters, int blocks, double *us_out) {
    CHECK_PTR(ctx, "ctx");
    PR_TRY(set_device(ctx->c));
    return debug_graph(ctx->c, variant, iters, blocks, us_out);
}
#endif

}  // extern "C"
