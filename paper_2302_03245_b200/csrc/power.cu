// power.cu -- K8: the Power-method baseline (solvers.py:186-243) on the
// same degree-binned CSC gather as the dense push round.
//
// Per iteration (solvers.py:217-235):
//   z_u   = (c * pi_u) * inv_deg_u            (solvers.py:173, inv_deg = 1/deg or 0)
//   y_v   = sum_{u in in(v)} z_u               (_WalkMultiplier, in-adjacency order)
//   nxt_v = y_v + restart * p_v,  restart = c * sum_{dangling} pi + (1 - c)
//   pi'   = nxt / sum(nxt);  delta = ||pi' - pi||_1
// Two launches per iteration: gather (+ sum of nxt) and normalise (+ delta,
// converged count, next z, next dangling sum); both end with a
// deterministic last-block reduction that also drives the graph's WHILE node.
#include <algorithm>
#include <climits>
#include <cstring>
#include <vector>

#include "internal.cuh"
#include "reduce.cuh"
#include "bins.cuh"

namespace pr {

struct PowCtl {
    int64_t k;               // iteration index
    uint32_t blocks_done;
    int32_t done;
    double total;            // sum(nxt) of the current iteration
    double restart;          // restart coefficient for the current iteration
    double delta;
    unsigned long long unit_ctr;  // gather-unit dispatch counter (bins.cuh)
    unsigned long long err_bits;  // max relative error vs ref of this iteration (bits of a double >= 0)
    int64_t hit;                  // first k+1 whose iterate beat target_err (0: none)
};

struct PowArgs {
    int64_t n;
    const int64_t *in_off;
    const int32_t *in_src;
    const int32_t *deg;
    BinView T;               // rows with in-degree > 0
    const int32_t *zero_ids; // in-degree-0 vertices: nxt = restart * p
    int64_t n_zero;
    const double *p;         // personalization (null: uniform 1/n)
    double *pi, *nxt, *z;
    double *deltas;          // device [iterations]
    int64_t *conv;           // device [iterations]
    Partial *partials;
    PowCtl *ctl;
    double c, tolerance, threshold, uniform_p;
    const double *ref;       // target mode (bench.py:255-275): reference vector or null
    double target_err;
    int64_t iterations;
    int32_t use_graph;
    cudaGraphConditionalHandle h_loop;
};

__device__ __forceinline__ double pval(const PowArgs &A, int64_t v) { return A.p ? A.p[v] : A.uniform_p; }

__device__ __forceinline__ double z_of(const PowArgs &A, int64_t v, double x) {
    int32_t d = A.deg[v];
    double inv = d > 0 ? __ddiv_rn(1.0, (double)d) : 0.0;
    return __dmul_rn(__dmul_rn(A.c, x), inv);
}

// last-block protocol over Partial.l1 (sum) / .above (second sum) / .conv_all
template <class Fin>
__device__ void pow_finish(const PowArgs &A, Partial p, Fin fin) {
    __shared__ bool is_last;
    block_reduce(p);
    if (threadIdx.x == 0) {
        A.partials[blockIdx.x] = p;
        __threadfence();
        unsigned t = atomicAdd(&A.ctl->blocks_done, 1u);
        is_last = t == gridDim.x - 1;
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    Partial acc;
    zero(acc);
    for (int64_t b = threadIdx.x; b < gridDim.x; b += blockDim.x) add(acc, load_partial(A.partials + b));
    block_reduce(acc);
    if (threadIdx.x == 0) {
        A.ctl->blocks_done = 0;
        fin(acc);
    }
}

// pi = p; z = (c p) inv_deg; restart from the dangling mass of p
__global__ void __launch_bounds__(256) k_pw_init(PowArgs A) {
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    Partial p;
    zero(p);
    if (v < A.n) {
        double x = pval(A, v);
        A.pi[v] = x;
        A.z[v] = z_of(A, v, x);
        if (A.deg[v] == 0) p.l1 = x;
    }
    pow_finish(A, p, [&](const Partial &acc) {
        A.ctl->k = 0;
        A.ctl->done = A.iterations <= 0;
        A.ctl->restart = __dadd_rn(__dmul_rn(A.c, acc.l1), 1.0 - A.c);  // solvers.py:219
        if (A.use_graph) cudaGraphSetConditional(A.h_loop, A.ctl->done ? 0u : 1u);
    });
}

// nxt_v = sum z over in-edges + restart * p_v; block partial of sum(nxt)
template <bool STREAM>
__global__ void __launch_bounds__(256, 4) k_pw_gather(PowArgs A) {
    if (A.use_graph && ((volatile PowCtl *)A.ctl)->done) return;  // unrolled slot after the stop
    const double restart = A.ctl->restart;
    Partial p;
    zero(p);
    auto finish = [&](int32_t v, double sum) {
        double x = __dadd_rn(sum, __dmul_rn(restart, pval(A, v)));
        A.nxt[v] = x;
        p.l1 += x;
    };
    auto thread_row = [&](bool valid, int64_t row, double sum) {
        if (valid) finish(__ldg(&A.T.ids[row]), sum);
    };
    auto single_row = [&](int64_t row, double sum) { finish(__ldg(&A.T.ids[row]), sum); };
    const Src src{A.z, A.z, 0, 0};
    bins_run_plain<STREAM, 0>(A.T, 0, A.T.n_units, src, thread_row, single_row);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < A.n_zero;
         i += (int64_t)gridDim.x * blockDim.x)
        finish(A.zero_ids[i], 0.0);
    pow_finish(A, p, [&](const Partial &acc) {
        A.ctl->total = acc.l1;
        A.ctl->unit_ctr = 0;
    });
}

// pi' = nxt / total; delta, converged count; next z and dangling sum
__global__ void __launch_bounds__(256) k_pw_norm(PowArgs A) {
    if (A.use_graph && ((volatile PowCtl *)A.ctl)->done) return;
    double total = A.ctl->total;
    Partial p;
    zero(p);
    double err = 0.0;                                   // max |pi - ref| / ref (bench.py:266)
    // grid-stride over one resident wave (few partials for the last block)
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < A.n; v += (int64_t)gridDim.x * blockDim.x) {
        double x = __ddiv_rn(A.nxt[v], total);
        double d = fabs(x - A.pi[v]);
        p.l1 += d;                                      // delta (solvers.py:222)
        p.conv_all += d <= A.threshold ? 1 : 0;         // solvers.py:227
        A.pi[v] = x;
        A.z[v] = z_of(A, v, x);
        if (A.deg[v] == 0) p.above += x;                // dangling mass for the next restart
        if (A.ref) {
            const double r = A.ref[v];
            err = fmax(err, __ddiv_rn(fabs(x - r), r));
        }
    }
    if (A.ref) {
        // max is order-free: non-negative doubles order as their bit patterns
        for (int o = 16; o > 0; o >>= 1) err = fmax(err, __shfl_xor_sync(0xffffffffu, err, o));
        if ((threadIdx.x & 31) == 0 && err > 0.0)
            atomicMax(&A.ctl->err_bits, (unsigned long long)__double_as_longlong(err));
    }
    pow_finish(A, p, [&](const Partial &acc) {
        PowCtl *c = A.ctl;
        int64_t k = c->k;
        A.deltas[k] = acc.l1;
        A.conv[k] = acc.conv_all;
        c->delta = acc.l1;
        c->restart = __dadd_rn(__dmul_rn(A.c, acc.above), 1.0 - A.c);
        c->k = k + 1;
        bool stop = (k + 1 >= A.iterations) || (A.tolerance > 0.0 && acc.l1 < A.tolerance);
        if (A.ref) {
            // bench.py:263-268: the probe stops at the first iterate below the target
            const double e = __longlong_as_double((long long)__ldcg(&c->err_bits));
            c->err_bits = 0;
            if (e < A.target_err) {
                c->hit = k + 1;
                stop = true;
            }
        }
        c->done = stop;
        if (A.use_graph) cudaGraphSetConditional(A.h_loop, stop ? 0u : 1u);
    });
}

static int add_node(cudaGraph_t g, cudaGraphNode_t *node, const cudaGraphNode_t *deps, size_t nd, void *f,
                    unsigned grid, void **args, size_t smem = 0) {
    cudaKernelNodeParams kp;
    memset(&kp, 0, sizeof(kp));
    kp.func = f;
    kp.gridDim = dim3(grid);
    kp.blockDim = dim3(256);
    kp.sharedMemBytes = (unsigned)smem;
    kp.kernelParams = args;
    PR_CUDA(cudaGraphAddKernelNode(node, g, deps, nd, &kp));
    return PR_OK;
}

int power_device(Graph &g, double damping, int64_t iterations, double tolerance, double threshold,
                 const double *h_p, double *h_pi, double *h_deltas, int64_t *h_conv,
                 int (*on_iterate)(void *, int64_t, const double *), void *user, pr_run_result *res,
                 const double *d_ref, double target_err, int64_t *hit) {
    if (!(damping > 0.0 && damping < 1.0)) return fail(PR_ERR_ARG, "damping must be in (0,1)");
    if (iterations < 0) return fail(PR_ERR_ARG, "max_iterations must be non-negative");
    Ctx &ctx = *g.ctx;
    cudaStream_t st = ctx.stream;
    int per_sm = 0;
    PR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pw_gather<false>, 256, 0));
    if (per_sm < 1) per_sm = 1;
    PR_TRY(ensure_sched(g, 2));
    auto &S = g.sched[2];
    int64_t n = g.n;
    PowArgs A;
    memset(&A, 0, sizeof(A));
    const int64_t blk = (int64_t)ctx.sm_count * per_sm;
    PR_TRY(ensure_units(g, 2, blk));
    // stream the CSC when an iteration's working set overflows L2 (bins.cuh)
    const bool stream = 4.0 * (double)S.edges + 16.0 * (double)n >
                        0.6 * (double)(ctx.l2_bytes ? ctx.l2_bytes : (size_t)126 << 20);
    const void *gather_fn = stream ? (const void *)k_pw_gather<true> : (const void *)k_pw_gather<false>;
    int64_t maxb = blk > (n + 255) / 256 ? blk : (n + 255) / 256;
    int64_t it_cap = iterations > 0 ? iterations : 1;
    // workspace: pi, nxt, z, p (opt), deltas, conv, partials, ctl
    size_t off_pi = 0, off_nxt = off_pi + 8 * n, off_z = off_nxt + 8 * n, off_p = off_z + 8 * n;
    size_t off_d = off_p + (h_p ? 8 * n : 0), off_c = off_d + 8 * it_cap, off_part = off_c + 8 * it_cap;
    size_t off_ctl = off_part + sizeof(Partial) * (maxb + 8);
    size_t total = off_ctl + sizeof(PowCtl) + 64;
    PR_TRY(ensure(g.pw, total));
    char *base = g.pw.as<char>();
    A.n = n;
    A.in_off = g.in_off.as<int64_t>();
    A.in_src = g.in_src.as<int32_t>();
    A.deg = g.out_deg.as<int32_t>();
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
    A.zero_ids = S.zero_ids.as<int32_t>();
    A.n_zero = S.n_zero;
    A.pi = (double *)(base + off_pi);
    A.nxt = (double *)(base + off_nxt);
    A.z = (double *)(base + off_z);
    A.p = h_p ? (const double *)(base + off_p) : nullptr;
    A.deltas = (double *)(base + off_d);
    A.conv = (int64_t *)(base + off_c);
    A.partials = (Partial *)(base + off_part);
    A.ctl = (PowCtl *)(base + off_ctl);
    A.T.unit_ctr = &A.ctl->unit_ctr;
    A.c = damping;
    A.tolerance = tolerance;
    A.threshold = threshold;
    A.uniform_p = 1.0 / (double)n;
    A.iterations = iterations;
    A.ref = d_ref;
    A.target_err = target_err;
    if (h_p) PR_CUDA(cudaMemcpyAsync((void *)A.p, h_p, 8 * n, cudaMemcpyHostToDevice, st));
    PR_CUDA(cudaMemsetAsync(A.ctl, 0, sizeof(PowCtl), st));
    unsigned g_all = grid_for(n, 256), g_gather = (unsigned)blk;
    int occ_norm = 0;
    PR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_norm, k_pw_norm, 256, 0));
    const unsigned wave = (unsigned)(ctx.sm_count * (occ_norm > 0 ? occ_norm : 1));
    const unsigned g_norm = g_all < wave ? g_all : wave;

    cudaEvent_t e0, e1;
    PR_CUDA(cudaEventCreate(&e0));
    PR_CUDA(cudaEventCreate(&e1));
    if (on_iterate) {
        // host-driven iterations with a host copy of every iterate (solvers.py:232-233)
        A.use_graph = 0;
        std::vector<double> host_pi((size_t)n);
        PR_CUDA(cudaEventRecord(e0, st));
        k_pw_init<<<g_all, 256, 0, st>>>(A);
        for (int64_t k = 0; k < iterations; ++k) {
            if (stream) k_pw_gather<true><<<g_gather, 256, 0, st>>>(A);
            else k_pw_gather<false><<<g_gather, 256, 0, st>>>(A);
            k_pw_norm<<<g_norm, 256, 0, st>>>(A);
            PR_CUDA(cudaGetLastError());
            PowCtl hc;
            PR_CUDA(cudaMemcpyAsync(&hc, A.ctl, sizeof(hc), cudaMemcpyDeviceToHost, st));
            PR_CUDA(cudaMemcpyAsync(host_pi.data(), A.pi, 8 * n, cudaMemcpyDeviceToHost, st));
            PR_CUDA(cudaStreamSynchronize(st));
            if (on_iterate(user, k, host_pi.data())) break;
            if (hc.done) break;
        }
        PR_CUDA(cudaEventRecord(e1, st));
        PR_CUDA(cudaEventSynchronize(e1));
    } else {
        cudaGraph_t G;
        PR_CUDA(cudaGraphCreate(&G, 0));
        PR_CUDA(cudaGraphConditionalHandleCreate(&A.h_loop, G, 1, cudaGraphCondAssignDefault));
        A.use_graph = 1;
        void *args[] = {&A};
        cudaGraphNode_t n_init, n_while, n_a, n_b;
        PR_TRY(add_node(G, &n_init, nullptr, 0, (void *)k_pw_init, g_all, args));
        cudaGraphNodeParams wp = {};
        wp.type = cudaGraphNodeTypeConditional;
        wp.conditional.handle = A.h_loop;
        wp.conditional.type = cudaGraphCondTypeWhile;
        wp.conditional.size = 1;
        PR_CUDA(cudaGraphAddNode(&n_while, G, &n_init, 1, &wp));
        cudaGraph_t body = wp.conditional.phGraph_out[0];
        // body unrolled into plain kernel nodes (a conditional iteration
        // costs more than a kernel launch; slots after the stop exit at once)
        cudaGraphNode_t prev = nullptr;
        for (int k = 0; k < 4; ++k) {
            PR_TRY(add_node(body, &n_a, prev ? &prev : nullptr, prev ? 1 : 0, (void *)gather_fn, g_gather, args));
            PR_TRY(add_node(body, &n_b, &n_a, 1, (void *)k_pw_norm, g_norm, args));
            prev = n_b;
        }
        cudaGraphExec_t ex;
        PR_CUDA(cudaGraphInstantiate(&ex, G, 0));
        PR_CUDA(cudaEventRecord(e0, st));
        cudaError_t le = cudaGraphLaunch(ex, st);
        PR_CUDA(cudaEventRecord(e1, st));
        cudaError_t se = cudaEventSynchronize(e1);
        cudaGraphExecDestroy(ex);
        cudaGraphDestroy(G);
        PR_CUDA(le);
        PR_CUDA(se);
    }
    float ms = 0.f;
    PR_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    PowCtl hc;
    PR_CUDA(cudaMemcpy(&hc, A.ctl, sizeof(hc), cudaMemcpyDeviceToHost));
    int64_t k = hc.k;
    if (hit) *hit = hc.hit;
    if (h_pi) PR_CUDA(cudaMemcpy(h_pi, A.pi, 8 * n, cudaMemcpyDeviceToHost));
    if (h_deltas && k) PR_CUDA(cudaMemcpy(h_deltas, A.deltas, 8 * k, cudaMemcpyDeviceToHost));
    if (h_conv && k) PR_CUDA(cudaMemcpy(h_conv, A.conv, 8 * k, cudaMemcpyDeviceToHost));
    if (res) {
        memset(res, 0, sizeof(*res));
        memset(res, 0, sizeof(*res));
        res->rounds = k;
        res->rows = k;
        res->push_ops = k * g.m;
        res->mass_total = 1.0;
        res->push_ms = ms;
        res->round_ms = ms;
        res->bytes_moved = (double)k * (12.0 * (double)g.m + 32.0 * (double)n);
    }
    return PR_OK;
}

// ---------------------------------------------------------------------------
// max_relative_error (bench.py:90-112): ERR = max_v |est_v - ref_v| / ref_v,
// its first argmax (np.argmax), the L1 error, and the count of ref_v <= 0
// (the reference raises on any).  Per-element arithmetic is the reference's
// (one subtraction, fabs, one division), so ERR and the worst vertex are
// bit-identical for equal inputs; the L1 sum runs in a fixed order (a fixed
// grid, then one block over the block partials), not numpy's pairwise order.
struct ErrPart {
    double rel, l1;
    int64_t worst, nonpos;
};

__device__ __forceinline__ void err_merge(ErrPart &a, const ErrPart &b) {
    // larger error wins; ties go to the smaller index (np.argmax is the first)
    if (b.rel > a.rel || (b.rel == a.rel && b.worst < a.worst)) {
        a.rel = b.rel;
        a.worst = b.worst;
    }
    a.l1 += b.l1;
    a.nonpos += b.nonpos;
}

__device__ void err_block(ErrPart &p) {
    __shared__ ErrPart wp[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int o = 16; o > 0; o >>= 1) {
        ErrPart q;
        q.rel = __shfl_down_sync(0xffffffffu, p.rel, o);
        q.l1 = __shfl_down_sync(0xffffffffu, p.l1, o);
        q.worst = __shfl_down_sync(0xffffffffu, p.worst, o);
        q.nonpos = __shfl_down_sync(0xffffffffu, p.nonpos, o);
        if (lane + o < 32) err_merge(p, q);
    }
    __syncthreads();
    if (lane == 0) wp[wid] = p;
    __syncthreads();
    if (threadIdx.x == 0)
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) err_merge(p, wp[w]);
}

__global__ void __launch_bounds__(256) k_err(const double *est, const double *ref, int64_t n, ErrPart *parts) {
    ErrPart p{0.0, 0.0, INT64_MAX, 0};
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const double r = ref[v], d = fabs(est[v] - r);
        const double rel = __ddiv_rn(d, r);
        if (rel > p.rel || p.worst == INT64_MAX) {
            p.rel = rel;
            p.worst = v;
        }
        p.l1 += d;
        p.nonpos += r <= 0.0 ? 1 : 0;
    }
    err_block(p);
    if (threadIdx.x == 0) parts[blockIdx.x] = p;
}

__global__ void __launch_bounds__(256) k_err_final(ErrPart *parts, int nb) {
    ErrPart p{0.0, 0.0, INT64_MAX, 0};
    for (int b = threadIdx.x; b < nb; b += blockDim.x) err_merge(p, parts[b]);
    err_block(p);
    if (threadIdx.x == 0) parts[nb] = p;
}

int error_report(Ctx &ctx, const double *d_est, const double *d_ref, int64_t n, double *max_rel, double *l1,
                 int64_t *worst, int64_t *nonpositive) {
    if (n <= 0) return fail(PR_ERR_ARG, "empty vectors");
    const int nb = (int)std::min<int64_t>((int64_t)ctx.sm_count * 4, (n + 255) / 256);
    PR_TRY(ensure(ctx.scratch, sizeof(ErrPart) * (nb + 1)));
    ErrPart *parts = ctx.scratch.as<ErrPart>();
    k_err<<<nb, 256, 0, ctx.stream>>>(d_est, d_ref, n, parts);
    k_err_final<<<1, 256, 0, ctx.stream>>>(parts, nb);
    PR_CUDA(cudaGetLastError());
    ErrPart h;
    PR_CUDA(cudaMemcpyAsync(&h, parts + nb, sizeof(h), cudaMemcpyDeviceToHost, ctx.stream));
    PR_CUDA(cudaStreamSynchronize(ctx.stream));
    if (max_rel) *max_rel = h.rel;
    if (l1) *l1 = h.l1;
    if (worst) *worst = h.worst;
    if (nonpositive) *nonpositive = h.nonpos;
    return PR_OK;
}

}  // namespace pr
