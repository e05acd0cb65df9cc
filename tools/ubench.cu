// ubench.cu -- microbenchmarks of the gather pattern (diagnostics only; not
// part of the engine).  pr_debug_gather runs variants of a pure gather-sum
// over the run layout's compacted CSC (IFP2 schedule) to separate the
// memory system's limit from the segmented-reduction overhead.
#include <cstdlib>
#include <cstring>

#include "internal.cuh"

namespace pr {

// v0: thread-contiguous 8 edges, 16B index loads, 8 independent gathers
__global__ void ub_gather8(const int32_t *__restrict__ csc, int64_t edges, const double *__restrict__ x,
                           double *__restrict__ out) {
    double acc = 0.0;
    for (int64_t e0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 8; e0 < edges;
         e0 += (int64_t)gridDim.x * blockDim.x * 8) {
        const int4 *p = reinterpret_cast<const int4 *>(csc + e0);
        int4 a = __ldg(p), b = __ldg(p + 1);
        int idx[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (e0 + q < edges) acc += __ldg(&x[idx[q]]);
    }
    if (acc == 123.456) out[0] = acc;
}

// v1: as v0 but 16 edges per thread per step (16 gathers in flight)
__global__ void ub_gather16(const int32_t *__restrict__ csc, int64_t edges, const double *__restrict__ x,
                            double *__restrict__ out) {
    double acc = 0.0;
    for (int64_t e0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 16; e0 < edges;
         e0 += (int64_t)gridDim.x * blockDim.x * 16) {
        const int4 *p = reinterpret_cast<const int4 *>(csc + e0);
        int4 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2), d = __ldg(p + 3);
        int idx[16] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w, d.x, d.y, d.z, d.w};
        double t[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) t[q] = e0 + q < edges ? __ldg(&x[idx[q]]) : 0.0;
#pragma unroll
        for (int q = 0; q < 16; ++q) acc += t[q];
    }
    if (acc == 123.456) out[0] = acc;
}

// v2: coalesced lane-interleaved (e = base + lane + 32q), 8 per lane
__global__ void ub_gather_lanes(const int32_t *__restrict__ csc, int64_t edges, const double *__restrict__ x,
                                double *__restrict__ out) {
    const int lane = threadIdx.x & 31;
    double acc = 0.0;
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = warp * 256; base < edges; base += nw * 256) {
        int idx[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) idx[q] = base + lane + 32 * q < edges ? __ldg(&csc[base + lane + 32 * q]) : -1;
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (idx[q] >= 0) acc += __ldg(&x[idx[q]]);
    }
    if (acc == 123.456) out[0] = acc;
}

// v3: index stream only (no gathers): the CSC read bound
__global__ void ub_stream(const int32_t *__restrict__ csc, int64_t edges, double *__restrict__ out) {
    int acc = 0;
    for (int64_t e0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 8; e0 < edges;
         e0 += (int64_t)gridDim.x * blockDim.x * 8) {
        const int4 *p = reinterpret_cast<const int4 *>(csc + e0);
        int4 a = __ldg(p), b = __ldg(p + 1);
        acc += a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w;
    }
    if (acc == 123456789) out[0] = acc;
}

// v4: as v2, but each gather LDG is issued by one 8-lane group at a time
// (4 predicated LDGs per 32 gathers): wavefronts per LDG <= 8
__global__ void ub_gather_groups8(const int32_t *__restrict__ csc, int64_t edges, const double *__restrict__ x,
                                  double *__restrict__ out) {
    const int lane = threadIdx.x & 31, grp = lane >> 3;
    double acc = 0.0;
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = warp * 256; base < edges; base += nw * 256) {
        int idx[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) idx[q] = base + lane + 32 * q < edges ? __ldg(&csc[base + lane + 32 * q]) : -1;
        double t[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            double v = 0.0;
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                double w;
                const int on = grp == g && idx[q] >= 0;
                asm volatile("{ .reg .pred p; setp.ne.s32 p, %2, 0;\n"
                             "  mov.f64 %0, 0d0000000000000000;\n"
                             "  @p ld.global.nc.f64 %0, [%1]; }"
                             : "=d"(w) : "l"(x + (idx[q] >= 0 ? idx[q] : 0)), "r"(on));
                v += w;
            }
            t[q] = v;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) acc += t[q];
    }
    if (acc == 123.456) out[0] = acc;
}

// v5: uniformly random indices (hash of the edge position): no locality
// v6: sequential x[e mod n]: fully coalesced gathers (the LSU floor)
template <int KIND>
__global__ void ub_gather_synth(int64_t edges, int64_t n, const double *__restrict__ x, double *__restrict__ out) {
    const int lane = threadIdx.x & 31;
    double acc = 0.0;
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = warp * 256; base < edges; base += nw * 256) {
        double t[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint64_t e = (uint64_t)(base + lane + 32 * q);
            uint64_t i;
            if (KIND == 0) {
                uint64_t z = e * 0x9E3779B97F4A7C15ull;
                z = (z ^ (z >> 31)) * 0xBF58476D1CE4E5B9ull;
                i = (z ^ (z >> 29)) % (uint64_t)n;
            } else {
                i = e % (uint64_t)n;
            }
            t[q] = e < (uint64_t)edges ? __ldg(&x[i]) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) acc += t[q];
    }
    if (acc == 123.456) out[0] = acc;
}

// v7-v9: the gather split by source id at H (the run layout's hottest
// sources are the low ids; each row's sources are sorted, so a row's hot
// sources are a prefix of it):
//   MODE 0: cold only -- gathers of ids < H are skipped (no load): the floor
//           of a main pass that leaves the hot prefix to another pass
//   MODE 1: hot only  -- only ids < H are gathered (L1 then holds x[0, H))
//   MODE 2: both, hot ids from a shared-memory copy of x[0, H) filled per block
template <int MODE>
__global__ void __launch_bounds__(1024, 1) ub_gather_split(const int32_t *__restrict__ csc, int64_t edges, const double *__restrict__ x,
                                int H, double *__restrict__ out) {
    extern __shared__ double xs[];
    if (MODE == 2) {
        for (int i = threadIdx.x; i < H; i += blockDim.x) xs[i] = __ldg(&x[i]);
        __syncthreads();
    }
    const int lane = threadIdx.x & 31;
    double acc = 0.0;
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = warp * 256; base < edges; base += nw * 256) {
        int idx[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) idx[q] = base + lane + 32 * q < edges ? __ldcs(&csc[base + lane + 32 * q]) : -1;
        double t[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const bool hot = (unsigned)idx[q] < (unsigned)H;
            if (MODE == 0) t[q] = idx[q] >= 0 && !hot ? __ldg(&x[idx[q]]) : 0.0;
            else if (MODE == 1) t[q] = hot ? __ldg(&x[idx[q]]) : 0.0;
            else {
                // explicit predicated LDS / LDG.NC: a C++ select between the two pointers becomes one
                // generic load, which replays per address space (measured 16 ms per sweep at H = 4096)
                const unsigned sa = (unsigned)__cvta_generic_to_shared(xs) + 8u * (unsigned)(hot ? idx[q] : 0);
                const double *ga = x + (idx[q] >= 0 && !hot ? idx[q] : 0);
                double v;
                asm("{ .reg .pred p; setp.ne.u32 p, %3, 0;\n"
                    "  @p ld.shared.f64 %0, [%1];\n"
                    "  @!p ld.global.nc.f64 %0, [%2]; }"
                    : "=d"(v) : "r"(sa), "l"(ga), "r"((unsigned)hot));
                t[q] = idx[q] < 0 ? 0.0 : v;
            }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) acc += t[q];
    }
    if (acc == 123.456) out[0] = acc;
}

int debug_gather(Graph &g0, int variant, int iters, int blocks_per_sm, double *ms_out) {
    PR_TRY(ensure_run_layout(g0));
    Graph &g = *g0.run;
    PR_TRY(preprocess_ifp2_device(g));
    PR_TRY(ensure_sched(g, 1));
    auto &S = g.sched[1];
    Ctx &ctx = *g.ctx;
    cudaStream_t st = ctx.stream;
    DevBuf x, out;
    PR_TRY(ensure(x, 8 * g.n));
    PR_TRY(ensure(out, 8));
    PR_CUDA(cudaMemsetAsync(x.ptr, 0, 8 * g.n, st));
    unsigned grid = (unsigned)(ctx.sm_count * (blocks_per_sm > 0 ? blocks_per_sm : 8));
    const int H = getenv("PR_UB_H") ? atoi(getenv("PR_UB_H")) : 16384;
    const int TH = getenv("PR_UB_THREADS") ? atoi(getenv("PR_UB_THREADS")) : 256;   // v7-v9 block size
    if (variant == 9 && 8 * H > 48 * 1024)
        PR_CUDA(cudaFuncSetAttribute(ub_gather_split<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * H));
    cudaEvent_t e0, e1;
    PR_CUDA(cudaEventCreate(&e0));
    PR_CUDA(cudaEventCreate(&e1));
    for (int rep = 0; rep < 2; ++rep) {
        PR_CUDA(cudaEventRecord(e0, st));
        for (int it = 0; it < iters; ++it) {
            switch (variant) {
            case 0: ub_gather8<<<grid, 256, 0, st>>>(S.csc.as<int32_t>(), S.edges, x.as<double>(), out.as<double>()); break;
            case 1: ub_gather16<<<grid, 256, 0, st>>>(S.csc.as<int32_t>(), S.edges, x.as<double>(), out.as<double>()); break;
            case 2: ub_gather_lanes<<<grid, 256, 0, st>>>(S.csc.as<int32_t>(), S.edges, x.as<double>(), out.as<double>()); break;
            case 4: ub_gather_groups8<<<grid, 256, 0, st>>>(S.csc.as<int32_t>(), S.edges, x.as<double>(), out.as<double>()); break;
            case 5: ub_gather_synth<0><<<grid, 256, 0, st>>>(S.edges, g.n, x.as<double>(), out.as<double>()); break;
            case 6: ub_gather_synth<1><<<grid, 256, 0, st>>>(S.edges, g.n, x.as<double>(), out.as<double>()); break;
            case 7: ub_gather_split<0><<<grid, TH, 0, st>>>(S.csc.as<int32_t>(), S.edges, x.as<double>(), H, out.as<double>()); break;
            case 8: ub_gather_split<1><<<grid, TH, 0, st>>>(S.csc.as<int32_t>(), S.edges, x.as<double>(), H, out.as<double>()); break;
            case 9: ub_gather_split<2><<<grid, TH, 8 * H, st>>>(S.csc.as<int32_t>(), S.edges, x.as<double>(), H, out.as<double>()); break;
            default: ub_stream<<<grid, 256, 0, st>>>(S.csc.as<int32_t>(), S.edges, out.as<double>()); break;
            }
        }
        PR_CUDA(cudaEventRecord(e1, st));
        PR_CUDA(cudaEventSynchronize(e1));
    }
    float ms = 0.f;
    PR_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *ms_out = ms / iters;
    return PR_OK;
}


// ---- round-loop launch overhead: a trivial "round" kernel whose last block
// decrements a counter and drives the conditional(s), like k_pull's finaliser
struct UbCtl {
    int64_t left;
    uint32_t arrive;
};

__global__ void ub_round(UbCtl *c, cudaGraphConditionalHandle h_loop, cudaGraphConditionalHandle h_sw, int mode) {
    __shared__ bool last;
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(&c->arrive, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    c->arrive = 0;
    if (c->left > 0) c->left -= 1;
    __threadfence();
    if (mode >= 1) cudaGraphSetConditional(h_loop, c->left > 0 ? 1u : 0u);
    if (mode == 2) cudaGraphSetConditional(h_sw, 0u);
}

// same, for programmatic (PDL) edges: trigger early, wait for the upstream grid
__global__ void ub_round_pdl(UbCtl *c, cudaGraphConditionalHandle h_loop, cudaGraphConditionalHandle h_sw, int mode) {
    cudaTriggerProgrammaticLaunchCompletion();
    cudaGridDependencySynchronize();
    __shared__ bool last;
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(&c->arrive, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    c->arrive = 0;
    if (c->left > 0) c->left -= 1;
    __threadfence();
    cudaGraphSetConditional(h_loop, c->left > 0 ? 1u : 0u);
}

__global__ void ub_init(UbCtl *c, int64_t iters) {
    c->left = iters;
    c->arrive = 0;
}

// variant 0: stream launches; 1: WHILE{round}; 2: WHILE{SWITCH{round}};
// 3: WHILE{round x4}; 4: WHILE{round x8}; 5: WHILE{cooperative round};
// 6: WHILE{round x8, programmatic edges}; 7: same with launch-completion port
int debug_graph(Ctx &ctx, int variant, int64_t iters, int blocks, double *us_out) {
    cudaStream_t st = ctx.stream;
    DevBuf cb;
    PR_TRY(ensure(cb, sizeof(UbCtl)));
    UbCtl *c = cb.as<UbCtl>();
    cudaEvent_t e0, e1;
    PR_CUDA(cudaEventCreate(&e0));
    PR_CUDA(cudaEventCreate(&e1));
    cudaGraphExec_t ex = nullptr;
    cudaGraph_t G = nullptr;
    if (variant >= 1) {
        PR_CUDA(cudaGraphCreate(&G, 0));
        cudaGraphConditionalHandle hl = 0, hs = 0;
        PR_CUDA(cudaGraphConditionalHandleCreate(&hl, G, 1, cudaGraphCondAssignDefault));
        if (variant == 2) PR_CUDA(cudaGraphConditionalHandleCreate(&hs, G, 0, cudaGraphCondAssignDefault));
        cudaGraphNode_t n_init, n_while, n_sw, n_k;
        int64_t it64 = iters;
        void *a_init[] = {&c, &it64};
        cudaKernelNodeParams kp = {};
        kp.func = (void *)ub_init;
        kp.gridDim = dim3(1);
        kp.blockDim = dim3(1);
        kp.kernelParams = a_init;
        PR_CUDA(cudaGraphAddKernelNode(&n_init, G, nullptr, 0, &kp));
        cudaGraphNodeParams wp = {};
        wp.type = cudaGraphNodeTypeConditional;
        wp.conditional.handle = hl;
        wp.conditional.type = cudaGraphCondTypeWhile;
        wp.conditional.size = 1;
        PR_CUDA(cudaGraphAddNode(&n_while, G, &n_init, 1, &wp));
        cudaGraph_t body = wp.conditional.phGraph_out[0];
        if (variant == 2) {
            cudaGraphNodeParams sp = {};
            sp.type = cudaGraphNodeTypeConditional;
            sp.conditional.handle = hs;
            sp.conditional.type = cudaGraphCondTypeSwitch;
            sp.conditional.size = 2;
            PR_CUDA(cudaGraphAddNode(&n_sw, body, nullptr, 0, &sp));
            body = sp.conditional.phGraph_out[0];
        }
        int mode = variant == 2 ? 2 : 1;
        void *a_r[] = {&c, &hl, &hs, &mode};
        kp.func = variant >= 6 ? (void *)ub_round_pdl : (void *)ub_round;
        kp.gridDim = dim3((unsigned)blocks);
        kp.blockDim = dim3(256);
        kp.kernelParams = a_r;
        const int copies = variant == 3 ? 4 : (variant == 4 || variant >= 6) ? 8 : 1;
        cudaGraphNode_t prev = nullptr;
        for (int k = 0; k < copies; ++k) {
            if (variant >= 6 && prev) {
                cudaGraphNodeParams np = {};
                np.type = cudaGraphNodeTypeKernel;
                np.kernel.func = kp.func;
                np.kernel.gridDim = kp.gridDim;
                np.kernel.blockDim = kp.blockDim;
                np.kernel.sharedMemBytes = 0;
                np.kernel.kernelParams = kp.kernelParams;
                cudaGraphEdgeData ed = {};
                ed.from_port = variant == 6 ? cudaGraphKernelNodePortProgrammatic : cudaGraphKernelNodePortLaunchCompletion;
                ed.type = cudaGraphDependencyTypeProgrammatic;
                PR_CUDA(cudaGraphAddNode_v2(&n_k, body, &prev, &ed, 1, &np));
                prev = n_k;
                continue;
            }
            PR_CUDA(cudaGraphAddKernelNode(&n_k, body, prev ? &prev : nullptr, prev ? 1 : 0, &kp));
            if (variant == 5) {
                cudaKernelNodeAttrValue v = {};
                v.cooperative = 1;
                PR_CUDA(cudaGraphKernelNodeSetAttribute(n_k, cudaLaunchAttributeCooperative, &v));
            }
            prev = n_k;
        }
        PR_CUDA(cudaGraphInstantiate(&ex, G, 0));
    }
    float ms = 0.f;
    for (int rep = 0; rep < 3; ++rep) {
        PR_CUDA(cudaEventRecord(e0, st));
        if (variant == 0) {
            ub_init<<<1, 1, 0, st>>>(c, iters);
            for (int64_t i = 0; i < iters; ++i) ub_round<<<blocks, 256, 0, st>>>(c, 0, 0, 0);
        } else {
            PR_CUDA(cudaGraphLaunch(ex, st));
        }
        PR_CUDA(cudaEventRecord(e1, st));
        PR_CUDA(cudaEventSynchronize(e1));
        PR_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    }
    if (ex) cudaGraphExecDestroy(ex);
    if (G) cudaGraphDestroy(G);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *us_out = 1e3 * ms / (double)iters;
    return PR_OK;
}

}  // namespace pr

