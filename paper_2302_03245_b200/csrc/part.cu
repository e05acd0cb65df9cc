// part.cu -- local step of the vertex-range partitioned rounds (multi-GPU,
// SURVEY.md §8(e); host orchestration in distributed.py).
//
// A partition owns `owned` vertices and the in-edge rows of them, with
// source ids in the padded global space (rank r's vertices at [r*slot, ...)).
// Each call is one bulk-synchronous step on the context stream:
//   init   -- state 0 (h = 1): drain, shares of the owned slice, statistics
//   round  -- h_v = (active ? 0 : h_v) + sum_{u in in(v)} s_full[u] for owned
//             v (sequential ascending-source sums: the same order as the
//             single-GPU exact engine and np.bincount), then the drain
//   settle -- IFP2: reserved_d = h_d + sum x_full[u] over d's sources
// Statistics are reduced per block and then by one block in fixed order
// (deterministic) and returned to the host, which all-reduces them.
#include <cstring>
#include <vector>

#include "internal.cuh"
#include "reduce.cuh"

namespace pr {

struct Part {
    Ctx *ctx;
    int64_t owned, slot, edges;
    int algorithm;
    double c, xi;
    DevBuf in_off, in_src, deg, row_len, dtc, dang, recv;   // int64 offsets, int32 ids/degrees, uint8 flags
    DevBuf h, reserved, act, partials, stats;
};

struct PartArgs {
    int64_t owned;
    const int64_t *in_off;
    const int32_t *in_src;
    const int32_t *deg, *row_len, *dtc;
    const uint8_t *dang, *recv;
    double *h, *reserved;
    uint8_t *act;
    Partial *partials;
    double c, xi;
};

// per-block statistics of the drain (ints: nact, work, push_ops, push_dang,
// conv_all, conv_scan; floats in l1/above/nd_above)
__device__ __forceinline__ void part_drain(const PartArgs &A, int64_t v, double *s_mine, Partial &p) {
    const double hv = A.h[v];
    const int32_t dv = A.deg[v];
    const bool scan = !A.dang[v];
    const bool above = hv > A.xi;
    p.l1 += hv;
    if (above) {
        p.above += hv;
        if (scan) p.nd_above += hv;
    } else {
        p.conv_all += 1;
        if (scan) p.conv_scan += 1;
    }
    const bool active = above && scan;
    A.act[v] = active;
    if (active) {
        const int32_t len = A.row_len[v];
        A.reserved[v] = __dadd_rn(A.reserved[v], hv);
        s_mine[v] = len > 0 ? __ddiv_rn(__dmul_rn(A.c, hv), (double)dv) : 0.0;
        p.nact += 1;
        p.work += (int64_t)dv + 1;
        p.push_ops += len;
        p.push_dang += A.dtc[v];
    } else {
        s_mine[v] = 0.0;
    }
}

__global__ void __launch_bounds__(256) k_part_init(PartArgs A, double *s_mine) {
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    Partial p;
    zero(p);
    if (v < A.owned) {
        A.h[v] = 1.0;
        A.reserved[v] = 0.0;
        part_drain(A, v, s_mine, p);
    }
    block_reduce(p);
    if (threadIdx.x == 0) A.partials[blockIdx.x] = p;
}

__global__ void __launch_bounds__(256) k_part_round(PartArgs A, const double *__restrict__ s_full, double *s_mine) {
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    Partial p;
    zero(p);
    if (v < A.owned) {
        double acc = 0.0;
        if (A.recv[v])
            for (int64_t e = A.in_off[v]; e < A.in_off[v + 1]; ++e) acc = __dadd_rn(acc, __ldg(&s_full[A.in_src[e]]));
        A.h[v] = __dadd_rn(A.act[v] ? 0.0 : A.h[v], acc);
        part_drain(A, v, s_mine, p);
    }
    block_reduce(p);
    if (threadIdx.x == 0) A.partials[blockIdx.x] = p;
}

__global__ void k_part_shares(PartArgs A, double *x_mine) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < A.owned; v += (int64_t)gridDim.x * blockDim.x)
        x_mine[v] = A.deg[v] > 0 ? __ddiv_rn(__dmul_rn(A.c, A.reserved[v]), (double)A.deg[v]) : 0.0;
}

__global__ void __launch_bounds__(256) k_part_settle(PartArgs A, const double *__restrict__ x_full) {
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    Partial p;
    zero(p);
    if (v < A.owned) {
        if (A.dang[v]) {
            double acc = 0.0;
            for (int64_t e = A.in_off[v]; e < A.in_off[v + 1]; ++e) acc = __dadd_rn(acc, x_full[A.in_src[e]]);
            p.push_ops = A.in_off[v + 1] - A.in_off[v];
            A.reserved[v] = __dadd_rn(A.h[v], acc);
            A.h[v] = 0.0;
        }
        const double hv = A.h[v];
        const bool above = hv > A.xi, scan = !A.dang[v];
        p.l1 = hv;
        if (above) {
            p.above = hv;
            if (scan) p.nd_above = hv;
        } else {
            p.conv_all = 1;
            if (scan) p.conv_scan = 1;
        }
    }
    block_reduce(p);
    if (threadIdx.x == 0) A.partials[blockIdx.x] = p;
}

__global__ void __launch_bounds__(256) k_part_total(PartArgs A, int include_h) {
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    Partial p;
    zero(p);
    if (v < A.owned) p.l1 = include_h ? A.reserved[v] + A.h[v] : A.reserved[v];
    block_reduce(p);
    if (threadIdx.x == 0) A.partials[blockIdx.x] = p;
}

// one block: fixed-order reduction of the block partials
__global__ void k_part_reduce(const Partial *partials, int64_t blocks, Partial *out) {
    Partial acc;
    zero(acc);
    for (int64_t b = threadIdx.x; b < blocks; b += blockDim.x) add(acc, partials[b]);
    block_reduce(acc);
    if (threadIdx.x == 0) *out = acc;
}

static PartArgs args_of(Part &P) {
    PartArgs A;
    A.owned = P.owned;
    A.in_off = P.in_off.as<int64_t>();
    A.in_src = P.in_src.as<int32_t>();
    A.deg = P.deg.as<int32_t>();
    A.row_len = P.row_len.as<int32_t>();
    A.dtc = P.dtc.as<int32_t>();
    A.dang = P.dang.as<uint8_t>();
    A.recv = P.recv.as<uint8_t>();
    A.h = P.h.as<double>();
    A.reserved = P.reserved.as<double>();
    A.act = P.act.as<uint8_t>();
    A.partials = P.partials.as<Partial>();
    A.c = P.c;
    A.xi = P.xi;
    return A;
}

static int finish_stats(Part &P, unsigned blocks, int64_t *ints, double *floats) {
    cudaStream_t st = P.ctx->stream;
    k_part_reduce<<<1, 256, 0, st>>>(P.partials.as<Partial>(), blocks, P.stats.as<Partial>());
    Partial h;
    PR_CUDA(cudaMemcpyAsync(&h, P.stats.ptr, sizeof(h), cudaMemcpyDeviceToHost, st));
    PR_CUDA(cudaStreamSynchronize(st));
    PR_CUDA(cudaGetLastError());
    if (ints) {
        ints[0] = h.nact;
        ints[1] = h.work;
        ints[2] = h.push_ops;
        ints[3] = h.push_dang;
        ints[4] = h.conv_all;
        ints[5] = h.conv_scan;
    }
    if (floats) {
        floats[0] = h.l1;
        floats[1] = h.above;
        floats[2] = h.nd_above;
    }
    return PR_OK;
}

template <class T>
static int upload_as(Ctx &ctx, DevBuf &dst, const int64_t *src, int64_t count) {
    std::vector<T> tmp((size_t)(count > 0 ? count : 1));
    for (int64_t i = 0; i < count; ++i) tmp[(size_t)i] = (T)src[i];
    PR_TRY(ensure(dst, sizeof(T) * (count > 0 ? count : 1)));
    if (count) PR_CUDA(cudaMemcpyAsync(dst.ptr, tmp.data(), sizeof(T) * count, cudaMemcpyHostToDevice, ctx.stream));
    PR_CUDA(cudaStreamSynchronize(ctx.stream));
    return PR_OK;
}

int part_create(Ctx &ctx, int64_t owned, int64_t slot, const int64_t *in_off, const int64_t *in_src, int64_t edges,
                const int64_t *deg, const int64_t *row_len, const int64_t *dtc, const uint8_t *dang,
                const uint8_t *recv, int algorithm, double c, double xi, Part **out) {
    if (owned < 0 || slot < owned) return fail(PR_ERR_ARG, "partition: need 0 <= owned <= slot");
    if (!(c > 0.0 && c < 1.0)) return fail(PR_ERR_ARG, "damping must be in (0,1)");
    if (!(xi > 0.0)) return fail(PR_ERR_ARG, "threshold must be positive");
    Part *P = new Part();
    P->ctx = &ctx;
    P->owned = owned;
    P->slot = slot;
    P->edges = edges;
    P->algorithm = algorithm;
    P->c = c;
    P->xi = xi;
    int rc = PR_OK;
    do {
        if ((rc = ensure(P->in_off, 8 * (owned + 1)))) break;
        if (cudaMemcpyAsync(P->in_off.ptr, in_off, 8 * (owned + 1), cudaMemcpyHostToDevice, ctx.stream) != cudaSuccess) {
            rc = fail(PR_ERR_CUDA, "partition upload");
            break;
        }
        if ((rc = upload_as<int32_t>(ctx, P->in_src, in_src, edges))) break;
        if ((rc = upload_as<int32_t>(ctx, P->deg, deg, owned))) break;
        if ((rc = upload_as<int32_t>(ctx, P->row_len, row_len, owned))) break;
        if ((rc = upload_as<int32_t>(ctx, P->dtc, dtc, owned))) break;
        if ((rc = ensure(P->dang, owned ? owned : 1))) break;
        if ((rc = ensure(P->recv, owned ? owned : 1))) break;
        if (owned) {
            cudaMemcpyAsync(P->dang.ptr, dang, owned, cudaMemcpyHostToDevice, ctx.stream);
            cudaMemcpyAsync(P->recv.ptr, recv, owned, cudaMemcpyHostToDevice, ctx.stream);
        }
        if ((rc = ensure(P->h, 8 * (owned ? owned : 1)))) break;
        if ((rc = ensure(P->reserved, 8 * (owned ? owned : 1)))) break;
        if ((rc = ensure(P->act, owned ? owned : 1))) break;
        if ((rc = ensure(P->partials, sizeof(Partial) * (grid_for(owned, 256) + 1)))) break;
        if ((rc = ensure(P->stats, sizeof(Partial)))) break;
        if (cudaStreamSynchronize(ctx.stream) != cudaSuccess) rc = fail(PR_ERR_CUDA, "partition upload");
    } while (0);
    if (rc) { delete P; return rc; }
    *out = P;
    return PR_OK;
}

int part_init(Part &P, double *d_s_mine, int64_t *ints, double *floats) {
    unsigned g = grid_for(P.owned, 256);
    k_part_init<<<g, 256, 0, P.ctx->stream>>>(args_of(P), d_s_mine);
    return finish_stats(P, g, ints, floats);
}

int part_round(Part &P, const double *d_s_full, double *d_s_mine, int64_t *ints, double *floats) {
    unsigned g = grid_for(P.owned, 256);
    k_part_round<<<g, 256, 0, P.ctx->stream>>>(args_of(P), d_s_full, d_s_mine);
    return finish_stats(P, g, ints, floats);
}

int part_settle_shares(Part &P, double *d_x_mine) {
    k_part_shares<<<grid_for(P.owned, 256), 256, 0, P.ctx->stream>>>(args_of(P), d_x_mine);
    PR_CUDA(cudaStreamSynchronize(P.ctx->stream));
    return PR_OK;
}

int part_settle(Part &P, const double *d_x_full, int64_t *settled, int64_t *ints, double *floats) {
    unsigned g = grid_for(P.owned, 256);
    k_part_settle<<<g, 256, 0, P.ctx->stream>>>(args_of(P), d_x_full);
    int64_t tmp[6];
    PR_TRY(finish_stats(P, g, tmp, floats));
    if (settled) *settled = tmp[2];
    if (ints) memcpy(ints, tmp, sizeof(tmp));
    return PR_OK;
}

int part_total(Part &P, int include_h, double *total) {
    unsigned g = grid_for(P.owned, 256);
    k_part_total<<<g, 256, 0, P.ctx->stream>>>(args_of(P), include_h);
    double f[3];
    PR_TRY(finish_stats(P, g, nullptr, f));
    *total = f[0];
    return PR_OK;
}

int part_export(Part &P, double *reserved, double *pending) {
    cudaStream_t st = P.ctx->stream;
    if (reserved && P.owned)
        PR_CUDA(cudaMemcpyAsync(reserved, P.reserved.ptr, 8 * P.owned, cudaMemcpyDeviceToHost, st));
    if (pending && P.owned) PR_CUDA(cudaMemcpyAsync(pending, P.h.ptr, 8 * P.owned, cudaMemcpyDeviceToHost, st));
    PR_CUDA(cudaStreamSynchronize(st));
    return PR_OK;
}

void part_destroy(Part *P) {
    if (!P) return;
    cudaStreamSynchronize(P->ctx->stream);
    delete P;
}

Ctx &part_ctx(Part &P) { return *P.ctx; }

}  // namespace pr
