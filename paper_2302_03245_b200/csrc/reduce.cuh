// reduce.cuh -- deterministic block / grid reductions shared by the round
// engine and the power method.
#pragma once

#include "internal.cuh"

namespace pr {

// ---------------------------------------------------------------- helpers

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void zero(Partial &p) {
    p.l1 = p.above = p.nd_above = 0.0;
    p.conv_all = p.conv_scan = p.nact = p.work = p.push_ops = p.push_dang = 0;
    p.digest = 0;
}

__device__ __forceinline__ void add(Partial &a, const Partial &b) {
    a.l1 += b.l1;
    a.above += b.above;
    a.nd_above += b.nd_above;
    a.conv_all += b.conv_all;
    a.conv_scan += b.conv_scan;
    a.nact += b.nact;
    a.work += b.work;
    a.push_ops += b.push_ops;
    a.push_dang += b.push_dang;
    a.digest += b.digest;
}

// L1-bypassing load of a partial written by another block of this grid
__device__ __forceinline__ Partial load_partial(const Partial *q) {
    Partial p;
    p.l1 = __ldcg(&q->l1);
    p.above = __ldcg(&q->above);
    p.nd_above = __ldcg(&q->nd_above);
    p.conv_all = __ldcg((const long long *)&q->conv_all);
    p.conv_scan = __ldcg((const long long *)&q->conv_scan);
    p.nact = __ldcg((const long long *)&q->nact);
    p.work = __ldcg((const long long *)&q->work);
    p.push_ops = __ldcg((const long long *)&q->push_ops);
    p.push_dang = __ldcg((const long long *)&q->push_dang);
    p.digest = __ldcg((const unsigned long long *)&q->digest);
    return p;
}

__device__ __forceinline__ void shfl_add(Partial &p, int o) {
    p.l1 += __shfl_down_sync(0xffffffffu, p.l1, o);
    p.above += __shfl_down_sync(0xffffffffu, p.above, o);
    p.nd_above += __shfl_down_sync(0xffffffffu, p.nd_above, o);
    p.conv_all += __shfl_down_sync(0xffffffffu, p.conv_all, o);
    p.conv_scan += __shfl_down_sync(0xffffffffu, p.conv_scan, o);
    p.nact += __shfl_down_sync(0xffffffffu, p.nact, o);
    p.work += __shfl_down_sync(0xffffffffu, p.work, o);
    p.push_ops += __shfl_down_sync(0xffffffffu, p.push_ops, o);
    p.push_dang += __shfl_down_sync(0xffffffffu, p.push_dang, o);
    p.digest += __shfl_down_sync(0xffffffffu, p.digest, o);
}

// Fixed-order block reduction (deterministic); result valid in thread 0.
// All threads of the block must call it.
static __device__ void block_reduce(Partial &p) {
    __shared__ Partial warp_part[32];
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int o = 16; o > 0; o >>= 1) shfl_add(p, o);
    __syncthreads();
    if (lane == 0) warp_part[wid] = p;
    __syncthreads();
    if (wid == 0) {
        int nw = (blockDim.x + 31) >> 5;
        if (lane < nw) p = warp_part[lane]; else zero(p);
        for (int o = 16; o > 0; o >>= 1) shfl_add(p, o);
    }
}

}  // namespace pr
