// cubutil.cuh -- run CUB device algorithms with the context's scratch buffer.
#pragma once

#include "internal.cuh"

namespace pr {

// size query, grow ctx scratch, execute
template <class F> static int cub_run(Ctx &ctx, F &&f) {
    size_t bytes = 0;
    PR_CUDA(f((void *)nullptr, bytes));
    PR_TRY(ensure(ctx.scratch, bytes));
    PR_CUDA(f(ctx.scratch.ptr, bytes));
    return PR_OK;
}

#define GRID_STRIDE(i, count) \
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (count); i += (int64_t)gridDim.x * blockDim.x)

}  // namespace pr
