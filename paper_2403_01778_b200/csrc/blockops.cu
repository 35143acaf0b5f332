// Operations on the block matrix J(u) = (1/(d-1)) [B(m,n)] kept in HBM as its
// upper blocks (pair order, column-major; nepv.cpp:81-157).  All reductions
// use fixed grids and fixed-order trees: bit-reproducible, no atomics.
//
//   sumsq_device     sum of squares of a vector (||J||_F^2 * (d-1)^2 / 2)
//   block_matvec     y = J x      (SymBlockMatrix::matvec, nepv.cpp:110-134)
//   dot_device       x'y
#include "common.cuh"
#include "blockmv.cuh"

namespace r1 {

namespace {

constexpr int kRedBlocks = 296;  // fixed partial count (2 waves of 148 SMs)
constexpr int kRedThreads = 256;

__device__ __forceinline__ double block_sum(double v, double* sh) {
    // fixed-order tree: warp xor-butterfly then warp partials in order
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0) {
        const int nw = blockDim.x >> 5;
        for (int w = 0; w < nw; ++w) s += sh[w];
    }
    __syncthreads();
    return s;  // valid in thread 0
}

__global__ void sumsq_partial_kernel(const double* __restrict__ x, uint64_t n,
                                     double* __restrict__ part) {
    __shared__ double sh[32];
    double s = 0.0;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        s = fma(x[i], x[i], s);
    s = block_sum(s, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void dot_partial_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                   uint64_t n, double* __restrict__ part) {
    __shared__ double sh[32];
    double s = 0.0;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        s = fma(x[i], y[i], s);
    s = block_sum(s, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void sum_partials_kernel(const double* __restrict__ part, int n, double* out) {
    __shared__ double sh[32];
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
    s = block_sum(s, sh);
    if (threadIdx.x == 0) *out = s;
}

// ---- block matvec (blockmv.cuh), two launches over a fixed grid ----------
__global__ void mv_phase_a_kernel(const BlockOp* __restrict__ op, const double* __restrict__ x) {
    blockop_phase_a(*op, x);
}

__global__ void mv_phase_b_kernel(const BlockOp* __restrict__ op, double* __restrict__ y) {
    blockop_phase_b(*op, y, blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x,
                    static_cast<int64_t>(gridDim.x) * blockDim.x);
}

struct MvPlan {
    BlockOp op;
    DeviceBuffer coldot, rowpart;
    DescCache<BlockOp> dop;  // one device descriptor per block buffer in use
};

std::map<std::pair<r1_context*, std::vector<uint64_t>>, std::shared_ptr<MvPlan>>& mv_plans() {
    static std::map<std::pair<r1_context*, std::vector<uint64_t>>, std::shared_ptr<MvPlan>> m;
    return m;
}

}  // namespace

void sumsq_device(r1_context* ctx, const double* x, uint64_t n, double* out_dev) {
    ctx->ws_small.ensure(64 * 1024);
    double* part = ctx->ws_small.as<double>() + 1024;
    sumsq_partial_kernel<<<kRedBlocks, kRedThreads, 0, ctx->stream>>>(x, n, part);
    check_launch(ctx, "sumsq_partial_kernel");
    sum_partials_kernel<<<1, kRedThreads, 0, ctx->stream>>>(part, kRedBlocks, out_dev);
    check_launch(ctx, "sum_partials_kernel");
}

void dot_device(r1_context* ctx, const double* x, const double* y, uint64_t n, double* out_dev) {
    ctx->ws_small.ensure(64 * 1024);
    double* part = ctx->ws_small.as<double>() + 2048;
    dot_partial_kernel<<<kRedBlocks, kRedThreads, 0, ctx->stream>>>(x, y, n, part);
    check_launch(ctx, "dot_partial_kernel");
    sum_partials_kernel<<<1, kRedThreads, 0, ctx->stream>>>(part, kRedBlocks, out_dev);
    check_launch(ctx, "sum_partials_kernel");
}

void block_matvec(r1_context* ctx, const uint64_t* dims, int order, const double* blocks,
                  const double* x, double* y) {
    if (order < 2 || order > 16) fail(R1_ERR_INVALID_ARGUMENT, "block_matvec: bad order");
    std::lock_guard<std::mutex> cache_lock(cache_mutex());
    auto& P = mv_plans()[{ctx, std::vector<uint64_t>(dims, dims + order)}];
    if (!P) {
        P = std::make_shared<MvPlan>();
        int64_t cn = 0, rn = 0;
        blockop_layout(P->op, dims, order, &cn, &rn);
        P->coldot.ensure(std::max<int64_t>(cn, 1) * sizeof(double));
        P->rowpart.ensure(std::max<int64_t>(rn, 1) * sizeof(double));
        P->op.coldot = P->coldot.as<double>();
        P->op.rowpart = P->rowpart.as<double>();
    }
    P->op.blocks = blocks;
    const BlockOp* dop = P->dop.get(P->op, ctx->stream);
    const int ga = std::max(1, std::min(P->op.ntasks, 4 * ctx->num_sms));
    mv_phase_a_kernel<<<ga, 256, 0, ctx->stream>>>(dop, x);
    check_launch(ctx, "mv_phase_a_kernel");
    const int gb = static_cast<int>(std::min<int64_t>((P->op.n + 255) / 256, 1024));
    mv_phase_b_kernel<<<std::max(gb, 1), 256, 0, ctx->stream>>>(dop, y);
    check_launch(ctx, "mv_phase_b_kernel");
}

void forget_matvec_plans(r1_context* ctx) {
    std::lock_guard<std::mutex> cache_lock(cache_mutex());
    auto& plans = mv_plans();
    for (auto it = plans.begin(); it != plans.end();)
        if (it->first.first == ctx)
            it = plans.erase(it);
        else
            ++it;
}

}  // namespace r1
