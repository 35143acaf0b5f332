// Operations on the block matrix J(u) = (1/(d-1)) [B(m,n)] kept in HBM as its
// upper blocks (pair order, column-major; nepv.cpp:81-157).  All reductions
// use fixed grids and fixed-order trees: bit-reproducible, no atomics.
//
//   sumsq_device     sum of squares of a vector (||J||_F^2 * (d-1)^2 / 2)
//   block_matvec     y = J x      (SymBlockMatrix::matvec, nepv.cpp:110-134)
//   dot_device       x'y
#include "common.cuh"

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

// ---- block matvec ---------------------------------------------------------
// Pass 1: one CTA per (block, 64-column chunk): column dots (B' x_m)[j] for
// the chunk's columns (complete), and row partials (B x_n)[i] over the chunk.
// Pass 2: each output entry sums its contributions in a fixed order.
constexpr int kMvChunk = 64;

struct MvTask {
    const double* B;
    int64_t rows, cols;
    int64_t xm_off, xn_off;
    int64_t coldot_off;  // into coldot buffer (cols entries)
    int64_t part_off;    // into row-partial buffer (nchunk * rows)
    int chunk;
};

__global__ void mv_pass1_kernel(const MvTask* __restrict__ tasks, const double* __restrict__ x,
                                double* __restrict__ coldot, double* __restrict__ part) {
    const MvTask t = tasks[blockIdx.x];
    const int64_t j0 = static_cast<int64_t>(t.chunk) * kMvChunk;
    const int64_t nc = t.cols - j0 < kMvChunk ? t.cols - j0 : int64_t(kMvChunk);
    const double* xm = x + t.xm_off;
    const double* xn = x + t.xn_off;
    // row partials
    for (int64_t i = threadIdx.x; i < t.rows; i += blockDim.x) {
        double s = 0.0;
        for (int64_t j = 0; j < nc; ++j) s = fma(t.B[i + (j0 + j) * t.rows], xn[j0 + j], s);
        part[t.part_off + static_cast<int64_t>(t.chunk) * t.rows + i] = s;
    }
    // column dots: warp per column
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int64_t j = warp; j < nc; j += nw) {
        const double* c = t.B + (j0 + j) * t.rows;
        double s = 0.0;
        for (int64_t i = lane; i < t.rows; i += 32) s = fma(c[i], xm[i], s);
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) coldot[t.coldot_off + j0 + j] = s;
    }
}

struct MvOut {
    int order;
    int64_t dims[16];
    int64_t offs[17];
    // per pair (m<n): coldot offset and row-partial offset, nchunk
    int64_t pc_off[136];
    int64_t pp_off[136];
    int pnch[136];
    double scale;
};

__device__ __forceinline__ int pair_idx(int m, int n, int d) { return m * (2 * d - m - 1) / 2 + (n - m - 1); }

__global__ void mv_pass2_kernel(const MvOut* __restrict__ o, const double* __restrict__ coldot,
                                const double* __restrict__ part, double* __restrict__ y) {
    const int d = o->order;
    const int64_t total = o->offs[d];
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int m = 0;
        while (t >= o->offs[m + 1]) ++m;
        const int64_t i = t - o->offs[m];
        double s = 0.0;
        // y_m += B(k,m)' x_k for k < m, then B(m,n) x_n for n > m (pair order)
        for (int k = 0; k < m; ++k) s += coldot[o->pc_off[pair_idx(k, m, d)] + i];
        for (int n = m + 1; n < d; ++n) {
            const int p = pair_idx(m, n, d);
            const double* pp = part + o->pp_off[p] + i;
            double r = 0.0;
            for (int c = 0; c < o->pnch[p]; ++c) r += pp[static_cast<int64_t>(c) * o->dims[m]];
            s += r;
        }
        y[t] = s * o->scale;
    }
}

struct MvPlan {
    std::vector<uint64_t> dims;
    DeviceBuffer tasks, out, coldot, part;
    int ntasks = 0;
    const double* blocks = nullptr;
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
    std::vector<uint64_t> key(dims, dims + order);
    auto& plans = mv_plans();
    auto& P = plans[{ctx, key}];
    if (!P || P->blocks != blocks) {
        if (!P) P = std::make_shared<MvPlan>();
        P->dims = key;
        P->blocks = blocks;
        std::vector<MvTask> tasks;
        MvOut o{};
        o.order = order;
        o.offs[0] = 0;
        for (int k = 0; k < order; ++k) {
            o.dims[k] = static_cast<int64_t>(dims[k]);
            o.offs[k + 1] = o.offs[k] + o.dims[k];
        }
        o.scale = 1.0 / static_cast<double>(order - 1);
        int64_t coff = 0, poff = 0;
        uint64_t boff = 0;
        int p = 0;
        for (int m = 0; m < order; ++m)
            for (int n = m + 1; n < order; ++n, ++p) {
                const int64_t rows = o.dims[m], cols = o.dims[n];
                const int nch = static_cast<int>((cols + kMvChunk - 1) / kMvChunk);
                o.pc_off[p] = coff;
                o.pp_off[p] = poff;
                o.pnch[p] = nch;
                for (int c = 0; c < nch; ++c)
                    tasks.push_back(MvTask{blocks + boff, rows, cols, o.offs[m], o.offs[n], coff,
                                           poff, c});
                coff += cols;
                poff += static_cast<int64_t>(nch) * rows;
                boff += static_cast<uint64_t>(rows * cols);
            }
        P->ntasks = static_cast<int>(tasks.size());
        P->tasks.ensure(tasks.size() * sizeof(MvTask));
        P->out.ensure(sizeof(MvOut));
        P->coldot.ensure(std::max<int64_t>(coff, 1) * sizeof(double));
        P->part.ensure(std::max<int64_t>(poff, 1) * sizeof(double));
        R1_CUDA(cudaMemcpyAsync(P->tasks.ptr, tasks.data(), tasks.size() * sizeof(MvTask),
                                cudaMemcpyHostToDevice, ctx->stream));
        R1_CUDA(cudaMemcpyAsync(P->out.ptr, &o, sizeof(MvOut), cudaMemcpyHostToDevice,
                                ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    mv_pass1_kernel<<<P->ntasks, 256, 0, ctx->stream>>>(P->tasks.as<MvTask>(), x,
                                                       P->coldot.as<double>(),
                                                       P->part.as<double>());
    check_launch(ctx, "mv_pass1_kernel");
    const uint64_t total = [&] {
        uint64_t s = 0;
        for (int k = 0; k < order; ++k) s += dims[k];
        return s;
    }();
    const int g = static_cast<int>(std::min<uint64_t>((total + 255) / 256, 1024));
    mv_pass2_kernel<<<g, 256, 0, ctx->stream>>>(P->out.as<MvOut>(), P->coldot.as<double>(),
                                               P->part.as<double>(), y);
    check_launch(ctx, "mv_pass2_kernel");
}

void forget_matvec_plans(r1_context* ctx) {
    auto& plans = mv_plans();
    for (auto it = plans.begin(); it != plans.end();)
        if (it->first.first == ctx)
            it = plans.erase(it);
        else
            ++it;
}

}  // namespace r1
