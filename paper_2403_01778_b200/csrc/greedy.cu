// Greedy rank-R deflation with a device-resident residual (reference
// proj/src/greedy.cpp:7-35, rank_one_expand tensor.cpp:246-265).
//
// The residual is a device copy of A.  Per term: solve on the residual with
// seed + term (any solver of r1_solve), then ONE fused pass
//   R[i] -= lambda * u_0[i_0] * u_1[i_1] * ... * u_{d-1}[i_{d-1}]
// (the reference's left-to-right expansion product) that also accumulates
// ||R||_F^2 into fixed per-block partials (read R once, write it once — the
// reference expands the full term into a second tensor and re-reads both).
#include "common.cuh"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

namespace r1 {

void sumsq_device(r1_context* ctx, const double* x, uint64_t n, double* out_dev);

namespace {

constexpr int kMaxOrder = 16;
constexpr int kDeflThreads = 256;

struct DeflArgs {
    double* R;
    int64_t I0, rows;  // R viewed as I0 x rows (rows = prod of modes 1..d-1)
    int nout;          // d - 1
    int64_t dims[kMaxOrder];
    const double* u[kMaxOrder];  // u[0] = mode 0, u[1..] = modes 1..d-1
    double lambda;
    double* partials;  // [gridDim.x]
    int dot_only;      // 1: accumulate sum R[i] * e[i] (no write), 0: subtract + ||R||^2
};

__device__ double block_sum(double v, double* sh) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int k = 0; k < static_cast<int>(blockDim.x >> 5); ++k) s += sh[k];
    return s;
}

// Block b handles rows b, b + gridDim.x, ...; thread t the i0 = t, t + blockDim.x, ...
// Fixed grid => fixed summation order => bit-reproducible norm.
__global__ void __launch_bounds__(kDeflThreads) deflate_kernel(const DeflArgs a) {
    __shared__ double sh[32];
    double acc = 0.0;
    for (int64_t row = blockIdx.x; row < a.rows; row += gridDim.x) {
        double w[kMaxOrder];
        int64_t q = row;
        for (int k = 1; k <= a.nout; ++k) {
            w[k] = __ldg(a.u[k] + q % a.dims[k]);
            q /= a.dims[k];
        }
        double* r = a.R + row * a.I0;
        for (int64_t i = threadIdx.x; i < a.I0; i += blockDim.x) {
            double e = a.lambda * __ldg(a.u[0] + i);
            for (int k = 1; k <= a.nout; ++k) e *= w[k];
            if (a.dot_only) {
                acc = fma(r[i], e, acc);
            } else {
                const double v = r[i] - e;
                r[i] = v;
                acc = fma(v, v, acc);
            }
        }
    }
    const double s = block_sum(acc, sh);
    if (threadIdx.x == 0) a.partials[blockIdx.x] = s;
}

__global__ void sum_fixed_kernel(const double* p, int n, double* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < n; ++i) s += p[i];
        out[0] = s;
    }
}

}  // namespace

// R -= lambda * outer(u); returns ||R||_F^2 into *out_dev (device).
void rank_one_subtract(r1_context* ctx, r1_tensor* t, double lambda, const double* u_dev,
                       double* scratch, double* out_dev, bool dot_only = false) {
    const int d = static_cast<int>(t->dims.size());
    if (d > kMaxOrder) fail(R1_ERR_INVALID_ARGUMENT, "rank_one_subtract: unsupported order");
    DeflArgs a{};
    a.R = t->dev;
    a.I0 = static_cast<int64_t>(t->dims[0]);
    a.rows = static_cast<int64_t>(t->numel / t->dims[0]);
    a.nout = d - 1;
    uint64_t off = 0;
    for (int k = 0; k < d; ++k) {
        a.dims[k] = static_cast<int64_t>(t->dims[k]);
        a.u[k] = u_dev + off;
        off += t->dims[k];
    }
    a.lambda = lambda;
    a.partials = scratch;
    a.dot_only = dot_only ? 1 : 0;
    const int grid = 4 * ctx->num_sms;
    deflate_kernel<<<grid, kDeflThreads, 0, ctx->stream>>>(a);
    check_launch(ctx, "deflate_kernel");
    sum_fixed_kernel<<<1, 32, 0, ctx->stream>>>(scratch, grid, out_dev);
    check_launch(ctx, "sum_fixed_kernel");
}

}  // namespace r1

using namespace r1;

extern "C" {

int r1_rank_one_subtract(r1_context* ctx, r1_tensor* t, double lambda, const double* factors_host,
                         double* norm_out) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx || !t) fail(R1_ERR_INVALID_ARGUMENT, "null argument");
        R1_CUDA(cudaSetDevice(ctx->device));
        uint64_t n = 0;
        for (auto v : t->dims) n += v;
        DeviceBuffer buf;
        buf.ensure((n + 8 * ctx->num_sms + 8) * sizeof(double));
        double* u = buf.as<double>();
        double* part = u + n;
        double* out = part + 4 * ctx->num_sms;
        R1_CUDA(cudaMemcpyAsync(u, factors_host, n * sizeof(double), cudaMemcpyHostToDevice,
                                ctx->stream));
        rank_one_subtract(ctx, t, lambda, u, part, out);
        double h = 0.0;
        R1_CUDA(cudaMemcpyAsync(&h, out, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
        if (norm_out) *norm_out = std::sqrt(h);
    });
}

int r1_greedy_rank_r(r1_context* ctx, const r1_tensor* a, uint64_t r, const char* solver,
                     const r1_solve_options* opts, r1_greedy_report* rep) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx || !a || !opts || !rep || !solver) fail(R1_ERR_INVALID_ARGUMENT, "null argument");
        R1_CUDA(cudaSetDevice(ctx->device));
        // greedy.cpp:9-12
        if (r < 1) fail(R1_ERR_INVALID_ARGUMENT, "greedy_rank_r: rank must be >= 1");
        if (!rep->lambdas || !rep->factors || !rep->residual_ratios)
            fail(R1_ERR_INVALID_ARGUMENT, "greedy_rank_r: report arrays are required");
        const int d = static_cast<int>(a->dims.size());
        uint64_t n = 0;
        for (auto v : a->dims) n += v;
        rep->completed = 0;
        rep->terms = 0;
        rep->failure[0] = '\0';

        DeviceBuffer buf;
        buf.ensure((n + 8 * ctx->num_sms + 8) * sizeof(double));
        double* u = buf.as<double>();
        double* part = u + n;
        double* out = part + 4 * ctx->num_sms;
        sumsq_device(ctx, a->dev, a->numel, out);
        double h = 0.0;
        R1_CUDA(cudaMemcpyAsync(&h, out, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
        const double base_norm = std::sqrt(h);
        if (base_norm == 0.0) fail(R1_ERR_INVALID_ARGUMENT, "greedy_rank_r: zero input tensor");

        // the residual: a device copy of A (the input is left untouched)
        r1_tensor* res = nullptr;
        int rc = r1_tensor_create(ctx, a->dims.data(), d, &res);
        if (rc != R1_OK) fail(rc, r1_last_error());
        struct Guard {
            r1_tensor* t;
            ~Guard() { r1_tensor_destroy(t); }
        } guard{res};
        R1_CUDA(cudaMemcpyAsync(res->dev, a->dev, a->numel * sizeof(double),
                                cudaMemcpyDeviceToDevice, ctx->stream));

        std::vector<double> fac(n), fx(n);
        std::vector<r1_iteration_record> trace(std::max(1, opts->max_iters));
        for (uint64_t term = 0; term < r; ++term) {
            r1_solve_options o = *opts;
            o.seed = opts->seed + term;  // greedy.cpp:17
            r1_solve_report local{};
            r1_solve_report* sr = rep->solves ? &rep->solves[term] : &local;
            if (!rep->solves) {
                local.factors = fac.data();
                local.final_x = fx.data();
                local.trace = trace.data();
            }
            rc = r1_solve(ctx, solver, res, &o, sr);
            if (rc == R1_ERR_INVALID_ARGUMENT || rc == R1_ERR_RUNTIME) {
                // greedy.cpp:19-23: partial report
                std::snprintf(rep->failure, sizeof(rep->failure), "term %llu: %s",
                              static_cast<unsigned long long>(term + 1), r1_last_error());
                return;
            }
            if (rc != R1_OK) fail(rc, r1_last_error());
            std::memcpy(rep->factors + term * n, sr->factors, n * sizeof(double));
            rep->lambdas[term] = sr->lambda;
            R1_CUDA(cudaMemcpyAsync(u, sr->factors, n * sizeof(double), cudaMemcpyHostToDevice,
                                    ctx->stream));
            rank_one_subtract(ctx, res, sr->lambda, u, part, out);
            R1_CUDA(cudaMemcpyAsync(&h, out, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
            R1_CUDA(cudaStreamSynchronize(ctx->stream));
            rep->residual_ratios[term] = std::sqrt(h) / base_norm;
            rep->terms = static_cast<int32_t>(term + 1);
        }
        rep->completed = 1;
    });
}

// rank_one_expand (tensor.cpp:246-265): out = lambda u_0 o ... o u_{d-1}, the
// reference's left-to-right product, as the deflation of a zero tensor by
// -lambda (0 - (-x) = x exactly).
int r1_rank_one_expand(r1_context* ctx, double lambda, const double* factors_host,
                       const uint64_t* dims, int order, double* out_host) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx || !dims || !factors_host || !out_host) fail(R1_ERR_INVALID_ARGUMENT, "null argument");
        R1_CUDA(cudaSetDevice(ctx->device));
        if (order < 1 || order > kMaxOrder) fail(R1_ERR_INVALID_ARGUMENT, "rank_one_expand: order mismatch");
        const uint64_t numel = numel_of(dims, order);
        uint64_t n = 0;
        for (int k = 0; k < order; ++k) n += dims[k];
        const size_t tbytes = ((numel + 2) * sizeof(double) + 255) & ~size_t(255);
        ctx->ws_upload.ensure(tbytes);
        ctx->ws_io.ensure((n + 8 * ctx->num_sms + 16) * sizeof(double));
        r1_tensor& t = ctx->upload_view;
        t.ctx = ctx;
        t.dims.assign(dims, dims + order);
        t.numel = numel;
        t.dev = ctx->ws_upload.as<double>();
        t.owned = false;
        double* u = ctx->ws_io.as<double>();
        double* part = u + n;
        double* out = part + 4 * ctx->num_sms;
        R1_CUDA(cudaMemsetAsync(t.dev, 0, numel * sizeof(double), ctx->stream));
        R1_CUDA(cudaMemcpyAsync(u, factors_host, n * sizeof(double), cudaMemcpyHostToDevice,
                                ctx->stream));
        rank_one_subtract(ctx, &t, -lambda, u, part, out);
        R1_CUDA(cudaMemcpyAsync(out_host, t.dev, numel * sizeof(double), cudaMemcpyDeviceToHost,
                                ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

// residual_norm (tensor.cpp:267-287): ||A - lambda o u||_F; numel <= dense_threshold
// subtracts the expansion (fused, one pass), above it the expansion-free form
// sqrt(max(0, ||A||^2 - 2 lambda <A, o u> + lambda^2)) (unit factors assumed).
int r1_residual_norm(r1_context* ctx, const double* a_host, const uint64_t* dims, int order,
                     double lambda, const double* factors_host, uint64_t dense_threshold,
                     double* out_norm) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx || !dims || !a_host || !factors_host || !out_norm)
            fail(R1_ERR_INVALID_ARGUMENT, "null argument");
        R1_CUDA(cudaSetDevice(ctx->device));
        if (order < 1 || order > kMaxOrder) fail(R1_ERR_INVALID_ARGUMENT, "residual_norm: order mismatch");
        uint64_t n = 0;
        for (int k = 0; k < order; ++k) n += dims[k];
        const r1_tensor* view = upload_tensor(ctx, a_host, dims, order);
        r1_tensor& t = const_cast<r1_tensor&>(*view);
        ctx->ws_io.ensure((n + 8 * ctx->num_sms + 16) * sizeof(double));
        double* u = ctx->ws_io.as<double>();
        double* part = u + n;
        double* out = part + 4 * ctx->num_sms;
        R1_CUDA(cudaMemcpyAsync(u, factors_host, n * sizeof(double), cudaMemcpyHostToDevice,
                                ctx->stream));
        double h[2] = {0.0, 0.0};
        if (t.numel <= dense_threshold) {
            rank_one_subtract(ctx, &t, lambda, u, part, out);
            R1_CUDA(cudaMemcpyAsync(h, out, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
            R1_CUDA(cudaStreamSynchronize(ctx->stream));
            *out_norm = std::sqrt(h[0]);
            return;
        }
        sumsq_device(ctx, t.dev, t.numel, out + 1);
        rank_one_subtract(ctx, &t, 1.0, u, part, out, true);
        R1_CUDA(cudaMemcpyAsync(h, out, 2 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
        const double s = h[1] - 2.0 * lambda * h[0] + lambda * lambda;
        *out_norm = std::sqrt(std::max(0.0, s));
    });
}

}  // extern "C"
