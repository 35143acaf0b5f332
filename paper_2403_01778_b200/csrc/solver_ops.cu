// Per-iteration device steps of HOSCF / iHOSCF around the sweep and the
// eigen solve (reference proj/src/solvers.cpp:129-297):
//
//   split_stack   split_factors + stack_factors (stacked.cpp:40-73) fused:
//                 u_n = x_n/||x_n|| (degenerate if < 1e-12), xhat = u/sqrt(d)
//   post          ONE block matvec y = J(u) xhat feeds everything the
//                 reference computes with extra tensor passes:
//                   rho = xhat'y (= lambda, the full contraction),
//                   Eq. 11 = ||y - rho xhat|| / (||J||_F + |mu|)   (nepv.cpp:271-282)
//                   w_n = sqrt(d) y_n = A x_{-n} u  (contract_leaving_all),
//                   lambda = u_0'w_0, KKT residual_n = ||w_n - lambda u_n||
//                   (kkt_report, nepv.cpp:249-269)
//   dense         SymBlockMatrix::dense (nepv.cpp:136-150) for the RQI solve
//   rqi           rayleigh_quotient_step (sym_eig.cpp:411-438): Bunch-Kaufman
//                 LDL^T (cuSOLVER dsytrf, LAPACK's BK with alpha=(1+sqrt17)/8,
//                 the same algorithm family as sym_eig.cpp:233-320), the
//                 reference's D-block condition test (>1e14 -> reject,
//                 :381-407, :424) and one shift bump (:434-437).
#include "common.cuh"
#include "blockmv.cuh"
#include "solver_ops.cuh"


#include <cmath>
#include <cstdlib>
#include <vector>

namespace r1 {

namespace {

constexpr int kOpsThreads = 512;

__device__ double block_reduce_sum(double v, double* sh) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    double s = 0.0;
    for (int k = 0; k < static_cast<int>(blockDim.x >> 5); ++k) s += sh[k];
    return s;
}

struct Dims {
    int d;
    int64_t offs[17];
};

// Single CTA: per-block norms of x, normalise, stack.
__global__ void split_stack_kernel(Dims dm, const double* __restrict__ x, double* __restrict__ u,
                                   double* __restrict__ xhat, int* __restrict__ flags) {
    __shared__ double sh[32];
    const double inv_sqrt_d = 1.0 / sqrt(static_cast<double>(dm.d));
    int deg = 0;
    for (int k = 0; k < dm.d; ++k) {
        const int64_t o = dm.offs[k], len = dm.offs[k + 1] - dm.offs[k];
        double s = 0.0;
        for (int64_t i = threadIdx.x; i < len; i += blockDim.x) s = fma(x[o + i], x[o + i], s);
        const double nrm = sqrt(block_reduce_sum(s, sh));
        const bool dk = nrm < 1e-12;
        deg |= dk ? 1 : 0;
        for (int64_t i = threadIdx.x; i < len; i += blockDim.x) {
            const double v = dk ? 0.0 : x[o + i] / nrm;
            if (u) u[o + i] = v;
            if (xhat) xhat[o + i] = v * inv_sqrt_d;
        }
    }
    if (threadIdx.x == 0 && flags) flags[0] = deg;
}

// Single CTA after y = J(u) xhat.
//   out[0] rho (= lambda), out[1] eq11, out[2] kkt max residual,
//   out[3] ||J||_F, out[4] lambda = u_0'w_0, out[5..5+d) residual_n
__global__ void post_kernel(Dims dm, const double* __restrict__ y, const double* __restrict__ xhat,
                            const double* __restrict__ u, const double* __restrict__ fro2,
                            const double* __restrict__ mu_dev, double mu_host, int use_mu_dev,
                            double* __restrict__ out) {
    __shared__ double sh[32];
    const int64_t n = dm.offs[dm.d];
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s = fma(xhat[i], y[i], s);
    const double rho = block_reduce_sum(s, sh);
    s = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double r = y[i] - rho * xhat[i];
        s = fma(r, r, s);
    }
    const double res = sqrt(block_reduce_sum(s, sh));
    const double fro = sqrt(2.0 * fro2[0]) / static_cast<double>(dm.d - 1);
    const double sqd = sqrt(static_cast<double>(dm.d));
    // lambda = u_0' w_0
    s = 0.0;
    for (int64_t i = threadIdx.x; i < dm.offs[1]; i += blockDim.x) s = fma(u[i], sqd * y[i], s);
    const double lam = block_reduce_sum(s, sh);
    double mx = 0.0;
    for (int k = 0; k < dm.d; ++k) {
        s = 0.0;
        for (int64_t i = dm.offs[k] + threadIdx.x; i < dm.offs[k + 1]; i += blockDim.x) {
            const double r = sqd * y[i] - lam * u[i];
            s = fma(r, r, s);
        }
        const double rk = sqrt(block_reduce_sum(s, sh));
        if (threadIdx.x == 0) out[5 + k] = rk;
        mx = fmax(mx, rk);
    }
    // mu: the eigenvalue (device / host) or, for the sweep baselines, the
    // full contraction lambda of these factors (baseline_stop, solvers.cpp:112-118)
    const double mu = use_mu_dev == 1 ? mu_dev[0] : (use_mu_dev == 2 ? lam : mu_host);
    if (threadIdx.x == 0) {
        out[0] = rho;
        out[1] = res / (fro + fabs(mu));
        out[2] = mx;
        out[3] = fro;
        out[4] = lam;
    }
}

// Leave-one-out update of the power sweeps (solvers.cpp:316-331): for the
// modes k in [lo, hi), w_k = sqrt(d) y_k = A x_{-k} u, u_k = w_k / ||w_k||
// (normalize, matrix.cpp:62-67), norms[k] = ||w_k||, degenerate below 1e-300.
__global__ void loo_update_kernel(Dims dm, const double* __restrict__ y, double* __restrict__ u,
                                  int lo, int hi, double* __restrict__ norms,
                                  int* __restrict__ flags, int accumulate) {
    __shared__ double sh[32];
    const double sqd = sqrt(static_cast<double>(dm.d));
    int deg = 0;
    for (int k = lo; k < hi; ++k) {
        const int64_t o = dm.offs[k], len = dm.offs[k + 1] - dm.offs[k];
        double s = 0.0;
        for (int64_t i = threadIdx.x; i < len; i += blockDim.x) {
            const double v = sqd * y[o + i];
            s = fma(v, v, s);
        }
        const double nrm = sqrt(block_reduce_sum(s, sh));
        deg |= nrm < 1e-300 ? 1 : 0;
        for (int64_t i = threadIdx.x; i < len; i += blockDim.x) {
            const double v = sqd * y[o + i];
            u[o + i] = nrm > 0.0 ? v / nrm : v;
        }
        if (threadIdx.x == 0) norms[k] = nrm;
    }
    if (threadIdx.x == 0) flags[0] = (accumulate ? flags[0] : 0) | deg;
}

// ASVD pair update (top_singular_pair, solvers.cpp:358-381): x = the
// largest-magnitude eigenvector of [[0,B],[B',0]] (rows I_m then I_n); a
// negative eigenvalue flips the right block; both blocks are normalised
// (degenerate below 1e-12) into u_m, u_n.
__global__ void asvd_take_kernel(Dims dm, int m, int n, const double* __restrict__ x,
                                 const double* __restrict__ value, double* __restrict__ u,
                                 int* __restrict__ flags, int accumulate) {
    __shared__ double sh[32];
    const int64_t lm = dm.offs[m + 1] - dm.offs[m], ln = dm.offs[n + 1] - dm.offs[n];
    const double sgn = value[0] < 0.0 ? -1.0 : 1.0;
    int deg = 0;
    for (int part = 0; part < 2; ++part) {
        const int64_t len = part ? ln : lm, src = part ? lm : 0, dst = dm.offs[part ? n : m];
        const double f = part ? sgn : 1.0;
        double s = 0.0;
        for (int64_t i = threadIdx.x; i < len; i += blockDim.x) {
            const double v = f * x[src + i];
            s = fma(v, v, s);
        }
        const double nrm = sqrt(block_reduce_sum(s, sh));
        deg |= nrm < 1e-12 ? 1 : 0;
        for (int64_t i = threadIdx.x; i < len; i += blockDim.x) {
            const double v = f * x[src + i];
            u[dst + i] = nrm > 0.0 ? v / nrm : v;
        }
    }
    if (threadIdx.x == 0) flags[0] = (accumulate ? flags[0] : 0) | deg;
}

__global__ void dense_kernel(const BlockOp* __restrict__ opp, double* __restrict__ S) {
    const BlockOp& op = *opp;
    const int64_t n = op.n;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n * n;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = e % n, c = e / n;
        int mr = 0, mc = 0;
        while (r >= op.offs[mr + 1]) ++mr;
        while (c >= op.offs[mc + 1]) ++mc;
        double v = 0.0;
        if (mr < mc) {
            const int p = pair_index(mr, mc, op.d);
            v = op.blocks[op.boff[p] + (r - op.offs[mr]) + (c - op.offs[mc]) * op.dims[mr]];
        } else if (mr > mc) {
            const int p = pair_index(mc, mr, op.d);
            v = op.blocks[op.boff[p] + (c - op.offs[mc]) + (r - op.offs[mr]) * op.dims[mc]];
        }
        S[e] = v * op.scale;
    }
}

__global__ void flip_kernel(double* v, int64_t n, const double* lam_in, double* lam_out) {
    const double lam = lam_in[0];
    if (lam < 0.0)
        for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
             i += static_cast<int64_t>(gridDim.x) * blockDim.x)
            v[i] = -v[i];
    if (blockIdx.x == 0 && threadIdx.x == 0) lam_out[0] = fabs(lam);
}

// ---- RQI helpers --------------------------------------------------------
__global__ void shift_copy_kernel(const double* __restrict__ S, double* __restrict__ W, int64_t n,
                                  const double* __restrict__ shift) {
    const double sh = shift[0];
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n * n;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = e % n, c = e / n;
        W[e] = S[e] - (r == c ? sh : 0.0);
    }
}

// (Sx)_i, thread per row (column-major S: coalesced across threads).
// y = S x for symmetric S (column-major): y_j = S(:, j) . x, one warp per
// column (coalesced column reads, fixed-order lane sums: deterministic).
__global__ void dense_matvec_kernel(const double* __restrict__ S, const double* __restrict__ x,
                                    int64_t n, double* __restrict__ y) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5); j < n; j += warps) {
        const double* c = S + j * n;
        double s0 = 0.0, s1 = 0.0;
        int64_t i = lane;
        for (; i + 32 < n; i += 64) {
            s0 = fma(c[i], x[i], s0);
            s1 = fma(c[i + 32], x[i + 32], s1);
        }
        if (i < n) s0 = fma(c[i], x[i], s0);
        double s = s0 + s1;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) y[j] = s;
    }
}

inline int dense_matvec_grid(int64_t n, int num_sms) {
    return std::max(1, static_cast<int>(std::min<int64_t>((n + 7) / 8, 8 * static_cast<int64_t>(num_sms))));
}

// shifts[1] = bumped shift (sym_eig.cpp:435-436) from rho = shifts[0].
__global__ void bump_kernel(double* __restrict__ shifts, const double* __restrict__ fro2) {
    const double rho = shifts[0];
    shifts[1] = rho != 0.0 ? rho * (1.0 + 1e-10) : 1e-10 * fmax(sqrt(fro2[0]), 1e-300);
}

Dims make_dims(const uint64_t* dims, int order) {
    Dims dm{};
    dm.d = order;
    dm.offs[0] = 0;
    for (int k = 0; k < order; ++k) dm.offs[k + 1] = dm.offs[k] + static_cast<int64_t>(dims[k]);
    return dm;
}

struct SolverHandle {
    DeviceBuffer work;         // Bunch-Kaufman workspace, reused
    DeviceBuffer dense;        // dense J for r1_rqi_blocks_device
    DescCache<BlockOp> dops;   // block-operator descriptors (dense assembly)
};

std::map<r1_context*, std::shared_ptr<SolverHandle>>& solver_handles() {
    static std::map<r1_context*, std::shared_ptr<SolverHandle>> m;
    return m;
}

SolverHandle& handle_state(r1_context* ctx) {
    std::lock_guard<std::mutex> cache_lock(cache_mutex());
    auto& H = solver_handles()[ctx];
    if (!H) H = std::make_shared<SolverHandle>();
    return *H;
}

}  // namespace

void forget_solver_handles(r1_context* ctx) {
    std::lock_guard<std::mutex> cache_lock(cache_mutex());
    solver_handles().erase(ctx);
}

void split_stack(r1_context* ctx, const uint64_t* dims, int order, const double* x, double* u,
                 double* xhat, int* flags_dev) {
    split_stack_kernel<<<1, kOpsThreads, 0, ctx->stream>>>(make_dims(dims, order), x, u, xhat,
                                                          flags_dev);
    check_launch(ctx, "split_stack_kernel");
}

void post_step(r1_context* ctx, const uint64_t* dims, int order, const double* y,
               const double* xhat, const double* u, const double* fro2_dev, const double* mu_dev,
               double mu_host, double* out_dev) {
    post_kernel<<<1, kOpsThreads, 0, ctx->stream>>>(make_dims(dims, order), y, xhat, u, fro2_dev,
                                                   mu_dev, mu_host, mu_dev ? 1 : 0, out_dev);
    check_launch(ctx, "post_kernel");
}

void post_step_self(r1_context* ctx, const uint64_t* dims, int order, const double* y,
                    const double* xhat, const double* u, const double* fro2_dev, double* out_dev) {
    post_kernel<<<1, kOpsThreads, 0, ctx->stream>>>(make_dims(dims, order), y, xhat, u, fro2_dev,
                                                   nullptr, 0.0, 2, out_dev);
    check_launch(ctx, "post_kernel");
}

void loo_update(r1_context* ctx, const uint64_t* dims, int order, const double* y, double* u,
                int lo, int hi, double* norms_dev, int* flags_dev, bool accumulate) {
    loo_update_kernel<<<1, kOpsThreads, 0, ctx->stream>>>(make_dims(dims, order), y, u, lo, hi,
                                                         norms_dev, flags_dev, accumulate ? 1 : 0);
    check_launch(ctx, "loo_update_kernel");
}

void asvd_take(r1_context* ctx, const uint64_t* dims, int order, int m, int n, const double* x,
               const double* value_dev, double* u, int* flags_dev, bool accumulate) {
    asvd_take_kernel<<<1, kOpsThreads, 0, ctx->stream>>>(make_dims(dims, order), m, n, x, value_dev,
                                                        u, flags_dev, accumulate ? 1 : 0);
    check_launch(ctx, "asvd_take_kernel");
}

void flip_first(r1_context* ctx, double* u0, int64_t n0, const double* lam_in, double* lam_out) {
    flip_kernel<<<1, 256, 0, ctx->stream>>>(u0, n0, lam_in, lam_out);
    check_launch(ctx, "flip_kernel");
}

void dense_from_blocks(r1_context* ctx, const uint64_t* dims, int order, const double* blocks,
                       double* S) {
    SolverHandle& H = handle_state(ctx);
    BlockOp op{};
    int64_t cn, rn;
    blockop_layout(op, dims, order, &cn, &rn);
    op.blocks = blocks;
    const BlockOp* dop = H.dops.get(op, ctx->stream);
    const int64_t nn = op.n * op.n;
    const int g = static_cast<int>(std::min<int64_t>((nn + 255) / 256, ctx->num_sms * 16));
    dense_kernel<<<std::max(g, 1), 256, 0, ctx->stream>>>(dop, S);
    check_launch(ctx, "dense_kernel");
}

size_t bk_workspace_bytes(int64_t n, int num_sms);
void bk_factor(r1_context* ctx, int64_t n, double* A, void* ws, double* cond_dev);
void bk_solve(r1_context* ctx, int64_t n, const double* A, void* ws, const double* x, double* y,
              int* ok_dev);

// One RQI step on the dense symmetric S (device, n x n, column-major) and x
// (device): rayleigh_quotient_step (sym_eig.cpp:411-438) on the hand-written
// Bunch-Kaufman (bk.cu): rho = x'Sx, attempt(rho), then attempt(bumped) once.
// Returns true and y (device, unit) when accepted, false for std::nullopt.
// Synchronous (the accept decision is a host branch).
bool rqi_step(r1_context* ctx, int64_t n, const double* S, const double* x, double* y) {
    const size_t nn = static_cast<size_t>(n) * n;
    ctx->ws_rqi.ensure((nn + 2 * n + 128) * sizeof(double));
    double* W = ctx->ws_rqi.as<double>();
    double* scal = W + nn;  // [0] rho, [1] bumped, [2] cond, [3] ||S||_F^2
    int* okd = reinterpret_cast<int*>(scal + 8);
    double* sx = scal + 16;
    SolverHandle& H = handle_state(ctx);
    H.work.ensure(bk_workspace_bytes(n, ctx->num_sms));
    dense_matvec_kernel<<<dense_matvec_grid(n, ctx->num_sms), 256, 0, ctx->stream>>>(S, x, n, sx);
    check_launch(ctx, "dense_matvec_kernel");
    dot_device(ctx, x, sx, static_cast<uint64_t>(n), scal);
    sumsq_device(ctx, S, nn, scal + 3);
    bump_kernel<<<1, 1, 0, ctx->stream>>>(scal, scal + 3);
    check_launch(ctx, "bump_kernel");
    const int g = static_cast<int>(std::min<size_t>((nn + 255) / 256, ctx->num_sms * 16));
    for (int attempt = 0; attempt < 2; ++attempt) {
        shift_copy_kernel<<<std::max(g, 1), 256, 0, ctx->stream>>>(S, W, n, scal + attempt);
        check_launch(ctx, "shift_copy_kernel");
        bk_factor(ctx, n, W, H.work.ptr, scal + 2);
        double cond = 0.0;
        R1_CUDA(cudaMemcpyAsync(&cond, scal + 2, sizeof(double), cudaMemcpyDeviceToHost,
                                ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
        if (!(cond <= 1e14)) continue;  // singular or ill-conditioned shift (sym_eig.cpp:424)
        bk_solve(ctx, n, W, H.work.ptr, x, y, okd);
        int ok = 0;
        R1_CUDA(cudaMemcpyAsync(&ok, okd, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
        if (ok) return true;
    }
    return false;
}

}  // namespace r1

using namespace r1;

extern "C" {

// One RQI step on the block matrix J (device blocks, replicated on every rank
// of a distributed solve): dense J, then rayleigh_quotient_step
// (sym_eig.cpp:411-438).  *accepted = 0 for std::nullopt.
int r1_rqi_blocks_device(r1_context* ctx, const uint64_t* dims, int order, const double* blocks_dev,
                         const double* x_dev, double* y_dev, int* accepted) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx || !dims || !accepted) fail(R1_ERR_INVALID_ARGUMENT, "null argument");
        R1_CUDA(cudaSetDevice(ctx->device));
        int64_t n = 0;
        for (int k = 0; k < order; ++k) n += static_cast<int64_t>(dims[k]);
        SolverHandle& H = handle_state(ctx);
        H.dense.ensure(static_cast<size_t>(n) * n * sizeof(double));
        dense_from_blocks(ctx, dims, order, blocks_dev, H.dense.as<double>());
        *accepted = rqi_step(ctx, n, H.dense.as<double>(), x_dev, y_dev) ? 1 : 0;
    });
}

}  // extern "C"
