// Declarations of the per-iteration device steps (solver_ops.cu) and the
// eigen solve (lanczos.cu) used by the host solver driver (solver.cpp).
#pragma once

#include <cstdint>

struct r1_context;

namespace r1 {

void split_stack(r1_context* ctx, const uint64_t* dims, int order, const double* x, double* u,
                 double* xhat, int* flags_dev);
void post_step(r1_context* ctx, const uint64_t* dims, int order, const double* y,
               const double* xhat, const double* u, const double* fro2_dev, const double* mu_dev,
               double mu_host, double* out_dev);
// post_step with mu = the full contraction lambda it computes (baselines)
void post_step_self(r1_context* ctx, const uint64_t* dims, int order, const double* y,
                    const double* xhat, const double* u, const double* fro2_dev, double* out_dev);
void loo_update(r1_context* ctx, const uint64_t* dims, int order, const double* y, double* u,
                int lo, int hi, double* norms_dev, int* flags_dev, bool accumulate);
void asvd_take(r1_context* ctx, const uint64_t* dims, int order, int m, int n, const double* x,
               const double* value_dev, double* u, int* flags_dev, bool accumulate);
void flip_first(r1_context* ctx, double* u0, int64_t n0, const double* lam_in, double* lam_out);
void dense_from_blocks(r1_context* ctx, const uint64_t* dims, int order, const double* blocks,
                       double* S);
bool rqi_step(r1_context* ctx, int64_t n, const double* S, const double* x, double* y);
// solver_chain: x0 is the previous eigenvector of the same operator inside one
// solve (nullptr on its first iteration): the step-count hint is used / reset.
// decide_tol: relative Ritz residual at which the non-picked spectral end
// counts as decided (lanczos.cu t_extremes)
void eig_blocks(r1_context* ctx, const uint64_t* dims, int order, const double* blocks,
                const double* x0, double* value_dev, double* vec_dev, int* info_host,
                double* stats_host, bool solver_chain = false, double decide_tol = 1e-6);
void eig_dense(r1_context* ctx, int64_t n, const double* S, const double* x0, double* value_dev,
               double* vec_dev, int* info_host, double* stats_host);
void dot_device(r1_context* ctx, const double* x, const double* y, uint64_t n, double* out_dev);
void forget_solver_handles(r1_context* ctx);

}  // namespace r1
