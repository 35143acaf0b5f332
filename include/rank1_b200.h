/*
 * rank1_b200.h — C-ABI of the B200-native HOSCF / iHOSCF hot path.
 *
 * This is the drop-in boundary between a host driver (the C++ `rank1::` API in
 * include/rank1/, a Python ctypes mirror, or a foreign FFI) and the sm_100a
 * kernels.  Every entry point is `extern "C"`, takes plain pointers and sizes,
 * returns an `int` status and never lets a C++ exception cross.  No torch or
 * CUDA types appear in the signatures; device pointers are `double*` that live
 * on the context's device and streams are passed as `void*` (a cudaStream_t).
 *
 * Layout conventions follow the reference (proj/include/rank1/tensor.hpp:11-14,
 * matrix.hpp:10): tensors are column-major with the FIRST index fastest; a
 * factor set is passed "flat" as u(0) ++ u(1) ++ ... ++ u(d-1) (length sum I_k,
 * the StackedVector block order of stacked.hpp:11-12); the symmetric block
 * matrix J is passed as its strictly-upper blocks B(m,n), m<n, concatenated in
 * the reference's pair order (nepv.cpp:98-102: (0,1),(0,2),...,(0,d-1),(1,2),...),
 * each block column-major I_m x I_n (mode m = rows).  J = (1/(d-1)) [B] as in
 * nepv.cpp:91.
 *
 * Status codes map 1:1 onto the reference's exception types:
 *   R1_ERR_INVALID_ARGUMENT  <-> std::invalid_argument
 *   R1_ERR_RUNTIME           <-> std::runtime_error (zero factor, failure after
 *                                restart, eigen non-convergence)
 *   R1_ERR_CUDA / R1_ERR_NO_DEVICE  new: device failures; there is NO CPU fallback.
 * r1_last_error() returns the (thread-local) message of the last failure, with
 * the reference's wording where one exists.
 */
#ifndef RANK1_B200_H
#define RANK1_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define R1_ABI_VERSION 1

#define R1_OK 0
#define R1_ERR_INVALID_ARGUMENT 1
#define R1_ERR_RUNTIME 2
#define R1_ERR_CUDA 3
#define R1_ERR_NO_DEVICE 4
#define R1_ERR_INTERNAL 5

/* enum values mirror proj/include/rank1/solvers.hpp:13-15 */
#define R1_INIT_UNIFORM01 0
#define R1_INIT_PROVIDED 1
#define R1_RQI_MAGNITUDE 0
#define R1_RQI_SIGNED_INCREASE 1
#define R1_STOP_KKT 0
#define R1_STOP_EQ11 1
#define R1_STOP_LAMBDA_DELTA 2

typedef struct r1_context r1_context; /* device, stream, events, workspaces   */
typedef struct r1_tensor r1_tensor;   /* a dense order-d tensor resident in HBM */
typedef struct r1_comm r1_comm;       /* NCCL communicator of a sharded tensor's ranks */

/* Mirrors rank1::SolveOptions (solvers.hpp:17-31), same defaults via
 * r1_solve_options_default().  `init_factors` is flat (sum I_k) or NULL. */
typedef struct r1_solve_options {
    double tol;
    int32_t max_iters;
    int32_t init;
    uint64_t seed;
    const double* init_factors;
    int32_t determinism;
    int32_t rqi_accept_rule;
    int32_t stop_rule;
    int32_t threads;
    int32_t record_kkt;
    int32_t asvd_disjoint_pairs;
    int32_t reuse_intermediates;
    /* Extension (not in the reference): when nonzero the SCF solvers also stop
     * once |lambda_k - lambda_{k-1}| <= scf_lambda_rtol * |lambda_k|
     * (BASELINE config 1's "relative sigma change" rule).  0 = reference
     * behaviour (Eq. 11 residual only, solvers.cpp:175-178). */
    double scf_lambda_rtol;
    /* Extension: when nonzero HOSCF also stops once the stacked eigenvector
     * turns by less than this between iterations, |sin angle(x_k, x_{k-1})|
     * <= scf_angle_tol (the factor-change rule of PAPER.md:400-408).  Evaluated
     * on the device with Eq. 11 and the sigma rule.  0 = off. */
    double scf_angle_tol;
} r1_solve_options;

/* Mirrors rank1::IterationRecord (solvers.hpp:33-43). */
typedef struct r1_iteration_record {
    double lambda;
    double stop_value;
    double eq11_value;
    double kkt_max_residual;
    int32_t rqi_accepted;
    int32_t n_sweeps;      /* extension: build_j sweeps charged to this iteration */
    double lambda_pre_rqi;
    double t_build_j;      /* seconds, device-timed (events / %globaltimer)      */
    double t_eig;
    double t_other;
    /* extension: |sin angle(x_k, x_{k-1})| of the stacked eigenvectors (HOSCF;
     * -1 for the first iteration and where not computed) */
    double factor_change;
} r1_iteration_record;

/* Mirrors rank1::SolveReport (solvers.hpp:45-58).  The caller owns every
 * array: `factors` and `final_x` hold sum I_k doubles, `trace` holds
 * max_iters records. */
typedef struct r1_solve_report {
    double lambda;
    double* factors;
    int32_t converged;
    int32_t iterations;
    double lambda0;
    int32_t restarted;
    double* final_x;
    r1_iteration_record* trace;
    /* extension: device-measured totals */
    int32_t total_sweeps;
    double t_total;        /* seconds around the whole solve (events)           */
} r1_solve_report;

/* ---- library / context ------------------------------------------------ */
int r1_abi_version(void);
const char* r1_last_error(void);
int r1_device_count(int* n);
void r1_solve_options_default(r1_solve_options* o);

int r1_context_create(int device, r1_context** out);
int r1_context_destroy(r1_context* ctx);
/* Use a caller-owned cudaStream_t (e.g. torch's current stream) for every
 * subsequent launch on this context; NULL restores the context's own stream.
 * A sweep of an order >= 4 tensor also uses internal side streams for the
 * independent chains of its recursion; they are forked from and joined back
 * into this stream with events inside the call, so stream order (and a stream
 * capture) on the caller's stream covers all of the call's work. */
int r1_context_set_stream(r1_context* ctx, void* cuda_stream);
int r1_context_synchronize(r1_context* ctx);
/* Kernel launches issued on this context since creation (evidence counter). */
int r1_context_launch_count(const r1_context* ctx, uint64_t* count);

/* ---- tensors ------------------------------------------------------------- */
/* Allocate a device tensor (16-byte aligned, padded) and copy `host` into it. */
int r1_tensor_from_host(r1_context* ctx, const double* host, const uint64_t* dims, int order,
                        r1_tensor** out);
/* Allocate without copying (values undefined). */
int r1_tensor_create(r1_context* ctx, const uint64_t* dims, int order, r1_tensor** out);
/* Wrap caller-owned device memory (no copy, not freed).  `dev` must be 16-byte
 * aligned and readable up to 16*ceil(8N/16) bytes. */
int r1_tensor_wrap_device(r1_context* ctx, const double* dev, const uint64_t* dims, int order,
                          r1_tensor** out);
/* Page-lock a caller-owned host range for the copy engines (cudaHostRegister)
 * / release it.  Host-buffer entry points (r1_build_j, r1_tensor_from_host,
 * ...) copy pinned sources directly and stream pageable ones through the
 * context's pinned staging lanes (8 host threads x 2 x 16 MiB, memcpy and DMA
 * overlapped); they never register the caller's memory implicitly, because a
 * registration outlives a freed std::vector and would redirect later DMA. */
int r1_host_register(void* host, uint64_t bytes);
int r1_host_unregister(void* host);

/* Asynchronous H2D of the full tensor on the context stream (pageable sources
 * are staged; the call returns when the host buffer may be reused). */
int r1_tensor_copy_from_host(r1_context* ctx, r1_tensor* t, const double* host);
/* D2H of the whole tensor (synchronous on the context stream). */
int r1_tensor_copy_to_host(r1_context* ctx, const r1_tensor* t, double* host);
/* frobenius_norm (tensor.hpp:67, tensor.cpp:240-244) of a device tensor. */
int r1_tensor_frobenius(r1_context* ctx, const r1_tensor* t, double* out);
int r1_tensor_destroy(r1_tensor* t);
/* frobenius_norm of a HOST tensor (staged to the device). */
int r1_host_frobenius(r1_context* ctx, const double* a_host, const uint64_t* dims, int order,
                      double* out);
double* r1_tensor_device_ptr(const r1_tensor* t);

/* ---- sizes ----------------------------------------------------------------- */
/* Number of doubles of the concatenated upper blocks: sum_{m<n} I_m I_n. */
uint64_t r1_blocks_numel(const uint64_t* dims, int order);

/* ---- the TTVc sweep (replaces rank1::build_j, nepv.hpp:58 / nepv.cpp:199-231)
 * Device-pointer form, asynchronous on the context stream.  `factors_dev` is
 * flat (sum I_k), `blocks_dev` receives all P = d(d-1)/2 blocks (pair order),
 * `fro2_dev` (nullable) receives sum over blocks of sum of squared entries
 * (||J||_F = sqrt(2*fro2)/(d-1), nepv.cpp:152-157).  Factors are NOT validated
 * here (use r1_build_j for the reference's checks).  Deterministic: fixed
 * reduction order, no atomics; identical inputs give identical bits. */
int r1_build_j_device(r1_context* ctx, const r1_tensor* a, const double* factors_dev,
                      double* blocks_dev, double* fro2_dev);

/* Host form with the reference's argument checks (nepv.cpp:24-41, 199-207):
 * order>=2 (invalid_argument), factor lengths (invalid_argument), for d>2 every
 * factor nonzero (runtime_error "degenerate factor set: zero factor for mode k")
 * and unit to 1e-8 (invalid_argument).  `a_host` is copied on every call (into
 * the context's grow-only device buffer: no allocation per call) unless `a_dev`
 * (nullable) is given.  Blocks are returned to host. */
int r1_build_j(r1_context* ctx, const double* a_host, const r1_tensor* a_dev,
               const uint64_t* dims, int order, const double* factors_host, double* blocks_host);

/* One block B(m,n) (replaces rank1::build_block, nepv.hpp:54 / nepv.cpp:159-170);
 * m>n is swapped as in the reference; only the contracted factors are checked. */
int r1_build_block(r1_context* ctx, const double* a_host, const r1_tensor* a_dev,
                   const uint64_t* dims, int order, const double* factors_host, int m, int n,
                   double* block_host);

/* ---- block-matrix operations (nepv.cpp:110-157, 249-282) ------------------ */
/* y = J x (scale included), device pointers, async. */
int r1_block_matvec_device(r1_context* ctx, const uint64_t* dims, int order,
                           const double* blocks_dev, const double* x_dev, double* y_dev);
/* Host-buffer forms (SymBlockMatrix::matvec / dense / frobenius_norm,
 * nepv.cpp:110-157), computed on the device. */
int r1_block_matvec(r1_context* ctx, const uint64_t* dims, int order, const double* blocks_host,
                    const double* x_host, double* y_host);
int r1_block_dense(r1_context* ctx, const uint64_t* dims, int order, const double* blocks_host,
                   double* s_host);
int r1_block_frobenius(r1_context* ctx, const uint64_t* dims, int order, const double* blocks_host,
                       double* out);
/* Eq. 11: ||Jx - rho x|| / (||J||_F + |lambda|), rho = x'Jx (nepv.cpp:271-282).
 * Host form: blocks/x on host, result to *out. */
int r1_scf_stopping_value(r1_context* ctx, const uint64_t* dims, int order,
                          const double* blocks_host, const double* x_host, double lambda,
                          double* out);
/* contract_leaving_all (tensor.hpp:86-87, tensor.cpp:216-238): out = w_0 ++ ... ++
 * w_{d-1}, w_n = A x_{k != n} u_k, from one device sweep (any factor norms;
 * `a_host` staged to the device unless `a_dev` is given). */
int r1_contract_leaving_all(r1_context* ctx, const double* a_host, const r1_tensor* a_dev,
                            const uint64_t* dims, int order, const double* factors_host,
                            double* out_host);
/* KKT report derived from the blocks of J(u) (no tensor pass):
 * w_n = B(n,m) u_m, lambda = u_0' B(0,1) u_1, residual_n = ||w_n - lambda u_n||.
 * out: [lambda, max_residual, residual_0..residual_{d-1}] (d+2 doubles). */
int r1_kkt_from_blocks(r1_context* ctx, const uint64_t* dims, int order,
                       const double* blocks_host, const double* factors_host, double* out);
/* kkt_report(A,f) (nepv.hpp:72): one sweep + the block identities above. */
int r1_kkt_report(r1_context* ctx, const double* a_host, const r1_tensor* a_dev,
                  const uint64_t* dims, int order, const double* factors_host, double* out);

/* ---- eigen steps (sym_eig.hpp:30, 37-38) ------------------------------------ */
/* Largest-magnitude eigenpair of the block matrix J (Lanczos on device, both
 * spectral ends converged; reference pick rule sym_eig.cpp:214-216 and sign
 * canonicalisation :223-227).  x0_dev (nullable) warm-starts. */
int r1_eig_blocks_device(r1_context* ctx, const uint64_t* dims, int order,
                         const double* blocks_dev, const double* x0_dev, double* value_dev,
                         double* vec_dev);
/* largest_magnitude_eigenpair (sym_eig.hpp:30) of a dense symmetric n x n
 * host matrix (column-major): the reference's definition (sym_eig.cpp:206-229)
 * on the device full decomposition r1_sym_eig_full below — pick lo iff
 * |w_lo| > |w_hi| (1 + 1e-12), largest-|entry| positive. */
int r1_largest_magnitude_eigenpair(r1_context* ctx, int64_t n, const double* s_host,
                                   double* value, double* vec);
/* One Rayleigh-quotient step (sym_eig.cpp:411-438) on device: Bunch-Kaufman
 * LDL^T of S - rho I, diag-condition rejection (>1e14), one shift bump.
 * *accepted = 0 reproduces std::nullopt. */
int r1_rayleigh_quotient_step(r1_context* ctx, int64_t n, const double* s_host,
                              const double* x_host, double* y_host, int* accepted);
/* The same on the device block matrix J (blocks_dev as r1_build_j_device
 * writes them), x_dev / y_dev device vectors of sum I_k: the RQI of a
 * distributed solve, where J is replicated on every rank. */
int r1_rqi_blocks_device(r1_context* ctx, const uint64_t* dims, int order, const double* blocks_dev,
                         const double* x_dev, double* y_dev, int* accepted);

/* ---- dense-matrix / tensor utilities of the API (off the solvers' path) ----
 * One-thread-block device kernels that restate the reference's sequential
 * algorithms step for step (csrc/dense_api.cu, compiled without FMA
 * contraction): results follow the reference's rounding (glibc / libdevice
 * hypot and sqrt aside).  Matrices are host, column-major n x n. */
/* sym_eig_full (sym_eig.hpp:19, sym_eig.cpp:27-204): ascending values, vectors
 * column j <-> values[j].  Non-symmetric input (> 1e-10 relative):
 * R1_ERR_INVALID_ARGUMENT "sym_eig: matrix is not symmetric"; no QL convergence
 * within 60 sweeps: R1_ERR_RUNTIME. */
int r1_sym_eig_full(r1_context* ctx, int64_t n, const double* s_host, double* values,
                    double* vectors);
/* detail::ldlt_factor (sym_eig.hpp:49, sym_eig.cpp:233-320): unblocked
 * Bunch-Kaufman, the reference's storage (w: L below the diagonal, D in the
 * pivot blocks; ipiv >= 0 1x1 row swap, < 0 2x2 with kp = -ipiv-1). */
int r1_ldlt_factor(r1_context* ctx, int64_t n, const double* s_host, double* w_host, int* ipiv,
                   int* singular);
/* detail::ldlt_solve (sym_eig.hpp:50, sym_eig.cpp:323-377). */
int r1_ldlt_solve(r1_context* ctx, int64_t n, const double* w_host, const int* ipiv,
                  const double* b_host, double* x_host);
/* detail::ldlt_diag_condition (sym_eig.hpp:52, sym_eig.cpp:380-407) from the
 * pivot blocks: diag[k] = w(k,k), sub[k] = w(k+1,k). */
int r1_ldlt_diag_condition(r1_context* ctx, int64_t n, const double* diag, const double* sub,
                           const int* ipiv, int singular, double* out);
/* matricize (tensor.hpp:55, tensor.cpp:72-83), inverse = 1: dematricize
 * (tensor.hpp:58, tensor.cpp:85-98). */
int r1_matricize(r1_context* ctx, const double* in_host, const uint64_t* dims, int order, int mode,
                 int inverse, double* out_host);
/* ttvc / ttvc_scalar (tensor.hpp:65-75, tensor.cpp:100-199): contract the
 * `nmodes` distinct `modes` (vectors concatenated in that order) in descending
 * mode order, each ttv summing in the reference's order.  full = 0: the
 * remaining tensor into out_host; full = 1 (nmodes == order): *scalar_out. */
int r1_ttvc(r1_context* ctx, const double* a_host, const uint64_t* dims, int order,
            const double* vs_host, const int* modes, int nmodes, int full, double* out_host,
            double* scalar_out);
/* rank_one_expand (tensor.hpp:92, tensor.cpp:246-265). */
int r1_rank_one_expand(r1_context* ctx, double lambda, const double* factors_host,
                       const uint64_t* dims, int order, double* out_host);
/* residual_norm (tensor.hpp:98-99, tensor.cpp:267-287). */
int r1_residual_norm(r1_context* ctx, const double* a_host, const uint64_t* dims, int order,
                     double lambda, const double* factors_host, uint64_t dense_threshold,
                     double* out_norm);

/* ---- multi-GPU: slabs along the last (slowest) mode over NCCL ----------------
 * SURVEY §8e.  Rank r of W holds the slab [lo_r, hi_r) of the last mode
 * (sizes differ by at most one, larger first) as an ordinary r1_tensor of dims
 * (I_0, ..., I_{d-2}, hi_r - lo_r).  Per sweep the partial blocks (m, n < d-1)
 * are all-reduced and the blocks (m, d-1) gathered in place, all in one NCCL
 * group; the eigen step / RQI / stopping test run replicated on identical
 * bits.  NCCL is loaded at run time (libnccl.so.2). */
#define R1_COMM_ID_BYTES 128
/* A fresh NCCL unique id (rank 0 makes it; the caller ships it to the others). */
int r1_comm_unique_id(void* id_out);
/* One process (or thread) per GPU: join communicator `id` as `rank` of `nranks`
 * and attach it to ctx. */
int r1_comm_init(r1_context* ctx, int nranks, int rank, const void* id, r1_comm** out);
/* One process for ndev GPUs: ctxs[i] on devices[i] (created by the caller);
 * comms[i] attached to ctxs[i]. */
int r1_comm_init_all(int ndev, const int* devices, r1_context** ctxs, r1_comm** comms);
int r1_comm_destroy(r1_comm* c);
int r1_comm_info(const r1_comm* c, int* world, int* rank);
/* [lo, hi) of `rank`'s slab of an extent split over `world` ranks. */
int r1_slab_bounds(uint64_t extent, int world, int rank, uint64_t* lo, uint64_t* hi);
/* The sweep of a sharded tensor: `slab` is this rank's slab, `global_dims` the
 * whole tensor's, factors_dev the GLOBAL flat factors, blocks_dev / fro2_dev
 * the GLOBAL blocks (identical on every rank on return).  Needs the context's
 * communicator (r1_comm_init*). */
int r1_build_j_sharded(r1_context* ctx, const r1_tensor* slab, const uint64_t* global_dims, int order,
                       const double* factors_dev, double* blocks_dev, double* fro2_dev);
/* hoscf / ihoscf on a sharded tensor: every rank calls it with its slab; the
 * reports (global factors, trace) are identical on all ranks. */
int r1_solve_sharded(r1_context* ctx, const char* algorithm, const r1_tensor* slab,
                     const uint64_t* global_dims, int order, const r1_solve_options* opts,
                     r1_solve_report* report);

/* ---- synthetic inputs ----------------------------------------------------------- */
/* Fill `t` with elements [first, first + numel(t)) of BASELINE config `cfg`
 * (1..5, definitions in DESIGN.md §6) whose global reference dims are
 * `global_dims`; a contiguous slab along the last (slowest) mode is a tensor of
 * the global dims with a shorter last extent.  Counter-based: any rank can
 * generate its own slab.  (Not in the reference API: generators.cpp is out of
 * scope; this exists so benchmarks never stage 8-32 GB through the host.) */
int r1_generate_config(r1_context* ctx, r1_tensor* t, int cfg, uint64_t seed,
                       const uint64_t* global_dims, int order, uint64_t first);
/* generate(name, dims, seed) (generators.hpp, generators.cpp:101-116) into `t`
 * (the tensor's dims): "gaussian" (N(0,1), stream 1) | "exp" | "arcsin" | "tan"
 * — the reference's named inputs for the experiment harness.  exp / arcsin are
 * bit-identical to the reference; gaussian / tan to ~1 ulp (device log/cos/tan). */
int r1_generate(r1_context* ctx, r1_tensor* t, const char* name, uint64_t seed);

/* ---- solvers (solvers.hpp:63-88) -------------------------------------------- */
/* algorithm: "hoscf" | "ihoscf" (SCF on J(u)) | "hopm" | "jacobi_hopm" |
 * "asvd" | "jacobi_asvd" (the reference's baselines, solvers.cpp:299-447, on
 * the same device sweep).  Unknown names: R1_ERR_INVALID_ARGUMENT "unknown
 * solver".  report->final_x (SCF solvers: last stacked eigenvector) is zeroed
 * for the baselines (the reference leaves it empty, solvers.hpp:56). */
int r1_solve(r1_context* ctx, const char* algorithm, const r1_tensor* a,
             const r1_solve_options* opts, r1_solve_report* report);

/* r1_solve on a HOST tensor (rank1::solve(name, const DenseTensor&, opts)):
 * staged into the context's grow-only device buffer, then solved. */
int r1_solve_host(r1_context* ctx, const char* algorithm, const double* a_host,
                  const uint64_t* dims, int order, const r1_solve_options* opts,
                  r1_solve_report* report);

/* ---- greedy rank-R deflation (greedy.hpp:11-22, greedy.cpp:7-35) --------------- */
/* Mirrors GreedyReport: terms in deflation order, ||R||_F / ||A||_F after each
 * term, completed = 0 with `failure` = "term k: <solver error>" when a term's
 * solve fails (partial report, status R1_OK, like the reference).  The
 * residual lives on the device (a copy of `a`; `a` is not modified). */
typedef struct r1_greedy_report {
    int32_t completed;
    int32_t terms;              /* terms solved (<= r) */
    double* lambdas;            /* [r] caller-owned: FactorSet::lambda per term */
    double* factors;            /* [r * sum I_k] caller-owned: factors per term */
    double* residual_ratios;    /* [r] caller-owned */
    r1_solve_report* solves;    /* [r] optional per-term reports (their arrays caller-owned) */
    char failure[256];
} r1_greedy_report;

/* r >= 1 (else R1_ERR_INVALID_ARGUMENT "greedy_rank_r: rank must be >= 1");
 * a zero tensor is R1_ERR_INVALID_ARGUMENT "greedy_rank_r: zero input tensor".
 * Term k solves with opts->seed + k. */
int r1_greedy_rank_r(r1_context* ctx, const r1_tensor* a, uint64_t r, const char* solver,
                     const r1_solve_options* opts, r1_greedy_report* report);

/* t -= lambda * u_0 o u_1 o ... (rank_one_expand, tensor.cpp:246-265, fused
 * with the subtraction); *norm_out = ||t||_F afterwards (nullable). */
int r1_rank_one_subtract(r1_context* ctx, r1_tensor* t, double lambda, const double* factors_host,
                         double* norm_out);

/* ---- .dt1 files straight to / from the device (tensor_io.hpp:9-21) -------------- */
/* read_dt1 (tensor_io.cpp:66-100): same validation and messages (R1_ERR_RUNTIME:
 * "read_dt1: cannot open|bad magic|tensor order must be >= 2|invalid
 * dimension|size overflow|truncated payload|trailing bytes ..."); the payload
 * streams through pinned staging buffers into a new device tensor. */
int r1_tensor_read_dt1(r1_context* ctx, const char* path, r1_tensor** out);
/* write_dt1 (tensor_io.cpp:47-64). */
int r1_tensor_write_dt1(r1_context* ctx, const r1_tensor* t, const char* path);

#ifdef __cplusplus
}
#endif

#endif /* RANK1_B200_H */
