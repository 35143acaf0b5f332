// C-ABI entry points (include/rank1_b200.h): context, device tensors and the
// sweep.  Argument checks and messages follow the reference
// (proj/src/nepv.cpp:24-41, 159-170, 199-207) so the host driver can map
// status codes back onto the same exception types.
#include "common.cuh"

#include <cmath>
#include <cstring>
#include <string>

namespace r1 {

thread_local std::string g_last_error;

std::mutex& cache_mutex() {
    static std::mutex m;
    return m;
}

std::set<std::pair<const void*, int>>& configured_set() {
    static std::set<std::pair<const void*, int>> s;
    return s;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }

void forget_matvec_plans(r1_context* ctx);
void forget_eig_plans(r1_context* ctx);
void forget_solver_handles(r1_context* ctx);
void forget_solver_work(r1_context* ctx);
void dot_device(r1_context* ctx, const double* x, const double* y, uint64_t n, double* out_dev);
void sweep_plan_info(r1_context* ctx, const uint64_t* dims, int order, int64_t* info);

namespace {

void bind(r1_context* ctx) {
    if (!ctx) fail(R1_ERR_INVALID_ARGUMENT, "null context");
    R1_CUDA(cudaSetDevice(ctx->device));
}

void check_dims(const uint64_t* dims, int order, const char* who) {
    if (order < 1 || order > 16) fail(R1_ERR_INVALID_ARGUMENT, std::string(who) + ": unsupported order");
    for (int k = 0; k < order; ++k)
        if (dims[k] == 0) fail(R1_ERR_INVALID_ARGUMENT, "DenseTensor: all dims must be >= 1");
}

double norm2_seq(const double* v, uint64_t n) {
    double s = 0.0;
    for (uint64_t i = 0; i < n; ++i) s += v[i] * v[i];
    return std::sqrt(s);
}

// check_unit_nonzero (nepv.cpp:31-41) for the listed modes.
void check_unit_nonzero(const uint64_t* dims, int order, const double* flat, const int* modes,
                        int nmodes) {
    uint64_t off[17];
    off[0] = 0;
    for (int k = 0; k < order; ++k) off[k + 1] = off[k] + dims[k];
    for (int t = 0; t < nmodes; ++t) {
        const int k = modes[t];
        const double nrm = norm2_seq(flat + off[k], dims[k]);
        if (nrm < 1e-12)
            fail(R1_ERR_RUNTIME, "degenerate factor set: zero factor for mode " + std::to_string(k));
        if (std::abs(nrm - 1.0) > 1e-8)
            fail(R1_ERR_INVALID_ARGUMENT,
                 "factor for mode " + std::to_string(k) + " is not unit length");
    }
}

const r1_tensor* device_tensor(r1_context* ctx, const double* a_host, const r1_tensor* a_dev,
                               const uint64_t* dims, int order) {
    if (a_dev) {
        if (static_cast<int>(a_dev->dims.size()) != order ||
            !std::equal(a_dev->dims.begin(), a_dev->dims.end(), dims))
            fail(R1_ERR_INVALID_ARGUMENT, "device tensor dims do not match");
        return a_dev;
    }
    if (!a_host) fail(R1_ERR_INVALID_ARGUMENT, "no tensor given");
    return upload_tensor(ctx, a_host, dims, order);
}

// Grow-only per-context buffers of the host-buffer entry points: the flat
// factors (nf) then the blocks (nb).
struct IoBuffers {
    double* factors;
    double* blocks;
};
IoBuffers io_buffers(r1_context* ctx, uint64_t nf, uint64_t nb) {
    const uint64_t nfa = (nf + 31) & ~uint64_t(31);
    ctx->ws_io.ensure((nfa + nb + 32) * sizeof(double));
    return {ctx->ws_io.as<double>(), ctx->ws_io.as<double>() + nfa};
}

}  // namespace
}  // namespace r1

using namespace r1;

extern "C" {

int r1_abi_version(void) { return R1_ABI_VERSION; }

const char* r1_last_error(void) { return g_last_error.c_str(); }

int r1_device_count(int* n) {
    return abi_guard([&] {
        int c = 0;
        cudaError_t e = cudaGetDeviceCount(&c);
        if (e != cudaSuccess) {
            cudaGetLastError();
            c = 0;
        }
        *n = c;
    });
}

void r1_solve_options_default(r1_solve_options* o) {
    // solvers.hpp:17-31
    std::memset(o, 0, sizeof(*o));
    o->tol = 1e-4;
    o->max_iters = 500;
    o->seed = 0;
    o->init = R1_INIT_UNIFORM01;
    o->init_factors = nullptr;
    o->determinism = 1;
    o->rqi_accept_rule = R1_RQI_MAGNITUDE;
    o->stop_rule = R1_STOP_KKT;
    o->threads = 0;
    o->record_kkt = 1;
    o->asvd_disjoint_pairs = 0;
    o->reuse_intermediates = 0;
    o->scf_lambda_rtol = 0.0;
}

int r1_context_create(int device, r1_context** out) {
    return abi_guard([&] {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
            cudaGetLastError();
            fail(R1_ERR_NO_DEVICE, "no CUDA device visible: the B200 path has no CPU fallback");
        }
        if (device < 0 || device >= n) fail(R1_ERR_INVALID_ARGUMENT, "bad device index");
        R1_CUDA(cudaSetDevice(device));
        cudaDeviceProp prop{};
        R1_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major < 10)
            fail(R1_ERR_NO_DEVICE, std::string("device is not Blackwell (sm_100a required): ") +
                                       prop.name);
        auto* ctx = new r1_context();
        ctx->device = device;
        ctx->num_sms = prop.multiProcessorCount;
        ctx->smem_optin = prop.sharedMemPerBlockOptin;
        R1_CUDA(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
        ctx->stream = ctx->own_stream;
        for (auto& st : ctx->side_streams) R1_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        ctx->side_stream = ctx->side_streams[0];
        for (auto& e : ctx->ev_sweep) R1_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        for (auto& e : ctx->ev_done) R1_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        for (auto& e : ctx->ev_join) R1_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        *out = ctx;
    });
}

int r1_context_destroy(r1_context* ctx) {
    return abi_guard([&] {
        if (!ctx) return;
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        forget_matvec_plans(ctx);
        forget_eig_plans(ctx);
        forget_solver_handles(ctx);
        forget_solver_work(ctx);
        ctx->plans.clear();
        if (ctx->comm) ctx->comm->ctx = nullptr;  // the communicator outlives its context
        if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
        for (auto st : ctx->side_streams)
            if (st) {
                cudaStreamSynchronize(st);
                cudaStreamDestroy(st);
            }
        for (auto e : ctx->ev_sweep)
            if (e) cudaEventDestroy(e);
        for (auto e : ctx->ev_done)
            if (e) cudaEventDestroy(e);
        for (auto e : ctx->ev_join)
            if (e) cudaEventDestroy(e);
        delete ctx;
    });
}

int r1_context_set_stream(r1_context* ctx, void* s) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        bind(ctx);
        ctx->stream = s ? static_cast<cudaStream_t>(s) : ctx->own_stream;
    });
}

int r1_context_synchronize(r1_context* ctx) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        bind(ctx);
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int r1_context_launch_count(const r1_context* ctx, uint64_t* count) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx) fail(R1_ERR_INVALID_ARGUMENT, "null context");
        *count = ctx->launches;
    });
}

// ---------------------------------------------------------------- tensors --
int r1_tensor_create(r1_context* ctx, const uint64_t* dims, int order, r1_tensor** out) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        bind(ctx);
        check_dims(dims, order, "r1_tensor_create");
        auto* t = new r1_tensor();
        t->ctx = ctx;
        t->dims.assign(dims, dims + order);
        t->numel = numel_of(dims, order);
        // 16-byte padded so aligned bulk copies never read past the allocation.
        const size_t bytes = ((t->numel + 2) * sizeof(double) + 255) & ~size_t(255);
        cudaError_t e = cudaMalloc(&t->dev, bytes);
        if (e != cudaSuccess) {
            delete t;
            cuda_check(e, "cudaMalloc(tensor)", __FILE__, __LINE__);
        }
        t->owned = true;
        *out = t;
    });
}

int r1_tensor_from_host(r1_context* ctx, const double* host, const uint64_t* dims, int order,
                        r1_tensor** out) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        int rc = r1_tensor_create(ctx, dims, order, out);
        if (rc != R1_OK) fail(rc, g_last_error);
        h2d_bytes(ctx, (*out)->dev, host, (*out)->numel * sizeof(double));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int r1_tensor_wrap_device(r1_context* ctx, const double* dev, const uint64_t* dims, int order,
                          r1_tensor** out) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        bind(ctx);
        check_dims(dims, order, "r1_tensor_wrap_device");
        if (reinterpret_cast<uintptr_t>(dev) % 16 != 0)
            fail(R1_ERR_INVALID_ARGUMENT, "device tensor must be 16-byte aligned");
        auto* t = new r1_tensor();
        t->ctx = ctx;
        t->dims.assign(dims, dims + order);
        t->numel = numel_of(dims, order);
        t->dev = const_cast<double*>(dev);
        t->owned = false;
        *out = t;
    });
}

int r1_tensor_copy_from_host(r1_context* ctx, r1_tensor* t, const double* host) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        bind(ctx);
        if (!t || !host) fail(R1_ERR_INVALID_ARGUMENT, "null argument");
        h2d_bytes(ctx, t->dev, host, t->numel * sizeof(double));
    });
}

int r1_tensor_copy_to_host(r1_context* ctx, const r1_tensor* t, double* host) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        bind(ctx);
        if (!t || !host) fail(R1_ERR_INVALID_ARGUMENT, "null argument");
        R1_CUDA(cudaMemcpyAsync(host, t->dev, t->numel * sizeof(double), cudaMemcpyDeviceToHost,
                                ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

// frobenius_norm (tensor.cpp:240-244), deterministic fixed-order device sum.
int r1_tensor_frobenius(r1_context* ctx, const r1_tensor* t, double* out) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        bind(ctx);
        if (!t || !out) fail(R1_ERR_INVALID_ARGUMENT, "null argument");
        const IoBuffers io = io_buffers(ctx, 0, 8);
        sumsq_device(ctx, t->dev, t->numel, io.blocks);
        double h = 0.0;
        R1_CUDA(cudaMemcpyAsync(&h, io.blocks, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
        *out = std::sqrt(h);
    });
}

// frobenius_norm (tensor.cpp:240-244) of a host tensor: staged H2D + the
// fixed-order device sum of squares.
int r1_host_frobenius(r1_context* ctx, const double* a_host, const uint64_t* dims, int order,
                      double* out) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        bind(ctx);
        if (!a_host || !dims || !out) fail(R1_ERR_INVALID_ARGUMENT, "null argument");
        check_dims(dims, order, "frobenius_norm");
        const r1_tensor* t = upload_tensor(ctx, a_host, dims, order);
        const IoBuffers io = io_buffers(ctx, 0, 8);
        sumsq_device(ctx, t->dev, t->numel, io.blocks);
        double h = 0.0;
        R1_CUDA(cudaMemcpyAsync(&h, io.blocks, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
        *out = std::sqrt(h);
    });
}

int r1_tensor_destroy(r1_tensor* t) {
    return abi_guard([&] {
        if (!t) return;
        if (t->owned && t->dev) {
            cudaSetDevice(t->ctx->device);
            cudaFree(t->dev);
        }
        delete t;
    });
}

double* r1_tensor_device_ptr(const r1_tensor* t) { return t ? t->dev : nullptr; }

uint64_t r1_blocks_numel(const uint64_t* dims, int order) { return blocks_numel(dims, order); }

// ------------------------------------------------------------------ sweep --
int r1_build_j_device(r1_context* ctx, const r1_tensor* a, const double* factors_dev,
                      double* blocks_dev, double* fro2_dev) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        bind(ctx);
        if (!a) fail(R1_ERR_INVALID_ARGUMENT, "null tensor");
        const int order = static_cast<int>(a->dims.size());
        if (order < 2) fail(R1_ERR_INVALID_ARGUMENT, "build_j: tensor order must be >= 2");
        sweep_blocks(ctx, a->dev, a->dims.data(), order, factors_dev, blocks_dev);
        if (fro2_dev) sumsq_device(ctx, blocks_dev, blocks_numel(a->dims.data(), order), fro2_dev);
    });
}

int r1_build_j(r1_context* ctx, const double* a_host, const r1_tensor* a_dev,
               const uint64_t* dims, int order, const double* factors_host, double* blocks_host) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        bind(ctx);
        if (order < 2) fail(R1_ERR_INVALID_ARGUMENT, "build_j: tensor order must be >= 2");
        check_dims(dims, order, "build_j");
        if (order > 2) {
            int all[16];
            for (int k = 0; k < order; ++k) all[k] = k;
            check_unit_nonzero(dims, order, factors_host, all, order);
        }
        const r1_tensor* t = device_tensor(ctx, a_host, a_dev, dims, order);
        uint64_t nf = 0;
        for (int k = 0; k < order; ++k) nf += dims[k];
        const uint64_t nb = blocks_numel(dims, order);
        const IoBuffers io = io_buffers(ctx, nf, nb);
        R1_CUDA(cudaMemcpyAsync(io.factors, factors_host, nf * sizeof(double),
                                cudaMemcpyHostToDevice, ctx->stream));
        sweep_blocks(ctx, t->dev, dims, order, io.factors, io.blocks);
        R1_CUDA(cudaMemcpyAsync(blocks_host, io.blocks, nb * sizeof(double), cudaMemcpyDeviceToHost,
                                ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int r1_build_block(r1_context* ctx, const double* a_host, const r1_tensor* a_dev,
                   const uint64_t* dims, int order, const double* factors_host, int m, int n,
                   double* block_host) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        bind(ctx);
        if (order < 2) fail(R1_ERR_INVALID_ARGUMENT, "build_block: tensor order must be >= 2");
        if (m == n) fail(R1_ERR_INVALID_ARGUMENT, "build_block: block modes must differ");
        if (m > n) std::swap(m, n);
        if (m < 0 || n >= order) fail(R1_ERR_INVALID_ARGUMENT, "build_block: mode out of range");
        check_dims(dims, order, "build_block");
        int modes[16], nm = 0;
        for (int k = 0; k < order; ++k)
            if (k != m && k != n) modes[nm++] = k;
        check_unit_nonzero(dims, order, factors_host, modes, nm);
        const r1_tensor* t = device_tensor(ctx, a_host, a_dev, dims, order);
        uint64_t nf = 0;
        for (int k = 0; k < order; ++k) nf += dims[k];
        // Factors of the two kept modes never enter block (m, n); the other
        // blocks of the shared sweep are computed and dropped.
        const uint64_t nb = blocks_numel(dims, order);
        const IoBuffers io = io_buffers(ctx, nf, nb);
        R1_CUDA(cudaMemcpyAsync(io.factors, factors_host, nf * sizeof(double),
                                cudaMemcpyHostToDevice, ctx->stream));
        sweep_blocks(ctx, t->dev, dims, order, io.factors, io.blocks);
        const uint64_t off = block_offset(dims, order, m, n);
        R1_CUDA(cudaMemcpyAsync(block_host, io.blocks + off, dims[m] * dims[n] * sizeof(double),
                                cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int r1_block_matvec_device(r1_context* ctx, const uint64_t* dims, int order,
                           const double* blocks_dev, const double* x_dev, double* y_dev) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        bind(ctx);
        block_matvec(ctx, dims, order, blocks_dev, x_dev, y_dev);
    });
}

// Diagnostics (not in the public header): per-CTA {start,end,smid} of the
// top-level sweep kernel into a device buffer of 3*ncta uint64 (NULL: off).
int r1x_set_sweep_trace(r1_context* ctx, void* dev) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        bind(ctx);
        ctx->dbg_sweep_trace = static_cast<unsigned long long*>(dev);
    });
}

// Diagnostics (not in the public header): enable CUDA-event timing of the
// top-level sweep kernel; r1x_kernel_time syncs and returns the summed
// milliseconds and the number of timed launches since the last query.
int r1x_time_kernels(r1_context* ctx, int enable) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        bind(ctx);
        ctx->time_kernels = enable != 0;
    });
}

int r1x_kernel_time(r1_context* ctx, double* ms, uint64_t* launches) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        bind(ctx);
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
        double total = 0.0;
        for (auto& pr : ctx->kernel_events) {
            float t = 0.f;
            R1_CUDA(cudaEventElapsedTime(&t, pr.first, pr.second));
            total += t;
            cudaEventDestroy(pr.first);
            cudaEventDestroy(pr.second);
        }
        *ms = total;
        *launches = ctx->kernel_events.size();
        ctx->kernel_events.clear();
    });
}

// Test/diagnostic hook (not in the public header): the top-level sweep plan.
int r1x_sweep_plan_info(r1_context* ctx, const uint64_t* dims, int order, int64_t* info) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        bind(ctx);
        sweep_plan_info(ctx, dims, order, info);
    });
}

}  // extern "C"
