// Host driver of HOSCF / iHOSCF (C++), calling the device steps.  Mirrors the
// reference's control flow (proj/src/solvers.cpp):
//   validate            :28-32     initial_factors / random_unit_factors :34-66
//   with_restart        :78-91     finalize_sign :70-76
//   run_hoscf           :129-183   run_ihoscf    :185-297
// Every numeric step runs on the device; per iteration the host reads one
// small status record (degeneracy flag + the stop value) — plus, in iHOSCF,
// the RQI accept decision.  The tensor never leaves HBM.
#include "common.cuh"
#include "solver_ops.cuh"

#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <string>
#include <vector>

namespace r1 {

void forget_eig_plans(r1_context* ctx);
void sweep_plan_info(r1_context* ctx, const uint64_t* dims, int order, int64_t* info);

namespace {

constexpr double kNan = std::numeric_limits<double>::quiet_NaN();

// CounterRng (reference include/rank1/rng.hpp:10-37), host side.
struct CounterRng {
    uint64_t key, counter = 0;
    static uint64_t mix(uint64_t z) {
        z ^= z >> 30;
        z *= 0xbf58476d1ce4e5b9ull;
        z ^= z >> 27;
        z *= 0x94d049bb133111ebull;
        z ^= z >> 31;
        return z;
    }
    CounterRng(uint64_t seed, uint64_t stream) : key(mix(seed + 0x9e3779b97f4a7c15ull * (stream + 1))) {}
    double next_unit() { return static_cast<double>(mix(key + 0x9e3779b97f4a7c15ull * ++counter) >> 11) * 0x1.0p-53; }
};
constexpr uint64_t kStreamInit = 2, kStreamRestart = 3;

double norm2_seq(const double* v, size_t n) {
    double s = 0.0;
    for (size_t i = 0; i < n; ++i) s += v[i] * v[i];
    return std::sqrt(s);
}

// normalize (matrix.cpp:62-67): returns the original norm.
double normalize(double* v, size_t n) {
    const double nrm = norm2_seq(v, n);
    if (nrm > 0.0)
        for (size_t i = 0; i < n; ++i) v[i] /= nrm;
    return nrm;
}

// random_unit_factors (solvers.cpp:34-49).
std::vector<double> random_unit_factors(const std::vector<uint64_t>& dims, uint64_t seed,
                                        uint64_t stream) {
    CounterRng rng(seed, stream);
    std::vector<double> f;
    for (uint64_t len : dims) {
        std::vector<double> u(len);
        for (double& v : u) v = rng.next_unit();
        if (normalize(u.data(), len) == 0.0) {
            std::fill(u.begin(), u.end(), 1.0);
            normalize(u.data(), len);
        }
        f.insert(f.end(), u.begin(), u.end());
    }
    return f;
}

struct Degenerate : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// CUDA events for the phase timings, created once per working set and reused
// by every solve (reset() rewinds the pool).
struct Events {
    std::vector<cudaEvent_t> ev;
    size_t used = 0;
    ~Events() {
        for (auto e : ev) cudaEventDestroy(e);
    }
    void reset() { used = 0; }
    cudaEvent_t rec(cudaStream_t s) {
        if (used == ev.size()) {
            cudaEvent_t e;
            R1_CUDA(cudaEventCreate(&e));
            ev.push_back(e);
        }
        cudaEvent_t e = ev[used++];
        R1_CUDA(cudaEventRecord(e, s));
        return e;
    }
    static double secs(cudaEvent_t a, cudaEvent_t b) {
        float ms = 0.f;
        R1_CUDA(cudaEventElapsedTime(&ms, a, b));
        return ms * 1e-3;
    }
};

// Device working set of one solve.
struct Work {
    r1_context* ctx;
    const r1_tensor* A;         // the tensor, or this rank's slab of a sharded one
    std::vector<uint64_t> dims; // GLOBAL dims (J, factors and all vectors use these)
    int d;
    int64_t n;     // sum I_k
    uint64_t nb;   // block entries
    // sharded along the last mode (comm.cu): the slab [lo, hi) and its local blocks
    bool sharded = false;
    std::vector<uint64_t> ldims;
    uint64_t lo = 0, hi = 0;
    DeviceBuffer lblocks;
    DeviceBuffer mem;
    double *U, *Umid, *Urqi, *X, *Xprev, *Xhat, *XhatR, *Yr, *Y, *J, *Jmid, *S;
    double *fro2, *fro2mid, *mu, *post, *postmid, *dotv;
    int* flags;
    PinnedBuffer hst;  // host staging
    std::shared_ptr<void> hd;  // HoscfDev (device-loop state), created on first use
    Events events;             // phase-timing events (iHOSCF / baselines), reused

    Work(r1_context* c, const r1_tensor* a, bool dense, const uint64_t* gdims = nullptr)
        : ctx(c), A(a), dims(a->dims), d(static_cast<int>(a->dims.size())) {
        if (gdims) {
            sharded = true;
            ldims = a->dims;
            dims.assign(gdims, gdims + d);
            const r1_comm* cm = c->comm;
            if (dims[d - 1] < static_cast<uint64_t>(cm->world))
                fail(R1_ERR_INVALID_ARGUMENT, "sharded solve: the last mode has fewer entries (" +
                                                  std::to_string(dims[d - 1]) + ") than ranks (" +
                                                  std::to_string(cm->world) + ")");
            slab_bounds(dims[d - 1], cm->world, cm->rank, &lo, &hi);
            if (hi - lo != ldims[d - 1])
                fail(R1_ERR_INVALID_ARGUMENT, "sharded solve: slab extent does not match this rank's share");
            for (int k = 0; k + 1 < d; ++k)
                if (ldims[k] != dims[k]) fail(R1_ERR_INVALID_ARGUMENT, "sharded solve: slab dims mismatch");
            lblocks.ensure((blocks_numel(ldims.data(), d) + 32) * sizeof(double));
        }
        n = 0;
        for (auto v : dims) n += static_cast<int64_t>(v);
        nb = blocks_numel(dims.data(), d);
        auto al = [](int64_t k) { return (k + 31) & ~int64_t(31); };
        const int64_t vec = al(n);
        const int64_t total = 10 * vec + 2 * al(static_cast<int64_t>(nb)) +
                              (dense ? al(n * n) : 0) + 7 * 64 + 64;
        mem.ensure(total * sizeof(double));
        double* p = mem.as<double>();
        auto take = [&](int64_t k) {
            double* r = p;
            p += al(k);
            return r;
        };
        U = take(n);
        Umid = take(n);
        Urqi = take(n);
        X = take(n);
        Xprev = take(n);
        Xhat = take(n);
        XhatR = take(n);
        Yr = take(n);
        Y = take(n);
        take(n);
        J = take(static_cast<int64_t>(nb));
        Jmid = take(static_cast<int64_t>(nb));
        S = dense ? take(n * n) : nullptr;
        fro2 = take(64);
        fro2mid = take(64);
        mu = take(64);
        post = take(64);
        postmid = take(64);
        dotv = take(64);
        flags = reinterpret_cast<int*>(take(64));
        hst.ensure(64 * 1024);
    }

    cudaStream_t st() const { return ctx->stream; }

    // J(u) of the whole tensor: one fused pass (sharded: over this rank's slab,
    // reading its slice of the last factor, then the NCCL block exchange)
    void sweep(const double* u, double* jb, double* f2) {
        if (sharded) {
            const double* last = u + (n - static_cast<int64_t>(dims[d - 1])) + lo;
            sweep_blocks(ctx, A->dev, ldims.data(), d, u, lblocks.as<double>(), last);
            exchange_blocks(ctx, lblocks.as<double>(), jb, dims.data(), d);
        } else {
            sweep_blocks(ctx, A->dev, dims.data(), d, u, jb);
        }
        sumsq_device(ctx, jb, nb, f2);
    }
    // y = J xhat, then Eq.11 / KKT / lambda into out (see solver_ops.cu)
    void post_step(const double* jb, const double* f2, const double* xh, const double* u,
                   const double* mu_dev, double mu_host, double* out) {
        block_matvec(ctx, dims.data(), d, jb, xh, Y);
        r1::post_step(ctx, dims.data(), d, Y, xh, u, f2, mu_dev, mu_host, out);
    }
    template <typename T>
    void fetch(T* host, const T* dev, size_t count) {
        R1_CUDA(cudaMemcpyAsync(host, dev, count * sizeof(T), cudaMemcpyDeviceToHost, st()));
    }
    void sync() { R1_CUDA(cudaStreamSynchronize(st())); }
};

// Working sets are cached per (context, dims, dense): repeated solves on the
// same shape do not reallocate.
std::map<std::pair<r1_context*, std::vector<uint64_t>>, std::shared_ptr<Work>>& work_cache() {
    static std::map<std::pair<r1_context*, std::vector<uint64_t>>, std::shared_ptr<Work>> m;
    return m;
}

Work& work_for(r1_context* ctx, const r1_tensor* a, bool dense, const uint64_t* gdims = nullptr) {
    std::vector<uint64_t> key = a->dims;
    key.push_back(dense ? 1 : 0);
    if (gdims) {  // sharded: the global dims and the communicator shape are part of the key
        key.insert(key.end(), gdims, gdims + a->dims.size());
        key.push_back(static_cast<uint64_t>(ctx->comm->world));
        key.push_back(static_cast<uint64_t>(ctx->comm->rank));
    }
    std::lock_guard<std::mutex> cache_lock(cache_mutex());
    auto& w = work_cache()[{ctx, key}];
    if (!w) w = std::make_shared<Work>(ctx, a, dense, gdims);
    w->A = a;
    return *w;
}

struct RunResult {
    std::vector<double> factors;  // host, flat
    double lambda = 0.0;
    bool converged = false;
    int iterations = 0;
    double lambda0 = 0.0;
    std::vector<r1_iteration_record> trace;
    std::vector<double> final_x;
    int sweeps = 0;
};

// ---- HOSCF with the loop control on the device ----------------------------
// Each iteration k (solvers.cpp:143-179) is the same device sequence
//   eigen step on J(u_{k-1}) -> split / stack -> sweep J(u_k) -> post step ->
//   record (trace slot, stop decision, warm-start vector),
// so it is captured ONCE per solve as a CUDA graph (two parities: the factor /
// block buffers ping-pong) and replayed.  The stop test — Eq. 11 <= tol
// (:175-178), plus the extensions relative-sigma change and factor change
// |sin angle(x_k, x_{k-1})| — is evaluated on the device
// by the record kernel, which writes one status word.  Each replay is wrapped
// in a conditional IF node whose condition a gate kernel sets from that status,
// so the host enqueues iterations in batches and reads the 8-byte state once
// per batch: after a stop the remaining replays are empty.  Phase times come
// from %globaltimer stamps in the trace.  Without conditional-node support the
// graphs are replayed one per status read; without graphs the same kernels are
// launched directly.

// Lanczos: the non-picked spectral end counts as decided at this relative
// Ritz residual in the HOSCF chain (lanczos.cu t_extremes; iHOSCF keeps 1e-6)
constexpr double kHoscfDecideTol = 1e-4;

struct DevRecord {
    double lambda, stop_value, eq11, kkt, angle, pad;
    unsigned long long t[5];  // globaltimer: start, after eig, after split, after sweep, end
};

struct IterState {
    int counter;  // iterations completed
    int status;   // 0 running, 1 Eq.11, 2 sigma change, 3 factor change, 4 max_iters, 5 degenerate
};

struct IterParams {
    double tol, lambda_rtol, angle_tol;
    int max_iters, record_kkt;
    int64_t n;
    int debug;
};

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void stamp_kernel(const IterState* st, DevRecord* trace, int cap, int which) {
    const int k = st->counter;
    if (k < 0 || k > cap) {
        printf("[r1] stamp_kernel: iteration slot %d out of range (cap %d)\n", k, cap);
        __trap();
    }
    trace[k].t[which] = global_ns();
}

__global__ void gate_kernel(const IterState* st, cudaGraphConditionalHandle h) {
    cudaGraphSetConditional(h, st->status == 0 ? 1u : 0u);
}

constexpr int kRecThreads = 256;

__device__ double rec_block_sum(double v, double* sh) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
    for (int k = 0; k < kRecThreads / 32; ++k) s += sh[k];
    return s;
}

// post = [rho, eq11, kkt, fro, lambda, ...] of the new J (post_kernel)
__global__ void __launch_bounds__(kRecThreads) record_kernel(IterState* st, DevRecord* trace,
                                                             const IterParams* prm,
                                                             const double* __restrict__ post,
                                                             const double* __restrict__ mu,
                                                             const int* __restrict__ flags,
                                                             const double* __restrict__ X,
                                                             double* __restrict__ Xprev) {
    __shared__ double sh[32];
    const int k = st->counter + 1;
    const int64_t n = prm->n;
    double angle = -1.0;
    if (k > 1) {
        double s = 0.0;
        for (int64_t i = threadIdx.x; i < n; i += kRecThreads) s = fma(X[i], Xprev[i], s);
        const double c = rec_block_sum(s, sh);
        s = 0.0;
        for (int64_t i = threadIdx.x; i < n; i += kRecThreads) {
            const double r = X[i] - c * Xprev[i];
            s = fma(r, r, s);
        }
        angle = sqrt(rec_block_sum(s, sh));
    }
    __syncthreads();
    for (int64_t i = threadIdx.x; i < n; i += kRecThreads) Xprev[i] = X[i];
    if (threadIdx.x != 0) return;
    DevRecord& r = trace[k - 1];
    if (flags[0]) {  // split_factors found a zero block: the restart path (solvers.cpp:78-91)
        st->status = 5;
        return;
    }
    const double lam = mu[0];
    r.lambda = lam;
    r.eq11 = post[1];
    r.stop_value = post[1];
    r.kkt = prm->record_kkt ? post[2] : __longlong_as_double(0x7ff8000000000000ll);
    r.angle = angle;
    r.pad = k > 1 ? fabs(lam - trace[k - 2].lambda) / fabs(lam) : -1.0;  // sigma change (diagnostics)
    int status = 0;
    if (r.stop_value <= prm->tol)
        status = 1;
    else if (prm->lambda_rtol > 0.0 && k > 1 && fabs(lam - trace[k - 2].lambda) <= prm->lambda_rtol * fabs(lam))
        status = 2;
    else if (prm->angle_tol > 0.0 && k > 1 && angle <= prm->angle_tol)
        status = 3;
    else if (k >= prm->max_iters)
        status = 4;
    r.t[4] = global_ns();
    if (prm->debug && (k <= 2 || status))
        printf("[r1 record] k=%d tol=%g lrtol=%g atol=%g max=%d eq11=%g dl=%g angle=%g status=%d\n", k,
               prm->tol, prm->lambda_rtol, prm->angle_tol, prm->max_iters, r.eq11, r.pad, angle, status);
    st->status = status;
    st->counter = k;
}

struct HoscfDev {
    DeviceBuffer mem;     // IterState + IterParams + trace
    IterState* state = nullptr;
    IterParams* params = nullptr;
    DevRecord* trace = nullptr;
    int cap = 0;
    PinnedBuffer hst;
    cudaGraphExec_t exec[2] = {nullptr, nullptr};
    bool conditional = false;
    uint64_t launches_per_iter = 0;
    ~HoscfDev() {
        for (auto e : exec)
            if (e) cudaGraphExecDestroy(e);
    }
    void ensure(int max_iters) {
        if (max_iters <= cap) return;
        const size_t bytes = 256 + static_cast<size_t>(max_iters + 1) * sizeof(DevRecord);
        mem.ensure(bytes);
        state = mem.as<IterState>();
        params = reinterpret_cast<IterParams*>(mem.as<char>() + 64);
        trace = reinterpret_cast<DevRecord*>(mem.as<char>() + 256);
        cap = max_iters;
    }
};

// One HOSCF iteration on the device; p = parity (reads buffers p, writes p^1).
void enqueue_hoscf_iteration(Work& w, HoscfDev& D, int p, bool warm) {
    r1_context* ctx = w.ctx;
    const cudaStream_t st = w.st();
    static const bool dbg = dev_env("R1_GRAPH_DEBUG") != nullptr;
    auto note = [&](const char* what) {
        if (dbg) std::fprintf(stderr, "[r1 iter] p=%d %s\n", p, what);
    };
    double* Ub[2] = {w.U, w.Umid};
    double* Jb[2] = {w.J, w.Jmid};
    double* fb[2] = {w.fro2, w.fro2mid};
    double* pb[2] = {w.post, w.postmid};
    const int q = p ^ 1;
    stamp_kernel<<<1, 1, 0, st>>>(D.state, D.trace, D.cap, 0);
    check_launch(ctx, "stamp_kernel");
    note("eig");
    eig_blocks(ctx, w.dims.data(), w.d, Jb[p], warm ? w.Xprev : nullptr, w.mu, w.X, nullptr, nullptr,
               true, kHoscfDecideTol);
    stamp_kernel<<<1, 1, 0, st>>>(D.state, D.trace, D.cap, 1);
    check_launch(ctx, "stamp_kernel");
    note("split");
    split_stack(ctx, w.dims.data(), w.d, w.X, Ub[q], w.Xhat, w.flags);
    stamp_kernel<<<1, 1, 0, st>>>(D.state, D.trace, D.cap, 2);
    check_launch(ctx, "stamp_kernel");
    note("sweep");
    w.sweep(Ub[q], Jb[q], fb[q]);
    stamp_kernel<<<1, 1, 0, st>>>(D.state, D.trace, D.cap, 3);
    check_launch(ctx, "stamp_kernel");
    note("post");
    w.post_step(Jb[q], fb[q], w.Xhat, Ub[q], w.mu, 0.0, pb[q]);
    record_kernel<<<1, kRecThreads, 0, st>>>(D.state, D.trace, D.params, pb[q], w.mu, w.flags, w.X,
                                             w.Xprev);
    check_launch(ctx, "record_kernel");
    note("done");
}

// Capture the parity-p iteration as [gate] -> IF(status == 0) {iteration} (or
// the bare iteration when conditional = false) and instantiate it.
cudaGraphExec_t capture_iteration(Work& w, HoscfDev& D, int p, bool conditional, uint64_t* launches) {
    const cudaStream_t st = w.st();
    static const bool dbg = dev_env("R1_GRAPH_DEBUG") != nullptr;
    auto note = [&](const char* what) {
        if (dbg) std::fprintf(stderr, "[r1 graph] p=%d cond=%d %s\n", p, conditional ? 1 : 0, what);
    };
    note("begin");
    cudaGraph_t g = nullptr;
    R1_CUDA(cudaGraphCreate(&g, 0));
    struct G {
        cudaGraph_t g;
        ~G() {
            if (g) cudaGraphDestroy(g);
        }
    } guard{g};
    cudaGraph_t body = g;
    if (conditional) {
        cudaGraphConditionalHandle h;
        R1_CUDA(cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault));
        R1_CUDA(cudaStreamBeginCaptureToGraph(st, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        gate_kernel<<<1, 1, 0, st>>>(D.state, h);
        cudaGraph_t cap = nullptr;
        R1_CUDA(cudaStreamEndCapture(st, &cap));
        size_t nn = 0;
        R1_CUDA(cudaGraphGetNodes(g, nullptr, &nn));
        std::vector<cudaGraphNode_t> nodes(nn);
        R1_CUDA(cudaGraphGetNodes(g, nodes.data(), &nn));
        cudaGraphNodeParams cp{};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeIf;
        cp.conditional.size = 1;
        cudaGraphNode_t cnode;
        R1_CUDA(cudaGraphAddNode(&cnode, g, nodes.data(), nn, &cp));
        body = cp.conditional.phGraph_out[0];
        note("conditional node added");
    }
    const uint64_t l0 = w.ctx->launches;
    R1_CUDA(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    try {
        enqueue_hoscf_iteration(w, D, p, true);
    } catch (...) {
        cudaGraph_t junk = nullptr;
        cudaStreamEndCapture(st, &junk);
        cudaGetLastError();
        throw;
    }
    cudaGraph_t cap = nullptr;
    R1_CUDA(cudaStreamEndCapture(st, &cap));
    note("body captured");
    *launches = w.ctx->launches - l0;
    w.ctx->launches = l0;  // counted per executed replay instead
    cudaGraphExec_t exec = nullptr;
    R1_CUDA(cudaGraphInstantiate(&exec, g, 0));
    note("instantiated");
    return exec;
}

RunResult run_hoscf_dev(Work& w, const r1_solve_options& o, const std::vector<double>& u0) {
    RunResult rr;
    r1_context* ctx = w.ctx;
    const cudaStream_t st = w.st();
    const int d = w.d;
    const int64_t n = w.n;
    if (!w.hd) w.hd = std::make_shared<HoscfDev>();
    HoscfDev& D = *static_cast<HoscfDev*>(w.hd.get());
    D.ensure(o.max_iters);
    // parameters and state (pageable -> synchronous copies, before any capture)
    IterParams prm{o.tol, o.scf_lambda_rtol, o.scf_angle_tol, o.max_iters, o.record_kkt, n,
                   dev_env("R1_GRAPH_DEBUG") ? 1 : 0};
    IterState s0{0, 0};
    R1_CUDA(cudaMemcpyAsync(D.params, &prm, sizeof(prm), cudaMemcpyHostToDevice, st));
    R1_CUDA(cudaMemcpyAsync(D.state, &s0, sizeof(s0), cudaMemcpyHostToDevice, st));

    // lambda0 and J(u0) (the reference's build_j before the loop, solvers.cpp:131-141)
    R1_CUDA(cudaMemcpyAsync(w.U, u0.data(), n * sizeof(double), cudaMemcpyHostToDevice, st));
    split_stack(ctx, w.dims.data(), d, w.U, nullptr, w.Xhat, w.flags);
    stamp_kernel<<<1, 1, 0, st>>>(D.state, D.trace, D.cap, 2);  // trace[0].t[2..3]: the initial sweep
    check_launch(ctx, "stamp_kernel");
    w.sweep(w.U, w.J, w.fro2);
    stamp_kernel<<<1, 1, 0, st>>>(D.state, D.trace, D.cap, 3);
    check_launch(ctx, "stamp_kernel");
    unsigned long long t_init[2];
    R1_CUDA(cudaMemcpyAsync(t_init, &D.trace[0].t[2], sizeof(t_init), cudaMemcpyDeviceToHost, st));
    w.post_step(w.J, w.fro2, w.Xhat, w.U, nullptr, 0.0, w.post);
    double* h = w.hst.as<double>();
    w.fetch(h, w.post, 8);
    // iteration 1: cold eigen step, launched directly
    enqueue_hoscf_iteration(w, D, 0, false);
    IterState* hs = reinterpret_cast<IterState*>(h + 16);
    w.fetch(hs, D.state, 1);
    w.sync();
    rr.lambda0 = h[4];
    const double t_init_sweep = (t_init[1] - t_init[0]) * 1e-9;

    // iterations 2..kEager: direct launches, one status read each (short solves
    // never pay for a capture); then graph replays with the device stop test
    int done = hs->counter, status = hs->status;
    constexpr int kEager = 6;
    while (status == 0 && done < kEager) {
        enqueue_hoscf_iteration(w, D, done & 1, true);
        w.fetch(hs, D.state, 1);
        w.sync();
        done = hs->counter;
        status = hs->status;
    }
    if (status == 0) {
        bool graphs = true;
        static const char* nog = dev_env("R1_SOLVER_GRAPHS");  // development: 0 = direct launches
        if (nog && std::atoi(nog) == 0) graphs = false;
        if (w.sharded) graphs = false;  // NCCL exchange inside the iteration: direct launches
        uint64_t per_iter = 0;
        if (graphs) {
            for (auto& e : D.exec)
                if (e) {
                    cudaGraphExecDestroy(e);
                    e = nullptr;
                }
            static const char* cenv = dev_env("R1_GRAPH_COND");  // development: 0 = plain graphs
            D.conditional = !(cenv && std::atoi(cenv) == 0);
            try {
                if (!D.conditional) throw Error(R1_ERR_CUDA, "conditional graphs disabled");
                D.exec[1] = capture_iteration(w, D, 1, true, &per_iter);
                D.exec[0] = capture_iteration(w, D, 0, true, &per_iter);
            } catch (const Error&) {
                cudaGetLastError();
                for (auto& e : D.exec)
                    if (e) {
                        cudaGraphExecDestroy(e);
                        e = nullptr;
                    }
                D.conditional = false;
                try {
                    D.exec[1] = capture_iteration(w, D, 1, false, &per_iter);
                    D.exec[0] = capture_iteration(w, D, 0, false, &per_iter);
                } catch (const Error&) {
                    cudaGetLastError();
                    graphs = false;
                }
            }
        }
        ctx->solver_graph_mode = graphs ? (D.conditional ? 2 : 1) : 0;
        int batch = D.conditional && graphs ? 2 : 1;
        int k = done;  // iterations enqueued so far
        while (status == 0) {
            const int nb = std::min(batch, o.max_iters - k);
            for (int b = 0; b < nb; ++b, ++k) {
                const int p = k & 1;  // iteration k+1 reads the buffers of parity k & 1
                if (graphs) {
                    R1_CUDA(cudaGraphLaunch(D.exec[p], st));
                    static const bool sync_each = dev_env("R1_GRAPH_SYNC_EACH") != nullptr;
                    if (sync_each) {
                        cudaError_t e = cudaStreamSynchronize(st);
                        if (e != cudaSuccess)
                            fail(R1_ERR_CUDA, std::string("graph replay of iteration ") +
                                                  std::to_string(k + 1) + " (parity " + std::to_string(p) +
                                                  "): " + cudaGetErrorString(e));
                    }
                } else
                    enqueue_hoscf_iteration(w, D, p, true);
            }
            w.fetch(hs, D.state, 1);
            w.sync();
            if (graphs) ctx->launches += per_iter * static_cast<uint64_t>(hs->counter - done);
            done = hs->counter;
            status = hs->status;
            k = done;
            if (graphs && D.conditional) batch = std::min(batch * 2, 32);
        }
    }
    if (status == 5)
        throw Degenerate("hoscf: eigenvector block collapsed to zero");

    // trace and final state
    std::vector<DevRecord> tr(done);
    if (done) R1_CUDA(cudaMemcpyAsync(tr.data(), D.trace, done * sizeof(DevRecord), cudaMemcpyDeviceToHost, st));
    const int fin = done & 1;  // buffers written by the last iteration
    double* Ub[2] = {w.U, w.Umid};
    double* pb[2] = {w.post, w.postmid};
    rr.factors.resize(n);
    rr.final_x.resize(n);
    w.fetch(h, pb[fin], 8);
    w.fetch(rr.factors.data(), Ub[fin], n);
    w.fetch(rr.final_x.data(), w.Xprev, n);
    w.sync();
    if (fin == 1) {  // keep the Work's canonical buffers pointing at the current state
        std::swap(w.U, w.Umid);
        std::swap(w.J, w.Jmid);
        std::swap(w.fro2, w.fro2mid);
        std::swap(w.post, w.postmid);
    }
    double lam = h[4];
    if (lam < 0.0) {  // finalize_sign (solvers.cpp:70-76)
        lam = -lam;
        for (uint64_t i = 0; i < w.dims[0]; ++i) rr.factors[i] = -rr.factors[i];
    }
    rr.lambda = lam;
    rr.iterations = done;
    rr.converged = status >= 1 && status <= 3;
    rr.sweeps = 1 + done;
    for (int i = 0; i < done; ++i) {
        const DevRecord& q = tr[i];
        r1_iteration_record rec{};
        rec.lambda = q.lambda;
        rec.stop_value = q.stop_value;
        rec.eq11_value = q.eq11;
        rec.kkt_max_residual = q.kkt;
        rec.rqi_accepted = 0;
        rec.n_sweeps = i == 0 ? 2 : 1;
        rec.lambda_pre_rqi = std::numeric_limits<double>::quiet_NaN();
        rec.factor_change = q.angle;
        if (dev_env("R1_GRAPH_DEBUG") && i >= done - 30)
            std::fprintf(stderr, "[r1 trace] k=%d lambda=%.17g dl/l=%.6e angle=%.3e\n", i + 1, q.lambda,
                         q.pad, q.angle);
        rec.t_eig = (q.t[1] - q.t[0]) * 1e-9;
        rec.t_build_j = (q.t[3] - q.t[2]) * 1e-9 + (i == 0 ? t_init_sweep : 0.0);
        rec.t_other = (q.t[2] - q.t[1]) * 1e-9 + (q.t[4] - q.t[3]) * 1e-9;
        rr.trace.push_back(rec);
    }
    return rr;
}

RunResult run(Work& w, const r1_solve_options& o, const std::vector<double>& u0, bool accelerated) {
    RunResult rr;
    Events& ev = w.events;
    ev.reset();
    const cudaStream_t st = w.st();
    const int d = w.d;
    const int64_t n = w.n;
    R1_CUDA(cudaMemcpyAsync(w.U, u0.data(), n * sizeof(double), cudaMemcpyHostToDevice, st));
    // lambda0 and J(u0): stack u0 on device (split of a unit vector = itself)
    split_stack(w.ctx, w.dims.data(), d, w.U, nullptr, w.Xhat, w.flags);
    cudaEvent_t e0 = ev.rec(st);
    w.sweep(w.U, w.J, w.fro2);
    cudaEvent_t e1 = ev.rec(st);
    w.post_step(w.J, w.fro2, w.Xhat, w.U, nullptr, 0.0, w.post);
    double* h = w.hst.as<double>();
    w.fetch(h, w.post, 8);
    w.sync();
    rr.lambda0 = h[4];
    rr.sweeps = 1;
    struct Marks {
        cudaEvent_t a, b, c, d2, e;
        cudaEvent_t f = nullptr, g = nullptr;  // the accepted-RQI sweep (solvers.cpp:266-270)
    };
    std::vector<Marks> marks;
    bool have_prev = false;
    double lam_prev = 0.0;
    const double sqd = std::sqrt(static_cast<double>(d));
    (void)sqd;

    for (int k = 1; k <= o.max_iters; ++k) {
        r1_iteration_record rec{};
        rec.lambda_pre_rqi = kNan;
        rec.factor_change = -1.0;
        rec.n_sweeps = (k == 1) ? 2 : 1;
        Marks mk;
        mk.a = ev.rec(st);
        eig_blocks(w.ctx, w.dims.data(), d, w.J, have_prev ? w.Xprev : nullptr, w.mu, w.X, nullptr,
                   nullptr, true);
        mk.b = ev.rec(st);
        split_stack(w.ctx, w.dims.data(), d, w.X, w.Umid, w.Xhat, w.flags);
        mk.c = ev.rec(st);
        w.sweep(w.Umid, w.Jmid, w.fro2mid);
        mk.d2 = ev.rec(st);
        w.post_step(w.Jmid, w.fro2mid, w.Xhat, w.Umid, w.mu, 0.0, w.postmid);
        int* hf = reinterpret_cast<int*>(h + 32);
        w.fetch(h, w.postmid, 8);
        w.fetch(h + 8, w.mu, 1);
        w.fetch(hf, w.flags, 1);
        w.sync();
        if (hf[0]) throw Degenerate(accelerated ? "ihoscf: eigenvector block collapsed to zero"
                                                : "hoscf: eigenvector block collapsed to zero");
        const double mu = h[8];
        const double sv = h[1];
        const double kkt_mid = h[2];
        const double rho_mid = h[0];
        double* xfinal = w.X;

        if (!accelerated || sv <= o.tol) {
            // hoscf step (solvers.cpp:160-178) or the iHOSCF early exit (:220-234)
            std::swap(w.U, w.Umid);
            std::swap(w.J, w.Jmid);
            std::swap(w.fro2, w.fro2mid);
            std::swap(w.post, w.postmid);
            rec.lambda = mu;
            rec.eq11_value = sv;
            rec.stop_value = sv;
            rec.kkt_max_residual = o.record_kkt ? kkt_mid : kNan;
        } else {
            // skip-ahead RQI refinement (solvers.cpp:236-283)
            rec.lambda_pre_rqi = rho_mid;
            dense_from_blocks(w.ctx, w.dims.data(), d, w.Jmid, w.S);
            bool accepted = false;
            double rho_y = 0.0;
            if (rqi_step(w.ctx, n, w.S, w.Xhat, w.Yr)) {
                split_stack(w.ctx, w.dims.data(), d, w.Yr, w.Urqi, nullptr, w.flags);
                block_matvec(w.ctx, w.dims.data(), d, w.Jmid, w.Yr, w.Y);
                dot_device(w.ctx, w.Yr, w.Y, static_cast<uint64_t>(n), w.dotv);
                w.fetch(hf, w.flags, 1);
                w.fetch(h + 9, w.dotv, 1);
                w.sync();
                if (!hf[0]) {
                    rho_y = h[9];
                    const bool improves = o.rqi_accept_rule == R1_RQI_SIGNED_INCREASE
                                              ? rho_y > rho_mid
                                              : std::abs(rho_y) > std::abs(rho_mid);
                    accepted = improves;
                }
            }
            rec.rqi_accepted = accepted ? 1 : 0;
            if (accepted) {
                std::swap(w.U, w.Urqi);
                // xhat of the refined factors (stack_factors(u), :272)
                split_stack(w.ctx, w.dims.data(), d, w.U, nullptr, w.XhatR, w.flags);
                mk.f = ev.rec(st);
                w.sweep(w.U, w.J, w.fro2);
                mk.g = ev.rec(st);
                rec.n_sweeps += 1;
                w.post_step(w.J, w.fro2, w.XhatR, w.U, nullptr, rho_y, w.post);
                w.fetch(h + 16, w.post, 8);
                w.sync();
                rec.lambda = rho_y;
                rec.eq11_value = h[16 + 1];
                rec.stop_value = rec.eq11_value;
                rec.kkt_max_residual = o.record_kkt ? h[16 + 2] : kNan;
                xfinal = w.Yr;
            } else {
                std::swap(w.U, w.Umid);
                std::swap(w.J, w.Jmid);
                std::swap(w.fro2, w.fro2mid);
                std::swap(w.post, w.postmid);
                rec.lambda = rho_mid;
                rec.eq11_value = sv;
                rec.stop_value = sv;
                rec.kkt_max_residual = o.record_kkt ? kkt_mid : kNan;
            }
        }
        mk.e = ev.rec(st);
        marks.push_back(mk);
        rr.sweeps += rec.n_sweeps - (k == 1 ? 1 : 0);
        rr.trace.push_back(rec);
        rr.iterations = k;
        // final_x / warm start for the next eigen solve
        R1_CUDA(cudaMemcpyAsync(w.Xprev, xfinal, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
        have_prev = true;
        if (rec.stop_value <= o.tol) {
            rr.converged = true;
            break;
        }
        if (o.scf_lambda_rtol > 0.0 && k > 1 &&
            std::abs(rec.lambda - lam_prev) <= o.scf_lambda_rtol * std::abs(rec.lambda)) {
            rr.converged = true;
            break;
        }
        lam_prev = rec.lambda;
    }
    // finalize_sign (solvers.cpp:70-76): lambda = u_0' B(0,1)... of the final J(u)
    w.fetch(h, w.post, 8);
    w.sync();
    double lam = h[4];
    rr.factors.resize(n);
    rr.final_x.resize(n);
    w.fetch(rr.factors.data(), w.U, n);
    w.fetch(rr.final_x.data(), w.Xprev, n);
    w.sync();
    if (lam < 0.0) {
        lam = -lam;
        for (uint64_t i = 0; i < w.dims[0]; ++i) rr.factors[i] = -rr.factors[i];
    }
    rr.lambda = lam;
    // phase times (events)
    for (size_t k = 0; k < marks.size(); ++k) {
        auto& r = rr.trace[k];
        const Marks& m = marks[k];
        r.t_eig = Events::secs(m.a, m.b);
        const double t_rqi_sweep = m.f ? Events::secs(m.f, m.g) : 0.0;
        r.t_build_j = Events::secs(m.c, m.d2) + (k == 0 ? Events::secs(e0, e1) : 0.0) + t_rqi_sweep;
        r.t_other = Events::secs(m.b, m.c) + Events::secs(m.d2, m.e) - t_rqi_sweep;
    }
    return rr;
}

// ---- the reference's sweep baselines on the device sweep -------------------
// run_power_sweep (solvers.cpp:299-354) and run_asvd (:400-447).  Every
// contraction they need comes out of the fused sweep at the current factors:
//   contract_leaving(A, u, n) = w_n = sqrt(d) (J(u) xhat)_n (one pass over A,
//   like the reference's single-output TTV chain), contract_leaving_all = all
//   d of them from the same pass, build_block(A, u, m, n) = block (m, n) of
//   J(u), multilinear_value = u_0' w_0, kkt_report = the post step.
// The stop evaluation at the new factors (baseline_stop, :100-127) is one
// sweep whose J also feeds the next iteration's first contraction, so
// Jacobi-HOPM and Jacobi-ASVD cost one pass over A per iteration, HOPM d
// and ASVD one per pair whose inputs changed.
enum class Baseline { hopm, jacobi_hopm, asvd, jacobi_asvd };

// asvd_pairs (solvers.cpp:383-397)
std::vector<std::pair<int, int>> asvd_pairs(int d, bool disjoint, int iteration) {
    std::vector<std::pair<int, int>> pairs;
    if (disjoint) {
        const int offset = d > 2 ? (iteration - 1) % 2 : 0;
        for (int m = offset; m + 1 < d; m += 2) pairs.emplace_back(m, m + 1);
        return pairs;
    }
    for (int m = 0; m + 1 < d; ++m) pairs.emplace_back(m, m + 1);
    if (d > 2) pairs.emplace_back(0, d - 1);
    return pairs;
}

RunResult run_baseline(Work& w, const r1_solve_options& o, const std::vector<double>& u0,
                       Baseline kind) {
    RunResult rr;
    Events& ev = w.events;
    ev.reset();
    r1_context* ctx = w.ctx;
    const cudaStream_t st = w.st();
    const int d = w.d;
    const int64_t n = w.n;
    const uint64_t* dims = w.dims.data();
    double* h = w.hst.as<double>();
    int* hf = reinterpret_cast<int*>(h + 60);
    double* norms = w.dotv + 8;  // d <= 16 entries
    R1_CUDA(cudaMemcpyAsync(w.U, u0.data(), n * sizeof(double), cudaMemcpyHostToDevice, st));

    // ||A||_F for the kkt rule (solvers.cpp:305, 108)
    double a_norm = 0.0;
    if (o.stop_rule == R1_STOP_KKT) {
        sumsq_device(ctx, w.A->dev, numel_of(dims, d), w.dotv);
        w.fetch(h, w.dotv, 1);
        w.sync();
        a_norm = std::sqrt(h[0]);
    }
    struct Sweep {
        int iter;
        cudaEvent_t a, b;
    };
    std::vector<Sweep> sweeps;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> marks;
    auto sweep = [&](int iter) {
        cudaEvent_t a = ev.rec(st);
        w.sweep(w.U, w.J, w.fro2);
        sweeps.push_back({iter, a, ev.rec(st)});
        rr.sweeps += 1;
    };
    // y = J(u) xhat: the leave-one-out vectors of the current factors
    auto loo_eval = [&](int iter) {
        sweep(iter);
        split_stack(ctx, dims, d, w.U, nullptr, w.Xhat, nullptr);
        block_matvec(ctx, dims, d, w.J, w.Xhat, w.Y);
    };
    // loo_eval + lambda, Eq. 11 (mu = lambda of the iteration) and KKT
    auto full_eval = [&](int iter, const double* mu_dev) {
        loo_eval(iter);
        if (mu_dev)
            r1::post_step(ctx, dims, d, w.Y, w.Xhat, w.U, w.fro2, mu_dev, 0.0, w.post);
        else
            post_step_self(ctx, dims, d, w.Y, w.Xhat, w.U, w.fro2, w.post);
    };

    full_eval(0, nullptr);
    w.fetch(h, w.post, 5);
    w.sync();
    rr.lambda0 = h[4];  // multilinear_value(a, u) (solvers.cpp:303)
    double lambda_prev = rr.lambda0;
    const char* what = kind == Baseline::hopm          ? "hopm: zero contraction vector"
                       : kind == Baseline::jacobi_hopm ? "jacobi_hopm: zero contraction vector"
                                                       : "asvd: singular vector block collapsed to zero";
    std::vector<uint64_t> dims2(2);

    for (int k = 1; k <= o.max_iters; ++k) {
        r1_iteration_record rec{};
        rec.lambda_pre_rqi = kNan;
        rec.factor_change = -1.0;
        cudaEvent_t t0 = ev.rec(st);
        const size_t nsw0 = sweeps.size();
        double lambda = 0.0;
        switch (kind) {
            case Baseline::hopm:
                // Gauss-Seidel: mode n contracts against the already-updated 0..n-1
                for (int m = 0; m < d; ++m) {
                    if (m > 0) loo_eval(k);
                    loo_update(ctx, dims, d, w.Y, w.U, m, m + 1, norms, w.flags, m > 0);
                }
                // lambda = ||w_{d-1}|| (solvers.cpp:329)
                full_eval(k, norms + d - 1);
                break;
            case Baseline::jacobi_hopm:
                loo_update(ctx, dims, d, w.Y, w.U, 0, d, norms, w.flags, false);
                full_eval(k, nullptr);  // lambda = multilinear_value at the new u (:321)
                break;
            case Baseline::asvd:
            case Baseline::jacobi_asvd: {
                const bool jacobi = kind == Baseline::jacobi_asvd;
                std::vector<char> dirty(d, 0);
                bool first = true;
                for (auto [m, nn] : asvd_pairs(d, o.asvd_disjoint_pairs != 0, k)) {
                    if (!jacobi) {
                        bool stale = false;
                        for (int q = 0; q < d; ++q) stale |= dirty[q] && q != m && q != nn;
                        if (stale) {
                            sweep(k);
                            std::fill(dirty.begin(), dirty.end(), 0);
                        }
                    }
                    dims2[0] = dims[m];
                    dims2[1] = dims[nn];
                    eig_blocks(ctx, dims2.data(), 2, w.J + block_offset(dims, d, m, nn), nullptr,
                               w.mu, w.X, nullptr, nullptr);
                    asvd_take(ctx, dims, d, m, nn, w.X, w.mu, w.U, w.flags, !first);
                    dirty[m] = dirty[nn] = 1;
                    first = false;
                }
                full_eval(k, nullptr);  // lambda = multilinear_value (:423)
                break;
            }
        }
        w.fetch(h, w.post, 5);
        w.fetch(h + 8, norms, d);
        w.fetch(hf, w.flags, 1);
        w.sync();
        if (hf[0]) throw Degenerate(what);
        lambda = kind == Baseline::hopm ? h[8 + d - 1] : h[4];
        // baseline_stop (solvers.cpp:100-127)
        const double kkt_max = h[2];
        switch (o.stop_rule) {
            case R1_STOP_EQ11:
                rec.eq11_value = h[1];
                rec.stop_value = h[1];
                rec.kkt_max_residual = o.record_kkt ? kkt_max : kNan;
                break;
            case R1_STOP_LAMBDA_DELTA:
                rec.eq11_value = kNan;
                rec.stop_value = std::abs(lambda - lambda_prev) / std::max(std::abs(lambda), 1e-300);
                rec.kkt_max_residual = o.record_kkt ? kkt_max : kNan;
                break;
            default:
                rec.eq11_value = kNan;
                rec.kkt_max_residual = kkt_max;
                rec.stop_value = kkt_max / std::max(a_norm, 1e-300);
                break;
        }
        rec.lambda = lambda;
        rec.n_sweeps = static_cast<int>(sweeps.size() - nsw0);
        lambda_prev = lambda;
        marks.emplace_back(t0, ev.rec(st));
        rr.trace.push_back(rec);
        rr.iterations = k;
        if (rec.stop_value <= o.tol) {
            rr.converged = true;
            break;
        }
    }
    // finalize_sign (solvers.cpp:70-76) with lambda of the last evaluation
    double lam = h[4];
    rr.factors.resize(n);
    w.fetch(rr.factors.data(), w.U, n);
    w.sync();
    if (lam < 0.0) {
        lam = -lam;
        for (uint64_t i = 0; i < w.dims[0]; ++i) rr.factors[i] = -rr.factors[i];
    }
    rr.lambda = lam;
    // device sweep time per iteration -> t_build_j, the rest -> t_other
    for (size_t k = 0; k < marks.size(); ++k) {
        auto& r = rr.trace[k];
        double tb = 0.0;
        for (const auto& s : sweeps)
            if (s.iter == static_cast<int>(k) + 1) tb += Events::secs(s.a, s.b);
        r.t_build_j = tb;
        r.t_eig = 0.0;
        r.t_other = std::max(0.0, Events::secs(marks[k].first, marks[k].second) - tb);
    }
    return rr;
}

std::vector<double> initial_factors(const std::vector<uint64_t>& dims, const r1_solve_options& o) {
    const int d = static_cast<int>(dims.size());
    if (o.init == R1_INIT_PROVIDED) {
        if (!o.init_factors) fail(R1_ERR_INVALID_ARGUMENT, "solver: provided init has wrong order");
        uint64_t n = 0;
        for (auto v : dims) n += v;
        std::vector<double> f(o.init_factors, o.init_factors + n);
        uint64_t off = 0;
        for (int k = 0; k < d; ++k) {
            if (normalize(f.data() + off, dims[k]) == 0.0)
                fail(R1_ERR_INVALID_ARGUMENT, "solver: provided init factor is zero");
            off += dims[k];
        }
        return f;
    }
    return random_unit_factors(dims, o.seed, kStreamInit);
}

}  // namespace

void forget_solver_work(r1_context* ctx) {
    std::lock_guard<std::mutex> cache_lock(cache_mutex());
    auto& m = work_cache();
    for (auto it = m.begin(); it != m.end();)
        if (it->first.first == ctx)
            it = m.erase(it);
        else
            ++it;
}

}  // namespace r1

using namespace r1;

extern "C" {

static void solve_impl(r1_context* ctx, const char* algorithm, const r1_tensor* a,
                       const r1_solve_options* opts, r1_solve_report* report,
                       const uint64_t* gdims = nullptr);

int r1_solve(r1_context* ctx, const char* algorithm, const r1_tensor* a,
             const r1_solve_options* opts, r1_solve_report* report) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx) fail(R1_ERR_INVALID_ARGUMENT, "null context");
        R1_CUDA(cudaSetDevice(ctx->device));
        solve_impl(ctx, algorithm, a, opts, report);
    });
}

// rank1::solve(name, DenseTensor, opts) from a host tensor: staged once into the
// context's upload buffer (no allocation per call), then the device solve.
int r1_solve_host(r1_context* ctx, const char* algorithm, const double* a_host,
                  const uint64_t* dims, int order, const r1_solve_options* opts,
                  r1_solve_report* report) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx || !a_host || !dims) fail(R1_ERR_INVALID_ARGUMENT, "null argument");
        R1_CUDA(cudaSetDevice(ctx->device));
        if (order < 1 || order > 16) fail(R1_ERR_INVALID_ARGUMENT, "solver: unsupported order");
        const r1_tensor* t = upload_tensor(ctx, a_host, dims, order);
        solve_impl(ctx, algorithm, t, opts, report);
    });
}

int r1_solve_sharded(r1_context* ctx, const char* algorithm, const r1_tensor* slab,
                     const uint64_t* global_dims, int order, const r1_solve_options* opts,
                     r1_solve_report* report) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx || !slab || !global_dims) fail(R1_ERR_INVALID_ARGUMENT, "null argument");
        if (!ctx->comm) fail(R1_ERR_INVALID_ARGUMENT, "sharded solve: no communicator attached");
        if (order != static_cast<int>(slab->dims.size()))
            fail(R1_ERR_INVALID_ARGUMENT, "sharded solve: order mismatch");
        R1_CUDA(cudaSetDevice(ctx->device));
        solve_impl(ctx, algorithm, slab, opts, report, global_dims);
    });
}

int r1_build_j_sharded(r1_context* ctx, const r1_tensor* slab, const uint64_t* global_dims, int order,
                       const double* factors_dev, double* blocks_dev, double* fro2_dev) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx || !slab || !global_dims || !factors_dev || !blocks_dev)
            fail(R1_ERR_INVALID_ARGUMENT, "null argument");
        if (!ctx->comm) fail(R1_ERR_INVALID_ARGUMENT, "sharded sweep: no communicator attached");
        if (order < 2 || order != static_cast<int>(slab->dims.size()))
            fail(R1_ERR_INVALID_ARGUMENT, "sharded sweep: order mismatch");
        R1_CUDA(cudaSetDevice(ctx->device));
        if (global_dims[order - 1] < static_cast<uint64_t>(ctx->comm->world))
            fail(R1_ERR_INVALID_ARGUMENT, "sharded sweep: the last mode has fewer entries than ranks");
        uint64_t lo, hi;
        slab_bounds(global_dims[order - 1], ctx->comm->world, ctx->comm->rank, &lo, &hi);
        if (hi - lo != slab->dims[order - 1])
            fail(R1_ERR_INVALID_ARGUMENT, "sharded sweep: slab extent does not match this rank's share");
        // local blocks in the context's sweep-exchange buffer
        const uint64_t lnb = blocks_numel(slab->dims.data(), order);
        ctx->ws_xchg.ensure((lnb + 32) * sizeof(double));
        uint64_t off = 0;
        for (int k = 0; k + 1 < order; ++k) off += global_dims[k];
        sweep_blocks(ctx, slab->dev, slab->dims.data(), order, factors_dev, ctx->ws_xchg.as<double>(),
                     factors_dev + off + lo);
        exchange_blocks(ctx, ctx->ws_xchg.as<double>(), blocks_dev, global_dims, order);
        if (fro2_dev) sumsq_device(ctx, blocks_dev, blocks_numel(global_dims, order), fro2_dev);
    });
}

}  // extern "C"

static void solve_impl(r1_context* ctx, const char* algorithm, const r1_tensor* a,
                       const r1_solve_options* opts, r1_solve_report* report,
                       const uint64_t* gdims) {
    {
        const std::string alg = algorithm ? algorithm : "";
        const bool baseline =
            alg == "hopm" || alg == "jacobi_hopm" || alg == "asvd" || alg == "jacobi_asvd";
        if (alg != "hoscf" && alg != "ihoscf" && !baseline)
            fail(R1_ERR_INVALID_ARGUMENT, "unknown solver: " + alg);
        if (!a || !opts || !report) fail(R1_ERR_INVALID_ARGUMENT, "null argument");
        // validate (solvers.cpp:28-32)
        if (a->dims.size() < 2) fail(R1_ERR_INVALID_ARGUMENT, "solver: tensor order must be >= 2");
        if (!(opts->tol > 0.0)) fail(R1_ERR_INVALID_ARGUMENT, "solver: tol must be > 0");
        if (opts->max_iters < 1) fail(R1_ERR_INVALID_ARGUMENT, "solver: max_iters must be >= 1");
        const bool acc = alg == "ihoscf";
        auto t0 = std::chrono::steady_clock::now();
        if (gdims && baseline)
            fail(R1_ERR_INVALID_ARGUMENT, "sharded solves support hoscf and ihoscf: " + alg);
        Work& w = work_for(ctx, a, acc, gdims);
        RunResult rr;
        bool restarted = false;
        const Baseline bk = alg == "hopm"          ? Baseline::hopm
                            : alg == "jacobi_hopm" ? Baseline::jacobi_hopm
                            : alg == "asvd"        ? Baseline::asvd
                                                   : Baseline::jacobi_asvd;
        auto go = [&](const std::vector<double>& u0) {
            if (baseline) return run_baseline(w, *opts, u0, bk);
            static const char* host_loop = dev_env("R1_HOSCF_HOST_LOOP");  // development A/B
            if (acc || (host_loop && std::atoi(host_loop) != 0)) return run(w, *opts, u0, acc);
            return run_hoscf_dev(w, *opts, u0);
        };
        try {
            rr = go(initial_factors(w.dims, *opts));
        } catch (const Degenerate&) {
            try {
                rr = go(random_unit_factors(w.dims, opts->seed, kStreamRestart));
                restarted = true;
            } catch (const Degenerate& e) {
                fail(R1_ERR_RUNTIME, std::string("solver failed after restart: ") + e.what());
            }
        }
        auto t1 = std::chrono::steady_clock::now();
        report->lambda = rr.lambda;
        std::memcpy(report->factors, rr.factors.data(), rr.factors.size() * sizeof(double));
        report->converged = rr.converged ? 1 : 0;
        report->iterations = rr.iterations;
        report->lambda0 = rr.lambda0;
        report->restarted = restarted ? 1 : 0;
        // baselines: final_x stays empty (solvers.hpp:56), reported as zeros
        if (report->final_x) {
            std::memset(report->final_x, 0, rr.factors.size() * sizeof(double));
            std::memcpy(report->final_x, rr.final_x.data(), rr.final_x.size() * sizeof(double));
        }
        for (int i = 0; i < rr.iterations; ++i) report->trace[i] = rr.trace[i];
        report->total_sweeps = rr.sweeps;
        report->t_total = std::chrono::duration<double>(t1 - t0).count();
    }
}

extern "C" {

int r1_eig_blocks_device(r1_context* ctx, const uint64_t* dims, int order, const double* blocks_dev,
                         const double* x0_dev, double* value_dev, double* vec_dev) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx) fail(R1_ERR_INVALID_ARGUMENT, "null context");
        R1_CUDA(cudaSetDevice(ctx->device));
        eig_blocks(ctx, dims, order, blocks_dev, x0_dev, value_dev, vec_dev, nullptr, nullptr);
    });
}

// Diagnostics (not in the public header): the loop mode of the last HOSCF solve.
int r1x_solver_graph_mode(r1_context* ctx, int* mode) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx || !mode) fail(R1_ERR_INVALID_ARGUMENT, "null argument");
        *mode = ctx->solver_graph_mode;
    });
}

// Diagnostics (not in the public header): eig on host blocks with info/stats.
int r1x_eig_blocks_info(r1_context* ctx, const uint64_t* dims, int order, const double* blocks_host,
                        double* value, double* vec, int* info, double* stats) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx) fail(R1_ERR_INVALID_ARGUMENT, "null context");
        R1_CUDA(cudaSetDevice(ctx->device));
        const uint64_t nb = blocks_numel(dims, order);
        uint64_t n = 0;
        for (int k = 0; k < order; ++k) n += dims[k];
        DeviceBuffer b, v;
        b.ensure(nb * sizeof(double));
        v.ensure((n + 8) * sizeof(double));
        R1_CUDA(cudaMemcpyAsync(b.ptr, blocks_host, nb * sizeof(double), cudaMemcpyHostToDevice,
                                ctx->stream));
        eig_blocks(ctx, dims, order, b.as<double>(), nullptr, v.as<double>() + n,
                   v.as<double>(), info, stats);
        R1_CUDA(cudaMemcpyAsync(vec, v.ptr, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaMemcpyAsync(value, v.as<double>() + n, sizeof(double), cudaMemcpyDeviceToHost,
                                ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

// Diagnostics (not in the public header): Lanczos (the solvers' eigen step)
// on a dense host matrix.  The public dense entry r1_largest_magnitude_eigenpair
// is the reference's full decomposition (dense_api.cu).
int r1x_eig_dense_lanczos(r1_context* ctx, int64_t n, const double* s_host, double* value,
                          double* vec) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx) fail(R1_ERR_INVALID_ARGUMENT, "null context");
        R1_CUDA(cudaSetDevice(ctx->device));
        if (n <= 0) fail(R1_ERR_INVALID_ARGUMENT, "largest_magnitude_eigenpair: empty matrix");
        // check_symmetric (sym_eig.cpp:13-22)
        double scale = 0.0, dev = 0.0;
        for (int64_t i = 0; i < n * n; ++i) scale = std::max(scale, std::abs(s_host[i]));
        for (int64_t j = 0; j < n; ++j)
            for (int64_t i = j + 1; i < n; ++i)
                dev = std::max(dev, std::abs(s_host[i + j * n] - s_host[j + i * n]));
        if (dev > 1e-10 * std::max(scale, 1e-300))
            fail(R1_ERR_INVALID_ARGUMENT, "sym_eig: matrix is not symmetric");
        DeviceBuffer S, v;
        S.ensure(static_cast<size_t>(n) * n * sizeof(double));
        v.ensure((n + 8) * sizeof(double));
        R1_CUDA(cudaMemcpyAsync(S.ptr, s_host, static_cast<size_t>(n) * n * sizeof(double),
                                cudaMemcpyHostToDevice, ctx->stream));
        int info[5];
        eig_dense(ctx, n, S.as<double>(), nullptr, v.as<double>() + n, v.as<double>(), info, nullptr);
        if (!info[0]) fail(R1_ERR_RUNTIME, "sym_eig: Lanczos iteration did not converge");
        R1_CUDA(cudaMemcpyAsync(vec, v.ptr, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaMemcpyAsync(value, v.as<double>() + n, sizeof(double), cudaMemcpyDeviceToHost,
                                ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int r1_rayleigh_quotient_step(r1_context* ctx, int64_t n, const double* s_host, const double* x_host,
                              double* y_host, int* accepted) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx) fail(R1_ERR_INVALID_ARGUMENT, "null context");
        R1_CUDA(cudaSetDevice(ctx->device));
        if (n <= 0) fail(R1_ERR_INVALID_ARGUMENT, "rayleigh_quotient_step: size mismatch");
        DeviceBuffer S, v;
        S.ensure(static_cast<size_t>(n) * n * sizeof(double));
        v.ensure(2 * n * sizeof(double));
        R1_CUDA(cudaMemcpyAsync(S.ptr, s_host, static_cast<size_t>(n) * n * sizeof(double),
                                cudaMemcpyHostToDevice, ctx->stream));
        R1_CUDA(cudaMemcpyAsync(v.ptr, x_host, n * sizeof(double), cudaMemcpyHostToDevice,
                                ctx->stream));
        const bool ok = rqi_step(ctx, n, S.as<double>(), v.as<double>(), v.as<double>() + n);
        *accepted = ok ? 1 : 0;
        if (ok) {
            R1_CUDA(cudaMemcpyAsync(y_host, v.as<double>() + n, n * sizeof(double),
                                    cudaMemcpyDeviceToHost, ctx->stream));
            R1_CUDA(cudaStreamSynchronize(ctx->stream));
        }
    });
}

// contract_leaving_all (tensor.cpp:216-238) from one device sweep: with unit
// factors v_k = u_k / |u_k| (a zero factor is replaced by e_0 and its norm 0
// kept), w_n = A x_{k != n} u_k = (prod_{k != n} |u_k|) sqrt(d) (J(v) vhat)_n.
// out: flat sum I_k (w_0 ++ ... ++ w_{d-1}).
int r1_contract_leaving_all(r1_context* ctx, const double* a_host, const r1_tensor* a_dev,
                            const uint64_t* dims, int order, const double* factors_host,
                            double* out_host) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx || !dims || !factors_host || !out_host) fail(R1_ERR_INVALID_ARGUMENT, "null argument");
        R1_CUDA(cudaSetDevice(ctx->device));
        if (order < 2 || order > 16)
            fail(R1_ERR_INVALID_ARGUMENT, "contract_leaving_all: order mismatch");
        uint64_t n = 0;
        for (int k = 0; k < order; ++k) n += dims[k];
        std::vector<double> v(factors_host, factors_host + n), norms(order);
        uint64_t off = 0;
        for (int k = 0; k < order; ++k) {
            norms[k] = normalize(v.data() + off, dims[k]);
            if (norms[k] == 0.0) v[off] = 1.0;
            off += dims[k];
        }
        const r1_tensor* t = a_dev;
        if (!t) {
            if (!a_host) fail(R1_ERR_INVALID_ARGUMENT, "no tensor given");
            t = upload_tensor(ctx, a_host, dims, order);
        }
        const uint64_t nb = blocks_numel(dims, order);
        const uint64_t nba = (nb + 31) & ~uint64_t(31), na = (n + 31) & ~uint64_t(31);
        ctx->ws_io.ensure((nba + 3 * na + 64) * sizeof(double));
        double* b = ctx->ws_io.as<double>();
        double* u = b + nba;
        double* xh = u + na;
        double* y = xh + na;
        R1_CUDA(cudaMemcpyAsync(u, v.data(), n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        sweep_blocks(ctx, t->dev, dims, order, u, b);
        split_stack(ctx, dims, order, u, nullptr, xh, nullptr);
        block_matvec(ctx, dims, order, b, xh, y);
        R1_CUDA(cudaMemcpyAsync(out_host, y, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
        const double sqd = std::sqrt(static_cast<double>(order));
        off = 0;
        for (int k = 0; k < order; ++k) {
            double sc = sqd;
            for (int m = 0; m < order; ++m)
                if (m != k) sc *= norms[m];
            for (uint64_t i = 0; i < dims[k]; ++i) out_host[off + i] *= sc;
            off += dims[k];
        }
    });
}

// Host-buffer forms of the SymBlockMatrix operations (nepv.cpp:110-157) for the
// C++ container: y = J x, dense J, ||J||_F, all on the device.
int r1_block_matvec(r1_context* ctx, const uint64_t* dims, int order, const double* blocks_host,
                    const double* x_host, double* y_host) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx || !dims) fail(R1_ERR_INVALID_ARGUMENT, "null argument");
        R1_CUDA(cudaSetDevice(ctx->device));
        if (order < 2 || order > 16) fail(R1_ERR_INVALID_ARGUMENT, "SymBlockMatrix: order must be >= 2");
        const uint64_t nb = blocks_numel(dims, order);
        uint64_t n = 0;
        for (int k = 0; k < order; ++k) n += dims[k];
        ctx->ws_io.ensure((nb + 2 * n + 64) * sizeof(double));
        double* b = ctx->ws_io.as<double>();
        double* x = b + ((nb + 31) & ~uint64_t(31));
        double* y = x + ((n + 31) & ~uint64_t(31));
        R1_CUDA(cudaMemcpyAsync(b, blocks_host, nb * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        R1_CUDA(cudaMemcpyAsync(x, x_host, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        block_matvec(ctx, dims, order, b, x, y);
        R1_CUDA(cudaMemcpyAsync(y_host, y, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int r1_block_dense(r1_context* ctx, const uint64_t* dims, int order, const double* blocks_host,
                   double* s_host) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx || !dims) fail(R1_ERR_INVALID_ARGUMENT, "null argument");
        R1_CUDA(cudaSetDevice(ctx->device));
        if (order < 2 || order > 16) fail(R1_ERR_INVALID_ARGUMENT, "SymBlockMatrix: order must be >= 2");
        const uint64_t nb = blocks_numel(dims, order);
        uint64_t n = 0;
        for (int k = 0; k < order; ++k) n += dims[k];
        ctx->ws_io.ensure((nb + n * n + 64) * sizeof(double));
        double* b = ctx->ws_io.as<double>();
        double* S = b + ((nb + 31) & ~uint64_t(31));
        R1_CUDA(cudaMemcpyAsync(b, blocks_host, nb * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        dense_from_blocks(ctx, dims, order, b, S);
        R1_CUDA(cudaMemcpyAsync(s_host, S, n * n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int r1_block_frobenius(r1_context* ctx, const uint64_t* dims, int order, const double* blocks_host,
                       double* out) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx || !dims || !out) fail(R1_ERR_INVALID_ARGUMENT, "null argument");
        R1_CUDA(cudaSetDevice(ctx->device));
        if (order < 2 || order > 16) fail(R1_ERR_INVALID_ARGUMENT, "SymBlockMatrix: order must be >= 2");
        const uint64_t nb = blocks_numel(dims, order);
        ctx->ws_io.ensure((nb + 64) * sizeof(double));
        double* b = ctx->ws_io.as<double>();
        double* f2 = b + ((nb + 31) & ~uint64_t(31));
        R1_CUDA(cudaMemcpyAsync(b, blocks_host, nb * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        sumsq_device(ctx, b, nb, f2);
        double h = 0.0;
        R1_CUDA(cudaMemcpyAsync(&h, f2, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
        *out = std::sqrt(2.0 * h) / static_cast<double>(order - 1);  // nepv.cpp:152-157
    });
}

int r1_scf_stopping_value(r1_context* ctx, const uint64_t* dims, int order, const double* blocks_host,
                          const double* x_host, double lambda, double* out) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx) fail(R1_ERR_INVALID_ARGUMENT, "null context");
        R1_CUDA(cudaSetDevice(ctx->device));
        const uint64_t nb = blocks_numel(dims, order);
        uint64_t n = 0;
        for (int k = 0; k < order; ++k) n += dims[k];
        DeviceBuffer b, v;
        b.ensure(nb * sizeof(double));
        v.ensure((3 * n + 80) * sizeof(double));
        double* x = v.as<double>();
        double* y = x + n;
        double* f2 = y + n;
        double* out_d = f2 + 8;
        R1_CUDA(cudaMemcpyAsync(b.ptr, blocks_host, nb * sizeof(double), cudaMemcpyHostToDevice,
                                ctx->stream));
        R1_CUDA(cudaMemcpyAsync(x, x_host, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        sumsq_device(ctx, b.as<double>(), nb, f2);
        block_matvec(ctx, dims, order, b.as<double>(), x, y);
        // the u argument only feeds the KKT outputs, which are ignored here
        post_step(ctx, dims, order, y, x, x, f2, nullptr, lambda, out_d);
        double h[8];
        R1_CUDA(cudaMemcpyAsync(h, out_d, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
        *out = h[1];
    });
}

// out: [lambda, max_residual, r_0..r_{d-1}]
int r1_kkt_from_blocks(r1_context* ctx, const uint64_t* dims, int order, const double* blocks_host,
                       const double* factors_host, double* out) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx) fail(R1_ERR_INVALID_ARGUMENT, "null context");
        R1_CUDA(cudaSetDevice(ctx->device));
        const uint64_t nb = blocks_numel(dims, order);
        uint64_t n = 0;
        for (int k = 0; k < order; ++k) n += dims[k];
        DeviceBuffer b, v;
        b.ensure(nb * sizeof(double));
        v.ensure((4 * n + 80) * sizeof(double));
        double* u = v.as<double>();
        double* xh = u + n;
        double* y = xh + n;
        double* f2 = y + n;
        double* out_d = f2 + 8;
        R1_CUDA(cudaMemcpyAsync(b.ptr, blocks_host, nb * sizeof(double), cudaMemcpyHostToDevice,
                                ctx->stream));
        {
            // check_unit_nonzero (nepv.cpp:31-41) as kkt_report does
            uint64_t off = 0;
            for (int k = 0; k < order; ++k) {
                double s = 0.0;
                for (uint64_t i = 0; i < dims[k]; ++i) s += factors_host[off + i] * factors_host[off + i];
                const double nrm = std::sqrt(s);
                if (nrm < 1e-12)
                    fail(R1_ERR_RUNTIME, "degenerate factor set: zero factor for mode " + std::to_string(k));
                if (std::abs(nrm - 1.0) > 1e-8)
                    fail(R1_ERR_INVALID_ARGUMENT, "factor for mode " + std::to_string(k) + " is not unit length");
                off += dims[k];
            }
        }
        R1_CUDA(cudaMemcpyAsync(u, factors_host, n * sizeof(double), cudaMemcpyHostToDevice,
                                ctx->stream));
        split_stack(ctx, dims, order, u, nullptr, xh, nullptr);
        sumsq_device(ctx, b.as<double>(), nb, f2);
        block_matvec(ctx, dims, order, b.as<double>(), xh, y);
        post_step(ctx, dims, order, y, xh, u, f2, nullptr, 0.0, out_d);
        std::vector<double> h(5 + order);
        R1_CUDA(cudaMemcpyAsync(h.data(), out_d, h.size() * sizeof(double), cudaMemcpyDeviceToHost,
                                ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
        out[0] = h[4];
        out[1] = h[2];
        for (int k = 0; k < order; ++k) out[2 + k] = h[5 + k];
    });
}

int r1_kkt_report(r1_context* ctx, const double* a_host, const r1_tensor* a_dev, const uint64_t* dims,
                  int order, const double* factors_host, double* out) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx) fail(R1_ERR_INVALID_ARGUMENT, "null context");
        const uint64_t nb = blocks_numel(dims, order);
        std::vector<double> blocks(nb);
        int rc = r1_build_j(ctx, a_host, a_dev, dims, order, factors_host, blocks.data());
        if (rc != R1_OK) fail(rc, r1_last_error());
        rc = r1_kkt_from_blocks(ctx, dims, order, blocks.data(), factors_host, out);
        if (rc != R1_OK) fail(rc, r1_last_error());
    });
}

}  // extern "C"
