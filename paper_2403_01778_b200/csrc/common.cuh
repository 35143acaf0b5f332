// Shared host/device plumbing for the B200 HOSCF path: error handling across
// the C-ABI, the device context (stream, events, workspace arena, launch
// counter) and small PTX helpers.  sm_100a only.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#include <cstdint>
#include <cstdio>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "rank1_b200.h"

namespace r1 {

// ------------------------------------------------------------------ errors --
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess) {
        char buf[512];
        snprintf(buf, sizeof(buf), "CUDA error %s (%d) in %s at %s:%d", cudaGetErrorString(e),
                 static_cast<int>(e), what, file, line);
        fail(R1_ERR_CUDA, buf);
    }
}
#define R1_CUDA(x) ::r1::cuda_check((x), #x, __FILE__, __LINE__)

void set_last_error(const std::string& msg);

// Development switches exist only in the development build
// (build.py --dev -> librank1_b200_dev.so, -DR1_DEV_SWITCHES); the release
// library ignores the environment.
#ifdef R1_DEV_SWITCHES
inline const char* dev_env(const char* name) { return std::getenv(name); }
#else
inline const char* dev_env(const char*) { return nullptr; }
#endif

// Runs f, mapping exceptions onto the ABI status codes (never throws).
template <typename F>
int abi_guard(F&& f) {
    try {
        f();
        return R1_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::invalid_argument& e) {
        set_last_error(e.what());
        return R1_ERR_INVALID_ARGUMENT;
    } catch (const std::bad_alloc& e) {
        set_last_error("out of memory");
        return R1_ERR_INTERNAL;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return R1_ERR_RUNTIME;
    } catch (...) {
        set_last_error("unknown error");
        return R1_ERR_INTERNAL;
    }
}

// ---------------------------------------------------------- device buffers --
struct DeviceBuffer {
    void* ptr = nullptr;
    size_t bytes = 0;
    DeviceBuffer() = default;
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    ~DeviceBuffer() {
        if (ptr) cudaFree(ptr);
    }
    void ensure(size_t b) {
        if (b <= bytes) return;
        if (ptr) R1_CUDA(cudaFree(ptr));
        ptr = nullptr;
        bytes = 0;
        R1_CUDA(cudaMalloc(&ptr, b));
        bytes = b;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(ptr);
    }
};

// Device copies of small host descriptors (BlockOp ...) keyed by content: a
// descriptor uploaded before is reused, so the hot loops (HOSCF alternates two
// block buffers) do no host-to-device copy — which would make the host wait
// for the stream.  The host copies live in pinned memory, so an upload issued
// while the stream is being captured into a CUDA graph is a legal memcpy node
// (replayed from the same, unchanging slot).  Users share one stream, so
// reusing a slot is ordered after the kernels that read it.
template <typename T, int N = 4>
struct DescCache {
    T* host = nullptr;  // N pinned slots
    bool used[N] = {};
    int next = 0;
    void* dev[N] = {};
    // the upload of a pinned slot must have run before the host rewrites the
    // slot (the host can be hundreds of launches ahead of the stream)
    cudaEvent_t sent[N] = {};
    bool sent_valid[N] = {};
    DescCache() = default;
    DescCache(const DescCache&) = delete;
    DescCache& operator=(const DescCache&) = delete;
    ~DescCache() {
        for (auto p : dev)
            if (p) cudaFree(p);
        for (auto e : sent)
            if (e) cudaEventDestroy(e);
        if (host) cudaFreeHost(host);
    }
    // All slots are allocated on the first (never captured) use, so a miss
    // while a graph is being captured only records a pinned-host memcpy node.
    const T* get(const T& d, cudaStream_t s) {
        if (!host) {
            R1_CUDA(cudaMallocHost(&host, N * sizeof(T)));
            for (int i = 0; i < N; ++i) R1_CUDA(cudaMalloc(&dev[i], sizeof(T)));
            for (int i = 0; i < N; ++i) R1_CUDA(cudaEventCreateWithFlags(&sent[i], cudaEventDisableTiming));
        }
        for (int i = 0; i < N; ++i)
            if (used[i] && std::memcmp(&host[i], &d, sizeof(T)) == 0) return static_cast<T*>(dev[i]);
        const int i = next;
        next = (next + 1) % N;
        used[i] = false;
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        R1_CUDA(cudaStreamIsCapturing(s, &cap));
        if (sent_valid[i] && cap == cudaStreamCaptureStatusNone) R1_CUDA(cudaEventSynchronize(sent[i]));
        std::memcpy(&host[i], &d, sizeof(T));
        R1_CUDA(cudaMemcpyAsync(dev[i], &host[i], sizeof(T), cudaMemcpyHostToDevice, s));
        if (cap == cudaStreamCaptureStatusNone) {
            R1_CUDA(cudaEventRecord(sent[i], s));
            sent_valid[i] = true;
        }
        used[i] = true;
        return static_cast<T*>(dev[i]);
    }
};

struct PinnedBuffer {
    void* ptr = nullptr;
    size_t bytes = 0;
    ~PinnedBuffer() {
        if (ptr) cudaFreeHost(ptr);
    }
    void ensure(size_t b) {
        if (b <= bytes) return;
        if (ptr) R1_CUDA(cudaFreeHost(ptr));
        ptr = nullptr;
        bytes = 0;
        R1_CUDA(cudaMallocHost(&ptr, b));
        bytes = b;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(ptr);
    }
};

struct SweepPlan;  // sweep.cu

// Per-context pinned staging lanes for pageable host -> device copies (host_io.cu).
constexpr int kStageLanes = 8;
struct HostStaging {
    struct Lane {
        cudaStream_t stream = nullptr;
        void* buf[2] = {nullptr, nullptr};
        cudaEvent_t done[2] = {nullptr, nullptr};
        cudaEvent_t joined = nullptr;
    };
    Lane lane[kStageLanes];
    bool ready = false;
    void ensure(int device);
    HostStaging() = default;
    HostStaging(const HostStaging&) = delete;
    HostStaging& operator=(const HostStaging&) = delete;
    ~HostStaging();
};

// Process-wide lock for the caches keyed by context (plans, work sets,
// handles): lookups and inserts only; the objects themselves belong to one
// context, whose calls are serialised by the context's own mutex.
std::mutex& cache_mutex();

// Runs `f` (kernel attribute setup) once per (key, device), under the cache
// lock so a concurrent launcher on the same device waits until it is done.
std::set<std::pair<const void*, int>>& configured_set();
template <typename F>
void configure_once(const void* key, int device, F&& f) {
    std::lock_guard<std::mutex> g(cache_mutex());
    if (configured_set().count({key, device})) return;
    f();
    configured_set().insert({key, device});
}

}  // namespace r1

// An NCCL communicator of the ranks sharing a sharded tensor (comm.cu).
struct r1_comm {
    void* comm = nullptr;  // ncclComm_t
    int world = 1;
    int rank = 0;
    bool owns = true;
    r1_context* ctx = nullptr;  // the context it is attached to (detached on destroy)
};

struct r1_tensor {
    r1_context* ctx = nullptr;
    std::vector<uint64_t> dims;
    uint64_t numel = 0;
    double* dev = nullptr;
    bool owned = false;
};

struct r1_context {
    int device = 0;
    int num_sms = 148;
    size_t smem_optin = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    // second lane of a sweep (sweep.cu): independent subtrees of the recursion
    // and the B01 second stage run beside the main stream, joined by events
    cudaStream_t side_stream = nullptr;                    // lane 1 (= side_streams[0])
    cudaStream_t side_streams[3] = {nullptr, nullptr, nullptr};  // lanes 1..3
    cudaEvent_t ev_sweep[3] = {nullptr, nullptr, nullptr};  // [0] root box kernel done
    cudaEvent_t ev_done[16] = {};   // outputs of the spine level at depth k done
    cudaEvent_t ev_join[3] = {};    // lane 1..3 finished
    uint64_t launches = 0;
    unsigned long long* dbg_sweep_trace = nullptr;  // diagnostics: per-CTA timing of level 0
    // diagnostics: CUDA events around every top-level sweep kernel launch
    bool time_kernels = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> kernel_events;
    // Workspace arena, grow-only: sweeps, eigen solver, RQI.
    r1::DeviceBuffer ws_sweep;
    r1::DeviceBuffer ws_eig;
    r1::DeviceBuffer ws_rqi;
    r1::DeviceBuffer ws_small;   // factors, scalars, flags
    r1::PinnedBuffer pinned;     // small host staging
    // host-buffer entry points (host_io.cu): device copy of the caller's
    // tensor, its view, factor / block buffers, pinned staging lanes
    r1::DeviceBuffer ws_upload;
    r1::DeviceBuffer ws_xchg;    // local slab blocks of r1_build_j_sharded
    r1::DeviceBuffer ws_io;
    r1_tensor upload_view;
    r1::HostStaging staging;
    r1_comm* comm = nullptr;  // attached communicator (sharded sweeps / solves)
    // diagnostics: how the last HOSCF solve drove its loop (0 direct launches,
    // 1 CUDA-graph replays, 2 graph replays behind conditional IF nodes)
    int solver_graph_mode = -1;
    // calls on one context are serialised (SURVEY §8b threading contract)
    std::recursive_mutex mu;
    std::map<std::vector<uint64_t>, std::shared_ptr<r1::SweepPlan>> plans;
};

namespace r1 {

// Host -> device upload of plan metadata / tables from pageable memory, complete
// on return.  (A synchronous cudaMemcpy from pageable memory returns once the
// data is STAGED; its DMA is ordered with the legacy default stream only, not
// with the context's non-blocking stream — a kernel launched right behind it
// could read the destination before the data landed.  Found with the
// randomised sweep probe: new plans' segment tables read early.)
inline void upload_now(r1_context* ctx, void* dst, const void* src, size_t bytes) {
    if (bytes == 0) return;
    R1_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    R1_CUDA(cudaStreamIsCapturing(ctx->stream, &st));
    if (st == cudaStreamCaptureStatusNone) R1_CUDA(cudaStreamSynchronize(ctx->stream));
}

inline void count_launch(r1_context* ctx, uint64_t n = 1) { ctx->launches += n; }

inline void check_launch(r1_context* ctx, const char* what) {
    count_launch(ctx);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) cuda_check(e, what, __FILE__, __LINE__);
}

inline uint64_t numel_of(const uint64_t* dims, int order) {
    uint64_t n = 1;
    for (int k = 0; k < order; ++k) n *= dims[k];
    return n;
}

inline uint64_t blocks_numel(const uint64_t* dims, int order) {
    uint64_t s = 0;
    for (int m = 0; m < order; ++m)
        for (int n = m + 1; n < order; ++n) s += dims[m] * dims[n];
    return s;
}

// Offset of block (m,n), m<n, in the concatenated pair order (nepv.cpp:98-102).
inline uint64_t block_offset(const uint64_t* dims, int order, int m, int n) {
    uint64_t s = 0;
    for (int a = 0; a < order; ++a)
        for (int b = a + 1; b < order; ++b) {
            if (a == m && b == n) return s;
            s += dims[a] * dims[b];
        }
    return s;
}

// Serialises the calls on one context (null-safe; the entry point reports the
// null context itself).
struct CtxLock {
    r1_context* c;
    explicit CtxLock(r1_context* ctx) : c(ctx) {
        if (c) c->mu.lock();
    }
    explicit CtxLock(const r1_context* ctx) : CtxLock(const_cast<r1_context*>(ctx)) {}
    ~CtxLock() {
        if (c) c->mu.unlock();
    }
    CtxLock(const CtxLock&) = delete;
    CtxLock& operator=(const CtxLock&) = delete;
};

// --------------------------------------------------------- component APIs --
// comm.cu: slabs along the last mode and the per-sweep block exchange
struct ExchangeOp {
    int m, n;
    uint64_t local_off, global_off, local_count, rows;
    int gathered;  // 1: (m, d-1) columns gathered, 0: partial block all-reduced
};
void slab_bounds(uint64_t extent, int world, int rank, uint64_t* lo, uint64_t* hi);
void exchange_plan(const uint64_t* gdims, int order, int world, int rank, std::vector<ExchangeOp>& ops);
void exchange_blocks(r1_context* ctx, const double* lblocks, double* gblocks, const uint64_t* gdims,
                     int order);
// host_io.cu
void h2d_bytes(r1_context* ctx, void* dst, const void* src, size_t bytes);
const r1_tensor* upload_tensor(r1_context* ctx, const double* host, const uint64_t* dims, int order);
// sweep.cu
// last_factor (nullable): read the last mode's factor from there instead of
// factors_dev + sum_{k<d-1} I_k (a slab of a tensor sharded along its last mode)
void sweep_blocks(r1_context* ctx, const double* a, const uint64_t* dims, int order,
                  const double* factors_dev, double* blocks_dev,
                  const double* last_factor = nullptr);
// blockops.cu
void sumsq_device(r1_context* ctx, const double* x, uint64_t n, double* out_dev);
void block_matvec(r1_context* ctx, const uint64_t* dims, int order, const double* blocks,
                  const double* x, double* y);

}  // namespace r1
