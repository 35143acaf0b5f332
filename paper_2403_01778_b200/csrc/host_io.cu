// Host <-> device movement of whole tensors for the host-buffer entry points
// (r1_build_j / r1_build_block / r1_kkt_report / r1_tensor_from_host, i.e. the
// C-ABI behind rank1::build_j(const DenseTensor&, ...), nepv.hpp:58).
//
// The reference's DenseTensor owns a pageable std::vector<double>.  A plain
// cudaMemcpy from pageable memory runs through the driver's single staging
// buffer (~10-20 GB/s); a one-time cudaHostRegister of the caller's vector
// would make later calls fast but is unsafe behind a by-const& API: the
// registration outlives a freed vector and silently redirects DMA for whatever
// is allocated at that address next.  So:
//  * pinned sources (cudaHostAlloc / cudaHostRegister'ed by the caller, e.g.
//    through r1_host_register) go straight to the copy engine;
//  * pageable sources stream through per-context pinned staging rings: T host
//    threads each own a lane (chunks t, t+T, ...), copy their chunk into one
//    of two pinned buffers and issue its H2D on the lane's own stream, so host
//    memcpy and PCIe DMA overlap; the lanes join the context stream by events.
// Device destination buffers are grow-only per context (no cudaMalloc per call).
#include "common.cuh"

#include <algorithm>
#include <cstring>
#include <thread>

namespace r1 {

namespace {

constexpr size_t kChunkBytes = size_t(16) << 20;  // 16 MiB per staging buffer
constexpr int kLanes = 8;

bool is_pinned(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

}  // namespace

void HostStaging::ensure(int device) {
    if (ready) return;
    R1_CUDA(cudaSetDevice(device));
    for (int l = 0; l < kStageLanes; ++l) {
        R1_CUDA(cudaStreamCreateWithFlags(&lane[l].stream, cudaStreamNonBlocking));
        for (int b = 0; b < 2; ++b) {
            R1_CUDA(cudaMallocHost(&lane[l].buf[b], kChunkBytes));
            R1_CUDA(cudaEventCreateWithFlags(&lane[l].done[b], cudaEventDisableTiming));
        }
        R1_CUDA(cudaEventCreateWithFlags(&lane[l].joined, cudaEventDisableTiming));
    }
    ready = true;
}

HostStaging::~HostStaging() {
    if (!ready) return;
    for (int l = 0; l < kStageLanes; ++l) {
        if (lane[l].stream) cudaStreamSynchronize(lane[l].stream);
        for (int b = 0; b < 2; ++b) {
            if (lane[l].buf[b]) cudaFreeHost(lane[l].buf[b]);
            if (lane[l].done[b]) cudaEventDestroy(lane[l].done[b]);
        }
        if (lane[l].joined) cudaEventDestroy(lane[l].joined);
        if (lane[l].stream) cudaStreamDestroy(lane[l].stream);
    }
}

// dst (device) <- src (host), `bytes` bytes, ordered on ctx->stream.
void h2d_bytes(r1_context* ctx, void* dst, const void* src, size_t bytes) {
    if (bytes == 0) return;
    if (bytes <= kChunkBytes || is_pinned(src)) {
        R1_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
        return;
    }
    HostStaging& S = ctx->staging;
    S.ensure(ctx->device);
    static_assert(kLanes == kStageLanes, "lane count");
    // the destination may still be read by earlier work on the context stream
    cudaEvent_t start;
    R1_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
    R1_CUDA(cudaEventRecord(start, ctx->stream));
    const size_t nchunks = (bytes + kChunkBytes - 1) / kChunkBytes;
    const int lanes = static_cast<int>(std::min<size_t>(kLanes, nchunks));
    std::vector<std::string> errors(lanes);
    auto lane_fn = [&](int l) {
        try {
            R1_CUDA(cudaSetDevice(ctx->device));
            HostStaging::Lane& L = S.lane[l];
            R1_CUDA(cudaStreamWaitEvent(L.stream, start, 0));
            int b = 0;
            for (size_t c = l; c < nchunks; c += lanes) {
                const size_t off = c * kChunkBytes;
                const size_t len = std::min(kChunkBytes, bytes - off);
                R1_CUDA(cudaEventSynchronize(L.done[b]));  // buffer b free again
                std::memcpy(L.buf[b], static_cast<const char*>(src) + off, len);
                R1_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, L.buf[b], len,
                                        cudaMemcpyHostToDevice, L.stream));
                R1_CUDA(cudaEventRecord(L.done[b], L.stream));
                b ^= 1;
            }
            R1_CUDA(cudaEventRecord(L.joined, L.stream));
        } catch (const std::exception& e) {
            errors[l] = e.what();
        }
    };
    std::vector<std::thread> th;
    for (int l = 1; l < lanes; ++l) th.emplace_back(lane_fn, l);
    lane_fn(0);
    for (auto& t : th) t.join();
    cudaEventDestroy(start);
    for (auto& e : errors)
        if (!e.empty()) fail(R1_ERR_CUDA, e);
    for (int l = 0; l < lanes; ++l) R1_CUDA(cudaStreamWaitEvent(ctx->stream, S.lane[l].joined, 0));
}

// A device copy of a host tensor in the context's grow-only upload buffer,
// returned as a (non-owning) tensor view valid until the next upload.
const r1_tensor* upload_tensor(r1_context* ctx, const double* host, const uint64_t* dims, int order) {
    const uint64_t n = numel_of(dims, order);
    const size_t bytes = ((n + 2) * sizeof(double) + 255) & ~size_t(255);
    ctx->ws_upload.ensure(bytes);
    r1_tensor& t = ctx->upload_view;
    t.ctx = ctx;
    t.dims.assign(dims, dims + order);
    t.numel = n;
    t.dev = ctx->ws_upload.as<double>();
    t.owned = false;
    h2d_bytes(ctx, t.dev, host, n * sizeof(double));
    return &t;
}

}  // namespace r1

using namespace r1;

extern "C" {

int r1_host_register(void* host, uint64_t bytes) {
    return abi_guard([&] {
        if (!host || bytes == 0) fail(R1_ERR_INVALID_ARGUMENT, "r1_host_register: empty range");
        R1_CUDA(cudaHostRegister(host, bytes, cudaHostRegisterPortable));
    });
}

int r1_host_unregister(void* host) {
    return abi_guard([&] {
        if (!host) fail(R1_ERR_INVALID_ARGUMENT, "r1_host_unregister: null pointer");
        R1_CUDA(cudaHostUnregister(host));
    });
}

}  // extern "C"
