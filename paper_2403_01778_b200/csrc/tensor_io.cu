// .dt1 tensor files straight to / from HBM (reference proj/src/tensor_io.cpp:47-100,
// format tensor_io.hpp:9-14): magic "DTEN1\0", u8 order d >= 2, d little-endian
// u64 dims, prod(dims) little-endian f64 values, first index fastest — i.e.
// exactly the device layout, so the payload streams file -> pinned staging ->
// HBM in chunks with the disk read of chunk k+1 overlapping the H2D copy of
// chunk k.  Validation and messages follow the reference loader.
#include "common.cuh"

#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

namespace r1 {
namespace {

constexpr char kMagic[6] = {'D', 'T', 'E', 'N', '1', '\0'};
constexpr size_t kChunk = size_t(64) << 20;  // bytes per staging buffer

struct File {
    FILE* f = nullptr;
    ~File() {
        if (f) std::fclose(f);
    }
};

bool get_u64le(FILE* f, uint64_t* v) {
    unsigned char b[8];
    if (std::fread(b, 1, 8, f) != 8) return false;
    uint64_t x = 0;
    for (int i = 0; i < 8; ++i) x |= static_cast<uint64_t>(b[i]) << (8 * i);
    *v = x;
    return true;
}

void put_u64le(FILE* f, uint64_t v) {
    unsigned char b[8];
    for (int i = 0; i < 8; ++i) b[i] = static_cast<unsigned char>((v >> (8 * i)) & 0xff);
    std::fwrite(b, 1, 8, f);
}

struct Staging {
    PinnedBuffer buf[2];
    cudaEvent_t ev[2] = {nullptr, nullptr};
    Staging() {
        for (int i = 0; i < 2; ++i) {
            buf[i].ensure(kChunk);
            R1_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
        }
    }
    ~Staging() {
        for (auto e : ev)
            if (e) cudaEventDestroy(e);
    }
};

}  // namespace
}  // namespace r1

using namespace r1;

extern "C" {

int r1_tensor_read_dt1(r1_context* ctx, const char* path, r1_tensor** out) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx || !path || !out) fail(R1_ERR_INVALID_ARGUMENT, "null argument");
        R1_CUDA(cudaSetDevice(ctx->device));
        const std::string p(path);
        File file;
        file.f = std::fopen(path, "rb");
        if (!file.f) fail(R1_ERR_RUNTIME, "read_dt1: cannot open " + p);
        char magic[6];
        if (std::fread(magic, 1, 6, file.f) != 6 || std::memcmp(magic, kMagic, 6) != 0)
            fail(R1_ERR_RUNTIME, "read_dt1: bad magic in " + p);
        unsigned char d = 0;
        if (std::fread(&d, 1, 1, file.f) != 1 || d < 2)
            fail(R1_ERR_RUNTIME, "read_dt1: tensor order must be >= 2");
        std::vector<uint64_t> dims(d);
        uint64_t count = 1;
        for (auto& dim : dims) {
            if (!get_u64le(file.f, &dim) || dim == 0) fail(R1_ERR_RUNTIME, "read_dt1: invalid dimension");
            if (count > ~uint64_t(0) / dim) fail(R1_ERR_RUNTIME, "read_dt1: size overflow");
            count *= dim;
        }
        // the declared shape must account for the file exactly (tensor_io.cpp:86-96)
        const long header = std::ftell(file.f);
        std::fseek(file.f, 0, SEEK_END);
        const long end = std::ftell(file.f);
        std::fseek(file.f, header, SEEK_SET);
        const uint64_t payload = static_cast<uint64_t>(end - header);
        if (count > ~uint64_t(0) / 8 || payload < count * 8)
            fail(R1_ERR_RUNTIME, "read_dt1: truncated payload in " + p);
        if (payload > count * 8) fail(R1_ERR_RUNTIME, "read_dt1: trailing bytes in " + p);
        if (d > 16) fail(R1_ERR_INVALID_ARGUMENT, "read_dt1: order > 16 is not supported on the device");

        r1_tensor* t = nullptr;
        int rc = r1_tensor_create(ctx, dims.data(), d, &t);
        if (rc != R1_OK) fail(rc, r1_last_error());
        try {
            Staging st;
            const uint64_t total = count * 8;
            uint64_t done = 0;
            int k = 0;
            while (done < total) {
                const size_t len = static_cast<size_t>(std::min<uint64_t>(kChunk, total - done));
                R1_CUDA(cudaEventSynchronize(st.ev[k]));  // staging buffer k is free again
                if (std::fread(st.buf[k].ptr, 1, len, file.f) != len)
                    fail(R1_ERR_RUNTIME, "read_dt1: truncated payload in " + p);
                R1_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(t->dev) + done, st.buf[k].ptr, len,
                                        cudaMemcpyHostToDevice, ctx->stream));
                R1_CUDA(cudaEventRecord(st.ev[k], ctx->stream));
                done += len;
                k ^= 1;
            }
            R1_CUDA(cudaStreamSynchronize(ctx->stream));
        } catch (...) {
            r1_tensor_destroy(t);
            throw;
        }
        *out = t;
    });
}

int r1_tensor_write_dt1(r1_context* ctx, const r1_tensor* t, const char* path) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx || !t || !path) fail(R1_ERR_INVALID_ARGUMENT, "null argument");
        R1_CUDA(cudaSetDevice(ctx->device));
        const std::string p(path);
        // tensor_io.cpp:47-50
        if (t->dims.size() < 2) fail(R1_ERR_INVALID_ARGUMENT, "write_dt1: tensor order must be >= 2");
        if (t->dims.size() > 255) fail(R1_ERR_INVALID_ARGUMENT, "write_dt1: tensor order exceeds 255");
        File file;
        file.f = std::fopen(path, "wb");
        if (!file.f) fail(R1_ERR_RUNTIME, "write_dt1: cannot open " + p);
        std::fwrite(kMagic, 1, 6, file.f);
        const unsigned char d = static_cast<unsigned char>(t->dims.size());
        std::fwrite(&d, 1, 1, file.f);
        for (auto v : t->dims) put_u64le(file.f, v);
        Staging st;
        const uint64_t total = t->numel * 8;
        // D2H of chunk k+1 overlaps the disk write of chunk k
        uint64_t issued = 0, written = 0;
        size_t len[2] = {0, 0};
        int k = 0;
        auto issue = [&](int b) {
            len[b] = static_cast<size_t>(std::min<uint64_t>(kChunk, total - issued));
            R1_CUDA(cudaMemcpyAsync(st.buf[b].ptr, reinterpret_cast<const char*>(t->dev) + issued,
                                    len[b], cudaMemcpyDeviceToHost, ctx->stream));
            R1_CUDA(cudaEventRecord(st.ev[b], ctx->stream));
            issued += len[b];
        };
        if (issued < total) issue(0);
        while (written < total) {
            R1_CUDA(cudaEventSynchronize(st.ev[k]));
            if (issued < total) issue(k ^ 1);
            if (std::fwrite(st.buf[k].ptr, 1, len[k], file.f) != len[k])
                fail(R1_ERR_RUNTIME, "write_dt1: write failed for " + p);
            written += len[k];
            k ^= 1;
        }
        if (std::fflush(file.f) != 0) fail(R1_ERR_RUNTIME, "write_dt1: write failed for " + p);
    });
}

}  // extern "C"
