// Multi-GPU sweep exchange over NCCL, behind the C-ABI.
//
// A tensor is split into contiguous slabs along its LAST (slowest) mode; rank
// r holds A[..., lo_r:hi_r] as an ordinary column-major tensor of dims
// (I_0, ..., I_{d-2}, hi_r - lo_r).  Its sweep (sweep_blocks with the slice
// u_{d-1}[lo_r:hi_r] of the global last factor) yields, per pair (m, n):
//   n <  d-1: a PARTIAL block (sum over the slab)        -> all-reduce (sum)
//   n == d-1: the block's complete columns lo_r..hi_r     -> gathered in place
// Block (m, d-1) is column-major I_m x I_{d-1}, so rank r's columns are one
// contiguous run of the global block: equal slabs use ncclAllGather straight
// into the global block, unequal ones one ncclBroadcast per root into its run.
// All of a sweep's collectives are issued in ONE ncclGroupStart/End (NCCL
// fuses the partial-block all-reduces).  NCCL hands every rank the same
// reduced bits, so the replicated eigen step, RQI and stopping test take the
// same branches everywhere (the solver needs no extra agreement step).
//
// NCCL is opened at run time (dlopen "libnccl.so.2"): the library has no link
// dependency, and inside a process that already loaded NCCL (torch) the loaded
// copy is reused.  Communicators: one process per GPU (r1_comm_init with an id
// from r1_comm_unique_id, exchanged by the caller — torch.distributed, MPI, a
// file), or one process for several GPUs (r1_comm_init_all, thread per GPU).
#include "common.cuh"

#include <dlfcn.h>

#include <cstring>
#include <string>
#include <vector>

namespace r1 {

namespace {

// ---- the slice of the NCCL API we use (nccl.h, ABI-stable across 2.x) -------
typedef struct ncclComm* ncclComm_t;
typedef struct {
    char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;  // ncclSuccess == 0
constexpr int kNcclDouble = 8;   // ncclFloat64
constexpr int kNcclSum = 0;      // ncclSum

struct Nccl {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GetVersion)(int*) = nullptr;
};

Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            n.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (n.h) break;
        }
        if (!n.h) {
            err = std::string("NCCL not found (dlopen libnccl.so.2): ") + dlerror();
            return;
        }
        auto sym = [&](auto& fp, const char* s) {
            fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(n.h, s));
            if (!fp && err.empty()) err = std::string("NCCL symbol missing: ") + s;
        };
        sym(n.GetUniqueId, "ncclGetUniqueId");
        sym(n.CommInitRank, "ncclCommInitRank");
        sym(n.CommInitAll, "ncclCommInitAll");
        sym(n.CommDestroy, "ncclCommDestroy");
        sym(n.AllReduce, "ncclAllReduce");
        sym(n.AllGather, "ncclAllGather");
        sym(n.Broadcast, "ncclBroadcast");
        sym(n.GroupStart, "ncclGroupStart");
        sym(n.GroupEnd, "ncclGroupEnd");
        sym(n.GetErrorString, "ncclGetErrorString");
        sym(n.GetVersion, "ncclGetVersion");
    });
    if (!err.empty()) fail(R1_ERR_RUNTIME, err);
    return n;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != 0) {
        const char* m = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
        fail(R1_ERR_CUDA, std::string("NCCL error in ") + what + ": " + m);
    }
}

}  // namespace

// [lo, hi) of rank's slab of `extent`: sizes differ by at most one, larger first
// (paper_2403_01778_b200/distributed.py slab_bounds).
void slab_bounds(uint64_t extent, int world, int rank, uint64_t* lo, uint64_t* hi) {
    const uint64_t base = extent / world, rem = extent % world;
    *lo = rank * base + std::min<uint64_t>(rank, rem);
    *hi = *lo + base + (static_cast<uint64_t>(rank) < rem ? 1 : 0);
}

// One entry per block pair: where the rank's local block sits, where the
// global block sits, and how it is combined.
void exchange_plan(const uint64_t* gdims, int order, int world, int rank, std::vector<ExchangeOp>& ops) {
    ops.clear();
    uint64_t lo, hi;
    slab_bounds(gdims[order - 1], world, rank, &lo, &hi);
    uint64_t loff = 0, goff = 0;
    for (int m = 0; m < order; ++m)
        for (int n = m + 1; n < order; ++n) {
            ExchangeOp op{};
            op.m = m;
            op.n = n;
            op.local_off = loff;
            op.global_off = goff;
            op.rows = gdims[m];
            const bool gathered = n == order - 1;
            op.gathered = gathered ? 1 : 0;
            op.local_count = gdims[m] * (gathered ? (hi - lo) : gdims[n]);
            ops.push_back(op);
            loff += op.local_count;
            goff += gdims[m] * gdims[n];
        }
}

// Assemble the global blocks (gblocks) from this rank's local slab blocks.
void exchange_blocks(r1_context* ctx, const double* lblocks, double* gblocks,
                     const uint64_t* gdims, int order) {
    r1_comm* c = ctx->comm;
    if (!c) fail(R1_ERR_INVALID_ARGUMENT, "exchange: no communicator attached");
    const int world = c->world, rank = c->rank;
    std::vector<ExchangeOp> ops;
    exchange_plan(gdims, order, world, rank, ops);
    const uint64_t extent = gdims[order - 1];
    const bool even = extent % world == 0;
    Nccl& N = nccl();
    ncclComm_t comm = static_cast<ncclComm_t>(c->comm);
    nccl_check(N.GroupStart(), "ncclGroupStart");
    for (const ExchangeOp& op : ops) {
        if (!op.gathered) {
            nccl_check(N.AllReduce(lblocks + op.local_off, gblocks + op.global_off, op.local_count,
                                   kNcclDouble, kNcclSum, comm, ctx->stream),
                       "ncclAllReduce");
        } else if (even) {
            nccl_check(N.AllGather(lblocks + op.local_off, gblocks + op.global_off, op.local_count,
                                   kNcclDouble, comm, ctx->stream),
                       "ncclAllGather");
        } else {
            for (int r = 0; r < world; ++r) {
                uint64_t rlo, rhi;
                slab_bounds(extent, world, r, &rlo, &rhi);
                if (rhi == rlo) continue;
                double* dst = gblocks + op.global_off + op.rows * rlo;
                const double* src = r == rank ? lblocks + op.local_off : dst;
                nccl_check(N.Broadcast(src, dst, op.rows * (rhi - rlo), kNcclDouble, r, comm,
                                       ctx->stream),
                           "ncclBroadcast");
            }
        }
    }
    nccl_check(N.GroupEnd(), "ncclGroupEnd");
    count_launch(ctx);
}

void comm_destroy(r1_comm* c) {
    if (!c) return;
    if (c->ctx && c->ctx->comm == c) c->ctx->comm = nullptr;
    if (c->comm && c->owns) nccl().CommDestroy(static_cast<ncclComm_t>(c->comm));
    delete c;
}

}  // namespace r1

using namespace r1;

extern "C" {

int r1_comm_unique_id(void* id_out) {
    return abi_guard([&] {
        if (!id_out) fail(R1_ERR_INVALID_ARGUMENT, "null argument");
        ncclUniqueId id;
        nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(id_out, &id, sizeof(id));
    });
}

int r1_comm_init(r1_context* ctx, int nranks, int rank, const void* id, r1_comm** out) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx || !id || !out) fail(R1_ERR_INVALID_ARGUMENT, "null argument");
        if (nranks < 1 || rank < 0 || rank >= nranks)
            fail(R1_ERR_INVALID_ARGUMENT, "r1_comm_init: bad rank / world size");
        R1_CUDA(cudaSetDevice(ctx->device));
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof(uid));
        auto* c = new r1_comm();
        c->world = nranks;
        c->rank = rank;
        c->owns = true;
        ncclResult_t r = nccl().CommInitRank(reinterpret_cast<ncclComm_t*>(&c->comm), nranks, uid, rank);
        if (r != 0) {
            delete c;
            nccl_check(r, "ncclCommInitRank");
        }
        c->ctx = ctx;
        ctx->comm = c;
        *out = c;
    });
}

int r1_comm_init_all(int ndev, const int* devices, r1_context** ctxs, r1_comm** comms) {
    return abi_guard([&] {
        if (ndev < 1 || !devices || !ctxs || !comms) fail(R1_ERR_INVALID_ARGUMENT, "null argument");
        std::vector<ncclComm_t> cs(ndev);
        nccl_check(nccl().CommInitAll(cs.data(), ndev, devices), "ncclCommInitAll");
        for (int i = 0; i < ndev; ++i) {
            if (!ctxs[i] || ctxs[i]->device != devices[i])
                fail(R1_ERR_INVALID_ARGUMENT, "r1_comm_init_all: context i must be on devices[i]");
            auto* c = new r1_comm();
            c->world = ndev;
            c->rank = i;
            c->owns = true;
            c->comm = reinterpret_cast<void*>(cs[i]);
            c->ctx = ctxs[i];
            ctxs[i]->comm = c;
            comms[i] = c;
        }
    });
}

int r1_comm_destroy(r1_comm* c) {
    return abi_guard([&] { comm_destroy(c); });
}

int r1_comm_info(const r1_comm* c, int* world, int* rank) {
    return abi_guard([&] {
        if (!c) fail(R1_ERR_INVALID_ARGUMENT, "null communicator");
        if (world) *world = c->world;
        if (rank) *rank = c->rank;
    });
}

int r1_slab_bounds(uint64_t extent, int world, int rank, uint64_t* lo, uint64_t* hi) {
    return abi_guard([&] {
        if (world < 1 || rank < 0 || rank >= world || !lo || !hi)
            fail(R1_ERR_INVALID_ARGUMENT, "r1_slab_bounds: bad arguments");
        slab_bounds(extent, world, rank, lo, hi);
    });
}

// Diagnostics / tests (not in the public header): this rank's exchange plan,
// 6 int64 per pair: m, n, local_off, global_off, local_count, gathered.
int r1x_exchange_plan(const uint64_t* gdims, int order, int world, int rank, int64_t* out, int cap) {
    return abi_guard([&] {
        std::vector<ExchangeOp> ops;
        exchange_plan(gdims, order, world, rank, ops);
        if (static_cast<int>(ops.size()) > cap) fail(R1_ERR_INVALID_ARGUMENT, "plan buffer too small");
        for (size_t i = 0; i < ops.size(); ++i) {
            int64_t* o = out + 6 * i;
            o[0] = ops[i].m;
            o[1] = ops[i].n;
            o[2] = static_cast<int64_t>(ops[i].local_off);
            o[3] = static_cast<int64_t>(ops[i].global_off);
            o[4] = static_cast<int64_t>(ops[i].local_count);
            o[5] = ops[i].gathered;
        }
    });
}

}  // extern "C"
