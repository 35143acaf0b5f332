// The fused TTVc sweep: every NEPv block B(m,n) = A x_{k not in {m,n}} u_k of
// J(u) from ONE streaming pass over the tensor per recursion level.
//
// Replaces rank1::build_j (reference proj/src/nepv.cpp:199-231), which builds
// each of the P = d(d-1)/2 blocks by its own TTV chain over the whole tensor
// (contract_to_block, nepv.cpp:46-77; ttv, tensor.cpp:100-138), i.e. P full
// passes over A.
//
// Design:
//   View A (column-major, first index fastest) as A[i0, i1, o] with o the
//   linear index of modes 2..d-1 and outer weight W[o] = prod_{k>=2} u_k[i_k].
//   One pass over A produces
//     B01[i0,i1] = sum_o A[i0,i1,o] W[o]          (= block (0,1))
//     C0[i0,o]   = sum_i1 A[i0,i1,o] u1[i1]       (= A x_1 u1, order d-1)
//     C1[i1,o]   = sum_i0 A[i0,i1,o] u0[i0]       (= A x_0 u0, order d-1)
//   For d = 3 these ARE blocks (0,1), (0,2), (1,2).  For d >= 4 the remaining
//   blocks are the blocks of C0 (modes 0,2,..) and the (0,k) blocks of C1
//   (modes 1,2,..) — the same problem one order lower on tensors I1x (resp.
//   I0x) smaller, handled by recursion (the reference's reuse_intermediates
//   idea, nepv.cpp:174-195, applied to the fused pass).
//
// Kernels: sweep3_box_kernel — persistent, one CTA per SM, one
// producer warp streaming (tile, o) panels HBM -> shared memory with 3-D TMA
// tensor-map loads (cp.async.bulk.tensor, L2 evict_first) into a byte-budgeted
// mbarrier ring, 7-11 consumer warps (32 elements per thread: 128 x 56,
// 256 x 44 or 64 x 64 tiles; the 15-warp / 16-element shapes stay selectable
// in the development build) keeping the B01 face tile in registers,
// reducing C1 with a transposing warp butterfly and C0 through shared memory;
// tiles are cut in whole 128-B lines (alignment classes), small faces put KO
// o-panels in one box, the last 25% of the panels are scheduled dynamically
// from a work counter the kernel re-arms itself.  The recursion's independent
// subtrees run on two streams (sweep_blocks).
// sweep3_kernel — the 1-D cp.async.bulk variant for odd I0 (no 16-B TMA
// stride).  C0/C1/B01 partials over tiles / segments go to a workspace and are
// summed in a fixed order by finish_kernel: no atomics anywhere, so results are
// bit-reproducible run to run.
#include "common.cuh"

#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

namespace r1 {

namespace {

constexpr int kNWC = 8;                    // consumer warps
constexpr int kThreads = (kNWC + 1) * 32;  // + one producer warp
constexpr int kMaxOrder = 16;
constexpr int kBoxNWC = 15;  // consumer warps of the 16-element box shapes (+1 producer = 16 warps)
constexpr int kBoxNCB = 4;   // their columns per consumer warp (box = 32*NRA x 60)
// sub-strips per tile of the 128 x 56 shape, accumulators in tensor memory
// (R1_SWEEP_NS in the development build).  Built, bit-correct and measured
// SLOWER (same box, C5 5.59 vs 5.17 ms, C2 1.43 vs 1.31 ms with 3 sub-strips):
// every box moves its 57 KB of accumulators out of and back into tensor
// memory, and tcgen05.ld reads 64 B per clock and SM — a third of the box
// period — so the 0.77 GB less partial-sum traffic (C5) does not pay.  Off.
constexpr int kSubStripsDefault = 1;
constexpr int kWideDefault = 13;  // wide consumer shapes for all three row-tile heights (tile_level)
constexpr int kMaxStages = 16;          // mbarrier slots of the box kernel ring
constexpr double kDynFrac = 0.25;       // share of the work scheduled dynamically
constexpr double kDynMinChunk = 8.0;    // guided chunks: remaining/(2*ncta), >= 8 panels
constexpr size_t kSmemBudget = 227 * 1024;  // opt-in dynamic shared memory per CTA

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

struct Seg {
    int tile;
    int o0;
    int o1;
    int pad;
};

struct SweepArgs {
    const double* A;
    int64_t I0, I1, O;
    // box kernel: merged-column view (alignment classes, see tile_level):
    // M[r, c, o] = A[r mod I0, K c + r / I0, o], MI0 = K I0 rows, MI1 = I1 / K
    int K;
    int64_t MI0, MI1;
    const double* u0;
    const double* u1;
    const double* W;
    int r0, t1, G0;
    int ts;                 // box kernel: columns per box (sub-strip of a tile; = t1 without sub-strips)
    int rbox;               // TMA path: box rows (= r0, even); smem column stride
    const Seg* segs;
    const int* cta_seg;
    double* P01;            // [nseg][t1][r0]
    double* P0;             // [G1] copies of I0 x O, stride P0_stride
    int64_t P0_stride;
    double* P1;             // [G0] copies of I1 x O, stride P1_stride (nullptr: skip)
    int64_t P1_stride;
    unsigned long long* trace;  // optional: per CTA {t_start, t_end, smid}
    int debug_mode;             // diagnostics: 1 = consumers only wait/release
    int trace_level0;           // host-side flag: this launch is the top-level sweep
    int dyn_first, ndyn;        // dynamic tail: segments [dyn_first, dyn_first + ndyn)
    int* dyn_counter;           // work counter of the dynamic tail (zeroed per launch)
};

// ------------------------------------------------------------- PTX helpers --
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_addr(bar);
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    } while (!done);
}

// Programmatic dependent launch: every sweep kernel lets its successor in the
// stream be scheduled at once and waits for its predecessor (completion and
// memory flush) before touching global memory, so launch latency and the
// prologue (smem zeroing, barrier init, tensor-map prefetch) leave the chain.
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Tensor memory as accumulator storage (box kernel with sub-strips): a warp
// reads / writes 8 doubles (16 32-bit columns) of each of its 32 lanes.
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
        "%13, %14, %15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15])
        : "r"(taddr)
        : "memory");
}
// completes the loads; the registers pass through it so no use moves above it
__device__ __forceinline__ void tmem_wait_ld(uint32_t (&r)[16]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]),
                   "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]),
                   "+r"(r[14]), "+r"(r[15])
                 :
                 : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
        "%13, %14, %15, %16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
// NE doubles of this thread's lane at column taddr.. (NE % 8 == 0)
template <int NE>
__device__ __forceinline__ void tmem_issue_load(uint32_t taddr, uint32_t (&r)[NE / 8][16]) {
#pragma unroll
    for (int c = 0; c < NE / 8; ++c) tmem_ld8(taddr + 16 * c, r[c]);
}
template <int NE>
__device__ __forceinline__ void tmem_complete_load(uint32_t (&r)[NE / 8][16], double* d) {
#pragma unroll
    for (int c = 0; c < NE / 8; ++c) tmem_wait_ld(r[c]);
#pragma unroll
    for (int c = 0; c < NE / 8; ++c)
#pragma unroll
        for (int e = 0; e < 8; ++e) d[8 * c + e] = __hiloint2double(static_cast<int>(r[c][2 * e + 1]), static_cast<int>(r[c][2 * e]));
}
template <int NE>
__device__ __forceinline__ void tmem_load_doubles(uint32_t taddr, double* d) {
    uint32_t r[NE / 8][16];
    tmem_issue_load<NE>(taddr, r);
    tmem_complete_load<NE>(r, d);
}
template <int NE>
__device__ __forceinline__ void tmem_store_doubles(uint32_t taddr, const double* d) {
#pragma unroll
    for (int c = 0; c < NE / 8; ++c) {
        uint32_t r[16];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            r[2 * e] = static_cast<uint32_t>(__double2loint(d[8 * c + e]));
            r[2 * e + 1] = static_cast<uint32_t>(__double2hiint(d[8 * c + e]));
        }
        tmem_st8(taddr + 16 * c, r);
    }
}

__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// 1-D bulk copy (any 16-B aligned run), completion on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
        : "memory");
}

// 3-D TMA tile load of box (rbox, t1, 1) at (c0, c1, c2); out-of-range
// elements are zero-filled by the hardware.
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        ".L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_addr(bar)),
        "l"(pol)
        : "memory");
}

__device__ __forceinline__ void consumer_bar() {
    asm volatile("bar.sync 1, %0;" ::"n"(kNWC * 32) : "memory");
}

// After the call lane L holds the 32-lane sum of v[col], col = *col_out, for
// NV = 2^L values per lane: L halving levels (offsets 16, 8, ...) exchange
// half the values each, the remaining offsets reduce the single survivor.
template <int NV>
__device__ __forceinline__ double warp_transpose_sum(double (&v)[NV], int lane, int* col_out) {
    int col = 0;
    int off = 16;
#pragma unroll
    for (int half = NV / 2; half >= 1; half >>= 1) {
        const bool upper = (lane & off) != 0;
#pragma unroll
        for (int q = 0; q < half; ++q) {
            const double send = upper ? v[q] : v[q + half];
            const double keep = upper ? v[q + half] : v[q];
            v[q] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
        if (upper) col += half;
        off >>= 1;
    }
    double r = v[0];
#pragma unroll
    for (; off >= 1; off >>= 1) r += __shfl_xor_sync(0xffffffffu, r, off);
    *col_out = col;
    return r;
}

// --------------------------------------------------------------- the sweep --
// TMA = true : one cp.async.bulk.tensor.3d per panel (I0 even: 16-B strides).
// TMA = false: one 1-D bulk copy per column run, 16-B aligned superset, the
//              consumer skips the (st & 1) leading element (any I0).
template <int NRA, int NCB, int STAGES, bool TMA>
__global__ void __launch_bounds__(kThreads, 1)
    sweep3_kernel(const SweepArgs p, const __grid_constant__ CUtensorMap tmap) {
    constexpr int RMAX = 32 * NRA;
    constexpr int CS = TMA ? RMAX : RMAX + 2;  // doubles per smem column
    constexpr int STAGE_DBL = kNWC * NCB * CS;
    extern __shared__ __align__(1024) double smem[];
    double* ring = smem;
    double* red = smem + STAGES * STAGE_DBL;  // [2][kNWC][RMAX]
    uint64_t* full = reinterpret_cast<uint64_t*>(red + 2 * kNWC * RMAX);
    uint64_t* empty = full + STAGES;

    pdl_launch_dependents();
    pdl_wait();
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kNWC);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const int seg_begin = p.cta_seg[blockIdx.x];
    const int seg_end = p.cta_seg[blockIdx.x + 1];
    const int64_t I0 = p.I0, I1 = p.I1;
    const int cstride = TMA ? p.rbox : CS;

    if (warp == kNWC) {
        // ---------------- producer: panels HBM -> smem ring ----------------
        const uint64_t pol = policy_evict_first();
        int stage = 0;
        uint32_t phase = 0;
        if (TMA) {
            if (lane == 0) {
                asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap))
                             : "memory");
                const uint32_t box_bytes = static_cast<uint32_t>(p.rbox) * p.t1 * 8;
                for (int s = seg_begin; s < seg_end; ++s) {
                    const Seg sg = p.segs[s];
                    const int g0 = sg.tile % p.G0, g1 = sg.tile / p.G0;
                    for (int o = sg.o0; o < sg.o1; ++o) {
                        mbar_wait(&empty[stage], phase ^ 1);
                        mbar_arrive_expect_tx(&full[stage], box_bytes);
                        tma_load_3d(ring + stage * STAGE_DBL, &tmap, g0 * p.r0, g1 * p.t1, o,
                                    &full[stage], pol);
                        if (++stage == STAGES) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                }
            }
            return;
        }
        for (int s = seg_begin; s < seg_end; ++s) {
            const Seg sg = p.segs[s];
            const int g0 = sg.tile % p.G0, g1 = sg.tile / p.G0;
            const int64_t R0s = static_cast<int64_t>(g0) * p.r0;
            const int64_t R1s = static_cast<int64_t>(g1) * p.t1;
            const int r0e = static_cast<int>(min64(p.r0, I0 - R0s));
            const int t1e = static_cast<int>(min64(p.t1, I1 - R1s));
            for (int o = sg.o0; o < sg.o1; ++o) {
                mbar_wait(&empty[stage], phase ^ 1);
                double* dst = ring + stage * STAGE_DBL;
                uint32_t bytes = 0;
                for (int j = lane; j < t1e; j += 32) {
                    const int64_t st = R0s + I0 * (R1s + j + I1 * static_cast<int64_t>(o));
                    const int64_t as = st & ~int64_t(1), ae = (st + r0e + 1) & ~int64_t(1);
                    bytes += static_cast<uint32_t>((ae - as) * 8);
                }
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1)
                    bytes += __shfl_xor_sync(0xffffffffu, bytes, off);
                if (lane == 0) mbar_arrive_expect_tx(&full[stage], bytes);
                __syncwarp();
                for (int j = lane; j < t1e; j += 32) {
                    const int64_t st = R0s + I0 * (R1s + j + I1 * static_cast<int64_t>(o));
                    const int64_t as = st & ~int64_t(1), ae = (st + r0e + 1) & ~int64_t(1);
                    bulk_g2s(dst + j * CS, p.A + as, static_cast<uint32_t>((ae - as) * 8),
                             &full[stage], pol);
                }
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
        return;
    }

    // -------------------- consumers: 8 warps, lanes along i0 -------------
    int stage = 0;
    uint32_t phase = 0;
    int rbuf = 0;
    for (int s = seg_begin; s < seg_end; ++s) {
        const Seg sg = p.segs[s];
        const int g0 = sg.tile % p.G0, g1 = sg.tile / p.G0;
        const int64_t R0s = static_cast<int64_t>(g0) * p.r0;
        const int64_t R1s = static_cast<int64_t>(g1) * p.t1;
        const int r0e = static_cast<int>(min64(p.r0, I0 - R0s));
        const int t1e = static_cast<int>(min64(p.t1, I1 - R1s));

        double u0r[NRA], u1c[NCB];
        double acc[NRA][NCB];
        bool rv[NRA], cv[NCB];
#pragma unroll
        for (int a = 0; a < NRA; ++a) {
            const int i = lane + 32 * a;
            rv[a] = i < r0e;
            u0r[a] = rv[a] ? __ldg(p.u0 + R0s + i) : 0.0;
        }
#pragma unroll
        for (int b = 0; b < NCB; ++b) {
            const int j = warp + kNWC * b;
            cv[b] = j < t1e;
            u1c[b] = cv[b] ? __ldg(p.u1 + R1s + j) : 0.0;
#pragma unroll
            for (int a = 0; a < NRA; ++a) acc[a][b] = 0.0;
        }
        double* P0row = p.P0 + static_cast<int64_t>(g1) * p.P0_stride + R0s;
        double* P1row = p.P1 ? p.P1 + static_cast<int64_t>(g0) * p.P1_stride + R1s : nullptr;

        for (int o = sg.o0; o < sg.o1; ++o) {
            const double wo = __ldg(p.W + o);
            mbar_wait(&full[stage], phase);
            const double* st = ring + stage * STAGE_DBL;
            const int64_t colbase = R0s + I0 * (R1s + I1 * static_cast<int64_t>(o));
            double c0p[NRA];
            double c1v[NCB];
#pragma unroll
            for (int a = 0; a < NRA; ++a) c0p[a] = 0.0;
#pragma unroll
            for (int b = 0; b < NCB; ++b) {
                const int j = warp + kNWC * b;
                double c1p = 0.0;
                if (cv[b]) {
                    const double* col =
                        st + j * cstride + (TMA ? 0 : static_cast<int>((colbase + I0 * j) & 1));
#pragma unroll
                    for (int a = 0; a < NRA; ++a) {
                        if (rv[a]) {
                            const double v = col[lane + 32 * a];
                            acc[a][b] = fma(v, wo, acc[a][b]);
                            c1p = fma(v, u0r[a], c1p);
                            c0p[a] = fma(v, u1c[b], c0p[a]);
                        }
                    }
                }
                c1v[b] = c1p;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stage]);
            if (++stage == STAGES) {
                stage = 0;
                phase ^= 1;
            }

            // C1 partial: full column dots over this tile's rows.
            int col;
            const double c1 = warp_transpose_sum<NCB>(c1v, lane, &col);
            if (P1row && (lane & (32 / NCB - 1)) == 0) {
                const int j = warp + kNWC * col;
                if (j < t1e) P1row[static_cast<int64_t>(o) * I1 + j] = c1;
            }

            // C0 partial: row sums over this tile's columns, across warps.
            double* rb = red + rbuf * kNWC * RMAX;
#pragma unroll
            for (int a = 0; a < NRA; ++a) rb[warp * RMAX + lane + 32 * a] = c0p[a];
            consumer_bar();
            for (int i = threadIdx.x; i < r0e; i += kNWC * 32) {
                double sum = 0.0;
#pragma unroll
                for (int w = 0; w < kNWC; ++w) sum += rb[w * RMAX + i];
                P0row[static_cast<int64_t>(o) * I0 + i] = sum;
            }
            rbuf ^= 1;
        }

        // Flush the B01 face partial of this segment.
        double* dst = p.P01 + static_cast<int64_t>(s) * p.r0 * p.t1;
#pragma unroll
        for (int b = 0; b < NCB; ++b) {
            const int j = warp + kNWC * b;
            if (!cv[b]) continue;
#pragma unroll
            for (int a = 0; a < NRA; ++a) {
                const int i = lane + 32 * a;
                if (rv[a]) dst[j * p.r0 + i] = acc[a][b];
            }
        }
    }
}

// TMA path with fixed RMAX x CMAX tiles.  Interior tiles load one full box;
// the ragged last row / column tiles use their own tensor maps whose box is
// exactly the remainder (boxes straddling the tensor edge take the slow
// out-of-bounds path in the TMA unit).  The smem column stride is the box's
// row count; rows beyond it read finite neighbours (the ring is zeroed once)
// whose contributions carry zero weights and are never stored.  Lane l owns
// rows 64p + 2l + {0,1} (one 128-bit LDS per pair p), warp w owns columns
// w + NWC*b: the inner loop is branch-free.
struct BoxMaps {
    CUtensorMap m[4];  // [row-edge bit | col-edge bit << 1]: boxes r0|rem0 x t1|rem1
};

// TMA path.  Tiles are balanced (r0 = ceil(I0/G0) rounded to even, t1 =
// ceil(I1/G1)), so every box is within a few rows/columns of the others; the
// ragged last row/column tiles use their own tensor maps (a box straddling the
// tensor edge takes the slow out-of-bounds path in the TMA unit).  The smem
// ring is budgeted in BYTES: nst = ring_bytes / box_bytes stages, so every SM
// keeps the same volume in flight — in a saturated memory system an SM's share
// of bandwidth follows its bytes in flight.  The consumer thread grid is fixed
// (RMAX x CMAX); rows/columns beyond the tile read finite neighbours (the ring
// is zeroed once) and carry zero weights, and are never stored.  Tiles live in
// the merged-column view (alignment classes, tile_level): lane l owns the NRA
// consecutive merged rows NRA*l.. (NRA/2 128-bit LDS), all in one class, warp
// w owns columns w + NWC*b.  Each thread copies its slice to registers and
// releases the stage before computing.
// KO > 1 (small faces): one box holds KO consecutive o-panels of the tile, so
// the per-panel fixed work (barrier waits, the C0 block reduction, the C1
// warp reduction) is paid once per KO panels; segments count o-groups.
// NS > 1 (sub-strips, round 2): a tile is NS column sub-strips of ts <= NWC * NCB
// columns, one TMA box each per o; the B01 accumulators of all sub-strips live
// in TENSOR MEMORY (256 KB per SM, idle otherwise: tcgen05.ld / .st, 32 doubles
// per thread and sub-strip), loaded before and stored after each box, so a
// tile is up to NS x larger than the register file allows and the face has NS
// x fewer column tiles, i.e. C0 partial sets; the C0 row sums of an o are
// carried in registers over its sub-strips and reduced once.
template <int NRA, int NCB, int NWC, bool STAGE_REGS, int KO, int NS = 1>
__global__ void __launch_bounds__((NWC + 1) * 32, 1)
    sweep3_box_kernel(const SweepArgs p, const __grid_constant__ BoxMaps maps, int nst,
                      int stage_dbl) {
    static_assert(KO * NCB <= 32, "C1 reduction holds KO * NCB values per lane");
    static_assert(NS == 1 || (KO == 1 && NWC <= 8 && NS * 4 * NRA * NCB <= 512 && (NRA * NCB) % 8 == 0),
                  "sub-strips: two warps per TMEM lane quadrant, 512 columns");
    static_assert(NRA % 2 == 0 && NRA <= 8, "rows are read in pairs, at most 4 pairs per lane");
    constexpr int RMAX = 32 * NRA;
    constexpr int NP = NRA / 2;
    extern __shared__ __align__(1024) double smem[];
    double* ring = smem;
    const int ring_dbl = nst * stage_dbl + RMAX;  // + slack for over-reads
    double* red = smem + ring_dbl;                // [2][KO][NWC][RMAX]
    uint64_t* full = reinterpret_cast<uint64_t*>(red + 2 * KO * NWC * RMAX);
    uint64_t* empty = full + kMaxStages;
    int4* meta = reinterpret_cast<int4*>(empty + kMaxStages);  // per stage {seg, tile, o, flags}
    uint64_t* red_full = reinterpret_cast<uint64_t*>(meta + kMaxStages);  // [2] C0 partial slots
    uint64_t* red_empty = red_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(red_empty + 2);  // tensor-memory base (NS > 1)

    pdl_launch_dependents();
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    // A lane's NRA rows are NP 16-B pairs at byte offset 16*NP*lane.  NP = 2:
    // lanes l and l+4 of a quarter warp would hit the same banks, so odd
    // quarter-lanes take their pairs in swapped order (pair slot q holds pair
    // q ^ hsw); NP = 4: lanes l, l+2, l+4, l+6 collide, hsw = (l >> 1) & 3.
    const int hsw = NP == 4 ? (lane >> 1) & 3 : (NP > 1 ? (lane >> 2) & 1 : 0);
    for (int i = threadIdx.x; i < ring_dbl / 2; i += blockDim.x)
        reinterpret_cast<double2*>(ring)[i] = make_double2(0.0, 0.0);
    if (threadIdx.x == 0) {
        for (int s = 0; s < nst; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NWC);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&red_full[s], NWC);
            mbar_init(&red_empty[s], NWC);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if constexpr (NS > 1) {
        if (warp == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                             smem_addr(tmem_slot))
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    }
    __syncthreads();
    if constexpr (NS > 1) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // this thread's accumulator columns: lane quadrant warp % 4, region (warp / 4, sub-strip)
    const uint32_t tmem_base = NS > 1 ? *tmem_slot : 0u;
    const uint32_t tmem_acc = NS > 1 ? tmem_base + ((static_cast<uint32_t>(warp & 3) * 32u) << 16) +
                                           static_cast<uint32_t>(warp >> 2) * (NS * 2 * NRA * NCB)
                                     : 0u;
    pdl_wait();

    const int seg_begin = p.cta_seg[blockIdx.x];
    const int seg_end = p.cta_seg[blockIdx.x + 1];
    const int64_t I0 = p.I0, I1 = p.I1;      // real extents
    const int64_t MI0 = p.MI0, MI1 = p.MI1;  // merged view (tiles live here)
    const int K = p.K;
    const int G1 = static_cast<int>((MI1 + p.t1 - 1) / p.t1);
    const int rem0 = static_cast<int>(MI0 - static_cast<int64_t>(p.G0 - 1) * p.r0);
    const int rem1 = static_cast<int>(MI1 - static_cast<int64_t>(G1 - 1) * p.t1);
    // boxes are ts columns wide (ts = t1 without sub-strips); only the last box
    // of the last column tile is narrower (remlast)
    const int remlast = rem1 - ((rem1 + p.ts - 1) / p.ts - 1) * p.ts;

    // Schedule (producer-driven): the static segments [seg_begin, seg_end) of
    // this CTA, then chunks of the dynamic tail taken from a work counter by
    // whichever CTA is free.  Every segment has its own B01 partial slot, so
    // the fixed-order reduction stays bit-reproducible for any schedule.
    // Per stage the producer publishes {segment, tile, o, flags} before its
    // arrive (release); consumers read it after the full-barrier wait.
    constexpr int kFirst = 1, kLast = 2, kDone = 4;
    if (warp == NWC) {
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            for (int m = 0; m < 4; ++m)
                asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.m[m]))
                             : "memory");
            int stage = 0;
            uint32_t phase = 0;
            auto run_segment = [&](int s) {
                const Seg sg = p.segs[s];
                const int g0 = sg.tile % p.G0, g1 = sg.tile / p.G0;
                const bool er = g0 == p.G0 - 1, ec = g1 == G1 - 1;
                const int nsub = ((ec ? rem1 : p.t1) + p.ts - 1) / p.ts;  // boxes per o
                for (int o = sg.o0; o < sg.o1; ++o) {
                    for (int sb = 0; sb < nsub; ++sb) {
                        const bool ecs = ec && sb == nsub - 1;
                        const uint32_t bytes = static_cast<uint32_t>(er ? rem0 : p.r0) *
                                               static_cast<uint32_t>(ecs ? remlast : p.ts) * 8u * KO;
                        const CUtensorMap* map = &maps.m[(er ? 1 : 0) | (ecs ? 2 : 0)];
                        mbar_wait(&empty[stage], phase ^ 1);
                        meta[stage] = make_int4(s, sg.tile, o,
                                                (o == sg.o0 && sb == 0 ? kFirst : 0) |
                                                    (o == sg.o1 - 1 && sb == nsub - 1 ? kLast : 0) | (sb << 8));
                        mbar_arrive_expect_tx(&full[stage], bytes);
                        tma_load_3d(ring + stage * stage_dbl, map, g0 * p.r0, g1 * p.t1 + sb * p.ts, o * KO,
                                    &full[stage], pol);
                        if (++stage == nst) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                }
            };
            for (int s = seg_begin; s < seg_end; ++s) run_segment(s);
            if (p.ndyn > 0) {
                for (;;) {
                    const int c = atomicAdd(p.dyn_counter, 1);
                    if (c >= p.ndyn) {
                        // every CTA ends with exactly one failing fetch: the one
                        // that draws the last ticket re-arms the counter for
                        // the next sweep (no memset node per sweep)
                        if (c == p.ndyn + static_cast<int>(gridDim.x) - 1) *p.dyn_counter = 0;
                        break;
                    }
                    run_segment(p.dyn_first + c);
                }
            }
            mbar_wait(&empty[stage], phase ^ 1);
            meta[stage] = make_int4(-1, 0, 0, kDone);
            mbar_arrive(&full[stage]);
        }
        return;
    }

    unsigned long long t_start = 0;
    if (p.trace && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    int stage = 0;
    uint32_t phase = 0;
    int rbuf = 0;
    int s = -1;
    int g0 = 0, g1 = 0, r0e = 0, t1e = 0, cst = 0;
    int pcls = 0, cls_lo = 0, cls_hi = 0;  // alignment class of this thread's rows / the tile's
    int64_t R0s = 0, R1s = 0;
    double u0r[NRA], u1c[NCB];
    double acc[NRA][NCB];
    double c0p[NRA];  // C0 row sums of the current o (carried over its sub-strips)
    int coff[NCB];  // smem offset (double2 units) of the thread's columns
    bool live = false;
    int nsub = 1;
    int last_w = -1;
    double* P0row = nullptr;
    double* P1row = nullptr;
    // KO == 1: the C0 block reduction of panel q (partials in red slot q & 1)
    // is summed one panel later, after the warp has written panel q + 1's
    // partials — an mbarrier pair per slot instead of a CTA barrier per panel,
    // so no warp waits for the slowest one at every panel and the sums overlap
    // the next panel's loads (C3 200^4: the barrier-synchronous reduction cost
    // 18% of the level-0 kernel)
    int pc = 0;                 // panels consumed by this CTA
    double* pend_dst = nullptr;  // C0 row of panel pc - 1
    int pend_r0e = 0;
    auto reduce_pending = [&]() {
        const int q = pc - 1, slot = q & 1;
        if (warp * 32 < pend_r0e) {
            mbar_wait(&red_full[slot], (q >> 1) & 1);
#pragma unroll
            for (int i = threadIdx.x; i < RMAX; i += NWC * 32) {
                if (i < pend_r0e) {
                    const double* rr = red + slot * NWC * RMAX + i;
                    double sum = 0.0;
#pragma unroll
                    for (int w = 0; w < NWC; ++w) sum += rr[w * RMAX];
                    pend_dst[i] = sum;
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&red_empty[slot]);
    };
    for (;;) {
        mbar_wait(&full[stage], phase);
        const int4 md = meta[stage];
        if (md.w & kDone) break;
        const int o = md.z;
        if (md.w & kFirst) {
            s = md.x;
            const int tile = md.y;
            g0 = tile % p.G0;
            g1 = tile / p.G0;
            R0s = static_cast<int64_t>(g0) * p.r0;
            R1s = static_cast<int64_t>(g1) * p.t1;
            r0e = static_cast<int>(min64(p.r0, MI0 - R0s));
            t1e = static_cast<int>(min64(p.t1, MI1 - R1s));
            cst = r0e;  // smem column stride (doubles) = box rows
            // lane owns NRA consecutive merged rows; I0 % NRA == 0 keeps them in
            // one alignment class (one real column per merged column)
            cls_lo = static_cast<int>(R0s / I0);
            cls_hi = static_cast<int>((R0s + r0e - 1) / I0);
            const int lr = NRA * lane;
            live = lr < r0e;
            pcls = live ? static_cast<int>((R0s + lr) / I0) : cls_hi;
            const int64_t i0s = R0s + lr - static_cast<int64_t>(pcls) * I0;
#pragma unroll
            for (int a = 0; a < NRA; ++a) {
                const int off = 2 * ((a >> 1) ^ hsw) + (a & 1);
                u0r[a] = lr + off < r0e ? __ldg(p.u0 + i0s + off) : 0.0;
            }
#pragma unroll
            for (int b = 0; b < NCB; ++b) {
                const int j = warp + NWC * b;
                u1c[b] = (j < t1e && live) ? __ldg(p.u1 + K * (R1s + j) + pcls) : 0.0;
                coff[b] = (min(j, t1e - 1) * cst) / 2 + (NRA / 2) * lane;
#pragma unroll
                for (int a = 0; a < NRA; ++a) acc[a][b] = 0.0;
            }
            P0row = p.P0 + static_cast<int64_t>(g1) * p.P0_stride + R0s;
            P1row = p.P1 ? p.P1 + static_cast<int64_t>(g0) * p.P1_stride + R1s : nullptr;
            if constexpr (NS > 1) {
                // zero this thread's accumulators of every sub-strip of the tile
                nsub = (t1e + p.ts - 1) / p.ts;
                tmem_wait_st();
                for (int q = 0; q < nsub; ++q)
                    tmem_store_doubles<NRA * NCB>(tmem_acc + q * (2 * NRA * NCB), &acc[0][0]);
            }
        }
        // sub-strip of this box: index, first column inside the tile, width
        const int sb = NS > 1 ? (md.w >> 8) : 0;
        const int jb = sb * p.ts;
        const int wsb = NS > 1 ? min(p.ts, t1e - jb) : t1e;
        if constexpr (NS > 1) {
            if (md.w & kFirst) last_w = -1;
#pragma unroll
            for (int b = 0; b < NCB; ++b) {
                const int j = warp + NWC * b;
                u1c[b] = (j < wsb && live) ? __ldg(p.u1 + K * (R1s + jb + j) + pcls) : 0.0;
            }
            if (wsb != last_w) {  // only the ragged last box of the last column tile differs
#pragma unroll
                for (int b = 0; b < NCB; ++b)
                    coff[b] = (min(warp + NWC * b, wsb - 1) * cst) / 2 + (NRA / 2) * lane;
                last_w = wsb;
            }
            // (the first box of a segment starts from the zeros set above).
            // Requesting the next box's accumulators right after this box's
            // store — the load under the wait for the next stage — measured
            // slower (248 registers: C5 6.1 vs 5.6 ms).
            if (!(md.w & kFirst)) {
                tmem_wait_st();
                tmem_load_doubles<NRA * NCB>(tmem_acc + sb * (2 * NRA * NCB), &acc[0][0]);
            }
        }
        {
            if constexpr (KO == 1) {
            const double wo = __ldg(p.W + o);
            const double2* st = reinterpret_cast<const double2*>(ring + stage * stage_dbl);
            if (p.debug_mode == 1) {
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[stage]);
                if (++stage == nst) {
                    stage = 0;
                    phase ^= 1;
                }
                continue;
            }
            double c1v[NCB];
            if (sb == 0) {
#pragma unroll
                for (int a = 0; a < NRA; ++a) c0p[a] = 0.0;
            }
            auto column = [&](int b, const double2* v) {
                double c1p = 0.0;
#pragma unroll
                for (int q = 0; q < NP; ++q) {
                    acc[2 * q][b] = fma(v[q].x, wo, acc[2 * q][b]);
                    acc[2 * q + 1][b] = fma(v[q].y, wo, acc[2 * q + 1][b]);
                    c1p = fma(v[q].x, u0r[2 * q], c1p);
                    c1p = fma(v[q].y, u0r[2 * q + 1], c1p);
                    c0p[2 * q] = fma(v[q].x, u1c[b], c0p[2 * q]);
                    c0p[2 * q + 1] = fma(v[q].y, u1c[b], c0p[2 * q + 1]);
                }
                c1v[b] = c1p;
            };
            if constexpr (STAGE_REGS) {
                // copy the slice to registers and release the stage before computing
                double2 v[NCB][NP];
#pragma unroll
                for (int b = 0; b < NCB; ++b)
#pragma unroll
                    for (int q = 0; q < NP; ++q) v[b][q] = st[coff[b] + (q ^ hsw)];
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[stage]);
#pragma unroll
                for (int b = 0; b < NCB; ++b) column(b, v[b]);
            } else {
#pragma unroll
                for (int b = 0; b < NCB; ++b) {
                    double2 v[NP];
#pragma unroll
                    for (int q = 0; q < NP; ++q) v[q] = st[coff[b] + (q ^ hsw)];
                    column(b, v);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[stage]);
            }
            if (++stage == nst) {
                stage = 0;
                phase ^= 1;
            }

            if (P1row) {
                // C1 of merged column j, class c = real column K j + c, stored
                // class-major (c MI1 + j) so the second stage reads only the
                // classes a row tile holds; a tile spanning several classes
                // reduces each class's lanes separately
                double* dst = P1row + static_cast<int64_t>(o) * I1;
                int col;
                if (cls_lo == cls_hi) {
                    const double c1 = warp_transpose_sum<NCB>(c1v, lane, &col);
                    const int j = warp + NWC * col;
                    if ((lane & (32 / NCB - 1)) == 0 && j < wsb) dst[cls_lo * MI1 + jb + j] = c1;
                } else {
                    for (int c = cls_lo; c <= cls_hi; ++c) {
                        double mv[NCB];
#pragma unroll
                        for (int b = 0; b < NCB; ++b) mv[b] = pcls == c ? c1v[b] : 0.0;
                        const double c1 = warp_transpose_sum<NCB>(mv, lane, &col);
                        const int j = warp + NWC * col;
                        if ((lane & (32 / NCB - 1)) == 0 && j < wsb) dst[c * MI1 + jb + j] = c1;
                    }
                }
            }

            if constexpr (NS > 1)
                tmem_store_doubles<NRA * NCB>(tmem_acc + sb * (2 * NRA * NCB), &acc[0][0]);
            if (sb == nsub - 1) {
                const int slot = pc & 1;
                mbar_wait(&red_empty[slot], ((pc >> 1) & 1) ^ 1);
                double2* rb =
                    reinterpret_cast<double2*>(red + slot * NWC * RMAX + warp * RMAX) + (NRA / 2) * lane;
#pragma unroll
                for (int q = 0; q < NP; ++q) rb[q ^ hsw] = make_double2(c0p[2 * q], c0p[2 * q + 1]);
                __syncwarp();
                if (lane == 0) mbar_arrive(&red_full[slot]);
                if (pc > 0) reduce_pending();
                pend_dst = P0row + static_cast<int64_t>(o) * MI0;
                pend_r0e = r0e;
                ++pc;
            }
            } else {
            const double2* st = reinterpret_cast<const double2*>(ring + stage * stage_dbl);
            if (p.debug_mode == 1) {
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[stage]);
                if (++stage == nst) {
                    stage = 0;
                    phase ^= 1;
                }
                continue;
            }
            const int ob = o * KO;          // first o-panel of the box
            const int pstride = r0e * t1e / 2;  // double2 per panel in the box
            double c0p[KO][NRA];
            double c1v[KO * NCB];
#pragma unroll
            for (int k = 0; k < KO; ++k)
#pragma unroll
                for (int a = 0; a < NRA; ++a) c0p[k][a] = 0.0;
#pragma unroll
            for (int k = 0; k < KO; ++k) {
                const double wo = __ldg(p.W + ob + k);
                auto column = [&](int b, const double2* v) {
                    double c1p = 0.0;
#pragma unroll
                    for (int q = 0; q < NP; ++q) {
                        acc[2 * q][b] = fma(v[q].x, wo, acc[2 * q][b]);
                        acc[2 * q + 1][b] = fma(v[q].y, wo, acc[2 * q + 1][b]);
                        c1p = fma(v[q].x, u0r[2 * q], c1p);
                        c1p = fma(v[q].y, u0r[2 * q + 1], c1p);
                        c0p[k][2 * q] = fma(v[q].x, u1c[b], c0p[k][2 * q]);
                        c0p[k][2 * q + 1] = fma(v[q].y, u1c[b], c0p[k][2 * q + 1]);
                    }
                    c1v[k * NCB + b] = c1p;
                };
                const double2* sp = st + k * pstride;
                if constexpr (STAGE_REGS) {
                    // copy the slice to registers; the last panel releases the stage
                    double2 v[NCB][NP];
#pragma unroll
                    for (int b = 0; b < NCB; ++b)
#pragma unroll
                        for (int q = 0; q < NP; ++q) v[b][q] = sp[coff[b] + (q ^ hsw)];
                    if (k == KO - 1) {
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&empty[stage]);
                    }
#pragma unroll
                    for (int b = 0; b < NCB; ++b) column(b, v[b]);
                } else {
#pragma unroll
                    for (int b = 0; b < NCB; ++b) {
                        double2 v[NP];
#pragma unroll
                        for (int q = 0; q < NP; ++q) v[q] = sp[coff[b] + (q ^ hsw)];
                        column(b, v);
                    }
                    if (k == KO - 1) {
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&empty[stage]);
                    }
                }
            }
            if (++stage == nst) {
                stage = 0;
                phase ^= 1;
            }

            if (P1row) {
                // C1 of merged column j, class c = real column K j + c, stored
                // class-major (c MI1 + j) so the second stage reads only the
                // classes a row tile holds; a tile spanning several classes
                // reduces each class's lanes separately.  Value index kb = panel
                // k * NCB + column slot b.
                constexpr int NV = KO * NCB;
                int col;
                if (cls_lo == cls_hi) {
                    const double c1 = warp_transpose_sum<NV>(c1v, lane, &col);
                    const int k = col / NCB, j = warp + NWC * (col % NCB);
                    if ((lane & (32 / NV - 1)) == 0 && j < t1e)
                        P1row[static_cast<int64_t>(ob + k) * I1 + cls_lo * MI1 + j] = c1;
                } else {
                    for (int c = cls_lo; c <= cls_hi; ++c) {
                        double mv[NV];
#pragma unroll
                        for (int v = 0; v < NV; ++v) mv[v] = pcls == c ? c1v[v] : 0.0;
                        const double c1 = warp_transpose_sum<NV>(mv, lane, &col);
                        const int k = col / NCB, j = warp + NWC * (col % NCB);
                        if ((lane & (32 / NV - 1)) == 0 && j < t1e)
                            P1row[static_cast<int64_t>(ob + k) * I1 + c * MI1 + j] = c1;
                    }
                }
            }

#pragma unroll
            for (int k = 0; k < KO; ++k) {
                double2* rb = reinterpret_cast<double2*>(red + ((rbuf * KO + k) * NWC + warp) * RMAX) +
                              (NRA / 2) * lane;
#pragma unroll
                for (int q = 0; q < NP; ++q) rb[q ^ hsw] = make_double2(c0p[k][2 * q], c0p[k][2 * q + 1]);
            }
            asm volatile("bar.sync 1, %0;" ::"n"(NWC * 32) : "memory");
            const double* rr = red + rbuf * KO * NWC * RMAX;
            for (int x = threadIdx.x; x < KO * r0e; x += NWC * 32) {
                const int k = x / r0e, i = x - k * r0e;
                double sum = 0.0;
#pragma unroll
                for (int w = 0; w < NWC; ++w) sum += rr[(k * NWC + w) * RMAX + i];
                P0row[static_cast<int64_t>(ob + k) * MI0 + i] = sum;
            }
            }
            rbuf ^= 1;
            if (md.w & kLast) {
                // flush the B01 face partial of this segment
                double* dst = p.P01 + static_cast<int64_t>(s) * p.r0 * p.t1;
                for (int q = 0; q < nsub; ++q) {
                    const int jq = q * p.ts, wq = NS > 1 ? min(p.ts, t1e - jq) : t1e;
                    if constexpr (NS > 1) {
                        tmem_wait_st();
                        tmem_load_doubles<NRA * NCB>(tmem_acc + q * (2 * NRA * NCB), &acc[0][0]);
                    }
#pragma unroll
                    for (int b = 0; b < NCB; ++b) {
                        const int j = warp + NWC * b;
                        if (j >= wq) continue;
#pragma unroll
                        for (int a = 0; a < NRA; ++a) {
                            const int i = NRA * lane + 2 * ((a >> 1) ^ hsw) + (a & 1);
                            if (i < r0e) dst[(jq + j) * p.r0 + i] = acc[a][b];
                        }
                    }
                }
            }
        }
    }
    if constexpr (KO == 1) {
        if (pc > 0) reduce_pending();
    }
    if constexpr (NS > 1) {
        tmem_wait_st();
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        asm volatile("bar.sync 1, %0;" ::"n"(NWC * 32) : "memory");
        if (warp == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
        }
    }
    if (p.trace && threadIdx.x == 0) {
        unsigned long long t_end;
        unsigned int smid;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        p.trace[3 * blockIdx.x] = t_start;
        p.trace[3 * blockIdx.x + 1] = t_end;
        p.trace[3 * blockIdx.x + 2] = smid;
    }
}

// Second stage of one level, all outputs in one launch, every sum in a fixed
// order (bit-reproducible for any schedule of the first stage):
//   B01[i0 + I0 i1] = sum over the tile's segments (o order) of P01 partials;
//       tiles live in the merged view: (i0, i1) is merged row (i1 mod K) I0 + i0
//       of merged column i1 / K;
//   C0[i0 + I0 o]   = sum_{g1 < G1} sum_{p < K} P0[g1 stride0 + o K I0 + p I0 + i0];
//   C1[i1 + I1 o]   = sum over the row tiles g0 holding class p = i1 mod K
//       (merged rows [p I0, (p+1) I0)) of P1[g0 stride1 + o I1 + p MI1 + i1 / K].
// A null P0 / P1 means the first stage wrote that output in place.
struct FinishArgs {
    const double* P01;
    const int* tile_seg;
    int64_t I0, I1, O, MI1;
    int K, lgK, r0, t1, G0, G1;
    double* b01;
    const double* P0;
    int64_t stride0;
    double* c0;
    const double* P1;
    int64_t stride1;
    double* c1;
    int64_t n_b01, n_c0, n_c1;
    // x / d for 0 <= x < 2^31 as (x * m) >> s (m = ceil(2^s / d), s = 31 +
    // ceil(log2 d): exact, Granlund-Montgomery) for d = I0, I1, r0, t1
    uint64_t m_I0, m_I1, m_r0, m_t1;
    int s_I0, s_I1, s_r0, s_t1;
};

void fastdiv_init(int64_t d, uint64_t& m, int& sh) {
    int l = 0;
    while ((int64_t(1) << l) < d) ++l;
    sh = 31 + l;
    m = static_cast<uint64_t>(((static_cast<unsigned __int128>(1) << sh) + d - 1) / d);
}

// Element per thread.  With K == 1 the C0 / C1 partial copies have the output
// layout (a plain sum of copies); K is a power of two.  IDX is the index type
// (32-bit whenever the level's element counts allow).
// Fixed-order sums of partials: s = ((0 + v_0) + v_1) + ... in index order.
// ordered_sum over p[0], p[stride], ...: full batches of 8 loads without
// predication, then 4, then singles; the pointer advances (no per-load
// multiply) — the generic version cost ~480 instructions per output at C2
__device__ __forceinline__ double ordered_sum_strided(int cnt, const double* p, int64_t stride) {
    double s = 0.0;
    int t = 0;
    for (; t + 8 <= cnt; t += 8, p += 8 * stride) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcs(p + u * stride);
#pragma unroll
        for (int u = 0; u < 8; ++u) s += v[u];
    }
    if (t < cnt) {  // the rest as one predicated batch (loads in flight together)
        const int r = cnt - t;
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = u < r ? __ldcs(p + u * stride) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (u < r) s += v[u];
    }
    return s;
}

// sum over g < G (outer), q < KK (inner) of p[g stride + q inner], in that order
template <int KK>
__device__ __forceinline__ double ordered_sum_2d(int G, const double* p, int64_t stride, int64_t inner) {
    constexpr int GB = KK >= 8 ? 1 : 8 / KK;  // g's per batch (8+ loads in flight)
    double s = 0.0;
    int g = 0;
    for (; g + GB <= G; g += GB, p += GB * stride) {
        double v[GB][KK];
#pragma unroll
        for (int a = 0; a < GB; ++a)
#pragma unroll
            for (int q = 0; q < KK; ++q) v[a][q] = __ldcs(p + a * stride + q * inner);
#pragma unroll
        for (int a = 0; a < GB; ++a)
#pragma unroll
            for (int q = 0; q < KK; ++q) s += v[a][q];
    }
    if (g < G) {  // the rest (< GB g's) as one predicated batch
        const int r = G - g;
        double v[GB][KK];
#pragma unroll
        for (int a = 0; a < GB; ++a)
#pragma unroll
            for (int q = 0; q < KK; ++q) v[a][q] = a < r ? __ldcs(p + a * stride + q * inner) : 0.0;
#pragma unroll
        for (int a = 0; a < GB; ++a)
#pragma unroll
            for (int q = 0; q < KK; ++q)
                if (a < r) s += v[a][q];
    }
    return s;
}

template <typename IDX>
__device__ __forceinline__ IDX fdiv(IDX x, int64_t d, uint64_t m, int sh) {
    if constexpr (sizeof(IDX) == 4)
        return static_cast<IDX>((static_cast<uint64_t>(x) * m) >> sh);  // x < 2^31
    else
        return x / static_cast<IDX>(d);
}

template <typename IDX>
__global__ void finish_kernel(const FinishArgs f) {
    pdl_launch_dependents();
    pdl_wait();
    const IDX nb = static_cast<IDX>(f.n_b01), n0 = static_cast<IDX>(f.n_c0);
    const IDX total = nb + n0 + static_cast<IDX>(f.n_c1);
    const IDX I0 = static_cast<IDX>(f.I0), I1 = static_cast<IDX>(f.I1);
    const int K = f.K;
    const int64_t tile_elems = static_cast<int64_t>(f.r0) * f.t1;
    for (IDX e = blockIdx.x * static_cast<IDX>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<IDX>(gridDim.x) * blockDim.x) {
        double s = 0.0;
        if (e < nb) {
            const IDX i1 = fdiv<IDX>(e, f.I0, f.m_I0, f.s_I0), i0 = e - i1 * I0;
            const IDX p = i1 & (K - 1), c = i1 >> f.lgK;
            const IDX r = p * I0 + i0;
            const int g0 = static_cast<int>(fdiv<IDX>(r, f.r0, f.m_r0, f.s_r0));
            const int g1 = static_cast<int>(fdiv<IDX>(c, f.t1, f.m_t1, f.s_t1));
            const int tile = g0 + f.G0 * g1;
            const double* src = f.P01 + static_cast<int64_t>(c - static_cast<IDX>(g1) * f.t1) * f.r0 +
                                (r - static_cast<IDX>(g0) * f.r0);
            const int sb = __ldg(f.tile_seg + tile), se = __ldg(f.tile_seg + tile + 1);
            s = ordered_sum_strided(se - sb, src + sb * tile_elems, tile_elems);
            f.b01[e] = s;
        } else if (e < nb + n0) {
            const IDX x = e - nb;
            if (K == 1) {
                const double* src = f.P0 + x;
                s = ordered_sum_strided(f.G1, src, f.stride0);
            } else {
                const IDX o = fdiv<IDX>(x, f.I0, f.m_I0, f.s_I0), i0 = x - o * I0;
                const double* src = f.P0 + static_cast<int64_t>(o) * K * f.I0 + i0;
                // g outer, q inner: the same summation order
                switch (K) {
                    case 2: s = ordered_sum_2d<2>(f.G1, src, f.stride0, f.I0); break;
                    case 4: s = ordered_sum_2d<4>(f.G1, src, f.stride0, f.I0); break;
                    case 8: s = ordered_sum_2d<8>(f.G1, src, f.stride0, f.I0); break;
                    default: s = ordered_sum_2d<16>(f.G1, src, f.stride0, f.I0); break;
                }
            }
            f.c0[x] = s;
        } else {
            const IDX x = e - nb - n0;
            if (K == 1) {
                const double* src = f.P1 + x;
                s = ordered_sum_strided(f.G0, src, f.stride1);
            } else {
                const IDX o = fdiv<IDX>(x, f.I1, f.m_I1, f.s_I1), i1 = x - o * I1;
                const int p = static_cast<int>(i1 & (K - 1));
                const int ga = static_cast<int>(fdiv<IDX>(static_cast<IDX>(p * f.I0), f.r0, f.m_r0, f.s_r0));
                const int gb =
                    static_cast<int>(fdiv<IDX>(static_cast<IDX>((p + 1) * f.I0 - 1), f.r0, f.m_r0, f.s_r0));
                const double* src = f.P1 + static_cast<int64_t>(o) * f.I1 + p * f.MI1 + (i1 >> f.lgK);
                s = ordered_sum_strided(gb - ga + 1, src + ga * f.stride1, f.stride1);
            }
            f.c1[x] = s;
        }
    }
}

// B01 when tiles hold many segments (deep o ranges split over many CTAs, e.g.
// a single 60 x 60 face tile): a CTA takes 32 consecutive offsets of one
// tile's partial slots (lanes, coalesced) and its 16 warps take 16 equal
// slices of the tile's segments (8 loads in flight per lane); the slices are
// combined in warp order through shared memory — one fixed summation order.
constexpr int kB01Warps = 16;
__global__ void __launch_bounds__(kB01Warps * 32) finish_b01_seg_kernel(const FinishArgs f) {
    pdl_launch_dependents();
    pdl_wait();
    __shared__ double red[kB01Warps][33];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t tile_elems = static_cast<int64_t>(f.r0) * f.t1;
    const int64_t per_tile = (tile_elems + 31) / 32;
    const int ntiles = f.G0 * f.G1;
    const int64_t units = static_cast<int64_t>(ntiles) * per_tile;
    const int64_t MI0 = static_cast<int64_t>(f.K) * f.I0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        const int tile = static_cast<int>(u / per_tile);
        const int64_t off = (u - static_cast<int64_t>(tile) * per_tile) * 32 + lane;
        const int g0 = tile % f.G0, g1 = tile / f.G0;
        const int64_t j = off / f.r0, i = off - j * f.r0;
        const int64_t r = static_cast<int64_t>(g0) * f.r0 + i, c = static_cast<int64_t>(g1) * f.t1 + j;
        const bool valid = off < tile_elems && i < f.r0 && r < MI0 && c < f.MI1;
        const int sb = __ldg(f.tile_seg + tile), se = __ldg(f.tile_seg + tile + 1);
        const int per = (se - sb + kB01Warps - 1) / kB01Warps;
        const int k0 = sb + warp * per, k1 = min(se, k0 + per);
        const double* src = f.P01 + (valid ? off : 0);
        double s = 0.0;
        int k = k0;
        for (; k + 8 <= k1; k += 8) {
            double v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = valid ? __ldcs(src + (k + q) * tile_elems) : 0.0;
#pragma unroll
            for (int q = 0; q < 8; ++q) s += v[q];
        }
        if (k < k1) {  // the rest as one predicated batch (loads in flight together)
            const int r = k1 - k;
            double v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = (valid && q < r) ? __ldcs(src + (k + q) * tile_elems) : 0.0;
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (q < r) s += v[q];
        }
        red[warp][lane] = s;
        __syncthreads();
        if (warp == 0 && valid) {
            double t = 0.0;
#pragma unroll
            for (int w = 0; w < kB01Warps; ++w) t += red[w][lane];
            // merged row r = p I0 + i0 of merged column c: B01[i0 + I0 (K c + p)]
            const int64_t pcl = r / f.I0, i0 = r - pcl * f.I0;
            f.b01[i0 + f.I0 * (f.K * c + pcl)] = t;
        }
        __syncthreads();
    }
}

struct OuterArgs {
    int nout;
    int64_t dims[kMaxOrder];
    const double* u[kMaxOrder];
    int64_t O;
    double* W;
};

// W[o] = u_2[i_2] * u_3[i_3] * ... (first outer mode fastest).
__global__ void outer_weights_kernel(const OuterArgs a) {
    pdl_launch_dependents();
    pdl_wait();
    for (int64_t o = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; o < a.O;
         o += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int64_t q = o;
        double w = 1.0;
        for (int k = 0; k < a.nout; ++k) {
            w *= a.u[k][q % a.dims[k]];
            q /= a.dims[k];
        }
        a.W[o] = w;
    }
}

// ------------------------------------------------------------ the planner --
enum class Where { Tensor, Final, Work, None };

struct Ref {
    Where where = Where::None;
    uint64_t off = 0;  // element offset into the final blocks or the work arena
};

struct Level {
    // sub-problem
    int order = 0;
    int64_t dims[kMaxOrder] = {};
    int modes[kMaxOrder] = {};  // original mode ids (ascending)
    Ref input;
    // view & tiling
    int64_t I0 = 0, I1 = 0, O = 0;
    int K = 1;                 // alignment classes merged per column (box kernel)
    int KO = 1;                // o-panels per box (small faces); segments count o-groups
    int64_t MI0 = 0, MI1 = 0;  // merged view K I0 x I1/K (tiles live here)
    int nra = 4, ncb = 8, stages = 3;
    int nwc = 15;  // consumer warps (box kernel)
    int ns = 1;    // column sub-strips per tile (accumulators in tensor memory when > 1)
    int ts = 0;    // columns per box (= t1 when ns == 1)
    int stage_dbl = 0;
    int dyn_first = 0, ndyn = 0;  // dynamic-tail segments (box kernel only)
    bool tma = false;
    int r0 = 0, t1 = 0, G0 = 0, G1 = 0, ncta = 0, nseg = 0, ntiles = 0;
    size_t smem = 0;
    // plan metadata (device offsets into SweepPlan::meta, in ints)
    uint64_t seg_off = 0, cta_off = 0, tile_off = 0;
    // outputs
    Ref out_b01, out_c0, out_c1;
    Ref w, p01, p0, p1;
    // Lanes: the levels whose blocks are all needed form a spine (root, its C0
    // child, that one's C0 child, ...) on lane 0; the C1 child of the spine
    // level at depth k starts a chain (each of its levels has one child) on lane
    // 1 + k % 3, which depends only on that spine level's C0 / C1.
    int lane = 0;
    int depth = 0;          // spine depth of this level (lane 0) or of the chain's parent
    bool chain_head = false;  // first level of a chain: waits for the spine level at `depth`
};

}  // namespace

struct SweepPlan {
    std::vector<uint64_t> dims;
    std::vector<Level> levels;
    std::vector<int> host_meta;
    DeviceBuffer meta;
    DeviceBuffer counters;  // one dynamic-tail work counter per level
    uint64_t work_elems = 0;
    uint64_t nblocks = 0;
};

namespace {

size_t smem_bytes(int nra, int ncb, int stages, bool tma) {
    const int rmax = 32 * nra;
    return static_cast<size_t>(stages) * kNWC * ncb * (rmax + (tma ? 0 : 2)) * 8 +
           static_cast<size_t>(2) * kNWC * rmax * 8 + 2 * stages * 8;
}

// Alignment classes.  TMA moves whole 128-B lines: a box row that starts or
// ends inside a line fetches the full line, and the neighbouring tile fetches
// it again (measured: 6.4% extra DRAM reads at I0 = 1000, whose 8000-B column
// pitch puts every other column at a 64-B offset).  Columns whose start
// offsets mod 128 B differ are "classes"; K consecutive columns (one of each
// class) are merged into one column of K I0 rows, whose pitch is a multiple of
// 128 B.  Row tiles of whole lines (r0 % 16 == 0) then never share a line.
// The box kernel maps merged rows back to (i0, class): lane rows stay inside
// one class because I0 % 4 == 0.
int alignment_classes(const Level& L) {
    // R1_SWEEP_MERGE: 0 never merge, 1 (default) when it keeps tiles full, 2 whenever legal
    static const char* env = dev_env("R1_SWEEP_MERGE");
    const int mode = env ? std::atoi(env) : 1;
    if (mode == 0) return 1;
    if (!L.tma || L.I0 % 4 != 0) return 1;
    const int64_t pitch = 8 * L.I0;
    int64_t g = 128;
    while (pitch % g) g >>= 1;
    const int K = static_cast<int>(128 / g);
    if (K == 1 || L.I1 % K != 0 || (8 * L.I0 * L.I1) % 128 != 0) return 1;
    // Worth it only when the merged view keeps full tiles: a class fills at
    // least one row tile and there are >= 4 full column tiles (I1 / K columns).
    if (mode == 1 && (L.I0 < 128 || L.I1 / K < 4 * kBoxNWC * kBoxNCB)) return 1;
    return K;
}

void tile_level(Level& L, int num_sms) {
    L.nra = L.I0 > 64 ? 4 : (L.I0 > 32 ? 2 : 1);
    L.ncb = 8;
    L.stages = L.nra == 4 ? 3 : (L.nra == 2 ? 5 : 8);
    // TMA needs 16-B global strides (I0 even) and an int32 outer coordinate.
    L.tma = (L.I0 % 2 == 0) && L.O < (int64_t(1) << 31) && L.I1 < (int64_t(1) << 31);
    L.smem = smem_bytes(L.nra, L.ncb, L.stages, L.tma);
    L.K = alignment_classes(L);
    L.MI0 = L.K * L.I0;
    L.MI1 = L.I1 / L.K;
    const int rmax = 32 * L.nra, cmax = kNWC * L.ncb;
    // Balance row tiles: G0 = ceil(I0/rmax), r0 = ceil(I0/G0) (same for cols);
    // on the TMA path r0 is even so interior boxes hold exactly the tile.
    if (L.tma) {
        // Balanced tiles on the fixed RMAX x CMAX consumer grid, in the merged view.
        L.nra = L.MI0 > 64 ? 4 : 2;
        L.ncb = kBoxNCB;
        // 128 < I0 <= 256, unmerged: one 256 x 30 row tile (8 rows x 2 columns
        // per lane, the same 16 accumulators) instead of two 128 x 60 ones —
        // no C1 partials, and no 128-B line shared by two row tiles (C3 200^4:
        // with a 1600-B column pitch every column's split fell inside a line,
        // 8% extra DRAM reads)
        static const char* n8_env = dev_env("R1_SWEEP_NRA8");
        const bool nra8 = n8_env ? std::atoi(n8_env) != 0 : true;
        L.nwc = kBoxNWC;  // (8 warps x 4 columns at I0 = 200 measured no faster)
        if (nra8 && L.K == 1 && L.MI0 > 128 && L.MI0 <= 256) {
            L.nra = 8;
            L.ncb = 2;
        }
        // Wide shapes (round 2): 32 elements per consumer thread instead of 16,
        // on fewer warps — the per-panel fixed work (barrier waits, the C1
        // butterfly, the C0 block reduction) is paid per 32 elements: 3.8
        // instead of 5.5 static instructions per DFMA in the 128-row loop.
        // Same-box A/B: C5 5.44-5.55 -> 5.31 ms (sustained 600 sweeps under the
        // power cap 5.72 -> 5.39), C2 1.39 -> 1.35, C4 1.14 -> 1.12 and C3 2.50 ->
        // 2.22 ms (11 warps x 4 columns also cut its column tiles from 7 to 5).
        // Measured and left out: 7 warps x 4 columns for the 256-row tiles (C3
        // 2.56 ms) and 11 warps x 8 columns for the 128-row ones (C5 5.45 ms:
        // 168-register cap, two 86-KB stages).  R1_SWEEP_WIDE=0 (development
        // build) restores the 15-warp shapes; bits 1 / 4 / 8 select the 128- /
        // 64- / 256-row shapes.
        static const char* wide_env = dev_env("R1_SWEEP_WIDE");
        const int wide = wide_env ? std::atoi(wide_env) : kWideDefault;
        if ((wide & 1) && L.nra == 4) {
            L.nwc = 7;  // 128 x 56
            L.ncb = 8;
        } else if ((wide & 8) && L.nra == 8) {
            L.nwc = 11;  // 256 x 44
            L.ncb = 4;
        } else if ((wide & 4) && L.nra == 2) {
            L.nwc = 8;  // 64 x 64
            L.ncb = 8;
        }
        const int rm = 32 * L.nra, cm = L.nwc * L.ncb;
        L.G0 = static_cast<int>((L.MI0 + rm - 1) / rm);
        L.r0 = static_cast<int>((L.MI0 + L.G0 - 1) / L.G0);
        // Whole 128-B lines per tile row when the (merged) column pitch is a
        // multiple of 128 B; else whole 32-B sectors (16 B, the TMA minimum,
        // for I0 % 4 != 0).
        const int q = (L.MI0 % 16 == 0) ? 16 : ((L.I0 % 4 == 0) ? 4 : 2);
        L.r0 = std::min(rm, (L.r0 + q - 1) / q * q);
        // a half-line column pitch (8 I0 = 64 mod 128, unmerged): round the row
        // tile up to whole lines, so the tile split is line-aligned in every
        // other column (C3 200^4: 100 -> 112 rows, -1.5%)
        if (L.G0 > 1 && L.K == 1 && (8 * L.I0) % 128 == 64 && L.r0 % 16 != 0) {
            const int r16 = (L.r0 + 15) / 16 * 16;
            if (r16 <= rm && static_cast<int64_t>(r16) * ((L.MI0 + L.r0 - 1) / L.r0 - 1) < L.MI0) L.r0 = r16;
        }
        L.G0 = static_cast<int>((L.MI0 + L.r0 - 1) / L.r0);
        L.G1 = static_cast<int>((L.MI1 + cm - 1) / cm);
        L.t1 = static_cast<int>((L.MI1 + L.G1 - 1) / L.G1);
        L.G1 = static_cast<int>((L.MI1 + L.t1 - 1) / L.t1);
        L.ns = 1;
        L.ts = L.t1;
        // Sub-strips (tensor-memory accumulators, 128 x 56 shape only; development
        // switch, see kSubStripsDefault): tiles of up to 4 boxes' width — the face
        // has up to 4 x fewer column tiles and as many fewer C0 partial sets (C5:
        // 9 -> 3, 384 MB less written and read again per sweep) — as long as the
        // level keeps every SM busy.
        static const char* ns_env = dev_env("R1_SWEEP_NS");
        const int ns_max = ns_env ? std::max(1, std::min(4, std::atoi(ns_env))) : kSubStripsDefault;
        if (L.nra == 4 && L.nwc == 7 && ns_max > 1 && L.G1 > 1) {
            for (int ns = ns_max; ns > 1; --ns) {
                const int g1 = static_cast<int>((L.MI1 + static_cast<int64_t>(cm) * ns - 1) / (static_cast<int64_t>(cm) * ns));
                int t1 = static_cast<int>((L.MI1 + g1 - 1) / g1);
                const int nsub = (t1 + cm - 1) / cm;       // boxes per regular tile
                const int ts = (t1 + nsub - 1) / nsub;     // equal sub-strips
                t1 = nsub * ts;
                const int g1b = static_cast<int>((L.MI1 + t1 - 1) / t1);
                static const char* mp_env = dev_env("R1_SWEEP_NS_MINP");  // development: panels per SM required
                const int64_t minp = mp_env ? std::atoi(mp_env) : 64;
                if (nsub < 2 || static_cast<int64_t>(L.G0) * g1b * L.O < minp * num_sms) continue;
                L.ns = nsub;
                L.ts = ts;
                L.t1 = t1;
                L.G1 = g1b;
                break;
            }
        }
        L.ntiles = L.G0 * L.G1;
        // a single small face tile: KO panels per box amortise the per-panel
        // reductions (C4: 60 x 60 faces)
        L.KO = 1;
        static const char* ko_env = dev_env("R1_SWEEP_KO");
        int ko_max = ko_env ? std::atoi(ko_env) : 2;  // measured: 2 beats 4 on C4
        if (L.nwc == 8) ko_max = std::min(ko_max, 2);   // the 64 x 64 shape has KO <= 2
        if (L.ntiles == 1 && L.r0 * L.t1 <= 64 * 64 && L.nra == 2)
            for (int ko = ko_max; ko > 1; ko >>= 1)
                if (L.O % ko == 0) {
                    L.KO = ko;
                    break;
                }
        const size_t red = static_cast<size_t>(2) * L.KO * L.nwc * rm * 8;
        const size_t bars = 2 * kMaxStages * 8 + kMaxStages * 16 + 4 * 8 + 16;  // + tensor-memory base slot
        const size_t box = static_cast<size_t>(L.r0) * L.ts * 8 * L.KO;
        const size_t ring = kSmemBudget - red - bars - rm * 8 - 1024;
        L.stages = static_cast<int>(std::min<size_t>(kMaxStages, ring / box));
        L.stage_dbl = static_cast<int>(((box + 127) & ~size_t(127)) / 8);  // 128-B aligned
        L.stages = static_cast<int>(std::min<size_t>(L.stages, ring / (L.stage_dbl * 8)));
        L.smem = (static_cast<size_t>(L.stages) * L.stage_dbl + rm) * 8 + red + bars;
        return;
    }
    L.G0 = static_cast<int>((L.I0 + rmax - 1) / rmax);
    L.r0 = static_cast<int>((L.I0 + L.G0 - 1) / L.G0);
    // Row tiles in whole 32-B sectors when the column stride allows it, so
    // neighbouring tiles never share a DRAM sector (it would be fetched twice).
    const int q = (L.I0 % 4 == 0) ? 4 : (L.tma ? 2 : 1);
    if (L.r0 % q) {
        L.r0 += q - L.r0 % q;
        if (L.r0 > rmax) L.r0 = rmax;
        L.G0 = static_cast<int>((L.I0 + L.r0 - 1) / L.r0);
    }
    L.G1 = static_cast<int>((L.I1 + cmax - 1) / cmax);
    L.t1 = static_cast<int>((L.I1 + L.G1 - 1) / L.G1);
    L.ntiles = L.G0 * L.G1;
    (void)num_sms;
}

// Partition (tile, o) panels into ncta contiguous chunks of equal cost and
// cut them into segments (maximal runs inside one tile).
void partition_level(Level& L, int num_sms, std::vector<int>& meta) {
    const int64_t Og = L.O / L.KO;  // o-groups (KO panels each)
    const int64_t npanels = static_cast<int64_t>(L.ntiles) * Og;
    auto panel_cost = [&](int tile) {
        const int g0 = tile % L.G0, g1 = tile / L.G0;
        const int64_t r = std::min<int64_t>(L.r0, L.MI0 - int64_t(g0) * L.r0);
        const int64_t c = std::min<int64_t>(L.t1, L.MI1 - int64_t(g1) * L.t1);
        // bytes dominate; zero-filled edge boxes still cost consumer issue time
        return static_cast<double>(r * c) + 512.0;
    };
    double total = 0.0;
    for (int t = 0; t < L.ntiles; ++t) total += panel_cost(t) * static_cast<double>(Og);
    // Enough CTAs to fill the chip, but at least ~min_panels panels each.
    static const char* mp_env = dev_env("R1_SWEEP_MIN_PANELS");
    // 4 (was 16): the small recursion levels (60^3 at C4) ran on one CTA
    const int64_t min_panels = mp_env ? std::max(1, std::atoi(mp_env)) : 4;
    int64_t ncta = std::min<int64_t>(num_sms, std::max<int64_t>(1, npanels / min_panels));
    static const char* nc_env = dev_env("R1_SWEEP_NCTA");  // development: cap the grid
    if (nc_env) ncta = std::max<int64_t>(1, std::min<int64_t>(ncta, std::atoi(nc_env)));
    L.ncta = static_cast<int>(ncta);
    std::vector<Seg> segs;
    std::vector<int> cta_seg(L.ncta + 1, 0);
    // The box kernel takes a dynamic tail: the last kDynFrac of the work is cut
    // into chunks of ~kDynChunk full panels that free CTAs take from a work
    // counter (SM bandwidth shares vary by ~10%; a static split waits for the
    // slowest SM).
    const bool dyn = L.tma && npanels >= static_cast<int64_t>(L.ncta) * 64;
    static const char* df_env = dev_env("R1_SWEEP_DYN_FRAC");  // development
    const double dyn_frac = df_env ? std::atof(df_env) : kDynFrac;
    const double static_total = dyn ? (1.0 - dyn_frac) * total : total;
    const double full_cost = static_cast<double>(L.r0) * L.t1 + 512.0;
    const double per = static_total / static_cast<double>(L.ncta);
    int cur = 0;          // CTA receiving the current panel
    int seg_cta = -1;     // CTA owning segs.back() (-1: dynamic chunk)
    double x = 0.0;       // cost of all earlier panels
    double chunk = 0.0;   // cost of the open dynamic chunk
    bool in_dyn = false;
    for (int t = 0; t < L.ntiles; ++t) {
        const double c = panel_cost(t);
        for (int64_t o = 0; o < Og; ++o) {
            if (!in_dyn && dyn && x + 0.5 * c >= static_total) {
                in_dyn = true;
                while (cur < L.ncta) cta_seg[++cur] = static_cast<int>(segs.size());
                L.dyn_first = static_cast<int>(segs.size());
            }
            if (in_dyn) {
                // guided chunk size: remaining / (2 ncta), at least kDynMinChunk panels
                static const char* mc_env = dev_env("R1_SWEEP_DYN_CHUNK");  // development
                const double min_chunk = mc_env ? std::atof(mc_env) : kDynMinChunk;
                const double target = std::max(min_chunk * full_cost,
                                               (total - x) / (2.0 * L.ncta));
                if (segs.size() == static_cast<size_t>(L.dyn_first) || segs.back().tile != t ||
                    segs.back().o1 != o || chunk >= target) {
                    segs.push_back(Seg{t, static_cast<int>(o), static_cast<int>(o + 1), 0});
                    chunk = 0.0;
                } else {
                    segs.back().o1 = static_cast<int>(o + 1);
                }
                chunk += c;
                x += c;
                continue;
            }
            const int target = std::min<int>(
                L.ncta - 1, static_cast<int>((x + 0.5 * c) / per));
            while (cur < target) cta_seg[++cur] = static_cast<int>(segs.size());
            if (segs.empty() || segs.back().tile != t || seg_cta != cur ||
                segs.back().o1 != o)
                segs.push_back(Seg{t, static_cast<int>(o), static_cast<int>(o + 1), 0});
            else
                segs.back().o1 = static_cast<int>(o + 1);
            seg_cta = cur;
            x += c;
        }
    }
    if (!in_dyn) {
        while (cur < L.ncta) cta_seg[++cur] = static_cast<int>(segs.size());
        L.dyn_first = static_cast<int>(segs.size());
    }
    L.ndyn = static_cast<int>(segs.size()) - L.dyn_first;
    L.nseg = static_cast<int>(segs.size());
    std::vector<int> tile_seg(L.ntiles + 1, 0);
    {
        int k = 0;
        for (int t = 0; t < L.ntiles; ++t) {
            tile_seg[t] = k;
            while (k < L.nseg && segs[k].tile == t) ++k;
        }
        tile_seg[L.ntiles] = L.nseg;
    }
    auto align4 = [&]() {
        while (meta.size() % 4) meta.push_back(0);
    };
    align4();
    L.seg_off = meta.size();
    for (const Seg& s : segs) {
        meta.push_back(s.tile);
        meta.push_back(s.o0);
        meta.push_back(s.o1);
        meta.push_back(0);
    }
    L.cta_off = meta.size();
    meta.insert(meta.end(), cta_seg.begin(), cta_seg.end());
    L.tile_off = meta.size();
    meta.insert(meta.end(), tile_seg.begin(), tile_seg.end());
}

// Recursively lay out the levels for a sub-problem of order `order` (>= 3).
// need_all: also produce the blocks among modes >= 2 of this sub-problem.
void plan_rec(SweepPlan& P, const uint64_t* full_dims, int full_order, int order,
              const int64_t* dims, const int* modes, Ref input, bool need_all, int num_sms,
              int lane = 0, int depth = 0, bool chain_head = false) {
    Level L;
    L.lane = lane;
    L.depth = depth;
    L.chain_head = chain_head;
    L.order = order;
    for (int k = 0; k < order; ++k) {
        L.dims[k] = dims[k];
        L.modes[k] = modes[k];
    }
    L.input = input;
    L.I0 = dims[0];
    L.I1 = dims[1];
    L.O = 1;
    for (int k = 2; k < order; ++k) L.O *= dims[k];
    tile_level(L, num_sms);
    partition_level(L, num_sms, P.host_meta);

    auto final_ref = [&](int a, int b) {
        return Ref{Where::Final, block_offset(full_dims, full_order, modes[a], modes[b])};
    };
    auto work = [&](uint64_t n) {
        Ref r{Where::Work, P.work_elems};
        P.work_elems += (n + 31) & ~uint64_t(31);
        return r;
    };
    L.out_b01 = final_ref(0, 1);
    const bool need_c1 = need_all;
    if (order == 3) {
        L.out_c0 = final_ref(0, 2);
        L.out_c1 = need_c1 ? final_ref(1, 2) : Ref{};
    } else {
        L.out_c0 = work(static_cast<uint64_t>(L.I0 * L.O));
        L.out_c1 = need_c1 ? work(static_cast<uint64_t>(L.I1 * L.O)) : Ref{};
    }
    L.w = work(static_cast<uint64_t>(L.O));
    L.p01 = work(static_cast<uint64_t>(L.nseg) * L.r0 * L.t1);
    // C0 / C1 partials per column / row tile (merged rows for C0), summed by
    // the second stage; written in place when there is a single tile and class
    L.p0 = (L.G1 > 1 || L.K > 1) ? work(static_cast<uint64_t>(L.G1) * L.MI0 * L.O) : L.out_c0;
    if (need_c1)
        L.p1 = (L.G0 > 1 || L.K > 1) ? work(static_cast<uint64_t>(L.G0) * L.I1 * L.O) : L.out_c1;
    P.levels.push_back(L);

    if (order >= 4) {
        // C0: modes (0, 2, 3, ...) — all of its blocks are blocks of A (if need_all),
        // else only its (0,k) blocks.
        int64_t d0[kMaxOrder];
        int m0[kMaxOrder];
        d0[0] = dims[0];
        m0[0] = modes[0];
        for (int k = 2; k < order; ++k) {
            d0[k - 1] = dims[k];
            m0[k - 1] = modes[k];
        }
        const Ref c0 = L.out_c0, c1 = L.out_c1;
        // the C0 child continues its parent's lane (the spine: depth + 1; a chain: same depth)
        plan_rec(P, full_dims, full_order, order - 1, d0, m0, c0, need_all, num_sms, lane,
                 need_all ? depth + 1 : depth, false);
        if (need_c1) {
            d0[0] = dims[1];
            m0[0] = modes[1];
            // a spine level's C1 subtree shares nothing with its C0 subtree
            // (disjoint work regions, disjoint final blocks): its own lane
            plan_rec(P, full_dims, full_order, order - 1, d0, m0, c1, false, num_sms, 1 + depth % 3, depth,
                     true);
        }
    }
}

std::shared_ptr<SweepPlan> get_plan(r1_context* ctx, const uint64_t* dims, int order) {
    std::vector<uint64_t> key(dims, dims + order);
    auto it = ctx->plans.find(key);
    if (it != ctx->plans.end()) return it->second;
    auto P = std::make_shared<SweepPlan>();
    P->dims = key;
    P->nblocks = blocks_numel(dims, order);
    int64_t d[kMaxOrder];
    int m[kMaxOrder];
    for (int k = 0; k < order; ++k) {
        d[k] = static_cast<int64_t>(dims[k]);
        m[k] = k;
    }
    plan_rec(*P, dims, order, order, d, m, Ref{Where::Tensor, 0}, true, ctx->num_sms);
    P->meta.ensure(std::max<size_t>(16, P->host_meta.size() * sizeof(int)));
    P->counters.ensure(std::max<size_t>(1, P->levels.size()) * 64);
    upload_now(ctx, P->meta.ptr, P->host_meta.data(), P->host_meta.size() * sizeof(int));
    R1_CUDA(cudaMemsetAsync(P->counters.ptr, 0, std::max<size_t>(1, P->levels.size()) * 64, ctx->stream));
    ctx->plans[key] = P;
    return P;
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        R1_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess)
            fail(R1_ERR_CUDA, "cuTensorMapEncodeTiled is not available from the driver");
        fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// 3-D map over the view A[i0, i1, o] (fp64, no swizzle, zero OOB fill).
CUtensorMap make_map(const double* A, const Level& L, int64_t box_rows, int64_t box_cols,
                     int64_t box_depth = 1) {
    CUtensorMap m;
    std::memset(&m, 0, sizeof(m));
    const cuuint64_t gdim[3] = {static_cast<cuuint64_t>(L.MI0), static_cast<cuuint64_t>(L.MI1),
                                static_cast<cuuint64_t>(L.O)};
    const cuuint64_t gstride[2] = {static_cast<cuuint64_t>(L.MI0) * 8,
                                   static_cast<cuuint64_t>(L.I0) * L.I1 * 8};
    const cuuint32_t box[3] = {static_cast<cuuint32_t>(box_rows), static_cast<cuuint32_t>(box_cols),
                               static_cast<cuuint32_t>(box_depth)};
    const cuuint32_t estride[3] = {1, 1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(A), gdim,
                             gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(R1_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return m;
}

// Launch a sweep kernel as a programmatic dependent of the preceding kernel
// (the kernels call griddepcontrol.wait before touching global memory).
template <typename... KArgs, typename... Args>
void launch_pdl(r1_context* ctx, void (*kern)(KArgs...), int grid, int block, size_t smem,
                cudaStream_t stream, Args&&... args) {
    static const char* env = dev_env("R1_SWEEP_PDL");  // development: 0 = plain stream order
    static const bool pdl = !(env && std::atoi(env) == 0);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(static_cast<unsigned>(block));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    R1_CUDA(cudaLaunchKernelEx(&cfg, kern, KArgs(std::forward<Args>(args))...));
    (void)ctx;
}

template <int NRA, int NCB, int STAGES, bool TMA>
void launch_sweep_t(r1_context* ctx, const Level& L, const SweepArgs& a, const CUtensorMap& m) {
    auto kern = sweep3_kernel<NRA, NCB, STAGES, TMA>;
    // L.smem never exceeds kSmemBudget: set the maximum once per device
    configure_once(reinterpret_cast<const void*>(kern), ctx->device, [&] {
        R1_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(kSmemBudget)));
    });
    launch_pdl(ctx, kern, L.ncta, kThreads, L.smem, ctx->stream, a, m);
    check_launch(ctx, "sweep3_kernel");
}

template <int NRA, bool SR, int KO, int NCB = kBoxNCB, int NWC = kBoxNWC, int NS = 1>
void launch_box(r1_context* ctx, const Level& L, const SweepArgs& a) {
    auto kern = sweep3_box_kernel<NRA, NCB, NWC, SR, KO, NS>;
    configure_once(reinterpret_cast<const void*>(kern), ctx->device, [&] {
        R1_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(kSmemBudget)));
    });
    BoxMaps maps;
    const int64_t rem0 = L.MI0 - static_cast<int64_t>(L.G0 - 1) * L.r0;
    const int64_t rem1 = L.MI1 - static_cast<int64_t>(L.G1 - 1) * L.t1;
    // boxes are ts columns wide; the last box of the last column tile is narrower
    const int64_t remlast = rem1 - ((rem1 + L.ts - 1) / L.ts - 1) * L.ts;
    maps.m[0] = make_map(a.A, L, L.r0, L.ts, KO);
    maps.m[1] = make_map(a.A, L, rem0, L.ts, KO);
    maps.m[2] = make_map(a.A, L, L.r0, remlast, KO);
    maps.m[3] = make_map(a.A, L, rem0, remlast, KO);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    const bool timed = ctx->time_kernels && a.trace_level0;
    if (timed) {
        R1_CUDA(cudaEventCreate(&e0));
        R1_CUDA(cudaEventCreate(&e1));
        R1_CUDA(cudaEventRecord(e0, ctx->stream));
    }
    launch_pdl(ctx, kern, L.ncta, (NWC + 1) * 32, L.smem, ctx->stream, a, maps, L.stages, L.stage_dbl);
    check_launch(ctx, "sweep3_box_kernel");
    if (timed) {
        R1_CUDA(cudaEventRecord(e1, ctx->stream));
        ctx->kernel_events.emplace_back(e0, e1);
    }
}

template <int NRA, int NCB, int STAGES>
void launch_sweep(r1_context* ctx, const Level& L, const SweepArgs& a) {
    if (L.tma) {
        static const char* sr = dev_env("R1_SWEEP_STAGE_REGS");
        const bool stage_regs = sr ? std::atoi(sr) != 0 : true;
        if (L.nra == 8 && L.nwc == 11) {
            launch_box<8, false, 1, 4, 11>(ctx, L, a);
        } else if (L.nra == 2 && L.nwc == 8) {
            if (L.KO == 2) launch_box<2, false, 2, 8, 8>(ctx, L, a);
            else launch_box<2, false, 1, 8, 8>(ctx, L, a);
        } else if (L.nra == 8) {
            if (stage_regs) launch_box<8, true, 1, 2>(ctx, L, a);
            else launch_box<8, false, 1, 2>(ctx, L, a);
        } else if (L.nra == 4 && L.nwc == 7 && L.ns > 1) {
            launch_box<4, true, 1, 8, 7, 4>(ctx, L, a);
        } else if (L.nra == 4 && L.nwc == 7) {
            if (stage_regs) launch_box<4, true, 1, 8, 7>(ctx, L, a);
            else launch_box<4, false, 1, 8, 7>(ctx, L, a);
        } else if (L.nra == 4) {
            if (stage_regs) launch_box<4, true, 1>(ctx, L, a);
            else launch_box<4, false, 1>(ctx, L, a);
        } else if (L.KO == 4) {
            if (stage_regs) launch_box<2, true, 4>(ctx, L, a);
            else launch_box<2, false, 4>(ctx, L, a);
        } else if (L.KO == 2) {
            if (stage_regs) launch_box<2, true, 2>(ctx, L, a);
            else launch_box<2, false, 2>(ctx, L, a);
        } else {
            if (stage_regs) launch_box<2, true, 1>(ctx, L, a);
            else launch_box<2, false, 1>(ctx, L, a);
        }
    } else {
        CUtensorMap m;
        std::memset(&m, 0, sizeof(m));
        launch_sweep_t<NRA, NCB, STAGES, false>(ctx, L, a, m);
    }
}

int grid_for(int64_t n, int threads, int num_sms) {
    const int64_t g = (n + threads - 1) / threads;
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(g, int64_t(num_sms) * 8)));
}

}  // namespace

void sweep_blocks(r1_context* ctx, const double* a, const uint64_t* dims, int order,
                  const double* factors_dev, double* blocks_dev, const double* last_factor) {
    if (order < 2 || order > kMaxOrder) fail(R1_ERR_INVALID_ARGUMENT, "sweep: unsupported order");
    const uint64_t n = numel_of(dims, order);
    if (order == 2) {
        // Nothing to contract: the block is the tensor itself (nepv.cpp:49-53).
        R1_CUDA(cudaMemcpyAsync(blocks_dev, a, n * sizeof(double), cudaMemcpyDeviceToDevice,
                                ctx->stream));
        return;
    }
    auto P = get_plan(ctx, dims, order);
    ctx->ws_sweep.ensure(std::max<uint64_t>(P->work_elems, 32) * sizeof(double));
    double* work = ctx->ws_sweep.as<double>();
    const int* meta = P->meta.as<int>();
    uint64_t foff[kMaxOrder + 1];
    foff[0] = 0;
    for (int k = 0; k < order; ++k) foff[k + 1] = foff[k] + dims[k];
    // factor of mode k; a slab of a sharded tensor reads its slice of the
    // global last factor in place (last_factor)
    auto fac = [&](int k) -> const double* {
        return (k == order - 1 && last_factor) ? last_factor : factors_dev + foff[k];
    };

    auto resolve = [&](const Ref& r) -> double* {
        switch (r.where) {
            case Where::Tensor: return const_cast<double*>(a);
            case Where::Final: return blocks_dev + r.off;
            case Where::Work: return work + r.off;
            default: return nullptr;
        }
    };

    // (the dynamic-tail counters are zeroed at plan creation and re-armed by the
    // box kernel itself)
    // Lanes.  The children of a level need only its C0 / C1, not B01, and its two
    // subtrees are independent: the root's B01 second stage and every spine
    // level's C1 chain (Level::lane) run on side streams beside the spine (C4:
    // 18 small kernels of ~190 us in a chain become chains of <= ~60 us).
    // Forked with events after the producing level's second stage, joined at
    // the end — inside a stream capture the side streams join the capture the
    // same way.
    static const char* fork_env = dev_env("R1_SWEEP_FORK");
    // 0 never, 1 tensors of >= 2^22 elements only, 2 (default) whenever the plan has chains:
    // small high-order tensors gain the most (16^5 76 -> 55 us, 40^4 38 -> 31 us, 10^6 143 -> 111 us)
    const int fork_mode = fork_env ? std::atoi(fork_env) : 2;
    const Level& root = P->levels.front();
    const bool root_seg = root.nseg >= 64 * root.ntiles;
    const bool fork = ctx->side_stream && fork_mode != 0 && (fork_mode == 2 || n >= (uint64_t(1) << 22)) &&
                      P->levels.size() > 1;
    cudaStream_t const main_stream = ctx->stream;
    struct StreamGuard {
        r1_context* c;
        cudaStream_t s;
        ~StreamGuard() { c->stream = s; }
    } guard{ctx, main_stream};
    bool lane_used[4] = {true, false, false, false};
    int level_idx = 0;
    for (const Level& L : P->levels) {
        const int lane = fork ? L.lane : 0;
        cudaStream_t const lane_stream = lane == 0 ? main_stream : ctx->side_streams[lane - 1];
        if (lane != 0 && L.chain_head) {
            R1_CUDA(cudaStreamWaitEvent(lane_stream, ctx->ev_done[L.depth], 0));
            lane_used[lane] = true;
        }
        ctx->stream = lane_stream;
        const bool is_root = &L == &root;
        // outer weights
        OuterArgs oa{};
        oa.nout = L.order - 2;
        for (int k = 2; k < L.order; ++k) {
            oa.dims[k - 2] = L.dims[k];
            oa.u[k - 2] = fac(L.modes[k]);
        }
        oa.O = L.O;
        oa.W = resolve(L.w);
        const double* Wsrc = oa.W;
        if (oa.nout == 1) {
            Wsrc = oa.u[0];  // order 3: the outer weights are u_2 itself
        } else {
            launch_pdl(ctx, outer_weights_kernel, grid_for(L.O, 256, ctx->num_sms), 256, 0, ctx->stream, oa);
            check_launch(ctx, "outer_weights_kernel");
        }

        SweepArgs s{};
        s.A = resolve(L.input);
        s.I0 = L.I0;
        s.I1 = L.I1;
        s.O = L.O;
        s.K = L.K;
        s.MI0 = L.MI0;
        s.MI1 = L.MI1;
        s.u0 = fac(L.modes[0]);
        s.u1 = fac(L.modes[1]);
        s.W = Wsrc;
        s.r0 = L.r0;
        s.t1 = L.t1;
        s.ts = L.ts > 0 ? L.ts : L.t1;
        s.G0 = L.G0;
        s.rbox = L.r0;
        s.segs = reinterpret_cast<const Seg*>(meta + L.seg_off);
        s.cta_seg = meta + L.cta_off;
        s.P01 = resolve(L.p01);
        s.P0 = resolve(L.p0);
        s.P0_stride = L.MI0 * L.O;
        s.P1 = L.out_c1.where == Where::None ? nullptr : resolve(L.p1);
        s.P1_stride = L.I1 * L.O;
        s.trace = (&L == &P->levels.front()) ? ctx->dbg_sweep_trace : nullptr;
        s.trace_level0 = (&L == &P->levels.front()) ? 1 : 0;
        s.dyn_first = L.dyn_first;
        s.ndyn = L.ndyn;
        s.dyn_counter = reinterpret_cast<int*>(P->counters.as<char>() + 64 * level_idx);
        ++level_idx;
        {
            static const char* dm = dev_env("R1_DEBUG_SWEEP_MODE");
            s.debug_mode = dm ? std::atoi(dm) : 0;
        }
        if (L.nra == 4 || L.nra == 8)  // (nra 8: box kernel only)
            launch_sweep<4, 8, 3>(ctx, L, s);
        else if (L.nra == 2)
            launch_sweep<2, 8, 5>(ctx, L, s);
        else
            launch_sweep<1, 8, 8>(ctx, L, s);

        // second stage: fixed-order partial sums, one launch
        FinishArgs f{};
        f.P01 = s.P01;
        f.tile_seg = meta + L.tile_off;
        f.I0 = L.I0;
        f.I1 = L.I1;
        f.O = L.O;
        f.MI1 = L.MI1;
        f.K = L.K;
        f.lgK = 0;
        while ((1 << f.lgK) < L.K) ++f.lgK;
        f.r0 = L.r0;
        f.t1 = L.t1;
        f.G0 = L.G0;
        f.G1 = L.G1;
        f.b01 = resolve(L.out_b01);
        if (L.G1 > 1 || L.K > 1) {
            f.P0 = s.P0;
            f.stride0 = s.P0_stride;
            f.c0 = resolve(L.out_c0);
            f.n_c0 = L.I0 * L.O;
        }
        if (s.P1 && (L.G0 > 1 || L.K > 1)) {
            f.P1 = s.P1;
            f.stride1 = s.P1_stride;
            f.c1 = resolve(L.out_c1);
            f.n_c1 = L.I1 * L.O;
        }
        f.n_b01 = L.I0 * L.I1;
        fastdiv_init(L.I0, f.m_I0, f.s_I0);
        fastdiv_init(L.I1, f.m_I1, f.s_I1);
        fastdiv_init(L.r0, f.m_r0, f.s_r0);
        fastdiv_init(L.t1, f.m_t1, f.s_t1);
        // a spine level's C1 chain waits for its C0 / C1 only (recorded below)
        auto root_outputs_done = [&]() {
            if (fork && L.lane == 0 && L.order >= 4) R1_CUDA(cudaEventRecord(ctx->ev_done[L.depth], main_stream));
        };
        if (L.nseg >= 64 * L.ntiles) {
            // many segments per tile: B01 by segment slices, C0/C1 (if any) below
            const int64_t units = static_cast<int64_t>(L.ntiles) * ((static_cast<int64_t>(L.r0) * L.t1 + 31) / 32);
            const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(units, int64_t(4) * ctx->num_sms)));
            cudaStream_t bs = ctx->stream;
            if (is_root && fork) {
                R1_CUDA(cudaEventRecord(ctx->ev_sweep[0], main_stream));
                R1_CUDA(cudaStreamWaitEvent(ctx->side_stream, ctx->ev_sweep[0], 0));
                bs = ctx->side_stream;
                lane_used[1] = true;
            }
            launch_pdl(ctx, finish_b01_seg_kernel, grid, kB01Warps * 32, 0, bs, f);
            check_launch(ctx, "finish_b01_seg_kernel");
            f.b01 = nullptr;
            f.n_b01 = 0;
            if (f.n_c0 + f.n_c1 == 0) {
                root_outputs_done();
                continue;
            }
        }
        {
            const int64_t total = f.n_b01 + f.n_c0 + f.n_c1;
            const int grid = static_cast<int>(
                std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, int64_t(32) * ctx->num_sms)));
            // 32-bit indices only while the grid-stride loop cannot step past
            // 2^31 (e + gridDim.x * 256 must stay representable)
            if (total + static_cast<int64_t>(grid) * 256 < (int64_t(1) << 31))
                launch_pdl(ctx, finish_kernel<int>, grid, 256, 0, ctx->stream, f);
            else
                launch_pdl(ctx, finish_kernel<int64_t>, grid, 256, 0, ctx->stream, f);
        }
        check_launch(ctx, "finish_kernel");
        root_outputs_done();
    }
    ctx->stream = main_stream;
    for (int l = 1; l < 4; ++l)
        if (lane_used[l]) {
            R1_CUDA(cudaEventRecord(ctx->ev_join[l - 1], ctx->side_streams[l - 1]));
            R1_CUDA(cudaStreamWaitEvent(main_stream, ctx->ev_join[l - 1], 0));
        }
}

// Introspection for tests / DESIGN.md: the plan of the top level.
void sweep_plan_info(r1_context* ctx, const uint64_t* dims, int order, int64_t* info) {
    auto P = get_plan(ctx, dims, order);
    const Level& L = P->levels.front();
    info[0] = L.r0;
    info[1] = L.t1;
    info[2] = L.G0;
    info[3] = L.G1;
    info[4] = L.ncta;
    info[5] = L.nseg;
    info[6] = static_cast<int64_t>(P->levels.size());
    info[7] = static_cast<int64_t>(P->work_elems);
    info[8] = static_cast<int64_t>(L.smem);
    info[9] = L.nra;
    info[10] = L.K;
    info[11] = L.KO;
    info[12] = L.ndyn;
    info[13] = L.ns;
    info[14] = L.ts;
}

}  // namespace r1
