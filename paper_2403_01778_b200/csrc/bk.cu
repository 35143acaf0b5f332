// Bunch-Kaufman LDL^T (lower) of a dense symmetric matrix, hand-written for
// the iHOSCF Rayleigh-quotient step (reference proj/src/sym_eig.cpp:233-438:
// ldlt_factor, ldlt_solve, ldlt_diag_condition, rayleigh_quotient_step).
//
// Same pivot rule as the reference's unblocked factorisation (alpha =
// (1+sqrt17)/8; 1x1 without interchange, 1x1 with k <-> imax, 2x2 with
// k+1 <-> imax; ties to the first index; zero column -> singular), blocked the
// LAPACK dlasyf way so the O(n^3) work runs on all SMs:
//   * panel kernel (ONE thread-block cluster of <= 16 CTAs, rows split across
//     the CTAs, W / updated columns / raw columns in shared memory): for each
//     of <= 32 (+1 when a 2x2 pivot straddles the edge) columns, form the
//     updated column from the stored matrix minus the panel's delayed update
//     (W = unscaled pivot columns, L), find colmax / rowmax across the
//     cluster, pick the pivot, apply the symmetric interchange, eliminate.
//     Cross-CTA data moves as st.async messages counted on mbarriers (no
//     cluster barrier inside the column loop; bk_panel_smem_kernel);
//     bk_panel_kernel is the global-memory fallback for panels that do not
//     fit in shared memory;
//   * trailing update (all SMs): A22 -= W L^T on the lower triangle on the
//     FP64 tensor cores (bk_update_tc_kernel);
//   * solve (bk_solve_cluster_kernel: one cluster, z in shared memory, each
//     panel's interchanges composed once by bk_perm_kernel; bk_solve_kernel
//     is the cooperative-grid fallback).
// D, the pivot sequence and the solution are the reference's (its accept test
// only reads D).  Interchanges are applied to the rows of the CURRENT panel's
// L only, so each panel's L is stored in the row order at the end of that
// panel (the blocked LAPACK convention); the solve applies them panel by
// panel: forward (P_p, L_p), D^-1, backward (L_p^T, P_p^T).
#include "common.cuh"
#include "dsmem.cuh"

#include <cooperative_groups.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

namespace cg = cooperative_groups;

namespace r1 {

namespace {

constexpr int kBkNb = 32;          // panel columns (a 2x2 pivot may add one)
constexpr int kBkW = kBkNb + 1;    // columns of the panel workspace
constexpr int kBkThreads = 256;
constexpr int kBkSolveB = 64;      // substitution block
constexpr double kBkAlpha = 0.6403882032022076;  // (1 + sqrt(17)) / 8

struct BkArgs {
    int64_t n;
    double* A;    // n x n column-major: lower triangle in, L and D out
    double* Wp;   // n x kBkW panel workspace
    int* ipiv;    // >= 0: 1x1 with interchange k <-> ipiv; < 0: 2x2 (both columns) with k+1 <-> -ipiv-1
    int* ctl;     // [0] next panel start, [1] singular, [2] last panel start, [3] last panel width
    double* Ck;   // updated column k
    double* Ci;   // updated column imax
    double* red;  // 4 * gridDim partials
    int* perm;    // panel start columns (ctl[4] of them), for the panel-wise solve
    char* ps;     // 0: 1x1 pivot, 1 / 2: first / second column of a 2x2 pivot
    unsigned long long* trace;  // diagnostics: per-phase cycle sums of CTA trace_cta, or null
    int trace_cta;
};

// Workspace layout (bytes from bk_workspace_bytes).
struct BkLayout {
    double *Wp, *Ck, *Ci, *red, *part, *z;
    int *ctl, *ipiv, *perm;
    char* ps;
    int* pperm;  // per panel: composed interchanges for the cluster solve
};

// Per-panel record of the cluster solve: [0] number of rows >= the panel end
// touched by its interchanges, [1] / [2] bit mask (low / high word) of the
// panel's first-of-2x2 columns, then those rows, then the slot permutations
// of the forward (P) and backward (P^T) application.
constexpr int kPermStride = 4 + kBkW + 4 * kBkW;
inline int64_t max_panels(int64_t n) { return n / kBkNb + 2; }

BkLayout bk_layout(void* ws, int64_t n, int num_sms) {
    BkLayout L;
    double* d = static_cast<double*>(ws);
    auto take = [&](int64_t k) {
        double* p = d;
        d += (k + 7) & ~int64_t(7);
        return p;
    };
    L.Wp = take(n * kBkW);
    L.Ck = take(n);
    L.Ci = take(n);
    L.z = take(n);
    L.red = take(4 * 64 + 8);
    L.part = take(static_cast<int64_t>(num_sms) * kBkSolveB + 8);
    int* i = reinterpret_cast<int*>(d);
    L.ctl = i;
    L.ipiv = i + 16;
    L.perm = L.ipiv + n + 16;
    L.ps = reinterpret_cast<char*>(L.perm + n + 16);
    L.pperm = reinterpret_cast<int*>(L.ps + ((n + 64 + 15) & ~int64_t(15)));
    return L;
}

__global__ void bk_init_kernel(int* perm, char* ps, int64_t n) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        perm[i] = static_cast<int>(i);
        ps[i] = 0;
    }
}

// Programmatic dependent launch: a kernel launched with the programmatic
// stream-serialisation attribute may start while its predecessor runs; it
// lets its own dependents launch at once and waits for the predecessor's
// completion (and memory flush) before touching any data.
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

__device__ __forceinline__ void argmax_merge(double& v, int64_t& i, double v2, int64_t i2) {
    if (v2 > v || (v2 == v && i2 < i)) {
        v = v2;
        i = i2;
    }
}

// block-wide (value, index) arg-max; result valid in thread 0
__device__ void block_argmax(double& v, int64_t& i, double* sv, int64_t* si) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, v, off);
        const int64_t i2 = __shfl_xor_sync(0xffffffffu, i, off);
        argmax_merge(v, i, v2, i2);
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) {
        sv[warp] = v;
        si[warp] = i;
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) argmax_merge(v, i, sv[w], si[w]);
}

// The whole grid is ONE thread-block cluster: the per-column barriers are
// hardware cluster barriers (release/acquire at cluster scope), not grid syncs.
__global__ void __launch_bounds__(kBkThreads) bk_panel_kernel(const BkArgs a) {
    cg::cluster_group grid = cg::this_cluster();
    __shared__ double sv[32];
    __shared__ int64_t si[32];
    __shared__ double Lr[kBkW];  // row k (then imax) of the panel's L columns
    pdl_enter();
    const int64_t n = a.n;
    const int64_t k0 = a.ctl[0];
    if (k0 >= n) return;
    const int G = gridDim.x;
    const int64_t chunk = (n - k0 + G - 1) / G;
    const int64_t lo = k0 + chunk * blockIdx.x, hi = min(n, lo + chunk);
    const int64_t gtid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int64_t gthreads = static_cast<int64_t>(G) * blockDim.x;
    double* A = a.A;
    double* Wp = a.Wp;

    int64_t k = k0;
    int jp = 0;
    while (k < n && jp < kBkNb) {
        // ---- updated column k (rows >= k) and its arg-max below the diagonal
        double bv = -1.0;
        int64_t bi = n;
        if (threadIdx.x < jp) Lr[threadIdx.x] = A[k + (k0 + threadIdx.x) * n];
        __syncthreads();
        for (int64_t i = max(lo, k) + threadIdx.x; i < hi; i += blockDim.x) {
            double s = A[i + k * n];
            for (int t = 0; t < jp; ++t) s -= Wp[i + t * n] * Lr[t];
            a.Ck[i] = s;
            if (i > k) argmax_merge(bv, bi, fabs(s), i);
        }
        block_argmax(bv, bi, sv, si);
        if (threadIdx.x == 0) {
            a.red[2 * blockIdx.x] = bv;
            a.red[2 * blockIdx.x + 1] = static_cast<double>(bi);
        }
        grid.sync();
        double colmax = -1.0;
        int64_t imax = n;
        for (int c = 0; c < G; ++c)
            argmax_merge(colmax, imax, a.red[2 * c], static_cast<int64_t>(a.red[2 * c + 1]));
        if (colmax < 0.0) {
            colmax = 0.0;
            imax = k;
        }
        const double absakk = fabs(a.Ck[k]);
        int kstep = 1;
        int64_t kp = k;
        if (fmax(absakk, colmax) == 0.0) {
            // zero column (sym_eig.cpp:253-258): singular, no elimination
            for (int64_t i = max(lo, k) + threadIdx.x; i < hi; i += blockDim.x) {
                A[i + k * n] = a.Ck[i];
                Wp[i + jp * n] = 0.0;
            }
            if (gtid == 0) {
                a.ipiv[k] = static_cast<int>(k);
                a.ps[k] = 0;
                a.ctl[1] = 1;
            }
            k += 1;
            jp += 1;
            grid.sync();
            continue;
        }
        if (!(absakk >= kBkAlpha * colmax)) {
            // updated column imax (sym_eig.cpp:263-275)
            double rv = -1.0;
            __syncthreads();
            if (threadIdx.x < jp) Lr[threadIdx.x] = A[imax + (k0 + threadIdx.x) * n];
            __syncthreads();
            for (int64_t i = max(lo, k) + threadIdx.x; i < hi; i += blockDim.x) {
                double s = i >= imax ? A[i + imax * n] : A[imax + i * n];
                for (int t = 0; t < jp; ++t) s -= Wp[i + t * n] * Lr[t];
                a.Ci[i] = s;
                if (i != imax) rv = fmax(rv, fabs(s));
            }
            int64_t dummy = 0;
            block_argmax(rv, dummy, sv, si);
            if (threadIdx.x == 0) a.red[2 * G + blockIdx.x] = rv;
            grid.sync();
            double rowmax = 0.0;
            for (int c = 0; c < G; ++c) rowmax = fmax(rowmax, a.red[2 * G + c]);
            if (absakk * rowmax >= kBkAlpha * colmax * colmax) {
                kp = k;
            } else if (fabs(a.Ci[imax]) >= kBkAlpha * rowmax) {
                kp = imax;
            } else {
                kp = imax;
                kstep = 2;
            }
        }
        const int64_t kk = k + kstep - 1;
        const bool swap = kp != kk;
        // symmetric interchange kk <-> kp.  Column kk is rewritten below, so
        // its stored entries only move out (to column kp, row kp, diagonal);
        // the owner of each row moves its entry before overwriting it.
        auto move_out = [&](int64_t i) {
            if (!swap) return;
            if (i > kp) A[i + kp * n] = A[i + kk * n];
            else if (i > kk && i < kp) A[kp + i * n] = A[i + kk * n];
            else if (i == kk) A[kp + kp * n] = A[kk + kk * n];
        };
        if (swap) {
            // rows of this panel's L columns (earlier panels keep their order:
            // the solve applies the interchanges panel by panel) and of W
            for (int64_t t = k0 + gtid; t < k; t += gthreads) {
                const double u = A[kk + t * n];
                A[kk + t * n] = A[kp + t * n];
                A[kp + t * n] = u;
            }
            for (int64_t t = gtid; t < jp; t += gthreads) {
                const double u = Wp[kk + t * n];
                Wp[kk + t * n] = Wp[kp + t * n];
                Wp[kp + t * n] = u;
            }
        }
        if (kstep == 1) {
            const double d = kp == k ? a.Ck[k] : a.Ci[kp];
            const bool zero = d == 0.0;
            const double r1 = zero ? 0.0 : 1.0 / d;
            for (int64_t i = max(lo, k) + threadIdx.x; i < hi; i += blockDim.x) {
                const double v = kp == k ? a.Ck[i] : (i == k ? a.Ci[kp] : (i == kp ? a.Ci[k] : a.Ci[i]));
                move_out(i);
                if (i == k) {
                    A[k + k * n] = d;
                    Wp[k + jp * n] = zero ? 0.0 : d;
                } else {
                    Wp[i + jp * n] = zero ? 0.0 : v;  // dkk == 0: no elimination (sym_eig.cpp:288-290)
                    A[i + k * n] = zero ? v : v * r1;
                }
            }
            if (gtid == 0) {
                a.ipiv[k] = static_cast<int>(kp);
                a.ps[k] = 0;
                if (zero) a.ctl[1] = 1;
            }
        } else {
            auto nk = [&](int64_t i) {
                return kp == k + 1 ? a.Ck[i] : (i == k + 1 ? a.Ck[kp] : (i == kp ? a.Ck[k + 1] : a.Ck[i]));
            };
            auto nk1 = [&](int64_t i) {
                return kp == k + 1 ? a.Ci[i] : (i == k + 1 ? a.Ci[kp] : (i == kp ? a.Ci[k + 1] : a.Ci[i]));
            };
            // sym_eig.cpp:298-313
            const double d21 = nk(k + 1);
            const double d11 = nk1(k + 1) / d21;
            const double d22 = nk(k) / d21;
            const double tt = 1.0 / (d11 * d22 - 1.0);
            const double d21t = tt / d21;
            for (int64_t i = max(lo, k) + threadIdx.x; i < hi; i += blockDim.x) {
                const double x0 = nk(i), x1 = nk1(i);
                move_out(i);
                Wp[i + jp * n] = x0;
                Wp[i + (jp + 1) * n] = x1;
                if (i == k) {
                    A[k + k * n] = x0;
                } else if (i == k + 1) {
                    A[k + 1 + k * n] = x0;  // = d21
                    A[k + 1 + (k + 1) * n] = x1;
                } else {
                    A[i + k * n] = d21t * (d11 * x0 - x1);
                    A[i + (k + 1) * n] = d21t * (d22 * x1 - x0);
                }
            }
            if (gtid == 0) {
                a.ipiv[k] = static_cast<int>(-kp - 1);
                a.ipiv[k + 1] = static_cast<int>(-kp - 1);
                a.ps[k] = 1;
                a.ps[k + 1] = 2;
            }
        }
        k += kstep;
        jp += kstep;
        grid.sync();
    }
    if (gtid == 0) {
        a.perm[a.ctl[4]] = static_cast<int>(k0);  // panel starts, for the solve
        a.ctl[4] += 1;
        a.ctl[2] = static_cast<int>(k0);
        a.ctl[3] = jp;
        a.ctl[0] = static_cast<int>(k);
    }
}

// Panel kernel with the CTA's rows of W, of the two updated columns and of the
// raw stored columns k, k+1 held in shared memory (used when they fit).
//
// No cluster barrier inside the column loop: every value another CTA needs is
// PUSHED into that CTA's shared memory with st.async, which counts the bytes
// on the receiver's mbarrier (transaction count), and the receiver waits for
// exactly the bytes it expects.  Three messages per column:
//   CAND  (all -> all) each CTA's arg-max of column k (index, signed value) and,
//         from the owners, c_k(k), c_k(k+1);
//   RMAX  (all -> all, imax path) row-max partial of column imax, c_imax(imax),
//         c_imax(k), c_imax(k+1);
//   NEXT  (owners -> all) the final W rows of the next pivot rows k', k'+1, and
//         to kp's owner the raw entries the interchange moves into columns
//         k', k'+1.
// A cluster barrier's release waits for every outstanding global store of the
// CTA; a message's release (the complete_tx) is performed by the memory
// system, so the L / interchange stores of a column stream out behind the NEXT
// message instead of in front of it.  They are ordered before the next CAND
// message, which every reader of A inside the panel waits for first.
// The W row of imax is read from its owner's shared memory after CAND (one
// DSMEM round trip); the raw columns k', k'+1 are prefetched with cp.async
// while a column eliminates and the entries its interchange rewrites are
// patched in; interchanged rows of the panel's earlier L columns are rebuilt
// from the W rows (stores only).
constexpr size_t kBkPanelSmemMax = 200 * 1024;
constexpr int kBkMaxRowsPerThread = 3;  // rows of a CTA per thread when the panel fits (rcap <= 656)
constexpr int kBkMsg = 4;  // doubles per CAND / RMAX record

// Pivot coefficients of one panel step, kept by every CTA so a row of the
// panel's L can be rebuilt from the same row of W (bit-identical to the stored
// L): 1x1: L = W * r1; 2x2 (k, k+1): L_k = d21t (d11 W_k - W_k1),
// L_k1 = d21t (d22 W_k1 - W_k); zero / singular columns have W = 0.
struct StepCoef {
    int type;  // 0 W == 0, 1 1x1, 2 first of 2x2, 3 second of 2x2
    double c0, c1, c2;
};

__device__ __forceinline__ double l_1x1(double w, double r1) { return __dmul_rn(w, r1); }
__device__ __forceinline__ double l_2x2(double d21t, double dii, double wi, double wo) {
    return __dmul_rn(d21t, __fma_rn(dii, wi, -wo));
}

__device__ __forceinline__ double l_entry(const double* wrow, const StepCoef* cf, int t) {
    const StepCoef c = cf[t];
    if (c.type == 1) return l_1x1(wrow[t], c.c0);
    if (c.type == 2) return l_2x2(c.c0, c.c1, wrow[t], wrow[t + 1]);
    if (c.type == 3) return l_2x2(c.c0, c.c2, wrow[t], wrow[t - 1]);
    return 0.0;
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}

// Magnitude keys for the warp reductions: for v >= 0 the IEEE bit pattern
// orders like the value, so key = bits(v) + 1 (0 = no candidate / NaN) and a
// max / arg-max is three (two) redux.sync instead of a five-level butterfly.
// Same result as the (|v|, index) merge rule: largest value, then the first
// index; NaN never wins (as `fabs(x) > best` never holds for NaN).
__device__ __forceinline__ unsigned long long mag_key(double v) {
    return v >= 0.0 ? static_cast<unsigned long long>(__double_as_longlong(fabs(v))) + 1ull : 0ull;
}

__device__ __forceinline__ double key_mag(unsigned long long key, double none) {
    return key ? __longlong_as_double(static_cast<long long>(key - 1ull)) : none;
}

// warp arg-max of (key, idx): max key, then min idx among the max keys
__device__ __forceinline__ void warp_key_argmax(unsigned long long& key, unsigned& idx) {
    const unsigned hi = static_cast<unsigned>(key >> 32), lo = static_cast<unsigned>(key);
    const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
    idx = __reduce_min_sync(0xffffffffu, hi == mh && lo == ml ? idx : 0xffffffffu);
    key = (static_cast<unsigned long long>(mh) << 32) | ml;
}

__device__ __forceinline__ unsigned long long warp_key_max(unsigned long long key) {
    const unsigned hi = static_cast<unsigned>(key >> 32), lo = static_cast<unsigned>(key);
    const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
    return (static_cast<unsigned long long>(mh) << 32) | ml;
}

// Updated entry of one row: s0 - W(row, 0:jp) . Lr in the fixed order (groups
// of four into s0..s3, the tail into s0).  Rolled loops: the panel kernel's
// code stays small (a step runs through most of it once).
__device__ __forceinline__ double row_update(const double* w, const double* Lr, int jp, double s0) {
    double s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int t = 0;
#pragma unroll 1
    for (; t + 4 <= jp; t += 4) {
        s0 -= w[t] * Lr[t];
        s1 -= w[t + 1] * Lr[t + 1];
        s2 -= w[t + 2] * Lr[t + 2];
        s3 -= w[t + 3] * Lr[t + 3];
    }
#pragma unroll 1
    for (; t < jp; ++t) s0 -= w[t] * Lr[t];
    return (s0 + s1) + (s2 + s3);
}

// NT threads per CTA; TRACE compiles the phase timers in (their register
// array doubles the register count).
template <int NT, bool TRACE>
__global__ void __launch_bounds__(NT) bk_panel_smem_kernel(const BkArgs a, int rcap) {
    static_assert((NT & (NT - 1)) == 0, "row mapping uses a mask");
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) double dsm[];
    pdl_enter();
    double* Ws = dsm;                 // [rcap][kBkW] this CTA's rows of W
    double* Cs = Ws + rcap * kBkW;    // [rcap] updated column k
    double* Cis = Cs + rcap;          // [rcap] updated column imax
    double* Raw = Cis + rcap;         // [2 pairs][2][rcap] raw stored columns (k, k+1)
    __shared__ unsigned long long skey[NT / 32];  // per-warp reduction keys
    __shared__ unsigned sidx[NT / 32];
    __shared__ double Lr[kBkW], Wim[kBkW];  // L row being applied; W row of imax
    __shared__ double pend[2][kBkW];
    __shared__ int pend_row[2], pend_n[2];
    __shared__ StepCoef coef[kBkW + 1];
    __shared__ double own[5];  // this CTA's c_k(k), c_k(k+1), c_i(imax), c_i(k), c_i(k+1)
    // message buffers (written by the other CTAs), double-buffered by step parity
    __shared__ __align__(16) double candm[2][16][kBkMsg];
    __shared__ __align__(16) double rmaxm[2][16][kBkMsg];
    __shared__ __align__(16) double nextm[2][2 * kBkW + 2];  // rows k', k'+1, 2 patches
    __shared__ __align__(8) uint64_t bars[6];                 // CAND[2], RMAX[2], NEXT[2]
    const int n = static_cast<int>(a.n);
    const int k0 = a.ctl[0];
    if (k0 >= n) return;
    const int G = gridDim.x;
    const int me = static_cast<int>(blockIdx.x);
    const int tid = static_cast<int>(threadIdx.x);
    const int chunk = (n - k0 + G - 1) / G;
    const int lo = k0 + chunk * me, hi = min(n, lo + chunk);
    const int R = hi > lo ? hi - lo : 0;
    const int gtid = me * NT + tid;
    double* A = a.A;
    auto col = [&](int c) { return A + static_cast<size_t>(c) * static_cast<size_t>(n); };
    // owner CTA of row i: (i - k0) / chunk by a float reciprocal and a +-1 fixup
    const float inv_chunk = 1.0f / static_cast<float>(chunk);
    auto owner = [&](int i) {
        const int x = i - k0;
        int q = static_cast<int>(static_cast<float>(x) * inv_chunk);
        if (q * chunk > x) --q;
        else if ((q + 1) * chunk <= x) ++q;
        return q;
    };
    // local row r is always handled by thread r % NT (the thread that
    // prefetched / patched a raw entry is the one that reads it)
    auto first_row = [&](int grow) {
        const int r0 = grow > lo ? min(grow - lo, R) : 0;
        return r0 + ((tid - r0) & (NT - 1));
    };
    auto raw = [&](int pair, int slot) { return Raw + (2 * pair + slot) * rcap; };
    // diagnostics (R1_BK_TRACE): per-phase cycles of CTA 0 thread 0, kept in
    // registers (constant indices after inlining) and written once at the end
    const bool tr = TRACE && a.trace && me == min(a.trace_cta, G - 1) && tid == 0;
    long long tprev = 0;
    unsigned long long tacc[16] = {};
    auto mark = [&](int ph) {
        if (!tr) return;
        const long long t = clock64();
        if (ph >= 0) tacc[ph] += static_cast<unsigned long long>(t - tprev);
        tprev = t;
    };
    if (tid < 2) pend_row[tid] = -1;
    if (tid == 0) {
        for (int b = 0; b < 6; ++b) mbar_init1(&bars[b]);
        mbar_init_fence();
    }
    // raw columns k0, k0+1 of this panel
    for (int s = 0; s < 2; ++s) {
        const int c = k0 + s;
        if (c >= n) break;
        const double* src = col(c);
#pragma unroll 1
        for (int r = first_row(c); r < R; r += NT) cp_async8(raw(0, s) + r, src + lo + r);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    __syncthreads();
    cl.sync();  // barriers initialised and shared memory live everywhere
    mark(-1);

    int k = k0, jp = 0, cp = 0, step = 0, rstep = 0;
    // the previous step's interchange and NEXT message
    bool p_swap = false;
    int p_kp = 0, p_kks = 0;
    uint32_t p_next_bytes = 0;
    while (k < n && jp < kBkNb) {
        const int b = step & 1;
        const double* nx = nextm[b ^ 1];  // NEXT of the previous step
        if (step > 0) {
            if (tid == 0) expect_bytes(&bars[4 + (b ^ 1)], p_next_bytes);
            wait_parity(&bars[4 + (b ^ 1)], ((step - 1) >> 1) & 1);
        }
        mark(0);
        asm volatile("cp.async.wait_all;" ::: "memory");
        if (p_swap) {
            for (int s = 0; s < 2; ++s) {
                const int c = k + s;
                if (c >= n || c > p_kp) continue;
                double* dst = raw(cp, s);
                if (c == p_kp) {  // column kp <- raw column kk below kp
                    const double* src = raw(cp ^ 1, p_kks);
                    for (int r = first_row(p_kp + 1); r < R; r += NT) dst[r] = src[r];
                }
                if (p_kp >= lo && p_kp < hi && ((p_kp - lo) & (NT - 1)) == tid)
                    dst[p_kp - lo] = nx[2 * kBkW + s];
            }
        }
        for (int p = 0; p < 2; ++p)
            if (pend_row[p] >= 0)
                for (int t = tid; t < pend_n[p]; t += NT) Ws[pend_row[p] * kBkW + t] = pend[p][t];
        if (tid < jp) Lr[tid] = l_entry(nx, coef, tid);
        __syncthreads();
        if (tid < 2) pend_row[tid] = -1;
        mark(1);
        // ---- updated column k on the CTA's rows, its arg-max below the diagonal
        double bv = -1.0, bs = 0.0;
        int bi = n;
        {
            const double* rk = raw(cp, 0);
            for (int r = first_row(k); r < R; r += NT) {
                const int i = lo + r;
                const double sacc = row_update(Ws + r * kBkW, Lr, jp, rk[r]);
                Cs[r] = sacc;
                if (i > k && (fabs(sacc) > bv || (fabs(sacc) == bv && i < bi))) {
                    bv = fabs(sacc);
                    bi = i;
                    bs = sacc;
                }
                if (i == k) own[0] = sacc;
                if (i == k + 1) own[1] = sacc;
            }
        }
        {
            unsigned long long key = mag_key(bv);
            unsigned idx = key ? static_cast<unsigned>(bi) : 0xffffffffu;
            warp_key_argmax(key, idx);
            if ((tid & 31) == 0) {
                skey[tid >> 5] = key;
                sidx[tid >> 5] = idx;
            }
        }
        __syncthreads();
        if (tid < 32) {
            // CAND record of this CTA (arg-max index and signed value, or n / 0
            // without a candidate; c_k(k), c_k(k+1)) -> every CTA; warp 0 sends
            unsigned long long key = tid < NT / 32 ? skey[tid] : 0ull;
            unsigned idx = tid < NT / 32 ? sidx[tid] : 0xffffffffu;
            warp_key_argmax(key, idx);
            const double ci = key ? static_cast<double>(idx) : static_cast<double>(n);
            const double cs = key ? Cs[static_cast<int>(idx) - lo] : 0.0;
            for (int e = tid; e < kBkMsg * G; e += 32) {
                const int f = e & 3;
                const double v = f == 0 ? ci : (f == 1 ? cs : own[f - 2]);
                send8(&candm[b][me][f], v, &bars[b], e >> 2);
            }
        }
        mark(2);
        if (tid == 0) expect_bytes(&bars[b], static_cast<uint32_t>(G * kBkMsg * 8));
        wait_parity(&bars[b], (step >> 1) & 1);
        mark(3);
        double colmax, ckimax;
        int imax;
        {
            const int lane = tid & 31;
            const int ii = lane < G ? static_cast<int>(candm[b][lane][0]) : n;
            const double sg = lane < G ? candm[b][lane][1] : 0.0;
            unsigned long long key = ii < n ? mag_key(fabs(sg)) : 0ull;
            unsigned idx = key ? static_cast<unsigned>(ii) : 0xffffffffu;
            warp_key_argmax(key, idx);
            if (key) {
                colmax = key_mag(key, 0.0);
                imax = static_cast<int>(idx);
                const unsigned wl = __ballot_sync(0xffffffffu, ii == imax);
                ckimax = __shfl_sync(0xffffffffu, sg, __ffs(wl) - 1);
            } else {
                colmax = 0.0;
                imax = k;
                ckimax = 0.0;
            }
        }
        const double ckk = candm[b][owner(k)][2];
        const double ckk1 = k + 1 < n ? candm[b][owner(k + 1)][3] : 0.0;
        const double absakk = fabs(ckk);
        int kstep = 1, kp = k;
        double cimax = 0.0, cik = 0.0, cik1 = 0.0;
        const bool imax_path = !(absakk >= kBkAlpha * colmax);
        if (imax_path) {
            // the column imax of the stored matrix (own rows), loaded first: its
            // L2 latency overlaps the remote W-row read and the L-row build
            double araw[kBkMaxRowsPerThread];
            const int rfirst = first_row(k);
            {
                const double* ci = col(imax);
#pragma unroll
                for (int q = 0; q < kBkMaxRowsPerThread; ++q) {
                    const int r = rfirst + q * NT, i = lo + r;
                    araw[q] = r < R ? (i >= imax ? ci[i] : col(i)[imax]) : 0.0;
                }
            }
            const int oi = owner(imax);
            const int lo_i = k0 + chunk * oi;
            const double* wrem = cl.map_shared_rank(Ws, oi) + (imax - lo_i) * kBkW;
            if (tid < jp) {
                const double w0 = wrem[tid];
                const StepCoef c = coef[tid];
                double lv = 0.0;
                if (c.type == 1) lv = l_1x1(w0, c.c0);
                else if (c.type == 2) lv = l_2x2(c.c0, c.c1, w0, wrem[tid + 1]);
                else if (c.type == 3) lv = l_2x2(c.c0, c.c2, w0, wrem[tid - 1]);
                Wim[tid] = w0;
                Lr[tid] = lv;
            }
            __syncthreads();
            double rv = -1.0;
#pragma unroll 1
            for (int q = 0; q < kBkMaxRowsPerThread; ++q) {
                const int r = rfirst + q * NT;
                if (r >= R) break;
                const int i = lo + r;
                const double a0 = q == 0 ? araw[0] : (q == 1 ? araw[1] : araw[2]);
                const double sacc = row_update(Ws + r * kBkW, Lr, jp, a0);
                Cis[r] = sacc;
                if (i != imax) rv = fmax(rv, fabs(sacc));
                if (i == imax) own[2] = sacc;
                if (i == k) own[3] = sacc;
                if (i == k + 1) own[4] = sacc;
            }
            {
                const unsigned long long key = warp_key_max(mag_key(rv));
                if ((tid & 31) == 0) skey[tid >> 5] = key;
            }
            __syncthreads();
            const int rb = 2 + (rstep & 1);
            if (tid < 32) {
                // RMAX record (row-max partial or -1, c_imax(imax), c_imax(k),
                // c_imax(k+1)) -> every CTA; warp 0 sends
                const double rmx = key_mag(warp_key_max(tid < NT / 32 ? skey[tid] : 0ull), -1.0);
                for (int e = tid; e < kBkMsg * G; e += 32) {
                    const int f = e & 3;
                    send8(&rmaxm[rstep & 1][me][f], f == 0 ? rmx : own[f + 1], &bars[rb], e >> 2);
                }
            }
            mark(4);
            if (tid == 0) expect_bytes(&bars[rb], static_cast<uint32_t>(G * kBkMsg * 8));
            wait_parity(&bars[rb], (rstep >> 1) & 1);
            mark(5);
            const double rowmax =
                key_mag(warp_key_max((tid & 31) < G ? mag_key(rmaxm[rstep & 1][tid & 31][0]) : 0ull), 0.0);
            cimax = rmaxm[rstep & 1][oi][1];
            cik = rmaxm[rstep & 1][owner(k)][2];
            cik1 = k + 1 < n ? rmaxm[rstep & 1][owner(k + 1)][3] : 0.0;
            ++rstep;
            if (tr) tacc[8] += 1;
            if (absakk * rowmax >= kBkAlpha * colmax * colmax) {
                kp = k;
            } else if (fabs(cimax) >= kBkAlpha * rowmax) {
                kp = imax;
            } else {
                kp = imax;
                kstep = 2;
            }
        }
        const int kk = k + kstep - 1;
        const int kks = kstep - 1;  // slot of column kk in the raw pair
        const bool swap = kp != kk;
        const int kn = k + kstep, jn = jp + kstep;
        const bool more = kn < n && jn < kBkNb;
        const double* rkk = raw(cp, kks);
        const double* w_kk = nx + kks * kBkW;  // W row kk (NEXT of the previous step)
        mark(10);
        // ---- NEXT (W needs no division: the pivot coefficients come after
        // it), pivot coefficients (every CTA), new W column(s), pending W rows
        const bool same = kp == k + 1;
        const double d = kstep == 1 ? (kp == k ? ckk : cimax) : 0.0;
        const bool zero = kstep == 1 && d == 0.0;
        auto new_w = [&](int r, int i, double& x0, double& x1) {
            if (kstep == 1) {
                const double v = kp == k ? Cs[r] : (i == k ? cimax : (i == kp ? cik : Cis[r]));
                x0 = zero ? 0.0 : (i == k ? d : v);
                x1 = v;  // unscaled, for the L store
            } else {
                x0 = same ? Cs[r] : (i == k + 1 ? ckimax : (i == kp ? ckk1 : Cs[r]));
                x1 = same ? Cis[r] : (i == k + 1 ? cimax : (i == kp ? cik1 : Cis[r]));
            }
        };
        // NEXT first (everyone waits for it): the final W rows of kn, kn+1 are
        // their old part (the row itself, or the interchange partner kk's for
        // kp) and the new column value(s) of that row -> every CTA; the raw
        // entries an interchange moves into columns kn, kn+1 -> kp's owner
        uint32_t next_bytes = 0;
        if (more) {
            const int okp = owner(kp);
            for (int s = 0; s < 2; ++s) {
                const int q = kn + s;
                if (q >= n) break;
                next_bytes += 8u * jn;
                if (q >= lo && q < hi) {
                    const double* old = swap && q == kp ? w_kk : Ws + (q - lo) * kBkW;
                    double x0, x1;
                    new_w(q - lo, q, x0, x1);
                    // warp w -> CTAs w, w + NT/32, ...; lane -> entries lane, lane + 32
                    for (int dst = tid >> 5; dst < G; dst += NT / 32)
                        for (int t = tid & 31; t < jn; t += 32) {
                            const double v = t < jp ? old[t] : (t == jp ? x0 : x1);
                            send8(&nextm[b][s * kBkW + t], v, &bars[4 + b], dst);
                        }
                }
                if (swap && q <= kp) {
                    if (okp == me) next_bytes += 8u;
                    const int srow = q < kp ? q : kk;  // the raw entry's row in column kk
                    if (srow >= lo && srow < hi && ((srow - lo) & (NT - 1)) == tid)
                        send8(&nextm[b][2 * kBkW + s], rkk[srow - lo], &bars[4 + b], okp);
                }
            }
        }
        mark(6);
        double r1 = 0.0, d11 = 0.0, d22 = 0.0, d21t = 0.0;
        if (kstep == 1) {
            r1 = zero ? 0.0 : 1.0 / d;
        } else {
            const double d21 = same ? ckk1 : ckimax;
            d11 = cimax / d21;
            d22 = ckk / d21;
            const double tt = 1.0 / (d11 * d22 - 1.0);
            d21t = tt / d21;
        }
        mark(12);
        if (swap) {
            if (kk >= lo && kk < hi && tid < jp) pend[0][tid] = Wim[tid];
            if (kp >= lo && kp < hi && tid < jp) pend[1][tid] = w_kk[tid];
            if (tid == 0) {
                if (kk >= lo && kk < hi) {
                    pend_row[0] = kk - lo;
                    pend_n[0] = jn;
                }
                if (kp >= lo && kp < hi) {
                    pend_row[1] = kp - lo;
                    pend_n[1] = jn;
                }
            }
        }
        for (int r = first_row(k); r < R; r += NT) {
            const int i = lo + r;
            double x0, x1;
            new_w(r, i, x0, x1);
            Ws[r * kBkW + jp] = x0;
            if (kstep == 2) Ws[r * kBkW + jp + 1] = x1;
            if (swap && (i == kk || i == kp)) {
                double* pr = pend[i == kk ? 0 : 1];
                pr[jp] = x0;
                if (kstep == 2) pr[jp + 1] = x1;
            }
        }
        if (tid == 0) {
            if (kstep == 1) {
                coef[jp] = StepCoef{zero ? 0 : 1, r1, 0.0, 0.0};
            } else {
                coef[jp] = StepCoef{2, d21t, d11, d22};
                coef[jp + 1] = StepCoef{3, d21t, d11, d22};
            }
        }
        mark(13);
        __syncthreads();
        mark(14);
        // prefetch the raw columns kn, kn+1 (patched at the top of the next
        // step), issued after NEXT so they stream during the stores
        if (more) {
            for (int s = 0; s < 2; ++s) {
                const int c = kn + s;
                if (c >= n) break;
                const double* src = col(c);
#pragma unroll 1
                for (int r = first_row(c); r < R; r += NT) cp_async8(raw(cp ^ 1, s) + r, src + lo + r);
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        mark(11);
        // ---- global stores (stream out behind NEXT): L / D of the new
        // column(s), interchange moves, interchanged rows of earlier L columns
        if (swap) {
            // interchanged rows of the earlier L columns: by the CTAs after
            // CTA 0 (which sends NEXT and owns the panel's first rows)
            const int ns = G > 1 ? G - 1 : 1, sg = G > 1 ? me - 1 : 0;
            for (int e = sg >= 0 ? sg + ns * tid : 2 * jp; e < 2 * jp; e += ns * NT) {
                const int t = e >> 1;
                if (e & 1) col(k0 + t)[kp] = l_entry(w_kk, coef, t);
                else col(k0 + t)[kk] = l_entry(Wim, coef, t);
            }
        }
        mark(15);
        double* ck = col(k);
        double* ck1 = col(k + 1 < n ? k + 1 : k);
        double* ckp = col(kp);
        for (int r = first_row(k); r < R; r += NT) {
            const int i = lo + r;
            double x0, x1;
            new_w(r, i, x0, x1);
            if (swap && i >= kk) {
                const double rv = rkk[r];
                if (i > kp) ckp[i] = rv;
                else if (i > kk && i < kp) col(i)[kp] = rv;
                else if (i == kk) ckp[kp] = rv;
            }
            if (kstep == 1) {
                if (i == k) ck[k] = d;
                else ck[i] = zero ? x1 : l_1x1(x1, r1);
            } else if (i == k) {
                ck[k] = x0;
            } else if (i == k + 1) {
                ck[k + 1] = x0;
                ck1[k + 1] = x1;
            } else {
                ck[i] = l_2x2(d21t, d11, x0, x1);
                ck1[i] = l_2x2(d21t, d22, x1, x0);
            }
        }
        if (gtid == 0) {
            if (kstep == 1) {
                a.ipiv[k] = kp;
                a.ps[k] = 0;
                if (zero) a.ctl[1] = 1;
            } else {
                a.ipiv[k] = -kp - 1;
                a.ipiv[k + 1] = -kp - 1;
                a.ps[k] = 1;
                a.ps[k + 1] = 2;
            }
        }
        p_swap = swap;
        p_kp = kp;
        p_kks = kks;
        p_next_bytes = next_bytes;
        k = kn;
        jp = jn;
        cp ^= 1;
        ++step;
        mark(7);
        if (tr) tacc[9] += 1;
    }
    __syncthreads();
    for (int p = 0; p < 2; ++p)
        if (pend_row[p] >= 0)
            for (int t = tid; t < pend_n[p]; t += NT) Ws[pend_row[p] * kBkW + t] = pend[p][t];
    __syncthreads();
    // the panel's W rows of this CTA -> global, for the trailing update
    for (int t = 0; t < jp; ++t)
#pragma unroll 1
        for (int r = tid; r < R; r += NT) a.Wp[(lo + r) + static_cast<size_t>(t) * n] = Ws[r * kBkW + t];
    if (tr)
        for (int q = 0; q < 16; ++q) a.trace[q] += tacc[q];
    if (gtid == 0) {
        a.perm[a.ctl[4]] = k0;  // panel starts, for the solve
        a.ctl[4] += 1;
        a.ctl[2] = k0;
        a.ctl[3] = jp;
        a.ctl[0] = k;
    }
    cl.sync();  // no CTA exits while others may still read its shared memory
}

constexpr int kBkT2 = 128;  // trailing-update tile rows

// A22 -= W L^T on the FP64 tensor cores (mma.sync m8n8k4 f64): 128 x 64
// tiles of the trailing lower triangle (each 128 x 128 block of the triangle
// as two column halves), 8 warps of 32 x 32, two CTAs per SM so one CTA's
// memory phases overlap the other's.  The A tile goes straight into the
// accumulator fragments (negated: acc = W L^T - A, stored back negated, which
// is exact), so only the W / L panels are staged in shared memory (cp.async,
// row stride kBkUpdLd: conflict-free fragment loads).  One mma replaces 8 DFMA
// issue slots per lane; a DFMA version of this kernel ran its FP64 pipe at
// ~31% (2 warps per scheduler) and was 18% slower end to end.
constexpr int kBkUpdLd = kBkT2 + 8;                  // 136: t-rows 16 banks apart
constexpr int kBkUpdK = (kBkW + 3) / 4 * 4;          // 36: panel width rounded to k = 4
constexpr int kBkUpdCols = 64;                       // tile columns
constexpr size_t kBkUpdTcSmem =
    static_cast<size_t>(kBkUpdK) * (kBkUpdLd + kBkUpdCols + 8) * sizeof(double);

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(kBkThreads, 2) bk_update_tc_kernel(const BkArgs a) {
    constexpr int kLdL = kBkUpdCols + 8;  // 72
    extern __shared__ __align__(16) double usm[];
    double* Ws = usm;                      // [kBkUpdK][kBkUpdLd]  W(i0 + r, t)
    double* Ls = usm + kBkUpdK * kBkUpdLd;  // [kBkUpdK][kLdL]      L(j0 + c, t)
    pdl_enter();
    const int64_t n = a.n;
    const int64_t k0 = a.ctl[2];
    const int jp = a.ctl[3];
    const int64_t kend = k0 + jp;
    const int64_t m = n - kend;
    if (m <= 0 || jp == 0) return;
    const int kp4 = (jp + 3) / 4;
    const int64_t T = (m + kBkT2 - 1) / kBkT2;
    const int64_t ntiles = T * (T + 1);  // two column halves per 128 x 128 block
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;  // warp tile origin in the CTA tile
    const int fr = lane >> 2, fc = (lane & 3) * 2;            // accumulator fragment row / col pair
    for (int64_t xx = blockIdx.x; xx < ntiles; xx += gridDim.x) {
        const int64_t x = xx >> 1;
        int64_t bi = static_cast<int64_t>((sqrt(8.0 * static_cast<double>(x) + 1.0) - 1.0) * 0.5);
        while (bi * (bi + 1) / 2 > x) --bi;
        while ((bi + 1) * (bi + 2) / 2 <= x) ++bi;
        const int64_t bj = x - bi * (bi + 1) / 2;
        const int64_t i0 = kend + bi * kBkT2, j0 = kend + bj * kBkT2 + (xx & 1) * kBkUpdCols;
        if (j0 >= n) continue;
        const int rows = static_cast<int>(n - i0 < kBkT2 ? n - i0 : kBkT2);
        const int cols = static_cast<int>(n - j0 < kBkUpdCols ? n - j0 : kBkUpdCols);
        __syncthreads();  // the previous tile's fragment loads are done
        // W / L panels -> shared (zero outside the tile and for t >= jp)
        for (int e = threadIdx.x; e < kBkT2 * kp4 * 4; e += blockDim.x) {
            const int r = e % kBkT2, t = e / kBkT2;
            double* wd = &Ws[t * kBkUpdLd + r];
            if (t < jp && r < rows) cp_async8(wd, a.Wp + (i0 + r) + t * n);
            else *wd = 0.0;
        }
        for (int e = threadIdx.x; e < kBkUpdCols * kp4 * 4; e += blockDim.x) {
            const int r = e % kBkUpdCols, t = e / kBkUpdCols;
            double* ld = &Ls[t * kLdL + r];
            if (t < jp && r < cols) cp_async8(ld, a.A + (j0 + r) + (k0 + t) * n);
            else *ld = 0.0;
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        // accumulators <- -A (the loads overlap the panel copies)
        double acc[4][4][2];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int ni = 0; ni < 4; ++ni)
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int rr = wm + mi * 8 + fr, cc = wn + ni * 8 + fc + q;
                    acc[mi][ni][q] = rr < rows && cc < cols ? -a.A[(i0 + rr) + (j0 + cc) * n] : 0.0;
                }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        for (int k4 = 0; k4 < kp4; ++k4) {
            const int t = k4 * 4 + (lane & 3);
            double fa[4], fb[4];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) fa[mi] = Ws[t * kBkUpdLd + wm + mi * 8 + fr];
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) fb[ni] = Ls[t * kLdL + wn + ni * 8 + fr];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], fa[mi], fb[ni]);
        }
        // A <- -(W L^T - A), lower triangle only where the tile meets the diagonal
        const bool diag = j0 + kBkUpdCols > i0;
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int ni = 0; ni < 4; ++ni)
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int rr = wm + mi * 8 + fr, cc = wn + ni * 8 + fc + q;
                    const int64_t i = i0 + rr, j = j0 + cc;
                    if (rr < rows && cc < cols && (!diag || i >= j)) a.A[i + j * n] = -acc[mi][ni][q];
                }
    }
}

// The reference's D-block condition
// (ldlt_diag_condition, sym_eig.cpp:381-407); one CTA.
__global__ void bk_condition_kernel(const double* __restrict__ A, int64_t n,
                                    const int* __restrict__ ctl, const char* __restrict__ ps,
                                    double* __restrict__ cond) {
    __shared__ double slo[32], shi[32];
    double lo = INFINITY, hi = 0.0;
    for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
        if (ps[k] == 0) {
            const double m = fabs(A[k + k * n]);
            lo = fmin(lo, m);
            hi = fmax(hi, m);
        } else if (ps[k] == 1) {
            const double aa = A[k + k * n], c = A[(k + 1) + (k + 1) * n], bb = A[(k + 1) + k * n];
            const double mid = 0.5 * (aa + c);
            const double rad = hypot(0.5 * (aa - c), bb);
            const double e1 = fabs(mid + rad), e2 = fabs(mid - rad);
            lo = fmin(lo, fmin(e1, e2));
            hi = fmax(hi, fmax(e1, e2));
        }
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, off));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, off));
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        slo[warp] = lo;
        shi[warp] = hi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) {
            lo = fmin(lo, slo[w]);
            hi = fmax(hi, shi[w]);
        }
        cond[0] = (ctl[1] != 0 || lo == 0.0) ? INFINITY : hi / lo;
    }
}

struct SolveArgs {
    int64_t n;
    const double* A;      // factored
    const int* ipiv;
    const char* ps;       // 0 1x1, 1 first of a 2x2, 2 second of a 2x2
    const int* pstart;    // panel start columns
    const int* ctl;       // ctl[4] = number of panels
    const double* x;      // right-hand side
    double* z;            // n work
    double* y;            // n out (unit) when ok
    double* part;         // gridDim * kBkSolveB
    int* ok;
};

// L(i,k) (zero inside a 2x2 diagonal block)
__device__ __forceinline__ double lval(const SolveArgs& s, int64_t i, int64_t k) {
    return (i == k + 1 && s.ps[k] == 1) ? 0.0 : s.A[i + k * s.n];
}

// interchanges of columns [c0, c1) applied to z in order (forward) or reversed
__device__ void panel_swaps(const SolveArgs& s, int64_t c0, int64_t c1, double* z, bool reverse) {
    if (!reverse) {
        for (int64_t k = c0; k < c1; ++k) {
            if (s.ps[k] == 2) continue;
            const int64_t kk = s.ps[k] == 1 ? k + 1 : k;
            const int64_t kp = s.ps[k] == 1 ? -s.ipiv[k] - 1 : s.ipiv[k];
            if (kp != kk) {
                const double u = z[kk];
                z[kk] = z[kp];
                z[kp] = u;
            }
        }
    } else {
        for (int64_t k = c1 - 1; k >= c0; --k) {
            if (s.ps[k] == 2) continue;
            const int64_t kk = s.ps[k] == 1 ? k + 1 : k;
            const int64_t kp = s.ps[k] == 1 ? -s.ipiv[k] - 1 : s.ipiv[k];
            if (kp != kk) {
                const double u = z[kk];
                z[kk] = z[kp];
                z[kp] = u;
            }
        }
    }
}

// A x = b with P_p A P_p^T = L_p D L_p^T panel by panel (each panel's L is in
// the row order at the end of that panel): forward = (apply P_p, eliminate
// with L_p) for p = 1..; D^-1; backward = (L_p^T, then P_p^T) for p = last..1.
__global__ void __launch_bounds__(kBkThreads) bk_solve_kernel(const SolveArgs s) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double sh[kBkSolveB + 32];
    const int64_t n = s.n;
    const int G = gridDim.x;
    const int64_t gtid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int64_t gthreads = static_cast<int64_t>(G) * blockDim.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int np = s.ctl[4];
    for (int64_t i = gtid; i < n; i += gthreads) s.z[i] = s.x[i];
    grid.sync();
    // ---- forward
    for (int p = 0; p < np; ++p) {
        const int64_t c0 = s.pstart[p], c1 = p + 1 < np ? s.pstart[p + 1] : n;
        if (blockIdx.x == 0) {
            if (threadIdx.x == 0) panel_swaps(s, c0, c1, s.z, false);
            for (int64_t k = c0; k < c1; ++k) {
                __syncthreads();
                const double zk = s.z[k];
                for (int64_t i = k + 1 + threadIdx.x; i < c1; i += blockDim.x) s.z[i] -= lval(s, i, k) * zk;
            }
        }
        grid.sync();
        for (int64_t i = c1 + gtid; i < n; i += gthreads) {
            double acc = 0.0;
            for (int64_t k = c0; k < c1; ++k) acc += lval(s, i, k) * s.z[k];
            s.z[i] -= acc;
        }
        grid.sync();
    }
    // ---- D^-1 (sym_eig.cpp:338-352)
    for (int64_t k = gtid; k < n; k += gthreads) {
        if (s.ps[k] == 0) {
            s.z[k] /= s.A[k + k * n];
        } else if (s.ps[k] == 1) {
            const double akm1k = s.A[(k + 1) + k * n];
            const double akm1 = s.A[k + k * n] / akm1k;
            const double ak = s.A[(k + 1) + (k + 1) * n] / akm1k;
            const double denom = akm1 * ak - 1.0;
            const double bkm1 = s.z[k] / akm1k;
            const double bk = s.z[k + 1] / akm1k;
            s.z[k] = (ak * bkm1 - bk) / denom;
            s.z[k + 1] = (akm1 * bk - bkm1) / denom;
        }
    }
    grid.sync();
    // ---- backward
    for (int p = np - 1; p >= 0; --p) {
        const int64_t c0 = s.pstart[p], c1 = p + 1 < np ? s.pstart[p + 1] : n;
        const int64_t rows = n - c1;
        const int64_t chunk = (rows + G - 1) / G;
        const int64_t r0 = c1 + chunk * blockIdx.x, r1 = min(n, r0 + chunk);
        for (int64_t k = c0 + warp; k < c1; k += nw) {
            double acc = 0.0;
            for (int64_t i = r0 + lane; i < r1; i += 32) acc += lval(s, i, k) * s.z[i];
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
            if (lane == 0) s.part[blockIdx.x * kBkSolveB + (k - c0)] = acc;
        }
        grid.sync();
        if (blockIdx.x == 0) {
            for (int64_t k = c0 + threadIdx.x; k < c1; k += blockDim.x) {
                double acc = 0.0;
                for (int c = 0; c < G; ++c) acc += s.part[c * kBkSolveB + (k - c0)];
                sh[k - c0] = acc;
            }
            for (int64_t k = c1 - 1; k >= c0; --k) {
                __syncthreads();
                double acc = 0.0;
                for (int64_t i = k + 1 + lane; i < c1; i += 32) acc += lval(s, i, k) * s.z[i];
                if (warp == 0) {
#pragma unroll
                    for (int off = 16; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
                    if (lane == 0) s.z[k] -= acc + sh[k - c0];
                }
            }
            __syncthreads();
            if (threadIdx.x == 0) panel_swaps(s, c0, c1, s.z, true);
        }
        grid.sync();
    }
    // ---- normalise (sym_eig.cpp:425-431)
    if (blockIdx.x == 0) {
        double acc = 0.0;
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc = fma(s.z[i], s.z[i], acc);
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (lane == 0) sh[warp] = acc;
        __syncthreads();
        double tot = 0.0;
        for (int w = 0; w < nw; ++w) tot += sh[w];
        const double nrm = sqrt(tot);
        const bool good = isfinite(nrm) && nrm != 0.0;
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s.y[i] = good ? s.z[i] / nrm : s.z[i];
        if (threadIdx.x == 0) s.ok[0] = good ? 1 : 0;
    }
}

// Composed interchanges of each panel (one thread per panel): the rows a
// panel's interchanges touch are its own columns' rows plus a few rows below
// it ("outside" rows); applying the interchanges in order (forward) or in
// reverse (backward) is a fixed permutation of those slots.
__global__ void bk_perm_kernel(const int* __restrict__ ipiv, const char* __restrict__ ps,
                               const int* __restrict__ pstart, const int* __restrict__ ctl, int n,
                               int* __restrict__ pperm) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    const int np = ctl[4];
    if (p >= np) return;
    const int c0 = pstart[p], c1 = p + 1 < np ? pstart[p + 1] : n, w = c1 - c0;
    int* P = pperm + static_cast<size_t>(p) * kPermStride;
    int* out = P + 4;
    int* fwd = out + kBkW;
    int* bwd = fwd + 2 * kBkW;
    int nout = 0;
    unsigned long long first2 = 0;
    auto slot = [&](int row) {
        if (row < c1) return row - c0;
        for (int j = 0; j < nout; ++j)
            if (out[j] == row) return w + j;
        out[nout] = row;
        return w + nout++;
    };
    for (int j = 0; j < 2 * kBkW; ++j) fwd[j] = bwd[j] = j;
    for (int k = c0; k < c1; ++k) {
        if (ps[k] == 1) first2 |= 1ull << (k - c0);
        if (ps[k] == 2) continue;
        const int kk = ps[k] == 1 ? k + 1 : k;
        const int kp = ps[k] == 1 ? -ipiv[k] - 1 : ipiv[k];
        if (kp == kk) continue;
        const int a = slot(kk), b = slot(kp);
        const int t = fwd[a];
        fwd[a] = fwd[b];
        fwd[b] = t;
    }
    for (int k = c1 - 1; k >= c0; --k) {
        if (ps[k] == 2) continue;
        const int kk = ps[k] == 1 ? k + 1 : k;
        const int kp = ps[k] == 1 ? -ipiv[k] - 1 : ipiv[k];
        if (kp == kk) continue;
        const int a = slot(kk), b = slot(kp);
        const int t = bwd[a];
        bwd[a] = bwd[b];
        bwd[b] = t;
    }
    P[0] = nout;
    P[1] = static_cast<int>(first2 & 0xffffffffu);
    P[2] = static_cast<int>(first2 >> 32);
}

// A x = b on ONE thread-block cluster (<= 16 CTAs): z lives in shared memory,
// CTA c owning rows [c chunk, (c+1) chunk).  Per panel (forward: P_p, L_p^-1;
// backward: L_p^-T, P_p^T, same algebra as bk_solve_kernel) every CTA
// redundantly solves the panel's diagonal block on the panel's rows plus the
// outside rows its interchanges touch (slots), and updates its own rows below
// the panel; the slot values a panel needs are pushed to every CTA by their
// owners at the end of the previous panel, so one cluster barrier per panel
// orders everything.  Fixed partitions and summation orders: deterministic.
__global__ void __launch_bounds__(kBkThreads) bk_solve_cluster_kernel(const SolveArgs s, const int* pperm) {
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) double zs[];      // own rows of z, then Lr
    __shared__ double Lb[2][kBkW][kBkW + 1];          // panel diagonal block (see below)
    __shared__ double gsl[2][2 * kBkW];               // pushed slot values, by panel parity
    __shared__ double part[2][16][kBkW];              // pushed backward partials, by parity
    __shared__ double zp[2 * kBkW];
    __shared__ double nrm2[16];
    // message barriers by panel parity (dsmem.cuh): the slot values (and, in
    // the backward pass, the partials) a panel needs count on mbar[par]
    __shared__ __align__(8) uint64_t mbar[2];
    __shared__ double tok[2][16];  // forward-pass tokens (see recv)
    uint32_t mph[2] = {0, 0};
    const int n = static_cast<int>(s.n);
    const int G = gridDim.x, me = blockIdx.x, tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int chunk = (n + G - 1) / G;
    const int lo = chunk * me, hi = min(n, lo + chunk), R = hi > lo ? hi - lo : 0;
    const int np = s.ctl[4];
    const double* A = s.A;
    auto colp = [&](int c) { return A + static_cast<size_t>(c) * static_cast<size_t>(n); };
    // Lr[t * chunk + r] = L(lo + r, c0 + t): this CTA's rows of a panel's L21,
    // staged with cp.async one panel ahead (the update / partials read it)
    double* Lr = zs + ((chunk + 1) & ~1);
    auto rec = [&](int p) { return pperm + static_cast<size_t>(p) * kPermStride; };
    auto pbounds = [&](int p, int& c0, int& c1) {
        c0 = s.pstart[p];
        c1 = p + 1 < np ? s.pstart[p + 1] : n;
    };
    auto slot_row = [&](const int* P, int c0, int w, int j) { return j < w ? c0 + j : P[4 + j - w]; };
    auto is_first2 = [&](const int* P, int t) {
        return ((t < 32 ? static_cast<unsigned>(P[1]) >> t : static_cast<unsigned>(P[2]) >> (t - 32)) & 1u) != 0;
    };
    // every CTA's slot values of panel p (rows owned here) -> gsl[par] everywhere
    auto push_slots = [&](int p, int par) {
        int c0, c1;
        pbounds(p, c0, c1);
        const int* P = rec(p);
        const int w = c1 - c0, m = w + P[0];
        for (int e = tid; e < m * G; e += kBkThreads) {
            const int j = e % m, d = e / m;
            const int row = slot_row(P, c0, w, j);
            if (row >= lo && row < hi) send8(&gsl[par][j], zs[row - lo], &mbar[par], d);
        }
    };
    // panel p's messages at this CTA: its m slot values, plus G w partials
    // (backward) or one token from every CTA (forward).  Only the owners of a
    // panel's slot rows send slot values, so without the tokens a CTA with
    // nothing to send imposes no wait and others could run two panels ahead
    // into the same-parity buffer; a token is sent after its sender has read
    // the previous panel's buffer (the backward partials come from every CTA).
    auto recv = [&](int p, int par, bool partials) {
        int c0, c1;
        pbounds(p, c0, c1);
        const int w = c1 - c0, m = w + rec(p)[0];
        if (tid == 0) expect_bytes(&mbar[par], static_cast<uint32_t>((m + (partials ? G * w : G)) * 8));
        if (par == 0) {
            wait_parity(&mbar[0], mph[0] & 1);
            ++mph[0];
        } else {
            wait_parity(&mbar[1], mph[1] & 1);
            ++mph[1];
        }
    };
    // forward: Lb[par][t][i] = L(c0+i, c0+t), i > t (column t contiguous)
    auto load_fwd_block = [&](int p, int par) {
        int c0, c1;
        pbounds(p, c0, c1);
        const int* P = rec(p);
        const int w = c1 - c0;
        for (int e = tid; e < w * w; e += kBkThreads) {
            const int t = e / w, i = e - t * w;
            const bool z = i <= t || (i == t + 1 && is_first2(P, t));
            Lb[par][t][i] = z ? 0.0 : colp(c0 + t)[c0 + i];
        }
    };
    auto prefetch_rows = [&](int p) {
        int c0, c1;
        pbounds(p, c0, c1);
        const int w = c1 - c0;
        const int r0 = c1 > lo ? min(c1 - lo, R) : 0;
        const int nr = R - r0;
        for (int e = tid; e < w * nr; e += kBkThreads) {
            const int t = e / nr, r = r0 + (e - t * nr);
            cp_async8(&Lr[t * chunk + r], colp(c0 + t) + lo + r);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int r = tid; r < R; r += kBkThreads) zs[r] = s.x[lo + r];
    if (tid == 0) {
        mbar_init1(&mbar[0]);
        mbar_init1(&mbar[1]);
        mbar_init_fence();
    }
    __syncthreads();
    cl.sync();  // barriers initialised, every CTA running, before any DSMEM store
    auto token = [&](int par) {
        if (tid < G) send8(&tok[par][me], 0.0, &mbar[par], tid);
    };
    if (np > 0) {
        prefetch_rows(0);
        push_slots(0, 0);
        token(0);
        load_fwd_block(0, 0);
    }
    // ---- forward
    for (int p = 0; p < np; ++p) {
        const int par = p & 1;
        int c0, c1;
        pbounds(p, c0, c1);
        const int* P = rec(p);
        const int w = c1 - c0, m = w + P[0];
        recv(p, par, false);
        __syncthreads();  // load_fwd_block(p) of the previous iteration is complete
        if (tid < m) zp[tid] = gsl[par][P[4 + kBkW + tid]];
        __syncthreads();
        if (warp == 0) {
            double a0 = lane < w ? zp[lane] : 0.0, a1 = lane + 32 < w ? zp[lane + 32] : 0.0;
            for (int t = 0; t < w; ++t) {
                const double zt = __shfl_sync(0xffffffffu, t < 32 ? a0 : a1, t & 31);
                a0 -= Lb[par][t][lane] * zt;  // zero for lane <= t
                if (lane + 32 < w) a1 -= Lb[par][t][lane + 32] * zt;
            }
            if (lane < w) zp[lane] = a0;
            if (lane + 32 < w) zp[lane + 32] = a1;
        }
        if (p + 1 < np) load_fwd_block(p + 1, par ^ 1);
        __syncthreads();
        if (tid < m) {
            const int row = slot_row(P, c0, w, tid);
            if (row >= lo && row < hi) zs[row - lo] = zp[tid];
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
        {
            const int r0 = c1 > lo ? min(c1 - lo, R) : 0;
            for (int r = r0 + tid; r < R; r += kBkThreads) {
                double acc = 0.0;
                for (int t = 0; t < w; ++t) acc += Lr[t * chunk + r] * zp[t];
                zs[r] -= acc;
            }
        }
        __syncthreads();
        if (p + 1 < np) {
            prefetch_rows(p + 1);
            push_slots(p + 1, par ^ 1);
            token(par ^ 1);
        }
    }
    cl.sync();  // D^-1 below reads / writes a neighbour's z for straddling 2x2 blocks
    // ---- D^-1 (sym_eig.cpp:338-352); a 2x2 pair is solved by its first row's owner
    for (int r = tid; r < R; r += kBkThreads) {
        const int k = lo + r;
        if (s.ps[k] == 0) {
            zs[r] /= A[k + static_cast<size_t>(k) * n];
        } else if (s.ps[k] == 1) {
            double* zk1 = k + 1 < hi ? &zs[r + 1] : cl.map_shared_rank(zs, me + 1);
            const double akm1k = A[(k + 1) + static_cast<size_t>(k) * n];
            const double akm1 = A[k + static_cast<size_t>(k) * n] / akm1k;
            const double ak = A[(k + 1) + static_cast<size_t>(k + 1) * n] / akm1k;
            const double denom = akm1 * ak - 1.0;
            const double bkm1 = zs[r] / akm1k;
            const double bk = *zk1 / akm1k;
            zs[r] = (ak * bkm1 - bk) / denom;
            *zk1 = (akm1 * bk - bkm1) / denom;
        }
    }
    cl.sync();
    // ---- backward: per panel, partials of L21^T z over own rows + own slot
    // values -> every CTA; barrier; sum (fixed order), L11^-T, P^T, write back
    auto push_back = [&](int p, int par) {
        int c0, c1;
        pbounds(p, c0, c1);
        const int w = c1 - c0;
        const int r0 = c1 > lo ? min(c1 - lo, R) : 0;
        for (int t = warp; t < w; t += kBkThreads / 32) {
            const double* ct = Lr + t * chunk;
            double acc = 0.0;
            for (int r = r0 + lane; r < R; r += 32) acc += ct[r] * zs[r];
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
            if (lane < G) send8(&part[par][me][t], acc, &mbar[par], lane);
        }
        push_slots(p, par);
    };
    if (np > 0) {
        prefetch_rows(np - 1);
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
        push_back(np - 1, (np - 1) & 1);
    }
    for (int p = np - 1; p >= 0; --p) {
        const int par = p & 1;
        int c0, c1;
        pbounds(p, c0, c1);
        const int* P = rec(p);
        const int w = c1 - c0, m = w + P[0];
        recv(p, par, true);
        __syncthreads();  // push_back(p) finished reading Lr
        if (p > 0) prefetch_rows(p - 1);
        // backward block: Lb[par][i][t] = L(c0+i, c0+t), i > t (row i contiguous)
        for (int e = tid; e < w * w; e += kBkThreads) {
            const int i = e / w, t = e - i * w;
            const bool z = i <= t || (i == t + 1 && is_first2(P, t));
            Lb[par][i][t] = z ? 0.0 : colp(c0 + t)[c0 + i];
        }
        if (tid < m) {
            double v = gsl[par][tid];
            if (tid < w)
                for (int c = 0; c < G; ++c) v -= part[par][c][tid];
            zp[tid] = v;
        }
        __syncthreads();
        if (warp == 0) {
            double a0 = lane < w ? zp[lane] : 0.0, a1 = lane + 32 < w ? zp[lane + 32] : 0.0;
            for (int i = w - 1; i >= 1; --i) {
                const double zi = __shfl_sync(0xffffffffu, i < 32 ? a0 : a1, i & 31);
                a0 -= Lb[par][i][lane] * zi;  // zero for lane >= i
            }
            if (lane < w) zp[lane] = a0;
            if (lane + 32 < w) zp[lane + 32] = a1;
        }
        __syncthreads();
        if (tid < m) {
            const int row = slot_row(P, c0, w, tid);
            if (row >= lo && row < hi) zs[row - lo] = zp[P[4 + 3 * kBkW + tid]];
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
        if (p > 0) push_back(p - 1, par ^ 1);
    }
    // ---- normalise (sym_eig.cpp:425-431)
    {
        double acc = 0.0;
        for (int r = tid; r < R; r += kBkThreads) acc = fma(zs[r], zs[r], acc);
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (lane == 0) zp[warp] = acc;
        __syncthreads();
        if (tid < G) {
            double tot = 0.0;
            for (int w = 0; w < kBkThreads / 32; ++w) tot += zp[w];
            *cl.map_shared_rank(&nrm2[me], tid) = tot;
        }
        cl.sync();
        double tot = 0.0;
        for (int c = 0; c < G; ++c) tot += nrm2[c];
        const double nrm = sqrt(tot);
        const bool good = isfinite(nrm) && nrm != 0.0;
        for (int r = tid; r < R; r += kBkThreads) s.y[lo + r] = good ? zs[r] / nrm : zs[r];
        if (me == 0 && tid == 0) s.ok[0] = good ? 1 : 0;
    }
    cl.sync();  // no CTA exits while others may still access its shared memory
}

// Largest cluster (<= 16, <= one CTA per 256 rows) the device can schedule.
int panel_cluster_size(r1_context* ctx, int64_t n) {
    static std::map<int, int> max_by_device;
    configure_once(reinterpret_cast<const void*>(bk_panel_kernel), ctx->device, [&] {
        int max16 = cudaFuncSetAttribute(bk_panel_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                        cudaSuccess
                    ? 16
                    : 8;
        cudaGetLastError();
        if (max16 == 16) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(16);
            cfg.blockDim = dim3(kBkThreads);
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = 16;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            int clusters = 0;
            if (cudaOccupancyMaxActiveClusters(&clusters, bk_panel_kernel, &cfg) != cudaSuccess ||
                clusters < 1)
                max16 = 8;
            cudaGetLastError();
        }
        max_by_device[ctx->device] = max16;
    });
    int max16 = 8;
    {
        std::lock_guard<std::mutex> g(cache_mutex());
        max16 = max_by_device[ctx->device];
    }
    static const char* genv = dev_env("R1_BK_G");  // development: force the cluster size
    if (genv) return std::max(1, std::min(max16, std::atoi(genv)));
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(max16, (n + 255) / 256)));
}

int coop_grid(const void* fn, int want, int num_sms) {
    int per_sm = 0;
    R1_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kBkThreads, 0));
    if (per_sm < 1) fail(R1_ERR_CUDA, "bk kernel cannot be resident");
    return std::max(1, std::min(want, per_sm * num_sms));
}

}  // namespace

size_t bk_workspace_bytes(int64_t n, int num_sms) {
    return (static_cast<size_t>(n) * kBkW + 3 * static_cast<size_t>(n) + 64 * 8 +
            static_cast<size_t>(num_sms) * kBkSolveB + 96) * sizeof(double) +
           (2 * static_cast<size_t>(n) + 64) * sizeof(int) + static_cast<size_t>(n) + 64 + 16 +
           static_cast<size_t>(max_panels(n)) * kPermStride * sizeof(int);
}

// Factor A (n x n, device, lower triangle; overwritten) and write the D-block
// condition (inf when singular) to cond_dev.  Async on ctx->stream.
void bk_factor(r1_context* ctx, int64_t n, double* A, void* ws, double* cond_dev) {
    const BkLayout L = bk_layout(ws, n, ctx->num_sms);
    R1_CUDA(cudaMemsetAsync(L.ctl, 0, 16 * sizeof(int), ctx->stream));
    bk_init_kernel<<<std::max(1, static_cast<int>(std::min<int64_t>((n + 255) / 256, 64))), 256, 0,
                     ctx->stream>>>(L.perm, L.ps, n);
    check_launch(ctx, "bk_init_kernel");
    static const bool trace = dev_env("R1_BK_TRACE") != nullptr;
    static DeviceBuffer tbuf;
    if (trace) {
        tbuf.ensure(16 * sizeof(unsigned long long));
        R1_CUDA(cudaMemsetAsync(tbuf.ptr, 0, 16 * sizeof(unsigned long long), ctx->stream));
    }
    BkArgs a{n, A, L.Wp, L.ipiv, L.ctl, L.Ck, L.Ci, L.red, L.perm, L.ps,
             trace ? tbuf.as<unsigned long long>() : nullptr,
             0};
    if (const char* tenv = dev_env("R1_BK_TRACE")) a.trace_cta = std::max(0, std::atoi(tenv) - 1);
    // the panel grid is one cluster (<= 16 CTAs, non-portable size when the
    // device allows it): enough SMs for the column updates, hardware barriers
    const int gp = panel_cluster_size(ctx, n);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(gp);
    cfg.blockDim = dim3(kBkThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = gp;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // CTA rows of W + the two updated columns in shared memory when they fit
    const int rcap = static_cast<int>((n + gp - 1) / gp);
    const size_t psmem = static_cast<size_t>(rcap) * (kBkW + 6) * sizeof(double);
    const bool smem_panel = psmem <= kBkPanelSmemMax && gp <= 16 && rcap <= kBkMaxRowsPerThread * kBkThreads;
    configure_once(reinterpret_cast<const void*>(bk_update_tc_kernel), ctx->device, [&] {
        for (auto fn : {bk_panel_smem_kernel<kBkThreads, false>, bk_panel_smem_kernel<kBkThreads, true>}) {
            R1_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kBkPanelSmemMax)));
            R1_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        }
        R1_CUDA(cudaFuncSetAttribute(bk_update_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(kBkUpdTcSmem)));
    });
    // 256 threads even when a CTA owns 2 rows per thread (n = 6500): 512 was
    // measured 2% slower there (16-warp reductions and barriers)
    auto panel_fn = trace ? bk_panel_smem_kernel<kBkThreads, true> : bk_panel_smem_kernel<kBkThreads, false>;
    // panels and trailing updates alternate as programmatic dependent launches:
    // each kernel is launched while its predecessor runs and waits for it on
    // the device (griddepcontrol.wait), so launch latency leaves the chain
    static const char* pdl_env = dev_env("R1_BK_PDL");  // development: 0 = plain stream order
    const bool pdl = !(pdl_env && std::atoi(pdl_env) == 0);
    cudaLaunchAttribute pattr[2];
    pattr[0] = attr[0];
    pattr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pattr[1].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t pcfg = cfg;
    pcfg.dynamicSmemBytes = psmem;
    pcfg.attrs = pattr;
    pcfg.numAttrs = pdl ? 2 : 1;
    cudaLaunchConfig_t ucfg{};
    ucfg.gridDim = dim3(2 * ctx->num_sms);
    ucfg.blockDim = dim3(kBkThreads);
    ucfg.dynamicSmemBytes = kBkUpdTcSmem;
    ucfg.stream = ctx->stream;
    ucfg.attrs = pattr + 1;
    ucfg.numAttrs = pdl ? 1 : 0;
    // each panel factors >= kBkNb columns (or the rest); extra launches exit at once
    const int64_t panels = (n + kBkNb - 1) / kBkNb;
    for (int64_t p = 0; p < panels; ++p) {
        if (smem_panel)
            R1_CUDA(cudaLaunchKernelEx(&pcfg, panel_fn, a, rcap));
        else
            R1_CUDA(cudaLaunchKernelEx(&cfg, bk_panel_kernel, a));
        check_launch(ctx, "bk_panel_kernel");
        R1_CUDA(cudaLaunchKernelEx(&ucfg, bk_update_tc_kernel, a));
        check_launch(ctx, "bk_update_tc_kernel");
    }
    bk_condition_kernel<<<1, 1024, 0, ctx->stream>>>(A, n, L.ctl, L.ps, cond_dev);
    check_launch(ctx, "bk_condition_kernel");
    if (trace) {
        unsigned long long h[16];
        R1_CUDA(cudaMemcpyAsync(h, tbuf.ptr, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
        const double c = h[9] ? static_cast<double>(h[9]) : 1.0;
        std::fprintf(stderr,
                     "[r1 bk] n=%lld cols=%llu imax-path=%llu cycles/col: wait_next %.0f top %.0f step1 %.0f "
                     "wait_cand %.0f imax %.0f wait_rmax %.0f elim %.0f (decide %.0f prefetch %.0f coef %.0f "
                     "neww %.0f bar %.0f sends %.0f) swapL %.0f stores %.0f\n",
                     static_cast<long long>(n), h[9], h[8], h[0] / c, h[1] / c, h[2] / c, h[3] / c,
                     h[4] / c, h[5] / c, (h[10] + h[11] + h[12] + h[13] + h[14] + h[6]) / c, h[10] / c,
                     h[11] / c, h[12] / c, h[13] / c, h[14] / c, h[6] / c, h[15] / c, h[7] / c);
    }
}

// y = (factored A)^-1 x, normalised; *ok_dev = finite and nonzero.
void bk_solve(r1_context* ctx, int64_t n, const double* A, void* ws, const double* x, double* y,
              int* ok_dev) {
    const BkLayout L = bk_layout(ws, n, ctx->num_sms);
    SolveArgs s{n, A, L.ipiv, L.ps, L.perm, L.ctl, x, L.z, y, L.part, ok_dev};
    static const char* gsolve = dev_env("R1_BK_GRID_SOLVE");
    const int gp = panel_cluster_size(ctx, n);
    if (!(gsolve && std::atoi(gsolve)) && n < (int64_t(1) << 30)) {
        // cluster solve: interchanges composed per panel, z in shared memory
        const int64_t mp = max_panels(n);
        bk_perm_kernel<<<static_cast<int>((mp + 127) / 128), 128, 0, ctx->stream>>>(
            L.ipiv, L.ps, L.perm, L.ctl, static_cast<int>(n), L.pperm);
        check_launch(ctx, "bk_perm_kernel");
        configure_once(reinterpret_cast<const void*>(bk_solve_cluster_kernel), ctx->device, [&] {
            R1_CUDA(cudaFuncSetAttribute(bk_solve_cluster_kernel,
                                         cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            R1_CUDA(cudaFuncSetAttribute(bk_solve_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         190 * 1024));
        });
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(gp);
        cfg.blockDim = dim3(kBkThreads);
        const int64_t chunk = (n + gp - 1) / gp;
        cfg.dynamicSmemBytes = static_cast<size_t>(((chunk + 1) & ~int64_t(1)) + kBkW * chunk) * sizeof(double);
        cfg.stream = ctx->stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = gp;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (cfg.dynamicSmemBytes <= 190 * 1024) {
            R1_CUDA(cudaLaunchKernelEx(&cfg, bk_solve_cluster_kernel, s, static_cast<const int*>(L.pperm)));
            check_launch(ctx, "bk_solve_cluster_kernel");
            return;
        }
    }
    const int g = coop_grid(reinterpret_cast<const void*>(bk_solve_kernel),
                            static_cast<int>(std::min<int64_t>(ctx->num_sms, (n + 255) / 256 + 1)),
                            ctx->num_sms);
    void* args[] = {&s};
    R1_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(bk_solve_kernel), dim3(g),
                                        dim3(kBkThreads), args, 0, ctx->stream));
    check_launch(ctx, "bk_solve_kernel");
}

}  // namespace r1

using namespace r1;

extern "C" {

// Diagnostics (not in the public header): factor the host matrix S and return
// ipiv (reference encoding), D (diag[n], sub[n]: the 2x2 off-diagonal at the
// first column of each pair), the singular flag and the D-block condition.
int r1x_ldlt(r1_context* ctx, int64_t n, const double* s_host, int* ipiv, double* diag,
             double* sub, int* singular, double* cond) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx) fail(R1_ERR_INVALID_ARGUMENT, "null context");
        R1_CUDA(cudaSetDevice(ctx->device));
        DeviceBuffer A, ws, c;
        A.ensure(static_cast<size_t>(n) * n * sizeof(double));
        ws.ensure(bk_workspace_bytes(n, ctx->num_sms));
        c.ensure(64);
        R1_CUDA(cudaMemcpyAsync(A.ptr, s_host, static_cast<size_t>(n) * n * sizeof(double),
                                cudaMemcpyHostToDevice, ctx->stream));
        bk_factor(ctx, n, A.as<double>(), ws.ptr, c.as<double>());
        const BkLayout L = bk_layout(ws.ptr, n, ctx->num_sms);
        std::vector<double> h(static_cast<size_t>(n) * n);
        int ctl[4];
        R1_CUDA(cudaMemcpyAsync(h.data(), A.ptr, h.size() * sizeof(double), cudaMemcpyDeviceToHost,
                                ctx->stream));
        R1_CUDA(cudaMemcpyAsync(ipiv, L.ipiv, n * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaMemcpyAsync(ctl, L.ctl, sizeof(ctl), cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaMemcpyAsync(cond, c.ptr, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
        for (int64_t k = 0; k < n; ++k) {
            diag[k] = h[k + k * n];
            sub[k] = 0.0;
        }
        for (int64_t k = 0; k < n;) {
            if (ipiv[k] < 0) {
                sub[k] = h[(k + 1) + k * n];
                k += 2;
            } else {
                ++k;
            }
        }
        *singular = ctl[1];
    });
}

// Diagnostics: upload S once, then time `reps` factorisations of fresh copies
// with CUDA events on the context's stream (the device-to-device restore is
// outside the timed region); ms[r] = factorisation r.
int r1x_ldlt_time(r1_context* ctx, int64_t n, const double* s_host, int reps, double* ms) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx || reps < 1) fail(R1_ERR_INVALID_ARGUMENT, "r1x_ldlt_time: bad arguments");
        R1_CUDA(cudaSetDevice(ctx->device));
        const size_t bytes = static_cast<size_t>(n) * n * sizeof(double);
        DeviceBuffer S, A, ws, c;
        S.ensure(bytes);
        A.ensure(bytes);
        ws.ensure(bk_workspace_bytes(n, ctx->num_sms));
        c.ensure(64);
        R1_CUDA(cudaMemcpyAsync(S.ptr, s_host, bytes, cudaMemcpyHostToDevice, ctx->stream));
        cudaEvent_t e0, e1;
        R1_CUDA(cudaEventCreate(&e0));
        R1_CUDA(cudaEventCreate(&e1));
        for (int r = 0; r < reps; ++r) {
            R1_CUDA(cudaMemcpyAsync(A.ptr, S.ptr, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
            R1_CUDA(cudaEventRecord(e0, ctx->stream));
            bk_factor(ctx, n, A.as<double>(), ws.ptr, c.as<double>());
            R1_CUDA(cudaEventRecord(e1, ctx->stream));
            R1_CUDA(cudaEventSynchronize(e1));
            float t = 0.0f;
            R1_CUDA(cudaEventElapsedTime(&t, e0, e1));
            ms[r] = t;
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    });
}

}  // extern "C"
