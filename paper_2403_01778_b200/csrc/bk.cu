// Bunch-Kaufman LDL^T (lower) of a dense symmetric matrix, hand-written for
// the iHOSCF Rayleigh-quotient step (reference proj/src/sym_eig.cpp:233-438:
// ldlt_factor, ldlt_solve, ldlt_diag_condition, rayleigh_quotient_step).
//
// Same pivot rule as the reference's unblocked factorisation (alpha =
// (1+sqrt17)/8; 1x1 without interchange, 1x1 with k <-> imax, 2x2 with
// k+1 <-> imax; ties to the first index; zero column -> singular), blocked the
// LAPACK dlasyf way so the O(n^3) work runs on all SMs:
//   * panel kernel (cooperative, a few dozen CTAs): for each of <= 32 (+1 when
//     a 2x2 pivot straddles the edge) columns, form the updated column from
//     the stored matrix minus the panel's delayed update (W = unscaled pivot
//     columns, L), reduce colmax / rowmax over the grid, pick the pivot, apply
//     the symmetric interchange, eliminate.  2-4 grid barriers per column.
//   * trailing update kernel (all SMs): A22 -= W L^T on the lower triangle,
//     128x128 tiles, W / L panels and the A tile staged with cp.async.
// D, the pivot sequence and the solution are the reference's (its accept test
// only reads D).  Interchanges are applied to the rows of the CURRENT panel's
// L only, so each panel's L is stored in the row order at the end of that
// panel (the blocked LAPACK convention); the solve (one cooperative kernel)
// applies them panel by panel: forward (P_p, L_p), D^-1, backward (L_p^T, P_p^T).
#include "common.cuh"

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
    unsigned long long* trace;  // diagnostics: per-phase globaltimer sums (CTA 0), or null
};

// Workspace layout (bytes from bk_workspace_bytes).
struct BkLayout {
    double *Wp, *Ck, *Ci, *red, *part, *z;
    int *ctl, *ipiv, *perm;
    char* ps;
};

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
    return L;
}

__global__ void bk_init_kernel(int* perm, char* ps, int64_t n) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        perm[i] = static_cast<int>(i);
        ps[i] = 0;
    }
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

// Panel kernel with the CTA's rows of W and of the two updated columns held
// in shared memory (used when they fit).  The few scalars other CTAs need —
// c_k(k), c_k(k+1), the signed arg-max entry, c_imax(imax), c_imax(k),
// c_imax(k+1) — are published beside the reduction partials, so a column
// costs two cluster barriers (three on the imax path) and no global re-reads
// of the updated columns.  W rows exchanged by an interchange move through
// DSMEM and land at the top of the next column.
__device__ void block_argmax3(double& v, int64_t& i, double& sgn, double* sv, int64_t* si,
                              double* ss) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, v, off);
        const int64_t i2 = __shfl_xor_sync(0xffffffffu, i, off);
        const double s2 = __shfl_xor_sync(0xffffffffu, sgn, off);
        if (v2 > v || (v2 == v && i2 < i)) {
            v = v2;
            i = i2;
            sgn = s2;
        }
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) {
        sv[warp] = v;
        si[warp] = i;
        ss[warp] = sgn;
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w)
            if (sv[w] > v || (sv[w] == v && si[w] < i)) {
                v = sv[w];
                i = si[w];
                sgn = ss[w];
            }
}

// Pivot coefficients of one panel step, kept by every CTA so a row of the
// panel's L can be rebuilt from the same row of W (bit-identical to the stored
// L): 1x1: L = W * r1; 2x2 (k, k+1): L_k = d21t (d11 W_k - W_k1),
// L_k1 = d21t (d22 W_k1 - W_k); zero / singular columns have W = 0.
struct StepCoef {
    int type;  // 0 W == 0, 1 1x1, 2 first of 2x2, 3 second of 2x2
    double c0, c1, c2;
};

__device__ __forceinline__ void l_row(const double* wrow, const StepCoef* cf, int jp, double* out) {
    for (int t = threadIdx.x; t < jp; t += blockDim.x) {
        const StepCoef c = cf[t];
        double v = 0.0;
        if (c.type == 1) v = wrow[t] * c.c0;
        else if (c.type == 2) v = c.c0 * (c.c1 * wrow[t] - wrow[t + 1]);
        else if (c.type == 3) v = c.c0 * (c.c2 * wrow[t] - wrow[t - 1]);
        out[t] = v;
    }
}

__global__ void __launch_bounds__(kBkThreads) bk_panel_smem_kernel(const BkArgs a, int rcap) {
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) double dsm[];
    double* Ws = dsm;                 // [rcap][kBkW] this CTA's rows of W
    double* Cs = Ws + rcap * kBkW;    // [rcap] updated column k
    double* Cis = Cs + rcap;          // [rcap] updated column imax
    __shared__ double sv[32], ss[32];
    __shared__ int64_t si[32];
    __shared__ double Lr[kBkW];
    __shared__ double pend[2][kBkW];
    __shared__ int pend_row[2], pend_n[2];
    __shared__ StepCoef coef[kBkW + 1];
    // published for the other CTAs (read through DSMEM after a cluster barrier)
    __shared__ double pub_v, pub_s, pub_rv;
    __shared__ int64_t pub_i;
    __shared__ double scal[8];  // [0] c_k(k) [1] c_k(k+1) [2] c_i(imax) [3] c_i(k) [4] c_i(k+1)
    // this CTA's copy of the cluster-wide decision inputs
    __shared__ double g_colmax, g_ckimax, g_rowmax, g_sc[5];
    __shared__ int64_t g_imax;
    const int64_t n = a.n;
    const int64_t k0 = a.ctl[0];
    if (k0 >= n) return;
    const int G = gridDim.x;
    const int64_t chunk = (n - k0 + G - 1) / G;
    const int64_t lo = k0 + chunk * blockIdx.x, hi = min(n, lo + chunk);
    const int R = static_cast<int>(hi > lo ? hi - lo : 0);
    const int64_t gtid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int64_t gthreads = static_cast<int64_t>(G) * blockDim.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* A = a.A;
    auto owner = [&](int64_t i) { return static_cast<int>((i - k0) / chunk); };
    auto local = [&](int64_t i) { return i - (k0 + chunk * owner(i)); };
    // row q of the panel's L (columns k0 .. k0+jp-1) from the owner's W row; a
    // row moved by the previous interchange is read from the owner's pending
    // copy (its W row is rewritten at the top of this column, concurrently)
    int64_t last_kk = -1, last_kp = -1;
    auto load_lrow = [&](int64_t q, int jp) {
        const double* w;
        if (q == last_kk) w = cl.map_shared_rank(&pend[0][0], owner(q));
        else if (q == last_kp) w = cl.map_shared_rank(&pend[1][0], owner(q));
        else w = cl.map_shared_rank(Ws, owner(q)) + local(q) * kBkW;
        l_row(w, coef, jp, Lr);
    };
    const bool tr = a.trace && blockIdx.x == 0 && threadIdx.x == 0;
    unsigned long long tprev = 0, tnow = 0;
    auto mark = [&](int ph) {
        if (!tr) return;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
        if (ph >= 0) a.trace[ph] += tnow - tprev;
        tprev = tnow;
    };
    mark(-1);
    if (threadIdx.x < 2) pend_row[threadIdx.x] = -1;
    __syncthreads();
    cl.sync();  // every CTA's shared memory is live before DSMEM use

    int64_t k = k0;
    int jp = 0;
    while (k < n && jp < kBkNb) {
        for (int p = 0; p < 2; ++p)
            if (pend_row[p] >= 0)
                for (int t = threadIdx.x; t < pend_n[p]; t += blockDim.x) Ws[pend_row[p] * kBkW + t] = pend[p][t];
        __syncthreads();
        if (threadIdx.x < 2) pend_row[threadIdx.x] = -1;
        load_lrow(k, jp);
        last_kk = last_kp = -1;
        __syncthreads();
        mark(0);
        // ---- updated column k on the CTA's rows
        double bv = -1.0, bs = 0.0;
        int64_t bi = n;
        for (int r = static_cast<int>(k > lo ? k - lo : 0) + threadIdx.x; r < R; r += blockDim.x) {
            const int64_t i = lo + r;
            double sacc = A[i + k * n];
            for (int t = 0; t < jp; ++t) sacc -= Ws[r * kBkW + t] * Lr[t];
            Cs[r] = sacc;
            if (i > k && (fabs(sacc) > bv || (fabs(sacc) == bv && i < bi))) {
                bv = fabs(sacc);
                bi = i;
                bs = sacc;
            }
            if (i == k) scal[0] = sacc;
            if (i == k + 1) scal[1] = sacc;
        }
        block_argmax3(bv, bi, bs, sv, si, ss);
        if (threadIdx.x == 0) {
            pub_v = bv;
            pub_i = bi;
            pub_s = bs;
        }
        mark(1);
        cl.sync();
        mark(2);
        if (warp == 0) {
            // all remote reads issued together: lanes < G the partials, lanes
            // 16 / 17 the scalars c_k(k), c_k(k+1)
            double v = -1.0, sg = 0.0;
            int64_t ii = n;
            if (lane < G) {
                v = *cl.map_shared_rank(&pub_v, lane);
                ii = *cl.map_shared_rank(&pub_i, lane);
                sg = *cl.map_shared_rank(&pub_s, lane);
            } else if (lane == 16) {
                g_sc[0] = *cl.map_shared_rank(&scal[0], owner(k));
            } else if (lane == 17) {
                g_sc[1] = k + 1 < n ? *cl.map_shared_rank(&scal[1], owner(k + 1)) : 0.0;
            }
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) {
                const double v2 = __shfl_xor_sync(0xffffffffu, v, off);
                const int64_t i2 = __shfl_xor_sync(0xffffffffu, ii, off);
                const double s2 = __shfl_xor_sync(0xffffffffu, sg, off);
                if (v2 > v || (v2 == v && i2 < ii)) {
                    v = v2;
                    ii = i2;
                    sg = s2;
                }
            }
            if (lane == 0) {
                g_colmax = v;
                g_imax = ii;
                g_ckimax = sg;
            }
        }
        __syncthreads();
        double colmax = g_colmax;
        int64_t imax = g_imax;
        const double ckimax = g_ckimax;
        if (colmax < 0.0) {
            colmax = 0.0;
            imax = k;
        }
        const double ckk = g_sc[0], ckk1 = g_sc[1];
        const double absakk = fabs(ckk);
        int kstep = 1;
        int64_t kp = k;
        double cimax = 0.0, cik = 0.0, cik1 = 0.0;
        mark(3);
        if (fmax(absakk, colmax) == 0.0) {
            for (int r = static_cast<int>(k > lo ? k - lo : 0) + threadIdx.x; r < R; r += blockDim.x) {
                A[(lo + r) + k * n] = Cs[r];
                Ws[r * kBkW + jp] = 0.0;
            }
            if (threadIdx.x == 0) coef[jp] = StepCoef{0, 0.0, 0.0, 0.0};
            if (gtid == 0) {
                a.ipiv[k] = static_cast<int>(k);
                a.ps[k] = 0;
                a.ctl[1] = 1;
            }
            k += 1;
            jp += 1;
            __syncthreads();
            cl.sync();
            continue;
        }
        if (!(absakk >= kBkAlpha * colmax)) {
            load_lrow(imax, jp);
            __syncthreads();
            double rv = -1.0;
            for (int r = static_cast<int>(k > lo ? k - lo : 0) + threadIdx.x; r < R; r += blockDim.x) {
                const int64_t i = lo + r;
                double sacc = i >= imax ? A[i + imax * n] : A[imax + i * n];
                for (int t = 0; t < jp; ++t) sacc -= Ws[r * kBkW + t] * Lr[t];
                Cis[r] = sacc;
                if (i != imax) rv = fmax(rv, fabs(sacc));
                if (i == imax) scal[2] = sacc;
                if (i == k) scal[3] = sacc;
                if (i == k + 1) scal[4] = sacc;
            }
            int64_t dummy = 0;
            double dd = 0.0;
            block_argmax3(rv, dummy, dd, sv, si, ss);
            if (threadIdx.x == 0) pub_rv = rv;
            mark(4);
            cl.sync();
            if (warp == 0) {
                double v = 0.0;
                if (lane < G) v = *cl.map_shared_rank(&pub_rv, lane);
                else if (lane == 16) g_sc[2] = *cl.map_shared_rank(&scal[2], owner(imax));
                else if (lane == 17) g_sc[3] = *cl.map_shared_rank(&scal[3], owner(k));
                else if (lane == 18) g_sc[4] = k + 1 < n ? *cl.map_shared_rank(&scal[4], owner(k + 1)) : 0.0;
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
                if (lane == 0) g_rowmax = v;
            }
            __syncthreads();
            const double rowmax = fmax(g_rowmax, 0.0);
            cimax = g_sc[2];
            cik = g_sc[3];
            cik1 = g_sc[4];
            if (tr) a.trace[8] += 1;
            if (absakk * rowmax >= kBkAlpha * colmax * colmax) {
                kp = k;
            } else if (fabs(cimax) >= kBkAlpha * rowmax) {
                kp = imax;
            } else {
                kp = imax;
                kstep = 2;
            }
        }
        const int64_t kk = k + kstep - 1;
        const bool swap = kp != kk;
        if (swap) {
            // rows of this panel's L columns (earlier panels keep their order:
            // the solve applies the interchanges panel by panel)
            for (int64_t t = k0 + gtid; t < k; t += gthreads) {
                const double u = A[kk + t * n];
                A[kk + t * n] = A[kp + t * n];
                A[kp + t * n] = u;
            }
            // W rows kk <-> kp through DSMEM; applied at the top of the next column
            const int okk = owner(kk), okp = owner(kp);
            for (int side = 0; side < 2; ++side) {
                const int me = side == 0 ? okk : okp;
                if (static_cast<int>(blockIdx.x) != me) continue;
                const int64_t dst = side == 0 ? kk : kp, src = side == 0 ? kp : kk;
                const double* remote = cl.map_shared_rank(Ws, owner(src)) + local(src) * kBkW;
                for (int t = threadIdx.x; t < jp; t += blockDim.x) pend[side][t] = remote[t];
                if (threadIdx.x == 0) {
                    pend_row[side] = static_cast<int>(dst - lo);
                    pend_n[side] = jp + kstep;  // + the new column(s), stored below
                }
            }
        }
        auto move_out = [&](int64_t i) {
            if (!swap) return;
            if (i > kp) A[i + kp * n] = A[i + kk * n];
            else if (i > kk && i < kp) A[kp + i * n] = A[i + kk * n];
            else if (i == kk) A[kp + kp * n] = A[kk + kk * n];
        };
        if (kstep == 1) {
            const double d = kp == k ? ckk : cimax;
            const bool zero = d == 0.0;
            const double r1 = zero ? 0.0 : 1.0 / d;
            for (int r = static_cast<int>(k > lo ? k - lo : 0) + threadIdx.x; r < R; r += blockDim.x) {
                const int64_t i = lo + r;
                const double v = kp == k ? Cs[r] : (i == k ? cimax : (i == kp ? cik : Cis[r]));
                move_out(i);
                const double wv = zero ? 0.0 : (i == k ? d : v);
                Ws[r * kBkW + jp] = wv;
                if (swap && i == kk) pend[0][jp] = wv;
                if (swap && i == kp) pend[1][jp] = wv;
                if (i == k) A[k + k * n] = d;
                else A[i + k * n] = zero ? v : v * r1;
            }
            if (threadIdx.x == 0) coef[jp] = StepCoef{zero ? 0 : 1, r1, 0.0, 0.0};
            if (gtid == 0) {
                a.ipiv[k] = static_cast<int>(kp);
                a.ps[k] = 0;
                if (zero) a.ctl[1] = 1;
            }
        } else {
            const bool same = kp == k + 1;
            const double nk_k = ckk, nk_k1 = same ? ckk1 : ckimax;
            const double nk1_k1 = cimax;
            const double d21 = nk_k1;
            const double d11 = nk1_k1 / d21;
            const double d22 = nk_k / d21;
            const double tt = 1.0 / (d11 * d22 - 1.0);
            const double d21t = tt / d21;
            for (int r = static_cast<int>(k > lo ? k - lo : 0) + threadIdx.x; r < R; r += blockDim.x) {
                const int64_t i = lo + r;
                const double x0 = same ? Cs[r] : (i == k + 1 ? ckimax : (i == kp ? ckk1 : Cs[r]));
                const double x1 = same ? Cis[r] : (i == k + 1 ? cimax : (i == kp ? cik1 : Cis[r]));
                move_out(i);
                Ws[r * kBkW + jp] = x0;
                Ws[r * kBkW + jp + 1] = x1;
                if (swap && i == kk) {
                    pend[0][jp] = x0;
                    pend[0][jp + 1] = x1;
                }
                if (swap && i == kp) {
                    pend[1][jp] = x0;
                    pend[1][jp + 1] = x1;
                }
                if (i == k) {
                    A[k + k * n] = x0;
                } else if (i == k + 1) {
                    A[k + 1 + k * n] = x0;
                    A[k + 1 + (k + 1) * n] = x1;
                } else {
                    A[i + k * n] = d21t * (d11 * x0 - x1);
                    A[i + (k + 1) * n] = d21t * (d22 * x1 - x0);
                }
            }
            if (threadIdx.x == 0) {
                coef[jp] = StepCoef{2, d21t, d11, d22};
                coef[jp + 1] = StepCoef{3, d21t, d11, d22};
            }
            if (gtid == 0) {
                a.ipiv[k] = static_cast<int>(-kp - 1);
                a.ipiv[k + 1] = static_cast<int>(-kp - 1);
                a.ps[k] = 1;
                a.ps[k + 1] = 2;
            }
        }
        if (swap) {
            last_kk = kk;
            last_kp = kp;
        }
        k += kstep;
        jp += kstep;
        mark(5);
        __syncthreads();
        cl.sync();
        mark(6);
        if (tr) a.trace[9] += 1;
    }
    for (int p = 0; p < 2; ++p)
        if (pend_row[p] >= 0)
            for (int t = threadIdx.x; t < pend_n[p]; t += blockDim.x) Ws[pend_row[p] * kBkW + t] = pend[p][t];
    __syncthreads();
    // the panel's W rows of this CTA -> global, for the trailing update
    for (int t = 0; t < jp; ++t)
        for (int r = threadIdx.x; r < R; r += blockDim.x) a.Wp[(lo + r) + t * n] = Ws[r * kBkW + t];
    if (gtid == 0) {
        a.perm[a.ctl[4]] = static_cast<int>(k0);  // panel starts, for the solve
        a.ctl[4] += 1;
        a.ctl[2] = static_cast<int>(k0);
        a.ctl[3] = jp;
        a.ctl[0] = static_cast<int>(k);
    }
    cl.sync();  // no CTA exits while others may still read its shared memory
}

// A22 -= W L^T, 128 x 128 tiles, 8 x 8 per thread (rows tx + 16 r, cols ty + 16 c:
// coalesced A traffic, conflict-free / broadcast shared loads).  The A tile is
// staged into shared memory with cp.async while the W L^T product is formed,
// so its HBM read overlaps the FP64 work.
constexpr int kBkT2 = 128;
constexpr size_t kBkUpdSmem = (2 * kBkW * kBkT2 + kBkT2 * kBkT2) * sizeof(double);

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
                 "l"(gmem)
                 : "memory");
}

__global__ void __launch_bounds__(kBkThreads, 1) bk_update2_kernel(const BkArgs a) {
    extern __shared__ __align__(16) double usm[];
    double* Wt = usm;                  // [kBkW][kBkT2]
    double* Lt = usm + kBkW * kBkT2;   // [kBkW][kBkT2]
    double* At = Lt + kBkW * kBkT2;    // [kBkT2 cols][kBkT2 rows]
    const int64_t n = a.n;
    const int64_t k0 = a.ctl[2];
    const int jp = a.ctl[3];
    const int64_t kend = k0 + jp;
    const int64_t m = n - kend;
    if (m <= 0 || jp == 0) return;
    const int64_t T = (m + kBkT2 - 1) / kBkT2;
    const int64_t ntiles = T * (T + 1) / 2;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    for (int64_t x = blockIdx.x; x < ntiles; x += gridDim.x) {
        int64_t bi = static_cast<int64_t>((sqrt(8.0 * static_cast<double>(x) + 1.0) - 1.0) * 0.5);
        while (bi * (bi + 1) / 2 > x) --bi;
        while ((bi + 1) * (bi + 2) / 2 <= x) ++bi;
        const int64_t bj = x - bi * (bi + 1) / 2;
        const int64_t i0 = kend + bi * kBkT2, j0 = kend + bj * kBkT2;
        const int rows = static_cast<int>(n - i0 < kBkT2 ? n - i0 : kBkT2);
        const int cols = static_cast<int>(n - j0 < kBkT2 ? n - j0 : kBkT2);
        __syncthreads();
        // W / L panels (needed first), then the A tile (needed last)
        for (int e = threadIdx.x; e < kBkT2 * jp; e += blockDim.x) {
            const int r = e % kBkT2, t = e / kBkT2;
            if (r < rows) cp_async8(&Wt[t * kBkT2 + r], a.Wp + (i0 + r) + t * n);
            else Wt[t * kBkT2 + r] = 0.0;
            if (r < cols) cp_async8(&Lt[t * kBkT2 + r], a.A + (j0 + r) + (k0 + t) * n);
            else Lt[t * kBkT2 + r] = 0.0;
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        for (int e = threadIdx.x; e < kBkT2 * cols; e += blockDim.x) {
            const int r = e % kBkT2, c = e / kBkT2;
            if (r < rows) cp_async8(&At[c * kBkT2 + r], a.A + (i0 + r) + (j0 + c) * n);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncthreads();
        double acc[8][8];
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[r][c] = 0.0;
        for (int t = 0; t < jp; ++t) {
            double w[8], l[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) w[r] = Wt[t * kBkT2 + tx + 16 * r];
#pragma unroll
            for (int c = 0; c < 8; ++c) l[c] = Lt[t * kBkT2 + ty + 16 * c];
#pragma unroll
            for (int r = 0; r < 8; ++r)
#pragma unroll
                for (int c = 0; c < 8; ++c) acc[r][c] = fma(w[r], l[c], acc[r][c]);
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        const bool diag = bi == bj;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const int cc = ty + 16 * c;
            if (cc >= cols) continue;
            const int64_t j = j0 + cc;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const int rr = tx + 16 * r;
                const int64_t i = i0 + rr;
                if (rr < rows && (!diag || i >= j)) a.A[i + j * n] = At[cc * kBkT2 + rr] - acc[r][c];
            }
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

// Largest cluster (<= 16, <= one CTA per 256 rows) the device can schedule.
int panel_cluster_size(r1_context* ctx, int64_t n) {
    static int max16 = -1;
    if (max16 < 0) {
        max16 = cudaFuncSetAttribute(bk_panel_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
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
    }
    (void)ctx;
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
           (2 * static_cast<size_t>(n) + 64) * sizeof(int) + static_cast<size_t>(n) + 64;
}

// Factor A (n x n, device, lower triangle; overwritten) and write the D-block
// condition (inf when singular) to cond_dev.  Async on ctx->stream.
void bk_factor(r1_context* ctx, int64_t n, double* A, void* ws, double* cond_dev) {
    const BkLayout L = bk_layout(ws, n, ctx->num_sms);
    R1_CUDA(cudaMemsetAsync(L.ctl, 0, 16 * sizeof(int), ctx->stream));
    bk_init_kernel<<<std::max(1, static_cast<int>(std::min<int64_t>((n + 255) / 256, 64))), 256, 0,
                     ctx->stream>>>(L.perm, L.ps, n);
    check_launch(ctx, "bk_init_kernel");
    static const bool trace = std::getenv("R1_BK_TRACE") != nullptr;
    static DeviceBuffer tbuf;
    if (trace) {
        tbuf.ensure(16 * sizeof(unsigned long long));
        R1_CUDA(cudaMemsetAsync(tbuf.ptr, 0, 16 * sizeof(unsigned long long), ctx->stream));
    }
    BkArgs a{n, A, L.Wp, L.ipiv, L.ctl, L.Ck, L.Ci, L.red, L.perm, L.ps,
             trace ? tbuf.as<unsigned long long>() : nullptr};
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
    const size_t psmem = static_cast<size_t>(rcap) * (kBkW + 2) * sizeof(double);
    const bool smem_panel = psmem <= 160 * 1024 && gp <= 16;
    static int configured = -1;
    if (configured != ctx->device) {
        R1_CUDA(cudaFuncSetAttribute(bk_panel_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     160 * 1024));
        R1_CUDA(cudaFuncSetAttribute(bk_panel_smem_kernel,
                                     cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        R1_CUDA(cudaFuncSetAttribute(bk_update2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(kBkUpdSmem)));
        configured = ctx->device;
    }
    if (smem_panel) cfg.dynamicSmemBytes = psmem;
    // each panel factors >= kBkNb columns (or the rest); extra launches exit at once
    const int64_t panels = (n + kBkNb - 1) / kBkNb;
    for (int64_t p = 0; p < panels; ++p) {
        if (smem_panel)
            R1_CUDA(cudaLaunchKernelEx(&cfg, bk_panel_smem_kernel, a, rcap));
        else
            R1_CUDA(cudaLaunchKernelEx(&cfg, bk_panel_kernel, a));
        check_launch(ctx, "bk_panel_kernel");
        bk_update2_kernel<<<ctx->num_sms, kBkThreads, kBkUpdSmem, ctx->stream>>>(a);
        check_launch(ctx, "bk_update2_kernel");
    }
    bk_condition_kernel<<<1, 1024, 0, ctx->stream>>>(A, n, L.ctl, L.ps, cond_dev);
    check_launch(ctx, "bk_condition_kernel");
    if (trace) {
        unsigned long long h[16];
        R1_CUDA(cudaMemcpyAsync(h, tbuf.ptr, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
        const double c = h[9] ? static_cast<double>(h[9]) : 1.0;
        std::fprintf(stderr,
                     "[r1 bk] n=%lld cols=%llu imax-path=%llu us/col: top %.2f step1 %.2f sync1 %.2f "
                     "decide %.2f imax %.2f elim %.2f sync_end %.2f\n",
                     static_cast<long long>(n), h[9], h[8], h[0] / c * 1e-3, h[1] / c * 1e-3,
                     h[2] / c * 1e-3, h[3] / c * 1e-3, h[4] / c * 1e-3, h[5] / c * 1e-3, h[6] / c * 1e-3);
    }
}

// y = (factored A)^-1 x, normalised; *ok_dev = finite and nonzero.
void bk_solve(r1_context* ctx, int64_t n, const double* A, void* ws, const double* x, double* y,
              int* ok_dev) {
    const BkLayout L = bk_layout(ws, n, ctx->num_sms);
    SolveArgs s{n, A, L.ipiv, L.ps, L.perm, L.ctl, x, L.z, y, L.part, ok_dev};
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

}  // extern "C"
