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
//     64x64 tiles staged in shared memory.
// The interchanges are applied to whole rows of L ("full-swap" form, P A P^T =
// L D L^T) instead of the reference's stepwise convention; D, the pivot
// sequence and the solution are the same (the reference's accept test only
// reads D).  Solve: one cooperative kernel (permute, blocked forward
// substitution, D^-1, blocked backward substitution, un-permute, normalise).
#include "common.cuh"

#include <cooperative_groups.h>

#include <cmath>
#include <vector>

namespace cg = cooperative_groups;

namespace r1 {

namespace {

constexpr int kBkNb = 32;          // panel columns (a 2x2 pivot may add one)
constexpr int kBkW = kBkNb + 1;    // columns of the panel workspace
constexpr int kBkThreads = 256;
constexpr int kBkTile = 64;        // trailing-update tile
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
    int* perm;    // composed interchanges: row i of P A P^T is row perm[i] of A
    char* ps;     // 0: 1x1 pivot, 1 / 2: first / second column of a 2x2 pivot
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
            if (gtid == 0) {
                const int u = a.perm[kk];
                a.perm[kk] = a.perm[kp];
                a.perm[kp] = u;
            }
            // whole rows of L (all earlier columns) and of the panel workspace
            for (int64_t t = gtid; t < k; t += gthreads) {
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
        a.ctl[2] = static_cast<int>(k0);
        a.ctl[3] = jp;
        a.ctl[0] = static_cast<int>(k);
    }
}

// A22 -= W L^T on the lower triangle of the trailing matrix [kend, n)^2.
__global__ void __launch_bounds__(kBkThreads) bk_update_kernel(const BkArgs a) {
    __shared__ double Ws[kBkTile][kBkW + 1];
    __shared__ double Ls[kBkTile][kBkW + 1];
    const int64_t n = a.n;
    const int64_t k0 = a.ctl[2];
    const int jp = a.ctl[3];
    const int64_t kend = k0 + jp;
    const int64_t m = n - kend;
    if (m <= 0 || jp == 0) return;
    const int64_t T = (m + kBkTile - 1) / kBkTile;
    const int64_t ntiles = T * (T + 1) / 2;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const double* A = a.A;
    for (int64_t x = blockIdx.x; x < ntiles; x += gridDim.x) {
        int64_t bi = static_cast<int64_t>((sqrt(8.0 * static_cast<double>(x) + 1.0) - 1.0) * 0.5);
        while (bi * (bi + 1) / 2 > x) --bi;
        while ((bi + 1) * (bi + 2) / 2 <= x) ++bi;
        const int64_t bj = x - bi * (bi + 1) / 2;
        const int64_t i0 = kend + bi * kBkTile, j0 = kend + bj * kBkTile;
        __syncthreads();
        for (int e = threadIdx.x; e < kBkTile * jp; e += blockDim.x) {
            const int r = e % kBkTile, t = e / kBkTile;
            const int64_t i = i0 + r, j = j0 + r;
            Ws[r][t] = i < n ? a.Wp[i + t * n] : 0.0;
            Ls[r][t] = j < n ? A[j + (k0 + t) * n] : 0.0;
        }
        __syncthreads();
        double acc[4][4] = {};
        for (int t = 0; t < jp; ++t) {
            double w[4], l[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) w[r] = Ws[ty + 16 * r][t];
#pragma unroll
            for (int c = 0; c < 4; ++c) l[c] = Ls[tx + 16 * c][t];
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[r][c] = fma(w[r], l[c], acc[r][c]);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int64_t j = j0 + tx + 16 * c;
            if (j >= n) continue;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int64_t i = i0 + ty + 16 * r;
                if (i < n && i >= j) a.A[i + j * n] -= acc[r][c];
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
    const char* ps;       // 0 1x1, 1 first of a 2x2, 2 second of a 2x2
    const int* perm;      // n
    const double* x;      // right-hand side
    double* z;            // n work
    double* y;            // n out (unit) when ok
    double* part;         // gridDim * kBkSolveB
    int* ok;
};

// L(i,k) of the full-swap factor (zero inside a 2x2 diagonal block)
__device__ __forceinline__ double lval(const SolveArgs& s, int64_t i, int64_t k) {
    return (i == k + 1 && s.ps[k] == 1) ? 0.0 : s.A[i + k * s.n];
}

__global__ void __launch_bounds__(kBkThreads) bk_solve_kernel(const SolveArgs s) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double sh[kBkSolveB + 32];
    const int64_t n = s.n;
    const int G = gridDim.x;
    const int64_t gtid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int64_t gthreads = static_cast<int64_t>(G) * blockDim.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    // ---- P b (the composed interchanges)
    for (int64_t i = gtid; i < n; i += gthreads) s.z[i] = s.x[s.perm[i]];
    grid.sync();
    // ---- forward: L z = P b, blocks of kBkSolveB columns
    for (int64_t c0 = 0; c0 < n; c0 += kBkSolveB) {
        const int64_t c1 = min(n, c0 + kBkSolveB);
        if (blockIdx.x == 0) {
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
    // ---- backward: L^T x = z, blocks from the bottom
    const int64_t nblk = (n + kBkSolveB - 1) / kBkSolveB;
    for (int64_t b = nblk - 1; b >= 0; --b) {
        const int64_t c0 = b * kBkSolveB, c1 = min(n, c0 + kBkSolveB);
        // partial dots over rows >= c1 (final), CTA-contiguous row ranges
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
        }
        grid.sync();
    }
    // ---- un-permute and normalise (sym_eig.cpp:425-431)
    for (int64_t i = gtid; i < n; i += gthreads) s.y[s.perm[i]] = s.z[i];
    grid.sync();
    if (blockIdx.x == 0) {
        double acc = 0.0;
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc = fma(s.y[i], s.y[i], acc);
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (lane == 0) sh[warp] = acc;
        __syncthreads();
        double tot = 0.0;
        for (int w = 0; w < nw; ++w) tot += sh[w];
        const double nrm = sqrt(tot);
        const bool good = isfinite(nrm) && nrm != 0.0;
        if (good)
            for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s.y[i] /= nrm;
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
    BkArgs a{n, A, L.Wp, L.ipiv, L.ctl, L.Ck, L.Ci, L.red, L.perm, L.ps};
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
    // each panel factors >= kBkNb columns (or the rest); extra launches exit at once
    const int64_t panels = (n + kBkNb - 1) / kBkNb;
    for (int64_t p = 0; p < panels; ++p) {
        R1_CUDA(cudaLaunchKernelEx(&cfg, bk_panel_kernel, a));
        check_launch(ctx, "bk_panel_kernel");
        bk_update_kernel<<<4 * ctx->num_sms, kBkThreads, 0, ctx->stream>>>(a);
        check_launch(ctx, "bk_update_kernel");
    }
    bk_condition_kernel<<<1, 1024, 0, ctx->stream>>>(A, n, L.ctl, L.ps, cond_dev);
    check_launch(ctx, "bk_condition_kernel");
}

// y = (factored A)^-1 x, normalised; *ok_dev = finite and nonzero.
void bk_solve(r1_context* ctx, int64_t n, const double* A, void* ws, const double* x, double* y,
              int* ok_dev) {
    const BkLayout L = bk_layout(ws, n, ctx->num_sms);
    SolveArgs s{n, A, L.ps, L.perm, x, L.z, y, L.part, ok_dev};
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
