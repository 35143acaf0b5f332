// Largest-magnitude eigenpair of J on the device.
//
// Replaces rank1::largest_magnitude_eigenpair(J.dense()) (reference
// proj/src/sym_eig.cpp:206-229: tred2 + implicit QL on the dense sum(I) x
// sum(I) matrix, O(n^3) per HOSCF iteration) by Lanczos:
//
//   * lanczos_kernel: one persistent cooperative kernel (grid = #SMs,
//     grid.sync between phases) runs the whole solve, the matvec through the
//     blocks (blockmv.cuh, never forming dense J); lanczos_cluster_kernel
//     (n <= 1024): the same algorithm on ONE thread-block cluster with the
//     rows of J, V and w in shared memory and DSMEM partial sums;
//   * full reorthogonalisation, classical Gram-Schmidt applied twice;
//   * every `check_every` steps CTA 0 computes BOTH extreme eigenvalues of
//     the tridiagonal T by Sturm-count multisection, their T-eigenvectors by
//     inverse iteration and the Ritz residual bounds |beta_m s_m|; the picked
//     end must reach tol, the other end only as far as the pick rule needs
//     (or the Krylov space is the whole space, then T's spectrum is exact);
//   * inside a solve the start vector is the previous eigenvector plus the
//     previous other-end Ritz vector, and the first check follows the
//     previous step count (both reset by the solve's cold first call);
//   * the reference's pick rule (lo iff |lo| > |hi| (1 + 1e-12),
//     sym_eig.cpp:214-216) and sign rule (largest-|entry| positive, first
//     index on ties, :223-227) are applied to the Ritz pair;
//   * a breakdown (invariant subspace) injects a fresh random direction;
//     non-convergence at the size limit restarts from the two extreme Ritz
//     vectors.
// All reductions have a fixed order over a fixed grid: deterministic.
#include "common.cuh"
#include "blockmv.cuh"
#include "dsmem.cuh"

#include <cooperative_groups.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

namespace cg = cooperative_groups;

namespace r1 {

namespace {

constexpr int kEigThreads = 512;
constexpr int kMaxKrylov = 512;
constexpr size_t kEigDynSmem = sizeof(double) * 14 * kMaxKrylov;

struct EigArgs {
    const BlockOp* op;
    int64_t n;
    int maxm;
    int check_every;
    int min_steps;
    int max_restarts;
    double tol;
    const double* x0;
    double* V;       // n x (maxm + 1), column-major
    double* w;       // n
    double* h;       // maxm + 1
    double* h2;      // maxm + 1
    double* alpha;   // maxm
    double* beta;    // maxm
    double* part;    // 4 * gridDim
    double* pdot1;   // gridDim x (kMaxKrylov+1) partial dots (CGS pass 1)
    double* pdot2;   // same, pass 2
    double* sT;      // 2 * maxm: T-eigenvectors (lo, hi)
    int* ctl;        // [0] state, [1] picked end, [2] steps, [3] restarts, [4] breakdowns
    double* stats;   // [theta_lo, theta_hi, res_lo, res_hi, value]
    double* out_value;
    double* out_vec;
    int cluster;     // 1: the grid is one thread-block cluster (hardware cluster barriers)
    int* hint;       // steps the previous warm-started solve of this operator took
    int warm;        // 1: x0 is the previous eigenvector (use and update *hint)
    const double* x1;  // previous solve's other-end Ritz vector (start = x0 + x1), or null
    double* other_out; // this solve's other-end Ritz vector (unit), or null
    int debug_text;    // development: print the phase split of t_extremes
    double warm_noise; // weight of the random component of a warm start vector
    double decide_tol; // relative Ritz residual at which the non-picked end counts as decided
    const struct LzTiles* tl;  // tiled matvec plan (TILED grid kernel), device
    unsigned long long* lzt;   // diagnostics (R1_DEBUG_EIG): CTA 1's phase-A split, ns
};

__device__ __forceinline__ double hash_unit(uint64_t i, uint64_t salt) {
    uint64_t z = i * 0x9e3779b97f4a7c15ull + salt;
    z ^= z >> 30;
    z *= 0xbf58476d1ce4e5b9ull;
    z ^= z >> 27;
    z *= 0x94d049bb133111ebull;
    z ^= z >> 31;
    return static_cast<double>(z >> 11) * 0x1.0p-53 * 2.0 - 1.0;
}

// Fixed-order CTA reduction; result valid in every thread.
__device__ double cta_sum(double v, double* sh) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    double s = 0.0;
    const int nw = blockDim.x >> 5;
    for (int k = 0; k < nw; ++k) s += sh[k];
    return s;
}

// Sum of gridDim partials stored at part[slot*gridDim + b], identical in all threads.
__device__ double grid_total(const double* part, int slot) {
    double s = 0.0;
    for (int b = 0; b < static_cast<int>(gridDim.x); ++b) s += part[slot * gridDim.x + b];
    return s;
}

// Number of eigenvalues of the symmetric tridiagonal (a, b) that are < x:
// sign changes of the leading principal minors p_k(x) = (a_k - x) p_{k-1} -
// b_{k-1}^2 p_{k-2} (Sturm).  No division on the chain (a division per step
// made this ~160 cycles per row); the pair (p_{k-1}, p_k) is rescaled by an
// exact power of two every 8 rows, which keeps the signs.  A zero minor
// counts as a sign change (the pivmin convention of the LDL^T form: d_k =
// p_k / p_{k-1} = 0 is replaced by a tiny negative pivot).
__device__ int sturm_count(const double* a, const double* b2, int m, double x) {
    int c = 0;
    double pm = 1.0, p = a[0] - x;
    bool neg = !(p > 0.0);  // sign of the last minor as used for counting
    c += neg;
    auto step = [&](int i) {
        const double pn = fma(a[i] - x, p, -b2[i - 1] * pm);
        pm = p;
        p = pn;
        // sign / zero tests on the bits (integer pipe, not the FP64 pipe)
        const long long bits = __double_as_longlong(p);
        const bool ng = (bits << 1) == 0 ? !neg : bits < 0;
        c += ng != neg;
        neg = ng;
    };
    auto rescale = [&]() {
        const double mx = fmax(fabs(p), fabs(pm));
        const int e = mx > 0.0 && mx < INFINITY ? ilogb(mx) : 0;
        if (e > 512 || e < -512) {
            p = scalbn(p, -e);
            pm = scalbn(pm, -e);
        }
    };
    // blocks of 8 rows: the loads and a_i - x hoist off the chain, which is
    // then one FMA per row
    int i = 1;
    for (; i + 8 <= m; i += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) step(i + u);
        rescale();
    }
    for (; i < m; ++i) step(i);
    return c;
}

// Inverse iteration for the eigenvector of T (size m) at shift theta; s unit.
__device__ void tri_eigvec(const double* a, const double* b, int m, double theta, double tnorm,
                           double* s, double* work) {
    // work: d[m] (then 1 / d), du[m], du2[m], l[m], row-swap flags[m].  One
    // thread; the recurrences carry their running values in registers so a
    // step's chain is one or two FMAs (shared-memory round trips on the chain
    // made the three passes ~40 us at m = 64).
    double* d = work;
    double* du = work + m;
    double* du2 = work + 2 * m;
    double* l = work + 3 * m;
    double* sw = work + 4 * m;  // 1.0 if rows i,i+1 were swapped
    const double tiny = 1e-300 + 2.2e-16 * tnorm;
    // LU with partial pivoting of the tridiagonal (LAPACK dgttrf pattern); at
    // step i only d[i] / du[i] may differ from T's (changed by step i-1)
    double di = a[0] - theta, dui = m > 1 ? b[0] : 0.0;
    for (int i = 0; i + 1 < m; ++i) {
        const double sub = b[i];  // T(i+1, i)
        const double dn = a[i + 1] - theta;
        const double dun = i + 2 < m ? b[i + 1] : 0.0;
        if (fabs(di) >= fabs(sub)) {
            const double f = di != 0.0 ? sub / di : 0.0;
            sw[i] = 0.0;
            l[i] = f;
            d[i] = di;
            du[i] = dui;
            du2[i] = 0.0;
            di = dn - f * dui;
            dui = dun;
        } else {
            const double f = di / sub;
            sw[i] = 1.0;
            l[i] = f;
            d[i] = sub;
            du[i] = dn;
            du2[i] = dun;
            di = dui - f * dn;
            dui = -f * dun;
        }
    }
    d[m - 1] = di;
    du[m - 1] = 0.0;
    du2[m - 1] = 0.0;
    // reciprocals of U's diagonal (independent of each other), then the
    // substitution passes multiply.  theta is accurate to the last bits
    // (multisection), so one pass from the all-ones vector already amplifies
    // the eigencomponent by gap / |theta - lambda| (>= ~1e12); the second
    // leaves only rounding (a third, as in round 1, changed nothing but the
    // check's latency: ~4 us of a ~25 us check)
    for (int i = 0; i < m; ++i) {
        double v = d[i];
        if (fabs(v) < tiny) v = v < 0 ? -tiny : tiny;
        d[i] = 1.0 / v;
    }
    for (int i = 0; i < m; ++i) s[i] = 1.0;
    for (int it = 0; it < 2; ++it) {
        // forward: apply L^-1 P
        double prev = s[0];
#pragma unroll 4
        for (int i = 0; i + 1 < m; ++i) {
            const double nxt = s[i + 1], li = l[i];
            if (sw[i] == 0.0) {
                s[i] = prev;
                prev = nxt - li * prev;
            } else {
                s[i] = nxt;
                prev = prev - li * nxt;
            }
        }
        s[m - 1] = prev;
        // back: U^-1 (d holds 1 / U(i,i))
        double n1 = s[m - 1] * d[m - 1], n0 = 0.0;
        s[m - 1] = n1;
        if (m > 1) {
            n0 = (s[m - 2] - du[m - 2] * n1) * d[m - 2];
            s[m - 2] = n0;
        }
#pragma unroll 4
        for (int i = m - 3; i >= 0; --i) {
            const double v = (s[i] - du[i] * n0 - du2[i] * n1) * d[i];
            s[i] = v;
            n1 = n0;
            n0 = v;
        }
        double q0 = 0.0, q1 = 0.0;
        int i = 0;
        for (; i + 1 < m; i += 2) {
            q0 = fma(s[i], s[i], q0);
            q1 = fma(s[i + 1], s[i + 1], q1);
        }
        if (i < m) q0 = fma(s[i], s[i], q0);
        const double inv = 1.0 / sqrt(q0 + q1);
        for (int k = 0; k < m; ++k) s[k] *= inv;
    }
}

// CTA 0: extremes of T_m, eigenvectors, bounds, convergence decision.
__device__ void t_extremes(const EigArgs& a, int m, double beta_last, bool exact, int restarts,
                           double* scratch, int stride) {
    // tridiagonal, two inverse-iteration workspaces and the two T-eigenvectors
    // live in shared memory: 14 * stride doubles at scratch (stride >= m)
    double* ta = scratch;
    double* tb = ta + stride;
    double* work = tb + stride;
    double* work2 = work + 5 * stride;
    double* sv[2] = {work2 + 5 * stride, work2 + 6 * stride};
    __shared__ double lohi[4];  // [a_lo, b_lo, a_hi, b_hi] intervals
    __shared__ int cnt[kEigThreads];
    __shared__ double theta[2];
    // alpha/beta[m-1] were stored by thread 0 of this CTA: order them before the reads
    __threadfence_block();
    __syncthreads();
    unsigned long long t_dbg0 = 0, t_dbg1 = 0, t_dbg2 = 0, t_dbg3 = 0;
    if (a.debug_text && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_dbg0));

    double* b2 = work;  // squared off-diagonal for the Sturm counts (work is free until the eigvecs)
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        ta[i] = a.alpha[i];
        tb[i] = i + 1 < m ? a.beta[i] : 0.0;
        b2[i] = tb[i] * tb[i];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double lo = 1e300, hi = -1e300, tn = 0.0;
        for (int i = 0; i < m; ++i) {
            const double r = fabs(i > 0 ? tb[i - 1] : 0.0) + fabs(i + 1 < m ? tb[i] : 0.0);
            lo = fmin(lo, ta[i] - r);
            hi = fmax(hi, ta[i] + r);
            tn = fmax(tn, fabs(ta[i]) + r);
        }
        const double pad = 1e-14 * tn + 1e-300;
        lohi[0] = lo - pad;
        lohi[1] = hi + pad;
        lohi[2] = lo - pad;
        lohi[3] = hi + pad;
        theta[0] = tn;  // temp: T norm
    }
    __syncthreads();
    unsigned long long t_dbgA = 0;
    int rounds_dbg = 0;
    if (a.debug_text && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_dbgA));
    const double tnorm = theta[0];
    // 0: lowest, 1: highest; NP points per side and round (more points per
    // round only add FP64-pipe pressure: 128 -> 8 rounds to full precision)
    const int half = blockDim.x / 2;
    const int side = threadIdx.x < half ? 0 : 1;
    const int k = threadIdx.x - side * half;
    const int NP = min(half, 128);
    __shared__ int found[2];
    auto narrow = [&](int sd) {
        const double lo = lohi[2 * sd], hi = lohi[2 * sd + 1];
        return !(hi - lo <= 2.2e-16 * fmax(fabs(lo), fabs(hi)) + 1e-300);
    };
    for (int round = 0; round < 12; ++round) {
        // every thread takes every barrier: the two halves may finish in
        // different rounds, so a finished half idles instead of leaving
        if (!narrow(0) && !narrow(1)) break;  // uniform: read after a barrier
        ++rounds_dbg;
        const bool active = narrow(side) && k < NP;
        const double lo = lohi[2 * side], hi = lohi[2 * side + 1];
        if (active) {
            const double x = lo + (hi - lo) * static_cast<double>(k + 1) / static_cast<double>(NP + 1);
            cnt[threadIdx.x] = sturm_count(ta, b2, m, x);
        }
        if (k == 0) found[side] = NP;
        __syncthreads();
        // lowest: first point with count >= 1; highest: first with count >= m
        const int target = side == 0 ? 1 : m;
        if (active) {
            const bool hit = cnt[threadIdx.x] >= target;
            const bool prev = k > 0 && cnt[threadIdx.x - 1] >= target;
            if (hit && !prev) found[side] = k;  // counts are monotone: one writer
        }
        __syncthreads();
        if (k == 0 && narrow(side)) {
            const int f = found[side];
            const double nlo = f == 0 ? lo : lo + (hi - lo) * static_cast<double>(f) / (NP + 1);
            const double nhi = f == NP ? hi : lo + (hi - lo) * static_cast<double>(f + 1) / (NP + 1);
            lohi[2 * side] = nlo;
            lohi[2 * side + 1] = nhi;
        }
        __syncthreads();
    }
    if (a.debug_text && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_dbg1));
    if (threadIdx.x == 0 || threadIdx.x == half) {
        const double th = 0.5 * (lohi[2 * side] + lohi[2 * side + 1]);
        theta[side] = th;
        tri_eigvec(ta, tb, m, th, tnorm, sv[side], side == 0 ? work : work2);
    }
    __syncthreads();
    if (a.debug_text && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_dbg2));
    if (threadIdx.x == 0) {
        const double res_lo = fabs(beta_last * sv[0][m - 1]);
        const double res_hi = fabs(beta_last * sv[1][m - 1]);
        const double scale = fmax(fabs(theta[0]), fabs(theta[1]));
        const int pick = fabs(theta[0]) > fabs(theta[1]) * (1.0 + 1e-12) ? 0 : 1;
        // The picked end must be converged to tol.  The other end matters only
        // through the pick rule: it is enough that it is a Ritz value with a
        // small residual (decide_tol relative: 1e-6 by default, 1e-4 in the
        // HOSCF chain, where the warm start carries the previous iteration's
        // vector of that end, so it is not a stray Ritz value) whose magnitude
        // is on the losing side by a 100-residual margin (close calls keep
        // iterating).  At 1e-6 C1's eigen step took 40 Lanczos steps for a
        // decision the margin settles at ~24.  iHOSCF keeps 1e-6: its RQI
        // accept test compares Rayleigh quotients equal to the last ulp, and
        // the tighter eigen step keeps its trajectory closest to the reference.
        const double rp = pick ? res_hi : res_lo, ro = pick ? res_lo : res_hi;
        const double tp = fabs(theta[pick]), to = fabs(theta[1 - pick]);
        const bool decided = ro <= a.decide_tol * scale && to + 100.0 * ro < tp * (1.0 - 1e-6);
        const bool conv = exact || (rp <= a.tol * scale && (ro <= a.tol * scale || decided));
        a.stats[0] = theta[0];
        a.stats[1] = theta[1];
        a.stats[2] = res_lo;
        a.stats[3] = res_hi;
        a.stats[4] = theta[pick];
        a.ctl[0] = conv ? 1 : 0;
        a.ctl[1] = pick;
        a.ctl[2] = m;
        a.ctl[3] = restarts;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        a.sT[i] = sv[0][i];
        a.sT[kMaxKrylov + i] = sv[1][i];
    }
    if (a.debug_text && threadIdx.x == 0) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_dbg3));
        printf("[t_extremes] m=%d load+gersh %.1f us multisection %.1f us (%d rounds) eigvec %.1f us tail %.1f us\n",
               m, (t_dbgA - t_dbg0) * 1e-3, (t_dbg1 - t_dbgA) * 1e-3, rounds_dbg, (t_dbg2 - t_dbg1) * 1e-3,
               (t_dbg3 - t_dbg2) * 1e-3);
    }
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// ---------------------------------------------------------------------------
// Tiled block matvec of the grid kernel (block operators, n > kSmallN).
//
// Every block B(p) (I_m x I_n, column-major) is cut into row chunks of
// Rc <= 32 * kLzNQ rows; the (pair, row chunk, column) units are split into
// gridDim contiguous ranges of equal cost, one per CTA ("segments": the part
// of a range inside one row chunk).  A warp takes a column of its segment,
// lane l the rows l + 32 q: ONE read of each block entry (L2 evict_last, so
// the 88 MB of C5's blocks stay on chip across the Lanczos steps) feeds both
// the column dot (B' x_m)[c] over the chunk (warp-reduced, complete) and the
// lane's row accumulators (B x_n)[i] (summed over the warps in shared memory
// into one row partial per segment).  The CGS pass-1 dots V' (J x) are folded
// into the same phase from the partials (every contribution to J x lives in
// exactly one CTA), so a Lanczos step needs three grid barriers, not four.
// The plan is fixed per operator shape: every sum has a fixed order.
constexpr int kLzNQ = 4;     // rows per lane (row chunk <= 128)
constexpr int kLzWarps = kEigThreads / 32;

struct LzSeg {
    int p, rc, c0, c1;  // pair, row chunk, columns [c0, c1)
    long long rp;       // row-partial slot (rows of the chunk)
};

struct LzTiles {
    int nrc[kMvMaxPairs] = {};
    int Rc[kMvMaxPairs] = {};
    int rcseg_off[kMvMaxPairs] = {};  // index of (p, 0) in rc_first
    int64_t cd_off[kMvMaxPairs] = {}; // column dots of pair p: [rc][I_n]
    unsigned char v2[kMvMaxPairs] = {};  // pair p's columns are 16-B aligned (double2 loads)
    const LzSeg* segs = nullptr;
    const int* cta_seg = nullptr;     // [G + 1]
    // phase-B metadata, one int array: rc_first[nrcf + 1] (first segment of
    // each (p, rc) + sentinel), then seg_rp[nseg] (row-partial slot of each
    // segment); copied to shared memory when it fits kLzMetaInts
    const int* meta = nullptr;
    int nrcf = 0, nseg = 0;
    double* coldot = nullptr;
    double* rowpart = nullptr;
};

constexpr int kLzMetaInts = 6144;  // 24 KB of shared memory for the phase-B metadata
constexpr size_t kLzDynSmem = sizeof(double) * 14 * kMaxKrylov + sizeof(int) * kLzMetaInts;

__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ double ld_keep(const double* p, uint64_t pol) {
    double v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}

__device__ __forceinline__ double2 ld_keep2(const double* p, uint64_t pol) {
    double2 v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
        : "=d"(v.x), "=d"(v.y)
        : "l"(p), "l"(pol));
    return v;
}

// Phase A of the tiled matvec on x (= V[:, kmax]) plus the CGS pass-1 dot
// partials pdot[blockIdx.x * ld + k] = sum over this CTA's contributions c to
// J x (unscaled) of V[row(c), k] c, k <= kmax.  red: kLzWarps * 32 kLzNQ
// doubles, rps: 32 kLzNQ, dacc: kmax + 1 (shared memory).
__device__ __noinline__ void lz_phase_a(const BlockOp& op, const LzTiles& tl, const double* __restrict__ x,
                           const double* __restrict__ V, int64_t n, int kmax, double* pdot, int ld,
                           double* red, double* rps, double* dacc, unsigned long long* tdbg) {
    unsigned long long tq0 = 0, tq1 = 0, tq2 = 0;
    auto tmark = [&](int slot, unsigned long long& last) {
        if (tdbg && threadIdx.x == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (slot >= 0) tdbg[slot] += t - last;
            last = t;
        }
    };
    tmark(-1, tq0);
    constexpr int RMAX = 32 * kLzNQ;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t pol = policy_evict_last();
    for (int k = threadIdx.x; k <= kmax; k += blockDim.x) dacc[k] = 0.0;
    const int s_end = tl.cta_seg[blockIdx.x + 1];
    for (int s = tl.cta_seg[blockIdx.x]; s < s_end; ++s) {
        const LzSeg sg = tl.segs[s];
        const int p = sg.p, m = op.pm[p], nn = op.pn[p];
        const int64_t rows = op.dims[m], cols = op.dims[nn];
        const int64_t i0 = static_cast<int64_t>(sg.rc) * tl.Rc[p];
        const int nr = static_cast<int>(min(static_cast<int64_t>(tl.Rc[p]), rows - i0));
        const double* B = op.blocks + op.boff[p] + i0;
        const double* xm = x + op.offs[m] + i0;
        const double* xn = x + op.offs[nn];
        double* cd = tl.coldot + tl.cd_off[p] + static_cast<int64_t>(sg.rc) * cols;
        // lane rows: r(q) = 64 (q / 2) + 2 lane + (q & 1) — two consecutive
        // rows per lane and pair of q, so aligned columns load as double2
        double xr[kLzNQ], racc[kLzNQ];
#pragma unroll
        for (int q = 0; q < kLzNQ; ++q) {
            const int r = 64 * (q >> 1) + 2 * lane + (q & 1);
            xr[q] = r < nr ? xm[r] : 0.0;
            racc[q] = 0.0;
        }
        auto column_dot = [&](const double (&b)[kLzNQ], double xc) {
            double dd = 0.0;
#pragma unroll
            for (int q = 0; q < kLzNQ; ++q) {
                racc[q] = fma(b[q], xc, racc[q]);
                dd = fma(b[q], xr[q], dd);
            }
            return dd;
        };
        auto load_col = [&](double (&b)[kLzNQ], const double* col, bool v2) {
            if (v2) {
#pragma unroll
                for (int h = 0; h < kLzNQ / 2; ++h) {
                    const int r = 64 * h + 2 * lane;
                    double2 v = make_double2(0.0, 0.0);
                    if (r + 1 < nr) {
                        v = ld_keep2(col + r, pol);
                    } else if (r < nr) {
                        v.x = ld_keep(col + r, pol);
                    }
                    b[2 * h] = v.x;
                    b[2 * h + 1] = v.y;
                }
            } else {
#pragma unroll
                for (int q = 0; q < kLzNQ; ++q) {
                    const int r = 64 * (q >> 1) + 2 * lane + (q & 1);
                    b[q] = r < nr ? ld_keep(col + r, pol) : 0.0;
                }
            }
        };
        const bool v2 = tl.v2[p] != 0;
        // four columns per iteration: 4 * kLzNQ doubles in flight per lane
        // (software-pipelining two such sets measured slower: branches and
        // register pressure at the 128-register cap)
        constexpr int CU = 4;
        int c = sg.c0 + warp;
        for (; c + (CU - 1) * kLzWarps < sg.c1; c += CU * kLzWarps) {
            double b[CU][kLzNQ];
#pragma unroll
            for (int u = 0; u < CU; ++u) load_col(b[u], B + static_cast<int64_t>(c + u * kLzWarps) * rows, v2);
            double dd[CU];
#pragma unroll
            for (int u = 0; u < CU; ++u) dd[u] = column_dot(b[u], xn[c + u * kLzWarps]);
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1)
#pragma unroll
                for (int u = 0; u < CU; ++u) dd[u] += __shfl_xor_sync(0xffffffffu, dd[u], off);
            if (lane == 0)
#pragma unroll
                for (int u = 0; u < CU; ++u) cd[c + u * kLzWarps] = dd[u];
        }
        for (; c < sg.c1; c += kLzWarps) {
            double b[kLzNQ];
            load_col(b, B + static_cast<int64_t>(c) * rows, v2);
            double dd = column_dot(b, xn[c]);
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) dd += __shfl_xor_sync(0xffffffffu, dd, off);
            if (lane == 0) cd[c] = dd;
        }
        tq1 = tq0;
        tmark(0, tq1);  // column loop (thread 0's view)
        // row partial of the segment: the warps' accumulators in warp order
#pragma unroll
        for (int q = 0; q < kLzNQ; ++q) red[warp * RMAX + 64 * (q >> 1) + 2 * lane + (q & 1)] = racc[q];
        __syncthreads();
        for (int r = threadIdx.x; r < nr; r += blockDim.x) {
            double v = 0.0;
#pragma unroll
            for (int w = 0; w < kLzWarps; ++w) v += red[w * RMAX + r];
            rps[r] = v;
            tl.rowpart[sg.rp + r] = v;
        }
        __syncthreads();
        tq2 = tq1;
        tmark(1, tq2);
        // CGS pass-1 dot partials of this segment's contributions (warp per k)
        const double* vm = V + op.offs[m] + i0;
        const double* vn = V + op.offs[nn];
        for (int k = warp; k <= kmax; k += kLzWarps) {
            const int64_t ko = static_cast<int64_t>(k) * n;
            double t = 0.0;
#pragma unroll
            for (int q = 0; q < kLzNQ; ++q) {  // rows: all loads issued together
                const int r = lane + 32 * q;
                t = fma(r < nr ? vm[ko + r] : 0.0, r < nr ? rps[r] : 0.0, t);
            }
            int cc = sg.c0 + lane;
            for (; cc + 7 * 32 < sg.c1; cc += 8 * 32) {
                double vv[8], cv[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    vv[u] = vn[ko + cc + 32 * u];
                    cv[u] = cd[cc + 32 * u];
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) t = fma(vv[u], cv[u], t);
            }
            for (; cc < sg.c1; cc += 32) t = fma(vn[ko + cc], cd[cc], t);
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
            if (lane == 0) dacc[k] += t;
        }
        __syncthreads();
        tq0 = tq2;
        tmark(2, tq0);
    }
    for (int k = threadIdx.x; k <= kmax; k += blockDim.x) pdot[static_cast<int64_t>(blockIdx.x) * ld + k] = dacc[k];
}

// (J x)[t] / scale for one row t, summed by an 8-lane group (sub-lane sl):
// the column dots of the pairs (k, m), k < m (one per row chunk) and the row
// partials of the pairs (m, n), n > m (one per segment of the row's chunk),
// strided over the group in a fixed enumeration, then a fixed shuffle tree.
// All 32 lanes must call (shuffles); the result is in every lane of the group.
__device__ double lz_row_sum8(const BlockOp& op, const LzTiles& tl, const int* meta, int64_t t, int sl) {
    const int d = op.d;
    int m = 0;
    while (t >= op.offs[m + 1]) ++m;
    const int64_t i = t - op.offs[m];
    const int* rc_first = meta;
    const int* seg_rp = meta + tl.nrcf + 1;
    double s = 0.0;
    int base = 0;  // enumeration index of the next contribution
    for (int k = 0; k < m; ++k) {
        const int p = pair_index(k, m, d);
        const int cnt = tl.nrc[p];
        for (int e = (sl - base) & 7; e < cnt; e += 8)
            s += tl.coldot[tl.cd_off[p] + static_cast<int64_t>(e) * op.dims[m] + i];
        base += cnt;
    }
    for (int nn = m + 1; nn < d; ++nn) {
        const int p = pair_index(m, nn, d);
        const int rc = static_cast<int>(i / tl.Rc[p]);
        const int64_t r = i - static_cast<int64_t>(rc) * tl.Rc[p];
        const int sf = rc_first[tl.rcseg_off[p] + rc], se = rc_first[tl.rcseg_off[p] + rc + 1];
        const int cnt = se - sf;
        for (int e = (sl - base) & 7; e < cnt; e += 8) s += tl.rowpart[seg_rp[sf + e] + r];
        base += cnt;
    }
#pragma unroll
    for (int off = 4; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    return s;
}

// TILED = false: the round-1 kernel (dense operators; development switch
// R1_EIG_TILED=0 for block operators) — phase A partials, phase B, CGS2 with
// its own passes, four grid barriers per step.
// TILED = true (block operators): lz_phase_a (single read, CGS pass 1 folded),
// then own rows y -> w1 = y - V h1 with the pass-2 dots and ||w1||^2, then
// v_{j+1} = (w1 - V h2) / beta with beta^2 = ||w1||^2 - ||h2||^2: three
// grid barriers per step.
template <bool TILED>
__global__ void __launch_bounds__(kEigThreads, 1) lanczos_kernel(const EigArgs a) {
    cg::grid_group grid = cg::this_grid();
    // one-CTA launches (small operators) synchronise with the CTA barrier
    auto gsync = [&]() {
        if (gridDim.x == 1)
            __syncthreads();
        else if (a.cluster)
            cg::this_cluster().sync();
        else
            grid.sync();
    };
    // diagnostics: per-phase ns accumulated by CTA 0 thread 0 (stats[8..15])
    unsigned long long tacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    unsigned long long tlast = gtimer();
    auto mark = [&](int ph) {
        const unsigned long long t = gtimer();
        tacc[ph] += t - tlast;
        tlast = t;
    };
    __shared__ BlockOp op;
    __shared__ LzTiles tls;
    __shared__ double red[32];
    __shared__ double hsh[kMaxKrylov + 1];
    if (threadIdx.x == 0) {
        op = *a.op;
        if (TILED) tls = *a.tl;
    }
    __syncthreads();
    // phase-B metadata of the tiled matvec: shared memory when it fits
    const int* lzmeta = nullptr;
    if constexpr (TILED) {
        extern __shared__ double dsm[];
        const int cnt = tls.nrcf + 1 + tls.nseg;
        if (cnt <= kLzMetaInts) {
            int* sm = reinterpret_cast<int*>(dsm + 14 * kMaxKrylov);
            for (int e = threadIdx.x; e < cnt; e += blockDim.x) sm[e] = tls.meta[e];
            lzmeta = sm;
            __syncthreads();
        } else {
            lzmeta = tls.meta;
        }
    }
    const int64_t n = a.n;
    const int64_t gtid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t gstride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int G = gridDim.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    // Row ownership: CTA b owns rows [r0, r1) of every length-n vector; the
    // reorthogonalisation works on own rows + fixed-order partial sums.
    const int64_t R = (n + G - 1) / G;
    const int64_t r0 = min(n, static_cast<int64_t>(blockIdx.x) * R);
    const int64_t r1 = min(n, r0 + R);
    const int ld = kMaxKrylov + 1;

    // partial dots out[b*ld + k] = sum_{t in own rows} V[t,k] w[t], k <= kmax
    auto partial_dots = [&](double* out, int kmax) {
        for (int k = warp; k <= kmax; k += nw) {
            const double* vk = a.V + static_cast<int64_t>(k) * n;
            double s0 = 0.0, s1 = 0.0;
            int64_t t = r0 + lane;
            for (; t + 32 < r1; t += 64) {
                s0 = fma(vk[t], a.w[t], s0);
                s1 = fma(vk[t + 32], a.w[t + 32], s1);
            }
            if (t < r1) s0 = fma(vk[t], a.w[t], s0);
            double s = s0 + s1;
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
            if (lane == 0) out[static_cast<int64_t>(blockIdx.x) * ld + k] = s;
        }
    };
    // hsh[k] = sum_b in[b*ld + k]: warp per k, lanes over b, fixed shuffle
    // tree (the same order in every CTA -> the same bits everywhere)
    auto reduce_dots = [&](const double* in, int kmax) {
        for (int k = warp; k <= kmax; k += nw) {
            double s = 0.0;
            for (int b = lane; b < G; b += 32) s += in[static_cast<int64_t>(b) * ld + k];
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
            if (lane == 0) hsh[k] = s;
        }
        __syncthreads();
    };
    // sum of the G partials part[slot*G + b], broadcast to the CTA
    auto grid_sum = [&](const double* part, int slot) {
        if (warp == 0) {
            double s = 0.0;
            for (int b = lane; b < G; b += 32) s += part[slot * G + b];
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
            if (lane == 0) red[31] = s;
        }
        __syncthreads();
        const double v = red[31];
        __syncthreads();
        return v;
    };
    // own rows: w[t] -= sum_k V[t,k] hsh[k]; returns the CTA's sum of w^2 (thread 0)
    auto update_rows = [&](int kmax, bool norm) {
        double ss = 0.0;
        for (int64_t t = r0 + warp; t < r1; t += nw) {
            double s = 0.0;
            for (int k = lane; k <= kmax; k += 32) s = fma(a.V[t + static_cast<int64_t>(k) * n], hsh[k], s);
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
            const double wt = a.w[t] - s;
            if (lane == 0) a.w[t] = wt;
            ss = fma(wt, wt, ss);
        }
        __syncwarp();
        if (norm) {
            ss = lane == 0 ? ss : 0.0;
            ss = cta_sum(ss, red);
            if (threadIdx.x == 0) a.part[blockIdx.x] = ss;
        }
        __syncthreads();
    };
    // CGS2 of w (own rows) against V[:, 0..kmax]; leaves ||w||^2 partials in part[0..G)
    auto cgs2 = [&](int kmax) {
        partial_dots(a.pdot1, kmax);
        gsync();
        reduce_dots(a.pdot1, kmax);
        update_rows(kmax, false);
        partial_dots(a.pdot2, kmax);
        gsync();
        reduce_dots(a.pdot2, kmax);
        update_rows(kmax, true);
        gsync();
    };

    // ---- start vector -> V[:,0]
    auto set_v0_from_w = [&]() {
        double s = 0.0;
        for (int64_t t = r0 + threadIdx.x; t < r1; t += blockDim.x) s = fma(a.w[t], a.w[t], s);
        s = cta_sum(s, red);
        if (threadIdx.x == 0) a.part[blockIdx.x] = s;
        gsync();
        const double nrm = sqrt(grid_sum(a.part, 0));
        for (int64_t t = r0 + threadIdx.x; t < r1; t += blockDim.x) a.V[t] = a.w[t] / nrm;
        gsync();
    };
    for (int64_t t = r0 + threadIdx.x; t < r1; t += blockDim.x) {
        const double r = hash_unit(static_cast<uint64_t>(t), 0x5eedull);
        a.w[t] = a.x0 ? a.x0[t] + (a.x1 ? a.x1[t] : 0.0) + a.warm_noise * r / sqrt(static_cast<double>(n)) : r;
    }
    set_v0_from_w();

    int restarts = 0, breakdowns = 0;
    int j = 0;
    // A warm-started solve (x0 = previous eigenvector) needs about as many
    // steps as the previous one of the same operator: skip the convergence
    // checks before that (each check is a sequential T-eigen solve on CTA 0).
    // The hint is reset by every cold start, so a solve is reproducible.
    int first_check = a.min_steps;
    if (a.warm && a.hint) first_check = max(a.min_steps, (*a.hint / a.check_every - 1) * a.check_every);
    bool zero_op = false;
    double anorm = 0.0;
    double inv_beta = 1.0;  // V[:,j] = w * inv_beta for j > 0 (materialised in phase B)
    // TILED: a convergence check decided at the end of a step, run by CTA 0
    // during the next step's matvec
    bool pend_check = false, pend_full = false, pend_limit = false;
    double pend_beta = 0.0;
    for (;;) {
        if constexpr (TILED) {
            extern __shared__ double dsm[];
            // [A] J v_j partials (single read of the blocks) + CGS pass-1 dot
            // partials.  CTA 0 has no matvec share (build_tiles): it runs the
            // convergence check of the previous step meanwhile; the decision
            // is read after the barrier (an unneeded step's partials are
            // simply dropped).
            mark(7);
            if (pend_check && blockIdx.x == 0)
                t_extremes(a, j, pend_beta, pend_full, restarts, dsm, kMaxKrylov);
            mark(5);
            lz_phase_a(op, tls, a.V + static_cast<int64_t>(j) * n, a.V, n, j, a.pdot1, ld, dsm,
                       dsm + kLzWarps * 32 * kLzNQ, dsm + (kLzWarps + 1) * 32 * kLzNQ,
                       blockIdx.x == 1 ? a.lzt : nullptr);
            mark(0);
            gsync();
            mark(1);
            if (pend_check) {
                pend_check = false;
                if (a.ctl[0]) break;
                if (pend_limit) {
                    if (restarts >= a.max_restarts) break;  // best effort: ctl[0] stays 0
                    // restart from (x_lo + x_hi): both ends stay represented
                    ++restarts;
                    first_check = a.min_steps;
                    for (int64_t t = r0 + threadIdx.x; t < r1; t += blockDim.x) {
                        double s0 = 0.0, s1 = 0.0;
                        for (int k = 0; k < j; ++k) {
                            const double v = a.V[t + static_cast<int64_t>(k) * n];
                            s0 = fma(v, a.sT[k], s0);
                            s1 = fma(v, a.sT[kMaxKrylov + k], s1);
                        }
                        a.w[t] = s0 + s1;
                    }
                    gsync();
                    set_v0_from_w();
                    j = 0;
                    anorm = 0.0;
                    continue;
                }
            }
            // [B] own rows, an 8-lane group per row (group g = 4 warp + lane / 8,
            // rows r0 + g + 64 round): y = J v_j, w1 = y - V h1 (h1 from the
            // folded partials), the pass-2 dots V' w1 and ||w1||^2.  Round 0
            // keeps w1 and its V entries k = sl + 8u < 32 in registers for the
            // update after the next barrier.
            reduce_dots(a.pdot1, j);  // hsh = h1 / scale
            const double sc = op.scale;
            const int g = 4 * warp + (lane >> 3), sl = lane & 7;
            double w1r = 0.0, vr[4] = {0.0, 0.0, 0.0, 0.0}, acc2[4] = {0.0, 0.0, 0.0, 0.0}, ssq = 0.0;
            for (int64_t tb = r0; tb < r1; tb += 64) {
                const int64_t t = tb + g;
                const bool ok = t < r1;
                const double y = lz_row_sum8(op, tls, lzmeta, ok ? t : r0, sl) * sc;
                double v4[4];
                double s = 0.0;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int k = sl + 8 * u;
                    v4[u] = (ok && k <= j) ? a.V[t + static_cast<int64_t>(k) * n] : 0.0;
                    s = fma(v4[u], k <= j ? hsh[k] * sc : 0.0, s);
                }
                if (ok)
                    for (int k = sl + 32; k <= j; k += 8) s = fma(a.V[t + static_cast<int64_t>(k) * n], hsh[k] * sc, s);
#pragma unroll
                for (int off = 4; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
                const double w1 = ok ? y - s : 0.0;
                if (ok && sl == 0) a.w[t] = w1;
#pragma unroll
                for (int u = 0; u < 4; ++u) acc2[u] = fma(v4[u], w1, acc2[u]);
                if (sl == 0) ssq = fma(w1, w1, ssq);
                if (tb == r0) {
                    w1r = w1;
#pragma unroll
                    for (int u = 0; u < 4; ++u) vr[u] = v4[u];
                }
            }
            // pass-2 dot partials k < 32 in a fixed order: groups, then the CTA
            {
                double* d2 = dsm;  // [64 groups][32 k] + [64] norms (phase-A scratch, free here)
#pragma unroll
                for (int u = 0; u < 4; ++u) d2[g * 32 + sl + 8 * u] = acc2[u];
                if (sl == 0) d2[64 * 32 + g] = ssq;
                __syncthreads();
                if (threadIdx.x <= min(j, 31)) {
                    double v = 0.0;
                    for (int q = 0; q < 64; ++q) v += d2[q * 32 + threadIdx.x];
                    a.pdot2[static_cast<int64_t>(blockIdx.x) * ld + threadIdx.x] = v;
                }
                if (threadIdx.x == 32) {
                    double v = 0.0;
                    for (int q = 0; q < 64; ++q) v += d2[64 * 32 + q];
                    a.part[blockIdx.x] = v;
                }
                if (j >= 32) {  // long Krylov spaces (cold starts): k >= 32 from memory
                    for (int k = 32 + warp; k <= j; k += nw) {
                        const double* vk = a.V + static_cast<int64_t>(k) * n;
                        double t2 = 0.0;
                        for (int64_t t = r0 + lane; t < r1; t += 32) t2 = fma(vk[t], a.w[t], t2);
#pragma unroll
                        for (int off = 16; off >= 1; off >>= 1) t2 += __shfl_xor_sync(0xffffffffu, t2, off);
                        if (lane == 0) a.pdot2[static_cast<int64_t>(blockIdx.x) * ld + k] = t2;
                    }
                }
            }
            mark(2);
            gsync();
            mark(3);
            const double h1j = hsh[j] * sc;
            __syncthreads();
            reduce_dots(a.pdot2, j);  // hsh = h2
            double h2sq = 0.0;
            for (int k = 0; k <= j; ++k) h2sq = fma(hsh[k], hsh[k], h2sq);
            const double w1sq = grid_sum(a.part, 0);
            const double alpha = h1j + hsh[j];
            // ||w1 - V h2||^2 = ||w1||^2 - ||h2||^2 (V orthonormal, h2 = V' w1)
            double nrm = sqrt(fmax(w1sq - h2sq, 0.0));
            anorm = fmax(anorm, fabs(alpha) + nrm + (j > 0 ? a.beta[j - 1] : 0.0));
            if (j == 0 && restarts == 0 && anorm == 0.0) {
                zero_op = true;  // J == 0 (see below)
                break;
            }
            const bool space_full = (j + 1 == n);
            const bool breakdown = !space_full && nrm <= 1e-13 * anorm;
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                a.alpha[j] = alpha;
                a.beta[j] = breakdown ? 0.0 : nrm;
            }
            double* vnext = a.V + static_cast<int64_t>(j + 1) * n;
            if (breakdown) {
                ++breakdowns;
                for (int64_t t = r0 + threadIdx.x; t < r1; t += blockDim.x)
                    a.w[t] = hash_unit(static_cast<uint64_t>(t), 0xb00ull + breakdowns);
                __syncthreads();
                cgs2(j);
                nrm = sqrt(grid_sum(a.part, 0));
                for (int64_t t = r0 + threadIdx.x; t < r1; t += blockDim.x) vnext[t] = a.w[t] / nrm;
            } else if (!space_full) {
                // v_{j+1} = (w1 - V h2) / beta: round 0 from registers
                const double ib = 1.0 / nrm;
                for (int64_t tb = r0; tb < r1; tb += 64) {
                    const int64_t t = tb + g;
                    const bool ok = t < r1;
                    double s = 0.0, w1 = w1r;
                    if (tb == r0) {
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int k = sl + 8 * u;
                            s = fma(vr[u], k <= j ? hsh[k] : 0.0, s);
                        }
                    } else {
                        w1 = ok ? a.w[t] : 0.0;
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int k = sl + 8 * u;
                            if (ok && k <= j) s = fma(a.V[t + static_cast<int64_t>(k) * n], hsh[k], s);
                        }
                    }
                    if (ok)
                        for (int k = sl + 32; k <= j; k += 8) s = fma(a.V[t + static_cast<int64_t>(k) * n], hsh[k], s);
#pragma unroll
                    for (int off = 4; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
                    if (ok && sl == 0) vnext[t] = (w1 - s) * ib;
                }
            }
            ++j;
            const bool size_limit = (j == a.maxm) || space_full;
            pend_check = ((j >= first_check && j % a.check_every == 0) && !breakdown) || size_limit;
            pend_beta = breakdown ? 0.0 : nrm;
            pend_full = space_full;
            pend_limit = size_limit;
            mark(4);
            gsync();
            mark(6);
            continue;
        }
        // [A] matvec partials of v_j
        mark(7);
        if (j == 0)
            blockop_phase_a<false>(op, a.V);
        else
            blockop_phase_a<false>(op, a.w, inv_beta);
        mark(0);
        gsync();
        mark(1);
        // [B] materialise own rows of v_j, then w = J v_j (own rows), partial dots
        if (j > 0) {
            double* vj = a.V + static_cast<int64_t>(j) * n;
            for (int64_t t = r0 + threadIdx.x; t < r1; t += blockDim.x) vj[t] = a.w[t] * inv_beta;
            __syncthreads();
        }
        blockop_phase_b<false>(op, a.w, r0 + threadIdx.x, blockDim.x, r1);
        __syncthreads();
        mark(2);
        cgs2(j);
        mark(3);
        // alpha_j = h1[j] + h2[j]; h2 is in hsh, h1[j] is re-reduced (same order)
        double alpha = 0.0;
        {
            const double h2j = hsh[j];
            if (warp == 0) {
                double s1 = 0.0;
                for (int b = lane; b < G; b += 32) s1 += a.pdot1[static_cast<int64_t>(b) * ld + j];
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) s1 += __shfl_xor_sync(0xffffffffu, s1, off);
                if (lane == 0) red[30] = s1;
            }
            __syncthreads();
            alpha = red[30] + h2j;
            __syncthreads();
        }
        double nrm = sqrt(grid_sum(a.part, 0));
        anorm = fmax(anorm, fabs(alpha) + nrm + (j > 0 ? a.beta[j - 1] : 0.0));
        if (j == 0 && restarts == 0 && anorm == 0.0) {
            // J v0 == 0 for a dense random v0: J is the zero matrix.  The
            // reference's full decomposition then returns the identity's last
            // column for the picked (highest) end (sym_eig.cpp:206-229).
            zero_op = true;
            break;
        }
        const bool space_full = (j + 1 == n);
        const bool breakdown = !space_full && nrm <= 1e-13 * anorm;
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            a.alpha[j] = alpha;
            a.beta[j] = breakdown ? 0.0 : nrm;
        }
        if (breakdown) {
            // invariant subspace: continue with a fresh direction orthogonal to V
            ++breakdowns;
            for (int64_t t = r0 + threadIdx.x; t < r1; t += blockDim.x)
                a.w[t] = hash_unit(static_cast<uint64_t>(t), 0xb00ull + breakdowns);
            __syncthreads();
            cgs2(j);
            nrm = sqrt(grid_sum(a.part, 0));
        }
        inv_beta = 1.0 / nrm;
        ++j;
        const bool size_limit = (j == a.maxm) || space_full;
        mark(4);
        if (((j >= first_check && j % a.check_every == 0) && !breakdown) || size_limit) {
            if (blockIdx.x == 0) {
                extern __shared__ double dsm[];
                t_extremes(a, j, breakdown ? 0.0 : nrm, space_full, restarts, dsm, kMaxKrylov);
            }
            mark(5);
            gsync();
            mark(6);
            if (a.ctl[0]) break;
            if (size_limit) {
                if (restarts >= a.max_restarts) break;  // best effort: ctl[0] stays 0
                // restart from (x_lo + x_hi): both ends stay represented
                ++restarts;
                first_check = a.min_steps;
                for (int64_t t = r0 + threadIdx.x; t < r1; t += blockDim.x) {
                    double s0 = 0.0, s1 = 0.0;
                    for (int k = 0; k < j; ++k) {
                        const double v = a.V[t + static_cast<int64_t>(k) * n];
                        s0 = fma(v, a.sT[k], s0);
                        s1 = fma(v, a.sT[kMaxKrylov + k], s1);
                    }
                    a.w[t] = s0 + s1;
                }
                gsync();
                set_v0_from_w();
                j = 0;
                anorm = 0.0;
            }
        }
    }

    if (zero_op) {
        for (int64_t i = gtid; i < n; i += gstride) a.out_vec[i] = i == n - 1 ? 1.0 : 0.0;
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            *a.out_value = 0.0;
            a.ctl[0] = 1;
            a.ctl[1] = 1;
            a.ctl[2] = 1;
            a.ctl[3] = 0;
            a.ctl[4] = 0;
        }
        return;
    }
    // ---- Ritz vector of the picked end
    const int m = j;
    const int pick = a.ctl[1];
    const double* s = a.sT + (pick ? kMaxKrylov : 0);
    const double* so = a.sT + (pick ? 0 : kMaxKrylov);
    double best = -1.0;
    int64_t besti = 0;
    double ss = 0.0, sso = 0.0;
    for (int64_t i = gtid; i < n; i += gstride) {
        double x = 0.0, xo = 0.0;
        for (int k = 0; k < m; ++k) {
            const double v = a.V[i + static_cast<int64_t>(k) * n];
            x = fma(v, s[k], x);
            xo = fma(v, so[k], xo);
        }
        a.out_vec[i] = x;
        if (a.other_out) a.other_out[i] = xo;
        ss = fma(x, x, ss);
        sso = fma(xo, xo, sso);
        if (fabs(x) > best) {
            best = fabs(x);
            besti = i;
        }
    }
    // argmax |x| with the lowest index on ties (sym_eig.cpp:223-227), and ||x||
    __shared__ double bv[32];
    __shared__ int64_t bi[32];
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, off);
        const int64_t oi = __shfl_xor_sync(0xffffffffu, besti, off);
        if (ov > best || (ov == best && oi < besti)) {
            best = ov;
            besti = oi;
        }
    }
    // (warp, lane as above)
    if (lane == 0) {
        bv[warp] = best;
        bi[warp] = besti;
    }
    ss = cta_sum(ss, red);
    sso = cta_sum(sso, red);
    if (threadIdx.x == 0) {
        a.part[3 * G + blockIdx.x] = sso;
        double b0 = bv[0];
        int64_t i0 = bi[0];
        for (int k = 1; k < static_cast<int>(blockDim.x >> 5); ++k)
            if (bv[k] > b0 || (bv[k] == b0 && bi[k] < i0)) {
                b0 = bv[k];
                i0 = bi[k];
            }
        a.part[G + blockIdx.x] = b0;
        a.part[2 * G + blockIdx.x] = static_cast<double>(i0);
        a.part[blockIdx.x] = ss;
    }
    gsync();
    double b0 = -1.0;
    int64_t i0 = 0;
    for (int b = 0; b < G; ++b) {
        const double v = a.part[G + b];
        const int64_t ii = static_cast<int64_t>(a.part[2 * G + b]);
        if (v > b0 || (v == b0 && ii < i0)) {
            b0 = v;
            i0 = ii;
        }
    }
    const double nrm = sqrt(grid_total(a.part, 0));
    const double sgn = a.out_vec[i0] < 0.0 ? -1.0 : 1.0;
    gsync();
    double nrm_o = 0.0;
    for (int b = 0; b < G; ++b) nrm_o += a.part[3 * G + b];
    nrm_o = sqrt(nrm_o);
    for (int64_t i = gtid; i < n; i += gstride) {
        a.out_vec[i] = sgn * a.out_vec[i] / nrm;
        if (a.other_out && nrm_o > 0.0) a.other_out[i] /= nrm_o;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        for (int k = 0; k < 8; ++k) a.stats[8 + k] = static_cast<double>(tacc[k]);
        *a.out_value = a.stats[4];
        if (a.hint) *a.hint = restarts == 0 ? m : 0;
        a.ctl[2] = m;
        a.ctl[3] = restarts;
        a.ctl[4] = breakdowns;
    }
}

// ---------------------------------------------------------------------------
// Small operators (n <= kSmallN): the whole Lanczos run on ONE thread-block
// cluster (<= 16 CTAs).  CTA c owns rows [c R, (c+1) R) of every length-n
// vector; its rows of J (dense, built once per call from the blocks; shared
// memory when they fit, else an L2-resident scratch), of the Krylov basis and
// of w stay with it.  Three cluster barriers per step: after the partial dots
// of each CGS2 pass and after publishing the next (unnormalised) vector with
// the ||w||^2 partials; partials travel as DSMEM stores and every sum runs
// over the G partials in CTA order (deterministic).  Same start vector,
// convergence test (t_extremes), breakdown / restart handling and pick / sign
// rules as lanczos_kernel; the lanczos_kernel's grid syncs and L2 round
// trips cost ~20 us per step at n = 300..800, this ~4 us.
constexpr int kSmallN = 1024;
constexpr int kSmallMaxM = 192;

__global__ void __launch_bounds__(kEigThreads, 1)
    lanczos_cluster_kernel(const EigArgs a, double* __restrict__ Sg, int s_in_smem) {
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) double dsm[];
    const BlockOp& op = *a.op;
    const int n = static_cast<int>(a.n);
    const int G = gridDim.x, me = blockIdx.x, tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5, nw = kEigThreads / 32;
    const int R = (n + G - 1) / G;
    const int r0 = min(n, me * R), r1 = min(n, r0 + R), Rm = r1 - r0;
    const int ld = a.maxm + 1;
    double* text = dsm;             // t_extremes scratch, 14 * ld
    double* Vs = text + 14 * ld;    // own rows of V: Vs[k * R + r]
    double* hp1 = Vs + ld * R;      // pushed pass-1 partials [16][ld]
    double* hp2 = hp1 + 16 * ld;    // pushed pass-2 partials [16][ld]
    double* wfull = hp2 + 16 * ld;  // pushed next vector (unnormalised), n
    double* ws = wfull + n;         // own rows of w, R
    double* Sown = s_in_smem ? ws + R : Sg + static_cast<size_t>(me) * R * n;  // own rows of J, [R][n]
    __shared__ double hsh[kSmallMaxM + 1];
    __shared__ double red[32];
    __shared__ double nrmp[16];
    __shared__ double fin[5][16];
    // message barriers (dsmem.cuh): 0 CGS pass 1, 1 CGS pass 2, 2 publish;
    // their phases advance identically in every CTA (uniform control flow)
    __shared__ __align__(8) uint64_t mbar[3];
    uint32_t ph1 = 0, ph2 = 0, php = 0;
    if (tid == 0) {
        for (int b = 0; b < 3; ++b) mbar_init1(&mbar[b]);
        mbar_init_fence();
    }
    __syncthreads();
    cl.sync();  // barriers initialised, every CTA running, before any DSMEM store
    // diagnostics (R1_DEBUG_EIG): per-phase ns of CTA 0 thread 0 -> stats[8..15]
    unsigned long long tacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    unsigned long long tlast = gtimer();
    auto mark = [&](int ph) {
        const unsigned long long t = gtimer();
        tacc[ph] += t - tlast;
        tlast = t;
    };

    // ---- own rows of J (row t = column t: symmetric)
    for (int e = tid; e < Rm * n; e += kEigThreads) {
        const int r = e / n, u = e - r * n, t = r0 + r;
        double v;
        if (op.dense) {
            v = op.dense[t + static_cast<size_t>(u) * n];
        } else {
            int m = 0, q = 0;
            while (t >= op.offs[m + 1]) ++m;
            while (u >= op.offs[q + 1]) ++q;
            const int64_t i = t - op.offs[m], jj = u - op.offs[q];
            v = 0.0;
            if (q > m) v = op.blocks[op.boff[pair_index(m, q, op.d)] + i + jj * op.dims[m]];
            else if (q < m) v = op.blocks[op.boff[pair_index(q, m, op.d)] + jj + i * op.dims[q]];
        }
        Sown[static_cast<size_t>(r) * n + u] = v;
    }
    // publish own rows of w and the CTA's ||w||^2 partial to every CTA (st.async
    // messages); once all (G + n) values have arrived every CTA returns
    // sqrt(sum of the partials in CTA order).  Buffers are reused safely: a CTA
    // sends a phase's data only after receiving the previous phase from all.
    auto publish = [&]() {
        double ss = 0.0;
        for (int r = tid; r < Rm; r += kEigThreads) ss = fma(ws[r], ws[r], ss);
        ss = cta_sum(ss, red);
        if (tid < G) send8(&nrmp[me], ss, &mbar[2], tid);
        for (int e = tid; e < G * Rm; e += kEigThreads) {
            const int c = e / Rm, r = e - c * Rm;
            send8(&wfull[r0 + r], ws[r], &mbar[2], c);
        }
        if (tid == 0) expect_bytes(&mbar[2], static_cast<uint32_t>((G + n) * 8));
        wait_parity(&mbar[2], php & 1);
        ++php;
        double t = 0.0;
        for (int c = 0; c < G; ++c) t += nrmp[c];
        return sqrt(t);
    };
    // one classical Gram-Schmidt pass of w (own rows) against V[:, 0..j]
    auto cgs_pass = [&](double* hp, int j, uint64_t* bar, uint32_t& ph) {
        for (int k = warp; k <= j; k += nw) {
            const double* vk = Vs + k * R;
            double s = 0.0;
            for (int r = lane; r < Rm; r += 32) s = fma(vk[r], ws[r], s);
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
            if (lane < G) send8(&hp[me * ld + k], s, bar, lane);
        }
        if (tid == 0) expect_bytes(bar, static_cast<uint32_t>(G * (j + 1) * 8));
        wait_parity(bar, ph & 1);
        ++ph;
        for (int k = tid; k <= j; k += kEigThreads) {
            double h = 0.0;
            for (int c = 0; c < G; ++c) h += hp[c * ld + k];
            hsh[k] = h;
        }
        __syncthreads();
        for (int r = tid; r < Rm; r += kEigThreads) {
            double s = 0.0;
            for (int k = 0; k <= j; ++k) s = fma(Vs[k * R + r], hsh[k], s);
            ws[r] -= s;
        }
        __syncthreads();
    };

    for (int r = tid; r < Rm; r += kEigThreads) {
        const int t = r0 + r;
        const double rr = hash_unit(static_cast<uint64_t>(t), 0x5eedull);
        ws[r] = a.x0 ? a.x0[t] + (a.x1 ? a.x1[t] : 0.0) + a.warm_noise * rr / sqrt(static_cast<double>(n)) : rr;
    }
    __syncthreads();
    double inv_beta = 1.0 / publish();
    mark(0);

    int restarts = 0, breakdowns = 0;
    int j = 0;
    int first_check = a.min_steps;
    if (a.warm && a.hint) first_check = max(a.min_steps, (*a.hint / a.check_every - 1) * a.check_every);
    bool zero_op = false;
    double anorm = 0.0;
    for (;;) {
        // v_j = w * inv_beta (own rows into V, all rows from wfull), w = J v_j
        for (int r = tid; r < Rm; r += kEigThreads) Vs[j * R + r] = ws[r] * inv_beta;
        for (int r = warp; r < Rm; r += nw) {
            // 8 independent loads per lane in flight: at n > ~600 the rows
            // live in L2 (they do not fit next to V in shared memory) and a
            // 2-deep loop was latency-bound (~5 us per step at n = 800)
            const double* sr = Sown + static_cast<size_t>(r) * n;
            double s4[4] = {0.0, 0.0, 0.0, 0.0};
            int u = lane;
            for (; u + 7 * 32 < n; u += 8 * 32) {
                double x[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) x[k] = sr[u + 32 * k];
#pragma unroll
                for (int k = 0; k < 8; ++k) s4[k & 3] = fma(x[k], wfull[u + 32 * k], s4[k & 3]);
            }
#pragma unroll
            for (int k = 0; k < 7; ++k)
                if (u + 32 * k < n) s4[k & 3] = fma(sr[u + 32 * k], wfull[u + 32 * k], s4[k & 3]);
            double s = (s4[0] + s4[1]) + (s4[2] + s4[3]);
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
            if (lane == 0) ws[r] = s * inv_beta * op.scale;
        }
        __syncthreads();
        mark(1);
        cgs_pass(hp1, j, &mbar[0], ph1);
        const double h1j = hsh[j];
        mark(2);
        cgs_pass(hp2, j, &mbar[1], ph2);
        const double alpha = h1j + hsh[j];
        mark(3);
        double nrm = publish();
        mark(4);
        anorm = fmax(anorm, fabs(alpha) + nrm + (j > 0 ? a.beta[j - 1] : 0.0));
        if (j == 0 && restarts == 0 && anorm == 0.0) {
            zero_op = true;  // J v0 == 0 for a dense random v0: J == 0 (see lanczos_kernel)
            break;
        }
        const bool space_full = (j + 1 == n);
        const bool breakdown = !space_full && nrm <= 1e-13 * anorm;
        if (me == 0 && tid == 0) {
            a.alpha[j] = alpha;
            a.beta[j] = breakdown ? 0.0 : nrm;
        }
        if (breakdown) {
            ++breakdowns;
            for (int r = tid; r < Rm; r += kEigThreads)
                ws[r] = hash_unit(static_cast<uint64_t>(r0 + r), 0xb00ull + breakdowns);
            __syncthreads();
            cgs_pass(hp1, j, &mbar[0], ph1);
            cgs_pass(hp2, j, &mbar[1], ph2);
            nrm = publish();
        }
        inv_beta = 1.0 / nrm;
        ++j;
        const bool size_limit = (j == a.maxm) || space_full;
        if (((j >= first_check && j % a.check_every == 0) && !breakdown) || size_limit) {
            if (me == 0) t_extremes(a, j, breakdown ? 0.0 : nrm, space_full, restarts, text, ld);
            cl.sync();
            mark(5);
            if (*reinterpret_cast<volatile int*>(a.ctl)) break;
            if (size_limit) {
                if (restarts >= a.max_restarts) break;  // best effort: ctl[0] stays 0
                ++restarts;
                first_check = a.min_steps;
                for (int r = tid; r < Rm; r += kEigThreads) {
                    double s0 = 0.0, s1 = 0.0;
                    for (int k = 0; k < j; ++k) {
                        const double v = Vs[k * R + r];
                        s0 = fma(v, a.sT[k], s0);
                        s1 = fma(v, a.sT[kMaxKrylov + k], s1);
                    }
                    ws[r] = s0 + s1;
                }
                __syncthreads();
                inv_beta = 1.0 / publish();
                j = 0;
                anorm = 0.0;
            }
        }
    }

    if (zero_op) {
        for (int r = tid; r < Rm; r += kEigThreads) a.out_vec[r0 + r] = r0 + r == n - 1 ? 1.0 : 0.0;
        if (me == 0 && tid == 0) {
            *a.out_value = 0.0;
            a.ctl[0] = 1;
            a.ctl[1] = 1;
            a.ctl[2] = 1;
            a.ctl[3] = 0;
            a.ctl[4] = 0;
        }
        cl.sync();
        return;
    }
    // ---- Ritz vectors of both ends (own rows); sign rule needs the global
    // arg-max |x| (lowest index on ties) and both norms
    const int m = j;
    const int pick = *reinterpret_cast<volatile int*>(a.ctl + 1);
    const double* s = a.sT + (pick ? kMaxKrylov : 0);
    const double* so = a.sT + (pick ? 0 : kMaxKrylov);
    double* xo_s = hp1;  // reuse: own rows of the other-end vector
    double best = -1.0, bsg = 0.0, ss = 0.0, sso = 0.0;
    int besti = n;
    for (int r = tid; r < Rm; r += kEigThreads) {
        double x = 0.0, xo = 0.0;
        for (int k = 0; k < m; ++k) {
            const double v = Vs[k * R + r];
            x = fma(v, s[k], x);
            xo = fma(v, so[k], xo);
        }
        ws[r] = x;
        xo_s[r] = xo;
        ss = fma(x, x, ss);
        sso = fma(xo, xo, sso);
        if (fabs(x) > best) {
            best = fabs(x);
            besti = r0 + r;
            bsg = x;
        }
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, off);
        const int oi = __shfl_xor_sync(0xffffffffu, besti, off);
        const double os = __shfl_xor_sync(0xffffffffu, bsg, off);
        if (ov > best || (ov == best && oi < besti)) {
            best = ov;
            besti = oi;
            bsg = os;
        }
    }
    __shared__ double bv[32], bs[32];
    __shared__ int bi[32];
    if (lane == 0) {
        bv[warp] = best;
        bi[warp] = besti;
        bs[warp] = bsg;
    }
    ss = cta_sum(ss, red);
    sso = cta_sum(sso, red);
    if (tid < G) {
        double b0 = bv[0], s0 = bs[0];
        int i0 = bi[0];
        for (int k = 1; k < nw; ++k)
            if (bv[k] > b0 || (bv[k] == b0 && bi[k] < i0)) {
                b0 = bv[k];
                i0 = bi[k];
                s0 = bs[k];
            }
        *cl.map_shared_rank(&fin[0][me], tid) = b0;
        *cl.map_shared_rank(&fin[1][me], tid) = static_cast<double>(i0);
        *cl.map_shared_rank(&fin[2][me], tid) = s0;
        *cl.map_shared_rank(&fin[3][me], tid) = ss;
        *cl.map_shared_rank(&fin[4][me], tid) = sso;
    }
    cl.sync();
    double b0 = -1.0, s0 = 0.0, nrm2 = 0.0, nrm2o = 0.0;
    int i0 = n;
    for (int c = 0; c < G; ++c) {
        const int ii = static_cast<int>(fin[1][c]);
        if (fin[0][c] > b0 || (fin[0][c] == b0 && ii < i0)) {
            b0 = fin[0][c];
            i0 = ii;
            s0 = fin[2][c];
        }
        nrm2 += fin[3][c];
        nrm2o += fin[4][c];
    }
    const double nrm = sqrt(nrm2), nrm_o = sqrt(nrm2o);
    const double sgn = s0 < 0.0 ? -1.0 : 1.0;
    for (int r = tid; r < Rm; r += kEigThreads) {
        a.out_vec[r0 + r] = sgn * ws[r] / nrm;
        if (a.other_out && nrm_o > 0.0) a.other_out[r0 + r] = xo_s[r] / nrm_o;
    }
    if (me == 0 && tid == 0) {
        mark(6);
        for (int k = 0; k < 8; ++k) a.stats[8 + k] = static_cast<double>(tacc[k]);
        *a.out_value = a.stats[4];
        if (a.hint) *a.hint = restarts == 0 ? m : 0;
        a.ctl[2] = m;
        a.ctl[3] = restarts;
        a.ctl[4] = breakdowns;
    }
    cl.sync();  // no CTA exits while others may still write its shared memory
}

struct EigPlan {
    BlockOp op;
    DescCache<BlockOp> dop;
    DeviceBuffer hint;   // one int: steps of the last solve in the solver's chain
    DeviceBuffer dense_ws;  // dense J + scratch of the reference-algorithm eigen step
    DeviceBuffer other;  // n: other-end Ritz vector of the last solve in the chain
    bool other_valid = false;
    int64_t coldot_n = 0, rowpart_n = 0;
    // tiled matvec plan of the grid kernel (built for tl_G CTAs)
    LzTiles tl;
    DeviceBuffer tl_meta;
    DescCache<LzTiles> dtl;
    int tl_G = 0;
    int64_t tl_coldot_n = 0, tl_rowpart_n = 0;
};

// Split the (pair, row chunk, column) units of the blocks into G contiguous
// ranges of equal cost (rows of the chunk + a per-column overhead) and cut
// them into segments (one row chunk each).
void build_tiles(r1_context* ctx, EigPlan& P, int G) {
    const BlockOp& op = P.op;
    LzTiles& tl = P.tl;
    tl = LzTiles{};
    std::vector<LzSeg> segs;
    std::vector<int> cta_seg(G + 1, 0), rc_first;
    double total = 0.0;
    int64_t cdo = 0;
    const int group = 1;
    for (int p = 0; p < op.npairs; ++p) {
        const int64_t rows = op.dims[op.pm[p]], cols = op.dims[op.pn[p]];
        int nrc = static_cast<int>((rows + 32 * kLzNQ - 1) / (32 * kLzNQ));
        int rc_rows = static_cast<int>((rows + nrc - 1) / nrc);
        tl.nrc[p] = nrc;
        tl.Rc[p] = rc_rows;
        // double2 loads: even rows and an even block offset keep every column
        // and every (even) row chunk 16-B aligned
        tl.v2[p] = (rows % 2 == 0 && op.boff[p] % 2 == 0) ? 1 : 0;
        if (tl.v2[p] && tl.Rc[p] % 2) ++tl.Rc[p];
        tl.cd_off[p] = cdo;
        cdo += static_cast<int64_t>(nrc) * cols;
        for (int rc = 0; rc < nrc; ++rc) {
            const int64_t nr = std::min<int64_t>(tl.Rc[p], rows - static_cast<int64_t>(rc) * tl.Rc[p]);
            total += static_cast<double>(cols) * static_cast<double>(nr + 16);
        }
    }
    // CTA 0 runs the convergence checks while the others do the matvec
    const int first = G > 1 ? 1 : 0;
    const double per = total / (G - first);
    double x = 0.0;
    int cur = first;
    long long rp = 0;
    for (int p = 0; p < op.npairs; ++p) {
        const int64_t rows = op.dims[op.pm[p]], cols = op.dims[op.pn[p]];
        tl.rcseg_off[p] = static_cast<int>(rc_first.size());
        for (int rc = 0; rc < tl.nrc[p]; ++rc) {
            const int64_t nr = std::min<int64_t>(tl.Rc[p], rows - static_cast<int64_t>(rc) * tl.Rc[p]);
            const double c = static_cast<double>(nr + 16);
            rc_first.push_back(static_cast<int>(segs.size()));
            bool open = false;
            for (int64_t col = 0; col < cols; col += group) {
                const int64_t ce = std::min<int64_t>(cols, col + group);
                const double cg = c * static_cast<double>(ce - col);
                const int target = first + std::min(G - 1 - first, static_cast<int>((x + 0.5 * cg) / per));
                if (!open || target != cur) {
                    while (cur < target) cta_seg[++cur] = static_cast<int>(segs.size());
                    segs.push_back(LzSeg{p, rc, static_cast<int>(col), static_cast<int>(ce), rp});
                    rp += nr;
                    open = true;
                } else {
                    segs.back().c1 = static_cast<int>(ce);
                }
                x += cg;
            }
        }
    }
    while (cur < G) cta_seg[++cur] = static_cast<int>(segs.size());
    rc_first.push_back(static_cast<int>(segs.size()));
    if (rp >= (1ll << 31)) fail(R1_ERR_INVALID_ARGUMENT, "eig: operator too large for the tiled matvec");
    tl.nrcf = static_cast<int>(rc_first.size()) - 1;
    tl.nseg = static_cast<int>(segs.size());
    for (const LzSeg& sg : segs) rc_first.push_back(static_cast<int>(sg.rp));  // meta = rc_first ++ seg_rp
    const size_t seg_bytes = segs.size() * sizeof(LzSeg);
    const size_t cta_bytes = cta_seg.size() * sizeof(int);
    const size_t rcf_bytes = rc_first.size() * sizeof(int);
    const size_t off_cta = (seg_bytes + 15) & ~size_t(15);
    const size_t off_rcf = off_cta + ((cta_bytes + 15) & ~size_t(15));
    P.tl_meta.ensure(off_rcf + rcf_bytes + 16);
    char* base = P.tl_meta.as<char>();
    upload_now(ctx, base, segs.data(), seg_bytes);
    upload_now(ctx, base + off_cta, cta_seg.data(), cta_bytes);
    upload_now(ctx, base + off_rcf, rc_first.data(), rcf_bytes);
    tl.segs = reinterpret_cast<const LzSeg*>(base);
    tl.cta_seg = reinterpret_cast<const int*>(base + off_cta);
    tl.meta = reinterpret_cast<const int*>(base + off_rcf);
    P.tl_coldot_n = cdo;
    P.tl_rowpart_n = rp;
    P.tl_G = G;
}

}  // namespace

namespace {

void finish_lanczos(r1_context* ctx, const EigArgs& a, int* info_host, double* stats_host) {
    const int64_t n = a.n;
    static const bool dbg = dev_env("R1_DEBUG_EIG") != nullptr;
    if (dbg) {
        int ctl[5];
        double st[16];
        R1_CUDA(cudaMemcpyAsync(ctl, a.ctl, sizeof(ctl), cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaMemcpyAsync(st, a.stats, sizeof(st), cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
        static const bool dbg_t = dev_env("R1_DEBUG_EIG_T") != nullptr;
        if (dbg_t) {
            std::vector<double> al(ctl[2]), be(ctl[2]);
            R1_CUDA(cudaMemcpy(al.data(), a.alpha, al.size() * sizeof(double), cudaMemcpyDeviceToHost));
            R1_CUDA(cudaMemcpy(be.data(), a.beta, be.size() * sizeof(double), cudaMemcpyDeviceToHost));
            for (int k = 0; k < std::min(ctl[2], 24); ++k)
                std::fprintf(stderr, "  T[%d] alpha=%.6e beta=%.6e\n", k, al[k], be[k]);
        }
        std::fprintf(stderr,
                     "[r1 eig] n=%lld conv=%d pick=%d steps=%d restarts=%d breakdowns=%d "
                     "lo=%.17g hi=%.17g res_lo=%.3g res_hi=%.3g | us: A=%.1f syncA=%.1f B=%.1f "
                     "cgs2=%.1f tail=%.1f text=%.1f synct=%.1f other=%.1f\n",
                     static_cast<long long>(n), ctl[0], ctl[1], ctl[2], ctl[3], ctl[4], st[0], st[1],
                     st[2], st[3], st[8] * 1e-3, st[9] * 1e-3, st[10] * 1e-3, st[11] * 1e-3,
                     st[12] * 1e-3, st[13] * 1e-3, st[14] * 1e-3, st[15] * 1e-3);
        unsigned long long lz[3] = {0, 0, 0};
        if (a.lzt) R1_CUDA(cudaMemcpy(lz, a.lzt, sizeof(lz), cudaMemcpyDeviceToHost));
        std::fprintf(stderr, "[r1 eig] CTA 1 phase A: columns %.1f us, row partials %.1f us, pass-1 dots %.1f us\n",
                     lz[0] * 1e-3, lz[1] * 1e-3, lz[2] * 1e-3);
    }
    if (info_host || stats_host) {
        int ctl[5];
        double st[5];
        R1_CUDA(cudaMemcpyAsync(ctl, a.ctl, sizeof(ctl), cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaMemcpyAsync(st, a.stats, sizeof(st), cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
        if (info_host)
            for (int k = 0; k < 5; ++k) info_host[k] = ctl[k];
        if (stats_host)
            for (int k = 0; k < 5; ++k) stats_host[k] = st[k];
    }
}

void run_lanczos(r1_context* ctx, EigPlan& P, const double* x0, double* value_dev,
                 double* vec_dev, int* info_host, double* stats_host, bool solver_chain = false,
                 double decide_tol = 1e-6) {
    const int64_t n = P.op.n;
    const int maxm = static_cast<int>(std::min<int64_t>(n, 320));
    static const char* gs = dev_env("R1_EIG_GRID");
    static const char* gc = dev_env("R1_EIG_CLUSTER");
    static const char* gsm = dev_env("R1_EIG_SMALL");
    static const char* tz = dev_env("R1_EIG_TILED");  // development: 0 = the round-1 grid kernel
    const int grid_ctas = gs ? std::max(1, std::min(ctx->num_sms, std::atoi(gs))) : ctx->num_sms;
    const int cl_size = gc ? std::max(0, std::min(16, std::atoi(gc))) : 0;
    // small operators take the single-cluster kernel below (unless overridden)
    const bool small_pref = n <= kSmallN && !gs && !gc && !(gsm && std::atoi(gsm) == 0);
    const bool tiled = !P.op.dense && !small_pref && !(cl_size > 1 && !gs) && !(tz && std::atoi(tz) == 0);
    if (tiled && P.tl_G != grid_ctas) build_tiles(ctx, P, grid_ctas);
    const int64_t tl_n = tiled ? P.tl_coldot_n + P.tl_rowpart_n + 16 : 0;
    const int64_t need = n * (maxm + 1) + n + 2 * (maxm + 1) + 2 * maxm + 8 * ctx->num_sms +
                         2 * static_cast<int64_t>(ctx->num_sms) * (kMaxKrylov + 8) +
                         2 * kMaxKrylov + P.coldot_n + P.rowpart_n + 256 + tl_n +
                         (n <= kSmallN ? (n + 16) * n : 0);
    ctx->ws_eig.ensure(need * sizeof(double));
    double* base = ctx->ws_eig.as<double>();
    int64_t off = 0;
    auto take = [&](int64_t k) {
        double* p = base + off;
        off += (k + 7) & ~int64_t(7);
        return p;
    };
    EigArgs a{};
    a.n = n;
    a.maxm = maxm;
    static const char* ce = dev_env("R1_EIG_CHECK");
    static const char* ms = dev_env("R1_EIG_MIN_STEPS");
    // the tiled grid kernel hides a check behind the next step's matvec:
    // check every 2 steps from step 4 (warm C5 solves: 8 -> 6 steps)
    a.check_every = n <= 64 ? 1 : (ce ? std::max(1, std::atoi(ce)) : (tiled ? 2 : 8));
    // the warm start (previous eigenvector) converges the picked end within a
    // few steps; the first check comes after 8 (C2 solve 0.87 -> 0.33 ms)
    a.min_steps = static_cast<int>(std::min<int64_t>(n, ms ? std::max(1, std::atoi(ms)) : (tiled ? 4 : 8)));
    a.max_restarts = 6;
    a.tol = 1e-13;
    a.x0 = x0;
    a.V = take(n * (maxm + 1));
    a.w = take(n);
    a.h = take(maxm + 1);
    a.h2 = take(maxm + 1);
    a.alpha = take(maxm);
    a.beta = take(maxm);
    a.part = take(4 * ctx->num_sms + 8);
    a.pdot1 = take(static_cast<int64_t>(ctx->num_sms) * (kMaxKrylov + 1));
    a.pdot2 = take(static_cast<int64_t>(ctx->num_sms) * (kMaxKrylov + 1));
    a.sT = take(2 * kMaxKrylov);
    a.stats = take(16);
    static const bool dbg_eig = dev_env("R1_DEBUG_EIG") != nullptr;
    a.lzt = reinterpret_cast<unsigned long long*>(take(4));
    if (dbg_eig)
        R1_CUDA(cudaMemsetAsync(a.lzt, 0, 4 * sizeof(unsigned long long), ctx->stream));
    else
        a.lzt = nullptr;
    a.ctl = reinterpret_cast<int*>(take(4));
    BlockOp op = P.op;
    op.coldot = take(std::max<int64_t>(P.coldot_n, 1));
    op.rowpart = take(std::max<int64_t>(P.rowpart_n, 1));
    a.op = P.dop.get(op, ctx->stream);
    if (tiled) {
        LzTiles tl = P.tl;
        tl.coldot = take(std::max<int64_t>(P.tl_coldot_n, 1));
        tl.rowpart = take(std::max<int64_t>(P.tl_rowpart_n, 1));
        a.tl = P.dtl.get(tl, ctx->stream);
    }
    a.out_value = value_dev;
    a.out_vec = vec_dev;
    static const bool dbg_text = dev_env("R1_DEBUG_EIG_TEXT") != nullptr;
    a.debug_text = dbg_text ? 1 : 0;
    static const char* wn = dev_env("R1_EIG_WARM_NOISE");  // development
    // 1e-6 (was 1e-3): the previous Ritz vectors are good to ~1e-5 or better,
    // a 1e-3 random component only had to be filtered out again (C1 eigen -6%)
    a.warm_noise = wn ? std::atof(wn) : 1e-6;
    static const char* dt = dev_env("R1_EIG_DECIDE_TOL");  // development
    a.decide_tol = dt ? std::atof(dt) : decide_tol;
    if (solver_chain) {
        if (!P.hint.ptr) {
            P.hint.ensure(sizeof(int));
            R1_CUDA(cudaMemsetAsync(P.hint.ptr, 0, sizeof(int), ctx->stream));
        }
        a.hint = P.hint.as<int>();
        static const char* he = dev_env("R1_EIG_HINT");  // development: 0 disables the hint
        a.warm = x0 != nullptr && !(he && std::atoi(he) == 0) ? 1 : 0;
        P.other.ensure(static_cast<size_t>(n) * sizeof(double));
        a.x1 = x0 != nullptr && P.other_valid ? P.other.as<double>() : nullptr;
        a.other_out = P.other.as<double>();
        P.other_valid = true;
    }

    R1_CUDA(cudaMemsetAsync(a.ctl, 0, 4 * sizeof(int), ctx->stream));
    if (small_pref) {
        // one thread-block cluster, rows of J / V / w on chip
        const int G = static_cast<int>(std::min<int64_t>(16, std::max<int64_t>(1, (n + 15) / 16)));
        const int64_t R = (n + G - 1) / G;
        const int mm = static_cast<int>(std::min<int64_t>(n, kSmallMaxM));
        const int64_t ld = mm + 1;
        const int64_t base_d = 14 * ld + ld * R + 32 * ld + n + R;
        const int64_t with_s = base_d + R * n;
        constexpr int64_t cap = 215 * 1024 / 8;
        // capability probe once per device: can a 16-CTA cluster with the full
        // shared-memory budget be resident?
        static std::map<int, int> small_states;
        int small_state = 0;
        configure_once(reinterpret_cast<const void*>(lanczos_cluster_kernel), ctx->device, [&] {
            int st = 0;
            if (cudaFuncSetAttribute(lanczos_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                    cudaSuccess &&
                cudaFuncSetAttribute(lanczos_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(cap * 8)) == cudaSuccess) {
                cudaLaunchConfig_t q{};
                q.gridDim = dim3(16);
                q.blockDim = dim3(kEigThreads);
                q.dynamicSmemBytes = static_cast<size_t>(cap * 8);
                cudaLaunchAttribute qa[1];
                qa[0].id = cudaLaunchAttributeClusterDimension;
                qa[0].val.clusterDim.x = 16;
                qa[0].val.clusterDim.y = 1;
                qa[0].val.clusterDim.z = 1;
                q.attrs = qa;
                q.numAttrs = 1;
                int clusters = 0;
                if (cudaOccupancyMaxActiveClusters(&clusters, lanczos_cluster_kernel, &q) == cudaSuccess &&
                    clusters >= 1)
                    st = 1;
            }
            cudaGetLastError();
            small_states[ctx->device] = st;
        });
        {
            std::lock_guard<std::mutex> g(cache_mutex());
            small_state = small_states[ctx->device];
        }
        if (small_state == 1 && base_d <= cap) {
            const int s_in = with_s <= cap ? 1 : 0;
            double* Sg = s_in ? nullptr : take(static_cast<int64_t>(G) * R * n);
            a.maxm = mm;
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(G);
            cfg.blockDim = dim3(kEigThreads);
            cfg.dynamicSmemBytes = static_cast<size_t>(s_in ? with_s : base_d) * sizeof(double);
            cfg.stream = ctx->stream;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = G;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            R1_CUDA(cudaLaunchKernelEx(&cfg, lanczos_cluster_kernel, a, Sg, s_in));
            check_launch(ctx, "lanczos_cluster_kernel");
            finish_lanczos(ctx, a, info_host, stats_host);
            return;
        }
    }
    auto kern = tiled ? lanczos_kernel<true> : lanczos_kernel<false>;
    const size_t dyn_smem = tiled ? kLzDynSmem : kEigDynSmem;
    configure_once(reinterpret_cast<const void*>(kern), ctx->device, [&] {
        R1_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(dyn_smem)));
        R1_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    });
    int per_sm = 0;
    R1_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kEigThreads, dyn_smem));
    if (per_sm < 1) fail(R1_ERR_CUDA, "lanczos kernel cannot be resident");
    void* args[] = {&a};
    // (small operators took the cluster kernel above; R1_EIG_CLUSTER / R1_EIG_GRID
    // are development overrides for this grid kernel)
    if (cl_size > 1 && !gs) {
        // the whole Lanczos run on ONE thread-block cluster: cluster barriers
        // instead of cooperative grid syncs
        a.cluster = 1;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(cl_size);
        cfg.blockDim = dim3(kEigThreads);
        cfg.dynamicSmemBytes = kEigDynSmem;
        cfg.stream = ctx->stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = cl_size;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        R1_CUDA(cudaLaunchKernelEx(&cfg, lanczos_kernel<false>, a));
    } else {
        R1_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), dim3(grid_ctas),
                                            dim3(kEigThreads), args, dyn_smem, ctx->stream));
    }
    check_launch(ctx, "lanczos_kernel");
    finish_lanczos(ctx, a, info_host, stats_host);
}

using PlanKey = std::pair<r1_context*, std::vector<uint64_t>>;
std::map<PlanKey, std::shared_ptr<EigPlan>>& eig_plans() {
    static std::map<PlanKey, std::shared_ptr<EigPlan>> m;
    return m;
}

}  // namespace

void dense_from_blocks(r1_context* ctx, const uint64_t* dims, int order, const double* blocks,
                       double* S);
void eig_dense_reference_device(r1_context* ctx, int64_t n, double* S, double* ws, double* value_dev,
                                double* vec_dev);

void forget_eig_plans(r1_context* ctx) {
    std::lock_guard<std::mutex> cache_lock(cache_mutex());
    auto& m = eig_plans();
    for (auto it = m.begin(); it != m.end();)
        if (it->first.first == ctx)
            it = m.erase(it);
        else
            ++it;
}

// Eigen solve on the blocks of J (dims/order), async on ctx->stream: value_dev[0],
// vec_dev[0..n).  info_host/stats_host (nullable) force a synchronous read of
// [converged, picked end, steps, restarts, breakdowns] / [theta_lo, theta_hi,
// res_lo, res_hi, value].
void eig_blocks(r1_context* ctx, const uint64_t* dims, int order, const double* blocks,
                const double* x0, double* value_dev, double* vec_dev, int* info_host,
                double* stats_host, bool solver_chain, double decide_tol) {
    if (order < 2 || order > 16) fail(R1_ERR_INVALID_ARGUMENT, "eig: unsupported order");
    std::shared_ptr<EigPlan> P;
    {
        std::lock_guard<std::mutex> cache_lock(cache_mutex());
        auto& slot = eig_plans()[{ctx, std::vector<uint64_t>(dims, dims + order)}];
        if (!slot) {
            slot = std::make_shared<EigPlan>();
            blockop_layout(slot->op, dims, order, &slot->coldot_n, &slot->rowpart_n,
                           int64_t(1) << 40);
        }
        P = slot;
    }
    P->op.blocks = blocks;
    P->op.dense = nullptr;
    const int64_t n = P->op.n;
    static const char* dmax = dev_env("R1_EIG_DENSE_MAX");  // development: reference algorithm for small n
    if (dmax && n <= std::atoll(dmax) && !info_host && !stats_host) {
        P->dense_ws.ensure((static_cast<size_t>(n) * n + 4 * n + 32) * sizeof(double));
        double* S = P->dense_ws.as<double>();
        dense_from_blocks(ctx, dims, order, blocks, S);
        eig_dense_reference_device(ctx, n, S, S + n * n, value_dev, vec_dev);
        return;
    }
    run_lanczos(ctx, *P, x0, value_dev, vec_dev, info_host, stats_host, solver_chain, decide_tol);
}

// Same on a dense symmetric n x n matrix S (device, column-major).
void eig_dense(r1_context* ctx, int64_t n, const double* S, const double* x0, double* value_dev,
               double* vec_dev, int* info_host, double* stats_host) {
    std::shared_ptr<EigPlan> P;
    {
        std::lock_guard<std::mutex> cache_lock(cache_mutex());
        auto& slot = eig_plans()[{ctx, std::vector<uint64_t>{0, static_cast<uint64_t>(n)}}];
        if (!slot) {
            slot = std::make_shared<EigPlan>();
            denseop_layout(slot->op, n, &slot->rowpart_n);
            slot->coldot_n = 0;
        }
        P = slot;
    }
    P->op.dense = S;
    P->op.blocks = nullptr;
    run_lanczos(ctx, *P, x0, value_dev, vec_dev, info_host, stats_host);
}

}  // namespace r1
