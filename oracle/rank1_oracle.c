/*
 * ORACLE / TEST INFRASTRUCTURE — not product code.
 *
 * Plain-C restatement of the reference's hot-path arithmetic, used as the
 * CHECKER for the CUDA path (tests/, __graft_entry__.smoke(), bench.py's
 * cpu_baseline leg).  Each function cites the reference file:line it follows
 * (paths relative to /root/reference/proj).  It is pinned against the compiled
 * reference (oracle/_ref/librank1_ref.so) and the reference's own known-answer
 * tests in tests/test_oracle_pins.py; it must never be linked into the product.
 *
 * Contents
 *   - CounterRng (include/rank1/rng.hpp:10-37) and its Box-Muller gaussian
 *     (src/generators.cpp:11-24), counter-addressable so generation can be
 *     parallel and still bit-identical to gen_gaussian (generators.cpp:50-56).
 *   - The BASELINE.json config tensors in reference (column-major) dims.
 *   - TTV (src/tensor.cpp:100-138) and the per-block TTV chain with the
 *     largest-remaining-dimension-first order (src/nepv.cpp:46-77), giving
 *     build_j's blocks with the reference's exact operation order
 *     (no FMA contraction: compile with -ffp-contract=off).
 *   - Bunch-Kaufman LDL^T, its solve and the diagonal-condition estimate
 *     (src/sym_eig.cpp:233-407), for the iHOSCF RQI step (:411-438).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define GOLDEN 0x9e3779b97f4a7c15ull

/* ---------------------------------------------------------------- RNG -- */

/* splitmix64 finalizer, rng.hpp:24-31 */
static inline uint64_t mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xbf58476d1ce4e5b9ull;
    z ^= z >> 27;
    z *= 0x94d049bb133111ebull;
    z ^= z >> 31;
    return z;
}

/* key of CounterRng(seed, stream), rng.hpp:14-15 */
uint64_t r1o_rng_key(uint64_t seed, uint64_t stream) { return mix64(seed + GOLDEN * (stream + 1)); }

/* the c-th draw (c >= 1) of next_u64, rng.hpp:17 */
static inline uint64_t draw_u64(uint64_t key, uint64_t c) { return mix64(key + GOLDEN * c); }

/* next_unit at counter c, rng.hpp:20 */
static inline double draw_unit(uint64_t key, uint64_t c) {
    return (double)(draw_u64(key, c) >> 11) * 0x1.0p-53;
}

/* p-th value (0-based) of the next_gaussian() stream: Box-Muller pair p/2
 * consumes draws 2*(p/2)+1 (u1, nudged by 2^-54) and +2 (u2); even p is the
 * cosine branch, odd p the cached sine (generators.cpp:11-24). */
static inline double draw_gauss(uint64_t key, uint64_t p) {
    const uint64_t k = p >> 1;
    const double u1 = draw_unit(key, 2 * k + 1) + 0x1.0p-54;
    const double u2 = draw_unit(key, 2 * k + 2);
    const double r = sqrt(-2.0 * log(u1));
    const double a = 2.0 * 3.14159265358979323846 * u2;
    return (p & 1) ? r * sin(a) : r * cos(a);
}

void r1o_rng_units(uint64_t seed, uint64_t stream, uint64_t first, int64_t count, double* out) {
    const uint64_t key = r1o_rng_key(seed, stream);
    for (int64_t i = 0; i < count; ++i) out[i] = draw_unit(key, first + (uint64_t)i + 1);
}

void r1o_rng_u64(uint64_t seed, uint64_t stream, uint64_t first, int64_t count, uint64_t* out) {
    const uint64_t key = r1o_rng_key(seed, stream);
    for (int64_t i = 0; i < count; ++i) out[i] = draw_u64(key, first + (uint64_t)i + 1);
}

void r1o_rng_gauss(uint64_t seed, uint64_t stream, uint64_t first, int64_t count, double* out) {
    const uint64_t key = r1o_rng_key(seed, stream);
    for (int64_t i = 0; i < count; ++i) out[i] = draw_gauss(key, first + (uint64_t)i);
}

/* gen_gaussian(dims, seed): stream kStreamTensor = 1 (rng.hpp:40), layout order. */
void r1o_gen_gaussian(uint64_t n, uint64_t seed, double* out) {
    const uint64_t key = r1o_rng_key(seed, 1);
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < (int64_t)n; ++p) out[p] = draw_gauss(key, (uint64_t)p);
}

/* normalize(), matrix.cpp:62-67 (sequential sum of squares, divide) */
static double norm2_seq(const double* v, int64_t n) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += v[i] * v[i];
    return sqrt(s);
}

/* Planted unit factor for reference mode k: N(0,1)^I on stream 100+k, normalized. */
void r1o_planted_factor(uint64_t seed, int k, int64_t len, double* out) {
    const uint64_t key = r1o_rng_key(seed, 100 + (uint64_t)k);
    for (int64_t i = 0; i < len; ++i) out[i] = draw_gauss(key, (uint64_t)i);
    const double nrm = norm2_seq(out, len);
    if (nrm > 0.0)
        for (int64_t i = 0; i < len; ++i) out[i] /= nrm;
}

/* Fixed-order blocked sum of squares (2^20-entry chunks, sequential inside,
 * chunks summed in order) so a parallel host and any checker agree bitwise. */
double r1o_sumsq_blocked(const double* v, uint64_t n) {
    const uint64_t C = 1ull << 20;
    const uint64_t nb = (n + C - 1) / C;
    double* part = (double*)malloc(sizeof(double) * (nb ? nb : 1));
#pragma omp parallel for schedule(static)
    for (int64_t b = 0; b < (int64_t)nb; ++b) {
        const uint64_t lo = (uint64_t)b * C, hi = lo + C < n ? lo + C : n;
        double s = 0.0;
        for (uint64_t i = lo; i < hi; ++i) s += v[i] * v[i];
        part[b] = s;
    }
    double s = 0.0;
    for (uint64_t b = 0; b < nb; ++b) s += part[b];
    free(part);
    return s;
}

/*
 * BASELINE.json configs in REFERENCE dims (config dims reversed):
 *   cfg 1: gen_gaussian(dims, seed)                               (any dims)
 *   cfg 2: 10 * u0 o u1 o u2 + (0.01/sqrt(N)) * N(0,1)            (order 3)
 *   cfg 3: U(-1,1) = 2*next_unit()-1 on stream 1                  (any dims)
 *   cfg 4: 5 * o_k u_k + z/||z||_F, z = gen_gaussian              (any order)
 *   cfg 5: sum_r w_r sin((r+1) pi i/Ii) cos(r pi j/Ij) exp(-r k/Ik) + 1e-3 N(0,1)
 *          with config index (i,j,k) = (ref i2, ref i1, ref i0),  (order 3)
 *          config extents (Ii,Ij,Ik) = (4000,2000,500) at full size (= ref dims
 *          reversed), 0-based indices, w = (3, 1, 0.5).
 * Planted factors for cfg 2/4 use streams 100+k of the same seed.
 */
int r1o_gen_config(int cfg, const uint64_t* dims, int order, uint64_t seed, double* out) {
    uint64_t n = 1;
    for (int k = 0; k < order; ++k) n *= dims[k];
    if (cfg == 1) {
        r1o_gen_gaussian(n, seed, out);
        return 0;
    }
    if (cfg == 3) {
        const uint64_t key = r1o_rng_key(seed, 1);
#pragma omp parallel for schedule(static)
        for (int64_t p = 0; p < (int64_t)n; ++p)
            out[p] = 2.0 * draw_unit(key, (uint64_t)p + 1) - 1.0;
        return 0;
    }
    if (cfg == 2 || cfg == 4) {
        if (cfg == 2 && order != 3) return 1;
        double* fac[16];
        if (order > 16) return 1;
        for (int k = 0; k < order; ++k) {
            fac[k] = (double*)malloc(sizeof(double) * dims[k]);
            r1o_planted_factor(seed, k, (int64_t)dims[k], fac[k]);
        }
        r1o_gen_gaussian(n, seed, out); /* noise in place */
        double noise_scale;
        double weight;
        if (cfg == 2) {
            weight = 10.0;
            noise_scale = 0.01 / sqrt((double)n);
        } else {
            weight = 5.0;
            noise_scale = 1.0 / sqrt(r1o_sumsq_blocked(out, n));
        }
#pragma omp parallel for schedule(static)
        for (int64_t p = 0; p < (int64_t)n; ++p) {
            uint64_t q = (uint64_t)p;
            double prod = 1.0;
            for (int k = 0; k < order; ++k) {
                prod *= fac[k][q % dims[k]];
                q /= dims[k];
            }
            out[p] = weight * prod + noise_scale * out[p];
        }
        for (int k = 0; k < order; ++k) free(fac[k]);
        return 0;
    }
    if (cfg == 5) {
        if (order != 3) return 1;
        const double PI = 3.14159265358979323846;
        const uint64_t Ik = dims[0], Ij = dims[1], Ii = dims[2];
        const double w[3] = {3.0, 1.0, 0.5};
        double* si = (double*)malloc(sizeof(double) * 3 * Ii);
        double* cj = (double*)malloc(sizeof(double) * 3 * Ij);
        double* ek = (double*)malloc(sizeof(double) * 3 * Ik);
        for (int r = 1; r <= 3; ++r) {
            for (uint64_t i = 0; i < Ii; ++i)
                si[(r - 1) * Ii + i] = sin((double)(r + 1) * PI * (double)i / (double)Ii);
            for (uint64_t j = 0; j < Ij; ++j)
                cj[(r - 1) * Ij + j] = cos((double)r * PI * (double)j / (double)Ij);
            for (uint64_t k = 0; k < Ik; ++k)
                ek[(r - 1) * Ik + k] = exp(-(double)r * (double)k / (double)Ik);
        }
        r1o_gen_gaussian(n, seed, out);
#pragma omp parallel for schedule(static)
        for (int64_t p = 0; p < (int64_t)n; ++p) {
            const uint64_t k = (uint64_t)p % Ik;
            const uint64_t j = ((uint64_t)p / Ik) % Ij;
            const uint64_t i = (uint64_t)p / (Ik * Ij);
            double s = 0.0;
            for (int r = 0; r < 3; ++r) s += w[r] * si[r * Ii + i] * cj[r * Ij + j] * ek[r * Ik + k];
            out[p] = s + 1e-3 * out[p];
        }
        free(si);
        free(cj);
        free(ek);
        return 0;
    }
    return 1;
}

/* ---------------------------------------------------------------- TTV -- */

/* ttv(a, v, mode), tensor.cpp:100-138: pre==1 -> ordered dot products,
 * otherwise ordered axpy accumulation over the contracted index. */
static void ttv(const double* src, const uint64_t* dims, int order, int mode, const double* v,
                double* dst) {
    uint64_t pre = 1, post = 1;
    const uint64_t len = dims[mode];
    for (int k = 0; k < mode; ++k) pre *= dims[k];
    for (int k = mode + 1; k < order; ++k) post *= dims[k];
    if (pre == 1) {
        for (uint64_t q = 0; q < post; ++q) {
            const double* blk = src + q * len;
            double acc = 0.0;
            for (uint64_t i = 0; i < len; ++i) acc += blk[i] * v[i];
            dst[q] = acc;
        }
    } else {
        memset(dst, 0, sizeof(double) * pre * post);
        for (uint64_t q = 0; q < post; ++q) {
            double* o = dst + q * pre;
            for (uint64_t i = 0; i < len; ++i) {
                const double vi = v[i];
                const double* blk = src + (q * len + i) * pre;
                for (uint64_t p = 0; p < pre; ++p) o[p] += blk[p] * vi;
            }
        }
    }
}

/* One block B(ka,kb), ka<kb: the TTV chain of nepv.cpp:46-77 — repeatedly
 * contract the remaining non-kept mode of largest current extent (first such
 * mode on ties).  `fac[k]` is factor k.  out: I_ka x I_kb column-major. */
void r1o_block(const double* a, const uint64_t* dims, int order, const double* const* fac, int ka,
               int kb, double* out) {
    uint64_t n = 1;
    for (int k = 0; k < order; ++k) n *= dims[k];
    if (order == 2) {
        memcpy(out, a, sizeof(double) * n);
        return;
    }
    uint64_t cur_dims[32];
    int cur_modes[32];
    int m = order;
    for (int k = 0; k < order; ++k) {
        cur_dims[k] = dims[k];
        cur_modes[k] = k;
    }
    const double* src = a;
    double* buf = NULL;
    while (m > 2) {
        int pick = -1;
        uint64_t best = 0;
        for (int i = 0; i < m; ++i) {
            if (cur_modes[i] == ka || cur_modes[i] == kb) continue;
            if (pick < 0 || cur_dims[i] > best) {
                pick = i;
                best = cur_dims[i];
            }
        }
        uint64_t on = 1;
        for (int i = 0; i < m; ++i)
            if (i != pick) on *= cur_dims[i];
        double* nb = (double*)malloc(sizeof(double) * on);
        ttv(src, cur_dims, m, pick, fac[cur_modes[pick]], nb);
        if (buf) free(buf);
        buf = nb;
        src = nb;
        for (int i = pick; i + 1 < m; ++i) {
            cur_dims[i] = cur_dims[i + 1];
            cur_modes[i] = cur_modes[i + 1];
        }
        --m;
    }
    memcpy(out, src, sizeof(double) * cur_dims[0] * cur_dims[1]);
    free(buf);
}

/* All P blocks in pair order (nepv.cpp:211-229); blocks are independent, so
 * the OpenMP loop over pairs does not change any value. */
void r1o_build_j(const double* a, const uint64_t* dims, int order, const double* factors_flat,
                 double* blocks) {
    const double* fac[32];
    uint64_t off = 0;
    for (int k = 0; k < order; ++k) {
        fac[k] = factors_flat + off;
        off += dims[k];
    }
    int pm[512], pn[512];
    uint64_t boff[512];
    int np = 0;
    uint64_t bo = 0;
    for (int m = 0; m < order; ++m)
        for (int n = m + 1; n < order; ++n) {
            pm[np] = m;
            pn[np] = n;
            boff[np] = bo;
            bo += dims[m] * dims[n];
            ++np;
        }
#pragma omp parallel for schedule(dynamic)
    for (int i = 0; i < np; ++i) r1o_block(a, dims, order, fac, pm[i], pn[i], blocks + boff[i]);
}

/* ------------------------------------------------------- Bunch-Kaufman -- */

/* ldlt_factor, sym_eig.cpp:233-320 (lower storage, alpha=(1+sqrt 17)/8).
 * w: n x n column-major, overwritten; ipiv: >=0 1x1 pivot row, <0 2x2 with
 * kp = -ipiv-1.  Returns the singular flag. */
int r1o_ldlt_factor(int64_t n, double* w, int* ipiv) {
#define W(i, j) w[(i) + (j) * n]
    const double alpha = (1.0 + sqrt(17.0)) / 8.0;
    int singular = 0;
    int64_t k = 0;
    while (k < n) {
        int64_t kstep = 1, kp = k, imax = k;
        const double absakk = fabs(W(k, k));
        double colmax = 0.0;
        for (int64_t i = k + 1; i < n; ++i)
            if (fabs(W(i, k)) > colmax) {
                colmax = fabs(W(i, k));
                imax = i;
            }
        if ((absakk > colmax ? absakk : colmax) == 0.0) {
            singular = 1;
            ipiv[k] = (int)k;
            ++k;
            continue;
        }
        if (absakk >= alpha * colmax) {
            kp = k;
        } else {
            double rowmax = 0.0;
            for (int64_t j = k; j < imax; ++j)
                if (fabs(W(imax, j)) > rowmax) rowmax = fabs(W(imax, j));
            for (int64_t i = imax + 1; i < n; ++i)
                if (fabs(W(i, imax)) > rowmax) rowmax = fabs(W(i, imax));
            if (absakk * rowmax >= alpha * colmax * colmax)
                kp = k;
            else if (fabs(W(imax, imax)) >= alpha * rowmax)
                kp = imax;
            else {
                kp = imax;
                kstep = 2;
            }
        }
        const int64_t kk = k + kstep - 1;
        if (kp != kk) {
            double t;
            for (int64_t i = kp + 1; i < n; ++i) {
                t = W(i, kk);
                W(i, kk) = W(i, kp);
                W(i, kp) = t;
            }
            for (int64_t j = kk + 1; j < kp; ++j) {
                t = W(j, kk);
                W(j, kk) = W(kp, j);
                W(kp, j) = t;
            }
            t = W(kk, kk);
            W(kk, kk) = W(kp, kp);
            W(kp, kp) = t;
            if (kstep == 2) {
                t = W(k + 1, k);
                W(k + 1, k) = W(kp, k);
                W(kp, k) = t;
            }
        }
        if (kstep == 1) {
            const double dkk = W(k, k);
            if (dkk == 0.0) {
                singular = 1;
            } else {
                const double r1 = 1.0 / dkk;
                for (int64_t j = k + 1; j < n; ++j) {
                    const double cj = r1 * W(j, k);
                    for (int64_t i = j; i < n; ++i) W(i, j) -= W(i, k) * cj;
                }
                for (int64_t i = k + 1; i < n; ++i) W(i, k) *= r1;
            }
            ipiv[k] = (int)kp;
        } else {
            if (k + 2 < n) {
                const double d21 = W(k + 1, k);
                const double d11 = W(k + 1, k + 1) / d21;
                const double d22 = W(k, k) / d21;
                const double t = 1.0 / (d11 * d22 - 1.0);
                const double d21t = t / d21;
                for (int64_t j = k + 2; j < n; ++j) {
                    const double wk = d21t * (d11 * W(j, k) - W(j, k + 1));
                    const double wkp1 = d21t * (d22 * W(j, k + 1) - W(j, k));
                    for (int64_t i = j; i < n; ++i) W(i, j) -= W(i, k) * wk + W(i, k + 1) * wkp1;
                    W(j, k) = wk;
                    W(j, k + 1) = wkp1;
                }
            }
            ipiv[k] = (int)(-kp - 1);
            ipiv[k + 1] = ipiv[k];
        }
        k += kstep;
    }
    return singular;
}

/* ldlt_solve, sym_eig.cpp:322-379 (b overwritten with the solution). */
void r1o_ldlt_solve(int64_t n, const double* w, const int* ipiv, double* b) {
    int64_t k = 0;
    while (k < n) {
        if (ipiv[k] >= 0) {
            const int64_t kp = ipiv[k];
            if (kp != k) {
                double t = b[k];
                b[k] = b[kp];
                b[kp] = t;
            }
            for (int64_t i = k + 1; i < n; ++i) b[i] -= W(i, k) * b[k];
            b[k] /= W(k, k);
            ++k;
        } else {
            const int64_t kp = -ipiv[k] - 1;
            if (kp != k + 1) {
                double t = b[k + 1];
                b[k + 1] = b[kp];
                b[kp] = t;
            }
            for (int64_t i = k + 2; i < n; ++i) b[i] -= W(i, k) * b[k] + W(i, k + 1) * b[k + 1];
            const double akm1k = W(k + 1, k);
            const double akm1 = W(k, k) / akm1k;
            const double ak = W(k + 1, k + 1) / akm1k;
            const double denom = akm1 * ak - 1.0;
            const double bkm1 = b[k] / akm1k;
            const double bk = b[k + 1] / akm1k;
            b[k] = (ak * bkm1 - bk) / denom;
            b[k + 1] = (akm1 * bk - bkm1) / denom;
            k += 2;
        }
    }
    int64_t kb = n;
    while (kb > 0) {
        const int64_t kk = kb - 1;
        if (ipiv[kk] >= 0) {
            double acc = 0.0;
            for (int64_t i = kk + 1; i < n; ++i) acc += W(i, kk) * b[i];
            b[kk] -= acc;
            const int64_t kp = ipiv[kk];
            if (kp != kk) {
                double t = b[kk];
                b[kk] = b[kp];
                b[kp] = t;
            }
            --kb;
        } else {
            double acc0 = 0.0, acc1 = 0.0;
            for (int64_t i = kk + 1; i < n; ++i) {
                acc1 += W(i, kk) * b[i];
                acc0 += W(i, kk - 1) * b[i];
            }
            b[kk] -= acc1;
            b[kk - 1] -= acc0;
            const int64_t kp = -ipiv[kk] - 1;
            if (kp != kk) {
                double t = b[kk];
                b[kk] = b[kp];
                b[kp] = t;
            }
            kb -= 2;
        }
    }
}

/* ldlt_diag_condition, sym_eig.cpp:381-407. */
double r1o_ldlt_diag_condition(int64_t n, const double* w, const int* ipiv, int singular) {
    if (singular) return INFINITY;
    double lo = INFINITY, hi = 0.0;
    int64_t k = 0;
    while (k < n) {
        if (ipiv[k] >= 0) {
            const double m = fabs(W(k, k));
            if (m < lo) lo = m;
            if (m > hi) hi = m;
            ++k;
        } else {
            const double a = W(k, k), c = W(k + 1, k + 1), bb = W(k + 1, k);
            const double mid = 0.5 * (a + c);
            const double rad = hypot(0.5 * (a - c), bb);
            const double e1 = fabs(mid + rad), e2 = fabs(mid - rad);
            const double mn = e1 < e2 ? e1 : e2, mx = e1 > e2 ? e1 : e2;
            if (mn < lo) lo = mn;
            if (mx > hi) hi = mx;
            k += 2;
        }
    }
    if (lo == 0.0) return INFINITY;
    return hi / lo;
}
#undef W

/* rayleigh_quotient_step, sym_eig.cpp:411-438.  Returns 1 and y when the
 * step is accepted, 0 for nullopt.  s is n x n column-major (unchanged). */
int r1o_rqi_step(int64_t n, const double* s, const double* x, double* y) {
    double* sx = (double*)calloc((size_t)n, sizeof(double));
    for (int64_t j = 0; j < n; ++j) {
        const double xj = x[j];
        const double* c = s + j * n;
        for (int64_t i = 0; i < n; ++i) sx[i] += c[i] * xj;
    }
    double rho = 0.0;
    for (int64_t i = 0; i < n; ++i) rho += x[i] * sx[i];
    free(sx);
    double* w = (double*)malloc(sizeof(double) * (size_t)(n * n));
    int* ipiv = (int*)malloc(sizeof(int) * (size_t)n);
    int ok = 0;
    for (int attempt = 0; attempt < 2 && !ok; ++attempt) {
        double shift = rho;
        if (attempt == 1) {
            if (rho != 0.0) {
                shift = rho * (1.0 + 1e-10);
            } else {
                double f = 0.0;
                for (int64_t i = 0; i < n * n; ++i) f += s[i] * s[i];
                f = sqrt(f);
                shift = 1e-10 * (f > 1e-300 ? f : 1e-300);
            }
        }
        memcpy(w, s, sizeof(double) * (size_t)(n * n));
        for (int64_t i = 0; i < n; ++i) w[i + i * n] -= shift;
        const int sing = r1o_ldlt_factor(n, w, ipiv);
        if (sing || r1o_ldlt_diag_condition(n, w, ipiv, sing) > 1e14) continue;
        memcpy(y, x, sizeof(double) * (size_t)n);
        r1o_ldlt_solve(n, w, ipiv, y);
        double nrm = 0.0;
        for (int64_t i = 0; i < n; ++i) nrm += y[i] * y[i];
        nrm = sqrt(nrm);
        if (!isfinite(nrm) || nrm == 0.0) continue;
        for (int64_t i = 0; i < n; ++i) y[i] /= nrm;
        ok = 1;
    }
    free(w);
    free(ipiv);
    return ok;
}
