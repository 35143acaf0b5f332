// Block-operator matvec y = J x, J = scale * [B(m,n)] (upper blocks, pair
// order, column-major; reference nepv.cpp:110-134), as device functions that
// both the standalone matvec kernels and the persistent Lanczos kernel use.
//
// Phase A: task (pair, 32-column chunk, chunk of <= kMvRows rows) computes
//          the column dots (B' x_m)[j] of its columns over its rows and the
//          row partials (B x_n)[i] of its rows over its columns (row chunks
//          keep the tasks of tall and short blocks the same size: the grid's
//          barriers wait for the largest task).
// Phase B: every output entry sums its contributions in a fixed order.
// Tasks are assigned round-robin over a fixed grid: deterministic.
#pragma once

#include <cstdint>
#include <vector>

namespace r1 {

constexpr int kMvCols = 32;   // columns per phase-A task
constexpr int kMvRows = 512;  // rows per phase-A task
constexpr int kMvMaxPairs = 120;

struct BlockOp {
    int d = 0;
    int npairs = 0;
    int ntasks = 0;
    int64_t n = 0;                       // sum I_k
    int64_t dims[16] = {};
    int64_t offs[17] = {};               // stacked-vector offsets
    int64_t boff[kMvMaxPairs] = {};      // element offset of block p
    int64_t cd_off[kMvMaxPairs] = {};    // column dots of pair p (nrc * I_n entries, row-chunk major)
    int64_t rp_off[kMvMaxPairs] = {};    // row partials of pair p (nchunk * I_m)
    int task_first[kMvMaxPairs + 1] = {};
    int nrc[kMvMaxPairs] = {};           // row chunks of pair p
    int64_t rows_per_task = kMvRows;
    signed char pm[kMvMaxPairs] = {}, pn[kMvMaxPairs] = {};
    double scale = 1.0;
    const double* blocks = nullptr;
    double* coldot = nullptr;
    double* rowpart = nullptr;
    const double* dense = nullptr;  // dense mode: y = S x for an n x n column-major S
};

// Dense-operator layout: tasks are 32-column chunks of S, no scale.
inline void denseop_layout(BlockOp& op, int64_t n, int64_t* rowpart_n) {
    op = BlockOp{};
    op.d = 1;
    op.n = n;
    op.offs[0] = 0;
    op.offs[1] = n;
    op.dims[0] = n;
    op.scale = 1.0;
    op.ntasks = static_cast<int>((n + kMvCols - 1) / kMvCols);
    *rowpart_n = static_cast<int64_t>(op.ntasks) * n;
}

__host__ __device__ inline int pair_index(int m, int n, int d) {
    return m * (2 * d - m - 1) / 2 + (n - m - 1);
}

// Sizes (doubles) of the two scratch areas of a BlockOp.
// rows_per_task: the phase-A row chunk (the standalone matvec kernels use
// kMvRows; the persistent Lanczos kernel keeps whole blocks per task, where
// more, smaller tasks measured slower)
inline void blockop_layout(BlockOp& op, const uint64_t* dims, int d, int64_t* coldot_n,
                           int64_t* rowpart_n, int64_t rows_per_task = kMvRows) {
    op.d = d;
    op.rows_per_task = rows_per_task;
    op.offs[0] = 0;
    for (int k = 0; k < d; ++k) {
        op.dims[k] = static_cast<int64_t>(dims[k]);
        op.offs[k + 1] = op.offs[k] + op.dims[k];
    }
    op.n = op.offs[d];
    op.scale = 1.0 / static_cast<double>(d - 1);
    int p = 0, task = 0;
    int64_t bo = 0, co = 0, ro = 0;
    for (int m = 0; m < d; ++m)
        for (int n = m + 1; n < d; ++n, ++p) {
            op.pm[p] = static_cast<signed char>(m);
            op.pn[p] = static_cast<signed char>(n);
            op.boff[p] = bo;
            op.cd_off[p] = co;
            op.rp_off[p] = ro;
            op.task_first[p] = task;
            const int64_t nch = (op.dims[n] + kMvCols - 1) / kMvCols;
            const int64_t nrc = (op.dims[m] + rows_per_task - 1) / rows_per_task;
            op.nrc[p] = static_cast<int>(nrc);
            task += static_cast<int>(nch * nrc);
            bo += op.dims[m] * op.dims[n];
            co += nrc * op.dims[n];
            ro += nch * op.dims[m];
        }
    op.npairs = p;
    op.task_first[p] = task;
    op.ntasks = task;
    *coldot_n = co;
    *rowpart_n = ro;
}

#ifdef __CUDACC__
// Phase A over tasks [blockIdx.x :: gridDim.x] for the input xscale * x.
// CHUNKED = false: the layout has one row chunk per pair (the Lanczos
// kernel: no chunk decode, fewer registers at its 128-register cap)
template <bool CHUNKED = true>
__device__ inline void blockop_phase_a(const BlockOp& op, const double* __restrict__ x,
                                       double xscale = 1.0) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    if (op.dense) {
        const int64_t n = op.n;
        for (int t = blockIdx.x; t < op.ntasks; t += gridDim.x) {
            const int64_t j0 = static_cast<int64_t>(t) * kMvCols;
            const int nc = static_cast<int>(n - j0 < kMvCols ? n - j0 : kMvCols);
            double* rp = op.rowpart + static_cast<int64_t>(t) * n;
            for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
                const double* si = op.dense + i + j0 * n;
                double s = 0.0;
#pragma unroll
                for (int h = 0; h < kMvCols; h += 16) {
                    double sv[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j) sv[j] = h + j < nc ? si[(h + j) * n] : 0.0;
#pragma unroll
                    for (int j = 0; j < 16; ++j) s = fma(sv[j], h + j < nc ? x[j0 + h + j] : 0.0, s);
                }
                rp[i] = s * xscale;
            }
        }
        return;
    }
    for (int t = blockIdx.x; t < op.ntasks; t += gridDim.x) {
        int p = 0;
        while (t >= op.task_first[p + 1]) ++p;
        const int local = t - op.task_first[p];
        const int c = CHUNKED ? local / op.nrc[p] : local;
        const int rc = CHUNKED ? local - c * op.nrc[p] : 0;
        const int m = op.pm[p], n = op.pn[p];
        const int64_t rows = op.dims[m], cols = op.dims[n];
        const int64_t i0 = CHUNKED ? static_cast<int64_t>(rc) * op.rows_per_task : 0;
        const int64_t i1 = !CHUNKED || rows - i0 < op.rows_per_task ? rows : i0 + op.rows_per_task;
        const double* B = op.blocks + op.boff[p];
        const int64_t j0 = static_cast<int64_t>(c) * kMvCols;
        const int nc = static_cast<int>(cols - j0 < kMvCols ? cols - j0 : kMvCols);
        const double* xm = x + op.offs[m];
        const double* xn = x + op.offs[n] + j0;
        double* rp = op.rowpart + op.rp_off[p] + static_cast<int64_t>(c) * rows;
        // row partials: batches of 16 independent loads per row, FMAs in order
        for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
            const double* bi = B + i + j0 * rows;
            double s = 0.0;
#pragma unroll
            for (int h = 0; h < kMvCols; h += 16) {
                double bv[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) bv[j] = h + j < nc ? bi[(h + j) * rows] : 0.0;
#pragma unroll
                for (int j = 0; j < 16; ++j) s = fma(bv[j], h + j < nc ? xn[h + j] : 0.0, s);
            }
            rp[i] = s * xscale;
        }
        // column dots: warp per column, 4 independent accumulators per lane
        for (int j = warp; j < nc; j += nw) {
            const double* col = B + (j0 + j) * rows;
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
            int64_t i = i0 + lane;
            for (; i + 96 < i1; i += 128) {
                s0 = fma(col[i], xm[i], s0);
                s1 = fma(col[i + 32], xm[i + 32], s1);
                s2 = fma(col[i + 64], xm[i + 64], s2);
                s3 = fma(col[i + 96], xm[i + 96], s3);
            }
            for (; i < i1; i += 32) s0 = fma(col[i], xm[i], s0);
            double s = (s0 + s1) + (s2 + s3);
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
            if (lane == 0) op.coldot[op.cd_off[p] + (CHUNKED ? rc * cols : 0) + j0 + j] = s * xscale;
        }
    }
}

// Phase B: y[t] for t in [start, end) step stride (end < 0: n).
template <bool CHUNKED = true>
__device__ inline void blockop_phase_b(const BlockOp& op, double* __restrict__ y, int64_t start,
                                       int64_t stride, int64_t end = -1) {
    const int d = op.d;
    const int64_t stop = end < 0 ? op.n : end;
    if (op.dense) {
        for (int64_t t = start; t < stop; t += stride) {
            double s = 0.0;
            for (int c = 0; c < op.ntasks; ++c) s += op.rowpart[static_cast<int64_t>(c) * op.n + t];
            y[t] = s;
        }
        return;
    }
    for (int64_t t = start; t < stop; t += stride) {
        int m = 0;
        while (t >= op.offs[m + 1]) ++m;
        const int64_t i = t - op.offs[m];
        double s = 0.0;
        for (int k = 0; k < m; ++k) {
            const int p = pair_index(k, m, d);
            const double* cd = op.coldot + op.cd_off[p] + i;
            if (!CHUNKED) {
                s += cd[0];
            } else {
                for (int rc = 0; rc < op.nrc[p]; ++rc) s += cd[static_cast<int64_t>(rc) * op.dims[m]];
            }
        }
        for (int n = m + 1; n < d; ++n) {
            const int p = pair_index(m, n, d);
            const int64_t nch = (op.dims[n] + kMvCols - 1) / kMvCols;
            const double* rp = op.rowpart + op.rp_off[p] + i;
            double r = 0.0;
#pragma unroll 8
            for (int64_t c = 0; c < nch; ++c) r += rp[c * op.dims[m]];
            s += r;
        }
        y[t] = s * op.scale;
    }
}
#endif

}  // namespace r1
