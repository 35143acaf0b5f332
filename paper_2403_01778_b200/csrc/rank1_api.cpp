// The C++ rank1:: drop-in (include/rank1/*.hpp) on top of the C-ABI
// (include/rank1_b200.h).  Container types are host-side as in the reference;
// every numeric step of the hot path (sweep, eigen step, RQI, stopping test,
// KKT, solvers) goes through r1_* into the sm_100a kernels.  Status codes are
// mapped back to the reference's exception types (invalid_argument /
// runtime_error).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <stdexcept>
#include <string>

#include "rank1/greedy.hpp"
#include "rank1/nepv.hpp"
#include "rank1/solvers.hpp"
#include "rank1/stacked.hpp"
#include "rank1/sym_eig.hpp"
#include "rank1/tensor.hpp"
#include "rank1/tensor_io.hpp"
#include "rank1_b200.h"

namespace rank1 {

namespace {

void raise(int rc) {
    if (rc == R1_OK) return;
    const std::string msg = r1_last_error();
    if (rc == R1_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

// Process-wide device context on device 0 (created on first use).
r1_context* ctx() {
    static std::once_flag once;
    static r1_context* c = nullptr;
    static int rc = R1_OK;
    static std::string err;
    std::call_once(once, [] {
        rc = r1_context_create(0, &c);
        if (rc != R1_OK) err = r1_last_error();
    });
    if (rc != R1_OK) throw std::runtime_error(err);
    return c;
}

std::vector<uint64_t> u64(const std::vector<std::size_t>& d) { return {d.begin(), d.end()}; }

std::vector<double> flat(const FactorSet& f) {
    std::vector<double> v;
    for (const auto& u : f.factors) v.insert(v.end(), u.begin(), u.end());
    return v;
}

void check_shapes(const DenseTensor& a, const FactorSet& f) {
    if (f.order() != a.order()) throw std::invalid_argument("factor set order mismatch");
    for (std::size_t k = 0; k < a.order(); ++k)
        if (f.factors[k].size() != a.dim(k))
            throw std::invalid_argument("factor length does not match tensor dim");
}

std::vector<double> blocks_of(const SymBlockMatrix& j) {
    std::vector<double> b;
    for (std::size_t m = 0; m < j.order(); ++m)
        for (std::size_t n = m + 1; n < j.order(); ++n) {
            const Matrix& x = j.block(m, n);
            b.insert(b.end(), x.values().begin(), x.values().end());
        }
    return b;
}

SymBlockMatrix from_blocks(const std::vector<std::size_t>& dims, const std::vector<double>& b) {
    SymBlockMatrix j(dims);
    std::size_t off = 0;
    for (std::size_t m = 0; m < dims.size(); ++m)
        for (std::size_t n = m + 1; n < dims.size(); ++n) {
            Matrix& x = j.block(m, n);
            std::memcpy(x.data(), b.data() + off, sizeof(double) * x.rows() * x.cols());
            off += x.rows() * x.cols();
        }
    return j;
}

}  // namespace

// ------------------------------------------------------------------ Matrix --
Matrix transpose(const Matrix& m) {
    Matrix t(m.cols(), m.rows());
    for (std::size_t j = 0; j < m.cols(); ++j)
        for (std::size_t i = 0; i < m.rows(); ++i) t(j, i) = m(i, j);
    return t;
}

std::vector<double> matvec(const Matrix& m, std::span<const double> x) {
    if (x.size() != m.cols()) throw std::invalid_argument("matvec: size mismatch");
    std::vector<double> y(m.rows(), 0.0);
    for (std::size_t j = 0; j < m.cols(); ++j)
        for (std::size_t i = 0; i < m.rows(); ++i) y[i] += m(i, j) * x[j];
    return y;
}

std::vector<double> matvec_transposed(const Matrix& m, std::span<const double> x) {
    if (x.size() != m.rows()) throw std::invalid_argument("matvec_transposed: size mismatch");
    std::vector<double> y(m.cols(), 0.0);
    for (std::size_t j = 0; j < m.cols(); ++j) {
        double s = 0.0;
        for (std::size_t i = 0; i < m.rows(); ++i) s += m(i, j) * x[i];
        y[j] = s;
    }
    return y;
}

double frobenius_norm(const Matrix& m) {
    double s = 0.0;
    for (double v : m.values()) s += v * v;
    return std::sqrt(s);
}

double max_abs(const Matrix& m) {
    double s = 0.0;
    for (double v : m.values()) s = std::max(s, std::abs(v));
    return s;
}

double dot(std::span<const double> a, std::span<const double> b) {
    if (a.size() != b.size()) throw std::invalid_argument("dot: size mismatch");
    double s = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
    return s;
}

double norm2(std::span<const double> v) {
    double s = 0.0;
    for (double x : v) s += x * x;
    return std::sqrt(s);
}

double normalize(std::span<double> v) {
    const double n = norm2(v);
    if (n > 0.0)
        for (double& x : v) x /= n;
    return n;
}

// -------------------------------------------------------------- DenseTensor --
namespace {
std::size_t checked_numel(const std::vector<std::size_t>& dims) {
    if (dims.empty()) throw std::invalid_argument("DenseTensor: order must be >= 1");
    std::size_t n = 1;
    for (std::size_t d : dims) {
        if (d == 0) throw std::invalid_argument("DenseTensor: all dims must be >= 1");
        if (n > std::size_t(-1) / d) throw std::invalid_argument("DenseTensor: size overflow");
        n *= d;
    }
    return n;
}
}  // namespace

DenseTensor::DenseTensor(std::vector<std::size_t> dims)
    : dims_(std::move(dims)), data_(checked_numel(dims_), 0.0) {}

DenseTensor::DenseTensor(std::vector<std::size_t> dims, std::vector<double> data)
    : dims_(std::move(dims)), data_(std::move(data)) {
    if (checked_numel(dims_) != data_.size())
        throw std::invalid_argument("DenseTensor: data length does not match product of dims");
}

std::size_t DenseTensor::linear_index(std::span<const std::size_t> idx) const {
    if (idx.size() != dims_.size()) throw std::invalid_argument("DenseTensor: index arity mismatch");
    std::size_t p = 0, stride = 1;
    for (std::size_t k = 0; k < dims_.size(); ++k) {
        if (idx[k] >= dims_[k]) throw std::out_of_range("DenseTensor: index out of range");
        p += idx[k] * stride;
        stride *= dims_[k];
    }
    return p;
}

double max_unit_deviation(const FactorSet& f) {
    double dev = 0.0;
    for (const auto& u : f.factors) dev = std::max(dev, std::abs(norm2(u) - 1.0));
    return dev;
}

double frobenius_norm(const DenseTensor& a) {
    double s = 0.0;
    for (double v : a.values()) s += v * v;
    return std::sqrt(s);
}

double multilinear_value(const DenseTensor& a, const FactorSet& f, bool) {
    if (f.order() != a.order()) throw std::invalid_argument("multilinear_value: order mismatch");
    // lambda = u0' B(0,1) u1 of one device sweep; the sweep needs unit
    // factors, so contract with normalised ones and rescale by the norms.
    FactorSet g = f;
    double scale = 1.0;
    for (auto& u : g.factors) {
        const double n = normalize(u);
        if (n == 0.0) return 0.0;
        scale *= n;
    }
    const auto dims = u64(a.dims());
    std::vector<double> out(a.order() + 2);
    const auto fl = flat(g);
    raise(r1_kkt_report(ctx(), a.data(), nullptr, dims.data(), static_cast<int>(a.order()),
                        fl.data(), out.data()));
    return out[0] * scale;
}

// ----------------------------------------------------------- StackedVector --
namespace {
std::vector<std::size_t> offsets(const std::vector<std::size_t>& d) {
    std::vector<std::size_t> o(d.size(), 0);
    for (std::size_t n = 1; n < d.size(); ++n) o[n] = o[n - 1] + d[n - 1];
    return o;
}
}  // namespace

StackedVector::StackedVector(std::vector<std::size_t> block_dims)
    : dims_(std::move(block_dims)), offs_(offsets(dims_)),
      flat_(std::accumulate(dims_.begin(), dims_.end(), std::size_t{0}), 0.0) {}

StackedVector::StackedVector(std::vector<std::size_t> block_dims, std::vector<double> flat)
    : dims_(std::move(block_dims)), offs_(offsets(dims_)), flat_(std::move(flat)) {
    if (std::accumulate(dims_.begin(), dims_.end(), std::size_t{0}) != flat_.size())
        throw std::invalid_argument("StackedVector: flat length does not match block dims");
}

double StackedVector::block_norm(std::size_t n) const { return norm2(block(n)); }
double StackedVector::norm() const { return norm2(flat_); }

SplitResult split_factors(const StackedVector& x) {
    SplitResult r;
    r.factors.factors.resize(x.order());
    r.degenerate.assign(x.order(), 0);
    for (std::size_t n = 0; n < x.order(); ++n) {
        auto b = x.block(n);
        auto& u = r.factors.factors[n];
        u.assign(b.begin(), b.end());
        const double nrm = norm2(u);
        if (nrm < 1e-12) {
            std::fill(u.begin(), u.end(), 0.0);
            r.degenerate[n] = 1;
        } else {
            for (double& v : u) v /= nrm;
        }
    }
    return r;
}

StackedVector stack_factors(const FactorSet& f) {
    if (f.order() == 0) throw std::invalid_argument("stack_factors: empty factor set");
    if (max_unit_deviation(f) > 1e-8)
        throw std::invalid_argument("stack_factors: factors must have unit norm");
    std::vector<std::size_t> dims;
    for (const auto& u : f.factors) dims.push_back(u.size());
    StackedVector x(dims);
    const double s = 1.0 / std::sqrt(static_cast<double>(f.order()));
    for (std::size_t n = 0; n < f.order(); ++n) {
        auto b = x.block(n);
        for (std::size_t i = 0; i < b.size(); ++i) b[i] = f.factors[n][i] * s;
    }
    return x;
}

StackedVector flip_first_block(const StackedVector& x) {
    StackedVector y = x;
    for (double& v : y.block(0)) v = -v;
    return y;
}

FactorSet flip_first_factor(FactorSet f) {
    if (f.order() == 0) throw std::invalid_argument("flip_first_factor: empty factor set");
    for (double& v : f.factors[0]) v = -v;
    return f;
}

// ----------------------------------------------------------- SymBlockMatrix --
SymBlockMatrix::SymBlockMatrix(std::vector<std::size_t> block_dims)
    : dims_(std::move(block_dims)) {
    const std::size_t d = dims_.size();
    if (d < 2) throw std::invalid_argument("SymBlockMatrix: order must be >= 2");
    offs_ = offsets(dims_);
    upper_.resize(d * (d - 1) / 2);
    for (std::size_t m = 0; m < d; ++m)
        for (std::size_t n = m + 1; n < d; ++n) upper_[pair_index(m, n)] = Matrix(dims_[m], dims_[n]);
    scale_ = 1.0 / static_cast<double>(d - 1);
}

std::size_t SymBlockMatrix::total_dim() const {
    return std::accumulate(dims_.begin(), dims_.end(), std::size_t{0});
}

std::size_t SymBlockMatrix::pair_index(std::size_t m, std::size_t n) const {
    const std::size_t d = dims_.size();
    if (m >= n || n >= d) throw std::invalid_argument("SymBlockMatrix: bad block pair");
    return m * (2 * d - m - 1) / 2 + (n - m - 1);
}

const Matrix& SymBlockMatrix::block(std::size_t m, std::size_t n) const { return upper_[pair_index(m, n)]; }
Matrix& SymBlockMatrix::block(std::size_t m, std::size_t n) { return upper_[pair_index(m, n)]; }

std::vector<double> SymBlockMatrix::matvec(std::span<const double> x) const {
    if (x.size() != total_dim()) throw std::invalid_argument("SymBlockMatrix: matvec size mismatch");
    std::vector<double> y(x.size(), 0.0);
    for (std::size_t m = 0; m < dims_.size(); ++m)
        for (std::size_t n = m + 1; n < dims_.size(); ++n) {
            const Matrix& b = block(m, n);
            for (std::size_t j = 0; j < b.cols(); ++j) {
                double acc = 0.0;
                for (std::size_t i = 0; i < b.rows(); ++i) {
                    y[offs_[m] + i] += b(i, j) * x[offs_[n] + j];
                    acc += b(i, j) * x[offs_[m] + i];
                }
                y[offs_[n] + j] += acc;
            }
        }
    for (double& v : y) v *= scale_;
    return y;
}

Matrix SymBlockMatrix::dense() const {
    Matrix s(total_dim(), total_dim());
    for (std::size_t m = 0; m < dims_.size(); ++m)
        for (std::size_t n = m + 1; n < dims_.size(); ++n) {
            const Matrix& b = block(m, n);
            for (std::size_t j = 0; j < b.cols(); ++j)
                for (std::size_t i = 0; i < b.rows(); ++i) {
                    const double v = b(i, j) * scale_;
                    s(offs_[m] + i, offs_[n] + j) = v;
                    s(offs_[n] + j, offs_[m] + i) = v;
                }
        }
    return s;
}

double SymBlockMatrix::frobenius_norm() const {
    double s = 0.0;
    for (const Matrix& b : upper_)
        for (double v : b.values()) s += v * v;
    return std::sqrt(2.0 * s) * scale_;
}

// ------------------------------------------------------------- the sweep --
SymBlockMatrix build_j(const DenseTensor& a, const FactorSet& f, const BuildOptions&) {
    if (a.order() < 2) throw std::invalid_argument("build_j: tensor order must be >= 2");
    check_shapes(a, f);
    const auto dims = u64(a.dims());
    std::vector<double> blocks(r1_blocks_numel(dims.data(), static_cast<int>(a.order())));
    const auto fl = flat(f);
    raise(r1_build_j(ctx(), a.data(), nullptr, dims.data(), static_cast<int>(a.order()), fl.data(),
                     blocks.data()));
    return from_blocks(a.dims(), blocks);
}

SymBlockMatrix build_j_serial(const DenseTensor& a, const FactorSet& f) {
    if (a.order() < 2) throw std::invalid_argument("build_j_serial: tensor order must be >= 2");
    return build_j(a, f, BuildOptions{});
}

Matrix build_block(const DenseTensor& a, const FactorSet& f, std::size_t m, std::size_t n) {
    if (a.order() < 2) throw std::invalid_argument("build_block: tensor order must be >= 2");
    if (m == n) throw std::invalid_argument("build_block: block modes must differ");
    if (m > n) std::swap(m, n);
    if (n >= a.order()) throw std::invalid_argument("build_block: mode out of range");
    check_shapes(a, f);
    const auto dims = u64(a.dims());
    Matrix b(a.dim(m), a.dim(n));
    const auto fl = flat(f);
    raise(r1_build_block(ctx(), a.data(), nullptr, dims.data(), static_cast<int>(a.order()), fl.data(),
                         static_cast<int>(m), static_cast<int>(n), b.data()));
    return b;
}

KktReport kkt_report(const DenseTensor& a, const FactorSet& f, bool) {
    check_shapes(a, f);
    const auto dims = u64(a.dims());
    std::vector<double> out(a.order() + 2);
    const auto fl = flat(f);
    raise(r1_kkt_report(ctx(), a.data(), nullptr, dims.data(), static_cast<int>(a.order()), fl.data(),
                        out.data()));
    KktReport r;
    r.lambda = out[0];
    r.max_residual = out[1];
    r.per_mode_residuals.assign(out.begin() + 2, out.end());
    return r;
}

double scf_stopping_value(const SymBlockMatrix& j, const StackedVector& x, double lambda) {
    if (x.total_dim() != j.total_dim())
        throw std::invalid_argument("scf_stopping_value: dimension mismatch");
    const auto dims = u64(j.block_dims());
    const auto b = blocks_of(j);
    double v = 0.0;
    raise(r1_scf_stopping_value(ctx(), dims.data(), static_cast<int>(j.order()), b.data(),
                                x.flat().data(), lambda, &v));
    return v;
}

// -------------------------------------------------------------- eigen steps --
EigPair largest_magnitude_eigenpair(const Matrix& s) {
    if (s.rows() != s.cols()) throw std::invalid_argument("sym_eig: matrix must be square");
    if (s.rows() == 0) throw std::invalid_argument("largest_magnitude_eigenpair: empty matrix");
    EigPair p;
    p.vector.resize(s.rows());
    raise(r1_largest_magnitude_eigenpair(ctx(), static_cast<int64_t>(s.rows()), s.data(), &p.value,
                                         p.vector.data()));
    return p;
}

std::optional<std::vector<double>> rayleigh_quotient_step(const Matrix& s, std::span<const double> x) {
    if (s.cols() != s.rows() || x.size() != s.rows())
        throw std::invalid_argument("rayleigh_quotient_step: size mismatch");
    std::vector<double> y(x.size());
    int accepted = 0;
    raise(r1_rayleigh_quotient_step(ctx(), static_cast<int64_t>(s.rows()), s.data(), x.data(),
                                    y.data(), &accepted));
    if (!accepted) return std::nullopt;
    return y;
}

// ------------------------------------------------------------------ solvers --
double SolveReport::wall_build_j() const {
    double s = 0.0;
    for (const auto& r : trace) s += r.t_build_j;
    return s;
}
double SolveReport::wall_eig() const {
    double s = 0.0;
    for (const auto& r : trace) s += r.t_eig;
    return s;
}
double SolveReport::wall_total() const {
    double s = 0.0;
    for (const auto& r : trace) s += r.t_build_j + r.t_eig + r.t_other;
    return s;
}

namespace {

// SolveOptions -> r1_solve_options (init factors flattened into `init`).
r1_solve_options c_options(const DenseTensor& a, const SolveOptions& opts, std::vector<double>& init) {
    r1_solve_options o;
    r1_solve_options_default(&o);
    o.tol = opts.tol;
    o.max_iters = opts.max_iters;
    o.seed = opts.seed;
    o.determinism = opts.determinism ? 1 : 0;
    o.rqi_accept_rule = opts.rqi_accept_rule == RqiAcceptRule::signed_increase ? R1_RQI_SIGNED_INCREASE
                                                                               : R1_RQI_MAGNITUDE;
    o.stop_rule = opts.stop_rule == StopRule::eq11 ? R1_STOP_EQ11
                  : opts.stop_rule == StopRule::lambda_delta ? R1_STOP_LAMBDA_DELTA
                                                               : R1_STOP_KKT;
    o.threads = opts.threads;
    o.record_kkt = opts.record_kkt ? 1 : 0;
    o.reuse_intermediates = opts.reuse_intermediates ? 1 : 0;
    o.asvd_disjoint_pairs = opts.asvd_disjoint_pairs ? 1 : 0;
    init.clear();
    if (opts.init == InitKind::provided) {
        if (opts.init_factors.size() != a.order())
            throw std::invalid_argument("solver: provided init has wrong order");
        for (std::size_t k = 0; k < a.order(); ++k) {
            if (opts.init_factors[k].size() != a.dim(k))
                throw std::invalid_argument("solver: provided init factor length mismatch");
            init.insert(init.end(), opts.init_factors[k].begin(), opts.init_factors[k].end());
        }
        o.init = R1_INIT_PROVIDED;
        o.init_factors = init.data();
    }
    return o;
}

// caller-owned arrays of one r1_solve_report
struct ReportBuffers {
    std::vector<double> fac, fx;
    std::vector<r1_iteration_record> tr;
    r1_solve_report r{};
    ReportBuffers(std::size_t n, int max_iters) : fac(n), fx(n), tr(std::max(1, max_iters)) {
        r.factors = fac.data();
        r.final_x = fx.data();
        r.trace = tr.data();
    }
};

SolveReport from_c(const std::string& algorithm, const DenseTensor& a, const ReportBuffers& b) {
    const r1_solve_report& r = b.r;
    SolveReport rep;
    rep.algorithm = algorithm;
    rep.result.lambda = r.lambda;
    std::size_t off = 0;
    for (std::size_t k = 0; k < a.order(); ++k) {
        rep.result.factors.emplace_back(b.fac.begin() + off, b.fac.begin() + off + a.dim(k));
        off += a.dim(k);
    }
    rep.converged = r.converged != 0;
    rep.iterations = r.iterations;
    rep.lambda0 = r.lambda0;
    rep.restarted = r.restarted != 0;
    // SCF solvers: last stacked eigenvector; baselines leave it empty (solvers.hpp:56)
    if (algorithm == "hoscf" || algorithm == "ihoscf") rep.final_x = StackedVector(a.dims(), b.fx);
    for (int i = 0; i < r.iterations; ++i) {
        IterationRecord q;
        q.lambda = b.tr[i].lambda;
        q.stop_value = b.tr[i].stop_value;
        q.eq11_value = b.tr[i].eq11_value;
        q.kkt_max_residual = b.tr[i].kkt_max_residual;
        q.rqi_accepted = b.tr[i].rqi_accepted != 0;
        q.lambda_pre_rqi = b.tr[i].lambda_pre_rqi;
        q.t_build_j = b.tr[i].t_build_j;
        q.t_eig = b.tr[i].t_eig;
        q.t_other = b.tr[i].t_other;
        rep.trace.push_back(q);
    }
    return rep;
}

struct TensorGuard {
    r1_tensor* t = nullptr;
    ~TensorGuard() {
        if (t) r1_tensor_destroy(t);
    }
};

}  // namespace

SolveReport solve(const std::string& algorithm, const DenseTensor& a, const SolveOptions& opts) {
    if (algorithm != "hoscf" && algorithm != "ihoscf" && algorithm != "hopm" &&
        algorithm != "jacobi_hopm" && algorithm != "asvd" && algorithm != "jacobi_asvd")
        throw std::invalid_argument("unknown solver: " + algorithm);
    if (a.order() < 2) throw std::invalid_argument("solver: tensor order must be >= 2");
    std::vector<double> init;
    r1_solve_options o = c_options(a, opts, init);
    const auto dims = u64(a.dims());
    TensorGuard t;
    raise(r1_tensor_from_host(ctx(), a.data(), dims.data(), static_cast<int>(a.order()), &t.t));
    const std::size_t n = std::accumulate(a.dims().begin(), a.dims().end(), std::size_t{0});
    ReportBuffers b(n, opts.max_iters);
    raise(r1_solve(ctx(), algorithm.c_str(), t.t, &o, &b.r));
    return from_c(algorithm, a, b);
}

// greedy.hpp:21-22 on the device (residual resident in HBM).
GreedyReport greedy_rank_r(const DenseTensor& a, std::size_t r, const std::string& solver,
                           const SolveOptions& opts) {
    if (r < 1) throw std::invalid_argument("greedy_rank_r: rank must be >= 1");
    std::vector<double> init;
    r1_solve_options o = c_options(a, opts, init);
    const auto dims = u64(a.dims());
    TensorGuard t;
    raise(r1_tensor_from_host(ctx(), a.data(), dims.data(), static_cast<int>(a.order()), &t.t));
    const std::size_t n = std::accumulate(a.dims().begin(), a.dims().end(), std::size_t{0});
    std::vector<double> lam(r), fac(r * n), rat(r);
    std::vector<std::unique_ptr<ReportBuffers>> bufs;
    std::vector<r1_solve_report> reps(r);
    for (std::size_t i = 0; i < r; ++i) {
        bufs.push_back(std::make_unique<ReportBuffers>(n, opts.max_iters));
        reps[i] = bufs.back()->r;
    }
    r1_greedy_report g{};
    g.lambdas = lam.data();
    g.factors = fac.data();
    g.residual_ratios = rat.data();
    g.solves = reps.data();
    raise(r1_greedy_rank_r(ctx(), t.t, r, solver.c_str(), &o, &g));
    GreedyReport rep;
    for (int i = 0; i < g.terms; ++i) {
        bufs[i]->r = reps[i];
        SolveReport s = from_c(solver, a, *bufs[i]);
        rep.terms.push_back(s.result);
        rep.residual_ratios.push_back(rat[i]);
        rep.solves.push_back(std::move(s));
    }
    rep.completed = g.completed != 0;
    rep.failure = g.failure;
    return rep;
}

// tensor_io.hpp:16-20: the file is staged through the device loader, so the
// host API and r1_tensor_read_dt1 share one validation path.
DenseTensor read_dt1(const std::string& path) {
    TensorGuard t;
    raise(r1_tensor_read_dt1(ctx(), path.c_str(), &t.t));
    // dims from the validated header
    std::vector<std::size_t> dims;
    {
        std::FILE* f = std::fopen(path.c_str(), "rb");
        if (!f) throw std::runtime_error("read_dt1: cannot open " + path);
        unsigned char hdr[7];
        if (std::fread(hdr, 1, 7, f) != 7) {
            std::fclose(f);
            throw std::runtime_error("read_dt1: bad magic in " + path);
        }
        for (int k = 0; k < hdr[6]; ++k) {
            unsigned char b[8];
            if (std::fread(b, 1, 8, f) != 8) break;
            uint64_t v = 0;
            for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(b[i]) << (8 * i);
            dims.push_back(static_cast<std::size_t>(v));
        }
        std::fclose(f);
    }
    DenseTensor out(dims);
    raise(r1_tensor_copy_to_host(ctx(), t.t, out.data()));
    return out;
}

void write_dt1(const std::string& path, const DenseTensor& a) {
    if (a.order() < 2) throw std::invalid_argument("write_dt1: tensor order must be >= 2");
    const auto dims = u64(a.dims());
    TensorGuard t;
    raise(r1_tensor_from_host(ctx(), a.data(), dims.data(), static_cast<int>(a.order()), &t.t));
    raise(r1_tensor_write_dt1(ctx(), t.t, path.c_str()));
}

void write_dt1(const std::string& path, const Matrix& m) {
    DenseTensor t({m.rows(), m.cols()}, std::vector<double>(m.values().begin(), m.values().end()));
    write_dt1(path, t);
}

SolveReport hoscf(const DenseTensor& a, const SolveOptions& opts) { return solve("hoscf", a, opts); }
SolveReport ihoscf(const DenseTensor& a, const SolveOptions& opts) { return solve("ihoscf", a, opts); }
SolveReport hopm(const DenseTensor& a, const SolveOptions& opts) { return solve("hopm", a, opts); }
SolveReport jacobi_hopm(const DenseTensor& a, const SolveOptions& opts) {
    return solve("jacobi_hopm", a, opts);
}
SolveReport asvd(const DenseTensor& a, const SolveOptions& opts) { return solve("asvd", a, opts); }
SolveReport jacobi_asvd(const DenseTensor& a, const SolveOptions& opts) {
    return solve("jacobi_asvd", a, opts);
}

const std::vector<std::string>& solver_names() {
    static const std::vector<std::string> names = {"hoscf", "ihoscf", "hopm",
                                                   "jacobi_hopm", "asvd", "jacobi_asvd"};
    return names;
}

}  // namespace rank1
