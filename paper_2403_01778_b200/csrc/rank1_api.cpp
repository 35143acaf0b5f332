// The C++ rank1:: drop-in (include/rank1/*.hpp) on top of the C-ABI
// (include/rank1_b200.h).  Container types are host-side as in the reference
// (they own std::vector storage); every computation over a tensor or a block
// matrix — sweep, SymBlockMatrix matvec / dense / norm, eigen steps, RQI,
// LDL^T, stopping test, KKT, contractions, unfoldings, expansions, solvers,
// generators — goes through r1_* into the sm_100a kernels.  What stays on the
// host is O(sum I_k) container glue over the caller's vectors (Matrix / span
// helpers of matrix.hpp, StackedVector split / stack / flip of stacked.hpp,
// the CounterRng draws of rng.hpp), kept as API shims with the reference's
// semantics and messages.  Status codes are mapped back to the reference's
// exception types (invalid_argument / runtime_error).
#include <algorithm>
#include <cmath>
#include <functional>
#include <numbers>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>

#include "rank1/generators.hpp"
#include "rank1/greedy.hpp"
#include "rank1/nepv.hpp"
#include "rank1/rng.hpp"
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

struct TensorGuard {
    r1_tensor* t = nullptr;
    ~TensorGuard() {
        if (t) r1_tensor_destroy(t);
    }
};


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
// matrix.hpp container helpers (reference matrix.cpp:6-67): host glue over the
// caller's vectors, sequential sums in index order as the reference's.
Matrix transpose(const Matrix& m) {
    Matrix t(m.cols(), m.rows());
    for (std::size_t j = 0; j < m.cols(); ++j) {
        const auto c = m.col(j);
        for (std::size_t i = 0; i < c.size(); ++i) t(j, i) = c[i];
    }
    return t;
}

std::vector<double> matvec(const Matrix& m, std::span<const double> x) {
    if (x.size() != m.cols()) throw std::invalid_argument("matvec: size mismatch");
    std::vector<double> y(m.rows(), 0.0);
    for (std::size_t j = 0; j < m.cols(); ++j) {
        const auto c = m.col(j);
        const double xj = x[j];
        std::transform(y.begin(), y.end(), c.begin(), y.begin(),
                       [xj](double acc, double a) { return acc + a * xj; });
    }
    return y;
}

std::vector<double> matvec_transposed(const Matrix& m, std::span<const double> x) {
    if (x.size() != m.rows()) throw std::invalid_argument("matvec_transposed: size mismatch");
    std::vector<double> y(m.cols());
    for (std::size_t j = 0; j < m.cols(); ++j) {
        const auto c = m.col(j);
        y[j] = std::inner_product(c.begin(), c.end(), x.begin(), 0.0);
    }
    return y;
}

double frobenius_norm(const Matrix& m) { return norm2(m.values()); }

double max_abs(const Matrix& m) {
    return std::accumulate(m.values().begin(), m.values().end(), 0.0,
                           [](double acc, double v) { return std::max(acc, std::abs(v)); });
}

double dot(std::span<const double> a, std::span<const double> b) {
    if (a.size() != b.size()) throw std::invalid_argument("dot: size mismatch");
    return std::inner_product(a.begin(), a.end(), b.begin(), 0.0);
}

double norm2(std::span<const double> v) {
    return std::sqrt(std::inner_product(v.begin(), v.end(), v.begin(), 0.0));
}

double normalize(std::span<double> v) {
    const double len = norm2(v);
    if (len > 0.0) std::transform(v.begin(), v.end(), v.begin(), [len](double x) { return x / len; });
    return len;
}

// ------------------------------------------------------------------- rng.hpp --
// Box-Muller in pairs (reference generators.cpp:11-24): u1 nudged by 2^-54 so
// the log stays finite; the sine half is returned by the next call.
double CounterRng::next_gaussian() {
    if (has_cached_) {
        has_cached_ = false;
        return cached_;
    }
    const double u1 = next_unit() + 0x1.0p-54;
    const double u2 = next_unit();
    const double rad = std::sqrt(-2.0 * std::log(u1));
    const double ang = 2.0 * std::numbers::pi * u2;
    cached_ = rad * std::sin(ang);
    has_cached_ = true;
    return rad * std::cos(ang);
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
    const auto dims = u64(a.dims());
    double v = 0.0;
    raise(r1_host_frobenius(ctx(), a.data(), dims.data(), static_cast<int>(a.order()), &v));
    return v;
}

// ---------------------------------------------------------- ttv / ttvc chains --
namespace {

void check_ttvc_args(const DenseTensor& a, std::span<const std::vector<double>> vs,
                     std::span<const std::size_t> modes) {
    if (vs.size() != modes.size()) throw std::invalid_argument("ttvc: vectors/modes mismatch");
    std::vector<bool> seen(a.order(), false);
    for (std::size_t i = 0; i < modes.size(); ++i) {
        if (modes[i] >= a.order()) throw std::invalid_argument("ttvc: mode out of range");
        if (seen[modes[i]]) throw std::invalid_argument("ttvc: duplicate mode");
        seen[modes[i]] = true;
        if (vs[i].size() != a.dim(modes[i])) throw std::invalid_argument("ttvc: vector length mismatch");
    }
}

// the device chain (r1_ttvc); full = all modes -> scalar
DenseTensor ttvc_device(const DenseTensor& a, std::span<const std::vector<double>> vs,
                        std::span<const std::size_t> modes, bool full, double* scalar) {
    std::vector<double> flatv;
    std::vector<int> m;
    for (std::size_t i = 0; i < modes.size(); ++i) {
        flatv.insert(flatv.end(), vs[i].begin(), vs[i].end());
        m.push_back(static_cast<int>(modes[i]));
    }
    std::vector<std::size_t> out_dims;
    std::vector<bool> gone(a.order(), false);
    for (auto k : modes) gone[k] = true;
    for (std::size_t k = 0; k < a.order(); ++k)
        if (!gone[k]) out_dims.push_back(a.dim(k));
    const auto dims = u64(a.dims());
    DenseTensor out = full ? DenseTensor() : DenseTensor(out_dims);
    raise(r1_ttvc(ctx(), a.data(), dims.data(), static_cast<int>(a.order()), flatv.data(), m.data(),
                  static_cast<int>(m.size()), full ? 1 : 0, full ? nullptr : out.data(), scalar));
    return out;
}

}  // namespace

DenseTensor ttv(const DenseTensor& a, std::span<const double> v, std::size_t mode, bool) {
    if (mode >= a.order()) throw std::invalid_argument("ttv: mode out of range");
    if (v.size() != a.dim(mode)) throw std::invalid_argument("ttv: vector length mismatch");
    if (a.order() == 1) throw std::invalid_argument("ttv: full contraction needs ttvc_scalar");
    const std::vector<double> vv(v.begin(), v.end());
    const std::size_t md[1] = {mode};
    return ttvc_device(a, std::span<const std::vector<double>>(&vv, 1), md, false, nullptr);
}

DenseTensor ttvc(const DenseTensor& a, std::span<const std::vector<double>> vs,
                 std::span<const std::size_t> modes, bool) {
    check_ttvc_args(a, vs, modes);
    if (modes.size() >= a.order())
        throw std::invalid_argument("ttvc: contracting all modes yields a scalar, use ttvc_scalar");
    if (modes.empty()) return a;
    return ttvc_device(a, vs, modes, false, nullptr);
}

double ttvc_scalar(const DenseTensor& a, std::span<const std::vector<double>> vs,
                   std::span<const std::size_t> modes, bool) {
    check_ttvc_args(a, vs, modes);
    if (modes.size() != a.order()) throw std::invalid_argument("ttvc_scalar: all modes must be contracted");
    double v = 0.0;
    ttvc_device(a, vs, modes, true, &v);
    return v;
}

double multilinear_value(const DenseTensor& a, const FactorSet& f, bool parallel) {
    if (f.order() != a.order()) throw std::invalid_argument("multilinear_value: order mismatch");
    std::vector<std::size_t> modes(a.order());
    std::iota(modes.begin(), modes.end(), std::size_t{0});
    return ttvc_scalar(a, f.factors, modes, parallel);
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

// stacked.hpp container glue (reference stacked.cpp:36-85): O(sum I_k) on the
// caller's vectors.
SplitResult split_factors(const StackedVector& x) {
    SplitResult r;
    r.factors.factors.reserve(x.order());
    r.degenerate.reserve(x.order());
    for (std::size_t n = 0; n < x.order(); ++n) {
        const auto blk = x.block(n);
        std::vector<double> u(blk.begin(), blk.end());
        const double len = norm2(u);
        const bool deg = len < 1e-12;  // flagged, not thrown (stacked.cpp:47-50)
        if (deg)
            std::fill(u.begin(), u.end(), 0.0);
        else
            std::transform(u.begin(), u.end(), u.begin(), [len](double v) { return v / len; });
        r.factors.factors.push_back(std::move(u));
        r.degenerate.push_back(deg ? 1 : 0);
    }
    return r;
}

StackedVector stack_factors(const FactorSet& f) {
    if (f.order() == 0) throw std::invalid_argument("stack_factors: empty factor set");
    if (max_unit_deviation(f) > 1e-8)
        throw std::invalid_argument("stack_factors: factors must have unit norm");
    std::vector<std::size_t> dims;
    std::vector<double> flat;
    const double w = 1.0 / std::sqrt(static_cast<double>(f.order()));
    for (const auto& u : f.factors) {
        dims.push_back(u.size());
        std::transform(u.begin(), u.end(), std::back_inserter(flat), [w](double v) { return v * w; });
    }
    return StackedVector(std::move(dims), std::move(flat));
}

StackedVector flip_first_block(const StackedVector& x) {
    StackedVector y = x;
    auto b = y.block(0);
    std::transform(b.begin(), b.end(), b.begin(), std::negate<double>());
    return y;
}

FactorSet flip_first_factor(FactorSet f) {
    if (f.order() == 0) throw std::invalid_argument("flip_first_factor: empty factor set");
    std::transform(f.factors[0].begin(), f.factors[0].end(), f.factors[0].begin(),
                   std::negate<double>());
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

// The operator on the device (nepv.cpp:110-157): the blocks are staged and
// r1_block_matvec / r1_block_dense / r1_block_frobenius run the kernels the
// solvers use.
std::vector<double> SymBlockMatrix::matvec(std::span<const double> x) const {
    if (x.size() != total_dim()) throw std::invalid_argument("SymBlockMatrix: matvec size mismatch");
    const auto dims = u64(dims_);
    const auto b = blocks_of(*this);
    std::vector<double> y(x.size());
    raise(r1_block_matvec(ctx(), dims.data(), static_cast<int>(order()), b.data(), x.data(), y.data()));
    return y;
}

Matrix SymBlockMatrix::dense() const {
    const auto dims = u64(dims_);
    const auto b = blocks_of(*this);
    Matrix s(total_dim(), total_dim());
    raise(r1_block_dense(ctx(), dims.data(), static_cast<int>(order()), b.data(), s.data()));
    return s;
}

double SymBlockMatrix::frobenius_norm() const {
    const auto dims = u64(dims_);
    const auto b = blocks_of(*this);
    double v = 0.0;
    raise(r1_block_frobenius(ctx(), dims.data(), static_cast<int>(order()), b.data(), &v));
    return v;
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

// sym_eig.hpp:19 / :49-52 on the device (csrc/dense_api.cu).
EigDecomposition sym_eig_full(const Matrix& s) {
    if (s.rows() != s.cols()) throw std::invalid_argument("sym_eig: matrix must be square");
    const std::size_t n = s.rows();
    EigDecomposition d;
    d.values.assign(n, 0.0);
    if (n == 0) return d;
    d.vectors = Matrix(n, n);
    raise(r1_sym_eig_full(ctx(), static_cast<int64_t>(n), s.data(), d.values.data(),
                          d.vectors.data()));
    return d;
}

namespace detail {

LdltFactors ldlt_factor(Matrix s) {
    const std::size_t n = s.rows();
    if (s.cols() != n) throw std::invalid_argument("ldlt_factor: matrix must be square");
    LdltFactors f{Matrix(n, n), std::vector<int>(n, 0), false};
    int sing = 0;
    raise(r1_ldlt_factor(ctx(), static_cast<int64_t>(n), s.data(), f.w.data(), f.ipiv.data(), &sing));
    f.singular = sing != 0;
    return f;
}

std::vector<double> ldlt_solve(const LdltFactors& f, std::vector<double> b) {
    const std::size_t n = f.w.rows();
    if (b.size() != n) throw std::invalid_argument("ldlt_solve: size mismatch");
    std::vector<double> x(n);
    raise(r1_ldlt_solve(ctx(), static_cast<int64_t>(n), f.w.data(), f.ipiv.data(), b.data(), x.data()));
    return x;
}

double ldlt_diag_condition(const LdltFactors& f) {
    const std::size_t n = f.w.rows();
    std::vector<double> diag(n), sub(n, 0.0);
    for (std::size_t k = 0; k < n; ++k) {
        diag[k] = f.w(k, k);
        if (k + 1 < n) sub[k] = f.w(k + 1, k);
    }
    double c = 0.0;
    raise(r1_ldlt_diag_condition(ctx(), static_cast<int64_t>(n), diag.data(), sub.data(),
                                 f.ipiv.data(), f.singular ? 1 : 0, &c));
    return c;
}

}  // namespace detail

// ---------------------------------------------------------- tensor.hpp extras --
std::vector<std::vector<double>> contract_leaving_all(const DenseTensor& a, const FactorSet& f, bool) {
    if (f.order() != a.order()) throw std::invalid_argument("contract_leaving_all: order mismatch");
    check_shapes(a, f);
    const auto dims = u64(a.dims());
    const auto fl = flat(f);
    std::vector<double> w(fl.size());
    raise(r1_contract_leaving_all(ctx(), a.data(), nullptr, dims.data(), static_cast<int>(a.order()),
                                  fl.data(), w.data()));
    std::vector<std::vector<double>> out;
    std::size_t off = 0;
    for (std::size_t k = 0; k < a.order(); ++k) {
        out.emplace_back(w.begin() + off, w.begin() + off + a.dim(k));
        off += a.dim(k);
    }
    return out;
}

std::vector<double> contract_leaving(const DenseTensor& a, const FactorSet& f, std::size_t mode,
                                     bool parallel) {
    if (f.order() != a.order()) throw std::invalid_argument("contract_leaving: order mismatch");
    if (mode >= a.order()) throw std::invalid_argument("contract_leaving: mode out of range");
    return contract_leaving_all(a, f, parallel)[mode];
}

Matrix matricize(const DenseTensor& a, std::size_t mode) {
    if (mode >= a.order()) throw std::invalid_argument("matricize: mode out of range");
    const auto dims = u64(a.dims());
    Matrix m(a.dim(mode), a.size() / a.dim(mode));
    raise(r1_matricize(ctx(), a.data(), dims.data(), static_cast<int>(a.order()),
                       static_cast<int>(mode), 0, m.data()));
    return m;
}

DenseTensor dematricize(const Matrix& m, std::size_t mode, std::vector<std::size_t> dims) {
    if (mode >= dims.size()) throw std::invalid_argument("dematricize: mode out of range");
    std::size_t rest = 1;
    for (std::size_t k = 0; k < dims.size(); ++k)
        if (k != mode) rest *= dims[k];
    if (m.rows() != dims[mode] || m.cols() != rest)
        throw std::invalid_argument("dematricize: matrix shape does not match dims");
    DenseTensor a(dims);
    const auto d = u64(dims);
    raise(r1_matricize(ctx(), m.data(), d.data(), static_cast<int>(dims.size()), static_cast<int>(mode),
                       1, a.data()));
    return a;
}

DenseTensor rank_one_expand(const FactorSet& f, std::span<const std::size_t> dims) {
    if (f.order() != dims.size()) throw std::invalid_argument("rank_one_expand: order mismatch");
    for (std::size_t n = 0; n < dims.size(); ++n)
        if (f.factors[n].size() != dims[n])
            throw std::invalid_argument("rank_one_expand: factor length mismatch");
    DenseTensor out(std::vector<std::size_t>(dims.begin(), dims.end()));
    const auto d = u64(out.dims());
    const auto fl = flat(f);
    raise(r1_rank_one_expand(ctx(), f.lambda, fl.data(), d.data(), static_cast<int>(dims.size()),
                             out.data()));
    return out;
}

double residual_norm(const DenseTensor& a, const FactorSet& f, std::size_t dense_threshold) {
    if (f.order() != a.order()) throw std::invalid_argument("residual_norm: order mismatch");
    for (std::size_t n = 0; n < a.order(); ++n)
        if (f.factors[n].size() != a.dim(n))
            throw std::invalid_argument("residual_norm: factor length mismatch");
    const auto d = u64(a.dims());
    const auto fl = flat(f);
    double v = 0.0;
    raise(r1_residual_norm(ctx(), a.data(), d.data(), static_cast<int>(a.order()), f.lambda, fl.data(),
                           dense_threshold, &v));
    return v;
}

// ------------------------------------------------------------ generators.hpp --
// Generated on the device (r1_generate, one counter per element) into a
// device tensor and copied back (generators.cpp:50-116).
std::vector<std::size_t> default_dims(const std::string& name) {
    if (name == "gaussian") return {10, 10, 10};
    if (name == "exp") return {30, 30, 30};
    if (name == "arcsin") return {20, 20, 20, 20};
    if (name == "tan") return {10, 10, 10, 10, 10};
    throw std::invalid_argument("unknown generator: " + name);
}

namespace {
DenseTensor generate_on_device(const std::string& name, const std::vector<std::size_t>& dims,
                               std::uint64_t seed) {
    if (dims.size() < 2) throw std::invalid_argument("generator: tensor order must be >= 2");
    const auto d = u64(dims);
    TensorGuard t;
    raise(r1_tensor_create(ctx(), d.data(), static_cast<int>(dims.size()), &t.t));
    raise(r1_generate(ctx(), t.t, name.c_str(), seed));
    DenseTensor out(dims);
    raise(r1_tensor_copy_to_host(ctx(), t.t, out.data()));
    return out;
}
}  // namespace

DenseTensor gen_gaussian(const std::vector<std::size_t>& dims, std::uint64_t seed) {
    return generate_on_device("gaussian", dims, seed);
}
DenseTensor gen_exp(const std::vector<std::size_t>& dims) { return generate_on_device("exp", dims, 0); }
DenseTensor gen_arcsin(const std::vector<std::size_t>& dims) {
    return generate_on_device("arcsin", dims, 0);
}
DenseTensor gen_tan(const std::vector<std::size_t>& dims) { return generate_on_device("tan", dims, 0); }

DenseTensor generate(const std::string& name, std::vector<std::size_t> dims, std::uint64_t seed) {
    if (dims.empty()) dims = default_dims(name);
    if (name != "gaussian" && name != "exp" && name != "arcsin" && name != "tan")
        throw std::invalid_argument("unknown generator: " + name);
    return generate_on_device(name, dims, seed);
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


}  // namespace

namespace {

// Several GPUs of the node for the SCF solvers (opt-in: R1_NUM_GPUS = N):
// one context per device, one NCCL communicator set (r1_comm_init_all), the
// tensor split into slabs along its last mode and one host thread per GPU
// running the sharded solver (SURVEY §8b threading: "one thread per GPU").
struct MultiGpu {
    std::vector<r1_context*> ctxs;
    std::vector<r1_comm*> comms;
};

MultiGpu* multi_gpu() {
    static std::once_flag once;
    static MultiGpu* m = nullptr;
    std::call_once(once, [] {
        const char* env = std::getenv("R1_NUM_GPUS");
        if (!env) return;  // default: the process context on device 0
        const int want = std::atoi(env);
        int have = 0;
        if (want < 1 || r1_device_count(&have) != R1_OK || have < 1) return;
        const int ndev = std::min(want, have);  // 1 is allowed: the sharded path on one GPU
        auto* mg = new MultiGpu();
        std::vector<int> devs(ndev);
        for (int i = 0; i < ndev; ++i) {
            devs[i] = i;
            r1_context* c = nullptr;
            raise(r1_context_create(i, &c));
            mg->ctxs.push_back(c);
        }
        mg->comms.resize(ndev);
        raise(r1_comm_init_all(ndev, devs.data(), mg->ctxs.data(), mg->comms.data()));
        m = mg;
    });
    return m;
}

}  // namespace

SolveReport solve(const std::string& algorithm, const DenseTensor& a, const SolveOptions& opts) {
    if (algorithm != "hoscf" && algorithm != "ihoscf" && algorithm != "hopm" &&
        algorithm != "jacobi_hopm" && algorithm != "asvd" && algorithm != "jacobi_asvd")
        throw std::invalid_argument("unknown solver: " + algorithm);
    if (a.order() < 2) throw std::invalid_argument("solver: tensor order must be >= 2");
    std::vector<double> init;
    r1_solve_options o = c_options(a, opts, init);
    const auto dims = u64(a.dims());
    const std::size_t n = std::accumulate(a.dims().begin(), a.dims().end(), std::size_t{0});
    const int d = static_cast<int>(a.order());
    MultiGpu* mg = (algorithm == "hoscf" || algorithm == "ihoscf") ? multi_gpu() : nullptr;
    if (mg && dims[d - 1] >= mg->ctxs.size()) {
        // slabs of the last (slowest) mode are contiguous runs of the host array
        const int W = static_cast<int>(mg->ctxs.size());
        uint64_t prefix = 1;
        for (int k = 0; k + 1 < d; ++k) prefix *= dims[k];
        std::vector<std::unique_ptr<ReportBuffers>> bufs;
        for (int r = 0; r < W; ++r) bufs.push_back(std::make_unique<ReportBuffers>(n, opts.max_iters));
        std::vector<int> rcs(W, R1_OK);
        std::vector<std::string> msgs(W);
        auto rank_fn = [&](int r) {
            uint64_t lo = 0, hi = 0;
            r1_slab_bounds(dims[d - 1], W, r, &lo, &hi);
            std::vector<uint64_t> ld(dims);
            ld[d - 1] = hi - lo;
            r1_tensor* slab = nullptr;
            int rc = r1_tensor_from_host(mg->ctxs[r], a.data() + prefix * lo, ld.data(), d, &slab);
            if (rc == R1_OK)
                rc = r1_solve_sharded(mg->ctxs[r], algorithm.c_str(), slab, dims.data(), d, &o,
                                      &bufs[r]->r);
            if (rc != R1_OK) msgs[r] = r1_last_error();  // thread-local message
            if (slab) r1_tensor_destroy(slab);
            rcs[r] = rc;
        };
        std::vector<std::thread> th;
        for (int r = 1; r < W; ++r) th.emplace_back(rank_fn, r);
        rank_fn(0);
        for (auto& t : th) t.join();
        for (int r = 0; r < W; ++r)
            if (rcs[r] != R1_OK) {
                if (rcs[r] == R1_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msgs[r]);
                throw std::runtime_error(msgs[r]);
            }
        return from_c(algorithm, a, *bufs[0]);
    }
    ReportBuffers b(n, opts.max_iters);
    raise(r1_solve_host(ctx(), algorithm.c_str(), a.data(), dims.data(), static_cast<int>(a.order()),
                        &o, &b.r));
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
