// rank1:: drop-in (B200 build) — symmetric eigen steps.
// API-compatible with proj/include/rank1/sym_eig.hpp:11-54 (same types,
// fields and signatures).  Everything runs on the device:
//  * sym_eig_full and largest_magnitude_eigenpair(Matrix): the reference's
//    Householder + implicit-QL decomposition restated in one thread block
//    (csrc/dense_api.cu), with its pick / sign rules;
//  * rayleigh_quotient_step: the blocked Bunch-Kaufman LDL^T of csrc/bk.cu
//    (cluster panel + FP64 tensor-core update) with the 1e14 diagonal-
//    condition rejection and the one shift bump;
//  * detail::ldlt_*: the unblocked Bunch-Kaufman in the reference's storage.
// The solvers themselves use Lanczos on the block operator (csrc/lanczos.cu).
#pragma once

#include <optional>
#include <span>
#include <vector>

#include "rank1/matrix.hpp"

namespace rank1 {

struct EigDecomposition {
    std::vector<double> values;  // ascending
    Matrix vectors;              // column j pairs with values[j]; orthonormal
};

/// Throws std::invalid_argument on non-symmetric input (beyond 1e-10
/// relative) and std::runtime_error when QL does not converge.
EigDecomposition sym_eig_full(const Matrix& s);

struct EigPair {
    double value = 0.0;
    std::vector<double> vector;
};

EigPair largest_magnitude_eigenpair(const Matrix& s);
std::optional<std::vector<double>> rayleigh_quotient_step(const Matrix& s,
                                                          std::span<const double> x);

namespace detail {

struct LdltFactors {
    Matrix w;               // L below the diagonal, D in the pivot blocks
    std::vector<int> ipiv;  // >= 0: 1x1 pivot row swap; < 0: 2x2 block, kp = -ipiv-1
    bool singular = false;  // an exactly zero pivot column was met
};

LdltFactors ldlt_factor(Matrix s);
std::vector<double> ldlt_solve(const LdltFactors& f, std::vector<double> b);
double ldlt_diag_condition(const LdltFactors& f);  // inf when singular

}  // namespace detail

}  // namespace rank1
