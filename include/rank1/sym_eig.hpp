// rank1:: drop-in (B200 build) — eigen steps of the solvers.
// API-compatible with proj/include/rank1/sym_eig.hpp:22-38 (the reference's
// dense tred2/QL decomposition sym_eig_full and its LDL^T internals are not on
// the device path and are not declared).  largest_magnitude_eigenpair runs
// device Lanczos (both spectral ends, the reference's pick and sign rules);
// rayleigh_quotient_step runs a device Bunch-Kaufman LDL^T solve with the
// reference's 1e14 diagonal-condition rejection and shift bump.
#pragma once

#include <optional>
#include <span>
#include <vector>

#include "rank1/matrix.hpp"

namespace rank1 {

struct EigPair {
    double value = 0.0;
    std::vector<double> vector;
};

EigPair largest_magnitude_eigenpair(const Matrix& s);
std::optional<std::vector<double>> rayleigh_quotient_step(const Matrix& s,
                                                          std::span<const double> x);

}  // namespace rank1
