// rank1:: drop-in (B200 build) — .dt1 tensor files.
// API-compatible with proj/include/rank1/tensor_io.hpp:9-21 (format: magic
// "DTEN1\0", u8 order d >= 2, d little-endian u64 dims, prod(dims)
// little-endian f64 values, first index fastest).  Files stream through the
// device loader (r1_tensor_read_dt1 / r1_tensor_write_dt1): same validation
// and messages as the reference.
#pragma once

#include <string>

#include "rank1/matrix.hpp"
#include "rank1/tensor.hpp"

namespace rank1 {

void write_dt1(const std::string& path, const DenseTensor& a);
DenseTensor read_dt1(const std::string& path);
void write_dt1(const std::string& path, const Matrix& m);

}  // namespace rank1
