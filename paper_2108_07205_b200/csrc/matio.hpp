// Dense matrix interchange (reference nystrom.cpp:450-477).
#pragma once

#include <string>

#include "common.hpp"

namespace sbx {

// Column-major host matrix (ld) -> file in the reference's dump format.
void dump_matrix(const std::string& path, const double* m, i64 rows, i64 cols, i64 ld);
// File -> column-major host matrix.
HMat load_matrix(const std::string& path);

}  // namespace sbx
