// Dense device SVD (one-sided Jacobi) for the reference's Eigen::BDCSVD
// calls: truncated_svd (idlib.cpp:134-154), dense_cond / factor_cond
// (els.cpp:205-222).  Diagnostic paths: O(min(m,n)^2 max(m,n)) per sweep.
#pragma once

#include <vector>

#include "common.hpp"

namespace sbx {

// Singular values (descending) of the m x n device matrix A (column-major, lda).
std::vector<double> singular_values_device(const double* A, i64 m, i64 n, i64 lda, cudaStream_t s);

// idlib.cpp:134-154: k = #{ s_i > eps s_0 }; U (m x k), V (n x k)
// column-major on the device, sv (k) descending on the host.
struct TruncSvd {
  i64 m = 0, n = 0, k = 0;
  DevBuf<double> U, V;
  std::vector<double> sv;
};
TruncSvd truncated_svd_device(const double* A, i64 m, i64 n, i64 lda, double eps, cudaStream_t s);

}  // namespace sbx

namespace sbx {
// R (k x n, ld ldr) = diag(sv) V^T of a truncated SVD.
void svd_sv_vt(const TruncSvd& t, double* R, i64 ldr, cudaStream_t s);
}  // namespace sbx
