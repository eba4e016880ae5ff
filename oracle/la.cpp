// ORACLE — TEST INFRASTRUCTURE ONLY (see orc.hpp).
// Small dense linear algebra standing in for the Eigen3 routines the
// reference calls (Eigen is absent from this image).
#include <algorithm>
#include <cstring>
#include <limits>

#include "orc.hpp"

namespace orc {

Mat Mat::transpose() const {
  Mat t(c, r);
  for (Index j = 0; j < c; ++j)
    for (Index i = 0; i < r; ++i) t(j, i) = (*this)(i, j);
  return t;
}

Mat Mat::rows_of(const std::vector<Index>& rows) const {
  Mat s(Index(rows.size()), c);
  for (Index j = 0; j < c; ++j)
    for (size_t i = 0; i < rows.size(); ++i) s(Index(i), j) = (*this)(rows[i], j);
  return s;
}

Mat Mat::block(Index i0, Index j0, Index nr, Index nc) const {
  Mat b(nr, nc);
  for (Index j = 0; j < nc; ++j)
    for (Index i = 0; i < nr; ++i) b(i, j) = (*this)(i0 + i, j0 + j);
  return b;
}

void Mat::set_block(Index i0, Index j0, const Mat& b) {
  for (Index j = 0; j < b.c; ++j)
    for (Index i = 0; i < b.r; ++i) (*this)(i0 + i, j0 + j) = b(i, j);
}

double Mat::norm() const {
  double s = 0;
  for (double v : a) s += v * v;
  return std::sqrt(s);
}

Mat matmul(const Mat& a, const Mat& b) {
  require(a.c == b.r, "matmul: shape mismatch");
  Mat out(a.r, b.c);
  for (Index j = 0; j < b.c; ++j) {
    double* oc = out.col(j);
    for (Index p = 0; p < a.c; ++p) {
      const double bp = b(p, j);
      if (bp == 0.0) continue;
      const double* ac = a.col(p);
      for (Index i = 0; i < a.r; ++i) oc[i] += ac[i] * bp;
    }
  }
  return out;
}

Mat matmul_tn(const Mat& a, const Mat& b) {
  require(a.r == b.r, "matmul_tn: shape mismatch");
  Mat out(a.c, b.c);
  for (Index j = 0; j < b.c; ++j)
    for (Index i = 0; i < a.c; ++i) {
      const double* ac = a.col(i);
      const double* bc = b.col(j);
      double s = 0;
      for (Index p = 0; p < a.r; ++p) s += ac[p] * bc[p];
      out(i, j) = s;
    }
  return out;
}

Mat hcat(const Mat& a, const Mat& b) {
  require(a.r == b.r || a.c == 0 || b.c == 0, "hcat: rows mismatch");
  const Index r = a.c ? a.r : b.r;
  Mat o(r, a.c + b.c);
  std::copy(a.a.begin(), a.a.end(), o.a.begin());
  std::copy(b.a.begin(), b.a.end(), o.a.begin() + a.size());
  return o;
}

Mat vcat(const Mat& a, const Mat& b) {
  const Index c = a.r ? a.c : b.c;
  Mat o(a.r + b.r, c);
  for (Index j = 0; j < c; ++j) {
    for (Index i = 0; i < a.r; ++i) o(i, j) = a(i, j);
    for (Index i = 0; i < b.r; ++i) o(a.r + i, j) = b(i, j);
  }
  return o;
}

Mat sub(const Mat& a, const Mat& b) {
  Mat o = a;
  for (size_t i = 0; i < o.a.size(); ++i) o.a[i] -= b.a[i];
  return o;
}

namespace {

double sq_norm(const double* v, Index n) {
  double s = 0;
  for (Index i = 0; i < n; ++i) s += v[i] * v[i];
  return s;
}

// Eigen MatrixBase::makeHouseholderInPlace on x[0..n): returns tau, beta;
// x[1..n) becomes the essential part.
void make_householder(double* x, Index n, double& tau, double& beta) {
  const double tail = n > 1 ? sq_norm(x + 1, n - 1) : 0.0;
  const double c0 = x[0];
  const double tol = std::numeric_limits<double>::min();
  if (tail <= tol) {
    tau = 0;
    beta = c0;
    for (Index i = 1; i < n; ++i) x[i] = 0;
  } else {
    beta = std::sqrt(c0 * c0 + tail);
    if (c0 >= 0) beta = -beta;
    const double s = c0 - beta;
    for (Index i = 1; i < n; ++i) x[i] /= s;  // Eigen: tail / (c0 - beta)
    tau = (beta - c0) / beta;
  }
}

// Eigen applyHouseholderOnTheLeft: block rows [k, rows), the reflector
// I - tau [1; ess][1; ess]^T applied to columns cols of `m`.
void apply_householder_left(Mat& m, Index k, const double* ess, double tau, Index c0,
                            Index c1) {
  const Index rows = m.r - k;
  if (rows == 1) {
    for (Index j = c0; j < c1; ++j) m(k, j) *= (1.0 - tau);
    return;
  }
  if (tau == 0.0) return;
  for (Index j = c0; j < c1; ++j) {
    double* col = m.col(j) + k;
    double t = 0;
    for (Index i = 1; i < rows; ++i) t += ess[i - 1] * col[i];
    t += col[0];
    col[0] -= tau * t;
    const double tt = tau * t;
    for (Index i = 1; i < rows; ++i) col[i] -= ess[i - 1] * tt;
  }
}

}  // namespace

CPQR cpqr(const Mat& a) {
  CPQR out;
  out.qr = a;
  Mat& q = out.qr;
  const Index rows = q.r, cols = q.c, size = std::min(rows, cols);
  std::vector<double> upd(static_cast<size_t>(cols)), dir(static_cast<size_t>(cols));
  for (Index k = 0; k < cols; ++k) {
    dir[size_t(k)] = std::sqrt(sq_norm(q.col(k), rows));
    upd[size_t(k)] = dir[size_t(k)];
  }
  const double thr = std::sqrt(std::numeric_limits<double>::epsilon());
  std::vector<Index> transp(static_cast<size_t>(size));
  std::vector<double> ess;
  for (Index k = 0; k < size; ++k) {
    Index big = k;
    double bv = upd[size_t(k)];
    for (Index j = k + 1; j < cols; ++j)
      if (upd[size_t(j)] > bv) {
        bv = upd[size_t(j)];
        big = j;
      }
    transp[size_t(k)] = big;
    if (big != k) {
      std::swap_ranges(q.col(k), q.col(k) + rows, q.col(big));
      std::swap(upd[size_t(k)], upd[size_t(big)]);
      std::swap(dir[size_t(k)], dir[size_t(big)]);
    }
    double tau, beta;
    make_householder(q.col(k) + k, rows - k, tau, beta);
    q(k, k) = beta;
    ess.assign(q.col(k) + k + 1, q.col(k) + rows);
    apply_householder_left(q, k, ess.data(), tau, k + 1, cols);
    for (Index j = k + 1; j < cols; ++j) {
      if (upd[size_t(j)] != 0.0) {
        double t = std::fabs(q(k, j)) / upd[size_t(j)];
        t = (1.0 + t) * (1.0 - t);
        t = t < 0 ? 0 : t;
        const double r = upd[size_t(j)] / dir[size_t(j)];
        const double t2 = t * r * r;
        if (t2 <= thr) {
          dir[size_t(j)] = std::sqrt(sq_norm(q.col(j) + k + 1, rows - k - 1));
          upd[size_t(j)] = dir[size_t(j)];
        } else {
          upd[size_t(j)] *= std::sqrt(t);
        }
      }
    }
  }
  out.perm.resize(size_t(cols));
  for (Index i = 0; i < cols; ++i) out.perm[size_t(i)] = i;
  for (Index k = 0; k < size; ++k) std::swap(out.perm[size_t(k)], out.perm[size_t(transp[size_t(k)])]);
  return out;
}

Mat householder_q_thin(const Mat& a0, Index ncols) {
  Mat a = a0;
  const Index rows = a.r, cols = a.c, size = std::min(rows, cols);
  std::vector<double> taus(static_cast<size_t>(size));
  for (Index k = 0; k < size; ++k) {
    double tau, beta;
    make_householder(a.col(k) + k, rows - k, tau, beta);
    a(k, k) = beta;
    taus[size_t(k)] = tau;
    apply_householder_left(a, k, a.col(k) + k + 1, tau, k + 1, cols);
  }
  Mat q(rows, ncols);
  for (Index i = 0; i < std::min(rows, ncols); ++i) q(i, i) = 1.0;
  for (Index k = size - 1; k >= 0; --k)
    apply_householder_left(q, k, a.col(k) + k + 1, taus[size_t(k)], 0, ncols);
  return q;
}

LU::LU(const Mat& a) : lu(a) {
  require(a.r == a.c, "LU: matrix must be square");
  const Index n = a.r;
  for (Index j = 0; j < n; ++j) {
    double s = 0;
    for (Index i = 0; i < n; ++i) s += std::fabs(a(i, j));
    l1norm = std::max(l1norm, s);
  }
  piv.resize(size_t(n));
  for (Index i = 0; i < n; ++i) piv[size_t(i)] = i;
  for (Index k = 0; k < n; ++k) {
    Index big = k;
    double bv = std::fabs(lu(k, k));
    for (Index i = k + 1; i < n; ++i)
      if (std::fabs(lu(i, k)) > bv) {
        bv = std::fabs(lu(i, k));
        big = i;
      }
    if (bv != 0.0) {
      if (big != k) {
        for (Index j = 0; j < n; ++j) std::swap(lu(k, j), lu(big, j));
        std::swap(piv[size_t(k)], piv[size_t(big)]);
      }
      const double d = lu(k, k);
      for (Index i = k + 1; i < n; ++i) lu(i, k) /= d;
    }
    for (Index j = k + 1; j < n; ++j) {
      const double ukj = lu(k, j);
      if (ukj == 0.0) continue;
      double* cj = lu.col(j);
      const double* ck = lu.col(k);
      for (Index i = k + 1; i < n; ++i) cj[i] -= ck[i] * ukj;
    }
  }
}

Mat LU::solve(const Mat& b) const {
  const Index n = lu.r;
  Mat x(n, b.c);
  for (Index c = 0; c < b.c; ++c) {
    double* xc = x.col(c);
    for (Index i = 0; i < n; ++i) xc[i] = b(piv[size_t(i)], c);
    for (Index j = 0; j < n; ++j) {
      const double v = xc[j];
      if (v == 0.0) continue;
      const double* lj = lu.col(j);
      for (Index i = j + 1; i < n; ++i) xc[i] -= lj[i] * v;
    }
    for (Index j = n - 1; j >= 0; --j) {
      xc[j] /= lu(j, j);
      const double v = xc[j];
      if (v == 0.0) continue;
      const double* uj = lu.col(j);
      for (Index i = 0; i < j; ++i) xc[i] -= uj[i] * v;
    }
  }
  return x;
}

Mat LU::solve_t(const Mat& b) const {
  const Index n = lu.r;
  Mat x(n, b.c);
  std::vector<double> y(static_cast<size_t>(n));
  for (Index c = 0; c < b.c; ++c) {
    for (Index i = 0; i < n; ++i) y[size_t(i)] = b(i, c);
    for (Index i = 0; i < n; ++i) {  // U^T y = b
      double s = y[size_t(i)];
      const double* ui = lu.col(i);
      for (Index p = 0; p < i; ++p) s -= ui[p] * y[size_t(p)];
      y[size_t(i)] = s / lu(i, i);
    }
    for (Index i = n - 1; i >= 0; --i) {  // L^T z = y
      double s = y[size_t(i)];
      const double* li = lu.col(i);
      for (Index p = i + 1; p < n; ++p) s -= li[p] * y[size_t(p)];
      y[size_t(i)] = s;
    }
    for (Index i = 0; i < n; ++i) x(piv[size_t(i)], c) = y[size_t(i)];
  }
  return x;
}

Mat LU::inverse() const { return solve(Mat::identity(lu.r)); }

double LU::rcond() const {
  const Index n = lu.r;
  if (l1norm == 0.0) return 0.0;
  if (n == 1) return 1.0;
  auto l1 = [](const Mat& v) {
    double s = 0;
    for (double x : v.a) s += std::fabs(x);
    return s;
  };
  Mat v(n, 1);
  for (Index i = 0; i < n; ++i) v(i, 0) = 1.0 / double(n);
  v = solve(v);
  double lower = l1(v), old_lower = lower;
  std::vector<double> sign(static_cast<size_t>(n)), old_sign;
  Index vmax = -1, old_vmax = -1;
  for (int k = 0; k < 4; ++k) {
    for (Index i = 0; i < n; ++i) sign[size_t(i)] = v(i, 0) < 0 ? -1.0 : 1.0;
    if (k > 0 && sign == old_sign) break;
    Mat sv(n, 1);
    for (Index i = 0; i < n; ++i) sv(i, 0) = sign[size_t(i)];
    v = solve_t(sv);
    vmax = 0;
    double best = std::fabs(v(0, 0));
    for (Index i = 1; i < n; ++i)
      if (std::fabs(v(i, 0)) > best) {
        best = std::fabs(v(i, 0));
        vmax = i;
      }
    if (vmax == old_vmax) break;
    Mat e(n, 1);
    e(vmax, 0) = 1.0;
    v = solve(e);
    lower = l1(v);
    if (lower <= old_lower) break;
    old_sign = sign;
    old_vmax = vmax;
    old_lower = lower;
  }
  Mat alt(n, 1);
  double s = 1.0;
  for (Index i = 0; i < n; ++i) {
    alt(i, 0) = s * (1.0 + double(i) / double(n - 1));
    s = -s;
  }
  alt = solve(alt);
  const double alt_lower = 2.0 * l1(alt) / (3.0 * double(n));
  const double inv_norm = std::max(lower, alt_lower);
  return inv_norm == 0.0 ? 0.0 : (1.0 / inv_norm) / l1norm;
}

Mat upper_solve(const Mat& u, Index k, const Mat& b) {
  Mat x = b;
  for (Index c = 0; c < x.c; ++c) {
    double* xc = x.col(c);
    for (Index j = k - 1; j >= 0; --j) {
      xc[j] /= u(j, j);
      const double v = xc[j];
      for (Index i = 0; i < j; ++i) xc[i] -= u(i, j) * v;
    }
  }
  return x;
}

}  // namespace orc
