// Conditioning diagnostics of the extended system (reference els.cpp:205-270,
// linop.cpp:17-43) on the device operators.
#include <algorithm>
#include <cmath>
#include <limits>
#include <random>

#include "dense.hpp"
#include "els.hpp"
#include "entries.hpp"
#include "idengine.hpp"
#include "svd.hpp"

namespace sbx {

namespace {

__global__ void cond_scale_kernel(double* x, i64 n, double a) {
  for (i64 i = blockIdx.x * i64(blockDim.x) + threadIdx.x; i < n; i += i64(gridDim.x) * blockDim.x) x[i] *= a;
}

double ratio(const std::vector<double>& sv, i64 k) {
  if (k == 0 || sv.empty()) return 1.0;
  const double lo = sv[size_t(std::min<i64>(k, i64(sv.size())) - 1)];
  return lo > 0.0 ? sv[0] / lo : std::numeric_limits<double>::infinity();
}

// sigma_1 / sigma_k of a device matrix of declared rank k (factor_cond,
// els.cpp:216-222), by the device Jacobi SVD.
double factor_cond_device(const double* A, i64 m, i64 n, i64 k, cudaStream_t s) {
  if (k == 0) return 1.0;
  return ratio(singular_values_device(A, m, n, m, s), k);
}

// dense_cond (els.cpp:207-213): sigma_max / sigma_min.
double dense_cond_device(const double* A, i64 n, cudaStream_t s) {
  if (n == 0) return 1.0;
  const auto sv = singular_values_device(A, n, n, n, s);
  return sv.back() > 0.0 ? sv.front() / sv.back() : std::numeric_limits<double>::infinity();
}

// Largest singular value by power iteration on B B^T (linop.cpp:17-36).
template <class F, class Ft>
double operator_norm(i64 n, F apply, Ft apply_t, int iters, std::uint64_t seed, cudaStream_t s) {
  if (n == 0) return 0.0;
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss(0.0, 1.0);
  std::vector<double> h(static_cast<size_t>(n));
  for (auto& x : h) x = gauss(rng);
  double nv = 0.0;
  for (double x : h) nv += x * x;
  nv = std::sqrt(nv);
  for (auto& x : h) x /= nv;
  DevBuf<double> v(static_cast<size_t>(n)), w(static_cast<size_t>(n)), dot(1);
  v.upload(h, s);
  auto norm = [&](const double* x) {
    gemm_batched({{x, x, dot.get(), 1, 1, int(n), int(n), int(n), 1, 1, 0, 1.0, 0.0}}, s);
    double r = 0.0;
    dot.download(&r, 1, s);
    SBX_CUDA(cudaStreamSynchronize(s));
    return std::sqrt(r);
  };
  double sig = 0.0;
  for (int it = 0; it < iters; ++it) {
    apply(v.get(), w.get());
    sig = norm(w.get());
    if (sig == 0.0) return 0.0;
    apply_t(w.get(), v.get());
    const double nn = norm(v.get());
    if (nn == 0.0) return sig;
    cond_scale_kernel<<<unsigned(std::min<i64>((n + 255) / 256, 1184)), 256, 0, s>>>(v.get(), n, 1.0 / nn);
    SBX_LAUNCHED();
  }
  return sig;
}

}  // namespace

CondReport els_conditioning(Els& e, int iters, cudaStream_t s, bool dense) {
  CondReport r;
  const i64 k = e.k, n = e.n_ext();
  if (k > 0) {
    r.kappa_w = dense_cond_device(e.Wmat.get(), k, s);          // dense_cond (els.cpp:230)
    r.kappa_l = factor_cond_device(e.L->get(), n, k, k, s);     // factor_cond (els.cpp:231)
    r.kappa_r = factor_cond_device(e.R.get(), k, n, k, s);      // factor_cond (els.cpp:232)
  }
  if (dense) {  // dense oracles (els.cpp:234-240): SVDs of Atilde and Atilde + L R
    require(e.old_g && e.new_g, "conditioning_report: the ELS does not know its meshes");
    require(n <= 12000, "conditioning_report: dense oracles are limited to 12000 unknowns (nystrom.cpp:13)");
    DevBuf<double> A(static_cast<size_t>(n * n));
    A.zero(s);
    const i64 nkc = e.n_k + e.n_c;
    std::vector<i64> oc = e.kept_old_s;
    oc.insert(oc.end(), e.cut_s.begin(), e.cut_s.end());
    DevBuf<i64> d_oc, d_p;
    d_oc.upload(oc, s);
    EntryOracle eo(*e.old_g, e.form, e.mu, s);
    eo.submatrix(d_oc.get(), nkc, d_oc.get(), nkc, A.get(), n, s);
    if (e.n_p > 0) {
      d_p.upload(e.added_s, s);
      EntryOracle en(*e.new_g, e.form, e.mu, s);
      en.submatrix(d_p.get(), e.n_p, d_p.get(), e.n_p, A.get() + nkc + nkc * n, n, s);
    }
    DevBuf<double> X(static_cast<size_t>(n * n));
    SBX_CUDA(cudaMemcpyAsync(X.get(), A.get(), size_t(n * n) * 8, cudaMemcpyDeviceToDevice, s));
    r.kappa_tilde = dense_cond_device(A.get(), n, s);
    if (k > 0)
      gemm_batched({{e.L->get(), e.R.get(), X.get(), int(n), int(n), int(k), int(n), int(k), int(n), 0, 0, 1.0, 1.0}},
                   s);
    r.kappa_ext = dense_cond_device(X.get(), n, s);
    r.bound = std::min(r.kappa_l * r.kappa_l, r.kappa_r * r.kappa_r) * r.kappa_ext * r.kappa_tilde;
    r.bound_holds = r.kappa_w <= r.bound * 1.000001;
    return r;
  }
  // estimator route (els.cpp:250-264): power iteration on the operators and
  // on their solves, seeds 1 and 2 (condition_estimate, linop.cpp:38-43)
  auto fwd = [&](const double* v, double* w) { els_apply_forward_device(e, v, w, 1, s, false, true); };
  auto fwd_t = [&](const double* v, double* w) { els_apply_forward_device(e, v, w, 1, s, true, true); };
  auto inv = [&](const double* v, double* w) { els_solve_ext_device(e, v, w, 1, s); };
  auto inv_t = [&](const double* v, double* w) { els_solve_ext_t_device(e, v, w, 1, s); };
  r.kappa_ext = operator_norm(n, fwd, fwd_t, iters, 1, s) * operator_norm(n, inv, inv_t, iters, 2, s);
  auto tf = [&](const double* v, double* w) { els_apply_forward_device(e, v, w, 1, s, false, false); };
  auto tf_t = [&](const double* v, double* w) { els_apply_forward_device(e, v, w, 1, s, true, false); };
  auto ti = [&](const double* v, double* w) { els_atilde_solve(e, v, w, 1, s, false); };
  auto ti_t = [&](const double* v, double* w) { els_atilde_solve(e, v, w, 1, s, true); };
  r.kappa_tilde = operator_norm(n, tf, tf_t, iters, 1, s) * operator_norm(n, ti, ti_t, iters, 2, s);
  r.bound = std::min(r.kappa_l * r.kappa_l, r.kappa_r * r.kappa_r) * r.kappa_ext * r.kappa_tilde;
  r.bound_holds = r.kappa_w <= r.bound * 1.000001;
  return r;
}

}  // namespace sbx
