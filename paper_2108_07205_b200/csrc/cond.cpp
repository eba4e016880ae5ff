// Conditioning diagnostics of the extended system (reference els.cpp:205-270,
// linop.cpp:17-43) on the device operators.
#include <algorithm>
#include <cmath>
#include <limits>
#include <random>

#include "dense.hpp"
#include "els.hpp"
#include "idengine.hpp"

namespace sbx {

std::vector<double> jacobi_singular_values(std::vector<double> a, i64 m, i64 n) {
  require(m >= n, "jacobi_singular_values: expects m >= n");
  const double tol = 1e-15;
  for (int sweep = 0; sweep < 60; ++sweep) {
    bool rotated = false;
    for (i64 p = 0; p < n - 1; ++p)
      for (i64 q = p + 1; q < n; ++q) {
        double* ap = a.data() + p * m;
        double* aq = a.data() + q * m;
        double alpha = 0.0, beta = 0.0, gamma = 0.0;
        for (i64 i = 0; i < m; ++i) {
          alpha += ap[i] * ap[i];
          beta += aq[i] * aq[i];
          gamma += ap[i] * aq[i];
        }
        if (gamma == 0.0 || std::fabs(gamma) <= tol * std::sqrt(alpha * beta)) continue;
        rotated = true;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), sn = c * t;
        for (i64 i = 0; i < m; ++i) {
          const double x = ap[i], y = aq[i];
          ap[i] = c * x - sn * y;
          aq[i] = sn * x + c * y;
        }
      }
    if (!rotated) break;
  }
  std::vector<double> sv(static_cast<size_t>(n));
  for (i64 j = 0; j < n; ++j) {
    double s2 = 0.0;
    for (i64 i = 0; i < m; ++i) s2 += a[size_t(i + j * m)] * a[size_t(i + j * m)];
    sv[size_t(j)] = std::sqrt(s2);
  }
  std::sort(sv.begin(), sv.end(), std::greater<double>());
  return sv;
}

namespace {

__global__ void cond_scale_kernel(double* x, i64 n, double a) {
  for (i64 i = blockIdx.x * i64(blockDim.x) + threadIdx.x; i < n; i += i64(gridDim.x) * blockDim.x) x[i] *= a;
}

double ratio(const std::vector<double>& sv, i64 k) {
  if (k == 0 || sv.empty()) return 1.0;
  const double lo = sv[size_t(std::min<i64>(k, i64(sv.size())) - 1)];
  return lo > 0.0 ? sv[0] / lo : std::numeric_limits<double>::infinity();
}

// sigma_1 / sigma_k of a tall device matrix (M x k, ld M): the R factor of a
// column-pivoted device QR carries the same singular values.
double tall_factor_cond(const double* A, i64 M, i64 k, cudaStream_t s) {
  if (k == 0) return 1.0;
  DevBuf<double> w(static_cast<size_t>(M * k));
  SBX_CUDA(cudaMemcpyAsync(w.get(), A, size_t(M * k) * 8, cudaMemcpyDeviceToDevice, s));
  IdBatch b;
  b.factor({IdProblem{w.get(), int(M), int(k), int(M)}}, 1e-300, s);
  std::vector<double> top(static_cast<size_t>(k * k));
  SBX_CUDA(cudaMemcpy2DAsync(top.data(), size_t(k) * 8, w.get(), size_t(M) * 8, size_t(k) * 8, size_t(k),
                             cudaMemcpyDeviceToHost, s));
  SBX_CUDA(cudaStreamSynchronize(s));
  const auto& perm = b.perm(0);
  std::vector<double> R(static_cast<size_t>(k * k), 0.0);
  for (i64 l = 0; l < k; ++l)
    for (i64 i = 0; i <= l; ++i) R[size_t(i + l * k)] = top[size_t(i + i64(perm[size_t(l)]) * k)];
  return ratio(jacobi_singular_values(std::move(R), k, k), k);
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

CondReport els_conditioning(Els& e, int iters, cudaStream_t s) {
  CondReport r;
  const i64 k = e.k, n = e.n_ext();
  if (k > 0) {
    std::vector<double> W(static_cast<size_t>(k * k));
    e.Wmat.download(W.data(), W.size(), s);
    SBX_CUDA(cudaStreamSynchronize(s));
    r.kappa_w = ratio(jacobi_singular_values(std::move(W), k, k), k);  // dense_cond (els.cpp:207-213)
    r.kappa_l = tall_factor_cond(e.L->get(), n, k, s);                 // factor_cond (els.cpp:216-222)
    DevBuf<double> rt(static_cast<size_t>(n * k));                      // R^T: n x k
    copy_batched({{e.R.get(), rt.get(), int(n), int(k), int(k), int(n), 1, 0}}, s);
    r.kappa_r = tall_factor_cond(rt.get(), n, k, s);
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
