// Device low-rank update compression Q ~= L R (reference lowrank.cpp:253-327,
// proxy.cpp:46-302, two-step ID mode).
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "geometry.hpp"

namespace sbx {

struct AppSolver;

struct Update {
  i64 k = 0, k1 = 0, k_kc = 0, k_kp = 0, k_pk = 0;
  i64 nk2 = 0, nc2 = 0, np2 = 0;
  i64 n_ext() const { return nk2 + nc2 + np2; }
  // n_ext x k, column-major; shared with the ELS solvers built on it
  std::shared_ptr<DevBuf<double>> L = std::make_shared<DevBuf<double>>();
  DevBuf<double> R;  // k x n_ext, column-major
  std::vector<i64> skeleton;
  std::vector<std::string> notes;
  // A_pp^{-1} built alongside the compression (adopted by els_build when it
  // matches; null if its build failed, els_build then reports the error)
  std::shared_ptr<AppSolver> app;
};

struct ProxyCircleH {
  double cx, cy, r0;
};
// make_proxy_geometry (proxy.cpp:46-77): one circle per component gaining nodes.
std::vector<ProxyCircleH> make_proxy_circles(const Geom& new_g, const Plan& plan);

std::unique_ptr<Update> update_compress_device(const Geom& old_g, const Geom& new_g,
                                               const Plan& plan, int formulation, double mu,
                                               double eps, std::uint64_t seed, cudaStream_t s);
void update_download(const Update& u, int which, double* out, cudaStream_t s);
// CompressionMode::SvdOptimal (lowrank.cpp:329-362): dense truncated SVDs of
// the kc / kp / pk blocks, re-truncated through L1 (update_svd.cpp).
std::unique_ptr<Update> update_svd_optimal_device(const Geom& old_g, const Geom& new_g, const Plan& plan,
                                                  int formulation, double mu, double eps, cudaStream_t s);
std::unique_ptr<Update> update_from_factors(const Plan& plan, const double* L, const double* R,
                                            i64 n_ext, i64 k, cudaStream_t s);

}  // namespace sbx
