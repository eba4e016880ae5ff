// GMRES / PGMRES-Local on the refined system (reference gmres.cpp:14-126,
// driven as in scenario.cpp:694-727).  The Krylov basis, the operator
// (els_apply_forward restricted to the kept and added unknowns) and the
// left preconditioner (els_solve) stay on the device; the small Hessenberg
// least-squares problem (Givens rotations) runs on the host, which reads
// j + 2 numbers per iteration.
//
// Orthogonalisation: classical Gram-Schmidt applied twice (two GEMV pairs
// per iteration) where the reference runs modified Gram-Schmidt plus one
// clean-up pass; both keep the basis orthogonal to working precision, the
// iterates agree to rounding.  Everything else (exact outer residual before
// accepting convergence, restart, stagnation window of 50, iteration
// budget, ConvergenceError messages) follows the reference.
#include <cmath>

#include "dense.hpp"
#include "els.hpp"

namespace sbx {

namespace {

constexpr i64 kStagnationWindow = 50;

__global__ void scale_kernel(double* x, i64 n, const double* num, double alpha_host, int mode) {
  // mode 0: x *= alpha_host; mode 1: x /= sqrt(*num)
  const double a = mode == 0 ? alpha_host : 1.0 / sqrt(*num);
  for (i64 i = blockIdx.x * i64(blockDim.x) + threadIdx.x; i < n; i += i64(gridDim.x) * blockDim.x) x[i] *= a;
}

__global__ void sub_kernel(const double* a, const double* b, double* out, i64 n) {
  for (i64 i = blockIdx.x * i64(blockDim.x) + threadIdx.x; i < n; i += i64(gridDim.x) * blockDim.x)
    out[i] = a[i] - b[i];
}

unsigned grid1(i64 n) { return unsigned(std::max<i64>(1, std::min<i64>((n + 255) / 256, 148 * 8))); }

struct Ctx {
  Els& e;
  cudaStream_t s;
  i64 nk, nc, np, nr, next;
  DevBuf<double> ext_in, ext_out, dot;
  bool precond;

  // w = restrict((Atilde + L R) extend(v))
  void apply(const double* v, double* w) {
    SBX_CUDA(cudaMemsetAsync(ext_in.get() + nk, 0, size_t(nc) * 8, s));
    SBX_CUDA(cudaMemcpyAsync(ext_in.get(), v, size_t(nk) * 8, cudaMemcpyDeviceToDevice, s));
    SBX_CUDA(cudaMemcpyAsync(ext_in.get() + nk + nc, v + nk, size_t(np) * 8, cudaMemcpyDeviceToDevice, s));
    els_apply_forward_device(e, ext_in.get(), ext_out.get(), 1, s);
    SBX_CUDA(cudaMemcpyAsync(w, ext_out.get(), size_t(nk) * 8, cudaMemcpyDeviceToDevice, s));
    SBX_CUDA(cudaMemcpyAsync(w + nk, ext_out.get() + nk + nc, size_t(np) * 8, cudaMemcpyDeviceToDevice, s));
  }
  // in place: w <- M^{-1} w (els_solve on (kept, added) data)
  void left(double* w, double* tmp) {
    if (!precond) return;
    els_solve(e, w, nr, 1, tmp, nr, false, true, s);
    SBX_CUDA(cudaMemcpyAsync(w, tmp, size_t(nr) * 8, cudaMemcpyDeviceToDevice, s));
  }
  double norm(const double* x) {
    gemm_batched({{x, x, dot.get(), 1, 1, int(nr), int(nr), int(nr), 1, 1, 0, 1.0, 0.0}}, s);
    double h = 0;
    dot.download(&h, 1, s);
    SBX_CUDA(cudaStreamSynchronize(s));
    return std::sqrt(h);
  }
};

}  // namespace

GmresOutcome els_gmres(Els& e, const double* g_n, double* tau_n, bool precond, double tol, i64 max_iter,
                       i64 restart, cudaStream_t s) {
  require(tol > 0.0 && tol < 1.0, "gmres: tolerance out of (0,1)");
  require(max_iter >= 1, "gmres: iteration budget must be positive");
  const i64 nr = e.n_k + e.n_p;
  for (i64 i = 0; i < nr; ++i) require(std::isfinite(g_n[i]), "gmres: right-hand side not finite");
  Ctx c{e, s, e.n_k, e.n_c, e.n_p, nr, e.n_ext(), {}, {}, {}, precond};
  c.ext_in.resize(size_t(c.next));
  c.ext_out.resize(size_t(c.next));
  c.dot.resize(1);
  GmresOutcome out;
  const i64 cycle = restart > 0 ? std::min(restart, max_iter) : max_iter;
  DevBuf<double> V(static_cast<size_t>(nr * (cycle + 1))), b(static_cast<size_t>(nr)), x(static_cast<size_t>(nr)),
      w(static_cast<size_t>(nr)), tmp(static_cast<size_t>(nr)), hcol(static_cast<size_t>(cycle + 2)),
      ccol(static_cast<size_t>(cycle + 2)), y(static_cast<size_t>(cycle + 1));
  b.upload(g_n, size_t(nr), s);
  x.zero(s);
  // beta0 = |M^{-1} b|
  SBX_CUDA(cudaMemcpyAsync(w.get(), b.get(), size_t(nr) * 8, cudaMemcpyDeviceToDevice, s));
  c.left(w.get(), tmp.get());
  const double beta0 = c.norm(w.get());
  out.history.push_back(1.0);
  auto finish = [&]() {
    x.download(tau_n, size_t(nr), s);
    SBX_CUDA(cudaStreamSynchronize(s));
  };
  if (beta0 == 0.0) {
    finish();
    return out;
  }
  std::vector<double> h(static_cast<size_t>((cycle + 1) * cycle), 0.0), cs(static_cast<size_t>(cycle)),
      sn(static_cast<size_t>(cycle)), g(static_cast<size_t>(cycle + 1));
  auto H = [&](i64 i, i64 j) -> double& { return h[size_t(i + j * (cycle + 1))]; };
  double best = 1.0;
  i64 since_best = 0, total = 0;
  auto fold = [&](i64 m) {  // x += V(:, 0:m) y, y = H(0:m,0:m)^{-1} g(0:m)
    std::vector<double> yy(static_cast<size_t>(m));
    for (i64 i = m - 1; i >= 0; --i) {
      double acc = g[size_t(i)];
      for (i64 l = i + 1; l < m; ++l) acc -= H(i, l) * yy[size_t(l)];
      yy[size_t(i)] = acc / H(i, i);
    }
    y.upload(yy, s);
    gemm_batched({{V.get(), y.get(), x.get(), int(nr), 1, int(m), int(nr), int(m), int(nr), 0, 0, 1.0, 1.0}}, s);
  };
  for (;;) {
    // exact outer residual r = M^{-1}(b - A x)
    c.apply(x.get(), tmp.get());
    sub_kernel<<<grid1(nr), 256, 0, s>>>(b.get(), tmp.get(), w.get(), nr);
    SBX_LAUNCHED();
    c.left(w.get(), tmp.get());
    const double beta = c.norm(w.get());
    if (beta / beta0 <= tol) break;
    if (total >= max_iter) {
      out.error = "gmres hit the iteration budget before the residual target";
      break;
    }
    SBX_CUDA(cudaMemcpyAsync(V.get(), w.get(), size_t(nr) * 8, cudaMemcpyDeviceToDevice, s));
    scale_kernel<<<grid1(nr), 256, 0, s>>>(V.get(), nr, nullptr, 1.0 / beta, 0);
    SBX_LAUNCHED();
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    i64 j = 0;
    bool claimed = false, failed = false;
    for (; j < cycle && total < max_iter; ++j) {
      double* vj = V.get() + j * nr;
      c.apply(vj, w.get());
      c.left(w.get(), tmp.get());
      // two classical Gram-Schmidt passes
      for (int pass = 0; pass < 2; ++pass) {
        double* col = pass == 0 ? hcol.get() : ccol.get();
        gemm_batched({{V.get(), w.get(), col, int(j + 1), 1, int(nr), int(nr), int(nr), int(j + 1), 1, 0, 1.0, 0.0}},
                     s);
        gemm_batched({{V.get(), col, w.get(), int(nr), 1, int(j + 1), int(nr), int(j + 1), int(nr), 0, 0, -1.0, 1.0}},
                     s);
      }
      std::vector<double> h1(static_cast<size_t>(j + 1)), h2(static_cast<size_t>(j + 1));
      hcol.download(h1.data(), h1.size(), s);
      ccol.download(h2.data(), h2.size(), s);
      const double hnext = c.norm(w.get());  // synchronises
      for (i64 i = 0; i <= j; ++i) H(i, j) = h1[size_t(i)] + h2[size_t(i)];
      for (i64 i = 0; i < j; ++i) {
        const double t = cs[size_t(i)] * H(i, j) + sn[size_t(i)] * H(i + 1, j);
        H(i + 1, j) = -sn[size_t(i)] * H(i, j) + cs[size_t(i)] * H(i + 1, j);
        H(i, j) = t;
      }
      const double denom = std::hypot(H(j, j), hnext);
      cs[size_t(j)] = denom > 0 ? H(j, j) / denom : 1.0;
      sn[size_t(j)] = denom > 0 ? hnext / denom : 0.0;
      H(j, j) = denom;
      H(j + 1, j) = 0.0;
      g[size_t(j + 1)] = -sn[size_t(j)] * g[size_t(j)];
      g[size_t(j)] = cs[size_t(j)] * g[size_t(j)];
      const double rel = std::fabs(g[size_t(j + 1)]) / beta0;
      out.history.push_back(rel);
      out.n_iter = ++total;
      if (rel < best) {
        best = rel;
        since_best = 0;
      } else {
        ++since_best;
      }
      const bool converged = rel <= tol;
      if (converged || since_best >= kStagnationWindow || hnext == 0.0 || total >= max_iter) {
        fold(j + 1);
        if (converged || hnext == 0.0) {
          claimed = true;
          break;
        }
        out.error = since_best >= kStagnationWindow
                        ? "gmres stagnated: no residual decrease over " + std::to_string(kStagnationWindow) +
                              " iterations"
                        : "gmres hit the iteration budget before the residual target";
        failed = true;
        break;
      }
      double* vn = V.get() + (j + 1) * nr;
      SBX_CUDA(cudaMemcpyAsync(vn, w.get(), size_t(nr) * 8, cudaMemcpyDeviceToDevice, s));
      scale_kernel<<<grid1(nr), 256, 0, s>>>(vn, nr, nullptr, 1.0 / hnext, 0);
      SBX_LAUNCHED();
    }
    if (failed) break;
    if (!claimed && j == cycle) fold(cycle);
  }
  finish();
  return out;
}

}  // namespace sbx
