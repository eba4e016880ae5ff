// Extended linear system + Woodbury solver on the device (north-star
// subsystem 3; reference els.cpp:80-203).
//
// Extended ordering (kept, cut, added) scalars.  Atilde = diag(A_oo in
// old-mesh order, A_pp); A_oo^{-1} is the static HBS inverse, A_pp^{-1} an
// explicit dense inverse (2 N_p <= 2048, els.hpp:40) or its own HBS.
//   build:  X = Atilde^{-1} L  (multi-RHS sweep, nrhs = k),
//           W = I + R X        (DMMA GEMM),  W = P L U + rcond gate
//   solve:  y = Atilde^{-1} g ;  y -= X W^{-1} (R y)
#pragma once

#include "geometry.hpp"
#include "hbs.hpp"
#include "update.hpp"

#include <string>

namespace sbx {

// A_pp^{-1} for the added unknowns (els.cpp:98-118): explicit dense inverse
// when 2 N_p <= 2048 (kDenseAddedLimit, els.hpp:40), else A_pp's own
// inverted HBS.  It depends only on the refined mesh, so update compression
// starts building it concurrently (Update::app) and els_build adopts it.
struct AppSolver {
  const Geom* g = nullptr;
  int form = 0;
  double mu = 0, eps = 0;
  std::vector<i64> added;           // plan.added_new it was built for
  std::unique_ptr<HbsOp> h;         // HBS of A_pp above the dense limit
  DevBuf<double> inv;               // dense A_pp^{-1}
  DevBuf<double> fwd;               // dense A_pp (forward apply, els.cpp:67-74)
  bool matches(const Geom& g2, const Plan& p, int f, double m, double e) const {
    return g == &g2 && form == f && mu == m && eps == e && added == p.added_new;
  }
};
// Partial-pivot LU, explicit inverse into inv (ld n) and Eigen's
// PartialPivLU::rcond() estimate of an n x n device matrix a (destroyed).
double dense_inverse(double* a, i64 n, double* inv, cudaStream_t s);
std::shared_ptr<AppSolver> build_app_solver(const Geom& new_g, const Plan& plan, int formulation,
                                            double mu, double eps, cudaStream_t s);
// out = A_pp^{-1} v (or A_pp^{-T} v) for n_p x nrhs column-major device blocks
// (els.cpp:47: app_lu.solve / app_h solve).
void app_solve_device(AppSolver& a, const double* v, i64 ldv, double* out, i64 ldo, i64 nrhs, cudaStream_t s,
                      bool transpose = false);

struct Els {
  HbsOp* a_oo = nullptr;            // static wall solver (owned by the caller's handle)
  std::shared_ptr<AppSolver> app;   // A_pp^{-1}
  i64 n_k = 0, n_c = 0, n_p = 0;    // scalar counts
  i64 k = 0;
  i64 n_ext() const { return n_k + n_c + n_p; }
  DevBuf<double> R;                 // k x n_ext
  std::shared_ptr<DevBuf<double>> L;  // n_ext x k (the update's, shared)
  DevBuf<double> X;                 // n_ext x k
  DevBuf<double> Winv;              // k x k explicit (I + R X)^{-1}
  DevBuf<double> Wmat;              // k x k (I + R X), for inspection
  DevBuf<i64> d_old_of_ext;         // ext rows [0, n_k+n_c) -> old-mesh scalar
  std::vector<i64> kept_new_s, added_s;
  std::vector<i64> kept_old_s, cut_s;
  // the meshes and formulation it was built on (dense conditioning route);
  // the caller keeps the geometry alive while it uses that route
  const Geom* old_g = nullptr;
  const Geom* new_g = nullptr;
  int form = 0;
  double mu = 1.0;
  i64 n_new = 0;
  // Per-stream solve workspaces: the solver is immutable after build, so
  // concurrent solves on distinct streams are legal.
  struct Scratch {
    DevBuf<double> a, b;
    StreamMark mark;  // end of the last solve on this stream
    double* ws(size_t n, cudaStream_t s) {
      StreamScope ss(s);
      a.reserve(n);
      return a.get();
    }
    double* ws2(size_t n, cudaStream_t s) {
      StreamScope ss(s);
      b.reserve(n);
      return b.get();
    }
  };
  PerStream<Scratch> scratch;
  Scratch& scratch_for(cudaStream_t s) { return scratch.get(s); }
  void drain() {
    scratch.for_each([](Scratch& x) { x.mark.wait(); });
  }
};

std::unique_ptr<Els> els_build_device(HbsOp& a_oo, const Geom& old_g, const Geom& new_g,
                                      const Plan& plan, const Update& upd, int formulation,
                                      double mu, cudaStream_t s);
// raw: g has n_ext rows (kept, cut, added); else n_k + n_p rows (kept, added)
// and the dummy block is dropped from the output (els.cpp:165-179).
// transpose (raw only): els_solve_raw_t (els.cpp:154-163).
void els_solve(Els& e, const double* g, i64 ldg, i64 nrhs, double* y, i64 ldy, bool raw, bool dev,
               cudaStream_t s, bool transpose = false);
void els_density_on_refined(const Els& e, const double* tau_n, double* out);
void els_download_xw(const Els& e, double* X, double* W, cudaStream_t s);

// els_apply_forward (els.cpp:181-186): out = (Atilde + L R) v, v / out
// n_ext x nrhs device blocks (ld n_ext).
// transpose: els_apply_forward_t (els.cpp:188-193), out = (Atilde + L R)^T v.
// with_update = false: the block-diagonal part Atilde alone (els.cpp:67-74).
void els_apply_forward_device(Els& e, const double* v, double* out, i64 nrhs, cudaStream_t s,
                              bool transpose = false, bool with_update = true);
// Atilde^{-1} v or Atilde^{-T} v on extended blocks (els.cpp:58-65).
void els_atilde_solve(Els& e, const double* v, double* out, i64 nrhs, cudaStream_t s, bool transpose);

// conditioning_report (els.cpp:225-270) on the estimator route: kappa_w,
// kappa_l, kappa_r from the singular values of W and of the R factors of
// device QRs of L and R^T (one-sided Jacobi on the k x k factors, host);
// kappa_ext and kappa_tilde by seeded power iteration on the device
// operators and their solves (linop.cpp:17-43, mt19937_64 Gaussian starts).
struct CondReport {
  double kappa_w = 1.0, kappa_l = 1.0, kappa_r = 1.0, kappa_ext = 1.0, kappa_tilde = 1.0, bound = 1.0;
  bool bound_holds = true;
};
// dense = true: the dense-oracle route (els.cpp:234-240): kappa_tilde and
// kappa_ext from the singular values of the assembled Atilde and
// Atilde + L R (device Jacobi SVD, n_ext <= 12000).
CondReport els_conditioning(Els& e, int iters, cudaStream_t s, bool dense = false);

// GMRES / PGMRES-Local on the refined system in (kept, added) unknowns
// (gmres.cpp:14-126 driven like scenario.cpp:694-727): operator =
// els_apply_forward restricted to (kept, added), optional left
// preconditioner = els_solve.  Host g_n in, tau_n out; returns iterations,
// fills the relative residual history (iterations + 1 entries).
struct GmresOutcome {
  i64 n_iter = 0;
  std::vector<double> history;
  std::string error;  // non-empty: the reference's ConvergenceError message
};
GmresOutcome els_gmres(Els& e, const double* g_n, double* tau_n, bool precond, double tol, i64 max_iter,
                       i64 restart, cudaStream_t s);

// Device-resident solve for callers holding device buffers:
// y_ext (n_ext x nrhs, column-major ld n_ext) = ELS^{-1} g_ext.
void els_solve_ext_device(Els& e, const double* g_ext, double* y_ext, i64 nrhs, cudaStream_t s);
// y_ext = ELS^{-T} g_ext (els.cpp:154-163).
void els_solve_ext_t_device(Els& e, const double* g_ext, double* y_ext, i64 nrhs, cudaStream_t s);

}  // namespace sbx
