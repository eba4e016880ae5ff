// ELS / Woodbury build and solve on the device (reference els.cpp:25-203).
#include "els.hpp"

#include <cstdlib>
#include "idengine.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <limits>

#include "dense.hpp"
#include "entries.hpp"
#include "hbs_build.hpp"

namespace sbx {

namespace {

// widths (columns) of the last Woodbury build / solve sweeps: hints for
// build_app_solver's item-table prebuild
std::atomic<i64> g_hint_build_cols{0}, g_hint_solve_cols{0};

std::vector<i64> scalars(const std::vector<i64>& nodes) {
  std::vector<i64> o(2 * nodes.size());
  i64* d = o.data();
  const i64* n = nodes.data();
  for (size_t i = 0, e = nodes.size(); i < e; ++i) {  // indexed stores: this runs on the step's critical path
    d[2 * i] = 2 * n[i];
    d[2 * i + 1] = 2 * n[i] + 1;
  }
  return o;
}

}  // namespace

// Dense LU + explicit inverse + rcond (Eigen PartialPivLU::rcond) of an
// n x n device matrix a (destroyed); returns rcond.
double dense_inverse(double* a, i64 n, double* inv, cudaStream_t s) {
  require(n <= 2048, "dense block above 2048 unknowns (els.hpp:40 limit)");
  DevBuf<int> piv(static_cast<size_t>(n));
  DevBuf<double> rc(1), work(static_cast<size_t>(4 * n));
  LuJob j{};
  j.a = a;
  j.n = int(n);
  j.lda = int(n);
  j.piv = piv.get();
  j.inv = inv;
  j.rcond = rc.get();
  j.work = work.get();
  lu_batched({j}, s);
  double r = 0;
  rc.download(&r, 1, s);
  SBX_CUDA(cudaStreamSynchronize(s));
  return r;
}

namespace {

// out = Atilde^{-1} v for an n_ext x nrhs column-major device block
// (els.cpp:43-65): the old-mesh part goes through the HBS sweep in old
// ordering (scatter/gather fused into the layout kernels), the added part
// through the dense inverse or its own HBS.
void atilde_solve(Els& e, const double* v, i64 ldv, double* out, i64 ldo, i64 nrhs, cudaStream_t s,
                  bool tr = false) {
  HbsOp& A = *e.a_oo;
  hbs_ensure_solve_plan(A);
  if (tr) hbs_ensure_transpose(A, true, false, s);
  const i64 nkc = e.n_k + e.n_c;
  // scatter to old-mesh rows, sweep, gather: out row i <- old row map[i]
  hbs_sweep_rows(A, A.solve_plan, v, ldv, nkc, nrhs, out, ldo, e.d_old_of_ext.get(), tr, s);
  phase_mark("els:   a_oo sweep", s);
  if (e.n_p == 0) return;
  app_solve_device(*e.app, v + nkc, ldv, out + nkc, ldo, nrhs, s, tr);
}

}  // namespace

void app_solve_device(AppSolver& a, const double* vp, i64 ldv, double* op, i64 ldo, i64 nrhs, cudaStream_t s,
                      bool tr) {
  const i64 n_p = 2 * i64(a.added.size());
  if (n_p == 0 || nrhs == 0) return;
  if (a.h) {
    HbsOp& H = *a.h;
    hbs_ensure_solve_plan(H);
    if (tr) hbs_ensure_transpose(H, true, false, s);
    hbs_sweep_rows(H, H.solve_plan, vp, ldv, n_p, nrhs, op, ldo, nullptr, tr, s);
    phase_mark("els:   A_pp sweep", s);
  } else {  // explicit inverse of A_pp (els.cpp:47: app_lu.solve / app_lu.transpose().solve)
    gemm_batched({{a.inv.get(), vp, op, int(n_p), int(nrhs), int(n_p), int(n_p), int(ldv), int(ldo), tr ? 1 : 0, 0,
                   1.0, 0.0}},
                 s);
  }
}

std::shared_ptr<AppSolver> build_app_solver(const Geom& new_g, const Plan& plan, int form, double mu,
                                            double eps, cudaStream_t s) {
  auto a = std::make_shared<AppSolver>();
  a->g = &new_g;
  a->form = form;
  a->mu = mu;
  a->eps = eps;
  a->added = plan.added_new;
  const auto added_s = scalars(plan.added_new);
  const i64 n_p = i64(added_s.size());
  if (n_p == 0) return a;
  if (n_p <= 2048) {  // kDenseAddedLimit counts scalars (els.hpp:40)
    EntryOracle eo(new_g, form, mu, s);
    DevBuf<double> app(static_cast<size_t>(n_p * n_p));
    DevBuf<i64> idx;
    idx.upload(added_s, s);
    eo.submatrix(idx.get(), n_p, idx.get(), n_p, app.get(), n_p, s);
    a->inv.resize(size_t(n_p * n_p));
    a->fwd.resize(size_t(n_p * n_p));
    SBX_CUDA(cudaMemcpyAsync(a->fwd.get(), app.get(), size_t(n_p * n_p) * 8, cudaMemcpyDeviceToDevice, s));
    const double rc = dense_inverse(app.get(), n_p, a->inv.get(), s);
    if (rc < 1e-14) throw Error(4, "added-unknown diagonal block is singular at added block");
  } else {
    HbsBuildOptions o;
    o.eps = eps;
    static const bool unfused = std::getenv("SBX_APP_UNFUSED") != nullptr;  // diagnostics
    if (unfused) {
      a->h = hbs_compress_device(new_g, form, mu, plan.added_new.data(), i64(plan.added_new.size()), o, s);
      id_rendezvous_leave();  // no factorisations below (joint CPQR launches, update.cpp)
      hbs_invert_device(*a->h, s);
    } else {  // the inverse of each level overlaps the compression of the next
      a->h = hbs_compress_invert_device(new_g, form, mu, plan.added_new.data(), i64(plan.added_new.size()), o, s);
      id_rendezvous_leave();
    }
    hbs_build_solve_plan(*a->h);
    // this runs beside the update compression (update.cpp: A_pp thread); the
    // sweeps over the new A_pp come right after it, at the widths of the
    // previous step's Woodbury build and solve: build their item tables here
    // rather than on the critical path
    for (const auto* hint : {&g_hint_build_cols, &g_hint_solve_cols}) {
      const i64 w = hint->load(std::memory_order_relaxed);
      if (w > 0) hbs_prebuild_flow(*a->h, a->h->solve_plan, w, s);
    }
  }
  return a;
}

std::unique_ptr<Els> els_build_device(HbsOp& a_oo, const Geom& old_g, const Geom& new_g,
                                      const Plan& plan, const Update& upd, int form, double mu,
                                      cudaStream_t s) {
  require(a_oo.has_inverse, "els_build: diagonal solver lacks inverse");
  auto e = std::make_unique<Els>();
  e->a_oo = &a_oo;
  e->old_g = &old_g;
  e->new_g = &new_g;
  e->form = form;
  e->mu = mu;
  e->n_k = 2 * i64(plan.kept_old.size());
  e->n_c = 2 * i64(plan.cut_old.size());
  e->n_p = 2 * i64(plan.added_new.size());
  e->n_new = new_g.n_nodes();
  require(a_oo.n == e->n_k + e->n_c, "els_build: diagonal solver size does not match the old mesh");
  require(upd.n_ext() == e->n_ext(), "els_build: update factor size does not match the plan");
  {  // ext rows (kept, cut) -> old-mesh scalars: all the first sweep needs from the host
    std::vector<i64> old_of_ext(size_t(e->n_k + e->n_c));
    i64* d = old_of_ext.data();
    for (const i64 nd : plan.kept_old) {
      *d++ = 2 * nd;
      *d++ = 2 * nd + 1;
    }
    for (const i64 nd : plan.cut_old) {
      *d++ = 2 * nd;
      *d++ = 2 * nd + 1;
    }
    e->d_old_of_ext.upload(old_of_ext, s);
  }
  // the host-side index maps of the handle are filled while the device works
  auto fill_host_maps = [&] {
    e->kept_old_s = scalars(plan.kept_old);
    e->cut_s = scalars(plan.cut_old);
    e->kept_new_s = scalars(plan.kept_new);
    e->added_s = scalars(plan.added_new);
  };
  if (e->n_p > 0) {
    if (upd.app && upd.app->matches(new_g, plan, form, mu, a_oo.eps))
      e->app = upd.app;
    else
      e->app = build_app_solver(new_g, plan, form, mu, a_oo.eps, s);
  }
  phase_mark("els: A_pp", s);
  e->k = upd.k;
  const i64 k = e->k, n = e->n_ext();
  if (k > 0) {
    e->R.resize(size_t(k * n));
    SBX_CUDA(cudaMemcpyAsync(e->R.get(), upd.R.get(), size_t(k * n) * 8, cudaMemcpyDeviceToDevice, s));
    e->X.resize(size_t(n * k));
    e->L = upd.L;
    g_hint_build_cols.store(k, std::memory_order_relaxed);
    atilde_solve(*e, upd.L->get(), n, e->X.get(), n, k, s);
    phase_mark("els: X = Atilde^-1 L", s);
    // W = I + R X  (els.cpp:124)
    e->Wmat.resize(size_t(k * k));
    gemm_batched({{e->R.get(), e->X.get(), e->Wmat.get(), int(k), int(k), int(n), int(k), int(n), int(k), 0,
                   0, 1.0, 0.0}},
                 s);
    launch_add_identity(e->Wmat.get(), k, k, s);
    phase_mark("els:   W = I + R X", s);
    fill_host_maps();
    DevBuf<double> wlu(static_cast<size_t>(k * k));
    SBX_CUDA(cudaMemcpyAsync(wlu.get(), e->Wmat.get(), size_t(k * k) * 8, cudaMemcpyDeviceToDevice, s));
    e->Winv.resize(size_t(k * k));
    const double rc = dense_inverse(wlu.get(), k, e->Winv.get(), s);
    if (rc < std::sqrt(std::numeric_limits<double>::epsilon()))
      throw Error(4,
                  "woodbury operator numerically singular; consider the optimal-basis compression "
                  "mode at woodbury solve");
  } else {
    fill_host_maps();
  }
  SBX_CUDA(cudaStreamSynchronize(s));
  phase_mark("els: W, LU(W)", s);
  return e;
}

void els_apply_forward_device(Els& e, const double* v, double* out, i64 nrhs, cudaStream_t s, bool tr,
                              bool with_update) {
  const i64 n = e.n_ext(), nkc = e.n_k + e.n_c;
  HbsOp& A = *e.a_oo;
  hbs_ensure_apply_plan(A);
  if (tr) hbs_ensure_transpose(A, false, true, s);
  hbs_sweep_rows(A, A.apply_plan, v, n, nkc, nrhs, out, n, e.d_old_of_ext.get(), tr, s);
  if (e.n_p > 0) {
    if (e.app->h) {
      HbsOp& H = *e.app->h;
      hbs_ensure_apply_plan(H);
      if (tr) hbs_ensure_transpose(H, false, true, s);
      hbs_sweep_rows(H, H.apply_plan, v + nkc, n, e.n_p, nrhs, out + nkc, n, nullptr, tr, s);
    } else {
      gemm_batched({{e.app->fwd.get(), v + nkc, out + nkc, int(e.n_p), int(nrhs), int(e.n_p), int(e.n_p), int(n),
                     int(n), tr ? 1 : 0, 0, 1.0, 0.0}},
                   s);
    }
  }
  if (e.k == 0 || !with_update) return;
  double* t = e.scratch_for(s).ws2(size_t(e.k * nrhs), s);
  if (!tr) {
    // out += L (R v)   (els.cpp:184); L is reconstructed as the update factor
    gemm_batched({{e.R.get(), v, t, int(e.k), int(nrhs), int(n), int(e.k), int(n), int(e.k), 0, 0, 1.0, 0.0}}, s);
    gemm_batched({{e.L->get(), t, out, int(n), int(nrhs), int(e.k), int(n), int(e.k), int(n), 0, 0, 1.0, 1.0}}, s);
  } else {
    // out += R^T (L^T v)   (els.cpp:191)
    gemm_batched({{e.L->get(), v, t, int(e.k), int(nrhs), int(n), int(n), int(n), int(e.k), 1, 0, 1.0, 0.0}}, s);
    gemm_batched({{e.R.get(), t, out, int(n), int(nrhs), int(e.k), int(e.k), int(e.k), int(n), 1, 0, 1.0, 1.0}}, s);
  }
}

void els_solve_ext_device(Els& e, const double* g_ext, double* y, i64 nrhs, cudaStream_t s) {
  const i64 n = e.n_ext(), k = e.k;
  atilde_solve(e, g_ext, n, y, n, nrhs, s);
  if (k == 0) return;
  // y -= X W^{-1} (R y)   (els.cpp:150)
  double* t = e.scratch_for(s).ws2(size_t(2 * k * nrhs), s);
  double* u = t + k * nrhs;
  gemm_batched({{e.R.get(), y, t, int(k), int(nrhs), int(n), int(k), int(n), int(k), 0, 0, 1.0, 0.0}}, s);
  gemm_batched({{e.Winv.get(), t, u, int(k), int(nrhs), int(k), int(k), int(k), int(k), 0, 0, 1.0, 0.0}}, s);
  gemm_batched({{e.X.get(), u, y, int(n), int(nrhs), int(k), int(n), int(k), int(n), 0, 0, -1.0, 1.0}}, s);
}

void els_atilde_solve(Els& e, const double* v, double* out, i64 nrhs, cudaStream_t s, bool tr) {
  atilde_solve(e, v, e.n_ext(), out, e.n_ext(), nrhs, s, tr);
}

void els_solve_ext_t_device(Els& e, const double* g_ext, double* y, i64 nrhs, cudaStream_t s) {
  const i64 n = e.n_ext(), k = e.k;
  if (k == 0) {
    atilde_solve(e, g_ext, n, y, n, nrhs, s, true);
    return;
  }
  // z = g - R^T W^{-T} (X^T g);  y = Atilde^{-T} z   (els.cpp:157-162)
  double* t = e.scratch_for(s).ws2(size_t(2 * k * nrhs), s);
  double* u = t + k * nrhs;
  DevBuf<double> z(static_cast<size_t>(n * nrhs));
  SBX_CUDA(cudaMemcpyAsync(z.get(), g_ext, size_t(n * nrhs) * 8, cudaMemcpyDeviceToDevice, s));
  gemm_batched({{e.X.get(), g_ext, t, int(k), int(nrhs), int(n), int(n), int(n), int(k), 1, 0, 1.0, 0.0}}, s);
  gemm_batched({{e.Winv.get(), t, u, int(k), int(nrhs), int(k), int(k), int(k), int(k), 1, 0, 1.0, 0.0}}, s);
  gemm_batched({{e.R.get(), u, z.get(), int(n), int(nrhs), int(k), int(k), int(k), int(n), 1, 0, -1.0, 1.0}}, s);
  atilde_solve(e, z.get(), n, y, n, nrhs, s, true);
}

void els_solve(Els& e, const double* g, i64 ldg, i64 nrhs, double* y, i64 ldy, bool raw, bool dev,
               cudaStream_t s, bool tr) {
  require(raw || !tr, "els_solve: the transpose solve is defined on the extended system (els_solve_raw_t)");
  const i64 n = e.n_ext();
  const i64 rows_in = raw ? n : e.n_k + e.n_p;
  require(ldg >= rows_in && ldy >= rows_in, "els_solve: leading dimension too small");
  if (nrhs == 0) return;
  if (!tr) g_hint_solve_cols.store(nrhs, std::memory_order_relaxed);
  double* gx = e.scratch_for(s).ws(size_t(2 * n * nrhs), s);
  double* yx = gx + n * nrhs;
  const i64 nkc = e.n_k + e.n_c;
  // g_ext = (g_k, 0, g_p)  (els.cpp:167-169)
  if (raw) {
    if (dev)
      SBX_CUDA(cudaMemcpy2DAsync(gx, size_t(n) * 8, g, size_t(ldg) * 8, size_t(n) * 8, size_t(nrhs),
                                 cudaMemcpyDeviceToDevice, s));
    else
      SBX_CUDA(cudaMemcpy2DAsync(gx, size_t(n) * 8, g, size_t(ldg) * 8, size_t(n) * 8, size_t(nrhs),
                                 cudaMemcpyHostToDevice, s));
  } else {
    const auto kind = dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    SBX_CUDA(cudaMemset2DAsync(gx + e.n_k, size_t(n) * 8, 0, size_t(e.n_c) * 8, size_t(nrhs), s));
    if (e.n_k)
      SBX_CUDA(cudaMemcpy2DAsync(gx, size_t(n) * 8, g, size_t(ldg) * 8, size_t(e.n_k) * 8, size_t(nrhs),
                                 kind, s));
    if (e.n_p)
      SBX_CUDA(cudaMemcpy2DAsync(gx + nkc, size_t(n) * 8, g + e.n_k, size_t(ldg) * 8, size_t(e.n_p) * 8,
                                 size_t(nrhs), kind, s));
  }
  if (tr)
    els_solve_ext_t_device(e, gx, yx, nrhs, s);
  else
    els_solve_ext_device(e, gx, yx, nrhs, s);
  const auto kind = dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  if (raw) {
    SBX_CUDA(cudaMemcpy2DAsync(y, size_t(ldy) * 8, yx, size_t(n) * 8, size_t(n) * 8, size_t(nrhs), kind, s));
  } else {  // drop the dummy (cut) block
    if (e.n_k)
      SBX_CUDA(cudaMemcpy2DAsync(y, size_t(ldy) * 8, yx, size_t(n) * 8, size_t(e.n_k) * 8, size_t(nrhs),
                                 kind, s));
    if (e.n_p)
      SBX_CUDA(cudaMemcpy2DAsync(y + e.n_k, size_t(ldy) * 8, yx + nkc, size_t(n) * 8, size_t(e.n_p) * 8,
                                 size_t(nrhs), kind, s));
  }
  e.scratch_for(s).mark.record(s);
  if (!dev) SBX_CUDA(cudaStreamSynchronize(s));
}

void els_density_on_refined(const Els& e, const double* tau_n, double* out) {
  // els.cpp:195-203 (host scatter of a host vector)
  for (i64 i = 0; i < 2 * e.n_new; ++i) out[i] = 0.0;
  for (i64 i = 0; i < e.n_k; ++i) out[e.kept_new_s[size_t(i)]] = tau_n[i];
  for (i64 i = 0; i < e.n_p; ++i) out[e.added_s[size_t(i)]] = tau_n[e.n_k + i];
}

void els_download_xw(const Els& e, double* X, double* W, cudaStream_t s) {
  const i64 k = e.k, n = e.n_ext();
  if (k == 0) return;
  if (X) e.X.download(X, size_t(n * k), s);
  if (W) e.Wmat.download(W, size_t(k * k), s);
  SBX_CUDA(cudaStreamSynchronize(s));
}

}  // namespace sbx
