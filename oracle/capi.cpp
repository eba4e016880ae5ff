// ORACLE — TEST INFRASTRUCTURE ONLY (see orc.hpp).
// Flat C entry points so the Python test-suite / bench cpu_baseline can
// drive the restatement through ctypes.  Status codes follow the product's
// C-ABI (include/sbx.h): 0 ok, 1 invalid argument, 3 geometry, 4 singular,
// 5 proxy violation, 7 other runtime error.
#include <cstring>
#include <exception>
#include <memory>
#include <string>

#include "orc.hpp"

using namespace orc;

namespace {
thread_local std::string g_err;

struct GeomH {
  std::shared_ptr<const Discretization> d;
};
struct PlanH {
  RefinementPlan p;
};
struct AsmH {
  std::shared_ptr<const Assembler> a;
};
struct HbsH {
  std::shared_ptr<HbsOperator> h;
};
struct UpdH {
  LowRankUpdate u;
};
struct ElsH {
  std::unique_ptr<ElsSolver> s;
};

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const GeometryError& e) {
    g_err = e.what();
    return 3;
  } catch (const SingularMatrixError& e) {
    g_err = e.what();
    return 4;
  } catch (const ProxyViolationError& e) {
    g_err = e.what();
    return 5;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 7;
  }
}

Mat from_ptr(const double* p, Index r, Index c) {
  Mat m(r, c);
  if (r * c != 0) std::memcpy(m.a.data(), p, size_t(8 * r * c));
  return m;
}
void to_ptr(const Mat& m, double* p) {
  if (m.size()) std::memcpy(p, m.a.data(), size_t(8 * m.size()));
}
CurveParams curve_params(int kind, double cx, double cy, double scale, int prongs, double amp,
                         double aspect, int flip) {
  CurveParams cp;
  cp.kind = CurveKind(kind);
  cp.center = {cx, cy};
  cp.scale = scale;
  cp.n_prongs = prongs;
  cp.amplitude = amp;
  cp.aspect = aspect;
  cp.flip_normal = flip != 0;
  return cp;
}
}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

int orc_geom_create(int kind, double cx, double cy, double scale, int prongs, double amp,
                    double aspect, int n_panels, int q, void** out) {
  return guard([&] {
    Curve c(curve_params(kind, cx, cy, scale, prongs, amp, aspect, 0));
    *out = new GeomH{std::make_shared<Discretization>(panelize(c, n_panels, q))};
  });
}

// Any curve kind with its coefficient lists (Fourier / Channel).
int orc_geom_create_curve(int kind, double cx, double cy, double scale, int prongs, double amp, double aspect,
                          int n_cos, const double* cos_coef, int n_sin, const double* sin_coef, int n_panels, int q,
                          void** out) {
  return guard([&] {
    CurveParams cp = curve_params(kind, cx, cy, scale, prongs, amp, aspect, 0);
    cp.cos_coef.assign(cos_coef, cos_coef + n_cos);
    cp.sin_coef.assign(sin_coef, sin_coef + n_sin);
    Curve c(cp);
    *out = new GeomH{std::make_shared<Discretization>(panelize(c, n_panels, q))};
  });
}

// holes: per hole (cx, cy, radius, n_panels, q) as doubles.
int orc_geom_add_holes(void* wall, int nh, const double* holes, void** out_geom, void** out_plan) {
  return guard([&] {
    std::vector<HoleSpec> hs;
    for (int i = 0; i < nh; ++i) {
      HoleSpec h;
      h.curve = curve_params(0, holes[5 * i], holes[5 * i + 1], holes[5 * i + 2], 0, 0, 1, 1);
      h.n_panels = int(holes[5 * i + 3]);
      h.q = int(holes[5 * i + 4]);
      hs.push_back(h);
    }
    auto [d, p] = add_holes(*static_cast<GeomH*>(wall)->d, hs);
    *out_geom = new GeomH{std::make_shared<Discretization>(std::move(d))};
    *out_plan = new PlanH{std::move(p)};
  });
}

void orc_geom_free(void* g) { delete static_cast<GeomH*>(g); }
void orc_plan_free(void* p) { delete static_cast<PlanH*>(p); }

int orc_geom_info(void* g, std::int64_t* n_nodes, std::int64_t* n_panels,
                  std::int64_t* n_components) {
  const auto& d = *static_cast<GeomH*>(g)->d;
  *n_nodes = d.n_nodes();
  *n_panels = d.n_panels();
  *n_components = Index(d.components.size());
  return 0;
}

// out: 9 arrays of n_nodes doubles (x, y, nx, ny, tx, ty, w, curvature, param)
// and panel_of (int64).
int orc_geom_nodes(void* g, double* out9, std::int64_t* panel_of) {
  const auto& d = *static_cast<GeomH*>(g)->d;
  const Index n = d.n_nodes();
  for (Index i = 0; i < n; ++i) {
    size_t s = size_t(i);
    out9[0 * n + i] = d.x[s].x;
    out9[1 * n + i] = d.x[s].y;
    out9[2 * n + i] = d.normal[s].x;
    out9[3 * n + i] = d.normal[s].y;
    out9[4 * n + i] = d.tangent[s].x;
    out9[5 * n + i] = d.tangent[s].y;
    out9[6 * n + i] = d.w[s];
    out9[7 * n + i] = d.curvature[s];
    out9[8 * n + i] = d.param[s];
    panel_of[i] = d.panel_of[s];
  }
  return 0;
}

std::int64_t orc_panels_near_point(void* g, double px, double py, double radius,
                                   std::int64_t* out, std::int64_t cap) {
  auto v = panels_near_point(*static_cast<GeomH*>(g)->d, {px, py}, radius);
  for (size_t i = 0; i < v.size() && Index(i) < cap; ++i) out[i] = v[i];
  return Index(v.size());
}

int orc_refine(void* g, const std::int64_t* panels, std::int64_t n, int m, void** out_geom,
               void** out_plan) {
  return guard([&] {
    std::vector<Index> ids(panels, panels + n);
    auto [d, p] = refine(*static_cast<GeomH*>(g)->d, ids, m);
    *out_geom = new GeomH{std::make_shared<Discretization>(std::move(d))};
    *out_plan = new PlanH{std::move(p)};
  });
}

int orc_coarsen(void* g, void* plan, void** out_geom) {
  return guard([&] {
    *out_geom = new GeomH{std::make_shared<Discretization>(
        coarsen(*static_cast<GeomH*>(g)->d, static_cast<PlanH*>(plan)->p))};
  });
}

int orc_plan_sizes(void* plan, std::int64_t* nk, std::int64_t* nc, std::int64_t* np) {
  const auto& p = static_cast<PlanH*>(plan)->p;
  *nk = p.n_k();
  *nc = p.n_c();
  *np = p.n_p();
  return 0;
}

int orc_plan_maps(void* plan, std::int64_t* kept_old, std::int64_t* kept_new,
                  std::int64_t* cut_old, std::int64_t* added_new) {
  const auto& p = static_cast<PlanH*>(plan)->p;
  std::copy(p.kept_old.begin(), p.kept_old.end(), kept_old);
  std::copy(p.kept_new.begin(), p.kept_new.end(), kept_new);
  std::copy(p.cut_old.begin(), p.cut_old.end(), cut_old);
  std::copy(p.added_new.begin(), p.added_new.end(), added_new);
  return 0;
}

int orc_asm_create(void* g, int form, double mu, void** out) {
  return guard([&] {
    Formulation f{FormulationKind(form), mu};
    *out = new AsmH{std::make_shared<Assembler>(static_cast<GeomH*>(g)->d, f)};
  });
}
void orc_asm_free(void* a) { delete static_cast<AsmH*>(a); }

int orc_asm_submatrix(void* a, const std::int64_t* rows, std::int64_t nr,
                      const std::int64_t* cols, std::int64_t nc, double* out) {
  return guard([&] {
    std::vector<Index> r(rows, rows + nr), c(cols, cols + nc);
    to_ptr(static_cast<AsmH*>(a)->a->submatrix(r, c), out);
  });
}

int orc_hbs_compress(void* a, const std::int64_t* subset, std::int64_t nsub, double eps,
                     std::int64_t leaf, void** out) {
  return guard([&] {
    HbsOptions o;
    o.eps = eps;
    o.leaf_nodes = leaf;
    auto ap = static_cast<AsmH*>(a)->a;
    HbsSource src = subset ? make_hbs_source_subset(ap, std::vector<Index>(subset, subset + nsub))
                           : make_hbs_source(ap);
    *out = new HbsH{std::make_shared<HbsOperator>(hbs_compress(src, o))};
  });
}
void orc_hbs_free(void* h) { delete static_cast<HbsH*>(h); }

int orc_hbs_invert(void* h) {
  return guard([&] { hbs_invert(*static_cast<HbsH*>(h)->h); });
}

// mode: 0 solve, 1 solve_t, 2 apply, 3 apply_t
int orc_hbs_sweep(void* h, int mode, const double* b, std::int64_t nrhs, double* out) {
  return guard([&] {
    const auto& op = *static_cast<HbsH*>(h)->h;
    Mat bm = from_ptr(b, op.n, nrhs);
    Mat r = mode == 0 ? hbs_solve(op, bm)
                      : mode == 1 ? hbs_solve_t(op, bm) : mode == 2 ? hbs_apply(op, bm) : hbs_apply_t(op, bm);
    to_ptr(r, out);
  });
}

int orc_hbs_save(void* h, const char* path) {
  return guard([&] { hbs_save(*static_cast<HbsH*>(h)->h, path); });
}
int orc_hbs_load(const char* path, void** out) {
  return guard([&] { *out = new HbsH{std::make_shared<HbsOperator>(hbs_load(path))}; });
}

// info[0..7]: n, node count, total skeleton, max_block_drawn, has_inverse,
// solve-factor doubles (sum |f|+|g|+|e| non-root + |root_g|), max depth, max k
int orc_hbs_info(void* h, std::int64_t* info) {
  const auto& op = *static_cast<HbsH*>(h)->h;
  Index fd = op.root_g.size(), md = 0, mk = 0;
  for (size_t i = 1; i < op.nodes.size(); ++i)
    fd += op.nodes[i].f.size() + op.nodes[i].g.size() + op.nodes[i].e.size();
  for (const auto& nd : op.nodes) {
    md = std::max<Index>(md, nd.depth);
    mk = std::max<Index>(mk, nd.k);
  }
  info[0] = op.n;
  info[1] = Index(op.nodes.size());
  info[2] = op.total_skeleton();
  info[3] = op.max_block_drawn;
  info[4] = op.has_inverse ? 1 : 0;
  info[5] = fd;
  info[6] = md;
  info[7] = mk;
  return 0;
}

std::int64_t orc_hbs_node_k(void* h, std::int64_t* ks, std::int64_t cap) {
  const auto& op = *static_cast<HbsH*>(h)->h;
  for (size_t i = 0; i < op.nodes.size() && Index(i) < cap; ++i) ks[i] = op.nodes[i].k;
  return Index(op.nodes.size());
}

// ID entry points: P buffer must hold m*min(m,n) doubles.
int orc_row_id(const double* w, std::int64_t m, std::int64_t n, double eps, std::int64_t forced,
               std::int64_t* k, std::int64_t* J, double* P) {
  return guard([&] {
    Mat W = from_ptr(w, m, n);
    IdResult id = forced >= 0 ? row_id_rank(W, forced) : row_id(W, eps);
    *k = id.k;
    std::copy(id.J.begin(), id.J.end(), J);
    to_ptr(id.P, P);
  });
}

int orc_randomized_row_id(const double* w, std::int64_t m, std::int64_t n, double eps,
                          std::uint64_t seed, std::int64_t* k, std::int64_t* J, double* P) {
  return guard([&] {
    IdResult id = randomized_row_id(from_ptr(w, m, n), eps, seed);
    *k = id.k;
    std::copy(id.J.begin(), id.J.end(), J);
    to_ptr(id.P, P);
  });
}

int orc_gaussian_sketch(std::int64_t n, std::int64_t l, std::uint64_t seed, double* out) {
  to_ptr(gaussian_sketch(n, l, seed), out);
  return 0;
}

int orc_update_compress(void* old_a, void* new_a, void* plan, double eps, std::uint64_t seed,
                        void** out) {
  return guard([&] {
    BlockSource src(static_cast<AsmH*>(old_a)->a, static_cast<AsmH*>(new_a)->a,
                    static_cast<PlanH*>(plan)->p);
    ProxyGeometry pg = make_proxy_geometry(src.new_oracle().disc(), src.plan());
    CompressOptions o;
    o.seed = seed;
    *out = new UpdH{compress_update(src, pg, eps, o)};
  });
}
void orc_update_free(void* u) { delete static_cast<UpdH*>(u); }

// info: k, k1, kc.k, kp.k, pk.k, n_ext, nk2, nc2, np2
int orc_update_info(void* u, std::int64_t* info) {
  const auto& x = static_cast<UpdH*>(u)->u;
  Index v[9] = {x.k, x.k1, x.kc.k, x.kp.k, x.pk.k, x.n_ext(), x.nk2, x.nc2, x.np2};
  std::copy(v, v + 9, info);
  return 0;
}

// which: 0 L, 1 R, 2 L1, 3 R1
int orc_update_factor(void* u, int which, double* out) {
  const auto& x = static_cast<UpdH*>(u)->u;
  to_ptr(which == 0 ? x.L : which == 1 ? x.R : which == 2 ? x.L1 : x.R1, out);
  return 0;
}

int orc_update_skeleton(void* u, std::int64_t* out) {
  const auto& x = static_cast<UpdH*>(u)->u;
  std::copy(x.skeleton.begin(), x.skeleton.end(), out);
  return 0;
}

// Install externally supplied L (n_ext x k) and R (k x n_ext).
int orc_update_set(void* u, const double* L, const double* R, std::int64_t n_ext, std::int64_t k) {
  return guard([&] {
    auto& x = static_cast<UpdH*>(u)->u;
    x.L = from_ptr(L, n_ext, k);
    x.R = from_ptr(R, k, n_ext);
    x.k = k;
  });
}

// nystrom.cpp:450-477 interchange (column-major host buffers on this side)
int orc_dump_matrix(const char* path, const double* m, std::int64_t rows, std::int64_t cols) {
  return guard([&] { dump_matrix(path, from_ptr(m, rows, cols)); });
}

int orc_load_matrix_dims(const char* path, std::int64_t* rows, std::int64_t* cols) {
  return guard([&] {
    const Mat m = load_matrix(path);
    *rows = m.r;
    *cols = m.c;
  });
}

int orc_load_matrix(const char* path, double* out) {
  return guard([&] { to_ptr(load_matrix(path), out); });
}

int orc_block_eval_full(void* old_a, void* new_a, void* plan, int block, double* out) {
  return guard([&] {
    BlockSource src(static_cast<AsmH*>(old_a)->a, static_cast<AsmH*>(new_a)->a,
                    static_cast<PlanH*>(plan)->p);
    to_ptr(src.eval_full(BlockName(block)), out);
  });
}

int orc_els_build(void* hbs, void* old_a, void* new_a, void* plan, void* upd, void** out) {
  return guard([&] {
    BlockSource src(static_cast<AsmH*>(old_a)->a, static_cast<AsmH*>(new_a)->a,
                    static_cast<PlanH*>(plan)->p);
    *out = new ElsH{els_build(static_cast<HbsH*>(hbs)->h, src, static_cast<PlanH*>(plan)->p,
                              static_cast<UpdH*>(upd)->u)};
  });
}
void orc_els_free(void* e) { delete static_cast<ElsH*>(e); }

// info: n_k, n_c, n_p (scalars), k, app is hbs (1) or dense (0)
int orc_els_info(void* e, std::int64_t* info) {
  const auto& s = *static_cast<ElsH*>(e)->s;
  info[0] = s.n_k;
  info[1] = s.n_c;
  info[2] = s.n_p;
  info[3] = s.update.k;
  info[4] = s.app_h ? 1 : 0;
  return 0;
}

// mode 0: els_solve (g_n has n_k+n_p rows), 1: els_solve_raw (n_ext rows),
// 2: raw transpose, 3: forward apply (n_ext rows)
int orc_els_solve(void* e, int mode, const double* g, std::int64_t nrhs, double* out) {
  return guard([&] {
    const auto& s = *static_cast<ElsH*>(e)->s;
    if (mode == 0) {
      to_ptr(els_solve(s, from_ptr(g, s.n_k + s.n_p, nrhs)), out);
    } else {
      Mat gm = from_ptr(g, s.n_ext(), nrhs);
      to_ptr(mode == 1 ? els_solve_raw(s, gm) : mode == 2 ? els_solve_raw_t(s, gm)
                                                          : els_apply_forward(s, gm),
             out);
    }
  });
}

int orc_els_xw(void* e, double* X, double* W) {
  const auto& s = *static_cast<ElsH*>(e)->s;
  if (X) to_ptr(s.x, X);
  if (W) to_ptr(s.w, W);
  return 0;
}

// src: nsrc x (x, y, fx, fy)
int orc_boundary_data(void* g, std::int64_t nsrc, const double* src, double mu, double* out) {
  return guard([&] {
    std::vector<StokesletSource> s;
    for (Index i = 0; i < nsrc; ++i)
      s.push_back({{src[4 * i], src[4 * i + 1]}, {src[4 * i + 2], src[4 * i + 3]}});
    auto v = boundary_data(*static_cast<GeomH*>(g)->d, s, mu);
    std::copy(v.begin(), v.end(), out);
  });
}

int orc_field_velocity(std::int64_t nsrc, const double* src, double mu, std::int64_t nt,
                       const double* targets, double* out) {
  return guard([&] {
    std::vector<StokesletSource> s;
    for (Index i = 0; i < nsrc; ++i)
      s.push_back({{src[4 * i], src[4 * i + 1]}, {src[4 * i + 2], src[4 * i + 3]}});
    for (Index t = 0; t < nt; ++t) {
      V2 u = field_velocity(s, mu, {targets[2 * t], targets[2 * t + 1]});
      out[2 * t] = u.x;
      out[2 * t + 1] = u.y;
    }
  });
}

int orc_evaluate_velocity(void* g, int form, double mu, const double* tau, std::int64_t nt,
                          const double* targets, double* out) {
  return guard([&] {
    const auto& d = *static_cast<GeomH*>(g)->d;
    std::vector<double> t(tau, tau + d.n_unknowns());
    std::vector<V2> tg;
    for (Index i = 0; i < nt; ++i) tg.push_back({targets[2 * i], targets[2 * i + 1]});
    auto v = evaluate_velocity(d, Formulation{FormulationKind(form), mu}, t, tg);
    for (Index i = 0; i < nt; ++i) {
      out[2 * i] = v[size_t(i)].x;
      out[2 * i + 1] = v[size_t(i)].y;
    }
  });
}

int orc_log_rule_weights(int q, double u, double* out) {
  return guard([&] {
    auto w = log_rule_weights(q, u);
    std::copy(w.begin(), w.end(), out);
  });
}

int orc_gauss_rule(int n, double* nodes, double* weights) {
  return guard([&] {
    const auto& g = gauss_rule(n);
    std::copy(g.nodes.begin(), g.nodes.end(), nodes);
    std::copy(g.weights.begin(), g.weights.end(), weights);
  });
}

}  // extern "C"
