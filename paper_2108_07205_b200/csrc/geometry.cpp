// Wall discretization, refine/coarsen/add_holes (reference geometry.cpp).
// Node data must agree bit for bit with the reference's so kept nodes of a
// refinement and the entry oracle match exactly (test_geometry.cpp:147-187);
// the formulas below therefore keep the reference's evaluation order.
#include "geometry.hpp"

#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <set>

namespace sbx {

namespace {

// Legendre P_n and P_n' in extended precision (gauss.cpp:12-23).
void legendre_pn(int n, long double x, long double& p, long double& dp) {
  long double p0 = 1.0L, p1 = x;
  if (n == 0) {
    p = 1.0L;
    dp = 0.0L;
    return;
  }
  for (int k = 2; k <= n; ++k) {
    const long double p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
    p0 = p1;
    p1 = p2;
  }
  p = p1;
  dp = n * (x * p1 - p0) / (x * x - 1.0L);
}

GaussTable make_gauss(int n) {  // Newton on P_n from Chebyshev-like guesses (gauss.cpp:25-47)
  GaussTable g;
  g.x.assign(size_t(n), 0.0);
  g.w.assign(size_t(n), 0.0);
  for (int i = 0; i < (n + 1) / 2; ++i) {
    long double x = std::cos(kPi * (i + 0.75L) / (n + 0.5L));
    long double p, dp;
    for (int it = 0; it < 100; ++it) {
      legendre_pn(n, x, p, dp);
      const long double dx = p / dp;
      x -= dx;
      if (std::fabs(double(dx)) < 1e-19) break;
    }
    legendre_pn(n, x, p, dp);
    const long double w = 2.0L / ((1.0L - x * x) * dp * dp);
    g.x[size_t(n - 1 - i)] = double(x);
    g.x[size_t(i)] = double(-x);
    g.w[size_t(n - 1 - i)] = double(w);
    g.w[size_t(i)] = double(w);
  }
  if (n % 2 == 1) g.x[size_t(n / 2)] = 0.0;
  return g;
}

void check_curve(const sbx_curve& p) {  // geometry.cpp:11-34
  if (p.scale <= 0) throw Error(3, "curve scale must be positive");
  if (p.kind == SBX_STAR) {
    if (p.n_prongs < 2) throw Error(3, "star needs at least 2 prongs");
    if (std::fabs(p.amplitude) >= 1.0) throw Error(3, "star amplitude must keep radius positive");
  }
  if (p.kind == SBX_ELLIPSE && p.aspect <= 0) throw Error(3, "ellipse aspect must be positive");
  if (p.kind == SBX_CHANNEL) {
    if (p.n_prongs < 1) throw Error(3, "channel needs at least one wave period");
    if (std::fabs(p.amplitude) >= 1.0) throw Error(3, "channel amplitude must keep the width positive");
    if (p.aspect <= 0) throw Error(3, "channel length must be positive");
    if (p.n_cos != 40) throw Error(3, "channel needs its two degree-9 cap polynomials (40 coefficients)");
    if (p.n_sin != 2 || !(p.sin_coef[0] > 0.0 && p.sin_coef[1] > 0.0 && 2.0 * p.sin_coef[0] + p.sin_coef[1] < 1.0))
      throw Error(3, "channel parameter fractions must be positive and sum below 1");
  }
  if (p.kind < 0 || p.kind > 4) throw Error(1, "unknown curve kind");
  if (p.n_cos < 0 || p.n_cos > 64 || p.n_sin < 0 || p.n_sin > 64)
    throw Error(1, "fourier coefficient count out of range");
}

}  // namespace

const GaussTable& gauss_table(int q) {
  static std::map<int, GaussTable> cache;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(q);
  if (it == cache.end()) it = cache.emplace(q, make_gauss(q)).first;
  return it->second;
}

void CurveDef::eval(double t, double& px, double& py, double& dx, double& dy, double& ddx,
                    double& ddy) const {
  if (p.kind == SBX_CHANNEL) {
    channel_eval(t, px, py, dx, dy, ddx, ddy);
    return;
  }
  const double c = std::cos(t), s = std::sin(t);
  if (p.kind == SBX_ELLIPSE) {
    px = p.center_x + p.scale * c;
    py = p.center_y + p.scale * (p.aspect * s);
    dx = p.scale * (-s);
    dy = p.scale * (p.aspect * c);
    ddx = p.scale * (-c);
    ddy = p.scale * (-p.aspect * s);
    return;
  }
  double r = 1.0, dr = 0.0, ddr = 0.0;  // radial profile (geometry.cpp:36-69)
  if (p.kind == SBX_STAR) {
    const double cn = std::cos(p.n_prongs * t), sn = std::sin(p.n_prongs * t);
    const double n = p.n_prongs;
    r = 1.0 + p.amplitude * cn;
    dr = -p.amplitude * n * sn;
    ddr = -p.amplitude * n * n * cn;
  } else if (p.kind == SBX_FOURIER) {
    for (int j = 0; j < p.n_cos; ++j) {
      const double k = double(j + 1);
      r += p.cos_coef[j] * std::cos(k * t);
      dr -= p.cos_coef[j] * k * std::sin(k * t);
      ddr -= p.cos_coef[j] * k * k * std::cos(k * t);
    }
    for (int j = 0; j < p.n_sin; ++j) {
      const double k = double(j + 1);
      r += p.sin_coef[j] * std::sin(k * t);
      dr += p.sin_coef[j] * k * std::cos(k * t);
      ddr -= p.sin_coef[j] * k * k * std::sin(k * t);
    }
  }
  const double sr = p.scale * r;
  px = p.center_x + sr * c;
  py = p.center_y + sr * s;
  dx = p.scale * (dr * c - r * s);
  dy = p.scale * (dr * s + r * c);
  ddx = p.scale * (ddr * c - 2 * dr * s - r * c);
  ddy = p.scale * (ddr * s + 2 * dr * c - r * s);
}

// The closed wavy channel (sbx.h SBX_CHANNEL), piecewise in t; the same
// operations as the oracle's Curve::channel (oracle/geom.cpp), so nodes agree
// bit for bit.
void CurveDef::channel_eval(double t, double& px, double& py, double& dx, double& dy, double& ddx,
                            double& ddy) const {
  const double F = 2.0 * kPi, fw = p.sin_coef[0], fr = p.sin_coef[1], fl = 1.0 - 2.0 * fw - fr;
  const double h = p.scale, Lam = p.aspect, a = p.amplitude, k = 2.0 * kPi * double(p.n_prongs) / Lam;
  const double T0 = F * fw, T1 = T0 + F * fr, T2 = T1 + F * fw;
  // scaled coordinates (X, Y), derivatives in t
  double X, Y, X1, Y1, X2, Y2;
  auto cap = [&](const double* cx, const double* cy, double u, double ud) {  // degree-9 polynomial piece
    X = 0.0, Y = 0.0, X1 = 0.0, Y1 = 0.0, X2 = 0.0, Y2 = 0.0;
    for (int j = 9; j >= 0; --j) {  // Horner for the value and both derivatives
      X2 = X2 * u + 2.0 * X1;
      Y2 = Y2 * u + 2.0 * Y1;
      X1 = X1 * u + X;
      Y1 = Y1 * u + Y;
      X = X * u + cx[j];
      Y = Y * u + cy[j];
    }
    X1 *= ud;
    Y1 *= ud;
    X2 *= ud * ud;
    Y2 *= ud * ud;
  };
  if (t < T0 || t >= T2 + F * fl) {  // bottom wall, left to right (t >= 2 pi wraps)
    const double tt = t < T0 ? t : t - F;
    const double xd = Lam / (F * fw);
    X = tt * xd;
    const double sn = std::sin(k * X), cs = std::cos(k * X);
    Y = -(1.0 + a * sn);
    X1 = xd;
    Y1 = -a * k * cs * xd;
    X2 = 0.0;
    Y2 = a * k * k * sn * xd * xd;
  } else if (t < T1) {  // right cap, bottom to top
    cap(p.cos_coef, p.cos_coef + 10, (t - T0) / (F * fr), 1.0 / (F * fr));
  } else if (t < T2) {  // top wall, right to left
    const double xd = -Lam / (F * fw);
    X = Lam + (t - T1) * xd;
    const double sn = std::sin(k * X), cs = std::cos(k * X);
    Y = 1.0 + a * sn;
    X1 = xd;
    Y1 = a * k * cs * xd;
    X2 = 0.0;
    Y2 = -a * k * k * sn * xd * xd;
  } else {  // left cap, top to bottom
    cap(p.cos_coef + 20, p.cos_coef + 30, (t - T2) / (F * fl), 1.0 / (F * fl));
  }
  px = p.center_x + h * X;
  py = p.center_y + h * Y;
  dx = h * X1;
  dy = h * Y1;
  ddx = h * X2;
  ddy = h * Y2;
}

namespace {

void curve_checks(const CurveDef& cv) {  // positive radius / nonvanishing speed (geometry.cpp:20-33)
  double mn = 1e300, mx = 0;
  for (int i = 0; i < 2048; ++i) {
    const double t = 2 * kPi * i / 2048.0;
    double px, py, dx, dy, ddx, ddy;
    cv.eval(t, px, py, dx, dy, ddx, ddy);
    if (cv.p.kind != SBX_ELLIPSE && cv.p.kind != SBX_CHANNEL) {
      const double rr = std::hypot(px - cv.p.center_x, py - cv.p.center_y) / cv.p.scale;
      if (rr <= 1e-6) throw Error(3, "curve radius vanishes");
    }
    const double sp = std::sqrt(dx * dx + dy * dy);
    mn = std::min(mn, sp);
    mx = std::max(mx, sp);
  }
  if (mn <= 1e-9 * mx) throw Error(3, "curve speed vanishes");
}

bool seg_cross(double ax, double ay, double bx, double by, double cx, double cy, double dx,
               double dy) {
  auto cr = [](double ux, double uy, double vx, double vy) { return ux * vy - uy * vx; };
  const double d1 = cr(bx - ax, by - ay, cx - ax, cy - ay), d2 = cr(bx - ax, by - ay, dx - ax, dy - ay);
  const double d3 = cr(dx - cx, dy - cy, ax - cx, ay - cy), d4 = cr(dx - cx, dy - cy, bx - cx, by - cy);
  return ((d1 > 0) != (d2 > 0)) && ((d3 > 0) != (d4 > 0));
}

std::vector<std::pair<double, double>> polyline(const CurveDef& cv, int M) {
  std::vector<std::pair<double, double>> pts(static_cast<size_t>(M));
  for (int i = 0; i < M; ++i) {
    double px, py, a, b, c, d;
    cv.eval(2 * kPi * i / M, px, py, a, b, c, d);
    pts[size_t(i)] = {px, py};
  }
  return pts;
}

void check_simple(const CurveDef& cv) {  // geometry.cpp:136-147
  const int M = 512;
  auto p = polyline(cv, M);
  for (int i = 0; i < M; ++i)
    for (int j = i + 2; j < M; ++j) {
      if (i == 0 && j == M - 1) continue;
      const auto &a = p[size_t(i)], &b = p[size_t((i + 1) % M)], &c = p[size_t(j)],
                 &d = p[size_t((j + 1) % M)];
      if (seg_cross(a.first, a.second, b.first, b.second, c.first, c.second, d.first, d.second))
        throw Error(3, "curve self-intersects at sampling resolution");
    }
}

bool inside(const CurveDef& cv, double qx, double qy, int samples = 512) {  // geometry.cpp:419-432
  int crossings = 0;
  double ax, ay, t0, t1, t2, t3;
  cv.eval(0.0, ax, ay, t0, t1, t2, t3);
  for (int i = 1; i <= samples; ++i) {
    double bx, by;
    cv.eval(2 * kPi * i / samples, bx, by, t0, t1, t2, t3);
    if ((ay <= qy) != (by <= qy)) {
      const double xi = ax + (qy - ay) / (by - ay) * (bx - ax);
      if (xi > qx) ++crossings;
    }
    ax = bx;
    ay = by;
  }
  return crossings % 2 == 1;
}

// One Gauss node of panel pd appended to the node arrays (geometry.cpp:149-179).
inline void push_node(Geom& g, const Component& comp, const GaussTable& gt, const PanelDef& pd, double half,
                      int j, double sgn, i64 pid) {
  const double t = pd.a + half * (gt.x[size_t(j)] + 1.0);
  double px, py, dx, dy, ddx, ddy;
  comp.curve.eval(t, px, py, dx, dy, ddx, ddy);
  const double sp = std::sqrt(dx * dx + dy * dy);
  const double nn = std::sqrt(dy * dy + dx * dx);  // |(dy, -dx)|
  g.x.push_back(px);
  g.y.push_back(py);
  g.nx.push_back(sgn * (dy / nn));
  g.ny.push_back(sgn * (-dx / nn));
  g.tx.push_back(dx / sp);
  g.ty.push_back(dy / sp);
  g.w.push_back(gt.w[size_t(j)] * sp * half);
  g.kappa.push_back(sgn * ((dx * ddy - dy * ddx) / (sp * sp * sp)));
  g.t.push_back(t);
  g.panel_of.push_back(pid);
}

inline void reserve_nodes(Geom& g, size_t total) {
  for (auto* v : {&g.x, &g.y, &g.nx, &g.ny, &g.tx, &g.ty, &g.w, &g.kappa, &g.t}) v->reserve(total);
  g.panel_of.reserve(total);
}

void append_nodes(Geom& g, i64 ci) {  // geometry.cpp:149-179
  Component& comp = g.comps[size_t(ci)];
  const GaussTable& gt = gauss_table(comp.q);
  const int q = comp.q;
  const double sgn = comp.curve.p.flip_normal ? -1.0 : 1.0;
  reserve_nodes(g, size_t(g.n_nodes()) + comp.panels.size() * size_t(q));
  for (size_t pl = 0; pl < comp.panels.size(); ++pl) {
    const PanelDef& pd = comp.panels[pl];
    const i64 pid = i64(g.panels.size());
    g.panels.push_back({ci, i64(pl), pd.a, pd.b, pd.level, g.n_nodes(), q});
    const double half = 0.5 * (pd.b - pd.a);
    for (int j = 0; j < q; ++j) push_node(g, comp, gt, pd, half, j, sgn, pid);
  }
}

}  // namespace

double Geom::panel_arclength(i64 p) const {
  const PanelRow& pr = panels[size_t(p)];
  double s = 0;
  for (int j = 0; j < pr.q; ++j) s += w[size_t(pr.node_begin + j)];
  return s;
}

void Geom::upload(cudaStream_t s) {
  const i64 n = n_nodes();
  // staged through a per-thread pinned buffer (a pageable copy of the 8 N
  // doubles is a synchronous bounce through the driver's staging area)
  struct Pinned {
    void* p = nullptr;
    size_t bytes = 0;
    ~Pinned() {
      if (p) cudaFreeHost(p);
    }
  };
  static thread_local Pinned pin;
  const size_t need = size_t(8 * n) * sizeof(double) + size_t(n) * sizeof(int);
  if (pin.bytes < need) {
    if (pin.p) SBX_CUDA(cudaFreeHost(pin.p));
    pin.p = nullptr;
    SBX_CUDA(cudaMallocHost(&pin.p, need));
    pin.bytes = need;
  }
  double* h = static_cast<double*>(pin.p);
  const std::vector<double>* src[8] = {&x, &y, &nx, &ny, &w, &kappa, &tx, &ty};
  for (int a = 0; a < 8; ++a) std::copy(src[a]->begin(), src[a]->end(), h + a * n);
  int* cp = reinterpret_cast<int*>(h + 8 * n);
  for (i64 i = 0; i < n; ++i) cp[i] = int(component_of(i));
  dev.n = n;
  dev.buf.upload(h, size_t(8 * n), s);
  dev.comp.upload(cp, size_t(n), s);
  SBX_CUDA(cudaStreamSynchronize(s));  // the pinned buffer is reused by the next upload
}

std::vector<PanelDef> uniform_panels(int n_panels, int q) {  // geometry.cpp:112-125
  require(n_panels >= 4, "need at least 4 panels");
  require(q >= 4 && q <= 64, "nodes per panel out of range");
  std::vector<PanelDef> out(static_cast<size_t>(n_panels));
  double prev = 0.0;
  for (int i = 0; i < n_panels; ++i) {
    const double next = (i + 1 == n_panels) ? 2 * kPi : 2 * kPi * (i + 1) / n_panels;
    out[size_t(i)] = {prev, next, 0};
    prev = next;
  }
  return out;
}

std::unique_ptr<Geom> geom_panelize(const sbx_curve& c, int n_panels, int q) {
  return geom_build({c}, {uniform_panels(n_panels, q)}, {q}, {false});
}

std::unique_ptr<Geom> geom_build(const std::vector<sbx_curve>& curves,
                                 const std::vector<std::vector<PanelDef>>& meshes,
                                 const std::vector<int>& qs, const std::vector<bool>& holes) {
  require(!curves.empty() && curves.size() == meshes.size() && curves.size() == holes.size() &&
              qs.size() == curves.size(),
          "build_discretization: size mismatch");
  auto g = std::make_unique<Geom>();
  for (size_t i = 0; i < curves.size(); ++i) {
    check_curve(curves[i]);
    CurveDef cv{curves[i]};
    curve_checks(cv);
    check_simple(cv);
    g->comps.push_back({cv, meshes[i], qs[i], g->n_nodes(), i64(g->panels.size()), bool(holes[i])});
    append_nodes(*g, i64(i));
  }
  const size_t nc = g->comps.size();  // layout checks (geometry.cpp:239-268)
  const int S = 256;
  std::vector<std::vector<std::pair<double, double>>> poly(nc);
  std::vector<double> lox(nc, 1e300), loy(nc, 1e300), hix(nc, -1e300), hiy(nc, -1e300);
  for (size_t c = 0; c < nc; ++c) {
    poly[c] = polyline(g->comps[c].curve, S);
    for (auto& p : poly[c]) {
      lox[c] = std::min(lox[c], p.first);
      loy[c] = std::min(loy[c], p.second);
      hix[c] = std::max(hix[c], p.first);
      hiy[c] = std::max(hiy[c], p.second);
    }
  }
  for (size_t a = 0; a + 1 < nc; ++a)
    for (size_t b = a + 1; b < nc; ++b) {
      if (!(lox[a] <= hix[b] && lox[b] <= hix[a] && loy[a] <= hiy[b] && loy[b] <= hiy[a])) continue;
      for (int i = 0; i < S; ++i)
        for (int j = 0; j < S; ++j) {
          const auto &p0 = poly[a][size_t(i)], &p1 = poly[a][size_t((i + 1) % S)];
          const auto &q0 = poly[b][size_t(j)], &q1 = poly[b][size_t((j + 1) % S)];
          if (seg_cross(p0.first, p0.second, p1.first, p1.second, q0.first, q0.second, q1.first,
                        q1.second))
            throw Error(3, "components intersect");
        }
      const bool b_in_a = inside(g->comps[a].curve, poly[b][0].first, poly[b][0].second);
      const bool a_in_b = inside(g->comps[b].curve, poly[a][0].first, poly[a][0].second);
      const bool legal = !a_in_b && (!b_in_a || (a == 0 && !holes[0] && holes[b]));
      if (!legal) throw Error(3, "component nesting is not wall-plus-holes");
    }
  return g;
}

std::pair<std::unique_ptr<Geom>, std::unique_ptr<Plan>> geom_refine(const Geom& g,
                                                                    std::vector<i64> ids, int m) {
  // geometry.cpp:272-342
  require(m >= 2, "split factor must be at least 2");
  std::sort(ids.begin(), ids.end());
  ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
  require(!ids.empty(), "refine: empty panel list");
  const i64 np = i64(g.panels.size());
  for (i64 id : ids) require(id >= 0 && id < np, "refine: panel id out of range");
  std::vector<char> refined(static_cast<size_t>(np), 0);
  for (i64 id : ids) refined[size_t(id)] = 1;
  auto plan = std::make_unique<Plan>();
  plan->panel_ids = ids;
  plan->m = m;
  auto ng = std::make_unique<Geom>();
  // Unrefined panels keep their nodes bit for bit: runs of them are copied
  // from the old arrays in bulk; only the m sub-panels of a refined panel
  // evaluate the curve (this is the per-step path of a moving refinement).
  size_t total = 0;
  for (const auto& o : g.panels) total += size_t(o.q) * (refined[size_t(&o - g.panels.data())] ? size_t(m) : 1);
  reserve_nodes(*ng, total);
  ng->panels.reserve(g.panels.size() + ids.size() * size_t(m - 1));
  plan->kept_old.reserve(size_t(g.n_nodes()));
  plan->kept_new.reserve(size_t(g.n_nodes()));
  const std::vector<double>* src[9] = {&g.x, &g.y, &g.nx, &g.ny, &g.tx, &g.ty, &g.w, &g.kappa, &g.t};
  std::vector<double>* dst[9] = {&ng->x, &ng->y, &ng->nx, &ng->ny, &ng->tx, &ng->ty, &ng->w, &ng->kappa, &ng->t};
  for (size_t ci = 0; ci < g.comps.size(); ++ci) {
    const Component& comp = g.comps[ci];
    plan->old_panels.push_back(comp.panels);
    plan->old_q.push_back(comp.q);
    const GaussTable& gt = gauss_table(comp.q);
    const int q = comp.q;
    const double sgn = comp.curve.p.flip_normal ? -1.0 : 1.0;
    std::vector<PanelDef> mesh;
    mesh.reserve(comp.panels.size() + ids.size() * size_t(m - 1));
    const i64 node_offset = ng->n_nodes(), panel_offset = i64(ng->panels.size());
    i64 run_a = -1, run_b = -1;  // pending run of kept old nodes [run_a, run_b)
    auto flush = [&] {
      if (run_a < 0) return;
      for (int a = 0; a < 9; ++a) dst[a]->insert(dst[a]->end(), src[a]->begin() + run_a, src[a]->begin() + run_b);
      run_a = run_b = -1;
    };
    for (size_t pl = 0; pl < comp.panels.size(); ++pl) {
      const PanelDef& p = comp.panels[pl];
      const PanelRow& o = g.panels[size_t(comp.panel_offset + i64(pl))];
      if (refined[size_t(comp.panel_offset + i64(pl))]) {
        flush();
        for (int j = 0; j < o.q; ++j) plan->cut_old.push_back(o.node_begin + j);
        double prev = p.a;
        for (int sp = 1; sp <= m; ++sp) {
          const double next = (sp == m) ? p.b : p.a + (p.b - p.a) * sp / m;
          const PanelDef pd{prev, next, p.level + 1};
          const i64 pid = i64(ng->panels.size());
          ng->panels.push_back({i64(ci), i64(mesh.size()), pd.a, pd.b, pd.level, ng->n_nodes(), q});
          mesh.push_back(pd);
          const double half = 0.5 * (pd.b - pd.a);
          for (int j = 0; j < q; ++j) {
            plan->added_new.push_back(ng->n_nodes());
            push_node(*ng, comp, gt, pd, half, j, sgn, pid);
          }
          prev = next;
        }
      } else {
        const i64 pid = i64(ng->panels.size());
        // nodes already appended plus the pending run = this panel's first node
        const i64 nb = ng->n_nodes() + (run_a < 0 ? 0 : run_b - run_a);
        ng->panels.push_back({i64(ci), i64(mesh.size()), p.a, p.b, p.level, nb, q});
        mesh.push_back(p);
        if (run_a >= 0 && run_b == o.node_begin) {
          run_b += o.q;
        } else {
          flush();
          run_a = o.node_begin;
          run_b = o.node_begin + o.q;
        }
        for (int j = 0; j < o.q; ++j) {
          plan->kept_old.push_back(o.node_begin + j);
          plan->kept_new.push_back(nb + j);
        }
        ng->panel_of.insert(ng->panel_of.end(), size_t(o.q), pid);
      }
    }
    flush();
    ng->comps.push_back({comp.curve, std::move(mesh), comp.q, node_offset, panel_offset, comp.is_hole});
  }
  return {std::move(ng), std::move(plan)};
}

std::unique_ptr<Geom> geom_coarsen(const Geom& g, const Plan& p) {  // geometry.cpp:344-353
  require(p.old_panels.size() == g.comps.size(), "coarsen: plan mismatch");
  std::vector<sbx_curve> curves;
  std::vector<bool> holes;
  for (const auto& c : g.comps) {
    curves.push_back(c.curve.p);
    holes.push_back(c.is_hole);
  }
  return geom_build(curves, p.old_panels, p.old_q, holes);
}

std::pair<std::unique_ptr<Geom>, std::unique_ptr<Plan>> geom_add_holes(
    const Geom& wall, const std::vector<sbx_curve>& holes, const std::vector<int>& n_panels,
    const std::vector<int>& qs) {  // geometry.cpp:355-404
  require(wall.comps.size() == 1 && !wall.comps[0].is_hole,
          "add_holes expects a single-wall discretization");
  auto plan = std::make_unique<Plan>();
  plan->m = 1;
  plan->old_panels.push_back(wall.comps[0].panels);
  plan->old_q.push_back(wall.comps[0].q);
  std::vector<sbx_curve> curves{wall.comps[0].curve.p};
  std::vector<std::vector<PanelDef>> meshes{wall.comps[0].panels};
  std::vector<int> q{wall.comps[0].q};
  std::vector<bool> flags{false};
  for (size_t i = 0; i < holes.size(); ++i) {
    sbx_curve h = holes[i];
    h.flip_normal = 1;
    curves.push_back(h);
    meshes.push_back(uniform_panels(n_panels[i], qs[i]));
    q.push_back(qs[i]);
    flags.push_back(true);
  }
  auto ng = geom_build(curves, meshes, q, flags);
  for (size_t hi = 1; hi < ng->comps.size(); ++hi)
    for (int s = 0; s < 64; ++s) {
      double px, py, a, b, c, d;
      ng->comps[hi].curve.eval(2 * kPi * s / 64.0, px, py, a, b, c, d);
      if (!inside(ng->comps[0].curve, px, py)) throw Error(3, "hole not inside the domain");
      for (size_t hj = 1; hj < ng->comps.size(); ++hj)
        if (hj != hi && inside(ng->comps[hj].curve, px, py)) throw Error(3, "holes overlap");
    }
  const i64 nw = wall.n_nodes();
  for (i64 i = 0; i < nw; ++i) {
    const size_t s = size_t(i);
    plan->kept_old.push_back(i);
    plan->kept_new.push_back(i);
    ng->x[s] = wall.x[s];
    ng->y[s] = wall.y[s];
    ng->nx[s] = wall.nx[s];
    ng->ny[s] = wall.ny[s];
    ng->tx[s] = wall.tx[s];
    ng->ty[s] = wall.ty[s];
    ng->w[s] = wall.w[s];
    ng->kappa[s] = wall.kappa[s];
    ng->t[s] = wall.t[s];
  }
  for (i64 i = nw; i < ng->n_nodes(); ++i) plan->added_new.push_back(i);
  return {std::move(ng), std::move(plan)};
}

std::vector<i64> panels_near_point(const Geom& g, double px, double py, double radius) {
  std::vector<i64> out;  // geometry.cpp:406-417
  for (i64 p = 0; p < i64(g.panels.size()); ++p) {
    const PanelRow& pr = g.panels[size_t(p)];
    double lo = 1e300;
    for (int j = 0; j < pr.q; ++j) {
      const size_t s = size_t(pr.node_begin + j);
      lo = std::min(lo, std::sqrt((g.x[s] - px) * (g.x[s] - px) + (g.y[s] - py) * (g.y[s] - py)));
    }
    if (lo < radius) out.push_back(p);
  }
  return out;
}

}  // namespace sbx
