// Product-integration weights for the logarithmic singularity of the
// single-layer kernel (reference logquad.cpp:16-112), computed on the host in
// extended precision and uploaded once per discretization (SURVEY.md
// appendix: the device never evaluates these recursions).
//
// For a q-point Gauss-Legendre panel mapped to [-1, 1] and a target at
// parameter u, lambda_j(u) integrates log|u - s| against the degree-(q-1)
// interpolant through the nodes s_j:
//   m_0 = (1-u) log|1-u| + (1+u) log|1+u| - 2
//   m_k = 2/(2k+1) (Q_{k+1}(u) - Q_{k-1}(u)),  k >= 1
//   lambda_j = w_j sum_k (2k+1)/2 P_k(s_j) m_k
// with Legendre functions of the second kind Q_k: upward recurrence for
// |u| < 1, Miller's downward recurrence (normalised by Q_0) for |u| > 1.
#include "logquad.hpp"

#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <unordered_map>
#include <algorithm>

namespace sbx {

namespace {

using ld = long double;

std::vector<ld> legendre_q(int n, double u) {
  require(std::fabs(std::fabs(u) - 1.0) > 1e-14, "log quadrature: target too close to a panel end");
  std::vector<ld> q(size_t(n) + 1, 0.0L);
  const bool mirror = u < -1.0;  // Q_k(-u) = (-1)^{k+1} Q_k(u) for |u| > 1
  const ld x = mirror ? -ld(u) : ld(u);
  if (std::fabs(x) < 1.0L) {
    q[0] = 0.5L * std::log((1.0L + x) / (1.0L - x));
    if (n >= 1) q[1] = x * q[0] - 1.0L;
    for (int k = 2; k <= n; ++k) q[size_t(k)] = ((2 * k - 1) * x * q[size_t(k - 1)] - (k - 1) * q[size_t(k - 2)]) / k;
    return q;
  }
  // x > 1: recur downward from far above n with arbitrary seeds, rescale by Q_0
  const ld rho = x + std::sqrt(x * x - 1.0L);
  int extra = int(std::ceil(46.0L / std::log(rho)));
  extra = std::min(std::max(extra, 20), 20000);
  ld hi = 0.0L, cur = 1e-200L;
  for (int k = n + extra; k >= 1; --k) {
    const ld lo = ((2 * k + 1) * x * cur - (k + 1) * hi) / k;  // Q_{k-1}
    hi = cur;
    cur = lo;
    if (k - 1 <= n) q[size_t(k - 1)] = cur;
    if (std::fabs(cur) > 1e3500L) {
      cur *= 1e-3500L;
      hi *= 1e-3500L;
      for (auto& v : q) v *= 1e-3500L;
    }
  }
  const ld q0 = 0.5L * std::log((x + 1.0L) / (x - 1.0L));
  const ld scale = q0 / q[0];
  for (auto& v : q) v *= scale;
  if (mirror)
    for (int k = 0; k <= n; k += 2) q[size_t(k)] = -q[size_t(k)];
  return q;
}

std::vector<double> compute_weights(int q, double u) {
  const GaussTable& g = gauss_table(q);
  std::vector<ld> m(static_cast<size_t>(q), 0.0L);
  const ld ul = u;
  m[0] = (1.0L - ul) * std::log(std::fabs(1.0L - ul)) + (1.0L + ul) * std::log(std::fabs(1.0L + ul)) - 2.0L;
  if (q > 1) {
    const std::vector<ld> Q = legendre_q(q, u);
    for (int k = 1; k < q; ++k) m[size_t(k)] = 2.0L / (2 * k + 1) * (Q[size_t(k + 1)] - Q[size_t(k - 1)]);
  }
  std::vector<double> w(static_cast<size_t>(q)), P(static_cast<size_t>(q));
  for (int j = 0; j < q; ++j) {
    const double s = g.x[size_t(j)];  // P_k(s_j) in double, as the reference tabulates them
    P[0] = 1.0;
    if (q > 1) P[1] = s;
    for (int k = 2; k < q; ++k) P[size_t(k)] = ((2 * k - 1) * s * P[size_t(k - 1)] - (k - 1) * P[size_t(k - 2)]) / k;
    ld acc = 0.0L;
    for (int k = 0; k < q; ++k) acc += (2 * k + 1) * 0.5L * ld(P[size_t(k)]) * m[size_t(k)];
    w[size_t(j)] = double(ld(g.w[size_t(j)]) * acc);
  }
  return w;
}

struct Key {
  int q;
  std::uint64_t bits;
  bool operator==(const Key& o) const { return q == o.q && bits == o.bits; }
};
struct KeyHash {
  size_t operator()(const Key& k) const { return std::hash<std::uint64_t>()(k.bits * 31 + std::uint64_t(k.q)); }
};

}  // namespace

const std::vector<double>& log_weights(int q, double u) {
  // neighbours of equal length give the same u for every panel: cache by value
  static std::mutex mu;
  static std::unordered_map<Key, std::vector<double>, KeyHash> cache;
  std::uint64_t bits;
  std::memcpy(&bits, &u, sizeof(bits));
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find({q, bits});
  if (it == cache.end()) it = cache.emplace(Key{q, bits}, compute_weights(q, u)).first;
  return it->second;
}

const std::vector<double>& log_self_table(int q) {
  static std::mutex mu;
  static std::map<int, std::vector<double>> cache;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(q);
    if (it != cache.end()) return it->second;
  }
  const GaussTable& g = gauss_table(q);
  std::vector<double> t(size_t(q) * q);  // row i (target node), column j (source node), row-major
  for (int i = 0; i < q; ++i) {
    const std::vector<double> w = compute_weights(q, g.x[size_t(i)]);
    for (int j = 0; j < q; ++j) t[size_t(i) * q + j] = w[size_t(j)];
  }
  std::lock_guard<std::mutex> lk(mu);
  return cache.emplace(q, std::move(t)).first->second;
}

const SlTables& single_layer_tables(const Geom& g, const std::vector<char>& sl_comp, cudaStream_t s) {
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (g.sl && g.sl->mask == sl_comp) return *g.sl;
  auto T = std::make_shared<SlTables>();
  T->mask = sl_comp;
  const i64 n = g.n_nodes();
  T->n = n;
  int qmax = 1;
  for (const auto& c : g.comps) qmax = std::max(qmax, c.q);
  T->qmax = qmax;
  std::vector<int> ints(size_t(5 * n), 0);
  std::vector<double> dbl(size_t(4 * n), 0.0), lam(size_t(2 * n * qmax), 0.0), tab;
  std::map<int, int> tab_off;
  for (i64 i = 0; i < n; ++i) {
    const PanelRow& pr = g.panels[size_t(g.panel_of[size_t(i)])];
    const i64 c = pr.component;
    if (!sl_comp[size_t(c)]) continue;
    const Component& comp = g.comps[size_t(c)];
    const int q = pr.q;
    const int loc = int(i - pr.node_begin);
    const GaussTable& gt = gauss_table(q);
    if (!tab_off.count(q)) {
      tab_off[q] = int(tab.size());
      const auto& t = log_self_table(q);
      tab.insert(tab.end(), t.begin(), t.end());
    }
    const i64 np = i64(comp.panels.size());
    ints[size_t(i)] = loc;
    ints[size_t(n + i)] = q;
    ints[size_t(2 * n + i)] = int(pr.local);
    ints[size_t(3 * n + i)] = int(np);
    ints[size_t(4 * n + i)] = tab_off[q];
    dbl[size_t(i)] = gt.x[size_t(loc)];
    dbl[size_t(n + i)] = g.w[size_t(i)] / gt.w[size_t(loc)];
    const double t = g.t[size_t(i)];
    for (int dir = 0; dir < 2; ++dir) {  // previous, next panel of the closed curve
      const i64 nb = dir == 0 ? (pr.local + np - 1) % np : (pr.local + 1) % np;
      const PanelDef& pn = comp.panels[size_t(nb)];
      const double mid = 0.5 * (pn.a + pn.b);
      double tt = t;
      while (tt - mid > kPi) tt -= 2 * kPi;
      while (mid - tt > kPi) tt += 2 * kPi;
      const double u = 2.0 * (tt - pn.a) / (pn.b - pn.a) - 1.0;
      dbl[size_t((2 + dir) * n + i)] = u;
      const std::vector<double>& w = log_weights(comp.q, u);
      std::copy(w.begin(), w.end(), lam.begin() + (dir * n + i) * qmax);
    }
  }
  if (tab.empty()) tab.push_back(0.0);
  T->ints.upload(ints, s);
  T->dbl.upload(dbl, s);
  T->lam.upload(lam, s);
  T->tab.upload(tab, s);
  SBX_CUDA(cudaStreamSynchronize(s));
  g.sl = T;
  return *T;
}

}  // namespace sbx
