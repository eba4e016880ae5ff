// Device HBS compression + telescoping inverse (reference hbs.cpp:349-487).
//
// Host code owns the tree topology and index bookkeeping (near sets,
// candidate lists, rank rules); every floating-point step runs on the GPU,
// batched over all boxes of a level:
//   W^T assembly  (entries.cu proxy/near jobs)  ->  CPQR (dense.cu qr_kernel)
//   ->  ranks, sample doubling, rank equalisation (host, from |r_jj|)
//   ->  interpolation matrices (interp_kernel)  ->  b_sib blocks.
// The inverse is a per-level batch of LU/inverse/rcond + DMMA GEMMs.
#include <algorithm>
#include <cstdio>
#include <climits>
#include <cmath>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <unordered_map>

#include "dense.hpp"
#include "entries.hpp"
#include "hbs_build.hpp"
#include "idengine.hpp"
#include "multigpu.hpp"

namespace sbx {

namespace {

struct Region {
  double cx = 0, cy = 0, r0 = 0;
};

std::vector<i64> scalars_of_range(i64 b, i64 e) {
  std::vector<i64> s;
  s.reserve(size_t(2 * (e - b)));
  for (i64 i = b; i < e; ++i) {
    s.push_back(2 * i);
    s.push_back(2 * i + 1);
  }
  return s;
}

// Per-level device storage of the interpolation factors and couplings.
struct LevelStore {
  DevBuf<double> buf;
  std::vector<i64> o_u, o_v, o_b;  // per node in level order
};

struct Builder {
  const Geom& g;
  const HbsBuildOptions& o;
  cudaStream_t s;
  HbsOp& op;
  const EntryOracle& eo;
  bool has_null;
  std::vector<double> px, py;  // local node coordinates
  std::vector<Region> reg;
  std::vector<std::vector<i64>> levels;
  i64 max_block = 0;

  std::vector<i64> row_cand(const HbsNodeH& nd) const {
    if (nd.is_leaf()) return scalars_of_range(nd.begin, nd.end);
    std::vector<i64> c = op.nodes[size_t(nd.left)].row_skel;
    const auto& r = op.nodes[size_t(nd.right)].row_skel;
    c.insert(c.end(), r.begin(), r.end());
    return c;
  }
  std::vector<i64> col_cand(const HbsNodeH& nd) const {
    if (nd.is_leaf()) return scalars_of_range(nd.begin, nd.end);
    std::vector<i64> c = op.nodes[size_t(nd.left)].col_skel;
    const auto& r = op.nodes[size_t(nd.right)].col_skel;
    c.insert(c.end(), r.begin(), r.end());
    return c;
  }
};

// Near sets of one level (hbs.cpp:242-268).  Leaves use a uniform-grid
// neighbour search returning the same ascending node list as the
// reference's O(N) scan; internal nodes scan their level.
void near_sets(Builder& B, const std::vector<i64>& ids, std::vector<std::vector<i64>>& nc,
               std::vector<std::vector<i64>>& nr) {
  nc.assign(ids.size(), {});
  nr.assign(ids.size(), {});
  const auto& nodes = B.op.nodes;
  bool any_leaf = false;
  double h = 0;
  for (i64 id : ids)
    if (nodes[size_t(id)].is_leaf()) {
      any_leaf = true;
      h = std::max(h, B.o.div_factor * B.reg[size_t(id)].r0);
    }
  std::unordered_map<long long, std::vector<i64>> grid;
  auto key = [](long long a, long long b) { return (a << 32) ^ (b & 0xffffffffLL); };
  if (any_leaf) {
    h = std::max(h, 1e-300);
    const i64 n = i64(B.px.size());
    for (i64 j = 0; j < n; ++j)
      grid[key((long long)std::floor(B.px[size_t(j)] / h), (long long)std::floor(B.py[size_t(j)] / h))]
          .push_back(j);
  }
  for (size_t q = 0; q < ids.size(); ++q) {
    const i64 id = ids[q];
    const HbsNodeH& nd = nodes[size_t(id)];
    const Region& rg = B.reg[size_t(id)];
    const double rad = B.o.div_factor * rg.r0;
    if (nd.is_leaf()) {
      std::vector<i64> hits;
      const long long gx = (long long)std::floor(rg.cx / h), gy = (long long)std::floor(rg.cy / h);
      const long long span = (long long)std::ceil(rad / h) + 1;
      for (long long a = gx - span; a <= gx + span; ++a)
        for (long long b = gy - span; b <= gy + span; ++b) {
          auto it = grid.find(key(a, b));
          if (it == grid.end()) continue;
          for (i64 j : it->second) {
            if (j >= nd.begin && j < nd.end) continue;
            const double dx = B.px[size_t(j)] - rg.cx, dy = B.py[size_t(j)] - rg.cy;
            if (std::sqrt(dx * dx + dy * dy) <= rad) hits.push_back(j);
          }
        }
      std::sort(hits.begin(), hits.end());
      for (i64 j : hits) {
        nc[q].push_back(2 * j);
        nc[q].push_back(2 * j + 1);
      }
      nr[q] = nc[q];
      continue;
    }
    for (i64 other : B.levels[size_t(nd.depth)]) {
      if (other == id) continue;
      const Region& org = B.reg[size_t(other)];
      const double dx = org.cx - rg.cx, dy = org.cy - rg.cy;
      if (std::sqrt(dx * dx + dy * dy) > rad + org.r0) continue;
      const auto cc = B.col_cand(nodes[size_t(other)]);
      const auto rc = B.row_cand(nodes[size_t(other)]);
      nc[q].insert(nc[q].end(), cc.begin(), cc.end());
      nr[q].insert(nr[q].end(), rc.begin(), rc.end());
    }
  }
}

// One sample-count round of W^T for every (node, row|col) problem.
struct SampleRound {
  DevBuf<double> wt;
  std::vector<IdProblem> probs;  // 2 per node: row then col
  IdBatch ids;
};

void build_round(Builder& B, const std::vector<i64>& ids, const std::vector<int>& ns_of,
                 const std::vector<std::vector<i64>>& rcand, const std::vector<std::vector<i64>>& ccand,
                 const std::vector<std::vector<i64>>& nc, const std::vector<std::vector<i64>>& nr,
                 SampleRound& R) {
  const int wn = B.has_null ? 1 : 0;
  std::vector<i64> off;
  i64 total = 0;
  R.probs.clear();
  for (size_t q = 0; q < ids.size(); ++q) {
    for (int side = 0; side < 2; ++side) {
      const int n = int(side == 0 ? rcand[q].size() : ccand[q].size());
      const int M = 4 * ns_of[q] + wn + int(side == 0 ? nc[q].size() : nr[q].size());
      off.push_back(total);
      total += i64(M) * n;
      R.probs.push_back({nullptr, M, n, std::max(M, 1)});
    }
  }
  R.wt.resize(size_t(std::max<i64>(total, 1)));
  for (size_t p = 0; p < R.probs.size(); ++p) R.probs[p].wt = R.wt.get() + off[p];
  // index arrays: candidates and near lists, concatenated
  std::vector<i64> cand, nearv;
  std::vector<ProxyJob> pj;
  std::vector<NearJob> nj;
  int max_rows = 0, max_n = 0;
  i64 max_near = 0;
  for (size_t q = 0; q < ids.size(); ++q) {
    const Region& rg = B.reg[size_t(ids[q])];
    for (int side = 0; side < 2; ++side) {
      const auto& cv = side == 0 ? rcand[q] : ccand[q];
      const auto& nv = side == 0 ? nc[q] : nr[q];
      const IdProblem& pr = R.probs[2 * q + size_t(side)];
      const i64 coff = i64(cand.size());
      cand.insert(cand.end(), cv.begin(), cv.end());
      if (pr.n == 0) continue;
      ProxyJob j{};
      j.cand_off = coff;
      j.n = pr.n;
      j.ns = ns_of[q];
      j.cx = rg.cx;
      j.cy = rg.cy;
      j.rad = B.o.bas_factor * rg.r0;
      j.out_off = off[2 * q + size_t(side)];
      j.ld = pr.lda;
      j.kind = side;  // 0 outgoing rows, 1 incoming columns
      j.with_null = wn;
      pj.push_back(j);
      max_rows = std::max(max_rows, j.ns);
      max_n = std::max(max_n, j.n);
      if (!nv.empty()) {
        NearJob k{};
        k.cand_off = coff;
        k.near_off = i64(nearv.size());
        k.n = pr.n;
        k.n_near = int(nv.size());
        k.out_off = off[2 * q + size_t(side)] + 4 * ns_of[q] + wn;
        k.ld = pr.lda;
        k.transpose = side;  // row ID: A(cand, near)^T ; col ID: A(near, cand)
        nearv.insert(nearv.end(), nv.begin(), nv.end());
        nj.push_back(k);
        max_near = std::max<i64>(max_near, i64(k.n_near) * k.n);
        B.max_block = std::max<i64>(B.max_block, i64(k.n_near) * k.n);
      }
    }
  }
  DevBuf<i64> dcand, dnear;
  DevBuf<ProxyJob> dpj;
  DevBuf<NearJob> dnj;
  dcand.upload(cand, B.s);
  dnear.upload(nearv, B.s);
  dpj.upload(pj, B.s);
  dnj.upload(nj, B.s);
  launch_proxy_jobs(B.eo.view(), dpj.get(), int(pj.size()), max_rows, max_n, dcand.get(), R.wt.get(), B.s);
  if (B.o.entries)
    host_near_jobs(*B.o.entries, nj, cand, nearv, R.wt.get(), B.s);
  else
    launch_near_jobs(B.eo.view(), dnj.get(), int(nj.size()), max_near, dcand.get(), dnear.get(),
                     R.wt.get(), B.s);
  R.ids.factor(R.probs, 1e-15, B.s);  // keeps every row the forced-rank rule can use
}

}  // namespace

// ---------------------------------------------------------------- inverse
namespace {
// Where one node's inputs and outputs of the telescoping inverse live: the
// arena (hbs_invert_device) or the per-level staging of the fused build.
struct InvSrc {
  const double* d = nullptr;  // leaf diagonal block (c x c, ld ldd)
  int ldd = 0;
  const double* u = nullptr;  // c x k, ld c
  const double* v = nullptr;  // c x k, ld c
  const double* b = nullptr;  // b_sib: k x k_sib, ld k
  double* dhat = nullptr;     // k x k
  double* e = nullptr;        // c x k, ld c
  double* fg = nullptr;       // (k + c) x c, ld k + c
};

// rcond gates (hbs.cpp:429) of one level, checked after the last level:
// the levels run back to back on the stream without host round trips; a
// failing block is reported as the first one in factorisation order
struct Gate {
  std::vector<size_t> ids;
  DevBuf<double> rc;
  int depth = 0;
};

std::string sci(double v) {
  char b[32];
  std::snprintf(b, sizeof(b), "%.3e", v);
  return b;
}

void check_gates(HbsOp& op, std::vector<std::unique_ptr<Gate>>& gates, double thr, cudaStream_t s) {
  op.node_rcond.assign(op.nodes.size(), 1.0);
  for (const auto& gp : gates) {
    const Gate& gt = *gp;
    std::vector<double> hrc(gt.rc.size());
    gt.rc.download(hrc.data(), hrc.size(), s);
    SBX_CUDA(cudaStreamSynchronize(s));
    for (size_t q = 0; q < gt.ids.size(); ++q) {
      const auto& nd = op.nodes[gt.ids[q]];
      double r = nd.c > 0 ? hrc[2 * q] : 1.0;
      if (gt.ids[q] != 0 && nd.c > 0 && nd.k > 0) r = std::min(r, hrc[2 * q + 1]);
      op.node_rcond[gt.ids[q]] = r;
    }
    for (size_t q = 0; q < gt.ids.size(); ++q) {
      const auto& nd = op.nodes[gt.ids[q]];
      if (nd.c > 0 && !(hrc[2 * q] >= thr))
        throw Error(4, std::string("singular ") + (gt.ids[q] == 0 ? "root" : "diagonal") +
                           " block (rcond " + sci(hrc[2 * q]) + ") at tree node [" +
                           std::to_string(nd.begin) + "," + std::to_string(nd.end) + ") depth " +
                           std::to_string(nd.depth));
    }
    for (size_t q = 0; q < gt.ids.size(); ++q) {
      const auto& nd = op.nodes[gt.ids[q]];
      if (gt.ids[q] != 0 && nd.c > 0 && nd.k > 0 && !(hrc[2 * q + 1] >= thr))
        throw Error(4, "singular skeleton block (rcond " + sci(hrc[2 * q + 1]) + ") at tree node [" +
                           std::to_string(nd.begin) + "," + std::to_string(nd.end) + ") depth " +
                           std::to_string(nd.depth));
    }
  }
}

// One level of the telescoping inverse (hbs.cpp:427-487) for the nodes
// `ids` (all of one depth), batched: x blocks, LU/inverse/rcond of x,
// t = v^T xi, xu = xi u, tu = t u, dhat = tu^{-1}, e = xu dhat, f = dhat t,
// g = xi - e t.  The root (id 0) only gets root_g = x^{-1}.
void invert_level(const HbsOp& op, const std::vector<size_t>& ids, const std::vector<InvSrc>& P, double* root_g,
                  std::vector<std::unique_ptr<Gate>>& gates, cudaStream_t s) {
  // x blocks and scratch
  std::vector<i64> xo(ids.size()), io(ids.size()), to(ids.size()), tuo(ids.size()), xuo(ids.size());
  i64 tot = 0;
  for (size_t q = 0; q < ids.size(); ++q) {
    const auto& nd = op.nodes[ids[q]];
    const i64 c = nd.c, k = nd.k;
    xo[q] = tot;
    tot += c * c;
    io[q] = tot;
    tot += c * c;
    to[q] = tot;
    tot += k * c;
    tuo[q] = tot;
    tot += k * k;
    xuo[q] = tot;
    tot += c * k;
  }
  DevBuf<double> scr(static_cast<size_t>(std::max<i64>(tot, 1)));
  double* S = scr.get();
  std::vector<CopyJob> cj;
  for (size_t q = 0; q < ids.size(); ++q) {
    const auto& nd = op.nodes[ids[q]];
    const int c = int(nd.c);
    double* x = S + xo[q];
    if (nd.is_leaf()) {
      cj.push_back({P[ids[q]].d, x, c, c, P[ids[q]].ldd, c, 0, 0});
    } else {
      const InvSrc& l = P[size_t(nd.left)];
      const InvSrc& r = P[size_t(nd.right)];
      const int kl = int(op.nodes[size_t(nd.left)].k), kr = int(op.nodes[size_t(nd.right)].k);
      if (kl) cj.push_back({l.dhat, x, kl, kl, kl, c, 0, 0});
      if (kl && kr) cj.push_back({l.b, x + size_t(kl) * c, kl, kr, kl, c, 0, 0});
      if (kl && kr) cj.push_back({r.b, x + kl, kr, kl, kr, c, 0, 0});
      if (kr) cj.push_back({r.dhat, x + kl + size_t(kl) * c, kr, kr, kr, c, 0, 0});
    }
  }
  copy_batched(cj, s);
  DevBuf<int> piv(static_cast<size_t>(std::max<i64>(tot, 1)));
  gates.push_back(std::make_unique<Gate>());
  Gate& gt = *gates.back();
  gt.ids = ids;
  gt.depth = ids.empty() ? 0 : op.nodes[ids[0]].depth;
  gt.rc.resize(ids.size() * 2 + 1);
  DevBuf<double>& rc = gt.rc;
  SBX_CUDA(cudaMemsetAsync(rc.get(), 0x7f, rc.size() * sizeof(double), s));  // unset gates pass
  DevBuf<double> work;
  i64 wtot = 0;
  for (size_t q = 0; q < ids.size(); ++q) wtot += 4 * (op.nodes[ids[q]].c + op.nodes[ids[q]].k);
  work.resize(size_t(std::max<i64>(wtot, 1)));
  // LU + inverse + rcond of x
  std::vector<LuJob> lj;
  i64 pw = 0;
  for (size_t q = 0; q < ids.size(); ++q) {
    const auto& nd = op.nodes[ids[q]];
    if (nd.c == 0) continue;
    LuJob j{};
    j.a = S + xo[q];
    j.n = int(nd.c);
    j.lda = int(nd.c);
    j.piv = piv.get() + xo[q];
    j.inv = ids[q] == 0 ? root_g : S + io[q];
    j.rcond = rc.get() + 2 * q;
    j.work = work.get() + pw;
    pw += 4 * nd.c;
    lj.push_back(j);
  }
  lu_batched(lj, s);
  phase_mark("inv: x blocks + LU/inverse", s);
  if (ids.size() == 1 && ids[0] == 0) return;  // the root keeps only root_g (hbs.cpp:450-458)
  // t = v^T xi (k x c), tu = t u (k x k)
  std::vector<GemmJob> g1, g2;
  for (size_t q = 0; q < ids.size(); ++q) {
    const auto& nd = op.nodes[ids[q]];
    const InvSrc& p = P[ids[q]];
    const int c = int(nd.c), k = int(nd.k);
    if (c == 0 || k == 0) continue;
    g1.push_back({p.v, S + io[q], S + to[q], k, c, c, c, c, k, 1, 0, 1.0, 0.0});
    g1.push_back({S + io[q], p.u, S + xuo[q], c, k, c, c, c, c, 0, 0, 1.0, 0.0});
  }
  gemm_batched(g1, s);
  for (size_t q = 0; q < ids.size(); ++q) {
    const auto& nd = op.nodes[ids[q]];
    const int c = int(nd.c), k = int(nd.k);
    if (c == 0 || k == 0) continue;
    g2.push_back({S + to[q], P[ids[q]].u, S + tuo[q], k, k, c, k, c, k, 0, 0, 1.0, 0.0});
  }
  gemm_batched(g2, s);
  std::vector<LuJob> lj2;
  pw = 0;
  for (size_t q = 0; q < ids.size(); ++q) {
    const auto& nd = op.nodes[ids[q]];
    if (nd.c == 0 || nd.k == 0) continue;
    LuJob j{};
    j.a = S + tuo[q];
    j.n = int(nd.k);
    j.lda = int(nd.k);
    j.piv = piv.get() + xo[q];
    j.inv = P[ids[q]].dhat;
    j.rcond = rc.get() + 2 * q + 1;
    j.work = work.get() + pw;
    pw += 4 * nd.k;
    lj2.push_back(j);
  }
  lu_batched(lj2, s);
  // e = (xi u) dhat, f = dhat t, g = xi - e t   (hbs.cpp:480-483)
  std::vector<GemmJob> g3, g4;
  std::vector<CopyJob> cg;
  for (size_t q = 0; q < ids.size(); ++q) {
    const auto& nd = op.nodes[ids[q]];
    const InvSrc& p = P[ids[q]];
    const int c = int(nd.c), k = int(nd.k);
    if (c == 0) continue;
    const int ld = k + c;
    cg.push_back({S + io[q], p.fg + k, c, c, c, ld, 0, 0});  // g <- xi
    if (k == 0) continue;
    g3.push_back({S + xuo[q], p.dhat, p.e, c, k, k, c, k, c, 0, 0, 1.0, 0.0});
    g3.push_back({p.dhat, S + to[q], p.fg, k, c, k, k, k, ld, 0, 0, 1.0, 0.0});
  }
  copy_batched(cg, s);
  gemm_batched(g3, s);
  for (size_t q = 0; q < ids.size(); ++q) {
    const auto& nd = op.nodes[ids[q]];
    const InvSrc& p = P[ids[q]];
    const int c = int(nd.c), k = int(nd.k);
    if (c == 0 || k == 0) continue;
    g4.push_back({p.e, S + to[q], p.fg + k, c, c, k, c, k, k + c, 0, 0, -1.0, 1.0});
  }
  gemm_batched(g4, s);
  phase_mark("inv: skeleton LU + e,f,g GEMMs", s);
}
}  // namespace

namespace {
// The fused build (with_inverse): a second host thread runs invert_level for
// depth d on its own stream as soon as the compression of depth d (u, v,
// b_sib) is complete, while the compression moves on to depth d - 1; the
// inverse factors go to per-level staging and join the arena at the end.
struct FusedInverse {
  std::mutex mu;
  std::condition_variable cv;
  int ready = INT_MAX;  // lowest depth whose factors are complete
  bool abort = false;
  std::vector<InvSrc> P;
  std::vector<DevBuf<double>> stage;  // per depth: dhat | e | fg of its nodes
  DevBuf<double> rootg;
  std::vector<std::unique_ptr<Gate>> gates;
  std::exception_ptr err;
  std::thread th;
  cudaEvent_t done = nullptr;
  void publish(int depth) {
    std::lock_guard<std::mutex> lk(mu);
    ready = depth;
    cv.notify_all();
  }
  bool wait_for(int depth) {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [&] { return abort || ready <= depth; });
    return !abort;
  }
  ~FusedInverse() {
    if (th.joinable()) {
      {
        std::lock_guard<std::mutex> lk(mu);
        abort = true;
        cv.notify_all();
      }
      th.join();
    }
    if (done) cudaEventDestroy(done);
  }
};

cudaStream_t inverse_stream() {
  static const cudaStream_t w = [] {
    cudaStream_t x = nullptr;
    SBX_CUDA(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
    return x;
  }();
  return w;
}

std::unique_ptr<HbsOp> compress_impl(const Geom& g, int formulation, double mu, const i64* nodes, i64 n_nodes,
                                     const HbsBuildOptions& o, cudaStream_t s, bool with_inverse) {
  require(o.eps > 0.0 && o.eps <= 0.1, "hbs_compress: tolerance out of range");
  require(o.leaf_nodes >= 2, "hbs_compress: leaf size too small");
  const i64 N = nodes ? n_nodes : g.n_nodes();
  require(N > 0, "hbs_compress: empty source");
  DevBuf<i64> dmap;
  if (nodes) {
    for (i64 i = 0; i < N; ++i) require(nodes[i] >= 0 && nodes[i] < g.n_nodes(), "hbs_compress: node out of range");
    dmap.upload(nodes, size_t(N), s);
  }
  EntryOracle eo(g, formulation, mu, s, nodes ? dmap.get() : nullptr);
  auto op = std::make_unique<HbsOp>();
  op->n = 2 * N;
  op->leaf_nodes = o.leaf_nodes;
  op->eps = o.eps;
  require(!o.entries || !nodes, "hbs_compress: a custom entry oracle covers the whole discretization");
  const bool with_null = eo.has_nullspace() && (!o.entries || o.entries->with_completion);
  Builder B{g, o, s, *op, eo, with_null, {}, {}, {}, {}, 0};
  B.px.resize(size_t(N));
  B.py.resize(size_t(N));
  for (i64 i = 0; i < N; ++i) {
    const i64 nd = nodes ? nodes[i] : i;
    B.px[size_t(i)] = g.x[size_t(nd)];
    B.py[size_t(i)] = g.y[size_t(nd)];
  }
  // balanced BFS tree (hbs.cpp:360-384)
  struct Pending {
    i64 b, e, parent;
    int depth;
  };
  std::vector<Pending> queue{{0, N, -1, 0}};
  for (size_t qi = 0; qi < queue.size(); ++qi) {
    const Pending p = queue[qi];
    HbsNodeH nd;
    nd.begin = p.b;
    nd.end = p.e;
    nd.parent = p.parent;
    nd.depth = p.depth;
    const i64 id = i64(op->nodes.size());
    if (p.parent >= 0) {
      HbsNodeH& par = op->nodes[size_t(p.parent)];
      (par.left < 0 ? par.left : par.right) = id;
    }
    op->nodes.push_back(nd);
    if (p.e - p.b > o.leaf_nodes) {
      const i64 mid = p.b + (p.e - p.b) / 2;
      queue.push_back({p.b, mid, id, p.depth + 1});
      queue.push_back({mid, p.e, id, p.depth + 1});
    }
  }
  const size_t nn = op->nodes.size();
  int max_depth = 0;
  B.reg.resize(nn);
  for (size_t i = 0; i < nn; ++i) {  // node_region (hbs.cpp:107-117)
    const auto& nd = op->nodes[i];
    double sx = 0, sy = 0;
    for (i64 j = nd.begin; j < nd.end; ++j) {
      sx += B.px[size_t(j)];
      sy += B.py[size_t(j)];
    }
    Region r;
    r.cx = sx / double(nd.end - nd.begin);
    r.cy = sy / double(nd.end - nd.begin);
    for (i64 j = nd.begin; j < nd.end; ++j) {
      const double dx = B.px[size_t(j)] - r.cx, dy = B.py[size_t(j)] - r.cy;
      r.r0 = std::max(r.r0, std::sqrt(dx * dx + dy * dy));
    }
    r.r0 = std::max(r.r0, 1e-12);
    B.reg[i] = r;
    max_depth = std::max(max_depth, nd.depth);
  }
  B.levels.assign(size_t(max_depth + 1), {});
  for (size_t i = 0; i < nn; ++i) B.levels[size_t(op->nodes[i].depth)].push_back(i64(i));
  // subtree-sharded build (multi-GPU): rank p of G = 2^g compresses the nodes
  // of depth >= g under the p-th depth-g node, and every node above, itself
  std::vector<char> mine(nn, 1);
  Collective* comm = o.comm;
  int G = 1, P = 0, gdep = 0;
  if (comm && comm->world() > 1) {
    require(!with_inverse, "hbs_compress: the fused build is not sharded");
    require(!nodes && !o.entries, "hbs_compress: a sharded build covers the whole discretization");
    G = comm->world();
    P = comm->rank();
    while ((1 << gdep) < G) ++gdep;
    require((1 << gdep) == G, "hbs_compress: sharded builds need a power-of-two rank count");
    std::vector<i64> owner(nn, -1);
    i64 q = 0;
    for (size_t i = 0; i < nn; ++i) {
      if (op->nodes[i].is_leaf())
        require(op->nodes[i].depth >= gdep, "hbs_compress: tree has a leaf above the partition depth");
      if (op->nodes[i].depth == gdep) owner[i] = q++;
      else if (op->nodes[i].depth > gdep) owner[i] = owner[size_t(op->nodes[i].parent)];
    }
    require(q == G, "hbs_compress: tree has fewer subtrees than ranks");
    op->stored.assign(nn, 0);
    for (size_t i = 0; i < nn; ++i) {
      mine[i] = owner[i] < 0 || owner[i] == P;
      op->stored[i] = mine[i] || op->nodes[i].depth == gdep;  // subtree roots: coupling + dhat slots everywhere
    }
    op->shard_G = G;
    op->shard_p = P;
    op->shard_g = gdep;
    op->comm = comm;
  }

  // leaf diagonal blocks
  std::vector<i64> leaf_ids;
  for (size_t i = 0; i < nn; ++i)
    if (op->nodes[i].is_leaf() && mine[i]) leaf_ids.push_back(i64(i));
  std::vector<i64> d_off(nn, -1);
  DevBuf<double> dstore;
  {
    std::vector<i64> idx;
    std::vector<BlockJob> jobs;
    i64 tot = 0, mx = 0;
    for (i64 id : leaf_ids) {
      const auto& nd = op->nodes[size_t(id)];
      const int c = int(2 * (nd.end - nd.begin));
      BlockJob j{};
      j.row_off = i64(idx.size());
      j.col_off = i64(idx.size());
      j.nr = c;
      j.nc = c;
      j.out_off = tot;
      j.ld = c;
      d_off[size_t(id)] = tot;
      tot += i64(c) * c;
      mx = std::max<i64>(mx, i64(c) * c);
      B.max_block = std::max<i64>(B.max_block, i64(c) * c);
      for (i64 q = 2 * nd.begin; q < 2 * nd.end; ++q) idx.push_back(q);
      jobs.push_back(j);
    }
    dstore.resize(size_t(std::max<i64>(tot, 1)));
    DevBuf<i64> didx;
    DevBuf<BlockJob> djobs;
    didx.upload(idx, s);
    djobs.upload(jobs, s);
    if (o.entries)
      host_block_jobs(*o.entries, jobs, idx, idx, dstore.get(), s);
    else
      launch_block_jobs(eo.view(), djobs.get(), int(jobs.size()), mx, didx.get(), didx.get(), dstore.get(), s);
    SBX_CUDA(cudaStreamSynchronize(s));
  }

  std::unique_ptr<FusedInverse> fz;
  if (with_inverse) {
    fz = std::make_unique<FusedInverse>();
    fz->P.resize(nn);
    fz->stage.resize(size_t(max_depth + 1));
    for (i64 id : leaf_ids) {
      fz->P[size_t(id)].d = dstore.get() + d_off[size_t(id)];
      fz->P[size_t(id)].ldd = int(2 * (op->nodes[size_t(id)].end - op->nodes[size_t(id)].begin));
    }
    SBX_CUDA(cudaEventCreateWithFlags(&fz->done, cudaEventDisableTiming));
    int dev = 0;
    SBX_CUDA(cudaGetDevice(&dev));
    FusedInverse* F = fz.get();
    const HbsOp* opp = op.get();
    const std::vector<std::vector<i64>>* levels = &B.levels;
    F->th = std::thread([F, opp, levels, dev, max_depth] {
      const cudaStream_t w = inverse_stream();
      try {
        SBX_CUDA(cudaSetDevice(dev));
        StreamScope ss(w);
        phase_mark(nullptr, w);
        for (int d = max_depth; d >= 0; --d) {
          if (!F->wait_for(d)) break;
          std::vector<size_t> ids;
          for (i64 id : (*levels)[size_t(d)]) ids.push_back(size_t(id));
          invert_level(*opp, ids, F->P, d == 0 ? F->rootg.get() : nullptr, F->gates, w);
        }
      } catch (...) {
        F->err = std::current_exception();
      }
      cudaEventRecord(F->done, w);
      cudaStreamSynchronize(w);  // thread-local job tables die with the thread
    });
  }
  // bottom-up skeletonisation; the root keeps no factors (hbs.cpp:411-421)
  std::vector<std::unique_ptr<LevelStore>> stores(static_cast<size_t>(max_depth + 1));
  std::vector<i64> pos_in_level(nn, 0);
  std::vector<double> remote_b;  // sharded: the other subtree roots' couplings (gathered)
  std::vector<i64> remote_b_off(nn, -1);
  for (int depth = max_depth; depth >= 1; --depth) {
    std::vector<i64> ids;
    for (i64 id : B.levels[size_t(depth)])
      if (mine[size_t(id)]) ids.push_back(id);
    const size_t L = ids.size();
    for (size_t q = 0; q < L; ++q) pos_in_level[size_t(ids[q])] = i64(q);
    std::vector<std::vector<i64>> rc(L), cc(L), nc, nr;
    for (size_t q = 0; q < L; ++q) {
      rc[q] = B.row_cand(op->nodes[size_t(ids[q])]);
      cc[q] = B.col_cand(op->nodes[size_t(ids[q])]);
    }
    near_sets(B, ids, nc, nr);
    phase_mark("hbs: near sets", s);
    for (size_t q = 0; q < L; ++q) {
      B.max_block = std::max<i64>(B.max_block, i64(rc[q].size()) * i64(nc[q].size()));
      B.max_block = std::max<i64>(B.max_block, i64(nr[q].size()) * i64(cc[q].size()));
    }
    // sample doubling until the rank settles within 2 (hbs.cpp:198-213)
    std::vector<std::unique_ptr<SampleRound>> rounds;
    std::vector<int> row_round(L, -1), col_round(L, -1);   // round holding the final sample
    std::vector<size_t> row_pi(L, 0), col_pi(L, 0);        // problem index inside that round
    std::vector<i64> prev_kr(L, -1), prev_kc(L, -1);
    std::vector<char> row_done(L, 0), col_done(L, 0);
    std::vector<size_t> active(L);
    for (size_t q = 0; q < L; ++q) active[q] = q;
    // The first two sample counts are always both needed (hbs.cpp:201-206),
    // so they run as one batch; later doublings only for unsettled boxes.
    for (int ns = 64; ns <= 2048 && !active.empty(); ns *= 2) {
      const bool pair = ns == 64;
      std::vector<i64> aid;
      std::vector<int> ans;
      std::vector<std::vector<i64>> arc, acc, anc, anr;
      for (int rep = 0; rep < (pair ? 2 : 1); ++rep)
        for (size_t q : active) {
          aid.push_back(ids[q]);
          ans.push_back(ns << rep);
          arc.push_back(rc[q]);
          acc.push_back(cc[q]);
          anc.push_back(nc[q]);
          anr.push_back(nr[q]);
        }
      auto R = std::make_unique<SampleRound>();
      build_round(B, aid, ans, arc, acc, anc, anr, *R);
      const int ridx = int(rounds.size());
      const size_t na = active.size();
      std::vector<size_t> next;
      for (size_t a = 0; a < na; ++a) {
        const size_t q = active[a];
        for (int rep = 0; rep < (pair ? 2 : 1); ++rep) {
          const size_t pa = a + size_t(rep) * na;
          const i64 kr = R->ids.eps_rank(2 * pa, o.eps), kc = R->ids.eps_rank(2 * pa + 1, o.eps);
          if (!row_done[q]) {
            const bool settled = prev_kr[q] >= 0 && std::llabs(kr - prev_kr[q]) <= 2;
            row_round[q] = ridx;
            row_pi[q] = 2 * pa;
            prev_kr[q] = kr;
            if (settled) row_done[q] = 1;
          }
          if (!col_done[q]) {
            const bool settled = prev_kc[q] >= 0 && std::llabs(kc - prev_kc[q]) <= 2;
            col_round[q] = ridx;
            col_pi[q] = 2 * pa + 1;
            prev_kc[q] = kc;
            if (settled) col_done[q] = 1;
          }
        }
        if (!row_done[q] || !col_done[q]) next.push_back(q);
      }
      rounds.push_back(std::move(R));
      if (pair) ns *= 2;  // 64 and 128 done
      active = next;
    }
    for (size_t q = 0; q < L; ++q) {
      if (!row_done[q]) op->notes.push_back("hbs row: proxy sample cap reached");
      if (!col_done[q]) op->notes.push_back("hbs col: proxy sample cap reached");
    }
    phase_mark("hbs: sample rounds (W^T + CPQR)", s);
    // rank equalisation (hbs.cpp:309-314)
    std::vector<i64> kfin(L);
    for (size_t q = 0; q < L; ++q) {
      const IdBatch& RB = rounds[size_t(row_round[q])]->ids;
      const IdBatch& CB = rounds[size_t(col_round[q])]->ids;
      i64 kr = RB.eps_rank(row_pi[q], o.eps), kc = CB.eps_rank(col_pi[q], o.eps);
      i64 k = std::max(kr, kc);
      if (kr < k) kr = RB.forced_rank(row_pi[q], k);
      if (kc < k) kc = CB.forced_rank(col_pi[q], k);
      k = std::min(kr, kc);
      kfin[q] = k;
    }
    // skeletons (idlib.cpp:55-62: J[:k] of each ID)
    for (size_t q = 0; q < L; ++q) {
      HbsNodeH& nd = op->nodes[size_t(ids[q])];
      const IdBatch& RB = rounds[size_t(row_round[q])]->ids;
      const IdBatch& CB = rounds[size_t(col_round[q])]->ids;
      nd.k = kfin[q];
      nd.row_skel.resize(size_t(nd.k));
      nd.col_skel.resize(size_t(nd.k));
      for (i64 i = 0; i < nd.k; ++i) {
        nd.row_skel[size_t(i)] = rc[q][size_t(RB.perm(row_pi[q])[size_t(i)])];
        nd.col_skel[size_t(i)] = cc[q][size_t(CB.perm(col_pi[q])[size_t(i)])];
      }
      if (nd.k == i64(rc[q].size()))
        op->notes.push_back("node [" + std::to_string(nd.begin) + "," + std::to_string(nd.end) +
                            ") kept at full rank (stored dense)");
    }
    if (G > 1 && depth >= gdep) {  // the other subtrees' skeletons of this depth (near sets, couplings above)
      std::vector<double> pk;
      for (i64 id : ids) {
        const auto& nd = op->nodes[size_t(id)];
        pk.push_back(double(id));
        pk.push_back(double(nd.k));
        for (i64 v : nd.row_skel) pk.push_back(double(v));
        for (i64 v : nd.col_skel) pk.push_back(double(v));
      }
      const auto all = gather_host(*comm, pk, s);
      for (int r = 0; r < G; ++r) {
        if (r == P) continue;
        const auto& v = all[size_t(r)];
        for (size_t at = 0; at < v.size();) {
          HbsNodeH& nd = op->nodes[size_t(v[at])];
          nd.k = i64(v[at + 1]);
          nd.row_skel.assign(size_t(nd.k), 0);
          nd.col_skel.assign(size_t(nd.k), 0);
          for (i64 i = 0; i < nd.k; ++i) {
            nd.row_skel[size_t(i)] = i64(v[at + 2 + size_t(i)]);
            nd.col_skel[size_t(i)] = i64(v[at + 2 + size_t(nd.k + i)]);
          }
          at += 2 + size_t(2 * nd.k);
        }
      }
    }
    // interpolation matrices u (row) and v (col), c x k each, then b_sib
    auto st = std::make_unique<LevelStore>();
    st->o_u.resize(L);
    st->o_v.resize(L);
    st->o_b.resize(L);
    i64 tot = 0;
    for (size_t q = 0; q < L; ++q) {
      const i64 c = i64(rc[q].size());
      st->o_u[q] = tot;
      tot += c * kfin[q];
      st->o_v[q] = tot;
      tot += i64(cc[q].size()) * kfin[q];
    }
    for (size_t q = 0; q < L; ++q) {  // b_sib sizes need the sibling's k (remote when sharded)
      const i64 id = ids[q];
      const i64 sib = op->sib(id);
      st->o_b[q] = tot;
      tot += kfin[q] * op->nodes[size_t(sib)].k;
    }
    st->buf.resize(size_t(std::max<i64>(tot, 1)));
    for (size_t r = 0; r < rounds.size(); ++r) {
      std::vector<i64> ks(rounds[r]->probs.size(), 0);
      std::vector<double*> P(ks.size(), nullptr);
      std::vector<int> ldp(ks.size(), 1);
      for (size_t q = 0; q < L; ++q) {
        if (row_round[q] == int(r)) {
          ks[row_pi[q]] = kfin[q];
          P[row_pi[q]] = st->buf.get() + st->o_u[q];
          ldp[row_pi[q]] = std::max<int>(1, int(rc[q].size()));
        }
        if (col_round[q] == int(r)) {
          ks[col_pi[q]] = kfin[q];
          P[col_pi[q]] = st->buf.get() + st->o_v[q];
          ldp[col_pi[q]] = std::max<int>(1, int(cc[q].size()));
        }
      }
      rounds[r]->ids.interp(ks, P, ldp, s);
    }
    {  // b_sib = entries(row_skel, sibling col_skel)
      std::vector<i64> ri, ci;
      std::vector<BlockJob> jobs;
      i64 mx = 0;
      for (size_t q = 0; q < L; ++q) {
        const auto& nd = op->nodes[size_t(ids[q])];
        const auto& sb = op->nodes[size_t(op->sib(ids[q]))];
        BlockJob j{};
        j.row_off = i64(ri.size());
        j.col_off = i64(ci.size());
        j.nr = int(nd.k);
        j.nc = int(sb.k);
        j.out_off = st->o_b[q];
        j.ld = std::max<int>(1, int(nd.k));
        ri.insert(ri.end(), nd.row_skel.begin(), nd.row_skel.end());
        ci.insert(ci.end(), sb.col_skel.begin(), sb.col_skel.end());
        mx = std::max<i64>(mx, i64(j.nr) * j.nc);
        B.max_block = std::max<i64>(B.max_block, i64(j.nr) * j.nc);
        jobs.push_back(j);
      }
      DevBuf<i64> dri, dci;
      DevBuf<BlockJob> dj;
      dri.upload(ri, s);
      dci.upload(ci, s);
      dj.upload(jobs, s);
      if (o.entries)
        host_block_jobs(*o.entries, jobs, ri, ci, st->buf.get(), s);
      else
        launch_block_jobs(eo.view(), dj.get(), int(jobs.size()), mx, dri.get(), dci.get(), st->buf.get(), s);
      SBX_CUDA(cudaStreamSynchronize(s));
    }
    if (G > 1 && depth == gdep) {  // the subtree roots' couplings, for the top levels' inverse on every rank
      std::vector<double> pk;
      for (size_t q = 0; q < L; ++q) {
        const auto& nd = op->nodes[size_t(ids[q])];
        const i64 ks = op->nodes[size_t(op->sib(ids[q]))].k;
        std::vector<double> b(static_cast<size_t>(nd.k * ks));
        if (!b.empty()) {
          SBX_CUDA(cudaMemcpyAsync(b.data(), st->buf.get() + st->o_b[q], b.size() * 8, cudaMemcpyDeviceToHost, s));
          SBX_CUDA(cudaStreamSynchronize(s));
        }
        pk.push_back(double(ids[q]));
        pk.insert(pk.end(), b.begin(), b.end());
      }
      const auto all = gather_host(*comm, pk, s);
      for (int r = 0; r < G; ++r) {
        if (r == P) continue;
        const auto& v = all[size_t(r)];
        for (size_t at = 0; at < v.size();) {
          const i64 id = i64(v[at]);
          const i64 cnt = op->nodes[size_t(id)].k * op->nodes[size_t(op->sib(id))].k;
          remote_b_off[size_t(id)] = i64(remote_b.size());
          remote_b.insert(remote_b.end(), v.begin() + i64(at) + 1, v.begin() + i64(at) + 1 + cnt);
          at += 1 + size_t(cnt);
        }
      }
    }
    if (fz) {  // this level's inverse inputs are complete: hand it to the inversion thread
      const LevelStore& S = *st;
      i64 tot2 = 0;
      for (size_t q = 0; q < L; ++q) {
        HbsNodeH& nd = op->nodes[size_t(ids[q])];
        nd.c = i64(rc[q].size());
        tot2 += nd.k * nd.k + 2 * nd.c * nd.k + nd.c * nd.c;
      }
      DevBuf<double>& sb = fz->stage[size_t(depth)];
      sb.resize(size_t(std::max<i64>(tot2, 1)));
      i64 off = 0;
      for (size_t q = 0; q < L; ++q) {
        const HbsNodeH& nd = op->nodes[size_t(ids[q])];
        InvSrc& p = fz->P[size_t(ids[q])];
        p.u = S.buf.get() + S.o_u[q];
        p.v = S.buf.get() + S.o_v[q];
        p.b = S.buf.get() + S.o_b[q];
        p.dhat = sb.get() + off;
        off += nd.k * nd.k;
        p.e = sb.get() + off;
        off += nd.c * nd.k;
        p.fg = sb.get() + off;
        off += (nd.k + nd.c) * nd.c;
      }
    }
    stores[size_t(depth)] = std::move(st);
    phase_mark("hbs: interp + b_sib", s);
    SBX_CUDA(cudaStreamSynchronize(s));
    if (fz) fz->publish(depth);
  }
  if (fz) {  // the root: c_0 = k_l + k_r (or the whole single leaf)
    HbsNodeH& r0 = op->nodes[0];
    r0.c = r0.is_leaf() ? 2 * (r0.end - r0.begin) : op->nodes[size_t(r0.left)].k + op->nodes[size_t(r0.right)].k;
    fz->rootg.resize(size_t(std::max<i64>(r0.c * r0.c, 1)));
    fz->publish(0);
  }
  phase_mark("hbs: levels done", s);
  op->max_block_drawn = B.max_block;
  if (fz) {  // the layout below rewrites node fields the inversion thread reads
    fz->th.join();
    if (fz->err) std::rethrow_exception(fz->err);
  }
  // final arena: layout by ranks, then place u, v, v^T, d, b_sib
  hbs_layout(*op);
  std::vector<CopyJob> cj;
  double* A = op->arena.get();
  DevBuf<double> d_remote_b;
  if (!remote_b.empty()) d_remote_b.upload(remote_b, s);
  for (size_t i = 0; i < nn; ++i) {
    const auto& nd = op->nodes[i];
    const int k = int(nd.k), c = int(nd.c);
    if (!mine[i]) {  // sharded: another rank's subtree; its root's coupling block only
      const i64 ks = i ? op->nodes[size_t(op->sib(i64(i)))].k : 0;
      if (op->has(i) && remote_b_off[i] >= 0 && k > 0 && ks > 0)
        cj.push_back({d_remote_b.get() + remote_b_off[i], A + nd.o_b, k, int(ks), k, k, 0, 0});
      continue;
    }
    if (nd.is_leaf()) {  // d below v^T in vd
      const int vld = (i == 0) ? c : k + c;
      cj.push_back({dstore.get() + d_off[i], A + nd.o_vd + (i == 0 ? 0 : k), c, c, c, vld, 0, 0});
    }
    if (i == 0) continue;
    const LevelStore& st = *stores[size_t(nd.depth)];
    const size_t q = size_t(pos_in_level[i]);
    const double* u = st.buf.get() + st.o_u[q];
    const double* v = st.buf.get() + st.o_v[q];
    if (k > 0 && c > 0) {
      cj.push_back({u, A + nd.o_u, c, k, c, c, 0, 0});
      cj.push_back({v, A + nd.o_v, c, k, c, c, 0, 0});
      const int vld = k + (nd.is_leaf() ? c : 0);
      cj.push_back({v, A + nd.o_vd, k, c, c, vld, 1, 0});
    }
    const i64 ks = op->nodes[size_t(op->sib(i64(i)))].k;
    if (k > 0 && ks > 0) cj.push_back({st.buf.get() + st.o_b[q], A + nd.o_b, k, int(ks), k, k, 0, 0});
  }
  copy_batched(cj, s);
  SBX_CUDA(cudaStreamSynchronize(s));
  op->has_apply = true;
  if (fz) {
    SBX_CUDA(cudaStreamWaitEvent(s, fz->done, 0));
    std::vector<CopyJob> ij;
    double* A2 = op->arena.get();
    for (size_t i = 1; i < nn; ++i) {
      const auto& nd = op->nodes[i];
      const InvSrc& p = fz->P[i];
      const int k = int(nd.k), c = int(nd.c);
      if (k > 0) ij.push_back({p.dhat, A2 + nd.o_dhat, k, k, k, k, 0, 0});
      if (k > 0 && c > 0) ij.push_back({p.e, A2 + nd.o_e, c, k, c, c, 0, 0});
      if (c > 0) ij.push_back({p.fg, A2 + nd.o_fg, k + c, c, k + c, k + c, 0, 0});
    }
    const int c0 = int(op->nodes[0].c);
    if (c0 > 0) ij.push_back({fz->rootg.get(), A2 + op->o_root_g, c0, c0, c0, c0, 0, 0});
    copy_batched(ij, s);
    const double thr = std::max(std::min(10.0 * op->eps, 1e-6), 1e-14);  // hbs.cpp:429
    check_gates(*op, fz->gates, thr, s);
    SBX_CUDA(cudaStreamSynchronize(s));
    phase_mark("hbs: fused inverse joined", s);
    op->has_inverse = true;
    op->solve_plan.built = false;
  }
  return op;
}
}  // namespace

std::unique_ptr<HbsOp> hbs_compress_device(const Geom& g, int formulation, double mu, const i64* nodes,
                                           i64 n_nodes, const HbsBuildOptions& o, cudaStream_t s) {
  return compress_impl(g, formulation, mu, nodes, n_nodes, o, s, false);
}

std::unique_ptr<HbsOp> hbs_compress_invert_device(const Geom& g, int formulation, double mu, const i64* nodes,
                                                  i64 n_nodes, const HbsBuildOptions& o, cudaStream_t s) {
  return compress_impl(g, formulation, mu, nodes, n_nodes, o, s, true);
}

void hbs_invert_device(HbsOp& op, cudaStream_t s) {
  require(!op.nodes.empty(), "hbs_invert: empty operator");
  require(op.has_apply, "hbs_invert: operator has no forward factors");
  const double thr = std::max(std::min(10.0 * op.eps, 1e-6), 1e-14);  // hbs.cpp:429
  double* A = op.arena.get();
  const size_t nn = op.nodes.size();
  std::vector<InvSrc> P(nn);
  for (size_t i = 0; i < nn; ++i) {
    const auto& nd = op.nodes[i];
    InvSrc& p = P[i];
    if (nd.is_leaf()) {
      p.d = A + nd.o_vd + (i == 0 ? 0 : nd.k);
      p.ldd = int(i == 0 ? nd.c : nd.k + nd.c);
    }
    if (i == 0) continue;
    p.u = A + nd.o_u;
    p.v = A + nd.o_v;
    p.b = A + nd.o_b;
    p.dhat = A + nd.o_dhat;
    p.e = A + nd.o_e;
    p.fg = A + nd.o_fg;
  }
  // sharded operator: this rank inverts its subtree, then (after the subtree
  // roots' dhat blocks are exchanged) the top levels like every other rank
  std::vector<char> own(nn, 1);
  if (op.sharded()) {
    require(op.comm != nullptr, "hbs_invert: sharded operator without its communicator");
    std::vector<i64> owner(nn, -1);
    i64 q = 0;
    for (size_t i = 0; i < nn; ++i) {
      if (op.nodes[i].depth == op.shard_g) owner[i] = q++;
      else if (op.nodes[i].depth > op.shard_g) owner[i] = owner[size_t(op.nodes[i].parent)];
      own[i] = owner[i] < 0 || owner[i] == op.shard_p;
    }
  }
  std::vector<std::unique_ptr<Gate>> gates;
  for (int depth = op.max_depth; depth >= 0; --depth) {
    std::vector<size_t> ids;
    for (size_t i = 0; i < nn; ++i)
      if (op.nodes[i].depth == depth && own[i]) ids.push_back(i);
    invert_level(op, ids, P, A + op.o_root_g, gates, s);
    if (op.sharded() && op.shard_G > 1 && depth == op.shard_g) {
      std::vector<double> pk;
      for (size_t i : ids) {
        const i64 k = op.nodes[i].k;
        std::vector<double> d(static_cast<size_t>(k * k));
        if (!d.empty()) {
          SBX_CUDA(cudaMemcpyAsync(d.data(), A + op.nodes[i].o_dhat, d.size() * 8, cudaMemcpyDeviceToHost, s));
          SBX_CUDA(cudaStreamSynchronize(s));
        }
        pk.push_back(double(i));
        pk.insert(pk.end(), d.begin(), d.end());
      }
      const auto all = gather_host(*op.comm, pk, s);
      for (int r = 0; r < op.shard_G; ++r) {
        if (r == op.shard_p) continue;
        const auto& v = all[size_t(r)];
        for (size_t at = 0; at < v.size();) {
          const auto& nd = op.nodes[size_t(v[at])];
          const size_t cnt = size_t(nd.k * nd.k);
          if (cnt)
            SBX_CUDA(cudaMemcpyAsync(A + nd.o_dhat, v.data() + at + 1, cnt * 8, cudaMemcpyHostToDevice, s));
          at += 1 + cnt;
        }
      }
      SBX_CUDA(cudaStreamSynchronize(s));
    }
  }
  check_gates(op, gates, thr, s);
  phase_mark("inv: done", s);
  op.has_inverse = true;
  op.solve_plan.built = false;
}

}  // namespace sbx
