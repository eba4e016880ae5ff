// Device two-step ID update compression (reference lowrank.cpp:253-327 with
// proxy.cpp:46-302 and idlib.cpp).  Host code keeps the index bookkeeping
// (far/near split, partition trees, skeleton lists); W^T assembly, CPQR,
// interpolation, the hierarchical merges (DMMA GEMMs) and the R blocks run
// on the device.
//
// The final randomized_row_id of the stacked factor L1 (idlib.cpp:101-132)
// is evaluated as the deterministic row ID of L1: the reference's own
// comment (idlib.cpp:115-118) notes that its Gaussian sketch is reduced to an
// exact orthogonal rotation G of the row space, which leaves row norms,
// angles and the eps-rank rule unchanged, so CPQR((L1 G)^T) and CPQR(L1^T)
// select the same pivots and interpolation matrix in exact arithmetic.
#include "update.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <numeric>
#include <set>
#include <thread>
#include <memory>

#include "dense.hpp"
#include "els.hpp"
#include "entries.hpp"
#include "idengine.hpp"

namespace sbx {

namespace {
// Diagnostics (SBX_HOST_TIMING): host wall time between marks of the update's
// setup, without device synchronisation.
struct HostMarks {
  bool on = std::getenv("SBX_HOST_TIMING") != nullptr;
  std::chrono::steady_clock::time_point last = std::chrono::steady_clock::now();
  void operator()(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[sbx-host] %-28s %8.1f us\n", what,
                 std::chrono::duration<double, std::micro>(now - last).count());
    last = now;
  }
};
}  // namespace


namespace {

struct RowIdResult {
  i64 m = 0, k = 0;
  std::vector<i64> J;  // skeleton first
  DevBuf<double> P;    // m x k
};

// Fills W^T for each candidate list (row ids of the implied W) into buf.
using WtBuilder = std::function<void(const std::vector<std::vector<i64>>&, std::vector<IdProblem>&,
                                     DevBuf<double>&)>;

struct Chunk {
  std::vector<i64> rows, skel;
  const double* P = nullptr;  // |rows| x k (column-major)
  i64 k = 0;
};

// One hierarchy of row IDs: m rows cut into leaves, W^T built by `build`.
struct HierSpec {
  i64 m = 0;
  std::vector<std::vector<i64>> leaves;
  WtBuilder build;
};

// hierarchical_row_id (proxy.cpp:193-247) / chunked near_row_id
// (lowrank.cpp:76-124): leaf IDs, then pairwise merges of skeleton rows.
// Independent hierarchies (the far-field IDs at two proxy sample counts,
// the near-field blocks, ...) advance in lockstep: every tree level of all
// of them is one batched CPQR, so the step pays max(depth) dependent levels
// instead of the sum.
std::vector<RowIdResult> hierarchical_id_multi(const std::vector<HierSpec>& specs, double eps,
                                               cudaStream_t s) {
  const size_t H = specs.size();
  std::vector<std::unique_ptr<DevBuf<double>>> keep;
  std::vector<std::vector<Chunk>> level(H);
  static const bool no_defer = std::getenv("SBX_NO_DEFER") != nullptr;  // diagnostics
  std::function<void()> deferred;  // the previous round's interpolation / merge launches
  auto run_deferred = [&] {
    if (deferred) {
      auto f = std::move(deferred);
      deferred = nullptr;
      f();
    }
  };
  // leaves
  {
    std::vector<IdProblem> all;
    std::vector<std::pair<size_t, size_t>> who;  // problem -> (hierarchy, leaf)
    for (size_t h = 0; h < H; ++h) {
      if (specs[h].leaves.empty()) continue;
      std::vector<IdProblem> probs;
      auto buf = std::make_unique<DevBuf<double>>();
      specs[h].build(specs[h].leaves, probs, *buf);
      for (size_t q = 0; q < probs.size(); ++q) who.push_back({h, q});
      all.insert(all.end(), probs.begin(), probs.end());
      keep.push_back(std::move(buf));
    }
    auto idsp = std::make_shared<IdBatch>();
    IdBatch& ids = *idsp;
    HostMarks hm;
    ids.factor(all, eps, s);
    hm("  leaves: factor (host+sync)");
    std::vector<i64> ks(all.size()), off(all.size());
    i64 tot = 0;
    for (size_t p = 0; p < all.size(); ++p) {
      ks[p] = ids.eps_rank(p, eps);
      off[p] = tot;
      tot += i64(specs[who[p].first].leaves[who[p].second].size()) * ks[p];
    }
    auto pb = std::make_unique<DevBuf<double>>(size_t(std::max<i64>(tot, 1)));
    std::vector<double*> P(all.size());
    std::vector<int> ldp(all.size());
    for (size_t p = 0; p < all.size(); ++p) {
      P[p] = pb->get() + off[p];
      ldp[p] = std::max<int>(1, int(specs[who[p].first].leaves[who[p].second].size()));
    }
    hm("  leaves: ranks + alloc");
    // the interpolation matrices are not needed by the next round's W^T
    // assembly or its factorization: their launch (and its host-side job
    // tables) is queued after that assembly's launches, so the device
    // assembles while the host prepares them (SBX_NO_DEFER: at once)
    deferred = [idsp, ks, P, ldp, s] { idsp->interp(ks, P, ldp, s); };
    if (no_defer) run_deferred();
    hm("  leaves: interp launch");
    for (size_t p = 0; p < all.size(); ++p) {
      const auto& lf = specs[who[p].first].leaves[who[p].second];
      Chunk c;
      c.rows = lf;
      c.k = ks[p];
      for (i64 i = 0; i < c.k; ++i) c.skel.push_back(lf[size_t(ids.perm(p)[size_t(i)])]);
      c.P = P[p];
      level[who[p].first].push_back(std::move(c));
    }
    keep.push_back(std::move(pb));
    hm("  leaves: chunks");
    phase_mark("  hier: leaves", s);
  }
  for (;;) {
    bool any = false;
    for (size_t h = 0; h < H; ++h) any |= level[h].size() > 1;
    if (!any) break;
    std::vector<IdProblem> all;
    std::vector<std::vector<std::vector<i64>>> unis(H);
    std::vector<size_t> first(H, 0);
    for (size_t h = 0; h < H; ++h) {
      first[h] = all.size();
      const size_t npair = level[h].size() / 2;
      unis[h].resize(npair);
      for (size_t q = 0; q < npair; ++q) {
        unis[h][q] = level[h][2 * q].skel;
        unis[h][q].insert(unis[h][q].end(), level[h][2 * q + 1].skel.begin(),
                          level[h][2 * q + 1].skel.end());
      }
      if (npair == 0) continue;
      std::vector<IdProblem> probs;
      auto buf = std::make_unique<DevBuf<double>>();
      specs[h].build(unis[h], probs, *buf);
      all.insert(all.end(), probs.begin(), probs.end());
      keep.push_back(std::move(buf));
    }
    run_deferred();  // behind this round's W^T assembly launches
    auto idsp = std::make_shared<IdBatch>();
    IdBatch& ids = *idsp;
    ids.factor(all, eps, s);
    std::vector<i64> ks(all.size()), ioff(all.size()), poff(all.size());
    i64 itot = 0, ptot = 0;
    for (size_t h = 0; h < H; ++h)
      for (size_t q = 0; q < unis[h].size(); ++q) {
        const size_t p = first[h] + q;
        ks[p] = ids.eps_rank(p, eps);
        ioff[p] = itot;
        itot += i64(unis[h][q].size()) * ks[p];
        poff[p] = ptot;
        ptot += i64(level[h][2 * q].rows.size() + level[h][2 * q + 1].rows.size()) * ks[p];
      }
    auto ib = std::make_unique<DevBuf<double>>(size_t(std::max<i64>(itot, 1)));
    auto pb = std::make_unique<DevBuf<double>>(size_t(std::max<i64>(ptot, 1)));
    std::vector<double*> IP(all.size());
    std::vector<int> ldi(all.size());
    for (size_t h = 0; h < H; ++h)
      for (size_t q = 0; q < unis[h].size(); ++q) {
        const size_t p = first[h] + q;
        IP[p] = ib->get() + ioff[p];
        ldi[p] = std::max<int>(1, int(unis[h][q].size()));
      }
    std::vector<GemmJob> gj;
    for (size_t h = 0; h < H; ++h) {
      std::vector<Chunk> next;
      for (size_t q = 0; q < unis[h].size(); ++q) {
        const size_t p = first[h] + q;
        const Chunk& a = level[h][2 * q];
        const Chunk& b = level[h][2 * q + 1];
        Chunk c;
        c.rows = a.rows;
        c.rows.insert(c.rows.end(), b.rows.begin(), b.rows.end());
        c.k = ks[p];
        for (i64 i = 0; i < c.k; ++i) c.skel.push_back(unis[h][q][size_t(ids.perm(p)[size_t(i)])]);
        double* P = pb->get() + poff[p];
        c.P = P;
        const int ra = int(a.rows.size()), rb = int(b.rows.size()), ld = ra + rb;
        const int ka = int(a.skel.size()), kb = int(b.skel.size()), k = int(c.k);
        if (k > 0) {
          // out.P = [a.P * id.P(0:ka, :); b.P * id.P(ka:, :)]  (proxy.cpp:187-189)
          if (ka == 0 || kb == 0) SBX_CUDA(cudaMemsetAsync(P, 0, size_t(ld) * k * 8, s));
          if (ka > 0)
            gj.push_back({a.P, IP[p], P, ra, k, ka, std::max(ra, 1), ldi[p], ld, 0, 0, 1.0, 0.0});
          if (kb > 0)
            gj.push_back({b.P, IP[p] + ka, P + ra, rb, k, kb, std::max(rb, 1), ldi[p], ld, 0, 0, 1.0, 0.0});
        }
        next.push_back(std::move(c));
      }
      if (level[h].size() % 2 == 1) next.push_back(level[h].back());
      if (!unis[h].empty()) level[h] = std::move(next);
    }
    deferred = [idsp, ks, IP, ldi, gj, s] {
      idsp->interp(ks, IP, ldi, s);
      gemm_batched(gj, s);
    };
    if (no_defer) run_deferred();
    phase_mark("  hier: merge level", s);
    keep.push_back(std::move(ib));
    keep.push_back(std::move(pb));
  }
  run_deferred();
  std::vector<RowIdResult> outs(H);
  // the roots' interpolation matrices scattered into the m-row outputs: all
  // hierarchies in one launch (one upload of the concatenated row maps)
  std::vector<i64> maps;
  std::vector<std::pair<size_t, i64>> map_off(H, {0, -1});
  for (size_t h = 0; h < H; ++h) {
    if (level[h].empty() || level[h].front().k <= 0) continue;
    map_off[h] = {maps.size(), 0};
    maps.insert(maps.end(), level[h].front().rows.begin(), level[h].front().rows.end());
  }
  DevBuf<i64> d_maps;
  if (!maps.empty()) d_maps.upload(maps, s);
  std::vector<ScatterJob> root_jobs;
  for (size_t h = 0; h < H; ++h) {
    RowIdResult& out = outs[h];
    const i64 m = specs[h].m;
    out.m = m;
    if (level[h].empty()) {
      out.J.resize(size_t(m));
      std::iota(out.J.begin(), out.J.end(), i64(0));
      continue;
    }
    const Chunk& root = level[h].front();
    out.k = root.k;
    out.P.resize(size_t(std::max<i64>(m * out.k, 1)));
    if (out.k > 0) {
      SBX_CUDA(cudaMemsetAsync(out.P.get(), 0, size_t(m * out.k) * 8, s));
      root_jobs.push_back({root.P, out.P.get(), d_maps.get() + map_off[h].first, int(root.rows.size()), int(out.k),
                           std::max<int>(1, int(root.rows.size())), int(m), 0, 0, 1.0});
    }
    out.J = root.skel;
    std::vector<char> in(size_t(m), 0);
    for (i64 x : root.skel) in[size_t(x)] = 1;
    for (i64 x : root.rows)
      if (!in[size_t(x)]) out.J.push_back(x);
  }
  scatter_batched(root_jobs, s);
  return outs;
}

RowIdResult hierarchical_id(i64 m, const std::vector<std::vector<i64>>& leaves,
                            const WtBuilder& build, double eps, cudaStream_t s) {
  auto r = hierarchical_id_multi({HierSpec{m, leaves, build}}, eps, s);
  return std::move(r[0]);
}

// Direct row ID of one implicitly built W (row_id(eval(all rows))).
RowIdResult direct_id(i64 m, const WtBuilder& build, double eps, cudaStream_t s) {
  std::vector<std::vector<i64>> one(1);
  one[0].resize(size_t(m));
  std::iota(one[0].begin(), one[0].end(), i64(0));
  std::vector<IdProblem> probs;
  DevBuf<double> buf;
  build(one, probs, buf);
  IdBatch ids;
  ids.factor(probs, eps, s);
  RowIdResult out;
  out.m = m;
  out.k = ids.eps_rank(0, eps);
  out.P.resize(size_t(std::max<i64>(m * out.k, 1)));
  if (out.k > 0) ids.interp({out.k}, {out.P.get()}, {std::max<int>(1, int(m))}, s);
  out.J.assign(ids.perm(0).begin(), ids.perm(0).end());
  return out;
}

// W^T builder for the proxy interaction (proxy.cpp:136-162): rows of W are
// scalars 2p+c of the point list `nodes` (global ids in g); columns are four
// per circle sample plus the completion column.
WtBuilder proxy_builder(const EntryView& v, const std::vector<i64>& nodes,
                        const std::vector<ProxyCircleH>& circles, double factor, int ns, bool with_null,
                        cudaStream_t s) {
  return [&v, &nodes, &circles, factor, ns, with_null, s](
             const std::vector<std::vector<i64>>& lists, std::vector<IdProblem>& probs,
             DevBuf<double>& buf) {
    const int nc = int(circles.size());
    const int M = 4 * ns * nc + (with_null ? 1 : 0);
    std::vector<i64> off;
    i64 tot = 0;
    probs.clear();
    for (const auto& l : lists) {
      off.push_back(tot);
      tot += i64(M) * i64(l.size());
      probs.push_back({nullptr, M, int(l.size()), std::max(M, 1)});
    }
    buf.resize(size_t(std::max<i64>(tot, 1)));
    std::vector<i64> cand;
    std::vector<ProxyJob> jobs;
    int max_n = 0;
    for (size_t q = 0; q < lists.size(); ++q) {
      probs[q].wt = buf.get() + off[q];
      const i64 co = i64(cand.size());
      for (i64 r : lists[q]) cand.push_back(2 * nodes[size_t(r / 2)] + (r & 1));
      if (lists[q].empty()) continue;
      max_n = std::max(max_n, int(lists[q].size()));
      for (int c = 0; c < nc; ++c) {
        ProxyJob j{};
        j.cand_off = co;
        j.n = int(lists[q].size());
        j.ns = ns;
        j.cx = circles[size_t(c)].cx;
        j.cy = circles[size_t(c)].cy;
        j.rad = factor * circles[size_t(c)].r0;
        j.out_off = off[q] + i64(4) * ns * c;
        j.ld = M;
        j.kind = 2;
        j.with_null = (with_null && c == nc - 1) ? 1 : 0;
        jobs.push_back(j);
      }
    }
    DevBuf<i64> dc;
    DevBuf<ProxyJob> dj;
    dc.upload(cand, s);
    dj.upload(jobs, s);
    // index tables return to the stream-ordered pool: no host sync needed
    launch_proxy_jobs(v, dj.get(), int(jobs.size()), ns, max_n, dc.get(), buf.get(), s);
  };
}

// W^T builder for a block of the entry oracle: W(r, c) = A(rowsc[r], colsc[c]).
WtBuilder entry_builder(const EntryView& v, const std::vector<i64>& rowsc,
                        const std::vector<i64>& colsc, cudaStream_t s) {
  return [&v, &rowsc, &colsc, s](const std::vector<std::vector<i64>>& lists,
                                 std::vector<IdProblem>& probs, DevBuf<double>& buf) {
    const int M = int(colsc.size());
    std::vector<i64> off;
    i64 tot = 0;
    probs.clear();
    for (const auto& l : lists) {
      off.push_back(tot);
      tot += i64(M) * i64(l.size());
      probs.push_back({nullptr, M, int(l.size()), std::max(M, 1)});
    }
    buf.resize(size_t(std::max<i64>(tot, 1)));
    std::vector<i64> cand;
    std::vector<NearJob> jobs;
    i64 mx = 0;
    for (size_t q = 0; q < lists.size(); ++q) {
      probs[q].wt = buf.get() + off[q];
      const i64 co = i64(cand.size());
      for (i64 r : lists[q]) cand.push_back(rowsc[size_t(r)]);
      if (lists[q].empty() || M == 0) continue;
      NearJob j{};
      j.cand_off = co;
      j.near_off = 0;
      j.n = int(lists[q].size());
      j.n_near = M;
      j.out_off = off[q];
      j.ld = M;
      j.transpose = 0;
      jobs.push_back(j);
      mx = std::max<i64>(mx, i64(M) * j.n);
    }
    DevBuf<i64> dc, dn;
    DevBuf<NearJob> dj;
    dc.upload(cand, s);
    dn.upload(colsc, s);
    dj.upload(jobs, s);
    launch_near_jobs(v, dj.get(), int(jobs.size()), mx, dc.get(), dn.get(), buf.get(), s);
  };
}

bool inside_any_div(const std::vector<ProxyCircleH>& cs, double div, double x, double y) {
  for (const auto& c : cs)
    if (std::sqrt((x - c.cx) * (x - c.cx) + (y - c.cy) * (y - c.cy)) < div * c.r0) return true;
  return false;
}

// compress_block_far (proxy.cpp:251-302) over point list `nodes` of g.
RowIdResult compress_block_far(const EntryView& v, const Geom& g, const std::vector<i64>& nodes,
                               const std::vector<ProxyCircleH>& circles, bool basis, bool with_null,
                               const std::vector<std::vector<i64>>& tree_leaves, double eps,
                               cudaStream_t s) {
  const double bas = 1.5, div = 3.0;
  require(!circles.empty(), "proxy geometry has no circles");
  for (i64 nd : nodes) {
    const bool in_div = inside_any_div(circles, div, g.x[size_t(nd)], g.y[size_t(nd)]);
    if (basis && in_div) throw Error(5, "far row point inside a division circle");
    if (!basis && !in_div) throw Error(5, "row point outside every division circle");
  }
  const i64 m = 2 * i64(nodes.size());
  if (nodes.empty()) {
    RowIdResult out;
    return out;
  }
  std::vector<std::vector<i64>> leaves;
  for (const auto& lf : tree_leaves) {
    std::vector<i64> rows;
    for (i64 p : lf) {
      rows.push_back(2 * p);
      rows.push_back(2 * p + 1);
    }
    leaves.push_back(std::move(rows));
  }
  const double factor = basis ? bas : div;
  // 64 and 128 samples are always both computed (proxy.cpp:289-300): one batch
  auto two = hierarchical_id_multi({HierSpec{m, leaves, proxy_builder(v, nodes, circles, factor, 64, with_null, s)},
                                    HierSpec{m, leaves, proxy_builder(v, nodes, circles, factor, 128, with_null, s)}},
                                   eps, s);
  bool settled = std::llabs(two[1].k - two[0].k) <= 2;
  RowIdResult prev = std::move(two[1]);
  for (int n = 256; !settled && n <= 2048; n *= 2) {
    RowIdResult cur =
        hierarchical_id(m, leaves, proxy_builder(v, nodes, circles, factor, n, with_null, s), eps, s);
    settled = std::llabs(cur.k - prev.k) <= 2;
    prev = std::move(cur);
  }
  return prev;
}

// near_row_id (lowrank.cpp:62-125): W(r, c) = A(rowsc[r], colsc[c]).
RowIdResult near_row_id(const EntryView& v, const std::vector<i64>& rowsc,
                        const std::vector<i64>& colsc, double eps, std::vector<std::string>& notes,
                        const char* tag, cudaStream_t s) {
  const i64 nr = i64(rowsc.size()), ncl = i64(colsc.size());
  if (nr == 0 || ncl == 0) {
    RowIdResult out;
    out.m = nr;
    out.J.resize(size_t(nr));
    std::iota(out.J.begin(), out.J.end(), i64(0));
    return out;
  }
  const WtBuilder b = entry_builder(v, rowsc, colsc, s);
  if (nr * ncl <= (i64(1) << 22)) return direct_id(nr, b, eps, s);
  notes.push_back(std::string(tag) + ": near block over memory budget, using row partition");
  std::vector<std::vector<i64>> leaves;
  for (i64 st = 0; st < nr; st += 256) {
    std::vector<i64> l;
    for (i64 r = st; r < std::min(st + 256, nr); ++r) l.push_back(r);
    leaves.push_back(std::move(l));
  }
  return hierarchical_id(nr, leaves, b, eps, s);
}

// compress_block_far split for the lockstep driver: validation and the two
// first hierarchies (64 and 128 samples), then the doubling loop on the
// results (proxy.cpp:251-302).
struct FarPrep {
  bool basis = true;
  double factor = 1.5;
  i64 m = 0;
  std::vector<std::vector<i64>> leaves;
};
FarPrep far_prepare(const Geom& g, const std::vector<i64>& nodes, const std::vector<ProxyCircleH>& circles,
                    bool basis, const std::vector<std::vector<i64>>& tree_leaves) {
  const double div = 3.0;
  require(!circles.empty(), "proxy geometry has no circles");
  for (i64 nd : nodes) {
    const bool in_div = inside_any_div(circles, div, g.x[size_t(nd)], g.y[size_t(nd)]);
    if (basis && in_div) throw Error(5, "far row point inside a division circle");
    if (!basis && !in_div) throw Error(5, "row point outside every division circle");
  }
  FarPrep f;
  f.basis = basis;
  f.factor = basis ? 1.5 : div;
  f.m = 2 * i64(nodes.size());
  if (nodes.empty()) return f;
  for (const auto& lf : tree_leaves) {
    std::vector<i64> rows(2 * lf.size());
    for (size_t i = 0; i < lf.size(); ++i) {
      rows[2 * i] = 2 * lf[i];
      rows[2 * i + 1] = 2 * lf[i] + 1;
    }
    f.leaves.push_back(std::move(rows));
  }
  return f;
}

RowIdResult far_settle(const EntryView& v, const std::vector<i64>& nodes, const std::vector<ProxyCircleH>& circles,
                       bool with_null, const FarPrep& f, RowIdResult r64, RowIdResult r128, double eps,
                       cudaStream_t s) {
  if (f.leaves.empty()) return RowIdResult{};
  bool settled = std::llabs(r128.k - r64.k) <= 2;
  RowIdResult prev = std::move(r128);
  for (int n = 256; !settled && n <= 2048; n *= 2) {
    RowIdResult cur =
        hierarchical_id(f.m, f.leaves, proxy_builder(v, nodes, circles, f.factor, n, with_null, s), eps, s);
    settled = std::llabs(cur.k - prev.k) <= 2;
    prev = std::move(cur);
  }
  return prev;
}

// near_row_id as a hierarchy spec: one leaf (direct ID) up to 2^22 entries,
// else 256-row chunks (lowrank.cpp:62-125).
HierSpec near_spec(const EntryView& v, const std::vector<i64>& rowsc, const std::vector<i64>& colsc,
                   std::vector<std::string>& notes, const char* tag, cudaStream_t s) {
  HierSpec h;
  const i64 nr = i64(rowsc.size()), ncl = i64(colsc.size());
  h.m = nr;
  if (nr == 0 || ncl == 0) return h;
  h.build = entry_builder(v, rowsc, colsc, s);
  const i64 chunk = nr * ncl <= (i64(1) << 22) ? nr : 256;
  if (chunk < nr) notes.push_back(std::string(tag) + ": near block over memory budget, using row partition");
  for (i64 st = 0; st < nr; st += chunk) {
    std::vector<i64> l;
    for (i64 r = st; r < std::min(st + chunk, nr); ++r) l.push_back(r);
    h.leaves.push_back(std::move(l));
  }
  return h;
}

std::vector<i64> scalars(const std::vector<i64>& nodes) {
  std::vector<i64> o(2 * nodes.size());
  i64* d = o.data();
  const i64* n = nodes.data();
  for (size_t i = 0, e = nodes.size(); i < e; ++i) {  // indexed stores: per-step host path
    d[2 * i] = 2 * n[i];
    d[2 * i + 1] = 2 * n[i] + 1;
  }
  return o;
}

}  // namespace

std::vector<ProxyCircleH> make_proxy_circles(const Geom& g, const Plan& plan) {
  std::vector<ProxyCircleH> out;
  if (plan.added_new.empty()) return out;
  const size_t nc = g.comps.size();
  std::vector<std::vector<std::pair<double, double>>> pts(nc);
  std::vector<std::vector<i64>> pans(nc);  // the panels of the added nodes, ascending and unique per component
  for (auto& p : pts) p.reserve(plan.added_new.size() + 2 * 64);
  for (i64 node : plan.added_new) {
    const i64 pid = g.panel_of[size_t(node)];
    const i64 c = g.panels[size_t(pid)].component;
    pts[size_t(c)].push_back({g.x[size_t(node)], g.y[size_t(node)]});
    auto& pc = pans[size_t(c)];
    if (pc.empty() || pc.back() != pid) pc.push_back(pid);  // nodes come panel by panel
  }
  for (auto& pc : pans) {
    std::sort(pc.begin(), pc.end());
    pc.erase(std::unique(pc.begin(), pc.end()), pc.end());
  }
  for (size_t c = 0; c < nc; ++c) {
    auto& p = pts[c];
    if (p.empty()) continue;
    for (i64 pid : pans[c]) {
      const PanelRow& pr = g.panels[size_t(pid)];
      double x, y, a, b, e, f;
      g.comps[c].curve.eval(pr.a, x, y, a, b, e, f);
      p.push_back({x, y});
      g.comps[c].curve.eval(pr.b, x, y, a, b, e, f);
      p.push_back({x, y});
    }
    double sx = 0, sy = 0;
    for (auto& q : p) {
      sx += q.first;
      sy += q.second;
    }
    const double cx = sx / double(p.size()), cy = sy / double(p.size());
    double r0 = 0;
    for (auto& q : p)
      r0 = std::max(r0, std::sqrt((q.first - cx) * (q.first - cx) + (q.second - cy) * (q.second - cy)));
    if (!(r0 > 0.0)) throw Error(3, "refined region has zero spatial extent");
    out.push_back({cx, cy, r0});
  }
  return out;
}

std::unique_ptr<Update> update_compress_device(const Geom& og, const Geom& ng, const Plan& plan,
                                               int form, double mu, double eps, std::uint64_t seed,
                                               cudaStream_t s) {
  (void)seed;  // the sketch is an exact rotation; see the header comment
  require(eps > 0.0 && eps <= 0.1, "compression tolerance out of range");
  auto u = std::make_unique<Update>();
  u->nk2 = 2 * i64(plan.kept_old.size());
  u->nc2 = 2 * i64(plan.cut_old.size());
  u->np2 = 2 * i64(plan.added_new.size());
  if (u->nc2 == 0 && u->np2 == 0) return u;
  // (the entry oracles first: they build the meshes' lazily shared single-layer
  // tables, which the A_pp thread's own oracle must find in place)
  EntryOracle eold(og, form, mu, s), enew(ng, form, mu, s);
  const bool with_null = enew.has_nullspace();
  const double app_eps = eps;  // els_build adopts it when a_oo was built at this eps
  auto t_app = [&](cudaStream_t w) {
    if (plan.added_new.empty()) return;
    try {
      u->app = build_app_solver(ng, plan, form, mu, app_eps, w);
    } catch (const Error&) {
      u->app.reset();  // els_build rebuilds it and reports the error there
    }
    phase_mark("update: A_pp inverse (for els_build)", w);
  };
  static const int par_mode = [] {
    const char* e = std::getenv("SBX_PAR_MODE");
    return e ? std::atoi(e) : 4;
  }();
  // mode 4: the A_pp HBS build runs in a second host thread on the SAME
  // stream; its factorisations and the update's share joint CPQR launches
  // through a rendezvous until one side has no more of them.  The thread
  // starts before the host-side setup below (proxy circles, far / near
  // split, partition trees: ~0.8 ms during which the device would idle).
  std::unique_ptr<IdRendezvous> rv;
  bool rv_entered = true;  // false: the main thread still has to enter the rendezvous
  std::thread app_thread;
  std::exception_ptr app_err;
  if (par_mode == 4 && !plan.added_new.empty()) {
    // the A_pp thread alone at first: its rounds launch on their own until the
    // main thread has finished the setup below and enters with its first batch
    // (SBX_RV_WAIT=1: both counted from the start, the A_pp thread waits)
    static const bool rv_wait = std::getenv("SBX_RV_WAIT") != nullptr;
    rv = std::make_unique<IdRendezvous>(rv_wait ? 2 : 1);
    rv_entered = rv_wait;
    int dev = 0;
    SBX_CUDA(cudaGetDevice(&dev));
    app_thread = std::thread([&, dev] {
      try {
        SBX_CUDA(cudaSetDevice(dev));
        StreamScope ss(s);
        IdRendezvousScope rs(rv.get());
        phase_mark(nullptr, s);
        t_app(s);
      } catch (...) {
        app_err = std::current_exception();
      }
    });
  }
  // on any exception below: main_rs leaves the rendezvous first (so the
  // A_pp thread's pending and later factorisations launch on their own),
  // then the thread is joined before it is destroyed -- never terminate()
  struct JoinOnExit {
    std::thread& t;
    ~JoinOnExit() {
      if (t.joinable()) t.join();
    }
  } join_app{app_thread};
  // (counted from the start only with SBX_RV_WAIT; else it enters below)
  std::unique_ptr<IdRendezvousScope> main_rs_early;
  if (rv && rv_entered) main_rs_early = std::make_unique<IdRendezvousScope>(rv.get());
  HostMarks hm;
  const auto circles = make_proxy_circles(ng, plan);
  hm("circles");
  const double div = 3.0;
  // shared far-field ID over the kept rows (lowrank.cpp:275-287)
  std::vector<i64> far_pos, near_pos;
  for (size_t p = 0; p < plan.kept_new.size(); ++p) {
    const i64 nd = plan.kept_new[p];
    (inside_any_div(circles, div, ng.x[size_t(nd)], ng.y[size_t(nd)]) ? near_pos : far_pos)
        .push_back(i64(p));
  }
  std::vector<i64> far_nodes;
  for (i64 p : far_pos) far_nodes.push_back(plan.kept_new[size_t(p)]);
  hm("far/near split");
  // dyadic-by-distance partition (proxy.cpp:91-129)
  std::vector<std::vector<i64>> ktree;
  {
    const i64 n = i64(far_nodes.size());
    std::vector<i64> order(static_cast<size_t>(n));
    std::iota(order.begin(), order.end(), i64(0));
    std::vector<int> band(static_cast<size_t>(n), 0);
    if (!circles.empty()) {
      for (i64 i = 0; i < n; ++i) {
        double best = INFINITY;
        const double x = ng.x[size_t(far_nodes[size_t(i)])], y = ng.y[size_t(far_nodes[size_t(i)])];
        for (const auto& c : circles)
          best = std::min(best, std::sqrt((x - c.cx) * (x - c.cx) + (y - c.cy) * (y - c.cy)) / c.r0);
        // floor(log2(max(1, best))) (proxy.cpp:91-129) through the binary exponent;
        // log2 itself only within 64 ulp (1.4e-14) of the next power of two,
        // where its rounding decides the band
        const double bb = std::max(1.0, best);
        std::uint64_t bits;
        std::memcpy(&bits, &bb, sizeof bits);
        int e2 = int((bits >> 52) & 0x7ff) - 1023;  // bb >= 1: a normal number
        const std::uint64_t frac = bits & 0xfffffffffffffull;
        if (frac >= 0xfffffffffffffull - 64 || !std::isfinite(bb)) e2 = int(std::floor(std::log2(bb)));
        band[size_t(i)] = e2;
      }
      // stable order by band: a counting sort (bands are a handful of small integers)
      int bmax = 0;
      for (int b : band) bmax = std::max(bmax, b);
      std::vector<i64> start(size_t(bmax) + 2, 0);
      for (int b : band) ++start[size_t(b) + 1];
      for (size_t b = 1; b < start.size(); ++b) start[b] += start[b - 1];
      for (i64 i = 0; i < n; ++i) order[size_t(start[size_t(band[size_t(i)])]++)] = i;
    }
    size_t pos = 0;
    while (pos < order.size()) {
      size_t run = pos + 1;
      while (run < order.size() && band[size_t(order[run])] == band[size_t(order[pos])]) ++run;
      while (pos < run) {
        const size_t take = std::min<size_t>(128, run - pos);
        ktree.emplace_back(order.begin() + long(pos), order.begin() + long(pos + take));
        pos += take;
      }
    }
  }
  phase_mark("update: setup", s);
  hm("bands + ktree");
  const std::vector<i64> far_s = scalars(far_pos), near_s = scalars(near_pos);
  // kept-row blocks kc (old oracle) and kp (new oracle)  (lowrank.cpp:130-180)
  const std::vector<i64> kept_old_s = scalars(plan.kept_old), kept_new_s = scalars(plan.kept_new);
  const std::vector<i64> cut_s = scalars(plan.cut_old), added_s = scalars(plan.added_new);
  hm("scalars");
  auto mapped = [](const std::vector<i64>& map, const std::vector<i64>& idx) {
    std::vector<i64> o;
    o.reserve(idx.size());
    for (i64 i : idx) o.push_back(map[size_t(i)]);
    return o;
  };
  // The five row IDs (far kept, near kc, near kp, far/near pk) are
  // independent until the stacked factor is assembled; they run as
  // concurrent tasks on worker streams, together with the A_pp inverse the
  // following els_build needs (it depends only on the refined mesh).
  RowIdResult far, kc_near, kp_near, pk_far, pk_near;
  std::vector<std::string> notes_kc, notes_kp, notes_pk;
  const bool do_kc = !kept_old_s.empty() && !cut_s.empty();
  const bool do_kp = !kept_new_s.empty() && !added_s.empty();
  const bool do_pk_near = u->np2 > 0 && u->nk2 > 0;
  auto t_far = [&](cudaStream_t w) {
    far = compress_block_far(enew.view(), ng, far_nodes, circles, true, with_null, ktree, eps, w);
    phase_mark("update: far ID (kept)", w);
  };
  auto t_kc = [&](cudaStream_t w) {
    if (!do_kc) return;
    kc_near = near_row_id(eold.view(), mapped(kept_old_s, near_s), cut_s, eps, notes_kc, "kc", w);
    phase_mark("update: kc near ID", w);
  };
  auto t_kp = [&](cudaStream_t w) {
    if (!do_kp) return;
    kp_near = near_row_id(enew.view(), mapped(kept_new_s, near_s), added_s, eps, notes_kp, "kp", w);
    phase_mark("update: kp near ID", w);
  };
  // added rows against the division surface (lowrank.cpp:296-308, 183-238)
  auto t_pk_far = [&](cudaStream_t w) {
    if (plan.added_new.empty()) return;
    std::vector<std::vector<i64>> ptree;
    for (size_t st = 0; st < plan.added_new.size(); st += 128) {
      std::vector<i64> l;
      for (size_t r = st; r < std::min(st + 128, plan.added_new.size()); ++r) l.push_back(i64(r));
      ptree.push_back(std::move(l));
    }
    pk_far = compress_block_far(enew.view(), ng, plan.added_new, circles, false, with_null, ptree, eps, w);
    phase_mark("update: pk far ID", w);
  };
  auto t_pk_near = [&](cudaStream_t w) {
    if (!do_pk_near) return;
    pk_near = near_row_id(enew.view(), added_s, mapped(kept_new_s, near_s), eps, notes_pk, "pk", w);
    phase_mark("update: pk near ID", w);
  };
  // SBX_PAR_MODE:
  //   4 (default) the row-ID hierarchies of the update in lockstep on the
  //     library stream, and the A_pp HBS build in a second host thread on
  //     the SAME stream; both threads' CPQR batches meet in a rendezvous
  //     and go out as one launch per round (no cross-stream co-scheduling);
  //   2 the same without the second thread (A_pp after the IDs);
  //   3 the near-field row IDs in order on the library stream, then the
  //     far-field hierarchies beside the A_pp build on two worker streams,
  //     both restricted to engines without grid-wide barriers;
  //   1 / 0 all row IDs beside A_pp / every task on its own stream.
  // Measured on cfg2 (bench, 10 steps): mode 4 32-33 ms, mode 2 35 ms;
  // modes 0/1/3 vary widely from run to run (co-scheduling of the
  // large-smem CPQR kernels of two streams is not stable).
  if (par_mode == 2 || par_mode == 4) {
    // every row-ID hierarchy of the update advances in lockstep (one batched
    // CPQR per tree level across all of them)
    std::vector<std::vector<i64>> ptree;
    for (size_t st = 0; st < plan.added_new.size(); st += 128) {
      std::vector<i64> l;
      for (size_t r = st; r < std::min(st + 128, plan.added_new.size()); ++r) l.push_back(i64(r));
      ptree.push_back(std::move(l));
    }
    static const bool fault = [] {  // tests: a proxy violation while the A_pp thread is running
      const char* e = std::getenv("SBX_TEST_FAULT");
      return e && std::string(e) == "far_prepare";
    }();
    if (fault) throw Error(5, "far row point inside a division circle (injected by SBX_TEST_FAULT)");
    const FarPrep fk = far_prepare(ng, far_nodes, circles, true, ktree);
    FarPrep fp;
    if (!plan.added_new.empty()) fp = far_prepare(ng, plan.added_new, circles, false, ptree);
  hm("far_prepare");
    const std::vector<i64> kc_rows = do_kc ? mapped(kept_old_s, near_s) : std::vector<i64>{};
    const std::vector<i64> kp_rows = do_kp ? mapped(kept_new_s, near_s) : std::vector<i64>{};
    const std::vector<i64> pk_cols = do_pk_near ? mapped(kept_new_s, near_s) : std::vector<i64>{};
  hm("mapped");
    std::vector<HierSpec> specs;
    specs.push_back({fk.m, fk.leaves, proxy_builder(enew.view(), far_nodes, circles, fk.factor, 64, with_null, s)});
    specs.push_back({fk.m, fk.leaves, proxy_builder(enew.view(), far_nodes, circles, fk.factor, 128, with_null, s)});
    specs.push_back({fp.m, fp.leaves,
                     proxy_builder(enew.view(), plan.added_new, circles, fp.factor, 64, with_null, s)});
    specs.push_back({fp.m, fp.leaves,
                     proxy_builder(enew.view(), plan.added_new, circles, fp.factor, 128, with_null, s)});
    specs.push_back(near_spec(eold.view(), kc_rows, cut_s, notes_kc, "kc", s));
    specs.push_back(near_spec(enew.view(), kp_rows, added_s, notes_kp, "kp", s));
    specs.push_back(near_spec(enew.view(), added_s, pk_cols, notes_pk, "pk", s));
  hm("specs");
    std::unique_ptr<IdRendezvousScope> main_rs_late;
    if (rv && !rv_entered) main_rs_late = std::make_unique<IdRendezvousScope>(rv.get(), true);
    auto res = hierarchical_id_multi(specs, eps, s);
    phase_mark("update: lockstep row IDs", s);
    far = far_settle(enew.view(), far_nodes, circles, with_null, fk, std::move(res[0]), std::move(res[1]), eps, s);
    if (!plan.added_new.empty())
      pk_far = far_settle(enew.view(), plan.added_new, circles, with_null, fp, std::move(res[2]), std::move(res[3]),
                          eps, s);
    kc_near = std::move(res[4]);
    kp_near = std::move(res[5]);
    pk_near = std::move(res[6]);
    if (main_rs_late) main_rs_late->leave();
    if (main_rs_early) main_rs_early->leave();
    if (app_thread.joinable()) {
      app_thread.join();
      if (app_err) std::rethrow_exception(app_err);
    } else {
      t_app(s);
    }
  } else if (par_mode == 5) {
    // the A_pp build (the step's critical path) on a high-priority worker
    // stream, every row ID of the update on a normal-priority one
    parallel_tasks({[&](cudaStream_t w) {
                      t_far(w);
                      t_kc(w);
                      t_kp(w);
                      t_pk_far(w);
                      t_pk_near(w);
                    },
                    t_app},
                   s, {0, 1});
  } else if (par_mode == 3) {
    t_kc(s);
    t_kp(s);
    t_pk_near(s);
    parallel_tasks({[&](cudaStream_t w) {
                      NoCoopScope nc;
                      t_far(w);
                      t_pk_far(w);
                    },
                    [&](cudaStream_t w) {
                      NoCoopScope nc;
                      t_app(w);
                    }},
                   s, {1, 0});
  } else if (par_mode == 1) {
    parallel_tasks({[&](cudaStream_t w) {
                      t_far(w);
                      t_kc(w);
                      t_kp(w);
                      t_pk_far(w);
                      t_pk_near(w);
                    },
                    t_app},
                   s, {1, 0});
  } else {
    parallel_tasks({t_far, t_kc, t_kp, t_pk_far, t_pk_near, t_app}, s);
  }
  for (auto* n : {&notes_kc, &notes_kp, &notes_pk}) u->notes.insert(u->notes.end(), n->begin(), n->end());
  struct KeptFactor {
    i64 k = 0;
    std::vector<i64> skel;  // block-local kept rows
  };
  auto kept_factor = [&](bool on, const RowIdResult& nearid) {
    KeptFactor f;
    if (!on) return f;
    f.k = far.k + nearid.k;
    for (i64 i = 0; i < far.k; ++i) f.skel.push_back(far_s[size_t(far.J[size_t(i)])]);
    for (i64 i = 0; i < nearid.k; ++i) f.skel.push_back(near_s[size_t(nearid.J[size_t(i)])]);
    return f;
  };
  KeptFactor kc = kept_factor(do_kc, kc_near), kp = kept_factor(do_kp, kp_near);
  i64 k_pk = 0;
  if (do_pk_near) k_pk = pk_far.k + pk_near.k;
  u->k_kc = kc.k;
  u->k_kp = kp.k;
  u->k_pk = k_pk;
  u->k1 = k_pk + kc.k + kp.k;
  const i64 n_ext = u->n_ext(), k1 = u->k1;
  if (k1 == 0) return u;
  // stacked L1 (n_ext x k1) and R1 (k1 x n_ext)  (lowrank.cpp:240-251)
  phase_mark("update:   settle", s);
  DevBuf<double> L1(static_cast<size_t>(n_ext * k1)), R1(static_cast<size_t>(k1 * n_ext));
  phase_mark("update:   L1/R1 alloc", s);
  SBX_CUDA(cudaMemsetAsync(L1.get(), 0, size_t(n_ext * k1) * 8, s));
  SBX_CUDA(cudaMemsetAsync(R1.get(), 0, size_t(k1 * n_ext) * 8, s));
  phase_mark("update:   L1/R1 memset", s);
  const i64 ckc = k_pk, ckp = k_pk + kc.k;
  DevBuf<i64> d_far_s, d_near_s, d_added_rows;
  d_far_s.upload(far_s, s);
  d_near_s.upload(near_s, s);
  std::vector<i64> added_rows(static_cast<size_t>(u->np2));
  for (i64 r = 0; r < u->np2; ++r) added_rows[size_t(r)] = u->nk2 + u->nc2 + r;
  d_added_rows.upload(added_rows, s);
  std::vector<ScatterJob> sj;
  const int ldl = int(n_ext);
  auto scat = [&](const double* src, const i64* map, i64 rows, i64 cols, int col_off, double alpha) {
    if (rows * cols == 0) return;
    sj.push_back({src, L1.get(), map, int(rows), int(cols), int(std::max<i64>(rows, 1)), ldl, col_off, 0, alpha});
  };
  if (kc.k > 0) {  // -kc.L in the kept rows
    scat(far.P.get(), d_far_s.get(), far.m, far.k, int(ckc), -1.0);
    scat(kc_near.P.get(), d_near_s.get(), kc_near.m, kc_near.k, int(ckc + far.k), -1.0);
  }
  if (kp.k > 0) {  // kp.L
    scat(far.P.get(), d_far_s.get(), far.m, far.k, int(ckp), 1.0);
    scat(kp_near.P.get(), d_near_s.get(), kp_near.m, kp_near.k, int(ckp + far.k), 1.0);
  }
  if (k_pk > 0) {  // pk.L in the added rows
    scat(pk_far.P.get(), d_added_rows.get(), pk_far.m, pk_far.k, 0, 1.0);
    scat(pk_near.P.get(), d_added_rows.get(), pk_near.m, pk_near.k, int(pk_far.k), 1.0);
  }
  scatter_batched(sj, s);
  phase_mark("update:   L1 scatter", s);
  // R blocks straight into R1
  {
    std::vector<i64> ri_old, ci_old, ri_new, ci_new, dstc_new;
    std::vector<BlockJob> jo, jn;
    i64 mo = 0, mn = 0;
    auto push = [](std::vector<i64>& ri, std::vector<i64>& ci, std::vector<BlockJob>& jv, i64& mx,
                   const std::vector<i64>& rows, const std::vector<i64>& cols, i64 out_off, int ld,
                   i64 dst_col_off) {
      if (rows.empty() || cols.empty()) return;
      BlockJob j{};
      j.row_off = i64(ri.size());
      j.col_off = i64(ci.size());
      j.nr = int(rows.size());
      j.nc = int(cols.size());
      j.out_off = out_off;
      j.ld = ld;
      j.dst_col_off = dst_col_off;
      ri.insert(ri.end(), rows.begin(), rows.end());
      ci.insert(ci.end(), cols.begin(), cols.end());
      mx = std::max<i64>(mx, i64(j.nr) * j.nc);
      jv.push_back(j);
    };
    const int ldr = int(k1);
    // kc.R = A_old(kept_old_s[skel], cut_s) at rows ckc.., cols nk2..
    push(ri_old, ci_old, jo, mo, mapped(kept_old_s, kc.skel), cut_s, ckc + u->nk2 * k1, ldr, -1);
    // kp.R = A_new(kept_new_s[skel], added_s) at rows ckp.., cols nk2+nc2..
    push(ri_new, ci_new, jn, mn, mapped(kept_new_s, kp.skel), added_s, ckp + (u->nk2 + u->nc2) * k1, ldr, -1);
    // pk.R: far skeleton rows over the far kept columns, near over near
    if (k_pk > 0) {
      std::vector<i64> fr, nr_;
      for (i64 i = 0; i < pk_far.k; ++i) fr.push_back(added_s[size_t(pk_far.J[size_t(i)])]);
      for (i64 i = 0; i < pk_near.k; ++i) nr_.push_back(added_s[size_t(pk_near.J[size_t(i)])]);
      const i64 o1 = i64(dstc_new.size());
      dstc_new.insert(dstc_new.end(), far_s.begin(), far_s.end());
      push(ri_new, ci_new, jn, mn, fr, mapped(kept_new_s, far_s), 0, ldr, o1);
      const i64 o2 = i64(dstc_new.size());
      dstc_new.insert(dstc_new.end(), near_s.begin(), near_s.end());
      push(ri_new, ci_new, jn, mn, nr_, mapped(kept_new_s, near_s), pk_far.k, ldr, o2);
    }
    DevBuf<i64> a, b, c, d, e;
    DevBuf<BlockJob> ja, jb;
    a.upload(ri_old, s);
    b.upload(ci_old, s);
    c.upload(ri_new, s);
    d.upload(ci_new, s);
    e.upload(dstc_new, s);
    ja.upload(jo, s);
    jb.upload(jn, s);
    phase_mark("update:   R1 index upload", s);
    launch_block_jobs(eold.view(), ja.get(), int(jo.size()), mo, a.get(), b.get(), R1.get(), s);
    launch_block_jobs(enew.view(), jb.get(), int(jn.size()), mn, c.get(), d.get(), R1.get(), s, e.get());
  }
  phase_mark("update: L1/R1 assembly", s);
  // Final row ID of L1 (see header): CPQR of L1^T.  The rows of L1 fall in
  // three groups with disjoint column supports — far kept rows (shared far
  // P in the kc and kp columns), near kept rows (near P's), added rows (pk
  // P's); cut rows are zero.  Columns of L1^T from different groups are
  // orthogonal, so the greedy CPQR decouples: each group is factored on its
  // own, the eps-rank uses the global |r_00| = max over groups, and the
  // global pivot order is the merge of the groups' |r_jj| sequences.
  struct Group {
    std::vector<const double*> src;  // interpolation blocks (rows x kcols), stacked as W^T rows
    std::vector<i64> kcols;
    i64 rows = 0;
    const i64* rowmap = nullptr;  // group row -> L1 row
    std::vector<i64> hrowmap;
  };
  Group gf, gn, ga;
  gf.rows = far.m;
  gf.hrowmap = far_s;
  gf.rowmap = d_far_s.get();
  // far rows of L1 are (-x, x) (kc and kp share the far P): factor x once and
  // scale its |r_jj| by sqrt(2) (identical Gram matrix up to the factor 2)
  double far_scale = 1.0;
  if (far.k > 0 && (kc.k > 0 || kp.k > 0)) {
    gf.src.push_back(far.P.get());
    gf.kcols.push_back(far.k);
    if (kc.k > 0 && kp.k > 0) far_scale = std::sqrt(2.0);
  }
  gn.rows = i64(near_s.size());
  gn.hrowmap = near_s;
  gn.rowmap = d_near_s.get();
  if (kc.k > 0 && kc_near.k > 0) {
    gn.src.push_back(kc_near.P.get());
    gn.kcols.push_back(kc_near.k);
  }
  if (kp.k > 0 && kp_near.k > 0) {
    gn.src.push_back(kp_near.P.get());
    gn.kcols.push_back(kp_near.k);
  }
  ga.rows = u->np2;
  ga.hrowmap = added_rows;
  ga.rowmap = d_added_rows.get();
  if (k_pk > 0) {
    if (pk_far.k > 0) {
      ga.src.push_back(pk_far.P.get());
      ga.kcols.push_back(pk_far.k);
    }
    if (pk_near.k > 0) {
      ga.src.push_back(pk_near.P.get());
      ga.kcols.push_back(pk_near.k);
    }
  }
  Group* groups[3] = {&gf, &gn, &ga};
  std::vector<IdProblem> fprobs(3);
  std::vector<std::unique_ptr<DevBuf<double>>> gbufs;
  std::vector<CopyJob> tj;
  for (int g = 0; g < 3; ++g) {
    Group& G = *groups[g];
    i64 M = 0;
    for (i64 c : G.kcols) M += c;
    if (G.rows == 0) M = 0;
    auto buf = std::make_unique<DevBuf<double>>(size_t(std::max<i64>(M * G.rows, 1)));
    i64 r0 = 0;
    for (size_t b = 0; b < G.src.size(); ++b) {  // W^T rows r0.. = block^T
      if (G.rows > 0)
        tj.push_back({G.src[b], buf->get() + r0, int(G.kcols[b]), int(G.rows), int(G.rows), int(M), 1, 0});
      r0 += G.kcols[b];
    }
    fprobs[size_t(g)] = {buf->get(), int(M), int(G.rows), int(std::max<i64>(M, 1))};
    gbufs.push_back(std::move(buf));
  }
  copy_batched(tj, s);
  IdBatch fin;
  fin.factor(fprobs, eps * 1e-3, s);  // truncated well below the global threshold
  const double gscale[3] = {far_scale, 1.0, 1.0};
  auto rdiag = [&](int g, i64 i) { return gscale[g] * fin.diag(size_t(g))[size_t(i)]; };
  double r00 = 0.0;
  for (int g = 0; g < 3; ++g)
    if (!fin.diag(size_t(g)).empty()) r00 = std::max(r00, rdiag(g, 0));
  std::vector<i64> kg(3, 0);
  if (r00 > 0.0)
    for (int g = 0; g < 3; ++g) {
      const i64 dn = i64(fin.diag(size_t(g)).size());
      while (kg[size_t(g)] < dn && rdiag(g, kg[size_t(g)]) > eps * r00) ++kg[size_t(g)];
    }
  // global pivot order: merge by |r_jj| (descending; ties keep group order)
  struct Piv {
    double r;
    int g;
    i64 i;
  };
  std::vector<Piv> order;
  for (int g = 0; g < 3; ++g)
    for (i64 i = 0; i < kg[size_t(g)]; ++i) order.push_back({rdiag(g, i), g, i});
  std::stable_sort(order.begin(), order.end(), [](const Piv& a, const Piv& b) { return a.r > b.r; });
  u->k = i64(order.size());
  phase_mark("update: final ID of L1", s);
  const i64 k = u->k;
  u->skeleton.clear();
  for (const Piv& p : order)
    u->skeleton.push_back(groups[p.g]->hrowmap[size_t(fin.perm(size_t(p.g))[size_t(p.i)])]);
  u->L->resize(size_t(std::max<i64>(n_ext * k, 1)));
  u->R.resize(size_t(std::max<i64>(k * n_ext, 1)));
  if (k > 0) {
    std::vector<std::unique_ptr<DevBuf<double>>> pg;
    std::vector<double*> Pp(3, nullptr);
    std::vector<int> ldp(3, 1);
    for (int g = 0; g < 3; ++g) {
      pg.push_back(std::make_unique<DevBuf<double>>(size_t(std::max<i64>(groups[g]->rows * kg[size_t(g)], 1))));
      Pp[size_t(g)] = pg.back()->get();
      ldp[size_t(g)] = int(std::max<i64>(groups[g]->rows, 1));
    }
    fin.interp(kg, Pp, ldp, s);
    phase_mark("update: final interp", s);
    SBX_CUDA(cudaMemsetAsync(u->L->get(), 0, size_t(n_ext * k) * 8, s));
    std::vector<ScatterJob> lj;
    for (i64 col = 0; col < k; ++col) {  // L column `col` = group column order[col].i
      const Piv& p = order[size_t(col)];
      const Group& G = *groups[p.g];
      lj.push_back({Pp[size_t(p.g)] + size_t(p.i) * size_t(ldp[size_t(p.g)]), u->L->get(), G.rowmap,
                    int(G.rows), 1, ldp[size_t(p.g)], int(n_ext), int(col), 0, 1.0});
    }
    scatter_batched(lj, s);
    phase_mark("update: L scatter", s);
    // R = L1(J(0:k), :) * R1
    DevBuf<i64> sk;
    sk.upload(u->skeleton, s);
    DevBuf<double> L1s(static_cast<size_t>(k * k1));
    scatter_batched({{L1.get(), L1s.get(), sk.get(), int(k), int(k1), ldl, int(k), 0, 1, 1.0}}, s);
    gemm_batched({{L1s.get(), R1.get(), u->R.get(), int(k), int(n_ext), int(k1), int(k), int(k1), int(k),
                   0, 0, 1.0, 0.0}},
                 s);
  }
  SBX_CUDA(cudaStreamSynchronize(s));
  phase_mark("update: L, R", s);
  return u;
}

void update_download(const Update& u, int which, double* out, cudaStream_t s) {
  require(which == 0 || which == 1, "update factor: which must be 0 (L) or 1 (R)");
  const size_t n = size_t(u.n_ext() * u.k);
  if (n == 0) return;
  (which == 0 ? *u.L : u.R).download(out, n, s);
  SBX_CUDA(cudaStreamSynchronize(s));
}

std::unique_ptr<Update> update_from_factors(const Plan& plan, const double* L, const double* R,
                                            i64 n_ext, i64 k, cudaStream_t s) {
  auto u = std::make_unique<Update>();
  u->nk2 = 2 * i64(plan.kept_old.size());
  u->nc2 = 2 * i64(plan.cut_old.size());
  u->np2 = 2 * i64(plan.added_new.size());
  require(n_ext == u->n_ext(), "update factor size does not match the plan");
  require(k >= 0, "negative rank");
  u->k = k;
  u->k1 = k;
  u->L->upload(L, size_t(n_ext * k), s);
  u->R.upload(R, size_t(n_ext * k), s);
  SBX_CUDA(cudaStreamSynchronize(s));
  return u;
}

}  // namespace sbx
