// The sbx C-ABI (include/sbx.h): opaque handles over the host/device
// objects, exceptions mapped to status codes + sbx_last_error().
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <string>

#include "els.hpp"
#include "entries.hpp"
#include "geometry.hpp"
#include "hbs.hpp"
#include "hbs_build.hpp"
#include "idengine.hpp"
#include "matio.hpp"
#include "multigpu.hpp"
#include "sbx.h"
#include "update.hpp"

struct sbx_geom_s {
  std::unique_ptr<sbx::Geom> g;
};
struct sbx_plan_s {
  std::unique_ptr<sbx::Plan> p;
};
struct sbx_hbs_s {
  std::unique_ptr<sbx::HbsOp> h;
};
struct sbx_update_s {
  std::shared_ptr<sbx::Update> u;  // shared with an update cache entry
};
// Snapshot update cache (scenario.cpp:836-899): updates are determined by the
// refinement plan alone, so identical (panel ids, m) -- at the same
// tolerance, formulation and seed -- share one compression.
struct sbx_update_cache_s {
  std::mutex mu;
  std::map<std::tuple<std::vector<int64_t>, int, double, int, double, uint64_t>, std::shared_ptr<sbx::Update>> map;
  int64_t hits = 0, misses = 0;
};
struct sbx_els_s {
  std::unique_ptr<sbx::Els> e;
};
struct sbx_app_s {
  std::shared_ptr<sbx::AppSolver> a;
};

struct sbx_comm_s {
  std::unique_ptr<sbx::Collective> c;
};
struct sbx_els_shard_s {
  std::unique_ptr<sbx::ElsShard> e;
  std::shared_ptr<sbx::Update> keep_update;  // L, R read by the build only; kept for symmetry with sbx_els
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return SBX_OK;
  } catch (const sbx::Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return SBX_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SBX_RUNTIME_ERROR;
  }
}

// Releasing a handle waits, as cudaFree would, for the work that may still
// read its device memory (which returns to a stream-ordered pool): the
// library stream, and the last call on every caller stream the handle ran
// on (StreamMark events; no device-wide synchronisation).
void drain_handle(sbx_hbs_s* h) {
  if (h->h) h->h->drain();
}
void drain_handle(sbx_els_s* e) {
  if (e->e) e->e->drain();
}
void drain_handle(sbx_app_s* a) {
  if (a->a && a->a->h) a->a->h->drain();
}
void drain_handle(sbx_els_shard_s* e) {
  if (e->e) (void)cudaDeviceSynchronize();  // shard solves run on caller streams (no marks kept)
}
template <class T>
void drain_handle(T*) {}  // used on the library stream only

template <class T>
int destroy_handle(T* h) {
  if (h) {
    drain_handle(h);
    (void)cudaStreamSynchronize(sbx::lib_stream());
    delete h;
  }
  return SBX_OK;
}

cudaStream_t stream_of(void* s) {
  return s ? static_cast<cudaStream_t>(s) : sbx::lib_stream();
}

sbx::Geom& G(sbx_geom g) {
  sbx::require(g && g->g, "null geometry handle");
  return *g->g;
}
sbx::Collective& Cm(sbx_comm c) {
  sbx::require(c && c->c, "null comm handle");
  return *c->c;
}
sbx::HbsOp& H(sbx_hbs h) {
  sbx::require(h && h->h, "null hbs handle");
  return *h->h;
}
}  // namespace

extern "C" {

const char* sbx_last_error(void) { return g_err.c_str(); }

int sbx_init(int device) {
  return guard([&] {
    // The per-step path waits on the device between its ID rounds (perm /
    // diag come back to the host): spin-wait so a waiting host thread is not
    // descheduled (SBX_SCHEDULE=yield|block|auto restores the driver's choice).
    static const char* sched = std::getenv("SBX_SCHEDULE");
    const unsigned flag = !sched ? cudaDeviceScheduleSpin
                          : std::strcmp(sched, "yield") == 0 ? cudaDeviceScheduleYield
                          : std::strcmp(sched, "block") == 0 ? cudaDeviceScheduleBlockingSync
                          : cudaDeviceScheduleAuto;
    SBX_CUDA(cudaSetDevice(device));
    if (cudaSetDeviceFlags(flag) != cudaSuccess) (void)cudaGetLastError();  // context already set up: keep its flags
    (void)sbx::lib_stream();
  });
}

int sbx_sync(void) {
  return guard([&] { SBX_CUDA(cudaStreamSynchronize(sbx::lib_stream())); });
}

int64_t sbx_kernel_launches(int reset) { return sbx::launches(reset != 0); }

int sbx_kernel_timing(int enable) {
  return guard([&] { sbx::ktimer_enable(enable != 0); });
}

int sbx_kernel_time(const char* name, int reset, double* total_ms, int64_t* count) {
  return guard([&] {
    int64_t c = 0;
    *total_ms = sbx::ktimer_total(name, reset != 0, &c);
    if (count) *count = c;
  });
}

int sbx_kernel_flops(const char* name, int reset, double* flops) {
  return guard([&] { *flops = sbx::ktimer_flops(name, reset != 0); });
}

int sbx_row_id(const double* w, int64_t m, int64_t n, double eps, int64_t forced, int engine,
               int64_t* k, int64_t* J, double* P) {
  return guard([&] {
    sbx::require(m >= 0 && n >= 0, "row_id: negative size");
    if (forced < 0) sbx::require(eps > 0.0 && eps <= 0.1, "id tolerance must lie in (0, 0.1]");
    cudaStream_t s = sbx::lib_stream();
    if (m == 0 || n == 0 || (forced >= 0 && forced == 0)) {
      *k = 0;
      for (int64_t i = 0; i < m; ++i) J[i] = i;
      return;
    }
    // W^T (n x m)
    std::vector<double> wt(size_t(m * n));
    for (int64_t i = 0; i < m; ++i)
      for (int64_t j = 0; j < n; ++j) wt[size_t(j + i * n)] = w[i + j * m];
    sbx::DevBuf<double> d;
    d.upload(wt, s);
    sbx::IdBatch b;
    b.force_engine = engine;
    b.factor({{d.get(), int(n), int(m), int(n)}}, forced >= 0 ? 1e-15 : eps, s);
    const int64_t kk = forced >= 0 ? b.forced_rank(0, forced) : b.eps_rank(0, eps);
    *k = kk;
    for (int64_t i = 0; i < m; ++i) J[i] = b.perm(0)[size_t(i)];
    if (kk > 0) {
      sbx::DevBuf<double> dp(size_t(m * kk));
      b.interp({kk}, {dp.get()}, {int(m)}, s);
      dp.download(P, size_t(m * kk), s);
    }
    SBX_CUDA(cudaStreamSynchronize(s));
  });
}

int sbx_dense_inverse(const double* a, int64_t n, double* inv, double* rcond) {
  return guard([&] {
    sbx::require(n >= 1, "dense_inverse: empty matrix");
    cudaStream_t s = sbx::lib_stream();
    sbx::DevBuf<double> d(size_t(n * n)), di(size_t(n * n));
    SBX_CUDA(cudaMemcpyAsync(d.get(), a, size_t(n * n) * 8, cudaMemcpyHostToDevice, s));
    const double rc = sbx::dense_inverse(d.get(), n, di.get(), s);
    di.download(inv, size_t(n * n), s);
    SBX_CUDA(cudaStreamSynchronize(s));
    if (rcond) *rcond = rc;
  });
}

int sbx_matmul(const double* a, int64_t m, int64_t k, const double* b, int64_t n, double* c) {
  return guard([&] {
    sbx::require(m >= 1 && n >= 1 && k >= 1, "matmul: empty operand");
    cudaStream_t s = sbx::lib_stream();
    sbx::DevBuf<double> da(size_t(m * k)), db(size_t(k * n)), dc(size_t(m * n));
    SBX_CUDA(cudaMemcpyAsync(da.get(), a, size_t(m * k) * 8, cudaMemcpyHostToDevice, s));
    SBX_CUDA(cudaMemcpyAsync(db.get(), b, size_t(k * n) * 8, cudaMemcpyHostToDevice, s));
    sbx::gemm_batched({{da.get(), db.get(), dc.get(), int(m), int(n), int(k), int(m), int(k), int(m), 0, 0, 1.0, 0.0}},
                      s);
    dc.download(c, size_t(m * n), s);
    SBX_CUDA(cudaStreamSynchronize(s));
  });
}

void* sbx_stream(void) {
  try {
    return static_cast<void*>(sbx::lib_stream());
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// ---------------------------------------------------------------- geometry
int sbx_geom_create(const sbx_curve* curve, int n_panels, int q, sbx_geom* out) {
  return guard([&] {
    sbx::require(curve && out, "null argument");
    auto g = sbx::geom_panelize(*curve, n_panels, q);
    g->upload(sbx::lib_stream());
    *out = new sbx_geom_s{std::move(g)};
  });
}

int sbx_geom_add_holes(sbx_geom wall, int n_holes, const sbx_curve* holes, const int32_t* n_panels,
                       const int32_t* q, sbx_geom* out, sbx_plan* plan) {
  return guard([&] {
    std::vector<sbx_curve> hs(holes, holes + n_holes);
    std::vector<int> np(n_panels, n_panels + n_holes), qs(q, q + n_holes);
    auto r = sbx::geom_add_holes(G(wall), hs, np, qs);
    r.first->upload(sbx::lib_stream());
    *out = new sbx_geom_s{std::move(r.first)};
    *plan = new sbx_plan_s{std::move(r.second)};
  });
}

int sbx_geom_destroy(sbx_geom g) { return destroy_handle(g); }

int sbx_geom_info(sbx_geom g, int64_t* n_nodes, int64_t* n_panels, int64_t* n_components) {
  return guard([&] {
    const auto& d = G(g);
    *n_nodes = d.n_nodes();
    *n_panels = int64_t(d.panels.size());
    *n_components = int64_t(d.comps.size());
  });
}

int sbx_geom_nodes(sbx_geom g, double* out9, int64_t* panel_of) {
  return guard([&] {
    const auto& d = G(g);
    const int64_t n = d.n_nodes();
    const std::vector<double>* src[9] = {&d.x, &d.y, &d.nx, &d.ny, &d.tx, &d.ty, &d.w, &d.kappa, &d.t};
    for (int a = 0; a < 9; ++a) std::memcpy(out9 + a * n, src[a]->data(), size_t(8 * n));
    if (panel_of) std::memcpy(panel_of, d.panel_of.data(), size_t(8 * n));
  });
}

int sbx_panels_near_point(sbx_geom g, double px, double py, double radius, int64_t* out,
                          int64_t cap, int64_t* count) {
  return guard([&] {
    auto v = sbx::panels_near_point(G(g), px, py, radius);
    for (size_t i = 0; i < v.size() && int64_t(i) < cap; ++i) out[i] = v[i];
    *count = int64_t(v.size());
  });
}

int sbx_refine(sbx_geom g, const int64_t* panel_ids, int64_t n, int m, sbx_geom* out,
               sbx_plan* plan) {
  return guard([&] {
    auto r = sbx::geom_refine(G(g), std::vector<int64_t>(panel_ids, panel_ids + n), m);
    r.first->upload(sbx::lib_stream());
    *out = new sbx_geom_s{std::move(r.first)};
    *plan = new sbx_plan_s{std::move(r.second)};
  });
}

int sbx_coarsen(sbx_geom g, sbx_plan plan, sbx_geom* out) {
  return guard([&] {
    sbx::require(plan && plan->p, "null plan handle");
    auto c = sbx::geom_coarsen(G(g), *plan->p);
    c->upload(sbx::lib_stream());
    *out = new sbx_geom_s{std::move(c)};
  });
}

int sbx_plan_destroy(sbx_plan p) { return destroy_handle(p); }

int sbx_plan_sizes(sbx_plan p, int64_t* n_k, int64_t* n_c, int64_t* n_p) {
  return guard([&] {
    sbx::require(p && p->p, "null plan handle");
    *n_k = int64_t(p->p->kept_old.size());
    *n_c = int64_t(p->p->cut_old.size());
    *n_p = int64_t(p->p->added_new.size());
  });
}

int sbx_plan_maps(sbx_plan p, int64_t* kept_old, int64_t* kept_new, int64_t* cut_old,
                  int64_t* added_new) {
  return guard([&] {
    sbx::require(p && p->p, "null plan handle");
    const auto& q = *p->p;
    std::copy(q.kept_old.begin(), q.kept_old.end(), kept_old);
    std::copy(q.kept_new.begin(), q.kept_new.end(), kept_new);
    std::copy(q.cut_old.begin(), q.cut_old.end(), cut_old);
    std::copy(q.added_new.begin(), q.added_new.end(), added_new);
  });
}

// ---------------------------------------------------------------- entries / data
int sbx_submatrix(sbx_geom g, int formulation, double mu, const int64_t* rows, int64_t nr,
                  const int64_t* cols, int64_t nc, double* out) {
  return guard([&] {
    sbx::EntryOracle eo(G(g), formulation, mu, sbx::lib_stream());
    eo.submatrix_host(rows, nr, cols, nc, out, sbx::lib_stream());
  });
}

int sbx_boundary_data(sbx_geom g, int64_t n_src, const double* src_xyf, double mu, double* out) {
  return guard([&] { sbx::boundary_data_host(G(g), n_src, src_xyf, mu, out, sbx::lib_stream()); });
}

int sbx_evaluate_solution(sbx_geom g, int formulation, double mu, const double* tau, int64_t ldt, int64_t nrhs,
                          const double* targets, int64_t n_targets, int with_pressure, double* velocity,
                          double* pressure, uint8_t* near_boundary) {
  return guard([&] {
    sbx::evaluate_solution_host(G(g), formulation, mu, tau, ldt, nrhs, targets, n_targets, with_pressure != 0,
                                velocity, pressure, near_boundary, sbx::lib_stream());
  });
}

// ---------------------------------------------------------------- HBS
int sbx_hbs_compress(sbx_geom g, int formulation, double mu, const sbx_hbs_options* opts,
                     sbx_hbs* out) {
  return guard([&] {
    sbx::HbsBuildOptions o;
    if (opts) o = sbx::HbsBuildOptions::from(*opts);
    auto h = sbx::hbs_compress_device(G(g), formulation, mu, nullptr, 0, o, sbx::lib_stream());
    *out = new sbx_hbs_s{std::move(h)};
  });
}

int sbx_hbs_compress_subset(sbx_geom g, int formulation, double mu, const int64_t* nodes,
                            int64_t n_nodes, const sbx_hbs_options* opts, sbx_hbs* out) {
  return guard([&] {
    sbx::HbsBuildOptions o;
    if (opts) o = sbx::HbsBuildOptions::from(*opts);
    auto h = sbx::hbs_compress_device(G(g), formulation, mu, nodes, n_nodes, o, sbx::lib_stream());
    *out = new sbx_hbs_s{std::move(h)};
  });
}

int sbx_hbs_compress_sharded(sbx_geom g, int formulation, double mu, const sbx_hbs_options* opts, sbx_comm c,
                             sbx_hbs* out) {
  return guard([&] {
    sbx::HbsBuildOptions o;
    if (opts) o = sbx::HbsBuildOptions::from(*opts);
    o.comm = Cm(c).world() > 1 ? &Cm(c) : nullptr;
    auto h = sbx::hbs_compress_device(G(g), formulation, mu, nullptr, 0, o, sbx::lib_stream());
    *out = new sbx_hbs_s{std::move(h)};
  });
}

int sbx_hbs_compress_custom(sbx_geom g, int formulation, double mu, sbx_entries_fn entries, void* ctx,
                            int with_completion, const sbx_hbs_options* opts, sbx_hbs* out) {
  return guard([&] {
    sbx::require(entries != nullptr, "hbs_compress_custom: null entry oracle");
    sbx::HostEntries he;
    he.fn = reinterpret_cast<decltype(he.fn)>(entries);
    he.ctx = ctx;
    he.with_completion = with_completion != 0;
    sbx::HbsBuildOptions o;
    if (opts) o = sbx::HbsBuildOptions::from(*opts);
    o.entries = &he;
    auto h = sbx::hbs_compress_device(G(g), formulation, mu, nullptr, 0, o, sbx::lib_stream());
    *out = new sbx_hbs_s{std::move(h)};
  });
}

int sbx_hbs_invert(sbx_hbs h) {
  return guard([&] { sbx::hbs_invert_device(H(h), sbx::lib_stream()); });
}

int sbx_hbs_destroy(sbx_hbs h) { return destroy_handle(h); }

int sbx_hbs_solve(sbx_hbs h, const double* b, int64_t ldb, int64_t nrhs, double* x, int64_t ldx,
                  int flags, void* stream) {
  return guard([&] {
    sbx::StreamScope scope(stream_of(stream));
    const bool dev = (flags & SBX_DEVICE_PTRS) != 0;
    if (flags & SBX_ROW_MAJOR) {
      sbx::require(dev, "hbs_solve: row-major blocks must be device pointers");
      sbx::hbs_sweep_rm(H(h), false, (flags & SBX_TRANSPOSE) != 0, b, ldb, nrhs, x, ldx, stream_of(stream));
      return;
    }
    if (flags & SBX_TRANSPOSE)
      sbx::hbs_solve_t(H(h), b, ldb, nrhs, x, ldx, dev, stream_of(stream));
    else
      sbx::hbs_solve(H(h), b, ldb, nrhs, x, ldx, dev, stream_of(stream));
  });
}

int sbx_hbs_apply(sbx_hbs h, const double* v, int64_t ldv, int64_t nrhs, double* y, int64_t ldy,
                  int flags, void* stream) {
  return guard([&] {
    sbx::StreamScope scope(stream_of(stream));
    const bool dev = (flags & SBX_DEVICE_PTRS) != 0;
    if (flags & SBX_ROW_MAJOR) {
      sbx::require(dev, "hbs_apply: row-major blocks must be device pointers");
      sbx::hbs_sweep_rm(H(h), true, (flags & SBX_TRANSPOSE) != 0, v, ldv, nrhs, y, ldy, stream_of(stream));
      return;
    }
    if (flags & SBX_TRANSPOSE)
      sbx::hbs_apply_t(H(h), v, ldv, nrhs, y, ldy, dev, stream_of(stream));
    else
      sbx::hbs_apply(H(h), v, ldv, nrhs, y, ldy, dev, stream_of(stream));
  });
}

int sbx_hbs_shard_info(sbx_hbs h, int G, int p, int64_t* row0, int64_t* row1, int64_t* kmax) {
  return guard([&] {
    const sbx::ShardPlans& S = sbx::hbs_shard(H(h), G, p);
    *row0 = S.row0;
    *row1 = S.row1;
    *kmax = S.kmax;
  });
}

int sbx_hbs_solve_shard_up(sbx_hbs h, int G, int p, const double* b_local, int64_t ldb, int64_t nrhs,
                           double* hat_out, int flags, void* stream) {
  return guard([&] {
    sbx::StreamScope scope(stream_of(stream));
    sbx::hbs_solve_shard_up(H(h), G, p, b_local, ldb, nrhs, hat_out, (flags & SBX_DEVICE_PTRS) != 0,
                            stream_of(stream));
  });
}

int sbx_hbs_solve_shard_down(sbx_hbs h, int G, int p, const double* hats, int64_t nrhs, double* x_local,
                             int64_t ldx, int flags, void* stream) {
  return guard([&] {
    sbx::StreamScope scope(stream_of(stream));
    sbx::hbs_solve_shard_down(H(h), G, p, hats, nrhs, x_local, ldx, (flags & SBX_DEVICE_PTRS) != 0,
                              stream_of(stream));
  });
}

int sbx_hbs_save_hbs1(sbx_hbs h, const char* path) {
  return guard([&] { sbx::hbs_save_hbs1(H(h), path, sbx::lib_stream()); });
}

int sbx_hbs_load_hbs1(const char* path, sbx_hbs* out) {
  return guard([&] { *out = new sbx_hbs_s{sbx::hbs_load_hbs1(path, sbx::lib_stream())}; });
}

int sbx_hbs_info(sbx_hbs h, int64_t* info) {
  return guard([&] {
    const auto& op = H(h);
    int64_t mk = 0;
    for (const auto& nd : op.nodes) mk = std::max<int64_t>(mk, nd.k);
    info[0] = op.n;
    info[1] = int64_t(op.nodes.size());
    info[2] = op.total_skeleton();
    info[3] = op.max_block_drawn;
    info[4] = op.has_inverse ? 1 : 0;
    info[5] = op.has_inverse ? op.solve_factor_doubles() : 0;
    info[6] = op.max_depth;
    info[7] = mk;
    info[8] = op.apply_factor_doubles();
    info[9] = op.leaf_nodes;
    info[10] = op.top_L;
    info[11] = op.top_K;
    info[12] = op.arena_used;
    info[13] = op.sharded() ? 1 : 0;
  });
}

int sbx_hbs_node_ranks(sbx_hbs h, int64_t* k, int64_t cap) {
  return guard([&] {
    const auto& op = H(h);
    for (size_t i = 0; i < op.nodes.size() && int64_t(i) < cap; ++i) k[i] = op.nodes[i].k;
  });
}

// ---------------------------------------------------------------- update
int sbx_update_compress(sbx_geom old_g, sbx_geom new_g, sbx_plan plan, int formulation, double mu,
                        double eps, uint64_t seed, sbx_update* out) {
  return guard([&] {
    sbx::require(plan && plan->p, "null plan handle");
    auto u = sbx::update_compress_device(G(old_g), G(new_g), *plan->p, formulation, mu, eps, seed,
                                         sbx::lib_stream());
    *out = new sbx_update_s{std::move(u)};
  });
}

int sbx_update_cache_create(sbx_update_cache* out) {
  return guard([&] { *out = new sbx_update_cache_s; });
}

int sbx_update_cache_destroy(sbx_update_cache c) { return destroy_handle(c); }

int sbx_update_cache_compress(sbx_update_cache c, sbx_geom old_g, sbx_geom new_g, sbx_plan plan,
                              const int64_t* panel_ids, int64_t n_panels, int m, int formulation, double mu,
                              double eps, uint64_t seed, sbx_update* out, int* hit) {
  return guard([&] {
    sbx::require(c && plan && plan->p, "null handle");
    sbx::require(n_panels >= 0 && (n_panels == 0 || panel_ids), "update_cache: bad panel list");
    auto key = std::make_tuple(std::vector<int64_t>(panel_ids, panel_ids + n_panels), m, eps, formulation, mu,
                               seed);
    {
      std::lock_guard<std::mutex> lk(c->mu);
      auto it = c->map.find(key);
      if (it != c->map.end()) {
        ++c->hits;
        if (hit) *hit = 1;
        *out = new sbx_update_s{it->second};
        return;
      }
    }
    std::shared_ptr<sbx::Update> u = sbx::update_compress_device(G(old_g), G(new_g), *plan->p, formulation, mu,
                                                                 eps, seed, sbx::lib_stream());
    std::lock_guard<std::mutex> lk(c->mu);
    ++c->misses;
    c->map.emplace(std::move(key), u);
    if (hit) *hit = 0;
    *out = new sbx_update_s{std::move(u)};
  });
}

int sbx_update_cache_stats(sbx_update_cache c, int64_t* entries, int64_t* hits, int64_t* misses) {
  return guard([&] {
    sbx::require(c != nullptr, "null cache handle");
    std::lock_guard<std::mutex> lk(c->mu);
    if (entries) *entries = int64_t(c->map.size());
    if (hits) *hits = c->hits;
    if (misses) *misses = c->misses;
  });
}

int sbx_update_compress_mode(sbx_geom old_g, sbx_geom new_g, sbx_plan plan, int formulation, double mu,
                             double eps, uint64_t seed, int mode, sbx_update* out) {
  return guard([&] {
    sbx::require(plan && plan->p, "null plan handle");
    sbx::require(mode == SBX_TWO_STEP_ID || mode == SBX_SVD_OPTIMAL, "compress_update: unknown compression mode");
    std::unique_ptr<sbx::Update> u =
        mode == SBX_SVD_OPTIMAL
            ? sbx::update_svd_optimal_device(G(old_g), G(new_g), *plan->p, formulation, mu, eps, sbx::lib_stream())
            : sbx::update_compress_device(G(old_g), G(new_g), *plan->p, formulation, mu, eps, seed,
                                          sbx::lib_stream());
    *out = new sbx_update_s{std::move(u)};
  });
}

int sbx_update_destroy(sbx_update u) { return destroy_handle(u); }

int sbx_update_info(sbx_update u, int64_t* info) {
  return guard([&] {
    sbx::require(u && u->u, "null update handle");
    const auto& x = *u->u;
    const int64_t v[9] = {x.k, x.k1, x.k_kc, x.k_kp, x.k_pk, x.n_ext(), x.nk2, x.nc2, x.np2};
    std::copy(v, v + 9, info);
  });
}

int sbx_update_factor(sbx_update u, int which, double* out) {
  return guard([&] {
    sbx::require(u && u->u, "null update handle");
    sbx::update_download(*u->u, which, out, sbx::lib_stream());
  });
}

int sbx_dump_matrix(const char* path, const double* m, int64_t rows, int64_t cols, int64_t ld) {
  return guard([&] { sbx::dump_matrix(path, m, rows, cols, ld); });
}

int sbx_load_matrix_dims(const char* path, int64_t* rows, int64_t* cols) {
  return guard([&] {
    const sbx::HMat m = sbx::load_matrix(path);
    *rows = m.r;
    *cols = m.c;
  });
}

int sbx_load_matrix(const char* path, double* out, int64_t ld) {
  return guard([&] {
    const sbx::HMat m = sbx::load_matrix(path);
    sbx::require(ld >= m.r, "load_matrix: leading dimension smaller than rows");
    for (int64_t j = 0; j < m.c; ++j)
      for (int64_t i = 0; i < m.r; ++i) out[i + j * ld] = m.a[size_t(i + j * m.r)];
  });
}

int sbx_update_dump(sbx_update u, const char* path_L, const char* path_R) {
  return guard([&] {
    sbx::require(u && u->u, "null update handle");
    const auto& x = *u->u;
    const int64_t n = x.n_ext(), k = x.k;
    std::vector<double> L(size_t(n * k)), R(size_t(k * n));
    if (k > 0) {
      sbx::update_download(x, 0, L.data(), sbx::lib_stream());
      sbx::update_download(x, 1, R.data(), sbx::lib_stream());
    }
    sbx::dump_matrix(path_L, L.data(), n, k, std::max<int64_t>(n, 1));
    sbx::dump_matrix(path_R, R.data(), k, n, std::max<int64_t>(k, 1));
  });
}

int sbx_update_load(sbx_plan plan, const char* path_L, const char* path_R, sbx_update* out) {
  return guard([&] {
    sbx::require(plan && plan->p, "null plan handle");
    const sbx::HMat L = sbx::load_matrix(path_L), R = sbx::load_matrix(path_R);
    sbx::require(L.c == R.r && L.r == R.c, "update_load: L (n_ext x k) and R (k x n_ext) do not match");
    *out = new sbx_update_s{sbx::update_from_factors(*plan->p, L.a.data(), R.a.data(), L.r, L.c,
                                                     sbx::lib_stream())};
  });
}

int sbx_update_from_factors(sbx_plan plan, const double* L, const double* R, int64_t n_ext,
                            int64_t k, sbx_update* out) {
  return guard([&] {
    sbx::require(plan && plan->p, "null plan handle");
    *out = new sbx_update_s{sbx::update_from_factors(*plan->p, L, R, n_ext, k, sbx::lib_stream())};
  });
}

// ---------------------------------------------------------------- ELS
int sbx_els_build(sbx_hbs a_oo, sbx_geom old_g, sbx_geom new_g, sbx_plan plan, sbx_update upd,
                  int formulation, double mu, sbx_els* out) {
  return guard([&] {
    sbx::require(plan && plan->p && upd && upd->u, "null handle");
    auto e = sbx::els_build_device(H(a_oo), G(old_g), G(new_g), *plan->p, *upd->u, formulation, mu,
                                   sbx::lib_stream());
    *out = new sbx_els_s{std::move(e)};
  });
}

int sbx_app_build(sbx_geom new_g, sbx_plan plan, int formulation, double mu, double eps, sbx_app* out) {
  return guard([&] {
    sbx::require(plan && plan->p, "null plan handle");
    sbx::require(eps > 0.0 && eps <= 0.1, "app_build: tolerance out of range");
    auto h = new sbx_app_s;
    try {
      h->a = sbx::build_app_solver(G(new_g), *plan->p, formulation, mu, eps, sbx::lib_stream());
      SBX_CUDA(cudaStreamSynchronize(sbx::lib_stream()));
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int sbx_app_destroy(sbx_app a) { return destroy_handle(a); }

int sbx_app_info(sbx_app a, int64_t* info) {
  return guard([&] {
    sbx::require(a && a->a, "null app handle");
    info[0] = 2 * int64_t(a->a->added.size());
    info[1] = a->a->h ? 1 : 0;
  });
}

int sbx_app_solve(sbx_app a, const double* v, int64_t ldv, int64_t nrhs, double* out, int64_t ldo, int flags,
                  void* stream) {
  return guard([&] {
    sbx::require(a && a->a, "null app handle");
    const cudaStream_t s = stream_of(stream);
    sbx::StreamScope scope(s);
    const int64_t n = 2 * int64_t(a->a->added.size());
    sbx::require(nrhs >= 0 && ldv >= n && ldo >= n, "app_solve: bad sizes");
    if (n == 0 || nrhs == 0) return;
    const bool tr = (flags & SBX_TRANSPOSE) != 0;
    if (flags & SBX_DEVICE_PTRS) {
      sbx::app_solve_device(*a->a, v, ldv, out, ldo, nrhs, s, tr);
      return;
    }
    sbx::DevBuf<double> dv(size_t(n * nrhs)), dout(size_t(n * nrhs));
    SBX_CUDA(cudaMemcpy2DAsync(dv.get(), size_t(n) * 8, v, size_t(ldv) * 8, size_t(n) * 8, size_t(nrhs),
                               cudaMemcpyHostToDevice, s));
    sbx::app_solve_device(*a->a, dv.get(), n, dout.get(), n, nrhs, s, tr);
    SBX_CUDA(cudaMemcpy2DAsync(out, size_t(ldo) * 8, dout.get(), size_t(n) * 8, size_t(n) * 8, size_t(nrhs),
                               cudaMemcpyDeviceToHost, s));
    SBX_CUDA(cudaStreamSynchronize(s));
  });
}

int sbx_els_destroy(sbx_els e) { return destroy_handle(e); }

int sbx_els_info(sbx_els e, int64_t* info) {
  return guard([&] {
    sbx::require(e && e->e, "null els handle");
    const auto& s = *e->e;
    info[0] = s.n_k;
    info[1] = s.n_c;
    info[2] = s.n_p;
    info[3] = s.k;
    info[4] = (s.app && s.app->h) ? 1 : 0;
    // algorithmic doubles of one A_pp solve: its HBS factors or the dense inverse
    info[5] = (s.app && s.app->h) ? s.app->h->solve_factor_doubles() : s.n_p * s.n_p;
  });
}

int sbx_els_solve(sbx_els e, const double* g_n, int64_t ldg, int64_t nrhs, double* tau_n,
                  int64_t ldt, int flags, void* stream) {
  return guard([&] {
    sbx::StreamScope scope(stream_of(stream));
    sbx::require(e && e->e, "null els handle");
    sbx::els_solve(*e->e, g_n, ldg, nrhs, tau_n, ldt, false, (flags & SBX_DEVICE_PTRS) != 0,
                   stream_of(stream));
  });
}

namespace {
int els_apply_forward_host(sbx_els e, const double* v, int64_t ldv, int64_t nrhs, double* out, int64_t ldo,
                           bool tr) {
  return guard([&] {
    sbx::require(e && e->e, "null els handle");
    sbx::Els& E = *e->e;
    const int64_t n = E.n_ext();
    sbx::require(ldv >= n && ldo >= n, "els_apply_forward: size mismatch");
    cudaStream_t s = sbx::lib_stream();
    sbx::DevBuf<double> dv(static_cast<size_t>(n * nrhs)), dout(static_cast<size_t>(n * nrhs));
    SBX_CUDA(cudaMemcpy2DAsync(dv.get(), size_t(n) * 8, v, size_t(ldv) * 8, size_t(n) * 8, size_t(nrhs),
                               cudaMemcpyHostToDevice, s));
    sbx::els_apply_forward_device(E, dv.get(), dout.get(), nrhs, s, tr);
    SBX_CUDA(cudaMemcpy2DAsync(out, size_t(ldo) * 8, dout.get(), size_t(n) * 8, size_t(n) * 8, size_t(nrhs),
                               cudaMemcpyDeviceToHost, s));
    SBX_CUDA(cudaStreamSynchronize(s));
  });
}
}  // namespace

int sbx_els_apply_forward(sbx_els e, const double* v, int64_t ldv, int64_t nrhs, double* out, int64_t ldo) {
  return els_apply_forward_host(e, v, ldv, nrhs, out, ldo, false);
}

int sbx_els_apply_forward_t(sbx_els e, const double* v, int64_t ldv, int64_t nrhs, double* out, int64_t ldo) {
  return els_apply_forward_host(e, v, ldv, nrhs, out, ldo, true);
}

int sbx_els_gmres(sbx_els e, const double* g_n, double* tau_n, int precond, double tol, int64_t max_iter,
                  int64_t restart, int64_t* n_iter, double* history, int64_t history_cap) {
  return guard([&] {
    sbx::require(e && e->e, "null els handle");
    sbx::GmresOutcome r = sbx::els_gmres(*e->e, g_n, tau_n, precond != 0, tol, max_iter, restart,
                                         sbx::lib_stream());
    if (n_iter) *n_iter = r.n_iter;
    if (history)
      for (size_t i = 0; i < r.history.size() && int64_t(i) < history_cap; ++i) history[i] = r.history[i];
    if (!r.error.empty()) throw sbx::Error(SBX_NONCONVERGENCE, r.error);
  });
}

int sbx_els_solve_raw(sbx_els e, const double* g_ext, int64_t ldg, int64_t nrhs, double* y,
                      int64_t ldy, int flags, void* stream) {
  return guard([&] {
    sbx::StreamScope scope(stream_of(stream));
    sbx::require(e && e->e, "null els handle");
    sbx::els_solve(*e->e, g_ext, ldg, nrhs, y, ldy, true, (flags & SBX_DEVICE_PTRS) != 0,
                   stream_of(stream), (flags & SBX_TRANSPOSE) != 0);
  });
}

int sbx_els_conditioning(sbx_els e, int iters, double* out) {
  return guard([&] {
    sbx::require(e && e->e, "null els handle");
    sbx::require(iters >= 1, "conditioning: iteration count must be positive");
    const sbx::CondReport r = sbx::els_conditioning(*e->e, iters, sbx::lib_stream());
    out[0] = r.kappa_w;
    out[1] = r.kappa_l;
    out[2] = r.kappa_r;
    out[3] = r.kappa_ext;
    out[4] = r.kappa_tilde;
    out[5] = r.bound;
    out[6] = r.bound_holds ? 1.0 : 0.0;
  });
}

int sbx_els_conditioning_report(sbx_els e, int dense, int iters, double* out) {
  return guard([&] {
    sbx::require(e && e->e, "null els handle");
    sbx::require(dense || iters >= 1, "conditioning: iteration count must be positive");
    const sbx::CondReport r = sbx::els_conditioning(*e->e, iters, sbx::lib_stream(), dense != 0);
    out[0] = r.kappa_w;
    out[1] = r.kappa_l;
    out[2] = r.kappa_r;
    out[3] = r.kappa_ext;
    out[4] = r.kappa_tilde;
    out[5] = r.bound;
    out[6] = r.bound_holds ? 1.0 : 0.0;
  });
}

int sbx_els_density_on_refined(sbx_els e, const double* tau_n, double* out) {
  return guard([&] {
    sbx::require(e && e->e, "null els handle");
    sbx::els_density_on_refined(*e->e, tau_n, out);
  });
}

int sbx_els_xw(sbx_els e, double* X, double* W) {
  return guard([&] {
    sbx::require(e && e->e, "null els handle");
    sbx::els_download_xw(*e->e, X, W, sbx::lib_stream());
  });
}

// ---------------------------------------------------------------- multi-GPU
namespace {

// Runs f on device blocks: host inputs are staged in, host outputs copied back.
struct Staged {
  sbx::DevBuf<double> buf;
  const double* in(const double* h, int64_t rows, int64_t cols, int64_t ld, bool dev, cudaStream_t s) {
    if (dev || rows == 0 || cols == 0) return h;
    buf.resize(size_t(rows * cols));
    SBX_CUDA(cudaMemcpy2DAsync(buf.get(), size_t(rows) * 8, h, size_t(ld) * 8, size_t(rows) * 8, size_t(cols),
                               cudaMemcpyHostToDevice, s));
    return buf.get();
  }
  double* out(double* h, int64_t rows, int64_t cols, bool dev) {
    if (dev || rows == 0 || cols == 0) return h;
    buf.resize(size_t(rows * cols));
    return buf.get();
  }
  void back(double* h, int64_t rows, int64_t cols, int64_t ld, bool dev, cudaStream_t s) {
    if (dev || rows == 0 || cols == 0) return;
    SBX_CUDA(cudaMemcpy2DAsync(h, size_t(ld) * 8, buf.get(), size_t(rows) * 8, size_t(rows) * 8, size_t(cols),
                               cudaMemcpyDeviceToHost, s));
  }
};
}  // namespace

int sbx_comm_unique_id(uint8_t* id128) {
  return guard([&] { sbx::nccl_unique_id(id128); });
}

int sbx_comm_create(const uint8_t* id128, int world, int rank, sbx_comm* out) {
  return guard([&] { *out = new sbx_comm_s{sbx::make_nccl_collective(id128, world, rank)}; });
}

int sbx_comm_create_loopback(int world, sbx_comm* members) {
  return guard([&] {
    auto g = sbx::make_loopback_group(world);
    for (int r = 0; r < world; ++r) members[r] = new sbx_comm_s{std::move(g[size_t(r)])};
  });
}

int sbx_comm_destroy(sbx_comm c) { return destroy_handle(c); }

int sbx_comm_info(sbx_comm c, int* world, int* rank) {
  return guard([&] {
    *world = Cm(c).world();
    *rank = Cm(c).rank();
  });
}

int sbx_hbs_solve_sharded(sbx_hbs h, sbx_comm c, const double* b_local, int64_t ldb, int64_t nrhs, double* x_local,
                          int64_t ldx, int flags, void* stream) {
  return guard([&] {
    const cudaStream_t s = stream_of(stream);
    sbx::StreamScope scope(s);
    sbx::HbsOp& op = H(h);
    sbx::Collective& cm = Cm(c);
    const sbx::ShardPlans& S = sbx::hbs_shard(op, cm.world(), cm.rank());
    const int64_t rows = S.row1 - S.row0;
    sbx::require(nrhs >= 0 && ldb >= rows && ldx >= rows, "hbs_solve_sharded: bad sizes");
    if (nrhs == 0) return;
    const bool dev = (flags & SBX_DEVICE_PTRS) != 0;
    Staged bi, xo;
    const double* bd = bi.in(b_local, rows, nrhs, ldb, dev, s);
    double* xd = xo.out(x_local, rows, nrhs, dev);
    sbx::hbs_solve_sharded(op, cm, bd, dev ? ldb : rows, nrhs, xd, dev ? ldx : rows, s);
    xo.back(x_local, rows, nrhs, ldx, dev, s);
    SBX_CUDA(cudaStreamSynchronize(s));
  });
}

int sbx_els_shard_build(sbx_hbs a_oo, sbx_comm c, sbx_geom old_g, sbx_geom new_g, sbx_plan plan, sbx_update upd,
                        int formulation, double mu, void* stream, sbx_els_shard* out) {
  return guard([&] {
    sbx::require(plan && plan->p && upd && upd->u, "null handle");
    const cudaStream_t s = stream_of(stream);
    sbx::StreamScope scope(s);
    auto e = sbx::els_shard_build(H(a_oo), Cm(c), G(old_g), G(new_g), *plan->p, *upd->u, formulation, mu, s);
    *out = new sbx_els_shard_s{std::move(e), upd->u};
  });
}

int sbx_els_shard_info(sbx_els_shard e, int64_t* info) {
  return guard([&] {
    sbx::require(e && e->e, "null els shard handle");
    const auto& x = *e->e;
    const int64_t v[7] = {x.row0, x.row1, x.local_p(), x.k, x.n_k + x.n_c + x.n_p, x.G, x.p};
    std::copy(v, v + 7, info);
  });
}

int sbx_els_shard_rows(sbx_els_shard e, int64_t* ext_rows) {
  return guard([&] {
    sbx::require(e && e->e, "null els shard handle");
    std::copy(e->e->ext_of_local.begin(), e->e->ext_of_local.end(), ext_rows);
  });
}

int sbx_els_shard_solve(sbx_els_shard e, const double* g_local, int64_t ldg, const double* g_p, int64_t ldgp,
                        int64_t nrhs, double* y_local, int64_t ldy, double* y_p, int64_t ldyp, int flags,
                        void* stream) {
  return guard([&] {
    sbx::require(e && e->e, "null els shard handle");
    sbx::ElsShard& x = *e->e;
    const cudaStream_t s = stream_of(stream);
    sbx::StreamScope scope(s);
    const int64_t rows = x.rows(), np = x.local_p();
    sbx::require(nrhs >= 0 && ldg >= rows && ldy >= rows, "els_shard_solve: bad sizes");
    if (np > 0) sbx::require(g_p && y_p && ldgp >= np && ldyp >= np, "els_shard_solve: rank 0 needs the added rows");
    if (nrhs == 0) return;
    const bool dev = (flags & SBX_DEVICE_PTRS) != 0;
    Staged gi, gpi, yo, ypo;
    const double* gd = gi.in(g_local, rows, nrhs, ldg, dev, s);
    const double* gpd = np > 0 ? gpi.in(g_p, np, nrhs, ldgp, dev, s) : nullptr;
    double* yd = yo.out(y_local, rows, nrhs, dev);
    double* ypd = np > 0 ? ypo.out(y_p, np, nrhs, dev) : nullptr;
    sbx::els_shard_solve(x, gd, dev ? ldg : rows, gpd, dev ? ldgp : std::max<int64_t>(np, 1), nrhs, yd,
                         dev ? ldy : rows, ypd, dev ? ldyp : std::max<int64_t>(np, 1), s);
    yo.back(y_local, rows, nrhs, ldy, dev, s);
    if (np > 0) ypo.back(y_p, np, nrhs, ldyp, dev, s);
    SBX_CUDA(cudaStreamSynchronize(s));
  });
}

int sbx_els_shard_destroy(sbx_els_shard e) { return destroy_handle(e); }

}  // extern "C"
