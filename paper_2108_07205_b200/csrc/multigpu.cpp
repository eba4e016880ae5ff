// Multi-GPU partitioned solve and Woodbury; see multigpu.hpp.
#include "multigpu.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <limits>
#include <mutex>

#include "dense.hpp"

namespace sbx {

// ---------------------------------------------------------------- NCCL (loaded at run time)
namespace {
struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

// An NCCL the process already loaded (torch's) is reused; otherwise the
// system libnccl.  Loading it lazily keeps single-GPU users free of it.
const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW);
    if (!h) return;
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
  });
  if (!api.get_unique_id || !api.comm_init_rank || !api.all_gather || !api.all_reduce || !api.comm_destroy)
    throw Error(6, "NCCL not available (libnccl.so.2 could not be loaded)");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    const char* msg = nccl().error_string ? nccl().error_string(r) : "?";
    throw Error(6, std::string("NCCL error in ") + what + ": " + msg);
  }
}

class NcclCollective final : public Collective {
 public:
  NcclCollective(const unsigned char id[128], int world, int rank) : world_(world), rank_(rank) {
    ncclUniqueId uid;
    static_assert(sizeof(uid) == 128, "NCCL unique id size");
    std::memcpy(&uid, id, sizeof(uid));
    nccl_check(nccl().comm_init_rank(&comm_, world, uid, rank), "ncclCommInitRank");
  }
  ~NcclCollective() override {
    if (comm_) nccl().comm_destroy(comm_);
  }
  int world() const override { return world_; }
  int rank() const override { return rank_; }
  void all_gather(double* buf, size_t count, cudaStream_t s) override {
    if (count == 0) return;
    nccl_check(nccl().all_gather(buf + size_t(rank_) * count, buf, count, ncclDouble, comm_, s), "ncclAllGather");
  }
  void all_reduce_sum(double* buf, size_t count, cudaStream_t s) override {
    if (count == 0) return;
    nccl_check(nccl().all_reduce(buf, buf, count, ncclDouble, ncclSum, comm_, s), "ncclAllReduce");
  }

 private:
  ncclComm_t comm_ = nullptr;
  int world_, rank_;
};

// ---------------------------------------------------------------- loopback group
__global__ void sum_blocks_kernel(const double* __restrict__ tmp, int world, size_t count, double* __restrict__ out) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < count; i += size_t(gridDim.x) * blockDim.x) {
    double a = 0.0;
    for (int q = 0; q < world; ++q) a += tmp[size_t(q) * count + i];  // rank order: same bits on every rank
    out[i] = a;
  }
}

struct LoopShared {
  explicit LoopShared(int w) : world(w), bufs(size_t(w), nullptr), ready(size_t(w)), copied(size_t(w)) {
    for (int q = 0; q < w; ++q) {
      SBX_CUDA(cudaEventCreateWithFlags(&ready[size_t(q)], cudaEventDisableTiming));
      SBX_CUDA(cudaEventCreateWithFlags(&copied[size_t(q)], cudaEventDisableTiming));
    }
  }
  ~LoopShared() {
    for (auto e : ready) cudaEventDestroy(e);
    for (auto e : copied) cudaEventDestroy(e);
  }
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const unsigned long long g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return;
    }
    cv.wait(lk, [&] { return gen != g; });
  }
  int world;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long gen = 0;
  std::vector<double*> bufs;
  std::vector<cudaEvent_t> ready, copied;
};

// Member r of an in-process group: every collective is three host barriers
// around stream-ordered device copies (event waits, no device spinning).
class LoopbackMember final : public Collective {
 public:
  LoopbackMember(std::shared_ptr<LoopShared> g, int r) : g_(std::move(g)), r_(r) {}
  int world() const override { return g_->world; }
  int rank() const override { return r_; }
  void all_gather(double* buf, size_t count, cudaStream_t s) override {
    exchange(buf, count, s, [&](int q) {
      SBX_CUDA(cudaMemcpyAsync(buf + size_t(q) * count, g_->bufs[size_t(q)] + size_t(q) * count,
                               count * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }, nullptr);
  }
  void all_reduce_sum(double* buf, size_t count, cudaStream_t s) override {
    const int W = world();
    DevBuf<double> tmp(static_cast<size_t>(W) * count);
    exchange(buf, count, s, [&](int q) {
      SBX_CUDA(cudaMemcpyAsync(tmp.get() + size_t(q) * count, g_->bufs[size_t(q)], count * sizeof(double),
                               cudaMemcpyDeviceToDevice, s));
    }, [&] {
      SBX_CUDA(cudaMemcpyAsync(tmp.get() + size_t(r_) * count, buf, count * sizeof(double),
                               cudaMemcpyDeviceToDevice, s));
    });
    if (count) {
      sum_blocks_kernel<<<unsigned(std::min<size_t>((count + 255) / 256, 1024)), 256, 0, s>>>(tmp.get(), W, count, buf);
      SBX_LAUNCHED();
    }
    SBX_CUDA(cudaStreamSynchronize(s));  // tmp returns to the pool
  }

 private:
  template <class Copy, class Own>
  void exchange(double* buf, size_t count, cudaStream_t s, Copy copy_from, Own own) {
    const int W = world();
    g_->bufs[size_t(r_)] = buf;
    SBX_CUDA(cudaEventRecord(g_->ready[size_t(r_)], s));
    g_->barrier();  // every member's block is published (event recorded)
    for (int q = 0; q < W; ++q) {
      if (q == r_) continue;
      SBX_CUDA(cudaStreamWaitEvent(s, g_->ready[size_t(q)], 0));
      if (count) copy_from(q);
    }
    if constexpr (!std::is_same_v<Own, std::nullptr_t>) own();
    SBX_CUDA(cudaEventRecord(g_->copied[size_t(r_)], s));
    g_->barrier();  // every member has enqueued its reads of the others' blocks
    for (int q = 0; q < W; ++q)
      if (q != r_) SBX_CUDA(cudaStreamWaitEvent(s, g_->copied[size_t(q)], 0));
    g_->barrier();  // events may be recorded again by the next collective
  }
  std::shared_ptr<LoopShared> g_;
  int r_;
};

__global__ void gather_rows_kernel(const double* __restrict__ src, i64 lds, const i64* __restrict__ map, i64 rows,
                                   i64 cols, double* __restrict__ dst, i64 ldd) {
  const i64 total = rows * cols;
  for (i64 e = blockIdx.x * i64(blockDim.x) + threadIdx.x; e < total; e += i64(gridDim.x) * blockDim.x) {
    const i64 r = e % rows, c = e / rows;
    dst[r + c * ldd] = src[map[r] + c * lds];
  }
}

void gather_rows(const double* src, i64 lds, const i64* map, i64 rows, i64 cols, double* dst, i64 ldd,
                 cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return;
  const i64 total = rows * cols;
  gather_rows_kernel<<<unsigned(std::min<i64>((total + 255) / 256, 148 * 16)), 256, 0, s>>>(src, lds, map, rows,
                                                                                           cols, dst, ldd);
  SBX_LAUNCHED();
}

std::vector<i64> scalars(const std::vector<i64>& nodes) {
  std::vector<i64> o;
  o.reserve(2 * nodes.size());
  for (i64 n : nodes) {
    o.push_back(2 * n);
    o.push_back(2 * n + 1);
  }
  return o;
}

GemmJob gemm(const double* A, const double* B, double* C, i64 m, i64 n, i64 k, i64 lda, i64 ldb, i64 ldc, int ta,
             double alpha, double beta) {
  return {A, B, C, int(m), int(n), int(k), int(lda), int(ldb), int(ldc), ta, 0, alpha, beta};
}
}  // namespace

void nccl_unique_id(unsigned char out[128]) {
  ncclUniqueId uid;
  nccl_check(nccl().get_unique_id(&uid), "ncclGetUniqueId");
  std::memcpy(out, &uid, 128);
}

std::unique_ptr<Collective> make_nccl_collective(const unsigned char id[128], int world, int rank) {
  require(world >= 1 && rank >= 0 && rank < world, "comm: rank out of range");
  return std::make_unique<NcclCollective>(id, world, rank);
}

std::vector<std::unique_ptr<Collective>> make_loopback_group(int world) {
  require(world >= 1, "loopback group: world must be positive");
  auto g = std::make_shared<LoopShared>(world);
  std::vector<std::unique_ptr<Collective>> out;
  for (int r = 0; r < world; ++r) out.push_back(std::make_unique<LoopbackMember>(g, r));
  return out;
}

std::vector<std::vector<double>> gather_host(Collective& c, const std::vector<double>& mine, cudaStream_t s) {
  const int G = c.world(), p = c.rank();
  DevBuf<double> sz(static_cast<size_t>(G));
  sz.zero(s);
  const double me = double(mine.size());
  SBX_CUDA(cudaMemcpyAsync(sz.get() + p, &me, sizeof(double), cudaMemcpyHostToDevice, s));
  c.all_gather(sz.get(), 1, s);
  std::vector<double> hs(static_cast<size_t>(G));
  sz.download(hs.data(), hs.size(), s);
  SBX_CUDA(cudaStreamSynchronize(s));
  size_t mx = 1;
  for (double v : hs) mx = std::max(mx, size_t(v));
  DevBuf<double> buf(static_cast<size_t>(G) * mx);
  buf.zero(s);
  if (!mine.empty())
    SBX_CUDA(cudaMemcpyAsync(buf.get() + size_t(p) * mx, mine.data(), mine.size() * sizeof(double),
                             cudaMemcpyHostToDevice, s));
  c.all_gather(buf.get(), mx, s);
  std::vector<double> all(static_cast<size_t>(G) * mx);
  buf.download(all.data(), all.size(), s);
  SBX_CUDA(cudaStreamSynchronize(s));
  std::vector<std::vector<double>> out(static_cast<size_t>(G));
  for (int q = 0; q < G; ++q)
    out[size_t(q)].assign(all.begin() + i64(q) * i64(mx), all.begin() + i64(q) * i64(mx) + i64(hs[size_t(q)]));
  return out;
}

// ---------------------------------------------------------------- sharded solve
void hbs_solve_sharded(HbsOp& op, Collective& c, const double* b_local, i64 ldb, i64 nrhs, double* x_local,
                       i64 ldx, cudaStream_t s) {
  const int G = c.world(), p = c.rank();
  const ShardPlans& S = hbs_shard(op, G, p);
  require(nrhs >= 1, "sharded solve: nrhs must be positive");
  const size_t chunk = size_t(S.kmax * nrhs);
  DevBuf<double> hats(std::max<size_t>(size_t(G) * chunk, 1));
  // 1. local up-sweep; this rank's hat lands at block p of the gather buffer
  hbs_solve_shard_up(op, G, p, b_local, ldb, nrhs, hats.get() + size_t(p) * chunk, true, s);
  // 2. the only exchange: the G subtree-root hats (NCCL over NVLink)
  if (G > 1) c.all_gather(hats.get(), chunk, s);
  // 3. top g levels redundantly, then the local down-sweep
  hbs_solve_shard_down(op, G, p, hats.get(), nrhs, x_local, ldx, true, s);
  SBX_CUDA(cudaStreamSynchronize(s));  // hats returns to the pool
}

// ---------------------------------------------------------------- sharded Woodbury
std::unique_ptr<ElsShard> els_shard_build(HbsOp& a_oo, Collective& c, const Geom& old_g, const Geom& new_g,
                                          const Plan& plan, const Update& upd, int form, double mu, cudaStream_t s) {
  require(a_oo.has_inverse, "els_shard_build: diagonal solver lacks inverse");
  auto e = std::make_unique<ElsShard>();
  e->a_oo = &a_oo;
  e->comm = &c;
  e->G = c.world();
  e->p = c.rank();
  const ShardPlans& S = hbs_shard(a_oo, e->G, e->p);
  e->row0 = S.row0;
  e->row1 = S.row1;
  const auto kept_old_s = scalars(plan.kept_old), cut_s = scalars(plan.cut_old);
  e->n_k = i64(kept_old_s.size());
  e->n_c = i64(cut_s.size());
  e->n_p = 2 * i64(plan.added_new.size());
  e->k = upd.k;
  const i64 nkc = e->n_k + e->n_c, n = nkc + e->n_p, k = e->k, rows = e->rows();
  require(a_oo.n == nkc, "els_shard_build: diagonal solver size does not match the old mesh");
  require(upd.n_ext() == n, "els_shard_build: update factor size does not match the plan");
  // owned ext rows in old-mesh order (kept, cut rows map 1:1 onto the old mesh)
  e->ext_of_local.assign(size_t(rows), -1);
  for (i64 q = 0; q < nkc; ++q) {
    const i64 o = q < e->n_k ? kept_old_s[size_t(q)] : cut_s[size_t(q - e->n_k)];
    if (o >= e->row0 && o < e->row1) e->ext_of_local[size_t(o - e->row0)] = q;
  }
  for (i64 v : e->ext_of_local) require(v >= 0, "els_shard_build: ext rows do not cover the owned old-mesh rows");
  e->d_ext_of_local.upload(e->ext_of_local, s);
  if (e->p == 0 && e->n_p > 0) {
    if (upd.app && upd.app->matches(new_g, plan, form, mu, a_oo.eps))
      e->app = upd.app;
    else
      e->app = build_app_solver(new_g, plan, form, mu, a_oo.eps, s);
  }
  if (k == 0) {
    SBX_CUDA(cudaStreamSynchronize(s));
    return e;
  }
  // X_own = A_oo^{-1} L on the owned rows: the sharded solve with k columns
  DevBuf<double> Lloc(static_cast<size_t>(rows * k)), RT(static_cast<size_t>(n * k));
  gather_rows(upd.L->get(), n, e->d_ext_of_local.get(), rows, k, Lloc.get(), rows, s);
  e->X.resize(size_t(rows * k));
  hbs_solve_sharded(a_oo, c, Lloc.get(), rows, k, e->X.get(), rows, s);
  // owned columns of R, kept transposed (rows x k) so both products read them as column-major panels
  copy_batched({{upd.R.get(), RT.get(), int(n), int(k), int(k), int(n), 1, 0}}, s);
  e->Rt.resize(size_t(rows * k));
  gather_rows(RT.get(), n, e->d_ext_of_local.get(), rows, k, e->Rt.get(), rows, s);
  // W partial = R_own X_own (+ R_p X_p on rank 0), summed over the ranks
  DevBuf<double> Wp(static_cast<size_t>(k * k));
  gemm_batched({gemm(e->Rt.get(), e->X.get(), Wp.get(), k, k, rows, rows, rows, k, 1, 1.0, 0.0)}, s);
  if (e->app) {
    e->Xp.resize(size_t(e->n_p * k));
    app_solve_device(*e->app, upd.L->get() + nkc, n, e->Xp.get(), e->n_p, k, s);
    e->Rpt.resize(size_t(e->n_p * k));
    launch_copy2d(RT.get() + nkc, n, e->Rpt.get(), e->n_p, e->n_p, k, s);
    gemm_batched({gemm(e->Rpt.get(), e->Xp.get(), Wp.get(), k, k, e->n_p, e->n_p, e->n_p, k, 1, 1.0, 1.0)}, s);
  }
  c.all_reduce_sum(Wp.get(), size_t(k * k), s);
  // W = I + R X, inverse and the reference's rcond gate (els.cpp:124-135), on every rank
  e->Wmat.resize(size_t(k * k));
  SBX_CUDA(cudaMemcpyAsync(e->Wmat.get(), Wp.get(), size_t(k * k) * 8, cudaMemcpyDeviceToDevice, s));
  launch_add_identity(e->Wmat.get(), k, k, s);
  DevBuf<double> wlu(static_cast<size_t>(k * k));
  SBX_CUDA(cudaMemcpyAsync(wlu.get(), e->Wmat.get(), size_t(k * k) * 8, cudaMemcpyDeviceToDevice, s));
  e->Winv.resize(size_t(k * k));
  const double rc = dense_inverse(wlu.get(), k, e->Winv.get(), s);
  if (rc < std::sqrt(std::numeric_limits<double>::epsilon()))
    throw Error(4,
                "woodbury operator numerically singular; consider the optimal-basis compression "
                "mode at woodbury solve");
  SBX_CUDA(cudaStreamSynchronize(s));
  return e;
}

void els_shard_solve(ElsShard& e, const double* g_local, i64 ldg, const double* g_p, i64 ldgp, i64 nrhs,
                     double* y_local, i64 ldy, double* y_p, i64 ldyp, cudaStream_t s) {
  if (nrhs == 0) return;
  const i64 rows = e.rows(), k = e.k, np = e.local_p();
  // y = Atilde^{-1} g: the sharded A_oo solve, A_pp on rank 0
  hbs_solve_sharded(*e.a_oo, *e.comm, g_local, ldg, nrhs, y_local, ldy, s);
  if (np > 0) app_solve_device(*e.app, g_p, ldgp, y_p, ldyp, nrhs, s);
  if (k == 0) return;
  // t = R y summed over ranks; y -= X W^{-1} t   (els.cpp:147-152)
  DevBuf<double> t(static_cast<size_t>(k * nrhs)), z(static_cast<size_t>(k * nrhs));
  std::vector<GemmJob> jt = {gemm(e.Rt.get(), y_local, t.get(), k, nrhs, rows, rows, ldy, k, 1, 1.0, 0.0)};
  gemm_batched(jt, s);
  if (np > 0) gemm_batched({gemm(e.Rpt.get(), y_p, t.get(), k, nrhs, np, np, ldyp, k, 1, 1.0, 1.0)}, s);
  e.comm->all_reduce_sum(t.get(), size_t(k * nrhs), s);
  gemm_batched({gemm(e.Winv.get(), t.get(), z.get(), k, nrhs, k, k, k, k, 0, 1.0, 0.0)}, s);
  gemm_batched({gemm(e.X.get(), z.get(), y_local, rows, nrhs, k, rows, k, ldy, 0, -1.0, 1.0)}, s);
  if (np > 0) gemm_batched({gemm(e.Xp.get(), z.get(), y_p, np, nrhs, k, np, k, ldyp, 0, -1.0, 1.0)}, s);
  SBX_CUDA(cudaStreamSynchronize(s));  // t, z return to the pool
}

}  // namespace sbx
