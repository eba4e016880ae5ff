// Batched device IDs (see idengine.hpp).
#include "idengine.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <condition_variable>
#include <memory>
#include <mutex>

namespace sbx {

namespace {
thread_local IdRendezvous* tl_rv = nullptr;

int sm_count() {
  static const int sms = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  return sms;
}
}  // namespace

// Engine routing and launches for one batch of CPQR jobs (engine: 0 auto).
namespace {
// SBX_ID_DUMP=<dir>: every batch (shapes, stop rule and W^T) as
// <dir>/batch_NNNN.bin for offline engine comparisons (scripts/id_bench.cu).
void dump_batch(const std::vector<QrJob>& all, cudaStream_t s) {
  static const char* dir = std::getenv("SBX_ID_DUMP");
  if (!dir || all.empty()) return;
  static int seq = 0;
  char path[512];
  std::snprintf(path, sizeof(path), "%s/batch_%04d.bin", dir, seq++);
  FILE* f = std::fopen(path, "wb");
  if (!f) return;
  const long long np = static_cast<long long>(all.size());
  std::fwrite(&np, sizeof(np), 1, f);
  SBX_CUDA(cudaStreamSynchronize(s));
  for (const auto& j : all) {
    const long long hdr[4] = {j.M, j.n, j.max_steps, 0};
    std::fwrite(hdr, sizeof(hdr), 1, f);
    std::fwrite(&j.stop_eps, sizeof(double), 1, f);
    std::vector<double> h(size_t(j.M) * j.n);
    SBX_CUDA(cudaMemcpy2D(h.data(), size_t(j.M) * sizeof(double), j.a, size_t(j.lda) * sizeof(double),
                          size_t(j.M) * sizeof(double), size_t(j.n), cudaMemcpyDeviceToHost));
    std::fwrite(h.data(), sizeof(double), h.size(), f);
  }
  std::fclose(f);
}
}  // namespace

void launch_id_jobs(const std::vector<QrJob>& all, int force_engine, cudaStream_t s) {
  dump_batch(all, s);
  static const int env_engine = [] {  // diagnostics: one engine for every batch
    const char* e = std::getenv("SBX_FORCE_ENGINE");
    return e ? std::atoi(e) : 0;
  }();
  if (force_engine == 0) force_engine = env_engine;
  KernelTimer kt("id_factor", s);  // every CPQR engine launch of the batch (bench: step-dominant family)
  std::vector<QrJob> jobs, big, chip, clus, reg, strm, rows, push, rrow, bq;
  static const int tsqr_max_m = [] {
    const char* e = std::getenv("SBX_TSQR_MAXM");
    return e ? std::atoi(e) : 0;
  }();
  // streaming TSQR of crowded batches: candidates per problem (the quad
  // kernel holds n <= 128) and TSQR steps (row blocks x n) beyond which one
  // problem's latency would set the whole round
  static const int tsqr_max_n = [] {
    const char* e = std::getenv("SBX_TSQR_MAXN");
    return e ? std::atoi(e) : 128;  // measured (scripts/route_scan.sh): 129..144 on the warp kernel loses
  }();
  static const i64 tsqr_max_steps = [] {
    const char* e = std::getenv("SBX_TSQR_MAXSTEPS");
    return e ? std::atoll(e) : i64(1) << 40;
  }();
  // Routing (measured per batch on the per-step problem mix, see
  // scripts/id_bench.cu --replay): while the whole batch fits the chip in
  // about two waves, the on-chip cooperative engine (exact CTA counts, one
  // grid barrier per step) wins; crowded batches are throughput bound, where
  // streaming TSQR (one CTA per tall problem, R0 on chip) and the
  // register-resident cluster engine win.
  const int sms = sm_count();
  i64 chip_ctas = 0;
  for (const auto& j : all) {
    const int g = cpqr_smem_ctas(j.M, j.n);
    chip_ctas += g > 0 ? g : sms;
  }
  const bool crowded = chip_ctas > 2 * i64(sms);
  // streaming TSQR is slow per problem (all n Householder steps before the
  // pivoted ones) and only pays off by sheer numbers of tall problems
  i64 n_tall = 0;
  for (const auto& j : all) n_tall += (j.n <= 144 && j.M > j.n && j.M <= 4096) ? 1 : 0;
  const bool tsqr_crowd = crowded && n_tall >= sms / 2;
  static const bool log = std::getenv("SBX_ID_LOG") != nullptr;  // diagnostics
  static const bool no_cluster = std::getenv("SBX_NO_CLUSTER") != nullptr;  // diagnostics
  static const bool no_reg = std::getenv("SBX_NO_REG") != nullptr;          // diagnostics
  // Few tall problems (the late rounds of the lockstep hierarchies): the
  // row-split cluster engine (two O(n) DSMEM exchanges per step) beats the
  // grid-barrier engine's per-step latency (measured on the replayed cfg2
  // rounds of <= 19 problems: 0.65 -> 0.42 ms, 0.74 -> 0.39 ms, 0.85 -> 0.77 ms)
  static const bool no_rows = std::getenv("SBX_NO_ROWS") != nullptr;  // diagnostics
  bool rows_all = !no_rows && !crowded && !all.empty() && all.size() <= 24;
  for (const auto& j : all) rows_all = rows_all && cpqr_rows_cluster(j.M, j.n) > 0;
  // The register-resident row-split engine (engine 9: one pushed exchange
  // per step, no serial section) takes every tall problem it holds while
  // their minimal clusters need at most ~4.75 waves of SMs (replayed cfg2
  // rounds, routing cap 296 / 700 / 1000 / 3000 CTAs: step median 20.9 /
  // 19.9 / 19.8 / 22.8 ms; the 151- and 75-problem rounds 2.09 -> 1.06 and
  // 1.40 -> 0.83 ms, the <= 38-problem rounds 1.00 -> 0.46, 0.78 -> 0.34,
  // 0.43 -> 0.24, 0.40 -> 0.21 ms); crowded rounds keep the throughput
  // engines below.
  static const bool no_rr = std::getenv("SBX_NO_RR") != nullptr;  // diagnostics
  static const i64 rr_cap = [] {
    const char* e = std::getenv("SBX_RR_CAP");
    return e ? std::atoll(e) : i64(-1);  // default: 19/4 of the SM count (replayed cfg2 rounds)
  }();
  // (tall problems only: on W^T with M < 2n it loses to the throughput engines)
  auto rr_fit = [](const QrJob& j) { return j.M >= 2 * j.n ? cpqr_regrows_cluster(j.M, j.n) : 0; };
  i64 rr_ctas = 0;
  for (const auto& j : all) rr_ctas += rr_fit(j);
  const bool rr_route = !no_rr && rr_ctas > 0 && rr_ctas <= (rr_cap >= 0 ? rr_cap : 19 * i64(sms) / 4);
  // in crowded rounds engine 9 still takes the problems the register
  // cluster engine would (wide-ish W^T stopping after a few steps)
  static const bool rr_e5 = !no_rr && std::getenv("SBX_RR_E5") != nullptr;  // measured: slower (off)
  static const bool rr_tsqr = !no_rr && std::getenv("SBX_RR_TSQR") != nullptr;
  // crowded tall problems: the blocked DMMA QR (engine 10) instead of the
  // streaming TSQR where it holds them (replayed cfg2 batches: 8.3 -> 6.6,
  // 4.4 -> 3.7, 1.54 -> 1.22 ms)
  static const bool use_bqr = std::getenv("SBX_NO_BQR") == nullptr;
  std::string line;
  for (const auto& j : all) {
    int engine = force_engine;
    if (engine == 8 && cpqr_push_cluster(j.M, j.n) == 0) engine = 0;  // does not fit: auto route
    if (engine == 9 && cpqr_regrows_cluster(j.M, j.n) == 0) engine = 0;
    if (engine == 10 && !bqr_ok(j.M, j.n)) engine = 0;
    if (engine == 0 && rr_route && rr_fit(j) > 0) engine = 9;
    if (engine == 0 && rows_all) engine = 7;
    if (engine == 0) {
      const int g = cpqr_smem_ctas(j.M, j.n);
      const bool chip_ok = !no_coop_flag() && g > 0 && g <= sms;
      const bool tsqr_ok = j.n <= tsqr_max_n && j.M > j.n &&
                           (j.M <= tsqr_max_m ||
                            (tsqr_crowd && j.M <= 4096 && i64((j.M + 127) / 128) * j.n <= tsqr_max_steps));
      const bool one_cta = qr_smem_need(j.M, j.n) <= size_t(200 * 1024);
      int rg = 0;
      const int rc = no_reg ? -1 : cpqr_reg_config(j.M, j.n, &rg);
      const int cs = cpqr_cluster_size(j.M, j.n);
      if (!crowded && chip_ok) engine = 3;
      else if (tsqr_ok) engine = (rr_tsqr && rr_fit(j) > 0) ? 9 : (use_bqr && bqr_ok(j.M, j.n)) ? 10 : 1;
      else if (rc >= 0 && !(rc >= 3 && cs > 0 && cs < rg)) engine = (rr_e5 && rr_fit(j) > 0) ? 9 : 5;
      else if (one_cta) engine = 1;
      else if (!no_cluster && cs > 0) engine = 4;
      else if (chip_ok) engine = 3;
      else if (!no_coop_flag() && i64(j.M) * j.n >= IdBatch::kCoopEntries) engine = 2;
      else engine = 1;
    }
    if (log) line += " " + std::to_string(j.M) + "x" + std::to_string(j.n) + "/e" + std::to_string(engine);
    (engine == 2   ? big
     : engine == 3 ? chip
     : engine == 4 ? clus
     : engine == 5 ? reg
     : engine == 6 ? strm
     : engine == 7 ? rows
     : engine == 8 ? push
     : engine == 9 ? rrow
     : engine == 10 ? bq
                   : jobs)
        .push_back(j);
  }
  cudaEvent_t lg0 = nullptr, lg1 = nullptr;
  if (log) {
    SBX_CUDA(cudaEventCreate(&lg0));
    SBX_CUDA(cudaEventCreate(&lg1));
    SBX_CUDA(cudaEventRecord(lg0, s));
  }
  // The engine groups of a round hold no grid-wide barriers between each
  // other, so they run side by side: the first non-empty group on s, every
  // other one on a stream forked from s (pooled), all joined back into s.
  static const int fork_env = [] {
    const char* e = std::getenv("SBX_ID_FORK");
    return e ? std::atoi(e) : 1;
  }();
  struct Group {
    std::vector<QrJob>* v;
    void (*fn)(const std::vector<QrJob>&, cudaStream_t);
  };
  // (launch order = the block scheduler's order: the longest-running
  // throughput engines first, so the shorter ones fill their tail waves)
  const Group groups[] = {{&bq, bqr_batched},           {&jobs, qr_batched},          {&rrow, cpqr_regrows_batched},
                          {&reg, cpqr_reg_batched},     {&big, cpqr_coop_batched},    {&chip, cpqr_smem_batched},
                          {&clus, cpqr_cluster_batched}, {&strm, cpqr_stream_batched}, {&rows, cpqr_rows_batched},
                          {&push, cpqr_push_batched}};
  // (every side stream forks from s BEFORE anything of this round is
  // launched on s, so no group waits for another)
  std::vector<std::unique_ptr<SideStream>> sides;
  std::vector<std::pair<const Group*, cudaStream_t>> plan;
  bool first = true;
  for (const auto& g : groups) {
    if (g.v->empty()) continue;
    const bool forkable = fork_env == 1 || (fork_env == 2 && (g.v == &rrow || g.v == &reg));
    if (first || !forkable) {
      plan.push_back({&g, s});
      first = false;
      continue;
    }
    sides.emplace_back(new SideStream(s));
    plan.push_back({&g, sides.back()->get()});
  }
  for (const auto& pl : plan) {
    StreamScope ss(pl.second);
    pl.first->fn(*pl.first->v, pl.second);
  }
  for (auto& sd : sides) sd->join(s);
  if (log) {  // diagnostics: the batch's device time (serialises the stream)
    float ms = 0.f;
    SBX_CUDA(cudaEventRecord(lg1, s));
    SBX_CUDA(cudaEventSynchronize(lg1));
    SBX_CUDA(cudaEventElapsedTime(&ms, lg0, lg1));
    std::fprintf(stderr, "[sbx-id %.3f ms]%s\n", double(ms), line.c_str());
    SBX_CUDA(cudaEventDestroy(lg0));
    SBX_CUDA(cudaEventDestroy(lg1));
  }
}

// ---------------------------------------------------------------- rendezvous
IdRendezvous::IdRendezvous(int participants) : active_(participants) {}

void IdRendezvous::flush_locked(std::unique_lock<std::mutex>& lk, cudaStream_t s) {
  std::vector<QrJob> merged;
  for (auto* v : pending_) merged.insert(merged.end(), v->begin(), v->end());
  pending_.clear();
  waiting_ = 0;
  const unsigned long long gen = ++generation_;
  // the launch runs with the lock held: the waiters' job vectors (copied
  // above) are theirs again, but the next round must not start before this
  // launch is enqueued (stream order of the rounds)
  try {
    launch_id_jobs(merged, 0, s);
  } catch (...) {
    err_ = std::current_exception();
    err_gen_ = gen;
    cv_.notify_all();
    throw;
  }
  (void)lk;
  cv_.notify_all();
}

void IdRendezvous::submit(std::vector<QrJob>& jobs, cudaStream_t s) {
  std::unique_lock<std::mutex> lk(mu_);
  pending_.push_back(&jobs);
  ++waiting_;
  last_stream_ = s;
  if (waiting_ >= active_) {
    flush_locked(lk, s);
    return;
  }
  const unsigned long long gen = generation_;
  cv_.wait(lk, [&] { return generation_ != gen; });
  if (err_ && err_gen_ == gen + 1) std::rethrow_exception(err_);
}

void IdRendezvous::leave() noexcept {
  std::unique_lock<std::mutex> lk(mu_);
  --active_;
  if (waiting_ > 0 && waiting_ >= active_) {
    try {
      flush_locked(lk, last_stream_);
    } catch (...) {
      // recorded in err_ for the waiters of that round; the leaving thread
      // is done with the rendezvous (possibly unwinding already)
    }
  }
}

void IdRendezvous::enter() {
  std::lock_guard<std::mutex> lk(mu_);
  ++active_;
}

IdRendezvousScope::IdRendezvousScope(IdRendezvous* rv, bool enter) : rv_(rv), prev_(tl_rv) {
  if (rv && enter) rv->enter();
  tl_rv = rv;
}
IdRendezvousScope::~IdRendezvousScope() { leave(); }
void IdRendezvousScope::leave() noexcept {
  if (rv_) {
    rv_->leave();
    rv_ = nullptr;
    tl_rv = prev_;
  }
}

void id_rendezvous_leave() {
  if (tl_rv) {
    IdRendezvous* rv = tl_rv;
    tl_rv = nullptr;
    rv->leave();
  }
}

void IdBatch::factor(const std::vector<IdProblem>& probs, double stop_eps, cudaStream_t s) {
  probs_ = probs;
  const size_t np = probs.size();
  perm_off_.assign(np + 1, 0);
  std::vector<i64> diag_off(np + 1, 0);
  for (size_t p = 0; p < np; ++p) {
    perm_off_[p + 1] = perm_off_[p] + probs[p].n;
    diag_off[p + 1] = diag_off[p] + std::min(probs[p].M, probs[p].n);
  }
  d_perm_.reserve(size_t(std::max<i64>(perm_off_[np], 1)));
  d_diag_.reserve(size_t(std::max<i64>(diag_off[np], 1)));
  d_steps_.reserve(std::max<size_t>(np, 1));
  std::vector<QrJob> jobs;
  for (size_t p = 0; p < np; ++p) {
    const auto& pr = probs[p];
    if (pr.M == 0 || pr.n == 0) continue;
    QrJob j{};
    j.a = pr.wt;
    j.M = pr.M;
    j.n = pr.n;
    j.lda = pr.lda;
    j.pivot = 1;
    j.max_steps = 0;
    j.stop_eps = stop_eps;
    j.perm = d_perm_.get() + perm_off_[p];
    j.diag = d_diag_.get() + diag_off[p];
    j.steps = d_steps_.get() + p;
    jobs.push_back(j);
  }
  if (tl_rv && force_engine == 0)
    tl_rv->submit(jobs, s);  // one joint launch with the other participants' batches
  else
    launch_id_jobs(jobs, force_engine, s);
  std::vector<int> hperm(static_cast<size_t>(perm_off_[np]));
  std::vector<double> hdiag(static_cast<size_t>(diag_off[np]));
  std::vector<int> hsteps;
  if (ktimer_on() && np) hsteps.resize(np);
  {  // pivots, |r_jj| (and steps) through one pinned buffer: async copies, one sync
    const size_t b_diag = hdiag.size() * sizeof(double), b_perm = hperm.size() * sizeof(int),
                 b_steps = hsteps.size() * sizeof(int);
    PinnedLease pin(b_diag + b_perm + b_steps);
    char* h = static_cast<char*>(pin.get());
    if (b_diag) SBX_CUDA(cudaMemcpyAsync(h, d_diag_.get(), b_diag, cudaMemcpyDeviceToHost, s));
    if (b_perm) SBX_CUDA(cudaMemcpyAsync(h + b_diag, d_perm_.get(), b_perm, cudaMemcpyDeviceToHost, s));
    if (b_steps) SBX_CUDA(cudaMemcpyAsync(h + b_diag + b_perm, d_steps_.get(), b_steps, cudaMemcpyDeviceToHost, s));
    SBX_CUDA(cudaStreamSynchronize(s));
    if (b_diag) std::memcpy(hdiag.data(), h, b_diag);
    if (b_perm) std::memcpy(hperm.data(), h + b_diag, b_perm);
    if (b_steps) std::memcpy(hsteps.data(), h + b_diag + b_perm, b_steps);
  }
  if (!hsteps.empty()) {
    // algorithmic work of the pivoted Householder steps actually taken:
    // step j updates the (M-j) x (n-j) trailing block, 4 flops per entry
    // (column dot product + rank-1 update), whatever engine ran it
    double f = 0.0;
    for (size_t p = 0; p < np; ++p) {
      const auto& pr = probs[p];
      if (pr.M == 0 || pr.n == 0) continue;
      const int st = std::min({hsteps[p], pr.M, pr.n});
      for (int j = 0; j < st; ++j) f += 4.0 * double(pr.M - j) * double(pr.n - j);
    }
    ktimer_add_flops("id_factor", f);
  }
  diag_.assign(np, {});
  perm_.assign(np, {});
  for (size_t p = 0; p < np; ++p) {
    const auto& pr = probs[p];
    if (pr.M == 0 || pr.n == 0) {
      perm_[p].resize(size_t(pr.n));
      for (int i = 0; i < pr.n; ++i) perm_[p][size_t(i)] = i;
      continue;
    }
    perm_[p].assign(hperm.begin() + perm_off_[p], hperm.begin() + perm_off_[p + 1]);
    diag_[p].assign(hdiag.begin() + diag_off[p], hdiag.begin() + diag_off[p + 1]);
  }
}

i64 IdBatch::eps_rank(size_t p, double eps) const {
  const auto& d = diag_[p];
  if (d.empty()) return 0;
  const double r00 = d[0];
  i64 k = 0;
  if (r00 > 0.0)
    while (k < i64(d.size()) && d[size_t(k)] > eps * r00) ++k;
  return k;
}

i64 IdBatch::forced_rank(size_t p, i64 kf) const {
  const auto& d = diag_[p];
  if (d.empty() || kf <= 0) return 0;
  const double r00 = d[0];
  i64 k = 0;
  while (k < std::min<i64>(kf, i64(d.size())) && d[size_t(k)] > 1e-15 * r00) ++k;
  return k;
}

void IdBatch::interp(const std::vector<i64>& ks, const std::vector<double*>& P,
                     const std::vector<int>& ldp, cudaStream_t s) {
  std::vector<InterpJob> jobs;
  std::vector<i64> toff;
  i64 tsz = 0;
  for (size_t p = 0; p < probs_.size(); ++p) {
    toff.push_back(tsz);
    const i64 k = ks[p];
    if (k > 0) tsz += k * (probs_[p].n - k);
  }
  d_T_.reserve(size_t(std::max<i64>(tsz, 1)));
  for (size_t p = 0; p < probs_.size(); ++p) {
    const i64 k = ks[p];
    if (k <= 0) continue;
    InterpJob j{};
    j.a = probs_[p].wt;
    j.lda = probs_[p].lda;
    j.n = probs_[p].n;
    j.k = int(k);
    j.perm = d_perm_.get() + perm_off_[p];
    j.colmap = j.perm;  // every engine pivots in place: R(:, l) = A(:, perm[l])
    j.P = P[p];
    j.ldp = ldp[p];
    j.T = d_T_.get() + toff[p];
    jobs.push_back(j);
  }
  interp_batched(jobs, s);
}

}  // namespace sbx
