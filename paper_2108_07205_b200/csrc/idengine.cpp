// Batched device IDs (see idengine.hpp).
#include "idengine.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <condition_variable>
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
void launch_id_jobs(const std::vector<QrJob>& all, int force_engine, cudaStream_t s) {
  std::vector<QrJob> jobs, big, chip, clus;
  static const int tsqr_max_m = [] {
    const char* e = std::getenv("SBX_TSQR_MAXM");
    return e ? std::atoi(e) : 0;
  }();
  // Large batches have enough independent problems to fill the GPU with one
  // CTA each; cross-CTA engines only pay off when problems are few.  Count
  // the CTAs the cluster engine would need for the whole batch.
  const int sms = sm_count();
  i64 cluster_ctas = 0;
  for (const auto& j : all) cluster_ctas += std::max(1, cpqr_cluster_size(j.M, j.n));
  const bool crowded = cluster_ctas > 2 * i64(sms);
  static const bool log = std::getenv("SBX_ID_LOG") != nullptr;  // diagnostics
  std::string line;
  for (const auto& j : all) {
    int engine = force_engine;
    if (engine == 0) {
      // one CTA when the problem fits its shared memory (or is a short, tall
      // TSQR case); else a thread-block cluster, else the on-chip cooperative
      // engine when the slabs fit the GPU, else the L2-streaming cooperative
      // engine for big problems
      const bool tsqr_ok = j.n <= 144 && j.M > j.n && (j.M <= tsqr_max_m || (crowded && j.M <= 4096));
      const bool one_cta = qr_smem_need(j.M, j.n) <= size_t(200 * 1024) || tsqr_ok;
      const int g = cpqr_smem_ctas(j.M, j.n);
      static const bool no_cluster = std::getenv("SBX_NO_CLUSTER") != nullptr;  // diagnostics
      if (one_cta) engine = 1;
      else if (!no_cluster && cpqr_cluster_size(j.M, j.n) > 0) engine = 4;
      else if (no_coop_flag()) engine = 1;  // beside other streams: no grid-wide barriers
      else if (g > 0 && g <= sms) engine = 3;
      else if (i64(j.M) * j.n >= IdBatch::kCoopEntries) engine = 2;
      else engine = 1;
    }
    if (log) line += " " + std::to_string(j.M) + "x" + std::to_string(j.n) + "/e" + std::to_string(engine);
    (engine == 2 ? big : engine == 3 ? chip : engine == 4 ? clus : jobs).push_back(j);
  }
  if (log) std::fprintf(stderr, "[sbx-id]%s\n", line.c_str());
  qr_batched(jobs, s);
  cpqr_coop_batched(big, s);
  cpqr_smem_batched(chip, s);
  cpqr_cluster_batched(clus, s);
}

// ---------------------------------------------------------------- rendezvous
IdRendezvous::IdRendezvous(int participants) : active_(participants) {}

void IdRendezvous::flush_locked(cudaStream_t s) {
  std::vector<QrJob> merged;
  for (auto* v : pending_) merged.insert(merged.end(), v->begin(), v->end());
  launch_id_jobs(merged, 0, s);
  pending_.clear();
  waiting_ = 0;
  ++generation_;
  cv_.notify_all();
}

void IdRendezvous::submit(std::vector<QrJob>& jobs, cudaStream_t s) {
  std::unique_lock<std::mutex> lk(mu_);
  pending_.push_back(&jobs);
  ++waiting_;
  last_stream_ = s;
  if (waiting_ >= active_) {
    flush_locked(s);
    return;
  }
  const unsigned long long gen = generation_;
  cv_.wait(lk, [&] { return generation_ != gen; });
}

void IdRendezvous::leave() {
  std::lock_guard<std::mutex> lk(mu_);
  --active_;
  if (waiting_ > 0 && waiting_ >= active_) flush_locked(last_stream_);
}

IdRendezvousScope::IdRendezvousScope(IdRendezvous* rv) : rv_(rv), prev_(tl_rv) { tl_rv = rv; }
IdRendezvousScope::~IdRendezvousScope() { leave(); }
void IdRendezvousScope::leave() {
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
  if (!hperm.empty()) d_perm_.download(hperm.data(), hperm.size(), s);
  if (!hdiag.empty()) d_diag_.download(hdiag.data(), hdiag.size(), s);
  SBX_CUDA(cudaStreamSynchronize(s));
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
