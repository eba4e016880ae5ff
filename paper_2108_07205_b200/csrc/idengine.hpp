// Batched interpolative decompositions on the device (reference
// idlib.cpp:27-99).  Each problem is a row ID of W given as W^T (M x n,
// column-major, device resident): CPQR of W^T (dense.cu qr_kernel), rank by
// the reference's rules, then P = [I; R11^{-1} R12] scattered by the pivots.
#pragma once

#include <condition_variable>
#include <exception>
#include <mutex>
#include <vector>

#include "common.hpp"
#include "dense.hpp"

namespace sbx {

struct IdProblem {
  double* wt;  // W^T, factored in place
  int M, n, lda;
};

class IdBatch {
 public:
  // CPQR of every problem; stop_eps truncates at |r_jj| <= stop_eps*|r_00|
  // (1e-15 keeps every row the forced-rank rule can ask for).
  void factor(const std::vector<IdProblem>& probs, double stop_eps, cudaStream_t s);
  // engine override for tests: 0 auto, 1 one CTA per problem, 2 cooperative
  // (slabs in L2), 3 cooperative on chip (slabs in shared memory), 4 one
  // thread-block cluster per problem, 5 register-resident cluster
  int force_engine = 0;
  size_t size() const { return probs_.size(); }
  const IdProblem& problem(size_t p) const { return probs_[p]; }
  // idlib.cpp:47-51: #{ |r_kk| > eps |r_00| }
  i64 eps_rank(size_t p, double eps) const;
  // idlib.cpp:38-45: min(k, dmax) cut at 1e-15 |r_00|
  i64 forced_rank(size_t p, i64 k) const;
  const std::vector<int>& perm(size_t p) const { return perm_[p]; }
  const std::vector<double>& diag(size_t p) const { return diag_[p]; }
  // Writes P_p (n_p x k_p, column-major, ldp) for every problem with k_p > 0.
  void interp(const std::vector<i64>& ks, const std::vector<double*>& P,
              const std::vector<int>& ldp, cudaStream_t s);

  static constexpr i64 kCoopEntries = i64(1) << 18;  // 2 MB of W^T

 private:
  std::vector<IdProblem> probs_;
  std::vector<std::vector<double>> diag_;
  std::vector<std::vector<int>> perm_;
  std::vector<i64> perm_off_;
  DevBuf<int> d_perm_;
  DevBuf<double> d_diag_;
  DevBuf<int> d_steps_;
  DevBuf<double> d_T_;
};

// Engine routing + launches of one batch of CPQR jobs (force_engine 0: auto).
void launch_id_jobs(const std::vector<QrJob>& jobs, int force_engine, cudaStream_t s);

// Joint CPQR launches across independent algorithms running in separate host
// threads on ONE stream: every IdBatch::factor of a participating thread
// waits until each still-active participant has submitted its batch, then a
// single launch factors all of them (the update's row-ID hierarchies and the
// A_pp HBS build advance level by level together instead of one after the
// other).  A participant that has no more factorisations must leave().
class IdRendezvous {
 public:
  explicit IdRendezvous(int participants);
  // Throws the launch's error in every participant of the failed round.
  void submit(std::vector<QrJob>& jobs, cudaStream_t s);
  // Never throws (called during unwinding): a failed flush is handed to the
  // waiting participants instead.
  void leave() noexcept;
  // A participant that was not counted at construction joins (its rounds are
  // joint from its first submit on; the others never waited for it before).
  void enter();

 private:
  // Starts a new round BEFORE launching (pending jobs moved out, generation
  // bumped, waiters released), so a throwing launch never leaves a
  // participant blocked or a dangling pending entry behind.
  void flush_locked(std::unique_lock<std::mutex>& lk, cudaStream_t s);
  std::mutex mu_;
  std::condition_variable cv_;
  int active_ = 0, waiting_ = 0;
  unsigned long long generation_ = 0;
  std::vector<std::vector<QrJob>*> pending_;
  cudaStream_t last_stream_ = nullptr;
  // error of round `err_gen_` (its generation after the bump), if its launch threw
  std::exception_ptr err_;
  unsigned long long err_gen_ = 0;
};

// Installs a rendezvous for the calling thread's IdBatch::factor calls;
// leaves it (at the latest) on destruction.
class IdRendezvousScope {
 public:
  // enter: the thread was not counted in the rendezvous' participants yet
  explicit IdRendezvousScope(IdRendezvous* rv, bool enter = false);
  ~IdRendezvousScope();
  void leave() noexcept;
  IdRendezvousScope(const IdRendezvousScope&) = delete;
  IdRendezvousScope& operator=(const IdRendezvousScope&) = delete;

 private:
  IdRendezvous* rv_;
  IdRendezvous* prev_;
};

// Leaves the calling thread's rendezvous, if any (a producer whose remaining
// work has no factorisations).
void id_rendezvous_leave();

}  // namespace sbx
