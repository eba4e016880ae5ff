// Shared host-side plumbing for the sbx library: errors, device buffers,
// the library stream and launch accounting.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

namespace sbx {

using i64 = std::int64_t;
constexpr double kPi = 3.141592653589793238462643383279502884;

// Error carrying an sbx.h status code.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void require(bool c, const std::string& m) {
  if (!c) throw Error(1, m);
}

#define SBX_CUDA(x)                                                                   \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess)                                                            \
      throw ::sbx::Error(6, std::string("CUDA error: ") + cudaGetErrorString(e_) +    \
                                " (" #x ") at " + __FILE__ + ":" + std::to_string(__LINE__)); \
  } while (0)

#define SBX_LAUNCHED()                       \
  do {                                       \
    SBX_CUDA(cudaGetLastError());            \
    ::sbx::count_launch();                   \
  } while (0)

void count_launch();
std::int64_t launches(bool reset);

// Optional CUDA-event timing of named kernels (bench evidence: the
// roofline's per-launch duration on the stream the kernel runs on).
void ktimer_enable(bool on);
bool ktimer_on();
void ktimer_record(const char* name, cudaEvent_t begin, cudaEvent_t end);
// Total milliseconds and launch count of `name` since the last reset
// (synchronises on the recorded events).
double ktimer_total(const char* name, bool reset, std::int64_t* count);
// Algorithmic flops attributed to `name` while timing is on (reset with
// ktimer_flops(name, true)).
void ktimer_add_flops(const char* name, double flops);
double ktimer_flops(const char* name, bool reset);
class KernelTimer {
 public:
  KernelTimer(const char* name, cudaStream_t s);
  ~KernelTimer();
  KernelTimer(const KernelTimer&) = delete;
  KernelTimer& operator=(const KernelTimer&) = delete;

 private:
  const char* name_;
  cudaStream_t s_;
  cudaEvent_t b_ = nullptr;
};
cudaStream_t lib_stream();

// Stream-ordered caching device allocator (the per-step path allocates many
// short-lived blocks; cudaMalloc/cudaFree would serialise the device).
// Pools are per stream: the stream current on the calling thread (a
// parallel_tasks worker stream, else the library stream).
void* dev_alloc(size_t bytes);
void dev_free(void* p, size_t bytes);
cudaStream_t cur_stream();
// Makes `s` the calling thread's current stream (allocation pool and plan
// uploads follow it) for the scope's lifetime: C-ABI calls that take a
// caller stream run entirely on it.
cudaStream_t set_cur_stream(cudaStream_t s);
class StreamScope {
 public:
  explicit StreamScope(cudaStream_t s) : prev_(set_cur_stream(s)) {}
  ~StreamScope() { set_cur_stream(prev_); }
  StreamScope(const StreamScope&) = delete;
  StreamScope& operator=(const StreamScope&) = delete;

 private:
  cudaStream_t prev_;
};

// A stream forked from `parent` (its work starts after the parent's queued
// work) for launches that should run beside the parent's next ones; join()
// makes the parent wait for it.  Streams and their fork/join events come
// from a process-wide pool: the per-step host threads are short-lived, so
// thread-local streams would be created (a driver call that can stall for
// tens of milliseconds under contention) and leaked every step.
class SideStream {
 public:
  SideStream(cudaStream_t parent, bool high_priority = false);
  ~SideStream();
  SideStream(const SideStream&) = delete;
  SideStream& operator=(const SideStream&) = delete;
  cudaStream_t get() const { return s_; }
  void join(cudaStream_t parent);

 private:
  cudaStream_t s_ = nullptr;
  cudaEvent_t fork_ = nullptr, join_ = nullptr;
  bool high_ = false;
};

// A pinned host buffer of at least `bytes` from a process-wide pool (returned
// on destruction): small device-to-host reads the host waits for anyway go
// through it as one async copy + sync instead of a pageable staged copy.
class PinnedLease {
 public:
  explicit PinnedLease(size_t bytes);
  ~PinnedLease();
  PinnedLease(const PinnedLease&) = delete;
  PinnedLease& operator=(const PinnedLease&) = delete;
  void* get() const { return p_; }

 private:
  void* p_ = nullptr;
  size_t bytes_ = 0;
};

// Thread-local switch: while set, the ID engines avoid cooperative launches
// (grid-wide co-residency), which other streams' kernels can starve.
bool& no_coop_flag();
class NoCoopScope {
 public:
  NoCoopScope() : prev_(no_coop_flag()) { no_coop_flag() = true; }
  ~NoCoopScope() { no_coop_flag() = prev_; }
  NoCoopScope(const NoCoopScope&) = delete;
  NoCoopScope& operator=(const NoCoopScope&) = delete;

 private:
  bool prev_;
};

// Runs independent host+device tasks concurrently: task i gets its own
// thread and worker stream (forked from `main`, joined back into it), so the
// latency-bound ID factorisations of independent blocks overlap on the GPU.
// Device buffers a task allocates must either be released inside the task
// or handed back to the caller, who releases them on `main` after the join.
// high[i] != 0 puts task i on a high-priority stream (its pending CTAs are
// dispatched before those of normal-priority tasks).
void parallel_tasks(const std::vector<std::function<void(cudaStream_t)>>& tasks, cudaStream_t main,
                    const std::vector<int>& high = {});

// Optional host-side phase timer (SBX_TIMING=1): syncs the stream and prints
// the elapsed time since the previous mark to stderr.
void phase_mark(const char* what, cudaStream_t s);

// Owning device buffer.
template <class T>
class DevBuf {
 public:
  DevBuf() = default;
  explicit DevBuf(size_t n) { resize(n); }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_) {
    o.p_ = nullptr;
    o.n_ = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p_ = o.p_;
      n_ = o.n_;
      o.p_ = nullptr;
      o.n_ = 0;
    }
    return *this;
  }
  void resize(size_t n) {
    if (n == n_) return;
    release();
    if (n) p_ = static_cast<T*>(dev_alloc(n * sizeof(T)));
    n_ = n;
  }
  // Grows (never shrinks) without preserving contents.
  void reserve(size_t n) {
    if (n > n_) resize(n);
  }
  void release() {
    if (p_) dev_free(p_, n_ * sizeof(T));
    p_ = nullptr;
    n_ = 0;
  }
  T* get() const { return p_; }
  size_t size() const { return n_; }
  void upload(const T* h, size_t n, cudaStream_t s) {
    reserve(n);
    if (n) SBX_CUDA(cudaMemcpyAsync(p_, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void upload(const std::vector<T>& h, cudaStream_t s) { upload(h.data(), h.size(), s); }
  void download(T* h, size_t n, cudaStream_t s) const {
    if (n) SBX_CUDA(cudaMemcpyAsync(h, p_, n * sizeof(T), cudaMemcpyDeviceToHost, s));
  }
  void zero(cudaStream_t s) {
    if (n_) SBX_CUDA(cudaMemsetAsync(p_, 0, n_ * sizeof(T), s));
  }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
};

// Per-stream scratch of a shared, immutable handle (the reference's
// "concurrent solves with distinct right-hand sides allowed", SPEC.md:362,
// 445): calls on one stream reuse one scratch set (stream order protects
// it), calls on distinct streams never share one.  Entries live as long as
// the handle, so returned references stay valid.
template <class T>
class PerStream {
 public:
  T& get(cudaStream_t s) {
    std::lock_guard<std::mutex> lk(mu_);
    for (auto& e : items_)
      if (e.first == s) return *e.second;
    items_.emplace_back(s, std::make_unique<T>());
    return *items_.back().second;
  }
  template <class F>
  void for_each(F f) {
    std::lock_guard<std::mutex> lk(mu_);
    for (auto& e : items_) f(*e.second);
  }

 private:
  std::mutex mu_;
  std::vector<std::pair<cudaStream_t, std::unique_ptr<T>>> items_;
};

// Completion marker of the last call a handle ran on one stream: recorded
// at the end of each call, waited on when the handle is destroyed (its
// device memory returns to a stream-ordered pool while work enqueued on a
// caller's stream may still read it).  The event is ours, so waiting on it
// is safe even after the caller destroyed that stream.
struct StreamMark {
  cudaEvent_t ev = nullptr;
  StreamMark() = default;
  StreamMark(const StreamMark&) = delete;
  StreamMark& operator=(const StreamMark&) = delete;
  ~StreamMark() {
    if (ev) cudaEventDestroy(ev);
  }
  void record(cudaStream_t s) {
    if (!ev) SBX_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    SBX_CUDA(cudaEventRecord(ev, s));
  }
  void wait() const {
    if (ev) (void)cudaEventSynchronize(ev);
  }
};

// Column-major host matrix (the reference's Eigen storage order; used for
// HBS1 I/O and small host-side bookkeeping only).
struct HMat {
  i64 r = 0, c = 0;
  std::vector<double> a;
  HMat() = default;
  HMat(i64 rows, i64 cols) : r(rows), c(cols), a(size_t(rows * cols), 0.0) {}
  i64 size() const { return r * c; }
};

}  // namespace sbx
