// Library runtime: device selection, the library stream, launch counting,
// the caching device allocator and the optional phase timer.
#include <malloc.h>
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <map>
#include <mutex>
#include <thread>
#include <vector>

#include "common.hpp"

namespace sbx {

namespace {
std::atomic<std::int64_t> g_launches{0};
cudaStream_t g_stream = nullptr;
std::once_flag g_once;

// Size-class free lists, one set per stream.  A block is handed back to the
// pool of the stream current on the freeing thread, so the next allocation
// from that pool is stream-ordered after every use of the block: uses on
// other streams are joined (event wait) into the freeing stream before the
// owner releases it (see parallel_tasks).
std::mutex g_pool_mu;
std::map<cudaStream_t, std::map<size_t, std::vector<void*>>> g_pool;
thread_local cudaStream_t tl_stream = nullptr;

// worker streams for parallel_tasks (created on demand, reused), one free
// list per priority class (0 normal, 1 high)
std::mutex g_ws_mu;
std::vector<cudaStream_t> g_ws_free[2];

size_t size_class(size_t bytes) {
  if (bytes <= 4096) return 4096;
  size_t c = 4096;
  while (c < bytes) c <<= 1;
  if (c > (size_t(64) << 20)) {  // above 64 MB: 8 MB granularity
    const size_t g = size_t(8) << 20;
    return (bytes + g - 1) / g * g;
  }
  return c;
}
}  // namespace

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

namespace {
std::atomic<bool> g_ktimer{false};
std::mutex g_ktimer_mu;
std::map<std::string, std::vector<std::pair<cudaEvent_t, cudaEvent_t>>> g_ktimes;
}  // namespace

void ktimer_enable(bool on) { g_ktimer.store(on); }
bool ktimer_on() { return g_ktimer.load(std::memory_order_relaxed); }

void ktimer_record(const char* name, cudaEvent_t begin, cudaEvent_t end) {
  std::lock_guard<std::mutex> lk(g_ktimer_mu);
  g_ktimes[name].push_back({begin, end});
}

double ktimer_total(const char* name, bool reset, std::int64_t* count) {
  std::lock_guard<std::mutex> lk(g_ktimer_mu);
  auto& v = g_ktimes[name];
  double ms = 0.0;
  for (auto& e : v) {
    SBX_CUDA(cudaEventSynchronize(e.second));
    float t = 0.0f;
    SBX_CUDA(cudaEventElapsedTime(&t, e.first, e.second));
    ms += t;
  }
  if (count) *count = std::int64_t(v.size());
  if (reset) {
    for (auto& e : v) {
      cudaEventDestroy(e.first);
      cudaEventDestroy(e.second);
    }
    v.clear();
  }
  return ms;
}

namespace {
std::map<std::string, double> g_kflops;
}

void ktimer_add_flops(const char* name, double flops) {
  if (!ktimer_on()) return;
  std::lock_guard<std::mutex> lk(g_ktimer_mu);
  g_kflops[name] += flops;
}

double ktimer_flops(const char* name, bool reset) {
  std::lock_guard<std::mutex> lk(g_ktimer_mu);
  const double f = g_kflops[name];
  if (reset) g_kflops[name] = 0.0;
  return f;
}

KernelTimer::KernelTimer(const char* name, cudaStream_t s) : name_(name), s_(s) {
  if (!ktimer_on()) return;
  SBX_CUDA(cudaEventCreate(&b_));
  SBX_CUDA(cudaEventRecord(b_, s_));
}

KernelTimer::~KernelTimer() {
  if (!b_) return;
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) != cudaSuccess || cudaEventRecord(e, s_) != cudaSuccess) return;
  ktimer_record(name_, b_, e);
}

std::int64_t launches(bool reset) {
  return reset ? g_launches.exchange(0) : g_launches.load();
}

namespace {
// The per-step host path builds multi-megabyte index and node vectors; with
// glibc's defaults every one of them is a fresh mmap (page faults on first
// touch, munmap on free: ~0.6 ms of a 0.75 ms refine).  Keep blocks up to
// 32 MB on the heap and do not trim it between steps.  SBX_NO_MALLOPT=1
// leaves the host process's allocator alone.
void tune_host_allocator() {
#if defined(__GLIBC__)
  if (std::getenv("SBX_NO_MALLOPT")) return;
  mallopt(M_MMAP_THRESHOLD, 32 << 20);
  mallopt(M_TRIM_THRESHOLD, 512 << 20);
  mallopt(M_TOP_PAD, 64 << 20);
#endif
}
}  // namespace

cudaStream_t lib_stream() {
  std::call_once(g_once, [] {
    tune_host_allocator();
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
      throw Error(6, "no CUDA device visible: the sbx library has no CPU fallback");
    SBX_CUDA(cudaStreamCreateWithFlags(&g_stream, cudaStreamNonBlocking));
  });
  return g_stream;
}

cudaStream_t cur_stream() { return tl_stream ? tl_stream : lib_stream(); }

bool& no_coop_flag() {
  thread_local bool f = false;
  return f;
}

cudaStream_t set_cur_stream(cudaStream_t s) {
  const cudaStream_t prev = tl_stream;
  tl_stream = s;
  return prev;
}

void* dev_alloc(size_t bytes) {
  const size_t c = size_class(bytes);
  const cudaStream_t st = cur_stream();
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    auto& pool = g_pool[st];
    auto it = pool.find(c);
    if (it != pool.end() && !it->second.empty()) {
      void* p = it->second.back();
      it->second.pop_back();
      return p;
    }
    // Another stream's pool has a free block of this class (blocks migrate
    // between pools when a host thread frees on a different stream than it
    // allocated on): take it, ordered after every use queued on that stream
    // so far (an event recorded there now).  A cudaMalloc in steady state
    // can stall the host for tens of milliseconds.
    for (auto& sp : g_pool) {
      if (sp.first == st) continue;
      auto jt = sp.second.find(c);
      if (jt == sp.second.end() || jt->second.empty()) continue;
      void* p = jt->second.back();
      jt->second.pop_back();
      static cudaEvent_t ev = [] {
        cudaEvent_t e = nullptr;
        SBX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        return e;
      }();
      SBX_CUDA(cudaEventRecord(ev, sp.first));
      SBX_CUDA(cudaStreamWaitEvent(st, ev, 0));
      return p;
    }
  }
  void* p = nullptr;
  static const bool alloc_log = std::getenv("SBX_ALLOC_LOG") != nullptr;  // diagnostics
  const auto ta = alloc_log ? std::chrono::steady_clock::now() : std::chrono::steady_clock::time_point{};
  cudaError_t e = cudaMalloc(&p, c);
  if (alloc_log)
    std::fprintf(stderr, "[sbx-alloc] %zu bytes %.3f ms\n", c,
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ta).count());
  if (e != cudaSuccess) {  // release cached blocks and retry once
    (void)cudaGetLastError();
    std::lock_guard<std::mutex> lk(g_pool_mu);
    SBX_CUDA(cudaDeviceSynchronize());
    for (auto& sp : g_pool)
      for (auto& kv : sp.second)
        for (void* q : kv.second) cudaFree(q);
    g_pool.clear();
    SBX_CUDA(cudaMalloc(&p, c));
  }
  return p;
}

void dev_free(void* p, size_t bytes) {
  if (!p) return;
  const cudaStream_t st = cur_stream();
  std::lock_guard<std::mutex> lk(g_pool_mu);
  g_pool[st][size_class(bytes)].push_back(p);
}

namespace {
struct SidePool {
  std::mutex mu;
  struct Entry {
    cudaStream_t s;
    cudaEvent_t fork, join;
  };
  std::vector<Entry> free[2];
};
SidePool& side_pool() {
  static SidePool* p = new SidePool;  // never destroyed (streams outlive static destruction order)
  return *p;
}
}  // namespace

SideStream::SideStream(cudaStream_t parent, bool high_priority) : high_(high_priority) {
  auto& pool = side_pool();
  {
    std::lock_guard<std::mutex> lk(pool.mu);
    auto& fl = pool.free[high_ ? 1 : 0];
    if (!fl.empty()) {
      s_ = fl.back().s;
      fork_ = fl.back().fork;
      join_ = fl.back().join;
      fl.pop_back();
    }
  }
  if (!s_) {
    int least = 0, greatest = 0;
    SBX_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    SBX_CUDA(cudaStreamCreateWithPriority(&s_, cudaStreamNonBlocking, high_ ? greatest : least));
    SBX_CUDA(cudaEventCreateWithFlags(&fork_, cudaEventDisableTiming));
    SBX_CUDA(cudaEventCreateWithFlags(&join_, cudaEventDisableTiming));
  }
  SBX_CUDA(cudaEventRecord(fork_, parent));
  SBX_CUDA(cudaStreamWaitEvent(s_, fork_, 0));
}

void SideStream::join(cudaStream_t parent) {
  SBX_CUDA(cudaEventRecord(join_, s_));
  SBX_CUDA(cudaStreamWaitEvent(parent, join_, 0));
}

SideStream::~SideStream() {
  if (!s_) return;
  auto& pool = side_pool();
  std::lock_guard<std::mutex> lk(pool.mu);
  pool.free[high_ ? 1 : 0].push_back({s_, fork_, join_});
}

namespace {
struct PinnedPool {
  std::mutex mu;
  std::vector<std::pair<void*, size_t>> free;
};
PinnedPool& pinned_pool() {
  static PinnedPool* p = new PinnedPool;  // never destroyed
  return *p;
}
}  // namespace

PinnedLease::PinnedLease(size_t bytes) {
  bytes = std::max<size_t>(bytes, 4096);
  auto& pool = pinned_pool();
  {
    std::lock_guard<std::mutex> lk(pool.mu);
    for (size_t i = 0; i < pool.free.size(); ++i)
      if (pool.free[i].second >= bytes) {
        p_ = pool.free[i].first;
        bytes_ = pool.free[i].second;
        pool.free.erase(pool.free.begin() + long(i));
        return;
      }
  }
  size_t sz = 4096;
  while (sz < bytes) sz <<= 1;
  SBX_CUDA(cudaMallocHost(&p_, sz));
  bytes_ = sz;
}

PinnedLease::~PinnedLease() {
  if (!p_) return;
  auto& pool = pinned_pool();
  std::lock_guard<std::mutex> lk(pool.mu);
  pool.free.push_back({p_, bytes_});
}

void parallel_tasks(const std::vector<std::function<void(cudaStream_t)>>& tasks, cudaStream_t main,
                    const std::vector<int>& high) {
  const size_t nt = tasks.size();
  if (nt == 0) return;
  static const bool serial = std::getenv("SBX_SERIAL") != nullptr;  // diagnostics
  if (serial) {
    for (const auto& t : tasks) t(main);
    return;
  }
  std::vector<cudaStream_t> ws(nt);
  {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    for (size_t i = 0; i < nt; ++i) {
      const int pc = (i < high.size() && high[i]) ? 1 : 0;
      auto& fl = g_ws_free[pc];
      if (fl.empty()) {
        int least = 0, greatest = 0;
        SBX_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        cudaStream_t w = nullptr;
        SBX_CUDA(cudaStreamCreateWithPriority(&w, cudaStreamNonBlocking, pc ? greatest : least));
        fl.push_back(w);
      }
      ws[i] = fl.back();
      fl.pop_back();
    }
  }
  cudaEvent_t fork = nullptr;
  SBX_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
  SBX_CUDA(cudaEventRecord(fork, main));
  int dev = 0;
  SBX_CUDA(cudaGetDevice(&dev));
  std::vector<std::exception_ptr> err(nt);
  std::vector<std::thread> th;
  th.reserve(nt);
  for (size_t i = 0; i < nt; ++i) {
    SBX_CUDA(cudaStreamWaitEvent(ws[i], fork, 0));
    th.emplace_back([&, i] {
      tl_stream = ws[i];
      try {
        SBX_CUDA(cudaSetDevice(dev));
        phase_mark(nullptr, ws[i]);
        tasks[i](ws[i]);
      } catch (...) {
        err[i] = std::current_exception();
      }
    });
  }
  for (auto& t : th) t.join();
  for (size_t i = 0; i < nt; ++i) {
    cudaEvent_t done = nullptr;
    SBX_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    SBX_CUDA(cudaEventRecord(done, ws[i]));
    SBX_CUDA(cudaStreamWaitEvent(main, done, 0));
    SBX_CUDA(cudaEventDestroy(done));
  }
  SBX_CUDA(cudaEventDestroy(fork));
  {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    for (size_t i = 0; i < nt; ++i) g_ws_free[(i < high.size() && high[i]) ? 1 : 0].push_back(ws[i]);
  }
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
}

void phase_mark(const char* what, cudaStream_t s) {
  static const bool on = std::getenv("SBX_TIMING") != nullptr;
  if (!on) return;
  thread_local auto last = std::chrono::steady_clock::now();
  if (!what) {  // reset (start of a worker task)
    last = std::chrono::steady_clock::now();
    return;
  }
  cudaStreamSynchronize(s);
  const auto now = std::chrono::steady_clock::now();
  std::fprintf(stderr, "[sbx] %-28s %9.3f ms%s\n", what,
               std::chrono::duration<double, std::milli>(now - last).count(), tl_stream ? " (worker)" : "");
  last = now;
}

}  // namespace sbx
