// Library runtime: device selection, the library stream, launch counting,
// the caching device allocator and the optional phase timer.
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <vector>

#include "common.hpp"

namespace sbx {

namespace {
std::atomic<std::int64_t> g_launches{0};
cudaStream_t g_stream = nullptr;
std::once_flag g_once;

// Size-class free lists.  Blocks are only ever handed back to the same
// process-wide pool; reuse is ordered because every library temporary lives
// on the library stream (or is synchronised before release).
std::mutex g_pool_mu;
std::map<size_t, std::vector<void*>> g_pool;

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

std::int64_t launches(bool reset) {
  return reset ? g_launches.exchange(0) : g_launches.load();
}

cudaStream_t lib_stream() {
  std::call_once(g_once, [] {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
      throw Error(6, "no CUDA device visible: the sbx library has no CPU fallback");
    SBX_CUDA(cudaStreamCreateWithFlags(&g_stream, cudaStreamNonBlocking));
  });
  return g_stream;
}

void* dev_alloc(size_t bytes) {
  const size_t c = size_class(bytes);
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    auto it = g_pool.find(c);
    if (it != g_pool.end() && !it->second.empty()) {
      void* p = it->second.back();
      it->second.pop_back();
      return p;
    }
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, c);
  if (e != cudaSuccess) {  // release cached blocks and retry once
    (void)cudaGetLastError();
    std::lock_guard<std::mutex> lk(g_pool_mu);
    SBX_CUDA(cudaDeviceSynchronize());
    for (auto& kv : g_pool)
      for (void* q : kv.second) cudaFree(q);
    g_pool.clear();
    SBX_CUDA(cudaMalloc(&p, c));
  }
  return p;
}

void dev_free(void* p, size_t bytes) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  g_pool[size_class(bytes)].push_back(p);
}

void phase_mark(const char* what, cudaStream_t s) {
  static const bool on = std::getenv("SBX_TIMING") != nullptr;
  if (!on) return;
  static auto last = std::chrono::steady_clock::now();
  cudaStreamSynchronize(s);
  const auto now = std::chrono::steady_clock::now();
  std::fprintf(stderr, "[sbx] %-28s %9.3f ms\n", what,
               std::chrono::duration<double, std::milli>(now - last).count());
  last = now;
}

}  // namespace sbx
