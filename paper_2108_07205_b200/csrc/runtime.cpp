// Library runtime: device selection, the library stream, launch counting.
#include <atomic>
#include <mutex>

#include "common.hpp"

namespace sbx {

namespace {
std::atomic<std::int64_t> g_launches{0};
cudaStream_t g_stream = nullptr;
std::once_flag g_once;
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

}  // namespace sbx
