// Size-bucketed caching device allocator behind DevBuf (see internal.h).
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "internal.h"

namespace gpfvm {

namespace {
struct Pool {
  std::mutex mu;
  std::map<std::pair<int, size_t>, std::vector<void*>> free_blocks;  // (device, rounded bytes)
};
Pool& pool() {
  static Pool* p = new Pool();  // intentionally leaked: no teardown-order issues at exit
  return *p;
}
size_t round_bytes(size_t b) {
  if (b <= (1u << 21)) {  // < 2 MiB: next power of two (>= 256 B)
    size_t r = 256;
    while (r < b) r <<= 1;
    return r;
  }
  const size_t g = 1u << 21;  // 2 MiB granules
  return (b + g - 1) / g * g;
}
}  // namespace

// GPFVM_NO_POOL (debugging with compute-sanitizer memcheck): exact-size
// cudaMalloc / synchronous cudaFree, so an out-of-bounds access leaves its
// allocation instead of landing in a neighbouring pooled block's padding
static bool no_pool() {
  static const bool v = getenv("GPFVM_NO_POOL") != nullptr;
  return v;
}

void* pool_alloc(size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (no_pool()) {
    void* q = nullptr;
    GPFVM_CUDA(cudaMalloc(&q, bytes ? bytes : 8));
    return q;
  }
  const size_t rb = round_bytes(bytes);
  {
    std::lock_guard<std::mutex> lk(pool().mu);
    auto it = pool().free_blocks.find({dev, rb});
    if (it != pool().free_blocks.end() && !it->second.empty()) {
      void* p = it->second.back();
      it->second.pop_back();
      return p;
    }
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, rb);
  if (e != cudaSuccess) {
    cudaGetLastError();
    // release every cached block of this device and retry once
    pool_trim();
    GPFVM_CUDA(cudaMalloc(&p, rb));
  }
  return p;
}

void pool_free(void* p, size_t bytes, int dev) {
  if (!p) return;
  if (no_pool()) {
    cudaDeviceSynchronize();
    cudaFree(p);
    return;
  }
  if (dev < 0) dev = current_device();
  std::lock_guard<std::mutex> lk(pool().mu);
  pool().free_blocks[{dev, round_bytes(bytes)}].push_back(p);
}

int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}

DevBuf& scratch(cudaStream_t s, int slot) {
  static thread_local std::map<std::tuple<int, cudaStream_t, int>, DevBuf> bufs;
  return bufs[std::make_tuple(current_device(), s, slot)];
}

void pool_trim() {
  int dev = 0;
  cudaGetDevice(&dev);
  std::vector<void*> victims;
  {
    std::lock_guard<std::mutex> lk(pool().mu);
    for (auto it = pool().free_blocks.begin(); it != pool().free_blocks.end(); ++it)
      if (it->first.first == dev) {
        victims.insert(victims.end(), it->second.begin(), it->second.end());
        it->second.clear();
      }
  }
  if (!victims.empty()) cudaDeviceSynchronize();
  for (void* v : victims) cudaFree(v);
}

}  // namespace gpfvm
