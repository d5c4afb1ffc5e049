// Pooled device / pinned-host allocation for libkotgpu (see common.cuh).
#include <algorithm>
#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace kot {

namespace {
std::mutex g_mu;
std::map<int, cudaStream_t> g_alloc_stream;              // per device, non-blocking
std::map<size_t, std::vector<void*>> g_pinned_free;     // size → cached pinned buffers

cudaStream_t alloc_stream_locked(int dev) {
  auto it = g_alloc_stream.find(dev);
  if (it != g_alloc_stream.end()) return it->second;
  cudaMemPool_t pool;
  KOT_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  unsigned long long keep = ~0ull;  // never trim the pool behind our back
  KOT_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  cudaStream_t s;
  KOT_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  g_alloc_stream[dev] = s;
  return s;
}
}  // namespace

void* dev_alloc(size_t bytes) {
  int dev = 0;
  KOT_CUDA(cudaGetDevice(&dev));
  cudaStream_t s;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    s = alloc_stream_locked(dev);
  }
  void* p = nullptr;
  KOT_CUDA(cudaMallocAsync(&p, bytes > 0 ? bytes : 8, s));
  KOT_CUDA(cudaStreamSynchronize(s));  // usable from every stream from here on
  return p;
}

void dev_free(void* p) {
  if (!p) return;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  cudaStream_t s;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    s = alloc_stream_locked(dev);
  }
  cudaFreeAsync(p, s);  // back to the pool; the caller's streams are idle
}

void* host_alloc_pinned(size_t bytes) {
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto& v = g_pinned_free[bytes];
    if (!v.empty()) {
      void* p = v.back();
      v.pop_back();
      return p;
    }
  }
  void* p = nullptr;
  KOT_CUDA(cudaMallocHost(&p, bytes > 0 ? bytes : 8));
  return p;
}

void host_free_pinned(void* p, size_t bytes) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_mu);
  g_pinned_free[bytes].push_back(p);
}

namespace {
std::map<std::pair<int, const void*>, int> g_smem_attr;
}

void ensure_smem_attr(const void* func, int bytes, bool nonportable_cluster) {
  int dev = 0;
  KOT_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_mu);
  int& have = g_smem_attr[{dev, func}];
  if (have >= bytes && have > 0) return;
  if (nonportable_cluster) KOT_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  if (bytes > 48 * 1024) KOT_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  have = std::max(bytes, 1);
}

}  // namespace kot
