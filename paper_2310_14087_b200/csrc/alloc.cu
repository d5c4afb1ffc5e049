// Pooled device / pinned-host allocation for libkotgpu (see common.cuh).
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace kot {

namespace {
std::mutex g_mu;
std::map<int, cudaStream_t> g_alloc_stream;              // per device, non-blocking
std::map<size_t, std::vector<void*>> g_pinned_free;     // size → cached pinned buffers

// The GEMM cores and the sytrd panel kernel prefer the maximum shared-memory carveout (KOT_CARVEOUT=0:
// driver defaults).  An SM takes a CTA only if its
// current L1/shared split leaves room: under per-kernel defaults an SM brought up for a 64 KB panel
// CTA could not take the CG GEMMs' CTAs beside it (measured with idle 64 KB CTAs on another stream:
// Newton chain 27.3 → 30.7 ms; with the max-shared preference 28.6).  Kernels without dynamic shared
// memory keep the default (max L1): a device-wide PreferShared cost the eigensolver its L1 (trial
// residual 27.5 → 28.6 ms), and so did the preference on every shared-memory kernel (tail, D&C…), so
// only the GEMMs and the panel kernel — the pair that must share SMs — carry it.
bool carveout_on() {
  static const bool on = [] {
    const char* e = std::getenv("KOT_CARVEOUT");
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}

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
// Debug canaries (KOT_CANARY=1): every device allocation gets kCanary guard bytes on both sides,
// filled with 0xAB and verified on free and by canary_check_all (out-of-bounds write detection
// without a sanitizer).
constexpr size_t kCanary = 64 * 1024;
struct Guarded {
  void* raw;
  size_t bytes;
  long seq;
};
std::map<void*, Guarded> g_guarded;
long g_seq = 0;
bool canary_on() {
  static const bool on = [] {
    const char* e = std::getenv("KOT_CANARY");
    return e && std::atoi(e) > 0;
  }();
  return on;
}
int check_one(void* user, const Guarded& g, const char* where) {
  std::vector<unsigned char> h(kCanary);
  int bad = 0;
  for (int side = 0; side < 2; ++side) {
    const char* src = side == 0 ? static_cast<const char*>(g.raw) : static_cast<const char*>(user) + g.bytes;
    if (cudaMemcpy(h.data(), src, kCanary, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    size_t first = kCanary, last = 0, cnt = 0;
    for (size_t i = 0; i < kCanary; ++i)
      if (h[i] != 0xAB) {
        first = std::min(first, i);
        last = i;
        ++cnt;
      }
    if (cnt) {
      std::fprintf(stderr, "[kot canary] %s: alloc #%ld (%zu B) %s guard: %zu bytes changed in [%zu, %zu]\n", where,
                   g.seq, g.bytes, side == 0 ? "LOW" : "HIGH", cnt, first, last);
      ++bad;
    }
  }
  return bad;
}
}  // namespace

int canary_check_all(const char* where) {
  if (!canary_on()) return 0;
  KOT_CUDA(cudaDeviceSynchronize());
  std::lock_guard<std::mutex> lk(g_mu);
  int bad = 0;
  for (auto& [u, g] : g_guarded) bad += check_one(u, g, where);
  return bad;
}

void* dev_alloc(size_t bytes) {
  int dev = 0;
  KOT_CUDA(cudaGetDevice(&dev));
  cudaStream_t s;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    s = alloc_stream_locked(dev);
  }
  void* p = nullptr;
  if (canary_on()) {
    const size_t b = ((bytes > 0 ? bytes : 8) + 255) / 256 * 256;
    KOT_CUDA(cudaMallocAsync(&p, b + 2 * kCanary, s));
    KOT_CUDA(cudaMemsetAsync(p, 0xAB, b + 2 * kCanary, s));
    KOT_CUDA(cudaStreamSynchronize(s));
    void* user = static_cast<char*>(p) + kCanary;
    std::lock_guard<std::mutex> lk(g_mu);
    g_guarded[user] = Guarded{p, b, g_seq++};
    return user;
  }
  KOT_CUDA(cudaMallocAsync(&p, bytes > 0 ? bytes : 8, s));
  // diagnostics: KOT_POISON fills fresh allocations (1: NaN bytes, 2: 0x55 bytes), restricted to
  // allocation numbers [lo, hi) by KOT_POISON_RANGE=lo:hi; KOT_ALLOC_LOG=1 lists the allocations
  static const int poison = [] {
    const char* e = std::getenv("KOT_POISON");
    return e ? std::atoi(e) : 0;
  }();
  static const std::pair<long, long> prange = [] {
    const char* e = std::getenv("KOT_POISON_RANGE");
    long lo = 0, hi = 1L << 60;
    if (e) std::sscanf(e, "%ld:%ld", &lo, &hi);
    return std::make_pair(lo, hi);
  }();
  static const bool alog = std::getenv("KOT_ALLOC_LOG") != nullptr;
  static std::atomic<long> aseq{0};
  const long seq = aseq++;
  if (alog) std::fprintf(stderr, "[kot alloc] #%ld %zu B\n", seq, bytes);
  if (poison && seq >= prange.first && seq < prange.second)
    KOT_CUDA(cudaMemsetAsync(p, poison == 1 ? 0xFF : 0x55, bytes > 0 ? bytes : 8, s));
  KOT_CUDA(cudaStreamSynchronize(s));  // usable from every stream from here on
  return p;
}

// Grows the device memory pool once (process set-up of a long-running service): `bytes` are allocated
// from the library's pool and given back to it; the pool never trims (release threshold = max), so later
// allocations find mapped memory.  Without it the first solve of a process pays the driver's mapping of
// the pool — 4 to 300 ms for the ≈ 3.5 GB of an ℓ = 2000 problem, depending on what ran on the GPU before.
void dev_reserve(size_t bytes) {
  int dev = 0;
  KOT_CUDA(cudaGetDevice(&dev));
  cudaStream_t s;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    s = alloc_stream_locked(dev);
  }
  void* p = nullptr;
  KOT_CUDA(cudaMallocAsync(&p, bytes > 0 ? bytes : 8, s));
  KOT_CUDA(cudaFreeAsync(p, s));
  KOT_CUDA(cudaStreamSynchronize(s));
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
  if (canary_on()) {
    Guarded g{};
    {
      std::lock_guard<std::mutex> lk(g_mu);
      auto it = g_guarded.find(p);
      if (it == g_guarded.end()) return;
      g = it->second;
      g_guarded.erase(it);
    }
    cudaDeviceSynchronize();
    check_one(p, g, "free");
    cudaFreeAsync(g.raw, s);
    return;
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

bool carveout_preferred() { return carveout_on(); }

void prefer_max_shared(const void* func) {
  if (!carveout_on()) return;
  std::lock_guard<std::mutex> lk(g_mu);
  static std::map<const void*, bool> done;
  if (done[func]) return;
  done[func] = true;
  KOT_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared));
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
