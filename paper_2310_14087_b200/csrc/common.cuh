// Shared helpers for libkotgpu (sm_100a, FP64).
#pragma once
#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

namespace kot {

// Status codes of the C ABI (include/kotgpu.h); map 1:1 onto the reference's
// exception classes.
enum Status : int {
  KOT_OK = 0,
  KOT_EINVAL = 1,        // ValueError
  KOT_EINDEFINITE = 2,   // IndefiniteKernelError (linalg.py:114)
  KOT_EEIG = 3,          // EigenSolveError (linalg.py:70)
  KOT_ENUMERICS = 4,     // SolverNumericsError (solver.py:28-33)
  KOT_ECG = 5,           // FloatingPointError in CG (linalg.py:146,156)
  KOT_ECUDA = 6,
  KOT_EASSERT = 7,       // AssertionError (psdcone.py:77)
  KOT_ECALLBACK = 8,     // the on_iteration observer raised (solver.py:170-181: propagates, ends the solve)
};

struct KotError : public std::runtime_error {
  int code;
  KotError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
// Thrown by an eigensolve whose caller cancelled it (speculative EG-pipeline work at the end of a
// solve); never escapes the library.
struct Cancelled {};

#define KOT_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) {                                                             \
      (void)cudaGetLastError(); /* clear non-sticky errors so later calls are clean */   \
      throw ::kot::KotError(::kot::KOT_ECUDA, std::string(#call) + ": " +              \
                                                  cudaGetErrorString(e_));               \
    }                                                                                    \
  } while (0)

// Every kernel launch of the library goes through KOT_LAUNCH_CHECK (counted:
// kot_launch_count() backs bench.py's "gpu_launches").
extern std::atomic<long long> g_kot_launches;
// launches by the calling thread (graph capture counts its own kernels with it)
inline long long& thread_launches() {
  static thread_local long long n = 0;
  return n;
}
#define KOT_LAUNCH_CHECK()                     \
  do {                                         \
    ::kot::g_kot_launches.fetch_add(1);        \
    ++::kot::thread_launches();                \
    KOT_CUDA(cudaGetLastError());              \
  } while (0)

inline void kot_require(bool ok, int code, const std::string& msg) {
  if (!ok) throw KotError(code, msg);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Deterministic block sum (fixed tree); every thread gets the result.
// `sh` must hold >= 32 doubles.  blockDim.x must be a multiple of 32.
__device__ __forceinline__ double block_sum(double v, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = (lane < nw) ? sh[lane] : 0.0;
  t = warp_sum(t);
  return t;
}

inline int ceil_div(long a, long b) { return (int)((a + b - 1) / b); }

// Device / pinned-host allocations of the library (alloc.cu).  Device memory
// comes from the device's stream-ordered pool with a high release threshold and
// pinned host buffers from a size-keyed free list, so creating a problem or an
// execution context after the first one costs no cudaMalloc/cudaFree (and no
// implicit device synchronisation) — this is what keeps solve()'s end-to-end
// time close to the device time.  Callers free only after their streams are idle.
void* dev_alloc(size_t bytes);
int canary_check_all(const char* where);  // KOT_CANARY=1: guard-byte check of every live allocation
void dev_free(void* p);
void dev_reserve(size_t bytes);  // grow the pool once (kot_reserve)
void* host_alloc_pinned(size_t bytes);
void host_free_pinned(void* p, size_t bytes);

// Raise `func`'s dynamic shared-memory limit to at least `bytes` on the CURRENT device (function
// attributes are per device), optionally allowing non-portable cluster sizes; cached per
// (device, kernel), thread-safe.
void ensure_smem_attr(const void* func, int bytes, bool nonportable_cluster = false);
// the kernel prefers the maximum shared-memory carveout (GEMM cores, sytrd panel; see alloc.cu)
void prefer_max_shared(const void* func);
bool carveout_preferred();

constexpr int kNumSMs = 148;

}  // namespace kot
