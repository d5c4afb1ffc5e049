// Background "panel-like" load for interference probes: G CTAs that hold their SM slots for `usec`
// microseconds (spinning on %globaltimer with __nanosleep), launched either as a cooperative grid or
// as a plain grid, on a private low-priority stream.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC spin.cu -o libspin.so
#include <cuda_runtime.h>

__global__ void spin_kernel(long long ns) {
  extern __shared__ double sm[];
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if ((long long)(t - t0) >= ns) break;
    __nanosleep(500);
  }
  if (threadIdx.x == 0 && ns < 0) sm[0] = 1.0;
}

static cudaStream_t g_st = nullptr;

extern "C" int spin_launch(int ctas, int threads, int usec, int coop, int smem_kb) {
  if (!g_st) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStreamCreateWithPriority(&g_st, cudaStreamNonBlocking, lo);
  }
  const size_t smem = (size_t)smem_kb * 1024;
  if (smem > 48 * 1024) cudaFuncSetAttribute(spin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  long long ns = (long long)usec * 1000;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = g_st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = coop;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return (int)cudaLaunchKernelEx(&cfg, spin_kernel, ns);
}

extern "C" int spin_sync() { return (int)cudaStreamSynchronize(g_st); }
