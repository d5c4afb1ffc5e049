// Cluster barrier / DSMEM latency microbenchmark (sizes 1..16, 256 threads per CTA).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void sync_loop(int iters, int mode, double* out) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double buf[64];
  if (threadIdx.x < 64) buf[threadIdx.x] = threadIdx.x;
  cl.sync();
  double acc = 0.0;
  const int CS = cl.num_blocks(), rank = cl.block_rank();
  for (int i = 0; i < iters; ++i) {
    if (mode == 1) {  // one remote DSMEM load per thread before each barrier
      const double* r = cl.map_shared_rank(buf, (rank + 1) % CS);
      acc += r[threadIdx.x & 63];
    } else if (mode == 2) {  // 16 remote loads per thread
      const double* r = cl.map_shared_rank(buf, (rank + 1) % CS);
#pragma unroll
      for (int k = 0; k < 16; ++k) acc += r[(threadIdx.x + k * 4) & 63];
    }
    if (mode == 3) {
      __syncthreads();
    } else {
      cl.sync();
    }
  }
  if (acc == 12345.0) out[0] = acc;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  cudaFuncSetAttribute(sync_loop, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 20000;
  for (int mode = 0; mode < 4; ++mode)
    for (int cs : {1, 2, 4, 8, 16}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs);
      cfg.blockDim = dim3(256);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, sync_loop, 10, mode, out);
      cudaEventRecord(a);
      cudaLaunchKernelEx(&cfg, sync_loop, iters, mode, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("mode %d cluster %2d: %.3f us per iteration (%s)\n", mode, cs, ms * 1e3 / iters,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
