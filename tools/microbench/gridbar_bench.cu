// Grid barrier variants at 148 CTAs × 256 threads: cooperative grid.sync vs a cluster-hierarchical
// barrier (cluster.sync + one atomic per cluster leader + generation flag), in a cooperative+cluster launch.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ unsigned int g_count;
__device__ unsigned int g_gen;

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void bar_grid(int iters, double* out) {
  cg::grid_group grid = cg::this_grid();
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    acc += threadIdx.x;
    grid.sync();
  }
  if (acc == -1) out[0] = acc;
}

__global__ void bar_cluster(int iters, int nclusters, double* out) {
  cg::cluster_group cl = cg::this_cluster();
  double acc = 0;
  const bool leader = cl.block_rank() == 0 && threadIdx.x == 0;
  for (int i = 0; i < iters; ++i) {
    acc += threadIdx.x;
    cl.sync();
    if (leader) {
      const unsigned gen = ld_acquire(&g_gen);
      __threadfence();
      if (atomicAdd(&g_count, 1u) == (unsigned)nclusters - 1) {
        g_count = 0;
        st_release(&g_gen, gen + 1);
      } else {
        while (ld_acquire(&g_gen) == gen) {
        }
      }
    }
    cl.sync();
  }
  if (acc == -1) out[0] = acc;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 20000;
  for (int G : {148, 128, 74, 37}) {
    void* args[] = {(void*)&iters, (void*)&out};
    int it0 = 10;
    void* args0[] = {(void*)&it0, (void*)&out};
    cudaLaunchCooperativeKernel((void*)bar_grid, G, 256, args0, 0, 0);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)bar_grid, G, 256, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("grid.sync   G=%3d: %.3f us  (%s)\n", G, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
  }
  for (int cs : {2, 4}) {
    const int G = (cs == 2) ? 148 : 144;
    const int ncl = G / cs;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(256);
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    cudaLaunchKernelEx(&cfg, bar_cluster, 10, ncl, out);
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, bar_cluster, iters, ncl, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("cluster bar cs=%d G=%3d: %.3f us  (%s)\n", cs, G, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
