// Microbenchmarks used to fix the FP64 roofline denominator on B200:
// DMMA (mma.sync m8n8k4 f64) vs DFMA throughput, cooperative grid-barrier
// latency, and L2/HBM streaming read bandwidth.
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; i++) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-9;
  double c[16];
#pragma unroll
  for (int i = 0; i < 16; i++) c[i] = i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) c[i] = fma(c[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) s += c[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void gridsync_loop(int iters, int* dummy) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; i++) g.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) dummy[0] = iters;
}

__global__ void read_bw(const double2* __restrict__ a, size_t n, double* out) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldcg(a + i);
    s += v.x + v.y;
  }
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0; cudaSetDevice(dev);
  cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  printf("device %s SMs %d clock %d kHz smemPerBlockOptin %zu L2 %d\n", p.name, p.multiProcessorCount, p.clockRate, p.sharedMemPerBlockOptin, p.l2CacheSize);
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int warps = 4; warps <= 16; warps *= 2) {
    int iters = 20000;
    dmma_loop<<<sms * 2, warps * 32>>>(out, 100);
    cudaEventRecord(e0);
    dmma_loop<<<sms * 2, warps * 32>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (sms * 2) * warps;
    printf("DMMA m8n8k4: %d warps/CTA x %d CTAs: %.2f TFLOP/s\n", warps, sms * 2, flops / ms / 1e9);
  }
  for (int warps = 4; warps <= 16; warps *= 2) {
    int iters = 20000;
    dfma_loop<<<sms * 2, warps * 32>>>(out, 100);
    cudaEventRecord(e0);
    dfma_loop<<<sms * 2, warps * 32>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * iters * 32.0 * warps * (sms * 2);
    printf("DFMA: %d warps/CTA x %d CTAs: %.2f TFLOP/s\n", warps, sms * 2, flops / ms / 1e9);
  }
  int* dummy; cudaMalloc(&dummy, 4);
  for (int ctas : {sms, 2 * sms}) {
    int iters = 10000;
    void* args[] = {&iters, &dummy};
    int it0 = 10; void* args0[] = {&it0, &dummy};
    cudaLaunchCooperativeKernel((void*)gridsync_loop, ctas, 256, args0, 0, 0);
    cudaEventRecord(e0);
    cudaError_t err = cudaLaunchCooperativeKernel((void*)gridsync_loop, ctas, 256, args, 0, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("grid.sync (%d CTAs): %.3f us each (%s)\n", ctas, ms * 1e3 / iters, cudaGetErrorString(err));
  }
  for (size_t mb : {16, 64, 2048}) {
    size_t bytes = mb << 20; size_t n = bytes / 16;
    double2* a; cudaMalloc(&a, bytes); cudaMemset(a, 0, bytes);
    read_bw<<<sms * 8, 512>>>(a, n, out);
    int reps = mb <= 64 ? 50 : 5;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; r++) read_bw<<<sms * 8, 512>>>(a, n, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("read bw %zu MB: %.1f GB/s\n", mb, (double)bytes * reps / ms / 1e6);
    cudaFree(a);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
