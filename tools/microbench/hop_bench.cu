// All-to-all hop through tagged 32-byte sectors (the sytrd mid kernel's exchange) and the block-level
// latencies around it: G CTAs × 512 threads, every CTA publishes S sectors (to R replicas) and polls all
// G·S sectors of its replica.  Variants of the load/store flavour; FP64 dependent-op latency; the cost
// of a 512-thread barrier and of a warp butterfly sum.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
namespace cg = cooperative_groups;

struct Sector { unsigned long long a, b, c, tag; };

template <int MODE>
__device__ __forceinline__ void put(Sector* s, unsigned long long v, unsigned long long tag) {
  if (MODE == 0)
    asm volatile("st.volatile.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(s), "l"(v), "l"(v), "l"(v), "l"(tag) : "memory");
  else
    asm volatile("st.relaxed.gpu.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(s), "l"(v), "l"(v), "l"(v), "l"(tag) : "memory");
}
template <int MODE>
__device__ __forceinline__ bool tryget(const Sector* s, unsigned long long tag, unsigned long long& v) {
  unsigned long long a, b, c, t;
  if (MODE == 0)
    asm volatile("ld.volatile.global.v4.b64 {%0, %1, %2, %3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(t) : "l"(s) : "memory");
  else
    asm volatile("ld.relaxed.gpu.global.v4.b64 {%0, %1, %2, %3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(t) : "l"(s) : "memory");
  v = a + b + c;
  return t == tag;
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) hop_kernel(Sector* buf, int S, int R, int iters, int work, long long* cyc, double* sink) {
  const int G = gridDim.x, g = blockIdx.x, tid = threadIdx.x;
  const int nsec = G * S;
  const int rep = g % R;
  __shared__ double sm[4096];
  for (int i = tid; i < 4096; i += 512) sm[i] = i;
  __syncthreads();
  unsigned long long acc = 0;
  double facc = 0.0;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const unsigned long long tag = it + 1;
    Sector* xb = buf + (long)(it & 1) * R * nsec;
    // optional compute between hops (smem traffic of `work` passes)
    for (int w = 0; w < work; ++w) facc += sm[(tid * 2 + w * 64 + it) & 4095];
    __syncthreads();
    if (tid < S * R) put<MODE>(xb + (long)(tid / S) * nsec + g * S + (tid % S), it + g, tag);
    const Sector* rb = xb + (long)rep * nsec;
    bool have[5];
#pragma unroll
    for (int u = 0; u < 5; ++u) have[u] = !(tid + u * 512 < nsec);
    while (true) {
      bool all = true;
#pragma unroll
      for (int u = 0; u < 5; ++u)
        if (!have[u]) {
          unsigned long long v;
          if (tryget<MODE>(rb + tid + u * 512, tag, v)) {
            have[u] = true;
            acc += v;
          } else
            all = false;
        }
      if (all) break;
    }
    __syncthreads();
  }
  const long long t1 = clock64();
  if (tid == 0) cyc[g] = t1 - t0;
  if (acc == 0x1234567 || facc == 1.2345) sink[0] = (double)acc;
}

__global__ void lat_kernel(long long* out, double* sink, int iters) {
  const int lane = threadIdx.x & 31;
  __shared__ double red[16];
  double x = threadIdx.x * 1e-3 + 1.0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = x + 1.0000001;  // dependent DADD
  long long t1 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, 1.0000001, 0.5);  // dependent DFMA
  long long t2 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    x *= 1e-2;
  }
  long long t3 = clock64();
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
  }
  long long t4 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (lane == 0) red[threadIdx.x >> 5] = x;
    __syncthreads();
    double s = 0;
#pragma unroll
    for (int w = 0; w < 16; ++w) s += red[w];
    x = s * 1e-2;
    __syncthreads();
  }
  long long t5 = clock64();
  for (int i = 0; i < iters; ++i) x = sqrt(x + 3.0);
  long long t6 = clock64();
  for (int i = 0; i < iters; ++i) x = 1.0 / (x + 3.0);
  long long t7 = clock64();
  for (int i = 0; i < iters; ++i) x = hypot(x, 3.0);
  long long t8 = clock64();
  if (threadIdx.x == 0) {
    out[0] = (t1 - t0) / iters; out[1] = (t2 - t1) / iters; out[2] = (t3 - t2) / iters; out[3] = (t4 - t3) / iters;
    out[4] = (t5 - t4) / iters; out[5] = (t6 - t5) / iters; out[6] = (t7 - t6) / iters; out[7] = (t8 - t7) / iters;
  }
  if (x == 1.2345) sink[0] = x;
}

template <int MODE>
static void run(Sector* buf, int G, int S, int R, int iters, int work, long long* cyc, double* sink, const char* name) {
  cudaMemset(buf, 0, sizeof(Sector) * 2 * 8 * 148 * 16);
  void* args[] = {&buf, &S, &R, &iters, &work, &cyc, &sink};
  cudaError_t e = cudaLaunchCooperativeKernel((void*)hop_kernel<MODE>, dim3(G), dim3(512), args, 0, 0);
  if (e != cudaSuccess) { printf("launch: %s\n", cudaGetErrorString(e)); return; }
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("sync: %s\n", cudaGetErrorString(e)); exit(1); }
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(long long) * G, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < G; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("%-10s G=%3d S=%2d R=%d work=%3d: %6.0f cycles/hop\n", name, G, S, R, work, (double)mx / iters);
}

int main() {
  Sector* buf; long long* cyc; double* sink;
  cudaMalloc(&buf, sizeof(Sector) * 2 * 8 * 148 * 16);
  cudaMalloc(&cyc, sizeof(long long) * 148);
  cudaMalloc(&sink, 8);
  const int iters = 2000;
  for (int G : {2, 16, 148})
    for (int S : {1, 8}) {
      run<0>(buf, G, S, 1, iters, 0, cyc, sink, "volatile");
      run<1>(buf, G, S, 1, iters, 0, cyc, sink, "relaxed");
    }
  for (int R : {1, 2, 4, 8}) run<1>(buf, 148, 8, R, iters, 0, cyc, sink, "relaxed");
  for (int R : {1, 4}) run<0>(buf, 148, 8, R, iters, 0, cyc, sink, "volatile");
  for (int S : {2, 4, 16}) run<1>(buf, 148, S, 1, iters, 0, cyc, sink, "relaxed");
  run<1>(buf, 148, 8, 1, iters, 64, cyc, sink, "relaxed");
  long long* out; cudaMalloc(&out, 64);
  lat_kernel<<<1, 512>>>(out, sink, 1000);
  cudaDeviceSynchronize();
  long long h[8]; cudaMemcpy(h, out, 64, cudaMemcpyDeviceToHost);
  printf("cycles: DADD %lld  DFMA %lld  warp_sum(f64)+mul %lld  syncthreads(512) %lld  block-sum(2 bar) %lld  sqrt %lld  div %lld  hypot %lld\n",
         h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
  return 0;
}
