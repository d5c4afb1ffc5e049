// Prototype: DMMA GEMM with larger CTA / warp tiles (compare with gemm.cuh's 64×64, 4 warps of 32×32).
// C = op(A) op(B), row-major, FP64 mma.sync m8n8k4; cp.async multistage, padded smem.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void cp8(void* smem, const void* g, int bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(g), "r"(bytes));
}
__device__ __forceinline__ void cp16(void* smem, const void* g, int bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(g), "r"(bytes));
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void waitg() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int BM, int BN, int WM, int WN, int BK, int ST, bool TA, bool TB>
__global__ void __launch_bounds__((BM / WM) * (BN / WN) * 32) gemm_big(int M, int N, int K, const double* A, int lda,
                                                                       const double* B, int ldb, double* C, int ldc) {
  constexpr int NT = (BM / WM) * (BN / WN) * 32;
  constexpr int MI = WM / 8, NJ = WN / 8;
  constexpr int PADK = BK + 4, PADM = BM + 4, PADN = BN + 4;
  constexpr int AT = TA ? BK * PADM : BM * PADK;
  constexpr int BT = TB ? BN * PADK : BK * PADN;
  extern __shared__ __align__(16) double sm[];
  double* As = sm;
  double* Bs = sm + ST * AT;
  const int tiles_m = (M + BM - 1) / BM;
  const int tm = blockIdx.x % tiles_m, tn = blockIdx.x / tiles_m;
  const int m0 = tm * BM, n0 = tn * BN;
  const int nkt = (K + BK - 1) / BK;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int wm = (warp / (BN / WN)) * WM, wn = (warp % (BN / WN)) * WN;
  auto issue = [&](int kt, int stg) {
    const int k0 = kt * BK;
    double* as = As + stg * AT;
    double* bs = Bs + stg * BT;
    if (TA) {  // A stored K×M: rows k, cols m (chunks of 2)
      for (int i = threadIdx.x; i < BK * BM / 2; i += NT) {
        const int r = i / (BM / 2), c = (i % (BM / 2)) * 2;
        const int gr = k0 + r, gc = m0 + c;
        const int v = (gr < K) ? min(max(M - gc, 0), 2) : 0;
        cp16(as + r * PADM + c, v ? A + (long)gr * lda + gc : A, v * 8);
      }
    } else {
      for (int i = threadIdx.x; i < BM * BK / 2; i += NT) {
        const int r = i / (BK / 2), c = (i % (BK / 2)) * 2;
        const int gr = m0 + r, gc = k0 + c;
        const int v = (gr < M) ? min(max(K - gc, 0), 2) : 0;
        cp16(as + r * PADK + c, v ? A + (long)gr * lda + gc : A, v * 8);
      }
    }
    if (TB) {  // B stored N×K
      for (int i = threadIdx.x; i < BN * BK / 2; i += NT) {
        const int r = i / (BK / 2), c = (i % (BK / 2)) * 2;
        const int gr = n0 + r, gc = k0 + c;
        const int v = (gr < N) ? min(max(K - gc, 0), 2) : 0;
        cp16(bs + r * PADK + c, v ? B + (long)gr * ldb + gc : B, v * 8);
      }
    } else {
      for (int i = threadIdx.x; i < BK * BN / 2; i += NT) {
        const int r = i / (BN / 2), c = (i % (BN / 2)) * 2;
        const int gr = k0 + r, gc = n0 + c;
        const int v = (gr < K) ? min(max(N - gc, 0), 2) : 0;
        cp16(bs + r * PADN + c, v ? B + (long)gr * ldb + gc : B, v * 8);
      }
    }
  };
  double acc[MI][NJ][2];
#pragma unroll
  for (int i = 0; i < MI; i++)
#pragma unroll
    for (int j = 0; j < NJ; j++) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
  for (int s = 0; s < ST - 1; ++s) {
    if (s < nkt) issue(s, s);
    commit();
  }
  for (int kt = 0; kt < nkt; ++kt) {
    waitg<ST - 2>();
    __syncthreads();
    if (kt + ST - 1 < nkt) issue(kt + ST - 1, (kt + ST - 1) % ST);
    commit();
    const double* as = As + (kt % ST) * AT;
    const double* bs = Bs + (kt % ST) * BT;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[MI], b[NJ];
#pragma unroll
      for (int i = 0; i < MI; i++) {
        const int m = wm + i * 8 + g;
        a[i] = TA ? as[(kk + t) * PADM + m] : as[m * PADK + kk + t];
      }
#pragma unroll
      for (int j = 0; j < NJ; j++) {
        const int n = wn + j * 8 + g;
        b[j] = TB ? bs[n * PADK + kk + t] : bs[(kk + t) * PADN + n];
      }
#pragma unroll
      for (int i = 0; i < MI; i++)
#pragma unroll
        for (int j = 0; j < NJ; j++) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  waitg<0>();
#pragma unroll
  for (int i = 0; i < MI; i++) {
    const int r = m0 + wm + i * 8 + g;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < NJ; j++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int c = n0 + wn + j * 8 + 2 * t + h;
        if (c < N) C[(long)r * ldc + c] = acc[i][j][h];
      }
  }
}

template <int BM, int BN, int WM, int WN, int BK, int ST, bool TA, bool TB>
void run(const char* name, int M, int N, int K, double* A, double* B, double* C) {
  constexpr int NT = (BM / WM) * (BN / WN) * 32;
  constexpr int AT = TA ? BK * (BM + 4) : BM * (BK + 4);
  constexpr int BT = TB ? BN * (BK + 4) : BK * (BN + 4);
  const int smem = ST * (AT + BT) * 8;
  auto k = gemm_big<BM, BN, WM, WN, BK, ST, TA, TB>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int grid = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  const int lda = TA ? M : K, ldb = TB ? K : N;
  k<<<grid, NT, smem>>>(M, N, K, A, lda, B, ldb, C, N);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 10;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) k<<<grid, NT, smem>>>(M, N, K, A, lda, B, ldb, C, N);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NT, smem);
  printf("%-34s BM%3d BN%3d W%2dx%2d BK%2d S%d occ %d  %5dx%5dx%5d  %7.3f ms  %6.2f TF/s  %s\n", name, BM, BN, WM, WN,
         BK, ST, occ, M, N, K, ms / reps, 2.0 * M * N * K / (ms / reps * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const long big = 8192L * 8192;
  double *A, *B, *C;
  cudaMalloc(&A, big * 8);
  cudaMalloc(&B, big * 8);
  cudaMalloc(&C, big * 8);
  cudaMemset(A, 0, big * 8);
  cudaMemset(B, 0, big * 8);
  run<128, 64, 64, 32, 8, 4, true, false>("TN matvec C", 1000, 2000, 2000, A, B, C);
  run<128, 64, 64, 32, 8, 4, false, true>("NT matvec F", 2000, 1000, 2000, A, B, C);
  run<128, 64, 64, 32, 8, 4, false, false>("NN 2000", 2000, 2000, 2000, A, B, C);
  run<128, 128, 64, 32, 8, 3, true, false>("TN matvec C", 1000, 2000, 2000, A, B, C);
  run<128, 128, 64, 32, 8, 3, false, true>("NT matvec F", 2000, 1000, 2000, A, B, C);
  run<128, 128, 64, 32, 8, 3, false, false>("NN 2000", 2000, 2000, 2000, A, B, C);
  run<128, 128, 64, 32, 16, 3, false, false>("NN 2000", 2000, 2000, 2000, A, B, C);
  run<128, 128, 64, 64, 8, 3, false, false>("NN 2000", 2000, 2000, 2000, A, B, C);
  run<64, 128, 32, 64, 8, 4, true, false>("TN matvec C", 1000, 2000, 2000, A, B, C);
  run<64, 128, 32, 64, 8, 4, false, true>("NT matvec F", 2000, 1000, 2000, A, B, C);
  run<64, 128, 32, 64, 8, 4, false, false>("NN 2000", 2000, 2000, 2000, A, B, C);
  run<128, 64, 64, 32, 8, 4, false, false>("NN 4096", 4096, 4096, 4096, A, B, C);
  run<128, 128, 64, 32, 8, 3, false, false>("NN 4096", 4096, 4096, 4096, A, B, C);
  return 0;
}
