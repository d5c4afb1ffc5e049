// TMA-staged vs cp.async DMMA GEMM core on the solver's shapes (correctness + throughput).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        tools/gemmbench/gemm_tma_bench.cu paper_2310_14087_b200/csrc/alloc.cu paper_2310_14087_b200/csrc/prof.cu -o gtb
#include <cmath>
#include <cstdio>
#include <vector>
#include "../../paper_2310_14087_b200/csrc/gemm.cuh"
namespace kot { std::atomic<long long> g_kot_launches{0}; }
using namespace kot;

__global__ void fill(double* p, long n, unsigned seed) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    unsigned x = (unsigned)(i * 2654435761u) ^ seed;
    x ^= x >> 13; x *= 0x5bd1e995; x ^= x >> 15;
    p[i] = (double)(x & 0xffffff) / 16777216.0 - 0.5;
  }
}

template <bool TA, bool TB, int BM, int BN, int WM, int WN, int ST = 4>
void run(int M, int N, int K, int reps, double* A, double* B, double* C, double* C2, const double* ks, int ksplit,
         double* ws, const char* name) {
  GemmShape s = make_shape(M, N, K, A, TA ? M + (M & 1) : K + (K & 1), B, TB ? K + (K & 1) : N + (N & 1));
  s.kscale = ks;
  s.ksplit = ksplit;
  s.ws = ws;
  EpiAxpby e{C, N, 1.0, 0.0}, e2{C2, N, 1.0, 0.0};
  auto old_launch = [&] { gemm_launch_tiled<TA, TB, GB_M, GB_N>(s, e2, 0); };
  auto new_launch = [&] { gemm_launch_tma<TA, TB, BM, BN, WM, WN, ST>(s, e, 0); };
  old_launch();
  if (!gemm_launch_tma<TA, TB, BM, BN, WM, WN, ST>(s, e, 0)) { printf("%s: TMA path refused\n", name); return; }
  cudaDeviceSynchronize();
  std::vector<double> h1((long)M * N), h2((long)M * N);
  cudaMemcpy(h1.data(), C, 8L * M * N, cudaMemcpyDeviceToHost);
  cudaMemcpy(h2.data(), C2, 8L * M * N, cudaMemcpyDeviceToHost);
  double num = 0, den = 0;
  for (long i = 0; i < (long)M * N; ++i) { num += (h1[i] - h2[i]) * (h1[i] - h2[i]); den += h2[i] * h2[i]; }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms_old, ms_new;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) old_launch();
  cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms_old, e0, e1);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) new_launch();
  cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms_new, e0, e1);
  const double f = 2.0 * M * N * K;
  printf("%-30s %dx%d/%dx%d st%d M=%5d N=%5d K=%5d ks=%d  old %7.3f ms %6.2f TF/s | tma %7.3f ms %6.2f TF/s | rel %.2e %s\n", name,
         BM, BN, WM, WN, ST, M, N, K, ksplit, ms_old / reps, f / (ms_old / reps * 1e-3) / 1e12, ms_new / reps,
         f / (ms_new / reps * 1e-3) / 1e12, std::sqrt(num / den), cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const long big = 4096L * 4200;
  double *A, *B, *C, *C2, *W, *ks;
  cudaMalloc(&A, big * 8); cudaMalloc(&B, big * 8); cudaMalloc(&C, big * 8); cudaMalloc(&C2, big * 8);
  cudaMalloc(&W, 4 * big * 8); cudaMalloc(&ks, 8192 * 8);
  fill<<<1024, 256>>>(A, big, 1); fill<<<1024, 256>>>(B, big, 2); fill<<<64, 256>>>(ks, 8192, 3);
#define G1(...) run<true, false, __VA_ARGS__>(1000, 1000, 2000, 20, A, B, C, C2, ks, 1, W, "GEMM1 TN kscale");
#define G1S(...) run<true, false, __VA_ARGS__>(1000, 1000, 2000, 20, A, B, C, C2, ks, 2, W, "GEMM1 TN kscale split2");
#define G2(...) run<false, true, __VA_ARGS__>(2000, 1000, 1000, 20, A, B, C, C2, nullptr, 1, W, "GEMM2 NT");
#define SQ(...) run<false, false, __VA_ARGS__>(2000, 2000, 2000, 10, A, B, C, C2, nullptr, 1, W, "NN 2000");
  for (int pass = 0; pass < 2; ++pass) {
    G1(64, 64, 32, 32, 4) G1(64, 64, 32, 32, 6) G1(64, 64, 32, 32, 3) G1(128, 64, 32, 32, 4) G1(64, 128, 32, 32, 4)
    G1(128, 128, 64, 32, 4) G1(128, 128, 32, 64, 4) G1(64, 64, 64, 32, 4) G1(64, 64, 32, 64, 4)
    G1S(64, 64, 32, 32, 4) G1S(128, 64, 32, 32, 4)
    G2(64, 64, 32, 32, 4) G2(64, 64, 32, 32, 6) G2(128, 64, 32, 32, 4) G2(128, 64, 64, 32, 4) G2(128, 64, 64, 32, 6)
    G2(64, 64, 64, 32, 4) G2(64, 64, 32, 64, 4)
    SQ(64, 64, 32, 32, 4) SQ(64, 64, 32, 32, 6) SQ(128, 64, 32, 32, 4) SQ(128, 128, 64, 32, 4) SQ(128, 128, 32, 64, 4)
  }
}
