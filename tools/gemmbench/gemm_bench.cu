// Standalone DMMA GEMM microbenchmark (shapes of the SSN hot path).
#include <cstdio>
#include <vector>
#include "../../paper_2310_14087_b200/csrc/gemm.cuh"
namespace kot { std::atomic<long long> g_kot_launches{0}; }
using namespace kot;

template <bool TA, bool TB>
double run(int M, int N, int K, int reps, double* A, double* B, double* C, const char* name, int ksplit = 1,
           double* ws = nullptr) {
  GemmShape s = make_shape(M, N, K, A, TA ? M : K, B, TB ? K : N);
  s.ksplit = ksplit;
  s.ws = ws;
  EpiAxpby e{C, N, 1.0, 0.0};
  gemm_launch<TA, TB>(s, e, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) gemm_launch<TA, TB>(s, e, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double t = ms / reps;
  printf("%-28s M=%5d N=%5d K=%5d ks=%d  %8.3f ms  %6.2f TF/s\n", name, M, N, K, ksplit, t,
         2.0 * M * N * K / (t * 1e-3) / 1e12);
  return t;
}

int main() {
  const long big = 8192L * 8192;
  double *A, *B, *C, *W;
  cudaMalloc(&A, big * 8);
  cudaMalloc(&B, big * 8);
  cudaMalloc(&C, big * 8);
  cudaMalloc(&W, 4 * big * 8);
  cudaMemset(A, 0, big * 8);
  cudaMemset(B, 0, big * 8);
  run<false, false>(2048, 2048, 2048, 10, A, B, C, "NN square 2048");
  run<false, false>(2000, 2000, 2000, 10, A, B, C, "NN square 2000");
  run<true, false>(2000, 2000, 2000, 10, A, B, C, "TN square 2000");
  run<false, true>(2000, 2000, 2000, 10, A, B, C, "NT square 2000");
  run<false, false>(4096, 4096, 4096, 5, A, B, C, "NN square 4096");
  run<true, false>(1000, 2000, 2000, 10, A, B, C, "TN matvec C (k=1000)");
  run<true, false>(1000, 1000, 2000, 20, A, B, C, "TN H-form GEMM1 split3", 3, W);
  run<false, true>(2000, 1000, 1000, 20, A, B, C, "NT H-form GEMM2");
  run<false, true>(2000, 1000, 2000, 10, A, B, C, "NT matvec F (k=1000)");
  run<true, false>(100, 2000, 2000, 10, A, B, C, "TN C k=100");
  run<true, false>(100, 2000, 2000, 10, A, B, C, "TN C k=100 split", 8, W);
  run<false, false>(2000, 2000, 128, 10, A, B, C, "NN ormtr update K=128");
  run<true, false>(128, 2000, 2000, 10, A, B, C, "TN ormtr W1 split", 4, W);
  run<false, false>(1000, 1000, 1000, 20, A, B, C, "NN square 1000");
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
