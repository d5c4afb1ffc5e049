// Blocked Cholesky with the reference jitter ladder (north-star item 2;
// reference linalg.py:86-114, called from problem.py:155).
//
// Right-looking, NB=64 panels: the diagonal block is factored in shared
// memory by one CTA, the panel below by a row-parallel triangular solve, and
// the trailing matrix by the DMMA core as a symmetric (one-triangle +
// mirror) rank-NB update.  A non-positive or NaN pivot (the dpotrf failure
// condition) raises a device flag; the host then retries with the next
// jitter of [0, 1e-10·s, …, 1e-6·s], s = tr(K)/ℓ, and raises
// IndefiniteKernelError at the cap.
#include "gemm.cuh"
#include "kernels.cuh"

namespace kot {

constexpr int CH_NB = 64;

__global__ void chol_copy_jitter_kernel(const double* __restrict__ K, double* __restrict__ W, int n,
                                        double jitter) {
  const long total = (long)n * n;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    const int r = (int)(i / n), c = (int)(i % n);
    // sym(K) = 0.5 (K + Kᵀ) as linalg.py:98, then + jitter·I
    double v = 0.5 * (K[i] + K[(long)c * n + r]);
    if (r == c) v += jitter;
    W[i] = v;
  }
}

// np.trace order (sequential) so the jitter ladder is bitwise the reference's.
__global__ void trace_kernel(const double* __restrict__ K, int n, double* __restrict__ out) {
  if (threadIdx.x != 0) return;
  double a = 0.0;
  for (int i = 0; i < n; ++i) a += K[(long)i * n + i];
  out[0] = a;
}

// Left-looking unblocked factor of the diagonal block in shared memory, with
// the rounding order of LAPACK/OpenBLAS potf2: a_jj − Σ l_jk² (no FMA), then
// the column is scaled by the reciprocal of the pivot.  This keeps the
// jitter-ladder decision identical on rank-deficient Grams
// (test_linalg.py:58-66).
__global__ void potrf_diag_kernel(double* __restrict__ W, int n, int p, int b, int* __restrict__ fail) {
  __shared__ double A[CH_NB][CH_NB + 1];
  __shared__ double inv_sh;
  for (int e = threadIdx.x; e < b * b; e += blockDim.x) {
    const int i = e / b, j = e % b;
    A[i][j] = W[(long)(p + i) * n + p + j];
  }
  __syncthreads();
  for (int j = 0; j < b; ++j) {
    if (threadIdx.x == 0) {
      double dot = 0.0;
      for (int k = 0; k < j; ++k) dot = __dadd_rn(dot, __dmul_rn(A[j][k], A[j][k]));
      const double ajj = __dsub_rn(A[j][j], dot);
      if (!(ajj > 0.0)) *fail = 1;
      const double r = sqrt(ajj);
      A[j][j] = r;
      inv_sh = 1.0 / r;
    }
    __syncthreads();
    const double inv = inv_sh;
    for (int i = j + 1 + threadIdx.x; i < b; i += blockDim.x) {
      double dot = 0.0;
      for (int k = 0; k < j; ++k) dot = __dadd_rn(dot, __dmul_rn(A[i][k], A[j][k]));
      A[i][j] = __dmul_rn(__dsub_rn(A[i][j], dot), inv);
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < b * b; e += blockDim.x) {
    const int i = e / b, j = e % b;
    W[(long)(p + i) * n + p + j] = (j <= i) ? A[i][j] : 0.0;
  }
}

// rows r >= p+b: solve x·L11ᵀ = W[r, p:p+b] in place (thread per row)
__global__ void trsm_rows_kernel(double* __restrict__ W, int n, int p, int b) {
  __shared__ double L[CH_NB][CH_NB + 1];
  for (int e = threadIdx.x; e < b * b; e += blockDim.x) {
    const int i = e / b, j = e % b;
    L[i][j] = W[(long)(p + i) * n + p + j];
  }
  __syncthreads();
  const int r = p + b + blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double x[CH_NB];
  double* row = W + (long)r * n + p;
#pragma unroll 8
  for (int j = 0; j < b; ++j) x[j] = row[j];
  for (int j = 0; j < b; ++j) {
    double s = x[j];
    for (int k = 0; k < j; ++k) s -= x[k] * L[j][k];
    x[j] = s / L[j][j];
  }
#pragma unroll 8
  for (int j = 0; j < b; ++j) row[j] = x[j];
}

// R[i][j] = L[j][i] for j >= i, 0 below the diagonal.
__global__ void lower_to_upper_kernel(const double* __restrict__ L, double* __restrict__ R, int n) {
  __shared__ double tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int r = by + k, c = bx + threadIdx.x;
    if (r < n && c < n) tile[k][threadIdx.x] = L[(long)r * n + c];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int i = bx + k, j = by + threadIdx.x;  // R[i][j] = L[j][i]
    if (i < n && j < n) R[(long)i * n + j] = (j >= i) ? tile[threadIdx.x][k] : 0.0;
  }
}

void cholesky_factor(double* W, int n, int* dfail, cudaStream_t st) {
  for (int p = 0; p < n; p += CH_NB) {
    const int b = std::min(CH_NB, n - p);
    potrf_diag_kernel<<<1, 256, 0, st>>>(W, n, p, b, dfail);
    KOT_LAUNCH_CHECK();
    const int rest = n - p - b;
    if (rest > 0) {
      trsm_rows_kernel<<<ceil_div(rest, 128), 128, 0, st>>>(W, n, p, b);
      KOT_LAUNCH_CHECK();
      // W22 -= L21 L21ᵀ  (one triangle, mirrored)
      double* L21 = W + (long)(p + b) * n + p;
      GemmShape s = make_shape(rest, rest, b, L21, n, L21, n);
      s.sym_tiles = 1;
      double* C = W + (long)(p + b) * n + p + b;
      EpiSymMirror epi{C, n, -1.0, C, 1.0, 0.0};
      gemm_launch<false, true>(s, epi, st);
    }
  }
}

double cholesky_psd_device(const double* K, int n, double* R, double* work, double* dscal, int* dflag,
                           cudaStream_t st) {
  // scale = tr(sym(K))/n
  double* dtr = dscal;
  trace_kernel<<<1, 32, 0, st>>>(K, n, dtr);
  KOT_LAUNCH_CHECK();
  double tr = 0.0;
  KOT_CUDA(cudaMemcpyAsync(&tr, dtr, sizeof(double), cudaMemcpyDeviceToHost, st));
  KOT_CUDA(cudaStreamSynchronize(st));
  const double scale = tr / n;
  // ladder identical to linalg.py:86-105
  double ladder[16];
  int nl = 0;
  ladder[nl++] = 0.0;
  for (double lev = 1e-10; lev <= 1e-6 * (1 + 1e-12); lev *= 10.0) ladder[nl++] = lev * scale;
  for (int i = 0; i < nl; ++i) {
    chol_copy_jitter_kernel<<<std::min(ceil_div((long)n * n, 256), 4096), 256, 0, st>>>(K, work, n, ladder[i]);
    KOT_LAUNCH_CHECK();
    KOT_CUDA(cudaMemsetAsync(dflag, 0, sizeof(int), st));
    cholesky_factor(work, n, dflag, st);
    int fail = 0;
    KOT_CUDA(cudaMemcpyAsync(&fail, dflag, sizeof(int), cudaMemcpyDeviceToHost, st));
    KOT_CUDA(cudaStreamSynchronize(st));
    if (!fail) {
      dim3 grid(ceil_div(n, 32), ceil_div(n, 32)), blk(32, 8);
      lower_to_upper_kernel<<<grid, blk, 0, st>>>(work, R, n);
      KOT_LAUNCH_CHECK();
      return ladder[i];
    }
  }
  throw KotError(KOT_EINDEFINITE, "kernel matrix numerically indefinite");
}

}  // namespace kot
