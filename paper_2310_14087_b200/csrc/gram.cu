// Gaussian Gram assembly (north-star item 1; reference kernels.py:61-94,
// problem.py:135-169).
//
// * Square Grams are computed one triangle at a time and mirrored, so Q and
//   K are bitwise symmetric with a unit diagonal per kernel, exactly as the
//   reference's sym(g)+fill_diagonal(1) produces (kernels.py:70-72).
// * Squared distances are accumulated dimension by dimension without FMA
//   contraction, the same order scipy's cdist('sqeuclidean') uses.
// * The mean embeddings (column means of the n×ℓ sample/filling Gram) and the
//   embedding norms (mean of the n×n sample Gram) are fused reductions: the
//   rectangular Grams are never materialised in HBM.
// Point tiles are staged in shared memory; each CTA owns a 32×32 output tile.
#include "kernels.cuh"

namespace kot {

constexpr int GT = 32;      // output tile
constexpr int GMAXD = 128;  // max point dimension staged (pair kernel: 2d)

__device__ __forceinline__ double sqdist_seq(const double* a, const double* b, int d) {
  double s = 0.0;
  for (int k = 0; k < d; ++k) {
    const double t = __dsub_rn(a[k], b[k]);
    s = __dadd_rn(s, __dmul_rn(t, t));
  }
  return s;
}

// out[i][j] = Σ_s exp(-||P_s[i]-P_s[j]||² / (2 bw_s)), s over 1 or 2 point sets
// with (d_s) dims each, upper tiles only, mirrored; diagonal = nsets.
// If `pair` (K on [x y] ∈ R^{2d}), the two sets are concatenated instead.
__global__ void gram_square_kernel(const double* __restrict__ P0, const double* __restrict__ P1, int n,
                                   int d, double twobw0, double twobw1, int nsets, int pair,
                                   double* __restrict__ out) {
  extern __shared__ double gsh[];
  const int tiles = (n + GT - 1) / GT;
  int t = blockIdx.x, ti = 0;
  while (t >= tiles - ti) {
    t -= tiles - ti;
    ++ti;
  }
  const int tj = ti + t;
  const int i0 = ti * GT, j0 = tj * GT;
  const int D = pair ? 2 * d : d;
  const int LD = D + 1;
  double* si = gsh;
  double* sj = gsh + GT * LD;
  const int sets = pair ? 1 : nsets;
  // thread layout: 256 threads, each computes 4 entries (rows ty*4.., col tx)
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 rows of 4
  double res[4] = {0, 0, 0, 0};
  for (int s = 0; s < sets; ++s) {
    const double* P = (s == 0) ? P0 : P1;
    const double twobw = (s == 0) ? twobw0 : twobw1;
    __syncthreads();
    for (int e = threadIdx.x; e < GT * D; e += blockDim.x) {
      const int r = e / D, k = e % D;
      double vi = 0.0, vj = 0.0;
      if (pair) {
        const double* src = (k < d) ? P0 : P1;
        const int kk = (k < d) ? k : k - d;
        if (i0 + r < n) vi = src[(long)(i0 + r) * d + kk];
        if (j0 + r < n) vj = src[(long)(j0 + r) * d + kk];
      } else {
        if (i0 + r < n) vi = P[(long)(i0 + r) * d + k];
        if (j0 + r < n) vj = P[(long)(j0 + r) * d + k];
      }
      si[r * LD + k] = vi;
      sj[r * LD + k] = vj;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = ty * 4 + q;
      const double dd = sqdist_seq(si + r * LD, sj + tx * LD, D);
      res[q] = __dadd_rn(res[q], exp(-dd / twobw));
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = i0 + ty * 4 + q, j = j0 + tx;
    if (i >= n || j >= n || i > j) continue;
    const double v = (i == j) ? (double)sets : res[q];
    out[(long)i * n + j] = v;
    out[(long)j * n + i] = v;
  }
}

// embed[j] = mean_i exp(-||S_i - F_j||²/(2bw)) summed over the (S,F) pairs
// (mu: xs/xt, nu: ys/yt).  Column mean accumulated row by row, as numpy's
// .mean(axis=0) on a C-contiguous array does.
__global__ void embed_kernel(const double* __restrict__ xs, int nx, const double* __restrict__ ys, int ny,
                             const double* __restrict__ xt, const double* __restrict__ yt, int l, int d,
                             double twobw_x, double twobw_y, double lambda2, double* __restrict__ embed,
                             double* __restrict__ z) {
  extern __shared__ double sh[];  // staged sample chunk: [CH][d]
  const int CH = 64;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  double fj[GMAXD];
  double tot = 0.0;
  for (int set = 0; set < 2; ++set) {
    const double* S = set ? ys : xs;
    const double* F = set ? yt : xt;
    const int ns = set ? ny : nx;
    const double twobw = set ? twobw_y : twobw_x;
    if (j < l)
      for (int k = 0; k < d; ++k) fj[k] = F[(long)j * d + k];
    double acc = 0.0;
    for (int c0 = 0; c0 < ns; c0 += CH) {
      __syncthreads();
      for (int e = threadIdx.x; e < CH * d; e += blockDim.x) {
        const int r = e / d, k = e % d;
        sh[e] = (c0 + r < ns) ? S[(long)(c0 + r) * d + k] : 0.0;
      }
      __syncthreads();
      if (j < l) {
        const int cn = min(CH, ns - c0);
        for (int r = 0; r < cn; ++r) {
          double s = 0.0;
          for (int k = 0; k < d; ++k) {
            const double t = __dsub_rn(sh[r * d + k], fj[k]);
            s = __dadd_rn(s, __dmul_rn(t, t));
          }
          acc = __dadd_rn(acc, exp(-s / twobw));
        }
      }
    }
    tot = (set == 0) ? acc / ns : tot + acc / ns;
  }
  if (j < l) {
    double cost = 0.0;
    for (int k = 0; k < d; ++k) {
      const double t = __dsub_rn(xt[(long)j * d + k], yt[(long)j * d + k]);
      cost = __dadd_rn(cost, __dmul_rn(t, t));
    }
    embed[j] = tot;
    z[j] = tot - lambda2 * cost;
  }
}

// Partial sums of the square sample Gram (unit diagonal) per row block,
// deterministic: part[blockIdx.x] = Σ_{i in block rows} Σ_j g_ij.
__global__ void gram_sum_kernel(const double* __restrict__ S, int n, int d, double twobw,
                                double* __restrict__ part) {
  __shared__ double red[32];
  const int i = blockIdx.x;  // one row per block
  double acc = 0.0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double v;
    if (j == i) {
      v = 1.0;
    } else {
      double s = 0.0;
      for (int k = 0; k < d; ++k) {
        const double t = __dsub_rn(S[(long)i * d + k], S[(long)j * d + k]);
        s = __dadd_rn(s, __dmul_rn(t, t));
      }
      v = exp(-s / twobw);
    }
    acc += v;
  }
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) part[i] = acc;
}

__global__ void sum_parts_kernel(const double* __restrict__ p0, int n0, const double* __restrict__ p1, int n1,
                                 double* __restrict__ out) {
  __shared__ double red[32];
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < n0; i += blockDim.x) a += p0[i];
  for (int i = threadIdx.x; i < n1; i += blockDim.x) b += p1[i];
  a = block_sum(a, red);
  b = block_sum(b, red);
  if (threadIdx.x == 0) out[0] = a / ((double)n0 * n0) + b / ((double)n1 * n1);
}

void gram_square(const double* P0, const double* P1, int n, int d, double bw0, double bw1, int nsets,
                 bool pair, double* out, cudaStream_t st) {
  kot_require((pair ? 2 * d : d) <= GMAXD, KOT_EINVAL, "point dimension too large for the Gram kernel");
  const int tiles = (n + GT - 1) / GT;
  const int D = pair ? 2 * d : d;
  const size_t smem = 2 * GT * (D + 1) * sizeof(double);
  ensure_smem_attr((const void*)gram_square_kernel, (int)smem);
  gram_square_kernel<<<tiles * (tiles + 1) / 2, 256, smem, st>>>(P0, P1, n, d, 2.0 * bw0,
                                                               2.0 * bw1, nsets, pair ? 1 : 0, out);
  KOT_LAUNCH_CHECK();
}

// Rectangular Gram: one thread per output entry, 32×8 tiles with both point tiles in shared memory.
__global__ void gram_rect_kernel(const double* __restrict__ A, int m, const double* __restrict__ B, int p, int d,
                                 double twobw, double* __restrict__ out) {
  extern __shared__ double gsh[];
  const int LD = d + 1;
  double* sa = gsh;            // 8 rows of A
  double* sb = gsh + 8 * LD;   // 32 rows of B
  const int i0 = blockIdx.y * 8, j0 = blockIdx.x * 32;
  for (int e = threadIdx.x; e < 8 * d; e += blockDim.x) {
    const int r = e / d, k = e % d;
    sa[r * LD + k] = (i0 + r < m) ? A[(long)(i0 + r) * d + k] : 0.0;
  }
  for (int e = threadIdx.x; e < 32 * d; e += blockDim.x) {
    const int r = e / d, k = e % d;
    sb[r * LD + k] = (j0 + r < p) ? B[(long)(j0 + r) * d + k] : 0.0;
  }
  __syncthreads();
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int i = i0 + ty, j = j0 + tx;
  if (i < m && j < p) out[(long)i * p + j] = exp(-sqdist_seq(sa + ty * LD, sb + tx * LD, d) / twobw);
}

void gram_rect(const double* A, int m, const double* B, int p, int d, double bw, double* out, cudaStream_t st) {
  kot_require(d >= 1 && d <= GMAXD, KOT_EINVAL, "point dimension must be in [1, 128]");
  if (m == 0 || p == 0) return;
  const size_t smem = 40 * (d + 1) * sizeof(double);
  gram_rect_kernel<<<dim3(ceil_div(p, 32), ceil_div(m, 8)), 256, smem, st>>>(A, m, B, p, d, 2.0 * bw, out);
  KOT_LAUNCH_CHECK();
}

// out[j] = mean_i k(S_i, F_j): the column mean of the n × m Gram accumulated row by row (numpy's
// .mean(axis=0) order), never materialised.
__global__ void mean_embed_kernel(const double* __restrict__ S, int n, const double* __restrict__ F, int m, int d,
                                  double twobw, double* __restrict__ out) {
  extern __shared__ double sh[];  // staged sample chunk: [CH][d]
  const int CH = 64;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  double fj[GMAXD];
  if (j < m)
    for (int k = 0; k < d; ++k) fj[k] = F[(long)j * d + k];
  double acc = 0.0;
  for (int c0 = 0; c0 < n; c0 += CH) {
    __syncthreads();
    for (int e = threadIdx.x; e < CH * d; e += blockDim.x) {
      const int r = e / d, k = e % d;
      sh[e] = (c0 + r < n) ? S[(long)(c0 + r) * d + k] : 0.0;
    }
    __syncthreads();
    if (j < m) {
      const int cn = min(CH, n - c0);
      for (int r = 0; r < cn; ++r) acc = __dadd_rn(acc, exp(-sqdist_seq(sh + r * d, fj, d) / twobw));
    }
  }
  if (j < m) out[j] = acc / n;
}

__global__ void mean_parts_kernel(const double* __restrict__ part, int n, double* __restrict__ out) {
  __shared__ double red[32];
  double a = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) a += part[i];
  a = block_sum(a, red);
  if (threadIdx.x == 0) out[0] = a / ((double)n * n);
}

void mean_embedding_device(const double* S, int n, const double* F, int m, int d, double bw, double* out,
                           cudaStream_t st) {
  kot_require(d >= 1 && d <= GMAXD, KOT_EINVAL, "point dimension must be in [1, 128]");
  kot_require(n >= 1, KOT_EINVAL, "sample set is empty");
  if (m == 0) return;
  mean_embed_kernel<<<ceil_div(m, 128), 128, 64 * d * sizeof(double), st>>>(S, n, F, m, d, 2.0 * bw, out);
  KOT_LAUNCH_CHECK();
}

void embedding_norm_sq_device(const double* S, int n, int d, double bw, double* scratch, double* out,
                              cudaStream_t st) {
  kot_require(d >= 1 && d <= GMAXD, KOT_EINVAL, "point dimension must be in [1, 128]");
  kot_require(n >= 1, KOT_EINVAL, "sample set is empty");
  gram_sum_kernel<<<n, 256, 0, st>>>(S, n, d, 2.0 * bw, scratch);
  KOT_LAUNCH_CHECK();
  mean_parts_kernel<<<1, 256, 0, st>>>(scratch, n, out);
  KOT_LAUNCH_CHECK();
}

// Natural-order unscrambled Sobol points (reference datagen.py:77-95, 111-132): point with natural
// index i = XOR of the direction numbers V[dim][b] over the set bits b of i, divided by 2^bits (exact),
// then mapped affinely into [lower, upper] per coordinate (same operations as the reference's NumPy
// expression lower + unit·(upper − lower), no FMA contraction).  One thread per (point, dimension).
__global__ void sobol_points_kernel(const unsigned long long* __restrict__ V, int dim, int bits, long first,
                                    int count, const double* __restrict__ lower, const double* __restrict__ upper,
                                    double* __restrict__ out) {
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (t >= (long)count * dim) return;
  const int j = (int)(t / dim), k = (int)(t % dim);
  unsigned long long idx = (unsigned long long)(first + j);
  unsigned long long x = 0;
  for (int b = 0; b < bits && idx; ++b, idx >>= 1)
    if (idx & 1ull) x ^= V[(long)k * bits + b];
  const double unit = (double)x / ldexp(1.0, bits);
  out[t] = __dadd_rn(lower[k], __dmul_rn(unit, __dsub_rn(upper[k], lower[k])));
}

void sobol_points_device(const unsigned long long* V, int dim, int bits, long first, int count,
                         const double* lower, const double* upper, double* out, cudaStream_t st) {
  kot_require(dim >= 1 && bits >= 1 && bits <= 64 && count >= 0 && first >= 0, KOT_EINVAL, "invalid Sobol request");
  if (count == 0) return;
  const long total = (long)count * dim;
  sobol_points_kernel<<<(int)((total + 255) / 256), 256, 0, st>>>(V, dim, bits, first, count, lower, upper, out);
  KOT_LAUNCH_CHECK();
}

void assemble_device(const double* xs, int nx, const double* ys, int ny, const double* xt, const double* yt,
                     int l, int d, double bw_x, double bw_y, double bw_xy, double lambda2, double* Q, double* Kmat,
                     double* embed, double* z, double* q_sq, double* scratch, cudaStream_t st) {
  kot_require(d <= GMAXD / 2 && d >= 1, KOT_EINVAL, "point dimension must be in [1, 64]");
  // Q = G_x(xt) + G_y(yt): unit diagonals sum to 2.
  gram_square(xt, yt, l, d, bw_x, bw_y, 2, false, Q, st);
  // K on [xt yt] ∈ R^{2d}
  gram_square(xt, yt, l, d, bw_xy, bw_xy, 1, true, Kmat, st);
  const int thr = 128;
  embed_kernel<<<ceil_div(l, thr), thr, 64 * d * sizeof(double), st>>>(xs, nx, ys, ny, xt, yt, l, d, 2.0 * bw_x,
                                                                       2.0 * bw_y, lambda2, embed, z);
  KOT_LAUNCH_CHECK();
  gram_sum_kernel<<<nx, 256, 0, st>>>(xs, nx, d, 2.0 * bw_x, scratch);
  KOT_LAUNCH_CHECK();
  gram_sum_kernel<<<ny, 256, 0, st>>>(ys, ny, d, 2.0 * bw_y, scratch + nx);
  KOT_LAUNCH_CHECK();
  sum_parts_kernel<<<1, 256, 0, st>>>(scratch, nx, scratch + nx, ny, q_sq);
  KOT_LAUNCH_CHECK();
}

}  // namespace kot

namespace kot {

// evaluate_map (reference problem.py:254-284): for each query q_j, fused over
// the samples and the filling points (no n×m Gram in HBM):
//   emb_j = mean_i k(x_i, q_j),            S_j = mean_i k(x_i, q_j) x_i
//   wgt_j = Σ_i γ_i k(x̃_i, q_j),           F_j = Σ_i γ_i k(x̃_i, q_j) x̃_i
//   u_j = (emb_j − wgt_j)/(2λ₂),  ∇u_j = ((S_j − emb_j q_j) − (F_j − wgt_j q_j)) / (2λ₂σ²),  T_j = q_j − ∇u_j
// One warp per query; lanes stride the points; fixed-order warp reductions.
constexpr int MAP_MAXD = 64;

__global__ void evaluate_map_kernel(const double* __restrict__ xs, int n, const double* __restrict__ xt,
                                    const double* __restrict__ gamma, int l, const double* __restrict__ qs, int m,
                                    int d, double twobw, double bw, double lambda2, double* __restrict__ u,
                                    double* __restrict__ tmap) {
  const int lane = threadIdx.x & 31;
  const int j = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (j >= m) return;
  double q[MAP_MAXD], S[MAP_MAXD], F[MAP_MAXD];
  for (int k = 0; k < d; ++k) {
    q[k] = qs[(long)j * d + k];
    S[k] = 0.0;
    F[k] = 0.0;
  }
  double emb = 0.0, wgt = 0.0;
  for (int i = lane; i < n; i += 32) {
    double s = 0.0;
    for (int k = 0; k < d; ++k) {
      const double t = __dsub_rn(xs[(long)i * d + k], q[k]);
      s = __dadd_rn(s, __dmul_rn(t, t));
    }
    const double kv = exp(-s / twobw);
    emb += kv;
    for (int k = 0; k < d; ++k) S[k] += kv * xs[(long)i * d + k];
  }
  for (int i = lane; i < l; i += 32) {
    double s = 0.0;
    for (int k = 0; k < d; ++k) {
      const double t = __dsub_rn(xt[(long)i * d + k], q[k]);
      s = __dadd_rn(s, __dmul_rn(t, t));
    }
    const double kv = gamma[i] * exp(-s / twobw);
    wgt += kv;
    for (int k = 0; k < d; ++k) F[k] += kv * xt[(long)i * d + k];
  }
  emb = warp_sum(emb) / n;
  wgt = warp_sum(wgt);
  const double tl = 2.0 * lambda2;
  for (int k = 0; k < d; ++k) {
    const double sk = warp_sum(S[k]) / n - emb * q[k];
    const double fk = warp_sum(F[k]) - wgt * q[k];
    if (lane == 0) tmap[(long)j * d + k] = q[k] - (sk - fk) / (tl * bw);
  }
  if (lane == 0) u[j] = (emb - wgt) / tl;
}

void evaluate_map_device(const double* xs, int n, const double* xt, const double* gamma, int l, const double* qs,
                         int m, int d, double bw, double lambda2, double* u, double* tmap, cudaStream_t st) {
  kot_require(d >= 1 && d <= MAP_MAXD, KOT_EINVAL, "query dimension must be in [1, 64]");
  evaluate_map_kernel<<<ceil_div(m, 4), 128, 0, st>>>(xs, n, xt, gamma, l, qs, m, d, 2.0 * bw, bw, lambda2, u,
                                                      tmap);
  KOT_LAUNCH_CHECK();
}

}  // namespace kot
