// Two-stage Householder tridiagonalisation for the eigensolver (eig.cu).
//
// The one-stage reduction (dlatrd structure) needs a grid-wide symv and two
// grid barriers per column: latency-bound on every SM for the whole
// reduction.  Here the work is split the way it maps onto B200:
//
//   stage 1 (sy2sb): dense → band of width SB = 16.  Per 16-column panel:
//     one thread-block CLUSTER factors the (ℓ−j−16)×16 sub-panel with
//     Householder QR (the panel lives in the cluster's shared memory, the two
//     reductions per column go through DSMEM), then the trailing matrix gets
//     the two-sided rank-32 update A22 −= V Wᵀ + W Vᵀ with
//     W = A22 V T − ½ V (Tᵀ Vᵀ A22 V T) — three DMMA GEMMs.
//   stage 2 (sb2st): band → tridiagonal by bulge chasing, ONE cluster whose
//     CTAs hold the whole band in shared memory (column blocks, DSMEM for the
//     neighbours').  Task (i, t) of sweep i annihilates column i (t = 0) or
//     the first column of the bulge block t; tasks with 2i + t = s are
//     element-disjoint and run concurrently (one warp each), one cluster
//     barrier per step s.
//   back-transform: Q = Q1·Q2.  Q2's reflectors are applied in blocks
//     G(I, t) = {H(i, t): i ∈ sweep block I} (sweep blocks last to first,
//     t ascending inside a block; tools/twostage_proto.py checks the order),
//     each as I − V T Vᵀ on a 31-row window; Q1 reuses ormtr's compact-WY
//     blocks (the stage-1 reflectors are stored in the same Vall layout).
//
// Both latency-bound parts run on ≤ 16 SMs, so concurrent eigensolves and the
// Newton chain's GEMMs share the GPU instead of queueing behind a grid-wide
// cooperative kernel.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "gemm.cuh"
#include "kernels.cuh"
#include "prof.cuh"

namespace cg = cooperative_groups;

namespace kot {

constexpr int SB = 16;            // band width
constexpr int SB_LDX = 3 * SB;    // stage-1 GEMM operand rows [V | W | V]
constexpr int PQR_THREADS = 512;  // 16 warps (column q) × 32 lanes (row group)
constexpr int PQR_LD = SB + 1;
constexpr int PQR_MAXCS = 16;
constexpr int SB2_LDB = 2 * SB;   // band column: d = r − c ∈ [0, 2·SB)  (bulge reaches 2·SB − 1)

static int eig_nt(int n) { return (n - 2) / SB + 1; }           // tasks per sweep (max)
static int eig_ni(int n) { return (n - 2 + SB - 1) / SB; }      // sweep blocks (sweeps 0..n−3)

long two_stage_q2_size(int n) { return n < 3 ? 1 : (long)eig_ni(n) * eig_nt(n) * SB * SB; }

// ============================================================== stage 1

__device__ __forceinline__ double half_sum(double v, unsigned mask) {
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o, 16);
  return v;
}

// Householder QR of the sub-panel A[j+SB:, j:j+SB] on one cluster (rows split
// over the CTAs, thread (q, rg) = column q × row group rg).  Per column: one
// cluster barrier for ‖x‖²/α, one for the 15 dot products vᵀP[:, q]; each
// half-warp gathers the CTA partials through DSMEM and reduces them in a fixed
// lane order, so every CTA derives bit-identical β, τ.  Writes R into A, the
// reflectors (explicit, zero above the unit entry, zero column if τ = 0) into
// Vall (ormtr layout) and Xs, τ, and the panel's T (forward, columnwise) into Tp.
constexpr int PQR_RPT = 16;  // rows per lane: ≤ 32·16 = 512 rows per CTA
unsigned long long* g_pqr_dbg = nullptr;
__global__ void __launch_bounds__(PQR_THREADS) sy2sb_panel_kernel(double* A, int n, int j, double* Vall,
                                                                  double* tau_out, double* Xs, double* Tp,
                                                                  unsigned long long* dbg) {
  cg::cluster_group cl = cg::this_cluster();
  const bool timing = dbg && threadIdx.x == 0 && cl.block_rank() == 0;
  long long tl = timing ? clock64() : 0;
  unsigned long long tseg[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#define PQM(k_)                     \
  if (timing) {                     \
    const long long t_ = clock64(); \
    tseg[k_] += t_ - tl;            \
    tl = t_;                        \
  }
  const int CS = (int)cl.num_blocks(), rank = (int)cl.block_rank();
  extern __shared__ double P[];  // [rows][PQR_LD]
  __shared__ double red_n[2];
  __shared__ double red_d[SB];
  __shared__ double Sk[SB][SB + 1];
  __shared__ double taus[SB];
  __shared__ double Ts[SB][SB + 1];
  const int m = n - j - SB;
  const int kb = min(SB, m);
  const int rc = (m + CS - 1) / CS;
  const int lo = rank * rc, hi = min(m, lo + rc);
  const int tid = threadIdx.x, q = tid >> 5, rg = tid & 31;
  for (int e = tid; e < (hi - lo) * SB; e += blockDim.x) {
    const int rr = e / SB, cc = e % SB;
    P[rr * PQR_LD + cc] = A[(long)(j + SB + lo + rr) * n + j + cc];
  }
  if (tid < SB) taus[tid] = 0.0;
  __syncthreads();
  if (q == 0) {  // ‖x[1:]‖² and α of column 0
    double s = 0.0;
#pragma unroll 4
    for (int jj = 0; jj < PQR_RPT; ++jj) {
      const int r = lo + rg + 32 * jj;
      if (r < hi && r > 0) {
        const double x = P[(r - lo) * PQR_LD];
        s += x * x;
      }
    }
    s = warp_sum(s);
    if (rg == 0) {
      red_n[0] = s;
      red_n[1] = (lo == 0 && hi > 0) ? P[0] : 0.0;
    }
  }
  PQM(0)
  for (int k = 0; k < kb; ++k) {
    cl.sync();
    PQM(1)
    double xn2 = 0.0, alpha = 0.0;
    if (rg < CS) {
      const double* rn = cl.map_shared_rank(red_n, rg);
      xn2 = rn[0];
      alpha = rn[1];
    }
    xn2 = warp_sum(xn2);
    alpha = warp_sum(alpha);
    double beta, tau, scale;
    if (xn2 == 0.0) {
      tau = 0.0;
      beta = alpha;
      scale = 1.0;
    } else {
      beta = -copysign(hypot(alpha, sqrt(xn2)), alpha);
      tau = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    PQM(2)
    // dots s_q = Σ_{r ≥ k} v_r P[r][q]  (q > k: apply to column q; q < k: T column), v cached per row
    double vc[PQR_RPT];
    double s = 0.0;
#pragma unroll
    for (int jj = 0; jj < PQR_RPT; ++jj) {
      const int r = lo + rg + 32 * jj;
      double v = 0.0;
      if (r < hi && r >= k) {
        v = (r == k) ? 1.0 : P[(r - lo) * PQR_LD + k] * scale;
        if (q != k) s += v * P[(r - lo) * PQR_LD + q];
      }
      vc[jj] = v;
    }
    s = warp_sum(s);
    if (rg == 0) red_d[q] = s;
    PQM(3)
    cl.sync();
    PQM(4)
    double tq = (rg < CS) ? cl.map_shared_rank(red_d, rg)[q] : 0.0;
    tq = warp_sum(tq);
    if (rg == 0 && q < k) Sk[k][q] = tq;
    if (tid == 0) taus[k] = tau;
    if (q > k && tau != 0.0) {
      const double f = tau * tq;
#pragma unroll
      for (int jj = 0; jj < PQR_RPT; ++jj) {
        const int r = lo + rg + 32 * jj;
        if (r < hi && r >= k) P[(r - lo) * PQR_LD + q] -= f * vc[jj];
      }
    } else if (q == k) {
#pragma unroll
      for (int jj = 0; jj < PQR_RPT; ++jj) {
        const int r = lo + rg + 32 * jj;
        if (r < hi && r >= k) P[(r - lo) * PQR_LD + k] = (r == k) ? beta : vc[jj];
      }
    }
    PQM(5)
    if (q == k + 1 && k + 1 < kb) {  // next column's ‖x[1:]‖² and α, from the just-updated values
      double s2 = 0.0;
#pragma unroll 4
      for (int jj = 0; jj < PQR_RPT; ++jj) {
        const int r = lo + rg + 32 * jj;
        if (r < hi && r > k + 1) {
          const double x = P[(r - lo) * PQR_LD + k + 1];
          s2 += x * x;
        }
      }
      s2 = warp_sum(s2);
      if (rg == 0) {
        red_n[0] = s2;
        red_n[1] = (k + 1 >= lo && k + 1 < hi) ? P[(k + 1 - lo) * PQR_LD + k + 1] : 0.0;
      }
    }
  }
  PQM(6)
  __syncthreads();
  if (tid < SB) {  // T row l: T[l][k] = −τ_k Σ_{l ≤ m < k} T[l][m] s_k[m]
    const int l = tid;
    for (int c = 0; c < SB; ++c) Ts[l][c] = 0.0;
    if (l < kb) {
      Ts[l][l] = taus[l];
      for (int c = l + 1; c < kb; ++c) {
        double acc = 0.0;
        for (int mm = l; mm < c; ++mm) acc += Ts[l][mm] * Sk[c][mm];
        Ts[l][c] = -taus[c] * acc;
      }
    }
  }
  __syncthreads();
  // ---- outputs
  for (int e = tid; e < (hi - lo) * SB; e += blockDim.x) {
    const int rr = e / SB, cc = e % SB, r = lo + rr;
    const long grow = (long)(j + SB + r);
    const double p = P[rr * PQR_LD + cc];
    double v = 0.0;
    if (cc < kb && taus[cc] != 0.0) v = (r == cc) ? 1.0 : (r > cc ? p : 0.0);
    A[grow * n + j + cc] = (r > cc && cc < kb) ? 0.0 : p;
    Vall[grow * n + j + cc] = v;
    Xs[grow * SB_LDX + cc] = v;
    Xs[grow * SB_LDX + 2 * SB + cc] = v;
  }
  if (rank == 0) {
    if (tid < SB) tau_out[j + tid] = taus[tid];
    for (int e = tid; e < SB * SB; e += blockDim.x) Tp[e] = Ts[e / SB][e % SB];
  }
  cl.sync();  // no CTA leaves while others may still read its red_n / red_d
  PQM(7)
  if (timing)
    for (int k2 = 0; k2 < 8; ++k2) atomicAdd(dbg + k2, tseg[k2]);
#undef PQM
}

// Xw = A22 V for a 64-row block and one K-split (partial) on the FP64 tensor cores
// (mma m8n8k4; 4 warps × 2×2 8×8 tiles), plus the partial S = V[rows]ᵀ Xw_partial[rows];
// both reduced in fixed order afterwards.  A22 and V chunks stream through a 2-stage
// cp.async pipeline (8-byte copies: A22 rows need not be 16-byte aligned).
constexpr int XW_ROWS = 64;
constexpr int XW_KC = 32;
constexpr int XW_LDA = XW_KC + 4;
constexpr int XW_LDV = SB + 4;
__global__ void __launch_bounds__(128) sy2sb_xw_kernel(const double* __restrict__ A22, int lda, int m,
                                                       const double* __restrict__ X0, double* Xwp,
                                                       double* Spart) {
  __shared__ double Ak[2][XW_ROWS][XW_LDA];
  __shared__ double Vk[2][XW_KC][XW_LDV];
  // after the K loop the A stages are reused for the Xw tile and the V rows
  double (*Xo)[SB + 1] = reinterpret_cast<double (*)[SB + 1]>(&Ak[0][0][0]);
  double (*Vr)[SB + 1] = reinterpret_cast<double (*)[SB + 1]>(&Ak[0][0][0] + XW_ROWS * (SB + 1));
  const int tid = threadIdx.x;
  const int rb = blockIdx.x * XW_ROWS;
  const int ks = gridDim.y, kid = blockIdx.y;
  const int kchunk = ((m + ks - 1) / ks + XW_KC - 1) / XW_KC * XW_KC;
  const int k0 = kid * kchunk, k1 = min(m, k0 + kchunk);
  auto issue = [&](int kb, int buf) {
    const int kn = min(XW_KC, k1 - kb);
    for (int e = tid; e < XW_ROWS * XW_KC; e += 128) {
      const int rr = e / XW_KC, kk = e % XW_KC;
      const bool ok = rb + rr < m && kk < kn;
      cp_async_8(&Ak[buf][rr][kk], ok ? A22 + (long)(rb + rr) * lda + kb + kk : A22, ok ? 8 : 0);
    }
    for (int e = tid; e < XW_KC * SB; e += 128) {
      const int kk = e / SB, c = e % SB;
      const bool ok = kk < kn;
      cp_async_8(&Vk[buf][kk][c], ok ? X0 + (long)(kb + kk) * SB_LDX + c : X0, ok ? 8 : 0);
    }
    cp_async_commit();
  };
  const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, tq = lane & 3;
  const int rt0 = warp * 2;  // row tiles rt0, rt0+1; column tiles 0, 1
  double acc[2][2][2] = {};
  int buf = 0;
  if (k0 < k1) issue(k0, 0);
  for (int kb = k0; kb < k1; kb += XW_KC) {
    if (kb + XW_KC < k1) {
      issue(kb + XW_KC, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < XW_KC; kk += 4) {
      const double a0 = Ak[buf][rt0 * 8 + g][kk + tq], a1 = Ak[buf][rt0 * 8 + 8 + g][kk + tq];
      const double b0 = Vk[buf][kk + tq][g], b1 = Vk[buf][kk + tq][8 + g];
      dmma(acc[0][0][0], acc[0][0][1], a0, b0);
      dmma(acc[0][1][0], acc[0][1][1], a0, b1);
      dmma(acc[1][0][0], acc[1][0][1], a1, b0);
      dmma(acc[1][1][0], acc[1][1][1], a1, b1);
    }
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int jt = 0; jt < 2; ++jt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int rr = (rt0 + i) * 8 + g, c = jt * 8 + 2 * tq + h;
        Xo[rr][c] = acc[i][jt][h];
        if (rb + rr < m) Xwp[((long)kid * m + rb + rr) * SB + c] = acc[i][jt][h];
      }
  for (int e = tid; e < XW_ROWS * SB; e += 128) {
    const int rr = e / SB, c = e % SB;
    Vr[rr][c] = (rb + rr < m) ? X0[(long)(rb + rr) * SB_LDX + c] : 0.0;
  }
  __syncthreads();
  for (int e = tid; e < SB * SB; e += 128) {
    const int a = e >> 4, c = e & 15;
    double s0 = 0.0, s1 = 0.0;
    for (int rr = 0; rr < XW_ROWS; rr += 2) {
      s0 += Vr[rr][a] * Xo[rr][c];
      s1 += Vr[rr + 1][a] * Xo[rr + 1][c];
    }
    Spart[((long)kid * gridDim.x + blockIdx.x) * SB * SB + e] = s0 + s1;
  }
}

// Fixed-order sum of the S partials, first level: CTA b sums partials b, b + G, b + 2G, …
// (all loads of a thread issued together); the W kernel adds the G level-1 sums in order.
constexpr int SRED_G = 16;
__global__ void __launch_bounds__(256) sy2sb_sred_kernel(const double* __restrict__ Spart, int nparts, double* S1) {
  const int e = threadIdx.x, b = blockIdx.x;
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int p = b, u = 0;
  for (; p < nparts; p += SRED_G, ++u) acc[u & 7] += __ldg(Spart + (long)p * SB * SB + e);
  S1[b * SB * SB + e] = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
}

// W = Xw T − ½ V M with M = Tᵀ S T, S = Σ partials (fixed order), Xw = Σ_k Xwp[k] (fixed order);
// W overwrites columns SB..2SB of Xs.
__global__ void __launch_bounds__(256) sy2sb_w_kernel(double* Xs, int r0, int m, const double* Tp,
                                                      const double* Sg, const double* Xwp, int ks) {
  __shared__ double T[SB][SB + 1], TS[SB][SB + 1], M[SB][SB + 1], S[SB][SB + 1];
  __shared__ double xw[16][SB + 1], vv[16][SB + 1];
  const int tid = threadIdx.x, a = tid >> 4, c = tid & 15;
  T[a][c] = Tp[a * SB + c];
  {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int b = 0; b < SRED_G; b += 2) {
      s0 += Sg[b * SB * SB + tid];
      s1 += Sg[(b + 1) * SB * SB + tid];
    }
    S[a][c] = s0 + s1;
  }
  __syncthreads();
  {
    double s = 0.0;
    for (int k = 0; k < SB; ++k) s += T[k][a] * S[k][c];
    TS[a][c] = s;
  }
  __syncthreads();
  {
    double s = 0.0;
    for (int k = 0; k < SB; ++k) s += TS[a][k] * T[k][c];
    M[a][c] = s;
  }
  for (int rb = blockIdx.x * 16; rb < m; rb += gridDim.x * 16) {
    const int r = rb + a;
    __syncthreads();
    if (r < m) {
      double x = 0.0;
      for (int k = 0; k < ks; ++k) x += Xwp[((long)k * m + r) * SB + c];
      xw[a][c] = x;
      vv[a][c] = Xs[(long)(r0 + r) * SB_LDX + c];
    }
    __syncthreads();
    if (r < m) {
      double s = 0.0, u = 0.0;
      for (int k = 0; k < SB; ++k) {
        s += xw[a][k] * T[k][c];
        u += vv[a][k] * M[k][c];
      }
      Xs[(long)(r0 + r) * SB_LDX + SB + c] = s - 0.5 * u;
    }
  }
}

// A22 −= V Wᵀ + W Vᵀ for one 64×64 lower tile (tm ≥ tn) + its mirror: K = 2·SB = 32,
// both operands staged whole in shared memory, one triangle computed (exact symmetry).
constexpr int S2K_T = 64;
constexpr int S2K_LD = 2 * SB + 1;
constexpr int S2K_SMEM = (2 * S2K_T * S2K_LD + S2K_T * (S2K_T + 1)) * 8;
// Tile sets: mode 0 = every lower tile; 1 = column strip 0 only (the next panel's columns, for the
// look-ahead); 2 = the lower tiles right of strip 0.
__global__ void __launch_bounds__(256) sy2sb_syr2k_kernel(double* C, int ldc, int m, const double* __restrict__ X0,
                                                          int mode) {
  extern __shared__ double s2k[];
  double (*Ash)[S2K_LD] = reinterpret_cast<double (*)[S2K_LD]>(s2k);
  double (*Bsh)[S2K_LD] = reinterpret_cast<double (*)[S2K_LD]>(s2k + S2K_T * S2K_LD);
  double (*Ct)[S2K_T + 1] = reinterpret_cast<double (*)[S2K_T + 1]>(s2k + 2 * S2K_T * S2K_LD);
  int tm, tn;
  if (mode == 1) {
    tm = blockIdx.x;
    tn = 0;
  } else {  // blockIdx.x → lower tile (tm, tn), tm ≥ tn, of the (sub)triangle
    const int b = blockIdx.x;
    tm = (int)((sqrt(8.0 * b + 1.0) - 1.0) * 0.5);
    while ((tm + 1) * (tm + 2) / 2 <= b) ++tm;
    while (tm * (tm + 1) / 2 > b) --tm;
    tn = b - tm * (tm + 1) / 2;
    if (mode == 2) {
      ++tm;
      ++tn;
    }
  }
  const int i0 = tm * S2K_T, j0 = tn * S2K_T;
  const int tid = threadIdx.x;
  for (int e = tid; e < S2K_T * 2 * SB; e += 256) {
    const int rr = e / (2 * SB), k = e % (2 * SB);
    Ash[rr][k] = (i0 + rr < m) ? __ldg(X0 + (long)(i0 + rr) * SB_LDX + k) : 0.0;       // [V | W]
    Bsh[rr][k] = (j0 + rr < m) ? __ldg(X0 + (long)(j0 + rr) * SB_LDX + SB + k) : 0.0;  // [W | V]
  }
  __syncthreads();
  // 8 warps × (2 row tiles × 4 column tiles) of 8×8 on the FP64 tensor cores, K = 2·SB = 32
  const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, tq = lane & 3;
  const int rt0 = (warp >> 1) * 2, ct0 = (warp & 1) * 4;
  double acc[2][4][2] = {};
#pragma unroll
  for (int k0 = 0; k0 < 2 * SB; k0 += 4) {
    const double a0 = Ash[rt0 * 8 + g][k0 + tq], a1 = Ash[rt0 * 8 + 8 + g][k0 + tq];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double bv = Bsh[(ct0 + u) * 8 + g][k0 + tq];
      dmma(acc[0][u][0], acc[0][u][1], a0, bv);
      dmma(acc[1][u][0], acc[1][u][1], a1, bv);
    }
  }
#pragma unroll
  for (int v = 0; v < 2; ++v)
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int li = (rt0 + v) * 8 + g, lj = (ct0 + u) * 8 + 2 * tq + h;
        const int i = i0 + li, j = j0 + lj;
        double o = 0.0;
        if (i < m && j < m && i >= j) {
          o = C[(long)i * ldc + j] - acc[v][u][h];
          C[(long)i * ldc + j] = o;
        }
        Ct[li][lj] = o;
      }
  __syncthreads();
  // mirror: C[j][i] = C[i][j] for i > j, coalesced along i
  const int tr = tid >> 4, tc = tid & 15;
#pragma unroll
  for (int v = 0; v < 4; ++v)
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int jj = tr + 16 * v, ii = tc + 16 * u;  // row j0+jj, column i0+ii
      const int i = i0 + ii, j = j0 + jj;
      if (i < m && j < m && i > j) C[(long)j * ldc + i] = Ct[ii][jj];
    }
}

static int pqr_cluster(int m) { return std::max(1, std::min(PQR_MAXCS, (m + 191) / 192)); }

static void sy2sb(const double* Z, int n, EigWork& w, cudaStream_t st) {
  KOT_CUDA(cudaMemcpyAsync(w.A, Z, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, st));
  KOT_CUDA(cudaMemsetAsync(w.Vall, 0, sizeof(double) * n * n, st));
  KOT_CUDA(cudaMemsetAsync(w.tau, 0, sizeof(double) * n, st));
  // Look-ahead: after panel p's W is known, the update of the next panel's columns (tile strip 0)
  // runs on the main stream, so panel p+1's QR can start while the rest of the rank-32 update runs
  // on a second stream; Xs is double-buffered (panel parity) because that update still reads it.
  w.ensure_two_stage();
  cudaStream_t sb = w.st2;
  double* Xs = w.X;      // n × SB_LDX, two buffers
  double* Tp = w.Tf;     // SB × SB
  double* Sred = w.Tf + SB * SB;  // SRED_G level-1 sums of S
  ensure_smem_attr((const void*)sy2sb_syr2k_kernel, S2K_SMEM);
  int pidx = 0;
  for (int j = 0; j + SB + 1 < n; j += SB, ++pidx) {
    if ((pidx & 7) == 0) w.check_cancel(st);
    const int m = n - j - SB;
    Xs = w.X + (long)(pidx & 1) * n * SB_LDX;
    const int cs = pqr_cluster(m);
    kot_require(ceil_div(m, cs) <= 32 * PQR_RPT, KOT_EINVAL, "matrix order too large for the band reduction");
    const int rows = (m + cs - 1) / cs;
    const size_t smem = sizeof(double) * std::max(rows, 1) * PQR_LD;
    ensure_smem_attr((const void*)sy2sb_panel_kernel, (int)smem, true);
    {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs);
      cfg.blockDim = dim3(PQR_THREADS);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      ProfScope ps("sy2sb_panel", st);
      KOT_CUDA(cudaLaunchKernelEx(&cfg, sy2sb_panel_kernel, w.A, n, j, w.Vall, w.tau, Xs, Tp, g_pqr_dbg));
      KOT_LAUNCH_CHECK();
    }
    const int r0 = j + SB;
    double* A22 = w.A + (long)r0 * n + r0;
    double* X0 = Xs + (long)r0 * SB_LDX;
    {  // Xw = A22 V (row blocks × K-splits) and the partial S = Vᵀ Xw; then W
      const int nb = ceil_div(m, XW_ROWS);
      const int ks = std::max(1, std::min(8, m / 1024));  // K-splits: keep ≥ ~2 CTAs per SM busy at large m
      double* Xwp = w.W1;       // [ks][m][SB]
      double* Spart = w.splitws;  // [ks·nb][SB·SB]
      if (pidx > 0) KOT_CUDA(cudaStreamWaitEvent(st, w.ev_rest, 0));  // A22 fully updated by panel p−1
      sy2sb_xw_kernel<<<dim3(nb, ks), 128, 0, st>>>(A22, n, m, X0, Xwp, Spart);
      KOT_LAUNCH_CHECK();
      sy2sb_sred_kernel<<<SRED_G, 256, 0, st>>>(Spart, ks * nb, Sred);
      KOT_LAUNCH_CHECK();
      sy2sb_w_kernel<<<std::min(ceil_div(m, 16), 2 * kNumSMs), 256, 0, st>>>(Xs, r0, m, Tp, Sred, Xwp, ks);
      KOT_LAUNCH_CHECK();
    }
    {  // A22 −= V Wᵀ + W Vᵀ  (one triangle + mirror): strip 0 now, the rest beside the next panel's QR
      const int nt = ceil_div(m, S2K_T);
      sy2sb_syr2k_kernel<<<nt, 256, S2K_SMEM, st>>>(A22, n, m, X0, 1);
      KOT_LAUNCH_CHECK();
      if (nt > 1) {
        KOT_CUDA(cudaEventRecord(w.ev_w, st));
        KOT_CUDA(cudaStreamWaitEvent(sb, w.ev_w, 0));
        sy2sb_syr2k_kernel<<<(nt - 1) * nt / 2, 256, S2K_SMEM, sb>>>(A22, n, m, X0, 2);
        KOT_LAUNCH_CHECK();
      }
      KOT_CUDA(cudaEventRecord(w.ev_rest, sb));
    }
  }
  KOT_CUDA(cudaStreamWaitEvent(st, w.ev_rest, 0));
}

// ============================================================== stage 2

struct Sb2Args {
  const double* A;
  int n, cw, NT;
  double* d;
  double* e;
  double* Vq2;
  double* tq2;
  unsigned long long* dbg;  // nullable: per-segment cycles of CTA 0 warp 0 (kot_debug_sb2st_timing)
};
unsigned long long* g_sb2_dbg = nullptr;

__device__ __forceinline__ long q2_index(int i, int t, int NT) {
  return ((long)(i / SB) * NT + t) * SB + (i % SB);
}

__device__ __forceinline__ int fdiv(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }
__device__ __forceinline__ int cdiv(int a, int b) { return -fdiv(-a, b); }

// Householder of x (lanes 0..len−1 of the warp, zeros elsewhere): returns v_lane, sets tau, beta.
__device__ __forceinline__ double warp_house(double x, int lane, double& tau, double& beta) {
  const double alpha = __shfl_sync(0xffffffffu, x, 0);
  double s = (lane >= 1) ? x * x : 0.0;
  s = warp_sum(s);
  double scale;
  if (s == 0.0) {
    tau = 0.0;
    beta = alpha;
    scale = 1.0;
  } else {
    // band entries are O(‖A‖): no over/underflow guard (hypot) needed on this path
    beta = -copysign(sqrt(fma(alpha, alpha, s)), alpha);
    tau = (beta - alpha) / beta;
    scale = 1.0 / (alpha - beta);
  }
  return lane == 0 ? 1.0 : x * scale;
}

__device__ __forceinline__ uint32_t dsm_map(const void* p, int rank) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(p), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ double dsm_ld(uint32_t a) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void dsm_st(uint32_t a, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}

constexpr int SB2_WARPS = 8;
constexpr int SB2_NTHREADS = 32 * SB2_WARPS;

__device__ __forceinline__ double sum16(const double (&p)[16]) {
  return ((((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]))) +
          (((p[8] + p[9]) + (p[10] + p[11])) + ((p[12] + p[13]) + (p[14] + p[15]))));
}

__device__ __forceinline__ void dsm_st_release_u64(uint32_t a, unsigned long long v) {
  asm volatile("st.release.cluster.shared::cluster.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long dsm_ld_acquire_u64(uint32_t a) {
  unsigned long long v;
  asm volatile("ld.acquire.cluster.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
  return v;
}

// Bulge chasing, one warp per SWEEP: warp g of the cluster chases sweeps g, g+W, g+2W, …
// (W = warps in the cluster) all the way down, keeping the previous reflector in
// registers.  Task (i, t) only has to wait for task (i−1, t+1): the predecessor
// sweep's warp publishes (sweep+1, tasks done) with a cluster-scope release store
// in its CTA's shared memory, the successor polls it with acquire loads.  Tasks
// running concurrently under this rule are element-disjoint (wavefront argument,
// tools/twostage_proto.py).  Lanes 0–15 hold the rows of the off-diagonal block
// C (or the column being annihilated for t = 0), lanes 16–31 the rows of the
// diagonal block D, in registers; the band lives in the cluster's shared memory.
__global__ void __launch_bounds__(SB2_NTHREADS, 1) sb2st_kernel(Sb2Args a) {
  cg::cluster_group cl = cg::this_cluster();
  const int CS = (int)cl.num_blocks(), rank = (int)cl.block_rank();
  extern __shared__ double sm[];
  const int n = a.n, cw = a.cw;
  double* AB = sm;  // [cw][SB2_LDB]
  __shared__ unsigned long long prog[SB2_WARPS];
  __shared__ uint32_t cbase[16], pbase[16];  // shared::cluster addresses of AB / prog in every CTA
  if (threadIdx.x < CS) {
    cbase[threadIdx.x] = dsm_map(AB, threadIdx.x);
    pbase[threadIdx.x] = dsm_map(prog, threadIdx.x);
  }
  if (threadIdx.x < SB2_WARPS) prog[threadIdx.x] = 0ull;
  const int c0 = rank * cw, c1 = min(n, c0 + cw);
  for (int e = threadIdx.x; e < cw * SB2_LDB; e += blockDim.x) {
    const int c = c0 + e / SB2_LDB, dd = e % SB2_LDB;
    AB[e] = (c < n && dd <= SB && c + dd < n) ? a.A[(long)(c + dd) * n + c] : 0.0;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = lane & 15;
  const bool isC = lane < 16;
  const unsigned full = 0xffffffffu;
  const int W = CS * SB2_WARPS, g = rank * SB2_WARPS + warp;
  const int gp = (g + W - 1) % W;  // warp chasing the previous sweep
  cl.sync();
  const uint32_t my_prog = pbase[rank] + (uint32_t)(warp * 8);
  const uint32_t pred_prog = pbase[gp / SB2_WARPS] + (uint32_t)((gp % SB2_WARPS) * 8);
  const bool timing = a.dbg && lane == 0;
  unsigned long long tseg[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tl = timing ? clock64() : 0;
#define SBM(k)                      \
  if (timing) {                     \
    const long long t_ = clock64(); \
    tseg[k] += t_ - tl;             \
    tl = t_;                        \
  }
  for (int i = g; i <= n - 3; i += W) {
    const int tmax = (n - 2 - i) / SB;
    const int tmaxp = (i > 0) ? (n - 1 - i) / SB : 0;  // predecessor's last task
    double vp[16];
    double taup = 0.0;
#pragma unroll
    for (int c = 0; c < 16; ++c) vp[c] = 0.0;
    for (int t = 0; t <= tmax; ++t) {
      // ---- wait for task (i−1, t+1) (or the whole predecessor sweep near the end)
      if (i > 0) {
        const unsigned need = (unsigned)min(t + 2, tmaxp + 1);
        if (lane == 0) {
          while (true) {
            const unsigned long long pv = dsm_ld_acquire_u64(pred_prog);
            const unsigned ps = (unsigned)(pv >> 32), pd = (unsigned)pv;
            if (ps > (unsigned)i || (ps == (unsigned)i && pd >= need)) break;
            __nanosleep(32);  // keep the spinning warps off the issue slots / LSU of the working ones
          }
        }
        __syncwarp();
      }
      SBM(0)
      const int stp = i + 1 + (t - 1) * SB;  // C columns (t ≥ 1)
      const int st = (t == 0) ? i + 1 : stp + SB;
      const int ed = min(st + SB - 1, n - 1), len = ed - st + 1;
      const int R = st + r;
      // a task touches ≤ 32 consecutive band columns: at most two owning CTAs
      const int cfirst = (t == 0) ? i : stp;
      const int o0 = cfirst / cw;
      const int split = (o0 + 1) * cw;
      const uint32_t b0 = cbase[o0] - (uint32_t)(o0 * cw * SB2_LDB * 8);
      const uint32_t b1 = (o0 + 1 < CS) ? cbase[o0 + 1] - (uint32_t)(split * SB2_LDB * 8) : 0u;
      auto ea = [&](int c, int d) -> uint32_t { return (c < split ? b0 : b1) + (uint32_t)((c * SB2_LDB + d) * 8); };
      double row[16];
      double x = 0.0;
      // ---- load
      if (isC) {
        if (t == 0) {
          x = (r < len) ? dsm_ld(ea(i, 1 + r)) : 0.0;
        } else {
#pragma unroll
          for (int c = 0; c < 16; ++c) row[c] = (r < len) ? dsm_ld(ea(stp + c, R - stp - c)) : 0.0;
        }
      } else {
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          double v = 0.0;
          if (r < len && c < len) v = dsm_ld((c <= r) ? ea(st + c, r - c) : ea(R, c - r));
          row[c] = v;
        }
      }
      SBM(1)
      if (t > 0) {  // ---- (1) C ← C H_p
        if (isC && taup != 0.0) {
          double p[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) p[c] = row[c] * vp[c];
          const double u = taup * sum16(p);
#pragma unroll
          for (int c = 0; c < 16; ++c) row[c] -= u * vp[c];
        }
        x = (isC && r < len) ? row[0] : 0.0;
      }
      SBM(2)
      // ---- (2) Householder from x (lanes 0..len−1)
      double tau, beta;
      const double vr = warp_house(isC ? x : 0.0, lane, tau, beta);
      const double vmine = (isC && r < len) ? vr : 0.0;  // lanes ≥ 16 carry 0
      double v[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) v[c] = __shfl_sync(full, vmine, c);
      if (isC && r < len) {
        if (t == 0)
          dsm_st(ea(i, 1 + r), (r == 0) ? beta : 0.0);
        else
          row[0] = (r == 0) ? beta : 0.0;
      }
      SBM(3)
      if (tau != 0.0) {
        // ---- (3) C[:, 1:] ← H C[:, 1:]: column sums y_c = Σ_r v_r C[r][c] by a 16-lane reduce-scatter
        if (t > 0) {
          double vals[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) vals[c] = isC ? vmine * row[c] : 0.0;
#pragma unroll
          for (int off = 8; off >= 1; off >>= 1) {
            const bool up = lane & off;
#pragma unroll
            for (int k = 0; k < off; ++k) {
              const double send = up ? vals[k] : vals[k + off];
              const double keep = up ? vals[k + off] : vals[k];
              vals[k] = keep + __shfl_xor_sync(full, send, off);
            }
          }
          const double ty = tau * vals[0];  // lane c (< 16): τ y_c
#pragma unroll
          for (int c = 1; c < 16; ++c) {
            const double yc = __shfl_sync(full, ty, c);
            if (isC) row[c] -= vmine * yc;
          }
        }
        SBM(4)
        // ---- (4) D ← H D H  (lanes 16..31 own the rows)
        double wr = 0.0;
        if (!isC && r < len) {
          double p[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) p[c] = row[c] * v[c];
          wr = tau * sum16(p);
        }
        const double vme = __shfl_sync(full, vmine, r);  // v_r for the D lanes
        const double wv = warp_sum((!isC && r < len) ? wr * vme : 0.0);
        wr += (-0.5 * tau * wv) * vme;
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const double wc = __shfl_sync(full, wr, 16 + c);
          if (!isC && r < len) row[c] -= vme * wc + wr * v[c];
        }
      }
      SBM(5)
      // ---- store, publish, record
      if (isC) {
        if (t > 0 && r < len) {
#pragma unroll
          for (int c = 0; c < 16; ++c) dsm_st(ea(stp + c, R - stp - c), row[c]);
        }
      } else if (r < len) {
#pragma unroll
        for (int c = 0; c < 16; ++c)
          if (c <= r) dsm_st(ea(st + c, r - c), row[c]);
      }
      __syncwarp();
      if (lane == 0) dsm_st_release_u64(my_prog, ((unsigned long long)(i + 1) << 32) | (unsigned)(t + 1));
      const long qi = q2_index(i, t, a.NT);
      const double vs = (tau != 0.0) ? vmine : 0.0;
      if (isC && r < len) a.Vq2[qi * SB + r] = vs;
      if (lane == 0) a.tq2[qi] = tau;
#pragma unroll
      for (int c = 0; c < 16; ++c) vp[c] = (tau != 0.0) ? v[c] : 0.0;
      taup = tau;
      SBM(6)
    }
  }
  if (timing)
    for (int k = 0; k < 8; ++k) atomicAdd(a.dbg + (rank * 32 + warp) * 8 + k, tseg[k]);
#undef SBM
  cl.sync();
  for (int c = c0 + threadIdx.x; c < c1; c += blockDim.x) {
    const double* cc = AB + (long)(c - c0) * SB2_LDB;
    a.d[c] = cc[0];
    if (c < n - 1) a.e[c] = cc[1];
  }
  cl.sync();
}

static int sb2_cluster(int n) {
  static const int forced = [] {
    const char* e = std::getenv("KOT_SB2_CS");  // diagnostic override
    return e ? std::atoi(e) : 0;
  }();
  if (forced > 0) return std::min(16, forced);
  return std::max(1, std::min(16, (n + 127) / 128));
}

static void sb2st(int n, EigWork& w, cudaStream_t st) {
  const int cs = sb2_cluster(n);
  const int cw = (n + cs - 1) / cs;
  const size_t smem = sizeof(double) * ((size_t)cw * SB2_LDB);
  kot_require(smem <= 220 * 1024, KOT_EINVAL, "matrix order too large for the bulge-chasing cluster");
  ensure_smem_attr((const void*)sb2st_kernel, (int)smem, true);
  const long q2 = two_stage_q2_size(n);
  KOT_CUDA(cudaMemsetAsync(w.Vq2, 0, sizeof(double) * q2, st));
  KOT_CUDA(cudaMemsetAsync(w.tq2, 0, sizeof(double) * (q2 / SB), st));
  Sb2Args args{w.A, n, cw, eig_nt(n), w.d, w.e, w.Vq2, w.tq2, g_sb2_dbg};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs);
  cfg.blockDim = dim3(SB2_NTHREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  KOT_CUDA(cudaLaunchKernelEx(&cfg, sb2st_kernel, args));
  KOT_LAUNCH_CHECK();
}

void two_stage_tridiag(const double* Z, int n, EigWork& w, cudaStream_t st) {
  w.ensure_two_stage();
  {
    ProfScope ps("eig.sy2sb", st, 4.0 / 3.0 * n * (double)n * n);
    sy2sb(Z, n, w, st);
  }
  ProfScope ps("eig.sb2st", st);
  sb2st(n, w, st);
}

// ============================================================== Q2 back-transform

constexpr int QG = 32;                 // sweeps per application group G(I, t)
constexpr int QG_ROWS = QG + SB - 1;   // window rows touched by a group

__host__ __device__ static int q2_ngroups_i(int n) { return (n - 2 + QG - 1) / QG; }
long two_stage_t_size(int n) { return n < 3 ? 1 : (long)q2_ngroups_i(n) * eig_nt(n) * QG * QG; }

// v of stage-2 reflector (i, t) (16 entries, zero-padded)
__device__ __forceinline__ const double* q2_vec(const double* Vq2, int i, int t, int NT) {
  return Vq2 + q2_index(i, t, NT) * SB;
}

// T of each group (forward columnwise, QG reflectors; reflector j on window rows j..j+SB−1).
// One warp per group; T stored row-major QG×QG (upper triangle).
constexpr int QL_WARPS = 2;
__global__ void __launch_bounds__(32 * QL_WARPS) q2_larft_kernel(const double* __restrict__ Vq2,
                                                                 const double* __restrict__ tq2, double* Tq2, int n,
                                                                 int NT, int ngroups) {
  __shared__ double Vs[QL_WARPS][QG][SB + 1];
  __shared__ double Tsh[QL_WARPS][QG][QG + 1];
  __shared__ double sv[QL_WARPS][QG];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x * QL_WARPS + warp;
  if (g >= ngroups) return;
  const int I = g / NT, t = g % NT;
  for (int e = lane; e < QG * SB; e += 32) {
    const int jj = e / SB, q = e % SB, i = I * QG + jj;
    Vs[warp][jj][q] = (i <= n - 3) ? q2_vec(Vq2, i, t, NT)[q] : 0.0;
  }
  const int il = I * QG + lane;
  const double taul = (il <= n - 3) ? tq2[q2_index(il, t, NT)] : 0.0;
  __syncwarp();
  for (int jc = 0; jc < QG; ++jc) {
    double sl = 0.0;  // Σ_rows v_lane · v_jc   (lane < jc; overlap rows jc .. lane+SB−1)
    if (lane < jc)
      for (int row = jc; row <= lane + SB - 1; ++row) sl += Vs[warp][lane][row - lane] * Vs[warp][jc][row - jc];
    sv[warp][lane] = sl;
    __syncwarp();
    const double tj = __shfl_sync(0xffffffffu, taul, jc);
    if (lane < jc) {
      double acc = 0.0;
      for (int mm = lane; mm < jc; ++mm) acc += Tsh[warp][lane][mm] * sv[warp][mm];
      Tsh[warp][lane][jc] = -tj * acc;
    } else {
      Tsh[warp][lane][jc] = (lane == jc) ? tj : 0.0;
    }
    __syncwarp();
  }
  double* out = Tq2 + (long)g * QG * QG;
  for (int e = lane; e < QG * QG; e += 32) out[e] = Tsh[warp][e / QG][e % QG];
}

// One wave of the Q2 back-transform.  Groups G(I, t) with t − I = wave touch
// disjoint row windows (tools/twostage_proto.py: apply_q2_waves), so a wave is a
// batch of independent (I − V T Vᵀ) updates: blockIdx.y picks the group,
// blockIdx.x a 64-column tile of P.  The three products (Y = VᵀW, Y ← T Y,
// W −= V Y) run on the FP64 tensor cores (mma m8n8k4), with K ranges cut to the
// band of V and the upper triangle of T.
constexpr int QW_COLS = 64;
constexpr int QW_TPC = 4;                 // column tiles per CTA (V, T loaded once, W double-buffered)
constexpr int QW_RW = 48;                 // window rows incl. zero padding (≥ QG_ROWS)
constexpr int QW_LDW = QW_COLS + 4;       // stride ≡ 4 (mod 16) doubles
constexpr int QW_LDV = QG + 4;
constexpr int QW_SMEM = (2 * QW_RW * QW_LDW + QW_RW * QW_LDV + QG * QW_LDV + 2 * QG * QW_LDW) * 8;
__global__ void __launch_bounds__(256) q2_wave_kernel(double* P, int n, const double* __restrict__ Vq2,
                                                      const double* __restrict__ Tq2, int NT, int wave, int Ilo,
                                                      int tile0, int tile1, const int* dcols) {
  extern __shared__ double qw[];
  double* Wb = qw;                       // [2][QW_RW][QW_LDW]
  double* Vd = Wb + 2 * QW_RW * QW_LDW;  // [QW_RW][QW_LDV]: Vd[ρ][j] = v_j[ρ − j]
  double* T = Vd + QW_RW * QW_LDV;       // [QG][QW_LDV]
  double* Y = T + QG * QW_LDV;           // [QG][QW_LDW]
  double* Y2 = Y + QG * QW_LDW;          // [QG][QW_LDW]
  const int I = Ilo + blockIdx.y;
  const int t = wave + I;
  const int ilo = I * QG;
  const int r0 = ilo + 1 + t * SB;
  const int nr = min(QG_ROWS, n - r0);
  const int tbeg = tile0 + blockIdx.x * QW_TPC;
  int tend = min(tile1, tbeg + QW_TPC);
  if (dcols) tend = min(tend, (*dcols + QW_COLS - 1) / QW_COLS);  // α-only back-transform
  if (tbeg >= tend) return;
  const int tid = threadIdx.x;
  auto issue = [&](int tile, int buf) {
    const int c0 = tile * QW_COLS, wc = min(QW_COLS, n - c0);
    double* W = Wb + buf * QW_RW * QW_LDW;
    for (int e = tid; e < QW_RW * QW_COLS; e += 256) {
      const int rr = e / QW_COLS, c = e % QW_COLS;
      const bool ok = rr < nr && c < wc;
      cp_async_8(W + rr * QW_LDW + c, ok ? P + (long)(r0 + rr) * n + c0 + c : P, ok ? 8 : 0);
    }
    cp_async_commit();
  };
  if (tbeg < tend) issue(tbeg, 0);
  for (int e = tid; e < QW_RW * QG; e += 256) {
    const int rho = e / QG, jj = e % QG, q = rho - jj, i = ilo + jj;
    Vd[rho * QW_LDV + jj] = (q >= 0 && q < SB && i <= n - 3 && rho < nr) ? __ldg(q2_vec(Vq2, i, t, NT) + q) : 0.0;
  }
  const double* Tg = Tq2 + ((long)I * NT + t) * QG * QG;
  for (int e = tid; e < QG * QG; e += 256) T[(e / QG) * QW_LDV + e % QG] = __ldg(Tg + e);
  const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, tq = lane & 3;
  int buf = 0;
  for (int tile = tbeg; tile < tend; ++tile, buf ^= 1) {
    if (tile + 1 < tend) {
      issue(tile + 1, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* W = Wb + buf * QW_RW * QW_LDW;
    const int c0 = tile * QW_COLS, wc = min(QW_COLS, n - c0);
    {  // ---- Y = Vᵀ W: warp → row tile jt = warp/2, column tiles 4·(warp%2) .. +3
      const int jt = warp >> 1, ct0 = (warp & 1) * 4;
      double acc[4][2] = {};
      const int kb = 8 * jt, ke = min(QW_RW, 8 * jt + 8 + SB - 1);
      for (int k0 = kb; k0 < ke; k0 += 4) {
        const double a = Vd[(k0 + tq) * QW_LDV + jt * 8 + g];
#pragma unroll
        for (int u = 0; u < 4; ++u) dmma(acc[u][0], acc[u][1], a, W[(k0 + tq) * QW_LDW + (ct0 + u) * 8 + g]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        Y[(jt * 8 + g) * QW_LDW + (ct0 + u) * 8 + 2 * tq] = acc[u][0];
        Y[(jt * 8 + g) * QW_LDW + (ct0 + u) * 8 + 2 * tq + 1] = acc[u][1];
      }
    }
    __syncthreads();
    {  // ---- Y2 = T Y  (T upper triangular: K from the row tile on)
      const int jt = warp >> 1, ct0 = (warp & 1) * 4;
      double acc[4][2] = {};
      for (int k0 = 8 * jt; k0 < QG; k0 += 4) {
        const double a = T[(jt * 8 + g) * QW_LDV + k0 + tq];
#pragma unroll
        for (int u = 0; u < 4; ++u) dmma(acc[u][0], acc[u][1], a, Y[(k0 + tq) * QW_LDW + (ct0 + u) * 8 + g]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        Y2[(jt * 8 + g) * QW_LDW + (ct0 + u) * 8 + 2 * tq] = acc[u][0];
        Y2[(jt * 8 + g) * QW_LDW + (ct0 + u) * 8 + 2 * tq + 1] = acc[u][1];
      }
    }
    __syncthreads();
    {  // ---- W −= V Y2: warp → column tile ct = warp, row tiles 0..5 (K = j ∈ [8ρt − SB + 1, 8ρt + 7])
      const int ct = warp;
#pragma unroll
      for (int pt = 0; pt < QW_RW / 8; ++pt) {
        double acc0 = 0.0, acc1 = 0.0;
        const int kb = max(0, (8 * pt - SB + 1) & ~3), ke = min(QG, 8 * pt + 8);
        for (int k0 = kb; k0 < ke; k0 += 4)
          dmma(acc0, acc1, Vd[(pt * 8 + g) * QW_LDV + k0 + tq], Y2[(k0 + tq) * QW_LDW + ct * 8 + g]);
        const int rho = pt * 8 + g, c = ct * 8 + 2 * tq;
        if (rho < nr) {
          if (c < wc) P[(long)(r0 + rho) * n + c0 + c] = W[rho * QW_LDW + c] - acc0;
          if (c + 1 < wc) P[(long)(r0 + rho) * n + c0 + c + 1] = W[rho * QW_LDW + c + 1] - acc1;
        }
      }
    }
    __syncthreads();  // W[buf] and Y/Y2 are rewritten by the next tile
  }
}

void two_stage_q2_apply(int n, EigWork& w, double* P, cudaStream_t st, const int* dcols) {
  if (n < 3) return;
  ProfScope ps("eig.q2", st, 2.0 * n * (double)n * n);
  const int NT = eig_nt(n);
  const int NI = q2_ngroups_i(n);
  const int ng = NI * NT;
  ensure_smem_attr((const void*)q2_wave_kernel, QW_SMEM);
  q2_larft_kernel<<<ceil_div(ng, QL_WARPS), 32 * QL_WARPS, 0, st>>>(w.Vq2, w.tq2, w.Tq2, n, NT, ng);
  KOT_LAUNCH_CHECK();
  // Column batches sized so that the batch's columns of P (n × width doubles) stay resident in
  // L2 across all waves: every wave re-reads the rows it updates, so without batching P streams
  // from HBM once per wave at large ℓ.  Waves t − I = wv; group (I, t) exists for
  // 0 ≤ t ≤ tmax(I) = (n − 2 − I·QG)/SB.
  static const long l2_budget = [] {
    const char* e = std::getenv("KOT_Q2_BATCH_MB");  // diagnostic: column batching of P
    return (e ? std::atol(e) : 4096L) << 20;
  }();
  const int tiles = ceil_div(n, QW_COLS);
  const int btiles = std::max(1, std::min(tiles, (int)(l2_budget / ((long)n * QW_COLS * 8))));
  for (int tb = 0; tb < tiles; tb += btiles) {
    const int nt = std::min(btiles, tiles - tb);
    for (int wv = -(NI - 1); wv <= (n - 2) / SB; ++wv) {
      int Ilo = std::max(0, -wv), Ihi = NI - 1;
      while (Ihi >= Ilo && wv + Ihi > (n - 2 - Ihi * QG) / SB) --Ihi;
      if (Ihi < Ilo) continue;
      dim3 grid(ceil_div(nt, QW_TPC), Ihi - Ilo + 1);
      q2_wave_kernel<<<grid, 256, QW_SMEM, st>>>(P, n, w.Vq2, w.Tq2, NT, wv, Ilo, tb, tb + nt, dcols);
      KOT_LAUNCH_CHECK();
    }
  }
}

}  // namespace kot

extern "C" int kot_debug_sb2st_timing(int on, unsigned long long* out8) {
  using namespace kot;
  if (on) {
    if (!g_sb2_dbg && cudaMalloc(&g_sb2_dbg, 16 * 32 * 8 * sizeof(unsigned long long)) != cudaSuccess) return 6;
    cudaMemset(g_sb2_dbg, 0, 16 * 32 * 8 * sizeof(unsigned long long));
  } else if (g_sb2_dbg) {
    cudaDeviceSynchronize();
    cudaMemcpy(out8, g_sb2_dbg, 16 * 32 * 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    cudaFree(g_sb2_dbg);
    g_sb2_dbg = nullptr;
  }
  return 0;
}

extern "C" int kot_debug_pqr_timing(int on, unsigned long long* out8) {
  using namespace kot;
  if (on) {
    if (!g_pqr_dbg && cudaMalloc(&g_pqr_dbg, 8 * sizeof(unsigned long long)) != cudaSuccess) return 6;
    cudaMemset(g_pqr_dbg, 0, 8 * sizeof(unsigned long long));
  } else if (g_pqr_dbg) {
    cudaDeviceSynchronize();
    cudaMemcpy(out8, g_pqr_dbg, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    cudaFree(g_pqr_dbg);
    g_pqr_dbg = nullptr;
  }
  return 0;
}
