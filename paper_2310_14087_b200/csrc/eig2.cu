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

#include "gemm.cuh"
#include "kernels.cuh"
#include "prof.cuh"

namespace cg = cooperative_groups;

namespace kot {

constexpr int SB = 16;            // band width
constexpr int SB_LDX = 3 * SB;    // stage-1 GEMM operand rows [V | W | V]
constexpr int PQR_THREADS = 256;  // 16 columns × 16 row groups
constexpr int PQR_LD = SB + 1;
constexpr int PQR_MAXCS = 8;
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
// over the CTAs).  Writes R into A, the reflectors (explicit, zero above the
// unit entry, zero column if τ = 0) into Vall (ormtr layout) and Xs, τ, and
// the panel's T (forward, columnwise) into Tp.
__global__ void __launch_bounds__(PQR_THREADS) sy2sb_panel_kernel(double* A, int n, int j, double* Vall,
                                                                  double* tau_out, double* Xs, double* Tp) {
  cg::cluster_group cl = cg::this_cluster();
  const int CS = (int)cl.num_blocks(), rank = (int)cl.block_rank();
  extern __shared__ double P[];  // [rows][PQR_LD]
  __shared__ double red[2][2 * SB];
  __shared__ double tot[SB];
  __shared__ double Ts[SB][SB + 1];
  __shared__ double taus[SB];
  __shared__ double sc[4];
  __shared__ double gath[PQR_MAXCS][2 * SB];
  const int m = n - j - SB;
  const int kb = min(SB, m);
  const int rc = (m + CS - 1) / CS;
  const int lo = rank * rc, hi = min(m, lo + rc);
  const int tid = threadIdx.x, q = tid >> 4, rg = tid & 15;
  const unsigned hmask = 0xffffu << (16 * ((tid >> 4) & 1));
  for (int e = tid; e < (hi - lo) * SB; e += blockDim.x) {
    const int rr = e / SB, cc = e % SB;
    P[rr * PQR_LD + cc] = A[(long)(j + SB + lo + rr) * n + j + cc];
  }
  for (int e = tid; e < SB * (SB + 1); e += blockDim.x) (&Ts[0][0])[e] = 0.0;
  if (tid < SB) taus[tid] = 0.0;
  __syncthreads();
  int par = 0;
  for (int k = 0; k < kb; ++k) {
    // ---- (a) ‖x[1:]‖² and α = P[k][k] (owner only; the others add zeros)
    if (q == k) {
      double s = 0.0;
      for (int r = lo + rg; r < hi; r += 16)
        if (r > k) {
          const double x = P[(r - lo) * PQR_LD + k];
          s += x * x;
        }
      s = half_sum(s, hmask);
      if (rg == 0) {
        red[par][0] = s;
        red[par][1] = (k >= lo && k < hi) ? P[(k - lo) * PQR_LD + k] : 0.0;
      }
    }
    cl.sync();
    if (tid < 32) {  // fixed-order gather over the cluster: identical on every CTA
      double xn = 0.0, al = 0.0;
      if (tid < CS) {
        const double* rr = cl.map_shared_rank(&red[par][0], tid);
        xn = rr[0];
        al = rr[1];
      }
      if (tid < CS) {
        gath[tid][0] = xn;
        gath[tid][1] = al;
      }
      __syncwarp();
      if (tid == 0) {
        double xn2 = 0.0, alpha = 0.0;
        for (int c = 0; c < CS; ++c) {
          xn2 += gath[c][0];
          alpha += gath[c][1];
        }
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
        sc[0] = tau;
        sc[1] = beta;
        sc[2] = scale;
        taus[k] = tau;
      }
    }
    __syncthreads();
    par ^= 1;
    const double tau = sc[0], beta = sc[1], scale = sc[2];
    // ---- (b) v = x / (α − β) below the diagonal, β on it
    for (int r = lo + tid; r < hi; r += blockDim.x) {
      if (r > k) P[(r - lo) * PQR_LD + k] *= scale;
      if (r == k) P[(r - lo) * PQR_LD + k] = beta;
    }
    __syncthreads();
    // ---- (c) s_q = Σ_{r ≥ k} v_r P[r][q]  (q > k: reflector applied to column q; q < k: T column)
    {
      double s = 0.0;
      if (q != k)
        for (int r = lo + rg; r < hi; r += 16)
          if (r >= k) {
            const double v = (r == k) ? 1.0 : P[(r - lo) * PQR_LD + k];
            s += v * P[(r - lo) * PQR_LD + q];
          }
      s = half_sum(s, hmask);
      if (rg == 0) red[par][q] = s;
    }
    cl.sync();
    for (int e = tid; e < CS * SB; e += blockDim.x) {
      const int c = e / SB, qq = e % SB;
      gath[c][qq] = cl.map_shared_rank(&red[par][0], c)[qq];
    }
    __syncthreads();
    if (tid < SB) {
      double s = 0.0;
      for (int c = 0; c < CS; ++c) s += gath[c][tid];
      tot[tid] = s;
    }
    __syncthreads();
    par ^= 1;
    // ---- (d) P[:, q>k] −= τ v s_qᵀ;  T[0:k, k] = −τ T[0:k,0:k] s[0:k];  T[k][k] = τ
    if (tau != 0.0)
      for (int e = tid; e < (hi - lo) * SB; e += blockDim.x) {
        const int rr = e / SB, cc = e % SB, r = lo + rr;
        if (cc > k && r >= k) {
          const double v = (r == k) ? 1.0 : P[rr * PQR_LD + k];
          P[rr * PQR_LD + cc] -= tau * v * tot[cc];
        }
      }
    if (tid < k) {
      double s = 0.0;
      for (int l = tid; l < k; ++l) s += Ts[tid][l] * tot[l];
      Ts[tid][k] = -tau * s;
    }
    if (tid == k) Ts[k][k] = tau;
    __syncthreads();
  }
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
  cl.sync();  // no CTA leaves while others may still read its red[]
}

// W = Xw T − ½ V M with M = Tᵀ (Vᵀ Xw) T; Xw (rows r0.., cols SB..2SB of Xs) is overwritten by W.
__global__ void __launch_bounds__(256) sy2sb_w_kernel(double* Xs, int r0, int m, const double* Tp, const double* S) {
  __shared__ double T[SB][SB + 1], TS[SB][SB + 1], M[SB][SB + 1];
  __shared__ double xw[16][SB + 1], vv[16][SB + 1];
  const int tid = threadIdx.x, a = tid >> 4, c = tid & 15;
  T[a][c] = Tp[a * SB + c];
  __syncthreads();
  {
    double s = 0.0;
    for (int k = 0; k < SB; ++k) s += T[k][a] * S[k * SB + c];
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
      xw[a][c] = Xs[(long)(r0 + r) * SB_LDX + SB + c];
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

static int pqr_cluster(int m) { return std::max(1, std::min(PQR_MAXCS, (m + 255) / 256)); }

static void sy2sb(const double* Z, int n, EigWork& w, cudaStream_t st) {
  KOT_CUDA(cudaMemcpyAsync(w.A, Z, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, st));
  KOT_CUDA(cudaMemsetAsync(w.Vall, 0, sizeof(double) * n * n, st));
  KOT_CUDA(cudaMemsetAsync(w.tau, 0, sizeof(double) * n, st));
  double* Xs = w.X;      // n × SB_LDX
  double* Tp = w.Tf;     // SB × SB
  double* S = w.Tf + SB * SB;
  static int smem_set = 0;
  for (int j = 0; j + SB + 1 < n; j += SB) {
    const int m = n - j - SB;
    const int cs = pqr_cluster(m);
    kot_require(cs <= PQR_MAXCS, KOT_EINVAL, "matrix order too large for the band reduction");
    const int rows = (m + cs - 1) / cs;
    const size_t smem = sizeof(double) * std::max(rows, 1) * PQR_LD;
    if ((int)smem > smem_set) {
      KOT_CUDA(cudaFuncSetAttribute(sy2sb_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      smem_set = (int)smem;
    }
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
      KOT_CUDA(cudaLaunchKernelEx(&cfg, sy2sb_panel_kernel, w.A, n, j, w.Vall, w.tau, Xs, Tp));
      KOT_LAUNCH_CHECK();
    }
    const int r0 = j + SB;
    double* A22 = w.A + (long)r0 * n + r0;
    double* X0 = Xs + (long)r0 * SB_LDX;
    {  // Xw = A22 V
      GemmShape s = make_shape(m, SB, m, A22, n, X0, SB_LDX);
      s.ws = w.splitws;
      s.ksplit = choose_ksplit(s, w.splitws_cap);
      gemm_launch<false, false>(s, EpiAxpby{X0 + SB, SB_LDX, 1.0, 0.0}, st);
    }
    {  // S = Vᵀ Xw
      GemmShape s = make_shape(SB, SB, m, X0, SB_LDX, X0 + SB, SB_LDX);
      s.ws = w.splitws;
      s.ksplit = choose_ksplit(s, w.splitws_cap);
      gemm_launch<true, false>(s, EpiAxpby{S, SB, 1.0, 0.0}, st);
    }
    sy2sb_w_kernel<<<std::min(ceil_div(m, 16), 2 * kNumSMs), 256, 0, st>>>(Xs, r0, m, Tp, S);
    KOT_LAUNCH_CHECK();
    {  // A22 −= V Wᵀ + W Vᵀ  (one triangle + mirror)
      GemmShape s = make_shape(m, m, 2 * SB, X0, SB_LDX, X0 + SB, SB_LDX);
      s.sym_tiles = 1;
      gemm_launch<false, true>(s, EpiSymMirror{A22, n, -1.0, A22, 1.0, 0.0}, st);
    }
  }
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
    beta = -copysign(hypot(alpha, sqrt(s)), alpha);
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
constexpr int SB2_SLOT = SB + 1;  // v[16], τ
constexpr int SB2_NSLOT = 64;     // slots per step parity, keyed by t mod 64

__device__ __forceinline__ double sum16(const double (&p)[16]) {
  return ((((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]))) +
          (((p[8] + p[9]) + (p[10] + p[11])) + ((p[12] + p[13]) + (p[14] + p[15]))));
}

// Bulge chasing, one warp per task.  Lanes 0–15 hold the rows of the off-diagonal
// block C (or, for t = 0, the column being annihilated), lanes 16–31 the rows of
// the symmetric diagonal block D, all in registers.  The reflector of task
// (i, t−1), needed by (i, t) one step later, is handed over through a DSMEM slot
// of the producing CTA (slot [s & 1][t & 63]: within a CTA the live t's span < 64).
__global__ void __launch_bounds__(SB2_NTHREADS, 1) sb2st_kernel(Sb2Args a) {
  cg::cluster_group cl = cg::this_cluster();
  const int CS = (int)cl.num_blocks(), rank = (int)cl.block_rank();
  extern __shared__ double sm[];
  const int n = a.n, cw = a.cw;
  double* AB = sm;                                // [cw][SB2_LDB]
  double* slots = sm + (long)cw * SB2_LDB;        // [2][SB2_NSLOT][SB2_SLOT]
  __shared__ uint32_t cbase[16], sbase[16];  // shared::cluster addresses of AB / slots in every CTA
  if (threadIdx.x < CS) {
    cbase[threadIdx.x] = dsm_map(AB, threadIdx.x);
    sbase[threadIdx.x] = dsm_map(slots, threadIdx.x);
  }
  const int c0 = rank * cw, c1 = min(n, c0 + cw);
  for (int e = threadIdx.x; e < cw * SB2_LDB; e += blockDim.x) {
    const int c = c0 + e / SB2_LDB, dd = e % SB2_LDB;
    AB[e] = (c < n && dd <= SB && c + dd < n) ? a.A[(long)(c + dd) * n + c] : 0.0;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = lane & 15;
  const bool isC = lane < 16;
  const unsigned full = 0xffffffffu;
  cl.sync();

  const int smax = 2 * n - 6;
  const bool timing = a.dbg && (threadIdx.x & 31) == 0;
  unsigned long long tseg[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tl = timing ? clock64() : 0;
#define SBM(k)                        \
  if (timing) {                       \
    const long long t_ = clock64();   \
    tseg[k] += t_ - tl;               \
    tl = t_;                          \
  }
  for (int s = 0; s <= smax; ++s) {
    // tasks whose anchor column lies in [c0, c1): t = 0 (anchor i) and t ≥ 1 (anchor i + 1 + (t−1)·SB)
    const bool has0 = !(s & 1) && s / 2 <= n - 3 && s / 2 >= c0 && s / 2 < c1;
    int tlo = max(max(1, s - 2 * (n - 3)), cdiv(2 * c0 - s - 2 + 2 * SB, 2 * SB - 1));
    int thi = min(min(s, fdiv(2 * n - 4 - s, 2 * SB - 1)), fdiv(2 * c1 - s - 3 + 2 * SB, 2 * SB - 1));
    if ((tlo & 1) != (s & 1)) ++tlo;
    if ((thi & 1) != (s & 1)) --thi;
    const int ntask = (thi >= tlo ? (thi - tlo) / 2 + 1 : 0) + (has0 ? 1 : 0);
    for (int idx = warp; idx < ntask; idx += SB2_WARPS) {
      int i, t;
      if (has0 && idx == 0) {
        t = 0;
        i = s / 2;
      } else {
        t = tlo + 2 * (idx - (has0 ? 1 : 0));
        i = (s - t) / 2;
      }
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
      // shared::cluster address of band element (column c, d = row − c)
      auto ea = [&](int c, int d) -> uint32_t { return (c < split ? b0 : b1) + (uint32_t)((c * SB2_LDB + d) * 8); };
      double row[16];
      double x = 0.0;
      SBM(0)
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
      if (t > 0) {
        // ---- (1) C ← C H_p  with the reflector of (i, t−1) from its producer's slot
        const int pa = (t == 1) ? i : i + 1 + (t - 2) * SB;
        const uint32_t ps =
            sbase[pa / cw] + (uint32_t)(((((s - 1) & 1) * SB2_NSLOT + ((t - 1) & (SB2_NSLOT - 1))) * SB2_SLOT) * 8);
        double vp[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) vp[c] = dsm_ld(ps + 8 * c);
        const double taup = dsm_ld(ps + 8 * SB);
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
      // ---- store
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
      // ---- hand the reflector to (i, t+1) and record it for the back-transform
      double* slot = slots + (((s & 1) * SB2_NSLOT + (t & (SB2_NSLOT - 1))) * SB2_SLOT);
      const long qi = q2_index(i, t, a.NT);
      if (isC) {
        const double vs = (tau != 0.0) ? vmine : 0.0;
        slot[r] = vs;
        if (r < len) a.Vq2[qi * SB + r] = vs;
        if (r == 0) {
          slot[SB] = tau;
          a.tq2[qi] = tau;
        }
      }
      SBM(6)
    }
    SBM(0)
    cl.sync();
    SBM(7)
  }
  if (timing)
    for (int k = 0; k < 8; ++k) atomicAdd(a.dbg + (rank * SB2_WARPS + warp) * 8 + k, tseg[k]);
#undef SBM
  for (int c = c0 + threadIdx.x; c < c1; c += blockDim.x) {
    const double* cc = AB + (long)(c - c0) * SB2_LDB;
    a.d[c] = cc[0];
    if (c < n - 1) a.e[c] = cc[1];
  }
  cl.sync();
}

static int sb2_cluster(int n) { return std::max(1, std::min(16, (n + 127) / 128)); }

static void sb2st(int n, EigWork& w, cudaStream_t st) {
  const int cs = sb2_cluster(n);
  const int cw = (n + cs - 1) / cs;
  const size_t smem = sizeof(double) * ((size_t)cw * SB2_LDB + 2 * SB2_NSLOT * SB2_SLOT);
  kot_require(smem <= 220 * 1024, KOT_EINVAL, "matrix order too large for the bulge-chasing cluster");
  static size_t smem_set = 0;
  if (smem > smem_set) {
    KOT_CUDA(cudaFuncSetAttribute(sb2st_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    KOT_CUDA(cudaFuncSetAttribute(sb2st_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    smem_set = smem;
  }
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
// blockIdx.x a 64-column tile of P.
constexpr int QW_COLS = 64;
constexpr int QW_LD = QW_COLS + 1;
constexpr int QW_SMEM = QG_ROWS * QW_LD * 8;
__global__ void __launch_bounds__(256) q2_wave_kernel(double* P, int n, const double* __restrict__ Vq2,
                                                      const double* __restrict__ Tq2, int NT, int wave, int Ilo) {
  extern __shared__ double qw_dyn[];
  double (*W)[QW_LD] = reinterpret_cast<double (*)[QW_LD]>(qw_dyn);  // [QG_ROWS][QW_LD]
  __shared__ double Y[QG][QW_LD];
  __shared__ double Vw[QG][SB + 1];
  __shared__ double T[QG][QG + 1];
  const int I = Ilo + blockIdx.y;
  const int t = wave + I;
  const int ilo = I * QG;
  const int r0 = ilo + 1 + t * SB;
  const int nr = min(QG_ROWS, n - r0);
  const int c0 = blockIdx.x * QW_COLS;
  const int wc = min(QW_COLS, n - c0);
  const int tid = threadIdx.x;
  for (int e = tid; e < nr * QW_COLS; e += 256) {
    const int rr = e / QW_COLS, c = e % QW_COLS;
    W[rr][c] = (c < wc) ? P[(long)(r0 + rr) * n + c0 + c] : 0.0;
  }
  for (int e = tid; e < QG * SB; e += 256) {
    const int jj = e / SB, q = e % SB, i = ilo + jj;
    Vw[jj][q] = (i <= n - 3) ? __ldg(q2_vec(Vq2, i, t, NT) + q) : 0.0;
  }
  const double* Tg = Tq2 + ((long)I * NT + t) * QG * QG;
  for (int e = tid; e < QG * QG; e += 256) T[e / QG][e % QG] = __ldg(Tg + e);
  __syncthreads();
  // thread → (row j, columns cb + 8u): lanes of a warp read consecutive doubles
  const int jj = tid >> 3, cb = tid & 7;
  // Y = Vᵀ W
  {
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int q = 0; q < SB && jj + q < nr; ++q) {
      const double v = Vw[jj][q];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[u] += v * W[jj + q][cb + 8 * u];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) Y[jj][cb + 8 * u] = acc[u];
  }
  __syncthreads();
  // Y ← T Y (upper triangular)
  {
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int l = jj; l < QG; ++l) {
      const double tv = T[jj][l];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[u] += tv * Y[l][cb + 8 * u];
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 8; ++u) Y[jj][cb + 8 * u] = acc[u];
  }
  __syncthreads();
  // W −= V Y: row ρ gets Σ_{j ∈ [ρ−SB+1, ρ]} v_j[ρ − j] Y[j]
  for (int e = tid; e < nr * 8; e += 256) {
    const int rho = e >> 3, cc = e & 7;
    const int jlo = max(0, rho - SB + 1), jhi = min(QG - 1, rho);
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int j = jlo; j <= jhi; ++j) {
      const double v = Vw[j][rho - j];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[u] += v * Y[j][cc + 8 * u];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (cc + 8 * u < wc) P[(long)(r0 + rho) * n + c0 + cc + 8 * u] = W[rho][cc + 8 * u] - acc[u];
  }
}

void two_stage_q2_apply(int n, EigWork& w, double* P, cudaStream_t st) {
  if (n < 3) return;
  ProfScope ps("eig.q2", st, 2.0 * n * (double)n * n);
  const int NT = eig_nt(n);
  const int NI = q2_ngroups_i(n);
  const int ng = NI * NT;
  static bool attr = false;
  if (!attr) {
    KOT_CUDA(cudaFuncSetAttribute(q2_wave_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, QW_SMEM));
    attr = true;
  }
  q2_larft_kernel<<<ceil_div(ng, QL_WARPS), 32 * QL_WARPS, 0, st>>>(w.Vq2, w.tq2, w.Tq2, n, NT, ng);
  KOT_LAUNCH_CHECK();
  // waves t − I = wv; group (I, t) exists for 0 ≤ t ≤ tmax(I) = (n − 2 − I·QG)/SB
  for (int wv = -(NI - 1); wv <= (n - 2) / SB; ++wv) {
    int Ilo = std::max(0, -wv), Ihi = NI - 1;
    while (Ihi >= Ilo && wv + Ihi > (n - 2 - Ihi * QG) / SB) --Ihi;
    if (Ihi < Ilo) continue;
    dim3 grid(ceil_div(n, QW_COLS), Ihi - Ilo + 1);
    q2_wave_kernel<<<grid, 256, QW_SMEM, st>>>(P, n, w.Vq2, w.Tq2, NT, wv, Ilo);
    KOT_LAUNCH_CHECK();
  }
}

}  // namespace kot

extern "C" int kot_debug_sb2st_timing(int on, unsigned long long* out8) {
  using namespace kot;
  if (on) {
    if (!g_sb2_dbg && cudaMalloc(&g_sb2_dbg, 16 * 8 * 8 * sizeof(unsigned long long)) != cudaSuccess) return 6;
    cudaMemset(g_sb2_dbg, 0, 16 * 8 * 8 * sizeof(unsigned long long));
  } else if (g_sb2_dbg) {
    cudaDeviceSynchronize();
    cudaMemcpy(out8, g_sb2_dbg, 16 * 8 * 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    cudaFree(g_sb2_dbg);
    g_sb2_dbg = nullptr;
  }
  return 0;
}
