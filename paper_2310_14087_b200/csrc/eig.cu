// Hand-written FP64 symmetric eigensolver for the PSD-cone projection
// (north-star item 4; replaces np.linalg.eigh / LAPACK dsyevd called from
// reference linalg.py:60-83, four times per SSN iteration).
//
//   1. sytrd  — blocked Householder tridiagonalisation (LAPACK dlatrd
//      structure, lower).  Each NB=32 panel runs as ONE cooperative
//      persistent kernel (2 grid barriers per column: column update |
//      Householder + symv), followed by the DMMA core for the trailing
//      symmetric rank-2NB update (one triangle + mirror).
//   2. stedc  — tridiagonal divide & conquer: leaves (≤32) by implicit QL
//      in one warp each; merges by deflation (dlaed2 rules), a warp-per-root
//      secular-equation solver (middle-way rational steps inside a bisection
//      bracket, roots stored as pole-origin + offset so d_i − λ_j is exact),
//      Gu–Eisenstat recomputation of z for orthogonal eigenvectors, and the
//      eigenvector update as a DMMA GEMM with a column-scatter epilogue.
//   3. ormtr  — back-transform P = Q_H·Q_T with compact-WY blocks
//      (I − V T Vᵀ), two DMMA GEMMs per block (V·T formed beside the D&C).
//   4. descending order + k = #(σ > 0)  (strict, zero → ᾱ, linalg.py:74-83).
// Consumers (proj, 𝒯, M) are basis-invariant, so eigenvector signs and the
// basis inside clusters may differ from LAPACK.
#include <cooperative_groups.h>

#include <algorithm>
#include <atomic>
#include <cfloat>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <vector>

#include "gemm.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace kot {

constexpr int TRD_NB = 32;
constexpr int TRD_THREADS = 256;
constexpr int TRD_WARPS = TRD_THREADS / 32;
constexpr int TRD_PSTRIDE = 2 * TRD_NB + 2;
constexpr int TRD_GRP = 8;
constexpr int TRD_NGRP = (kNumSMs + TRD_GRP - 1) / TRD_GRP;
constexpr int DC_LEAF = 32;
constexpr double DEPS = DBL_EPSILON * 0.5;  // LAPACK dlamch('E')

// ============================================================== workspace

EigWork::EigWork(int n_) : n(n_) {
  const long nn = (long)n * n;
  auto alloc = [&](double** p, long cnt) { *p = static_cast<double*>(dev_alloc(std::max(cnt, 1L) * sizeof(double))); };
  alloc(&A, nn);
  alloc(&Vall, nn);
  alloc(&X, (long)n * 3 * TRD_NB);
  alloc(&d, n);
  alloc(&e, n);
  alloc(&tau, n);
  alloc(&xv, n);
  alloc(&yv, n);
  alloc(&part, (long)kNumSMs * TRD_PSTRIDE);
  alloc(&partn, kNumSMs);
  alloc(&gpart, (long)TRD_PSTRIDE * TRD_NGRP);
  gcnt = static_cast<int*>(dev_alloc(sizeof(int) * TRD_NGRP));
  alloc(&Tf, 256L * 256 * 2);
  alloc(&W1, 256L * n * 2);
  splitws_cap = 16L * 256 * n;
  alloc(&splitws, splitws_cap);
  alloc(&Q, nn);
  alloc(&Qw, nn + 2L * n + 8);
  alloc(&Qnd, nn + 2L * n + 8);
  alloc(&Dl, nn + 2L * n + 8);
  alloc(&Uw, nn + 2L * n + 8);
  alloc(&zs, n);
  alloc(&ds, n);
  alloc(&dlam, n);
  alloc(&wv, n);
  alloc(&what, n);
  alloc(&lam, n);
  alloc(&dfv, n);
  alloc(&rotcs, 2L * n);
  alloc(&rho, n + 1);  // merge ρ's, then the tridiagonal's max norm at [n]
  ibuf = static_cast<int*>(dev_alloc(sizeof(int) * (8L * n + 64)));
  dbuf = dev_alloc(16L * n + 4096 + 64L * n);
  hbuf = static_cast<int*>(host_alloc_pinned(sizeof(int) * (12L * n + 512)));
}

// two-stage buffers on first use (the default one-stage path never touches them)
void EigWork::ensure_two_stage() {
  if (Vq2 || n < 3) return;
  auto alloc = [&](double** p, long cnt) { *p = static_cast<double*>(dev_alloc(std::max(cnt, 1L) * sizeof(double))); };
  const long q2 = two_stage_q2_size(n);
  alloc(&Vq2, q2);
  alloc(&Tq2, two_stage_t_size(n));
  alloc(&tq2, q2 / 16);
  KOT_CUDA(cudaStreamCreateWithFlags(&st2, cudaStreamNonBlocking));
  KOT_CUDA(cudaEventCreateWithFlags(&ev_w, cudaEventDisableTiming));
  KOT_CUDA(cudaEventCreateWithFlags(&ev_rest, cudaEventDisableTiming));
}

void EigWork::ensure_panel_events() {
  if (ev_panel[0]) return;
  for (auto& e : ev_panel) KOT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
}

void EigWork::ensure_tfactors() {
  if (Tall) return;
  const int nblk = std::max(1, (n - 1 + 127) / 128);
  Tall = static_cast<double*>(dev_alloc(sizeof(double) * 128L * 128 * nblk));
  Sside = static_cast<double*>(dev_alloc(sizeof(double) * 128L * 128));
  VT = static_cast<double*>(dev_alloc(sizeof(double) * (long)n * n));
  ws_t = static_cast<double*>(dev_alloc(sizeof(double) * 16L * 128 * 128));
  int lo = 0, hi = 0;
  KOT_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  KOT_CUDA(cudaStreamCreateWithPriority(&st_t, cudaStreamNonBlocking, hi));
  KOT_CUDA(cudaEventCreateWithFlags(&ev_t0, cudaEventDisableTiming));
  KOT_CUDA(cudaEventCreateWithFlags(&ev_t1, cudaEventDisableTiming));
}

EigWork::~EigWork() {
  for (double* p : {A, Vall, X, d, e, tau, xv, yv, part, partn, Tf, W1, Q, Qw, Qnd, Dl, Uw, zs, ds, dlam, wv, what, lam,
                    dfv, rotcs, rho, splitws, gpart, Vq2, Tq2, tq2})
    dev_free(p);
  if (st2) {
    cudaStreamSynchronize(st2);
    cudaStreamDestroy(st2);
  }
  if (st_t) {
    cudaStreamSynchronize(st_t);
    cudaStreamDestroy(st_t);
  }
  for (auto e : ev_panel)
    if (e) cudaEventDestroy(e);
  if (ev_t0) cudaEventDestroy(ev_t0);
  if (ev_t1) cudaEventDestroy(ev_t1);
  for (double* q : {Tall, Sside, ws_t, VT}) dev_free(q);
  if (ev_w) cudaEventDestroy(ev_w);
  if (ev_rest) cudaEventDestroy(ev_rest);
  dev_free(gcnt);
  dev_free(mid_x);
  dev_free(mid_err);
  if (mid_err_host) host_free_pinned(mid_err_host, 2 * sizeof(int));
  dev_free(ibuf);
  dev_free(dbuf);
  host_free_pinned(hbuf, sizeof(int) * (12L * n + 512));
}

// ================================================================= sytrd

struct TrdArgs {
  double* A;
  int n, p0, nb;
  double* X;  // n × 3NB : [V | W | V]
  double* Vall;
  double* d;
  double* e;
  double* tau;
  double* xv;
  double* yv;
  double* part;   // [TRD_PSTRIDE][kNumSMs]: t1[NB], t2[NB], yvv per CTA (transposed: coalesced reduction)
  double* partn;  // [G]: Σ x_r², r >= c+2
  unsigned long long* dbg;  // nullable: per-segment ns accumulated by CTA 0 thread 0
  double* gpart;  // [TRD_PSTRIDE][TRD_NGRP]: per-group sums of the CTA partials
  int* gcnt;      // [TRD_NGRP] arrival counters (self-resetting)
};


__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// dlarfg scalars from α and Σx² (the part of the column below α): β = −sign(α)‖(α, x)‖,
// τ = (β − α)/β = 1 + |α|/‖·‖, 1/(α − β) = sign(α)/(|α| + ‖·‖).  Far from over/underflow the norm comes
// straight from the sum of squares with hardware rsqrt / reciprocal seeds and Newton steps — a short
// dependent chain (FP64 sqrt, hypot and two divisions cost ≈ 1 µs when a whole CTA waits for one
// thread, or when every thread runs them); dlapy2 otherwise.  Results within an ulp or two of dlarfg's.
__device__ __forceinline__ void dlarfg_scalars(double alpha, double xn2, double& beta, double& tau, double& scale) {
  if (xn2 == 0.0) {  // H = I
    tau = 0.0;
    beta = alpha;
    scale = 1.0;
    return;
  }
  const double s2 = fma(alpha, alpha, xn2), aa = fabs(alpha);
  double nrm, rn, rd;
  if (s2 > 1e-280 && s2 < 1e280) {
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(rn) : "d"(s2));
    const double hs = 0.5 * s2;
    rn = rn * fma(-hs * rn, rn, 1.5);
    rn = rn * fma(-hs * rn, rn, 1.5);
    nrm = s2 * rn;
    nrm = fma(0.5 * rn, fma(-nrm, nrm, s2), nrm);
    rn = fma(rn, fma(-nrm, rn, 1.0), rn);
    const double dsum = aa + nrm;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rd) : "d"(dsum));
    rd = fma(rd, fma(-dsum, rd, 1.0), rd);
    rd = fma(rd, fma(-dsum, rd, 1.0), rd);
    rd = fma(rd, fma(-dsum, rd, 1.0), rd);
  } else {
    nrm = hypot(alpha, sqrt(xn2));
    rn = 1.0 / nrm;
    rd = 1.0 / (aa + nrm);
  }
  beta = -copysign(nrm, alpha);
  tau = fma(aa, rn, 1.0);
  scale = copysign(rd, alpha);
}

// One cooperative launch per NB=32 panel.  Each warp owns up to TRD_RPW rows
// (r ≡ global-warp-id mod #warps, r ≥ p0); their V/W panel rows and the panel
// columns of A live in shared memory for the whole panel, the symv results in
// registers, so a column costs ~4 dependent global round trips + 2 grid
// barriers.  V/W are also written to global (X = [V | W | V]) for the trailing
// rank-2NB update and for the other CTAs (row c of V/W).
constexpr int TRD_RPW = 8;  // rows per warp: n ≤ TRD_RPW · 8 · 148 = 9472

__global__ void __launch_bounds__(TRD_THREADS, 2) sytrd_panel_kernel(TrdArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double dsm[];
  // dynamic smem: [Vs | Ws | Ac] (TRD_WARPS × TRD_RPW × NB each) then the Householder vector (n)
  typedef double RowBlk[TRD_RPW][TRD_NB];
  RowBlk* Vs = reinterpret_cast<RowBlk*>(dsm);
  RowBlk* Ws = Vs + TRD_WARPS;
  RowBlk* Ac = Ws + TRD_WARPS;
  double* vsh = reinterpret_cast<double*>(Ac + TRD_WARPS);
  __shared__ double sred[TRD_WARPS][TRD_PSTRIDE];
  __shared__ double tred[TRD_PSTRIDE];
  __shared__ double wrow[TRD_NB], vrow[TRD_NB];
  __shared__ double nrm_sh[TRD_WARPS];
  __shared__ double scal_sh[2];

  const int n = a.n, p0 = a.p0, nb = a.nb;
  const int G = gridDim.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int gw = blockIdx.x * TRD_WARPS + wid;
  const int NW = G * TRD_WARPS;
  constexpr int LDX = 3 * TRD_NB;
  double* V = a.X;
  double* Wm = a.X + TRD_NB;
  double* V2 = a.X + 2 * TRD_NB;
  // own rows: rbase + q·NW, q < TRD_RPW
  const int rbase = p0 + ((gw - p0) % NW + NW) % NW;
  double yreg[TRD_RPW];
#pragma unroll
  for (int q = 0; q < TRD_RPW; ++q) {
    const int r = rbase + q * NW;
    Vs[wid][q][lane] = 0.0;
    Ws[wid][q][lane] = 0.0;
    Ac[wid][q][lane] = (r < n && lane < nb) ? a.A[(long)r * n + p0 + lane] : 0.0;
    yreg[q] = 0.0;
  }
  __syncwarp();
  double tau_prev = 0.0;
  const bool timing = (a.dbg != nullptr) && blockIdx.x == 0 && threadIdx.x == 0;
  unsigned long long tseg[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long tl = timing ? gtimer() : 0;
#define TRD_MARK(i)                   \
  if (timing) {                       \
    const unsigned long long t_ = gtimer(); \
    tseg[i] += t_ - tl;               \
    tl = t_;                          \
  }

  for (int jj = 0; jj <= nb; ++jj) {
    const int c = p0 + jj;
    // ------------------------------------------------------------ phase Q
    if (jj > 0) {
      const int m = jj - 1;  // t-range of the previous column's corrections
      // prefetch row c of V/W (owned elsewhere) while the partials are reduced
      double pv = 0.0, pw = 0.0, pyc = 0.0;
      if (wid == TRD_WARPS - 1 && jj < nb) {
        if (lane < jj) pv = __ldcg(V + (long)c * LDX + lane);
        if (lane < m) pw = __ldcg(Wm + (long)c * LDX + lane);
        pyc = __ldcg(a.yv + c);
      }
      if (wid < TRD_WARPS - 1) {  // TRD_WARPS−1 warps share the partial columns; every load issued up front
        constexpr int QPW = (2 * TRD_NB + 1 + TRD_WARPS - 2) / (TRD_WARPS - 1);
        constexpr int GPL = (kNumSMs + 31) / 32;  // partials per lane (G ≤ 148)
        double sq[QPW];
#pragma unroll
        for (int i = 0; i < QPW; ++i) {
          const int q = wid + i * (TRD_WARPS - 1);
          const bool need = q <= 2 * TRD_NB && (q < m || (q >= TRD_NB && q < TRD_NB + m) || q == 2 * TRD_NB);
          double v[GPL];
#pragma unroll
          for (int u = 0; u < GPL; ++u) {
            const int g = lane + 32 * u;
            v[u] = (need && g < G) ? __ldcg(a.part + (long)q * kNumSMs + g) : 0.0;
          }
          double s = 0.0;
#pragma unroll
          for (int u = 0; u < GPL; ++u) s += v[u];
          sq[i] = s;
        }
#pragma unroll
        for (int i = 0; i < QPW; ++i) {
          const int q = wid + i * (TRD_WARPS - 1);
          const double s = warp_sum(sq[i]);
          if (lane == 0 && q <= 2 * TRD_NB) tred[q] = s;
        }
      }
      if (wid == TRD_WARPS - 1 && jj < nb) {
        vrow[lane] = pv;
        if (lane < m) wrow[lane] = pw;
      }
      __syncthreads();
      TRD_MARK(0)
      const double t1l = (lane < m) ? tred[lane] : 0.0, t2l = (lane < m) ? tred[TRD_NB + lane] : 0.0;
      const double t12 = warp_sum(t1l * t2l);
      // α = −½ τ (wᵀv),  wᵀv = τ (yᵀv − 2 t1·t2)
      const double alpha_prev = -0.5 * tau_prev * (tau_prev * (tred[2 * TRD_NB] - 2.0 * t12));
      // finish W[:, jj-1] for own rows r >= c: w_r = τ (y_r − V_r·t1 − W_r·t2) + α v_r
#pragma unroll
      for (int q = 0; q < TRD_RPW; ++q) {
        const int r = rbase + q * NW;
        if (r < c || r >= n) continue;
        double s = Vs[wid][q][lane] * t1l + Ws[wid][q][lane] * t2l;
        s = warp_sum(s);
        const double w = tau_prev * (yreg[q] - s) + alpha_prev * Vs[wid][q][jj - 1];
        if (lane == 0) {
          Ws[wid][q][jj - 1] = w;
          Wm[(long)r * LDX + jj - 1] = w;
        }
      }
      if (wid == TRD_WARPS - 1 && jj < nb) {  // row c, redundantly (identical arithmetic to its owner)
        double s = ((lane < m) ? vrow[lane] : 0.0) * t1l + ((lane < m) ? wrow[lane] : 0.0) * t2l;
        s = warp_sum(s);
        if (lane == 0) wrow[m] = tau_prev * (pyc - s) + alpha_prev * vrow[m];
      }
    } else if (wid == TRD_WARPS - 1) {
      vrow[lane] = 0.0;
      wrow[lane] = 0.0;
    }
    if (jj == nb) break;
    __syncthreads();
    TRD_MARK(1)
    // update column c for own rows r >= c; Σ x_r² over r >= c+2
    double nrm = 0.0;
    const double wl = (lane < jj) ? wrow[lane] : 0.0, vl = (lane < jj) ? vrow[lane] : 0.0;
#pragma unroll
    for (int q = 0; q < TRD_RPW; ++q) {
      const int r = rbase + q * NW;
      if (r < c || r >= n) continue;
      double s = Vs[wid][q][lane] * wl + Ws[wid][q][lane] * vl;
      s = warp_sum(s);
      const double x = Ac[wid][q][jj] - s;
      if (lane == 0) {
        a.xv[r] = x;
        if (r == c) a.d[c] = x;
        if (r >= c + 2) nrm += x * x;
      }
    }
    if (lane == 0) nrm_sh[wid] = nrm;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < TRD_WARPS; ++w) s += nrm_sh[w];
      a.partn[blockIdx.x] = s;
    }
    TRD_MARK(2)
    grid.sync();
    TRD_MARK(3)
    // ------------------------------------------------------------ phase S
    const int m = n - c - 1;
    // stage x (unscaled) while warp 0 reduces the norm partials
    {  // all loads in flight before the stores (one L2 round trip for m ≤ 2048)
      constexpr int XB = 8;
      for (int s0 = threadIdx.x; s0 < m; s0 += XB * TRD_THREADS) {
        double t[XB];
#pragma unroll
        for (int u = 0; u < XB; ++u) {
          const int s = s0 + u * TRD_THREADS;
          t[u] = (s < m) ? __ldcg(a.xv + c + 1 + s) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < XB; ++u) {
          const int s = s0 + u * TRD_THREADS;
          if (s < m) vsh[s] = t[u];
        }
      }
    }
    if (wid == 0) {
      const double alpha = __ldcg(a.xv + c + 1);  // issued together with the partial loads
      constexpr int GPL = (kNumSMs + 31) / 32;
      double v[GPL];
#pragma unroll
      for (int u = 0; u < GPL; ++u) v[u] = (lane + 32 * u < G) ? __ldcg(a.partn + lane + 32 * u) : 0.0;
      double s = 0.0;
#pragma unroll
      for (int u = 0; u < GPL; ++u) s += v[u];
      s = warp_sum(s);
      if (lane == 0) {
        const double xn2 = s;
        double beta, tau, scale;
        dlarfg_scalars(alpha, xn2, beta, tau, scale);
        scal_sh[0] = tau;
        scal_sh[1] = scale;
        if (blockIdx.x == 0) {
          a.e[c] = beta;
          a.tau[c] = tau;
        }
      }
    }
    __syncthreads();
    const double tau = scal_sh[0], scale = scal_sh[1];
    tau_prev = tau;
    TRD_MARK(4)
    for (int s = threadIdx.x; s < m; s += blockDim.x) vsh[s] = (s == 0) ? 1.0 : vsh[s] * scale;
    __syncthreads();
    double pt1 = 0.0, pt2 = 0.0, pyv = 0.0;  // lane t accumulates t1_t, t2_t
    // per own row: V/W bookkeeping once its symv result y is known
    auto finish_row = [&](int q, int r, double y) {
      const double vr = vsh[r - c - 1];
      yreg[q] = y;
      if (lane == jj) Vs[wid][q][jj] = vr;
      if (lane == 0) {
        if (r == c + 1) a.yv[r] = y;
        V[(long)r * LDX + jj] = vr;
        V2[(long)r * LDX + jj] = vr;
        a.Vall[(long)r * n + c] = (tau == 0.0) ? 0.0 : vr;  // H = I: no reflector for the back-transform
        pyv += y * vr;
      }
      if (lane < jj) {
        pt1 += Ws[wid][q][lane] * vr;
        pt2 += Vs[wid][q][lane] * vr;
      }
    };
    // L2-latency bound: 16-byte loads, 16 in flight per lane — from one row, or 8 + 8 from two rows
    // of the same warp (same length m and 16-byte phase s0 when n is even), so a warp with several
    // rows needs half the dependent round trips
    const bool pair_ok = (n & 1) == 0;
    // one row's symv (16 loads in flight per lane)
    auto symv_row = [&](int q, int r) {
      const double* Ar = a.A + (long)r * n + c + 1;
      double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      const int s0 = (int)((reinterpret_cast<uintptr_t>(Ar) >> 3) & 1);  // peel to 16 B alignment
      if (s0 && lane == 0 && m > 0) acc[0] = Ar[0] * vsh[0];
      const int m2 = (m - s0) >> 1;
      const double2* A2 = reinterpret_cast<const double2*>(Ar + s0);
      const double* vb = vsh + s0;
      int qq = lane;
      for (; qq + 15 * 32 < m2; qq += 16 * 32) {  // 16 × 16 B in flight per lane
        double2 av[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) av[u] = __ldcg(A2 + qq + u * 32);
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int s = 2 * (qq + u * 32);
          acc[u & 7] += av[u].x * vb[s] + av[u].y * vb[s + 1];
        }
      }
      for (; qq + 7 * 32 < m2; qq += 8 * 32) {
        double2 av[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) av[u] = __ldcg(A2 + qq + u * 32);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int s = 2 * (qq + u * 32);
          acc[u] += av[u].x * vb[s] + av[u].y * vb[s + 1];
        }
      }
      for (; qq < m2; qq += 32) {
        const double2 av = A2[qq];
        acc[0] += av.x * vb[2 * qq] + av.y * vb[2 * qq + 1];
      }
      if (((m - s0) & 1) && lane == 0) acc[1] += Ar[m - 1] * vsh[m - 1];
      double y = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
      y = warp_sum(y);
      finish_row(q, r, y);
    };
    // two rows of this warp together (8 + 8 loads in flight per lane)
    auto symv_pair = [&](int q, int r, int r1) {
        const double* Ar0 = a.A + (long)r * n + c + 1;
        const double* Ar1 = a.A + (long)r1 * n + c + 1;
        double acc0[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        double acc1[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        const int s0 = (int)((reinterpret_cast<uintptr_t>(Ar0) >> 3) & 1);
        if (s0 && lane == 0 && m > 0) {
          acc0[0] = Ar0[0] * vsh[0];
          acc1[0] = Ar1[0] * vsh[0];
        }
        const int m2 = (m - s0) >> 1;
        const double2* A20 = reinterpret_cast<const double2*>(Ar0 + s0);
        const double2* A21 = reinterpret_cast<const double2*>(Ar1 + s0);
        const double* vb = vsh + s0;
        int qq = lane;
        for (; qq + 7 * 32 < m2; qq += 8 * 32) {
          double2 av0[8], av1[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            av0[u] = __ldcg(A20 + qq + u * 32);
            av1[u] = __ldcg(A21 + qq + u * 32);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int s = 2 * (qq + u * 32);
            acc0[u] += av0[u].x * vb[s] + av0[u].y * vb[s + 1];
            acc1[u] += av1[u].x * vb[s] + av1[u].y * vb[s + 1];
          }
        }
        for (; qq < m2; qq += 32) {
          const double2 a0 = A20[qq], a1 = A21[qq];
          acc0[0] += a0.x * vb[2 * qq] + a0.y * vb[2 * qq + 1];
          acc1[0] += a1.x * vb[2 * qq] + a1.y * vb[2 * qq + 1];
        }
        if (((m - s0) & 1) && lane == 0) {
          acc0[1] += Ar0[m - 1] * vsh[m - 1];
          acc1[1] += Ar1[m - 1] * vsh[m - 1];
        }
        double y0 = ((acc0[0] + acc0[1]) + (acc0[2] + acc0[3])) + ((acc0[4] + acc0[5]) + (acc0[6] + acc0[7]));
        double y1 = ((acc1[0] + acc1[1]) + (acc1[2] + acc1[3])) + ((acc1[4] + acc1[5]) + (acc1[6] + acc1[7]));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          y0 += __shfl_xor_sync(0xffffffffu, y0, o);
          y1 += __shfl_xor_sync(0xffffffffu, y1, o);
        }
        finish_row(q, r, y0);
        finish_row(q + 1, r1, y1);
    };
#pragma unroll
    for (int q = 0; q < TRD_RPW; q += 2) {
      const int r = rbase + q * NW, r1 = r + NW;
      const bool v0 = r > c && r < n, v1 = r1 > c && r1 < n;
      if (v0 && v1 && pair_ok) {
        symv_pair(q, r, r1);
      } else {
        if (v0) symv_row(q, r);
        if (v1) symv_row(q + 1, r1);
      }
    }
    sred[wid][lane] = pt1;
    sred[wid][TRD_NB + lane] = pt2;
    if (lane == 0) sred[wid][2 * TRD_NB] = pyv;
    __syncthreads();
    TRD_MARK(5)
    for (int q = threadIdx.x; q <= 2 * TRD_NB; q += blockDim.x) {
      double s = 0.0;
      for (int w = 0; w < TRD_WARPS; ++w) s += sred[w][q];
      a.part[(long)q * kNumSMs + blockIdx.x] = s;
    }
    TRD_MARK(6)
    grid.sync();
    TRD_MARK(7)
  }
  if (timing)
    for (int i = 0; i < 8; ++i) a.dbg[i] += tseg[i];
#undef TRD_MARK
}

// ------------------------------------------------------------ sytrd tail (one cluster)
//
// The last m0 ≤ TAIL_MAX columns of the reduction are done by ONE 16-CTA thread-block cluster that
// holds the whole trailing matrix in its shared memory (rows r ≡ rank mod 16, full symmetric rows):
// unblocked dsytd2 (lower) — per column a distributed-shared-memory gather of the column + its norm,
// the Householder scalars computed identically in every CTA, a row-dot symv on the CTA's own rows,
// a DSMEM gather of y, and the rank-2 update in place.  Two cluster barriers per column instead of
// the panel kernel's two grid barriers and ~4 dependent L2 round trips (≈9.5 µs/column), and only 16
// SMs busy, which leaves the rest of the GPU to the solver's other chains.
constexpr int TAIL_CL = 16;
constexpr int TAIL_THREADS = 512;
constexpr int TAIL_MAX = 640;                   // rows per CTA ≤ 40: 40 × 640 × 8 B = 200 KB of smem
constexpr int TAIL_RPC = TAIL_MAX / TAIL_CL;    // 40
static_assert(TAIL_RPC <= 3 * (TAIL_THREADS / 32), "tail_rows_pass takes at most 3 rows per warp");

struct TailArgs {
  const double* A;  // n × n (ld n), trailing block at (c0, c0) fully updated and symmetric
  int n, c0;
  double* d;
  double* e;
  double* tau;
  double* Vall;     // reflector c (global index) in column c, rows > c; v_{c+1} = 1
  unsigned long long* dbg;  // nullable: per-segment ns accumulated by CTA 0 thread 0
};
unsigned long long* g_tail_dbg = nullptr;  // set by kot_debug_tail_timing

__device__ __forceinline__ double tail_block_sum(double v, double* sh) {
  // fixed-order block reduction (identical result in every CTA for identical inputs)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int w = 0; w < TAIL_THREADS / 32; ++w) t += sh[w];
  return t;
}

// R own rows of one warp (R warp-uniform): the pending rank-2 update applied in place (if pend) fused
// with y_r = Σ_{s>c} A_rs v_s.  Per row: lane-strided, two interleaved partial sums, butterfly — the
// same arithmetic whichever warp or R a row lands in.
template <int R>
__device__ __forceinline__ void tail_rows_pass(double* Aloc, int ld, int q0, int c, int m0, bool pend,
                                               const double* vp, const double* wp, const double* vn,
                                               double* yslot, int g, int lane) {
  cg::cluster_group cl = cg::this_cluster();
  double* A[R];
  double vr[R], wr[R], a0[R], a1[R];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const int q = q0 + j * (TAIL_THREADS / 32);
    const int r = g + TAIL_CL * q;
    A[j] = Aloc + (long)q * ld;
    vr[j] = pend ? vp[r] : 0.0;
    wr[j] = pend ? wp[r] : 0.0;
    a0[j] = 0.0;
    a1[j] = 0.0;
  }
  int s = c + 1 + lane;
  if (pend) {
    for (; s + 32 < m0; s += 64) {
      const double ws0 = wp[s], ws1 = wp[s + 32], us0 = vp[s], us1 = vp[s + 32];
      const double x0 = vn[s], x1 = vn[s + 32];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const double e0 = A[j][s] - vr[j] * ws0 - wr[j] * us0;
        const double e1 = A[j][s + 32] - vr[j] * ws1 - wr[j] * us1;
        A[j][s] = e0;
        A[j][s + 32] = e1;
        a0[j] += e0 * x0;
        a1[j] += e1 * x1;
      }
    }
    if (s < m0) {
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const double e = A[j][s] - vr[j] * wp[s] - wr[j] * vp[s];
        A[j][s] = e;
        a0[j] += e * vn[s];
      }
    }
  } else {
    for (; s + 32 < m0; s += 64) {
      const double x0 = vn[s], x1 = vn[s + 32];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        a0[j] += A[j][s] * x0;
        a1[j] += A[j][s + 32] * x1;
      }
    }
    if (s < m0) {
#pragma unroll
      for (int j = 0; j < R; ++j) a0[j] += A[j][s] * vn[s];
    }
  }
  double t[R];
#pragma unroll
  for (int j = 0; j < R; ++j) t[j] = a0[j] + a1[j];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int j = 0; j < R; ++j) t[j] += __shfl_xor_sync(0xffffffffu, t[j], o);
  }
  // (the butterfly leaves the same bits in every lane) lane k < 16 pushes y_r into CTA k's slot
  if (lane < TAIL_CL) {
#pragma unroll
    for (int j = 0; j < R; ++j) cl.map_shared_rank(yslot, lane)[g + TAIL_CL * (q0 + j * (TAIL_THREADS / 32))] = t[j];
  }
}

__global__ void __launch_bounds__(TAIL_THREADS, 1) sytrd_tail_kernel(TailArgs a) {
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ double tsm[];
  const int g = (int)cl.block_rank();
  const int n = a.n, c0 = a.c0, m0 = n - c0;
  const int nrows = (m0 - g + TAIL_CL - 1) / TAIL_CL;  // own rows r = g + 16 q, q < nrows
  const int ld = m0 + (m0 & 1);
  double* Aloc = tsm;                               // nrows × ld
  double* vwbuf = Aloc + (long)TAIL_RPC * ld;       // by column parity: [v | w], 2 × 2 × ld
  // Push model: every CTA stores its rows' column entries, partial norm and symv results straight into
  // every CTA's shared memory (remote stores before the cluster barrier), so each consumer reads them
  // locally after it: x_r lands in v's slot of the column (scaled in place), y_r in w's slot, the
  // partial norms in nfull[rank].  The slots are dead when written: the column's v / w buffers last
  // held column c−2's, and every CTA is past the barrier that ends their last use.
  __shared__ double nfull[TAIL_CL];
  __shared__ double red[TAIL_THREADS / 32];
  __shared__ double scal[3];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

  for (int q = wid; q < nrows; q += TAIL_THREADS / 32) {
    const double* src = a.A + (long)(c0 + g + TAIL_CL * q) * n + c0;
    double* dst = Aloc + (long)q * ld;
    for (int s = lane; s < m0; s += 32) dst[s] = src[s];
  }
  __syncthreads();

  const bool timing = (a.dbg != nullptr) && g == 0 && tid == 0;
  unsigned long long tseg[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long tl = timing ? gtimer() : 0;
#define TAIL_MARK(i)                        \
  if (timing) {                             \
    const unsigned long long t_ = gtimer(); \
    tseg[i] += t_ - tl;                     \
    tl = t_;                                \
  }
  // The rank-2 update of column c, A_rs −= v_r w_s + w_r v_s (r, s > c), is deferred into column c+1:
  // column c+1 is published with it applied on the fly, and the rest is applied inside column c+1's
  // symv pass (one read + one write of the own rows per column instead of a symv read plus a separate
  // read-modify-write).  Same expressions, same order: bit-identical to the undeferred update.
  bool pend = false;  // column c−1's update is still to be applied (uniform over the cluster)
  for (int c = 0; c + 1 < m0; ++c) {
    double* vn = vwbuf + (c & 1) * 2L * ld;  // v of column c, then its w
    double* wn = vn + ld;
    const double* vp = vwbuf + ((c + 1) & 1) * 2L * ld;  // column c−1's
    const double* wp = vp + ld;
    // (A) publish own entries of column c below the diagonal (pending update applied) and the partial norm
    double pn = 0.0;
    for (int q = tid; q < nrows; q += TAIL_THREADS) {
      const int r = g + TAIL_CL * q;
      double x = Aloc[(long)q * ld + c];
      if (pend && r >= c) x = x - vp[r] * wp[c] - wp[r] * vp[c];
      if (r > c) {
#pragma unroll
        for (int k = 0; k < TAIL_CL; ++k) cl.map_shared_rank(vn, k)[r] = x;
      }
      if (r >= c + 2) pn += x * x;
      if (r == c) a.d[c0 + c] = x;
    }
    pn = tail_block_sum(pn, red);
    if (tid < TAIL_CL) cl.map_shared_rank(nfull, tid)[g] = pn;
    TAIL_MARK(0)
    cl.sync();
    TAIL_MARK(1)
    // (B) the column is local now (pushed into vn), Householder scalars (dlarfg) identically in every
    // CTA, then v = x·scale in place with v_{c+1} = 1
    constexpr int XPT = (TAIL_MAX + TAIL_THREADS - 1) / TAIL_THREADS;
    double xr[XPT];
#pragma unroll
    for (int u = 0; u < XPT; ++u) {
      const int r = c + 1 + tid + u * TAIL_THREADS;
      xr[u] = (r < m0) ? vn[r] : 0.0;
    }
    const double alpha = vn[c + 1];  // read by every thread before the barrier below
    if (wid == 0) {
      double t = (lane < TAIL_CL) ? nfull[lane] : 0.0;
      t = warp_sum(t);  // fixed order over the 16 ranks
      if (lane == 0) scal[0] = t;
    }
    __syncthreads();
    const double xn2 = scal[0];
    double beta, tau, scale;
    dlarfg_scalars(alpha, xn2, beta, tau, scale);  // every thread, identically
    if (g == 0 && tid == 0) {
      a.e[c0 + c] = beta;
      a.tau[c0 + c] = tau;
    }
#pragma unroll
    for (int u = 0; u < XPT; ++u) {
      const int r = c + 1 + tid + u * TAIL_THREADS;
      if (r < m0) vn[r] = (r == c + 1) ? 1.0 : xr[u] * scale;
    }
    __syncthreads();
    TAIL_MARK(2)
    for (int q = tid; q < nrows; q += TAIL_THREADS) {
      const int r = g + TAIL_CL * q;
      if (r > c) a.Vall[(long)(c0 + r) * n + c0 + c] = (tau == 0.0) ? 0.0 : vn[r];
    }
    TAIL_MARK(3)
    if (tau == 0.0) {  // H = I: no symv and no new update; apply the pending one on its own
      if (pend) {
        for (int q = wid; q < nrows; q += TAIL_THREADS / 32) {
          const int r = g + TAIL_CL * q;
          if (r <= c) continue;
          double* Ar = Aloc + (long)q * ld;
          const double vr = vp[r], wr = wp[r];
          for (int s = c + 1 + lane; s < m0; s += 32) Ar[s] = Ar[s] - vr * wp[s] - wr * vp[s];
        }
      }
      pend = false;
      __syncthreads();
      cl.sync();  // keep the two-barrier rhythm
      continue;
    }
    // (C) pending update fused with y_r = Σ_{s>c} A_rs v_s for own rows r > c: the live rows
    // q ≥ qlo spread over the warps (warp w: qlo + w + 16 j), one pass of up to 3 rows per warp
    {
      const int qlo = (c + 1 - g + TAIL_CL - 1) / TAIL_CL > 0 ? (c + 1 - g + TAIL_CL - 1) / TAIL_CL : 0;
      const int q0 = qlo + wid;
      const int nr = q0 < nrows ? (nrows - q0 + TAIL_THREADS / 32 - 1) / (TAIL_THREADS / 32) : 0;
      if (nr == 1)
        tail_rows_pass<1>(Aloc, ld, q0, c, m0, pend, vp, wp, vn, wn, g, lane);
      else if (nr == 2)
        tail_rows_pass<2>(Aloc, ld, q0, c, m0, pend, vp, wp, vn, wn, g, lane);
      else if (nr >= 3)
        tail_rows_pass<3>(Aloc, ld, q0, c, m0, pend, vp, wp, vn, wn, g, lane);
    }
    TAIL_MARK(4)
    cl.sync();
    TAIL_MARK(5)
    // (D) gather y (registers), w = τ y − ½ τ² (yᵀv) v
    double yr[XPT];
    double pyv = 0.0;
#pragma unroll
    for (int u = 0; u < XPT; ++u) {
      const int r = c + 1 + tid + u * TAIL_THREADS;
      yr[u] = (r < m0) ? wn[r] : 0.0;  // pushed by the row's owner
    }
#pragma unroll
    for (int u = 0; u < XPT; ++u) {
      const int r = c + 1 + tid + u * TAIL_THREADS;
      if (r < m0) pyv += yr[u] * vn[r];
    }
    const double yv = tail_block_sum(pyv, red);
    const double alpha2 = -0.5 * tau * (tau * yv);
#pragma unroll
    for (int u = 0; u < XPT; ++u) {
      const int r = c + 1 + tid + u * TAIL_THREADS;
      if (r < m0) wn[r] = tau * yr[u] + alpha2 * vn[r];
    }
    pend = true;
    __syncthreads();
    TAIL_MARK(6)
  }
  if (timing)
    for (int i = 0; i < 8; ++i) a.dbg[i] += tseg[i];
#undef TAIL_MARK
  if (g == (m0 - 1) % TAIL_CL && tid == 0) {
    const int r = m0 - 1;
    double x = Aloc[(long)((m0 - 1) / TAIL_CL) * ld + r];
    if (pend && m0 >= 2) {  // the last column's update (c = m0 − 2) on the last diagonal entry
      const double* vp = vwbuf + ((m0 - 2) & 1) * 2L * ld;
      const double* wp = vp + ld;
      x = x - vp[r] * wp[r] - wp[r] * vp[r];
    }
    a.d[n - 1] = x;
  }
  cl.sync();  // no CTA leaves while its shared memory may still be read
}

__global__ void set_last_diag_kernel(const double* A, int n, double* d) { d[n - 1] = A[(long)(n - 1) * n + n - 1]; }

}  // namespace kot
#include "sytrd_mid.cuh"
namespace kot {

void EigWork::ensure_mid() {
  if (mid_x) return;
  const size_t bytes = sizeof(MidSector) * 2 * MID_REP_MAX * kNumSMs * MID_SPC;
  mid_x = dev_alloc(bytes);
  mid_err = static_cast<int*>(dev_alloc(sizeof(int)));
  mid_err_host = static_cast<int*>(host_alloc_pinned(2 * sizeof(int)));
  mid_err_host[0] = mid_err_host[1] = 0;
  mid_resident = reinterpret_cast<unsigned*>(mid_err_host + 1);
  KOT_CUDA(cudaMemset(mid_x, 0, bytes));
  KOT_CUDA(cudaMemset(mid_err, 0, sizeof(int)));
}


unsigned long long* g_trd_dbg = nullptr;  // set by kot_debug_sytrd_timing

// CTAs of the cooperative panel kernel (≤ one per SM).  KOT_TRD_GRID caps every
// lane, KOT_TRD_GRID_FG/_BG/_BG2 set the per-lane sizes under an EG pipeline (diagnostics).
static int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  const int v = e ? std::atoi(e) : 0;
  return v > 0 ? v : dflt;
}
// Number of live EG pipelines (solver.cu): while one runs, three eigensolve chains share the GPU.
static std::atomic<int> g_pipelines{0};
void eig_pipeline_active(int delta) { g_pipelines += delta; }

// Process-wide cap on every panel grid (KOT_TRD_GRID, or kot_set_panel_grid_cap at run time): several
// concurrent solves (config-5 batches) share the GPU better with thin grids.
static std::atomic<int> g_trd_cap{-1};
void set_panel_grid_cap(int cap) { g_trd_cap = cap > 0 ? std::min(cap, kNumSMs) : kNumSMs; }
static int trd_grid_cap_all() {
  if (g_trd_cap.load() < 0) g_trd_cap = std::min(env_int("KOT_TRD_GRID", kNumSMs), kNumSMs);
  return g_trd_cap.load();
}
static int trd_grid_cap(int lane) {
  if (g_trd_cap.load() < 0) g_trd_cap = std::min(env_int("KOT_TRD_GRID", kNumSMs), kNumSMs);
  const int cap = g_trd_cap.load();
  // With an EG pipeline running, four cooperative grids can be in flight — Newton chain 96, the EG
  // step's two projections (run side by side, eg_step_parallel) 48 each, residual at v 32 CTAs — and
  // they fit co-resident in the 2 × 148 slots, so no chain queues at the gate behind another's panel
  // (probe cfg3 with parallel EG projections: 96/96/64 → 10.2, 96/64/64 → 10.5, 96/64/48 → 10.7–11.0,
  // 112/56/48 → 10.7, 128/48/48 → 11.0, 96/64/32 → 10.8, 96/48/32 → 11.1, 96/32/32 → 11.1 it/s: the
  // EG chain has slack, ≈ 58 vs 90 ms per iteration).  Alone, lane 0 uses every SM.
  static const int fg = env_int("KOT_TRD_GRID_FG", 96);
  const int cap_fg = std::min(fg, cap);
  // Round 2, with the TMA GEMM core: thinner EG-chain grids leave CTA slots (registers) to the Newton
  // chain's CG GEMMs, whose CTAs co-reside with panel CTAs on the same SMs (cfg3: 48/32 → 24/16
  // CTAs: Newton direction 42.1 → 38.5 ms, 13.9 → 14.6 it/s; the EG chain, 51 → 56 ms, keeps slack).
  // With the mid kernel on the Newton chain the EG chain became the longer one: 32 / 32 (cfg3 16.55–16.65
  // it/s, tight profile 15.25) against 24 / 16 (16.26–16.33, 15.15), 48 / 16 (16.6, 15.0), 48 / 32 (16.5, 15.1).
  static const int bg = env_int("KOT_TRD_GRID_BG", 32);
  const int cap_bg = std::min(bg, cap);
  // lane 2 = the EG pipeline's residual thread, lane 1 = its EG-step threads
  static const int bg2 = env_int("KOT_TRD_GRID_BG2", 32);
  const int cap_bg2 = std::min(bg2, cap);
  if (lane == 0) return g_pipelines.load() > 0 ? cap_fg : cap;
  return lane == 2 ? cap_bg2 : cap_bg;
}
static int trd_grid(int rows, int lane) {
  // never below what the per-warp row capacity needs (TRD_RPW rows per warp)
  const int need = ceil_div(rows, TRD_WARPS * TRD_RPW);
  const int g = std::max(need, std::max(1, std::min(trd_grid_cap(lane), ceil_div(rows, TRD_WARPS))));
  return g;
}

// Cooperative sytrd grids from different streams/host threads must never need
// more co-resident CTAs than the SMs can hold at once (their blocks spin on a
// grid barrier).  This process-wide gate accounts CTA slots (occupancy × SMs):
// a grid is admitted when its CTAs fit, and background grids (lane ≠ 0) may
// only use what is left after reserving one full lane-0 grid, so a Newton-chain
// eigensolve never queues behind the EG pipeline.
//
// The grid-resident mid kernel needs WHOLE SMs (one 220 KB CTA each) and its CTAs spin on each other
// from the first column on, so it must never wait for SMs behind a stream of small background CTAs:
// its owner first makes the gate exclusive (no new background grid is admitted, the ones in flight
// retire — a panel launch lasts under a millisecond), launches, waits until the kernel reports every
// CTA resident (its first exchange completed), and then re-opens the gate with the slots of its SMs
// accounted, so the background chains' grids go on beside it on the remaining SMs.
namespace {
std::mutex g_coop_mu;
std::condition_variable g_coop_cv;
int g_coop_used = 0;
int g_coop_fg = 0;      // lane-0 grids in flight
bool g_coop_excl = false;  // an exclusive owner is waiting or launching: no new admissions
std::atomic<bool> g_coop_excl_hint{false};  // lock-free mirror, polled by the panel loops
struct CoopGate {
  int slots, lane, total, limit_bg;
  CoopGate(int total_, int want, int reserve, int lane_) : slots(want), lane(lane_), total(total_) {
    static const bool yield_bg = [] {  // diagnostic: background grids wait while a lane-0 grid runs
      const char* e = std::getenv("KOT_COOP_YIELD");
      return e && std::atoi(e) > 0;
    }();
    std::unique_lock<std::mutex> lk(g_coop_mu);
    limit_bg = total - reserve;
    const int limit = (lane == 0) ? total : limit_bg;
    g_coop_cv.wait(lk, [&] {
      if (g_coop_excl) return false;
      if (lane != 0 && yield_bg && g_coop_fg > 0) return false;
      return g_coop_used + want <= limit || g_coop_used == 0;
    });
    g_coop_used += want;
    if (lane == 0) ++g_coop_fg;
  }
  // no other grid in flight and none admitted until exclusive_end
  void exclusive_begin() {
    // (the caller's own grids have retired: its slots go back while it waits, so that two owners
    // cannot block each other)
    std::unique_lock<std::mutex> lk(g_coop_mu);
    g_coop_used -= slots;
    g_coop_cv.notify_all();
    g_coop_cv.wait(lk, [&] { return !g_coop_excl; });
    g_coop_excl = true;
    g_coop_excl_hint = true;
    g_coop_cv.wait(lk, [&] { return g_coop_used == 0; });
    g_coop_used += slots;
  }
  // Called by the other chains between two panel launches: when an exclusive owner waits, let the
  // grids in flight retire, give the slots back and come back once the owner's kernel is resident
  // (a gate is otherwise held for a whole tridiagonalisation, tens of milliseconds).
  void yield_to_exclusive(cudaStream_t st) {
    if (!g_coop_excl_hint.load(std::memory_order_relaxed)) return;
    if (st) KOT_CUDA(cudaStreamSynchronize(st));  // (no stream: the host-only self-test)
    std::unique_lock<std::mutex> lk(g_coop_mu);
    if (!g_coop_excl) return;
    g_coop_used -= slots;
    g_coop_cv.notify_all();
    const int limit = (lane == 0) ? total : limit_bg;
    g_coop_cv.wait(lk, [&] { return !g_coop_excl && (g_coop_used + slots <= limit || g_coop_used == 0); });
    g_coop_used += slots;
  }
  // the owner's kernel is resident on `sms` whole SMs: account them and admit the others again
  void exclusive_end(int sms, int per_sm) {
    {
      std::lock_guard<std::mutex> lk(g_coop_mu);
      const int hold = std::max(slots, limit_bg - per_sm * (kNumSMs - sms));
      g_coop_used += hold - slots;
      slots = hold;
      g_coop_excl = false;
      g_coop_excl_hint = false;
    }
    g_coop_cv.notify_all();
  }
  ~CoopGate() {
    {
      std::lock_guard<std::mutex> lk(g_coop_mu);
      g_coop_used -= slots;
      if (lane == 0) --g_coop_fg;
    }
    g_coop_cv.notify_all();
  }
};
}  // namespace

// Grid-resident mid kernel: KOT_TRD_MID = 0 off, 1 (default) for latency-critical eigensolves, 2 for
// every eigensolve (tests); KOT_TRD_MID_TAIL = trailing columns handed to the cluster tail (0: none).
static std::atomic<int> g_mid_mode{-1};
static std::atomic<int> g_mid_tail{-1};
static std::atomic<int> g_mid_head{-1};  // head launch on every SM beside an EG pipeline (KOT_TRD_MID_HEAD)
static std::atomic<int> g_mid_rep{1};  // replicas of the exchange sectors (KOT_TRD_MID_REP)
static int mid_mode() {
  if (g_mid_mode.load() < 0) {
    const char* e = std::getenv("KOT_TRD_MID");
    g_mid_mode = e ? std::max(0, std::atoi(e)) : 1;
    const char* t = std::getenv("KOT_TRD_MID_TAIL");
    g_mid_tail = t ? std::max(0, std::atoi(t)) : 0;
    const char* r = std::getenv("KOT_TRD_MID_REP");
    if (r) g_mid_rep = std::min(std::max(1, std::atoi(r)), MID_REP_MAX);
  }
  return g_mid_mode.load();
}
// the mid kernel needs one resident 512-thread CTA with the maximum shared memory per SM: if the
// device or its configuration cannot provide that, the panel + tail path is used
static bool mid_supported() {
  static const bool ok = [] {
    int dev = 0, sms = 0, per_sm = 0, coop = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    if (sms < kNumSMs || !coop) return false;
    if (cudaFuncSetAttribute((const void*)sytrd_mid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             200 * 1024) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sytrd_mid_kernel, MID_THREADS, 200 * 1024) !=
            cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return per_sm >= 1;
  }();
  return ok;
}
static size_t mid_smem_max() {
  static const size_t v = [] {
    int dev = 0, optin = 0;
    KOT_CUDA(cudaGetDevice(&dev));
    KOT_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa;
    KOT_CUDA(cudaFuncGetAttributes(&fa, (const void*)sytrd_mid_kernel));
    return (size_t)optin - fa.sharedSizeBytes;
  }();
  return v;
}

static void sytrd(const double* Z, int n, EigWork& w, cudaStream_t st, int lane, CoopGate* gate, int per_sm) {
  KOT_CUDA(cudaMemcpyAsync(w.A, Z, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, st));
  KOT_CUDA(cudaMemsetAsync(w.Vall, 0, sizeof(double) * n * n, st));
  static const bool use_tail = [] {
    const char* e = std::getenv("KOT_TRD_TAIL");
    return !(e && std::atoi(e) == 0);
  }();
  // columns [c0, n) go to the cluster-resident tail kernel (c0 on a panel boundary)
  int c0 = !use_tail ? n : (n <= TAIL_MAX ? 0 : ceil_div(n - TAIL_MAX, TRD_NB) * TRD_NB);
  // columns [cm, cm + mid_cols) go to the grid-resident mid kernel: a latency-critical eigensolve
  // (lane 0, not a background chain) whose grid's shared memory holds clearly more than the tail's 640
  int cm = n, mid_cols = 0, Gm = 0;
  int ch = n, Gh = 0;  // head launch: columns [ch, cm) on Gh CTAs (ch = cm: none)
  const int mode = mid_mode();
  if (mode > 0 && n >= 3 && ((lane == 0 && !background_thread()) || mode >= 2) && mid_supported()) {
    // beside an EG pipeline the mid kernel takes KOT_TRD_MID_GRID whole SMs (default 96) and the
    // background chains keep the others; alone, every SM
    static const int mid_grid_shared = env_int("KOT_TRD_MID_GRID", 96);
    if (g_mid_head.load() < 0) {
      const char* e = std::getenv("KOT_TRD_MID_HEAD");
      g_mid_head = e ? std::min(std::max(std::atoi(e), 0), 2) : 1;
    }
    // (2: the solver's two-launch schedule also for standalone eigensolves — tests)
    const bool shared_like = (g_pipelines.load() > 0 || g_mid_head.load() == 2) && lane == 0 && !background_thread();
    Gm = std::min(shared_like ? std::min(mid_grid_shared, trd_grid_cap_all()) : trd_grid_cap(lane), kNumSMs);
    const int cap = mid_capacity(Gm, mid_smem_max());
    if (cap >= TAIL_MAX + 256 && (n > TAIL_MAX || mode >= 2)) {
      cm = n <= cap ? 0 : ceil_div(n - cap, TRD_NB) * TRD_NB;
      const int m0 = n - cm;
      const int keep = use_tail ? std::min(g_mid_tail.load(), TAIL_MAX) : 0;  // columns left to the tail
      mid_cols = keep >= 2 && m0 - keep >= 1 ? m0 - keep : m0 - 1;
      c0 = mid_cols == m0 - 1 ? n : cm + mid_cols;
      // Beside an EG pipeline the columns between what every SM could hold and what Gm SMs hold (224 … 560
      // at ℓ = 2000) would go to the panel kernel at ≈ 19 µs per column: a *head* launch on every SM takes
      // them instead (the background chains wait ≈ 1.6 ms longer at the gate) and hands its block over.
      if (g_mid_head.load() >= 1 && shared_like) {
        const int Gall = std::min(trd_grid_cap_all(), kNumSMs);
        const int caph = mid_capacity(Gall, mid_smem_max());
        if (Gall > Gm && caph >= cap + 2 * TRD_NB && n > cap) {
          ch = n <= caph ? 0 : ceil_div(n - caph, TRD_NB) * TRD_NB;
          Gh = Gall;
          if (cm - ch < 2) ch = cm;  // nothing worth a launch
        }
      }
    }
  }
  if (ch > cm) ch = cm;
  // Under a batch's panel-grid cap (several solves share the GPU) every chain is throttled, the Newton
  // chains included: short queues interleave the solves more evenly (config-5 batch 2.77 → 2.81 problems/s;
  // without any throttle 2.70).  KOT_TRD_THROTTLE_ALL=0 restricts it to the background chains again.
  static const bool throttle_all = [] {
    const char* e = std::getenv("KOT_TRD_THROTTLE_ALL");
    return !(e && std::atoi(e) == 0);
  }();
  const bool throttle = gate != nullptr && mode > 0 && g_pipelines.load() > 0 &&
                        (lane != 0 || background_thread() || (throttle_all && trd_grid_cap_all() < kNumSMs));
  static const int depth = std::min(env_int("KOT_TRD_THROTTLE", 2), 8);  // panels enqueued ahead of the GPU
  if (throttle) w.ensure_panel_events();
  for (int p0 = 0; p0 < std::min(std::min(c0, ch), n - 1); p0 += TRD_NB) {
    const int nb = std::min(TRD_NB, n - 1 - p0);
    w.check_cancel(st);
    if (gate) {
      // background chains stay within a few panels of the GPU, so that they reach this point (and can
      // yield to a mid kernel's exclusive window) within a millisecond or two instead of having the
      // whole tridiagonalisation enqueued
      if (throttle) {
        const int pi = p0 / TRD_NB;
        if (pi >= depth) KOT_CUDA(cudaEventSynchronize(w.ev_panel[pi % depth]));
      }
      gate->yield_to_exclusive(st);
    }
    KOT_CUDA(cudaMemsetAsync(w.X, 0, sizeof(double) * n * 3 * TRD_NB, st));
    const int rows = n - p0;
    const int G = trd_grid(rows, lane);
    kot_require((long)G * TRD_WARPS * TRD_RPW >= rows, KOT_EINVAL, "matrix order too large for sytrd");
    TrdArgs args{w.A, n, p0, nb, w.X, w.Vall, w.d, w.e, w.tau, w.xv, w.yv, w.part, w.partn, g_trd_dbg,
                 w.gpart, w.gcnt};
    // algorithmic bytes: one read of the lower triangle of every trailing matrix this panel reflects
    double bytes = 0.0;
    for (int c = p0; c < p0 + nb; ++c) bytes += 8.0 * 0.5 * (double)(n - c - 1) * (n - c);
    const size_t smem = sizeof(double) * (std::max(rows, 1) + 3L * TRD_WARPS * TRD_RPW * TRD_NB);
    ensure_smem_attr((const void*)sytrd_panel_kernel, (int)smem);
    {
      ProfScope pscope("sytrd_panel", st, 0.0, bytes);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(G);
      cfg.blockDim = dim3(TRD_THREADS);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeCooperative;
      at[0].val.cooperative = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      // background chains' panels (lanes 1, 2) bring their SMs up with the maximum shared-memory
      // carveout, so that the Newton chain's GEMM CTAs fit beside them; the Newton chain's own panels
      // keep the default split (their L1 helps: trial eigensolve 27.8 vs 28.6 ms)
      if ((lane != 0 || background_thread()) && carveout_preferred()) {
        at[1].id = cudaLaunchAttributePreferredSharedMemoryCarveout;
        at[1].val.sharedMemCarveout = cudaSharedmemCarveoutMaxShared;
        cfg.numAttrs = 2;
      }
      KOT_CUDA(cudaLaunchKernelEx(&cfg, sytrd_panel_kernel, args));
      KOT_LAUNCH_CHECK();
    }
    // trailing update A22 -= V Wᵀ + W Vᵀ on rows/cols >= p0+nb
    const int t0 = p0 + nb;
    const int m2 = n - t0;
    if (m2 > 0) {
      constexpr int LDX = 3 * TRD_NB;
      GemmShape s = make_shape(m2, m2, 2 * TRD_NB, w.X + (long)t0 * LDX, LDX, w.X + (long)t0 * LDX + TRD_NB, LDX);
      s.sym_tiles = 1;
      double* C = w.A + (long)t0 * n + t0;
      EpiSymMirror epi{C, n, -1.0, C, 1.0, 0.0};
      gemm_launch<false, true>(s, epi, st);
    }
    if (throttle) KOT_CUDA(cudaEventRecord(w.ev_panel[(p0 / TRD_NB) % depth], st));
  }
  if (mid_cols > 0) {
    ensure_smem_attr((const void*)sytrd_mid_kernel, (int)mid_smem_max());  // static + dynamic may pass 48 KB below it
    w.ensure_mid();
    // columns [cs, cs + cols) of the block starting at cs on G CTAs; returns the launch epoch
    auto launch_mid = [&](int G, int cs, int cols) {
      const int m0 = n - cs;
      const int rpc = ceil_div(m0, G), ld = m0 + (m0 & 1);
      const size_t smem = sizeof(double) * ((size_t)rpc * ld + 4L * ld);
      ++w.mid_seq;  // 64-bit launch epoch: a tag never repeats within a buffer's lifetime
      MidArgs ma{w.A, n, cs, cols, w.d, w.e, w.tau, w.Vall, static_cast<MidSector*>(w.mid_x),
                 g_mid_rep.load(), w.mid_seq << 12, w.mid_err, w.mid_resident, g_mid_dbg, g_mid_trace,
                 g_mid_trace_c0, g_mid_trace_cta};
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(G);
      cfg.blockDim = dim3(MID_THREADS);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeCooperative;  // co-residency: the CTAs spin on each other's slots
      at[0].val.cooperative = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      double bytes = 0.0;
      for (int c = cs; c < cs + cols; ++c) bytes += 8.0 * 0.5 * (double)(n - c - 1) * (n - c);
      ProfScope ps("sytrd_mid", st, 0.0, bytes);
      KOT_CUDA(cudaLaunchKernelEx(&cfg, sytrd_mid_kernel, ma));
      KOT_LAUNCH_CHECK();
      return ma.epoch0;
    };
    // other cooperative grids may be in flight (EG pipeline, concurrent solves): launch exclusively
    const bool shared_gpu = gate != nullptr && (g_pipelines.load() > 0 || lane != 0 || background_thread());
    const auto tx0 = std::chrono::steady_clock::now();
    struct WindowGuard {  // a failed launch must not leave the gate closed for the other chains
      CoopGate* g = nullptr;
      int per_sm = 1;
      ~WindowGuard() {
        if (g) g->exclusive_end(0, per_sm);
      }
    } window;
    if (shared_gpu) {
      KOT_CUDA(cudaStreamSynchronize(st));  // our own panels have retired
      const auto tx1 = std::chrono::steady_clock::now();
      gate->exclusive_begin();
      window.g = gate;
      window.per_sm = per_sm;
      prof_host("host.mid_sync", std::chrono::duration<double, std::milli>(tx1 - tx0).count());
      prof_host("host.mid_excl", std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tx1).count());
    }
    if (ch < cm) launch_mid(Gh, ch, cm - ch);  // head: every SM, hands the block from column cm on back
    const unsigned long long epoch = launch_mid(Gm, cm, mid_cols);
    if (shared_gpu) {
      // every CTA is resident once CTA 0 has completed the first exchange
      const auto t0 = std::chrono::steady_clock::now();
      while (*reinterpret_cast<volatile unsigned*>(w.mid_resident) != (unsigned)epoch) {
        if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(4)) break;  // the kernel's own timeout reports
      }
      prof_host("host.mid_resident", std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
      window.g = nullptr;
      gate->exclusive_end(Gm, per_sm);
    }
    KOT_CUDA(cudaMemcpyAsync(w.mid_err_host, w.mid_err, sizeof(int), cudaMemcpyDeviceToHost, st));
    w.mid_used = true;
  }
  if (c0 < n) {
    if (gate) gate->yield_to_exclusive(st);
    const int m0 = n - c0;
    const size_t smem = sizeof(double) * ((size_t)TAIL_RPC * (m0 + 1) + 4L * (m0 + 1));
    ensure_smem_attr((const void*)sytrd_tail_kernel, (int)smem, true);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(TAIL_CL);
    cfg.blockDim = dim3(TAIL_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = TAIL_CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    TailArgs ta{w.A, n, c0, w.d, w.e, w.tau, w.Vall, g_tail_dbg};
    ProfScope ps("sytrd_tail", st);
    KOT_CUDA(cudaLaunchKernelEx(&cfg, sytrd_tail_kernel, ta));
    KOT_LAUNCH_CHECK();
  } else if (mid_cols == 0) {
    set_last_diag_kernel<<<1, 1, 0, st>>>(w.A, n, w.d);
    KOT_LAUNCH_CHECK();
  }
}

// ======================================================== tridiagonal D&C

// Subtract the rank-one couplings at every split point (dlaed0): d[s], d[s+1] -= |e[s]|.  First the
// tridiagonal's max norm (dstedc's orgnrm, over the couplings as given) goes to *scale: LAPACK runs
// the D&C on T/orgnrm, so its deflation tolerance 8·eps·max(d_max, z_max) mixes an O(1) d with the
// unit-norm z; the merges use 8·eps·max(d_max, orgnrm·z_max), the same test without rescaling T
// (a matrix of norm 1e-8 deflated at an absolute 1.8e-15 before: 3.7e-7 relative projection error).
constexpr int DC_SPLIT_THREADS = 256;
__global__ void __launch_bounds__(DC_SPLIT_THREADS) dc_split_kernel(double* d, const double* e, int n,
                                                                  const int* splits, int ns, double* scale) {
  __shared__ double red[DC_SPLIT_THREADS / 32];
  double mx = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    mx = fmax(mx, fabs(d[i]));
    if (i < n - 1) mx = fmax(mx, fabs(e[i]));
  }
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int w = 0; w < DC_SPLIT_THREADS / 32; ++w) mx = fmax(mx, red[w]);
  *scale = mx;
  for (int i = 0; i < ns; ++i) {
    const int s = splits[i];
    const double r = fabs(e[s]);
    d[s] -= r;
    d[s + 1] -= r;
  }
}

// Leaves: implicit QL (tqli) on a ≤32 tridiagonal, one warp per leaf, without local memory: lane i
// holds d[i], e[i] in registers (the recurrence reads them by warp broadcast, only lanes i, i+1 write),
// every lane runs the scalar recurrence redundantly (identical values), and the eigenvector matrix
// lives in shared memory column-major (column i = 32 consecutive doubles, lane k owns row k), so each
// rotation is two conflict-free shared accesses per lane.  Same arithmetic as the textbook tqli
// (dlaeq-free, the leaves are ≤ 32), eigenvalues finally ranked ascending (ties by index).
constexpr int LEAF_WARPS = 4;
__global__ void __launch_bounds__(32 * LEAF_WARPS) dc_leaf_kernel(double* d, const double* e, const int* leaf_off,
                                                                   const int* leaf_len, int nleaves, double* Q,
                                                                   int ldq, int* err) {
  __shared__ double zsh[LEAF_WARPS][DC_LEAF * DC_LEAF];
  const int w = threadIdx.x >> 5;
  const int leaf = blockIdx.x * LEAF_WARPS + w;
  if (leaf >= nleaves) return;
  const int lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu;
  const int o = leaf_off[leaf], m = leaf_len[leaf];
  double* Z = zsh[w];  // Z[i*32 + k] = row k, column i
  double D = lane < m ? d[o + lane] : 0.0;
  double E = lane < m - 1 ? e[o + lane] : 0.0;
  for (int i = 0; i < m; ++i) Z[i * 32 + lane] = (i == lane) ? 1.0 : 0.0;
  __syncwarp();
  auto dget = [&](int i) { return __shfl_sync(full, D, i); };
  auto eget = [&](int i) { return __shfl_sync(full, E, i); };
  bool failed = false;
  for (int l = 0; l < m && !failed; ++l) {
    int iter = 0, mm;
    do {
      for (mm = l; mm < m - 1; ++mm) {
        const double sd = fabs(dget(mm)) + fabs(dget(mm + 1));
        if (fabs(eget(mm)) + sd == sd) break;
      }
      if (mm != l) {
        if (iter++ == 60) {
          failed = true;
          break;
        }
        const double el = eget(l), dl = dget(l);
        double g = (dget(l + 1) - dl) / (2.0 * el);
        double r = hypot(g, 1.0);
        g = dget(mm) - dl + el / (g + copysign(r, g));
        double s = 1.0, c = 1.0, p = 0.0;
        int i;
        bool early = false;
        for (i = mm - 1; i >= l; --i) {
          const double ei = eget(i), di = dget(i), dip = dget(i + 1);
          double f = s * ei;
          const double b = c * ei;
          r = hypot(f, g);
          if (lane == i + 1) E = r;
          if (r == 0.0) {
            if (lane == i + 1) D = dip - p;
            if (lane == mm) E = 0.0;
            early = true;
            break;
          }
          s = f / r;
          c = g / r;
          g = dip - p;
          r = (di - g) * s + 2.0 * c * b;
          p = s * r;
          if (lane == i + 1) D = g + p;
          g = c * r - b;
          const double z0 = Z[i * 32 + lane], z1 = Z[(i + 1) * 32 + lane];
          Z[(i + 1) * 32 + lane] = s * z0 + c * z1;
          Z[i * 32 + lane] = c * z0 - s * z1;
        }
        if (early) continue;
        if (lane == l) {
          D -= p;
          E = g;
        }
        if (lane == mm) E = 0.0;
      }
    } while (mm != l);
  }
  if (failed) {
    if (lane == 0) atomicExch(err, 1);
    return;
  }
  __syncwarp();
  // ascending order: rank of lane's eigenvalue (ties broken by index), eigenvector columns follow
  int rank = 0;
  for (int j = 0; j < m; ++j) {
    const double dj = dget(j);
    rank += (dj < D) || (dj == D && j < lane);
  }
  if (lane < m) d[o + rank] = D;
  for (int i = 0; i < m; ++i) {
    const int ri = __shfl_sync(full, rank, i);
    if (lane < m) Q[(long)(o + lane) * ldq + o + ri] = Z[i * 32 + lane];
  }
}

constexpr int MS = 8;  // meta ints per merge: K, ndefl, nrot, c1 (top-only), c12 (top-only + mixed)

struct MergeDesc {
  int o, n1, n2;
  long off;  // offset of this merge's K×K / n×K scratch (prefix of n_m²)
};

// Per-merge bookkeeping (one CTA per merge, arrays staged in shared memory):
// z extraction, stable merge of the two ascending halves (parallel ranks by
// binary search), dlaed2 deflation (sequential scan on thread 0 over smem).
// Integer outputs (global, at the merge's offset o):
//   perm[o..o+n)   : sorted position → local column of the block
//   ndcol[o..)     : sorted positions of the K non-deflated columns
//   dcol[o..)      : sorted positions of the deflated columns (sorted by value)
//   rot[o..)       : (pj, nj) index pairs of the deflation rotations
//   meta[4*mi..]   : K, ndefl, nrot
constexpr int DC_PREP_THREADS = 256;

__device__ __forceinline__ int rank_lt(const double* a, int n, double v) {  // #{a_i < v}
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < v)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}
__device__ __forceinline__ int rank_le(const double* a, int n, double v) {  // #{a_i <= v}
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] <= v)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(DC_PREP_THREADS) dc_merge_prep_kernel(
    const MergeDesc* md, const double* Q, int ldq, const double* d, const double* e, double* zs, double* ds,
    double* dlam, double* wv, double* dfv, double* rotcs, double* rho_out, int* perm, int* ndcol, int* dcol,
    int* rot, int* meta, int* pidx, const double* tscale) {
  extern __shared__ double psm[];
  __shared__ double red[32];
  const MergeDesc m = md[blockIdx.x];
  const int o = m.o, n1 = m.n1, n = m.n1 + m.n2;
  double* Du = psm;         // unsorted d (n)
  double* D = psm + n;      // sorted d (n)
  double* Z = psm + 2 * n;  // sorted z (n)
  int* P = reinterpret_cast<int*>(psm + 3 * n);  // n ints
  const double esplit = e[o + n1 - 1];
  const double sgn = (esplit < 0.0) ? -1.0 : 1.0;
  const double rs2 = 1.0 / sqrt(2.0);  // dlaed2: z ← z/√2, ρ ← |2ρ|
  for (int i = threadIdx.x; i < n; i += blockDim.x) Du[i] = d[o + i];
  __syncthreads();
  double zmax = 0.0, dmax = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    // stable merge rank: left-half elements go first on ties
    const int pos = (i < n1) ? i + rank_lt(Du + n1, n - n1, Du[i]) : (i - n1) + rank_le(Du, n1, Du[i]);
    P[pos] = i;
    const double zz = (i < n1) ? Q[(long)(o + n1 - 1) * ldq + o + i] : sgn * Q[(long)(o + n1) * ldq + o + i];
    const double zv = zz * rs2;
    D[pos] = Du[i];
    Z[pos] = zv;
    zmax = fmax(zmax, fabs(zv));
    dmax = fmax(dmax, fabs(Du[i]));
  }
  zmax = warp_max(zmax);
  dmax = warp_max(dmax);
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5] = zmax;
    red[16 + (threadIdx.x >> 5)] = dmax;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) perm[o + i] = P[i];
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
    zmax = fmax(zmax, red[w]);
    dmax = fmax(dmax, red[16 + w]);
  }
  const double rho = fabs(2.0 * esplit);
  const double tol = 8.0 * DEPS * fmax(dmax, *tscale * zmax);  // dlaed2's test on T/orgnrm
  int* NDC = ndcol + o;
  int* DC = dcol + o;
  int* RT = rot + 2 * o;
  double* DFV = dfv + o;
  double* RCS = rotcs + 2 * o;
  double* WV = wv + o;
  double* DL = dlam + o;
  // ---- parallel fast path: if no close pair of non-small z triggers a deflation rotation, the
  // sequential dlaed2 scan reduces to "non-small → secular, small → deflated", in sorted order.
  __shared__ int trig_sh, tot_sh;
  __shared__ int csum[DC_PREP_THREADS];
  int* prevnz = reinterpret_cast<int*>(Du);  // Du is dead after the merge: reuse as int scratch
  if (threadIdx.x == 0) trig_sh = (rho * zmax <= tol) ? 1 : 0;  // everything deflates: sequential path
  __syncthreads();
  const int chunk = (n + blockDim.x - 1) / blockDim.x;
  const int j0 = threadIdx.x * chunk, j1 = min(n, j0 + chunk);
  {  // previous non-small index (chunk-local scan, then carry from the left chunks)
    int last = -1, cnt = 0;
    for (int j = j0; j < j1; ++j) {
      prevnz[j] = last;
      if (!(rho * fabs(Z[j]) <= tol)) {
        last = j;
        ++cnt;
      }
    }
    csum[threadIdx.x] = last;
    __syncthreads();
    int carry = -1;
    for (int q = threadIdx.x - 1; q >= 0 && carry < 0; --q) carry = csum[q];
    for (int j = j0; j < j1 && (prevnz[j] < 0); ++j) prevnz[j] = carry;
    __syncthreads();
    csum[threadIdx.x] = cnt;
  }
  // the dlaed2 close-pair test of every non-small j against its predecessor with the ORIGINAL values:
  // the sequential scan below reuses it wherever the predecessor was not itself rotated (then Z[pj],
  // D[pj] are still the original values, so the test is the same expression on the same inputs)
  unsigned long long fl = 0;  // bit j − j0: the test fired (chunk ≤ 64, i.e. n ≤ 64·DC_PREP_THREADS)
  for (int j = j0; j < j1; ++j) {
    if (rho * fabs(Z[j]) <= tol) continue;
    const int pj = prevnz[j];
    if (pj < 0) continue;
    double s = Z[pj], c = Z[j];
    const double tau = hypot(c, s);
    const double t = D[j] - D[pj];
    c /= tau;
    s = -s / tau;
    if (fabs(t * c * s) <= tol) {
      trig_sh = 1;
      fl |= 1ull << ((j - j0) & 63);
    }
  }
  __syncthreads();
  if (trig_sh) {  // prevnz is dead: it becomes the origin mask (bit 2 = the precomputed test fired)
    const bool exact = chunk <= 64;
    for (int j = j0; j < j1; ++j)
      prevnz[j] = ((P[j] < n1) ? 1 : 2) | ((!exact || ((fl >> (j - j0)) & 1ull)) ? 4 : 0);
    __syncthreads();
  }
  if (!trig_sh) {
    __shared__ int ctop[DC_PREP_THREADS];
    int tops = 0;
    for (int j = j0; j < j1; ++j)
      if (!(rho * fabs(Z[j]) <= tol) && P[j] < n1) ++tops;
    ctop[threadIdx.x] = tops;
    __syncthreads();
    // exclusive prefixes of the non-small and top-only counts over chunks
    if (threadIdx.x == 0) {
      int acc = 0, acct = 0;
      for (int q = 0; q < (int)blockDim.x; ++q) {
        const int v = csum[q], vt = ctop[q];
        csum[q] = acc;
        ctop[q] = acct;
        acc += v;
        acct += vt;
      }
      tot_sh = acct;
      rho_out[blockIdx.x] = rho;
      meta[MS * blockIdx.x + 0] = acc;
      meta[MS * blockIdx.x + 1] = n - acc;
      meta[MS * blockIdx.x + 2] = 0;
      meta[MS * blockIdx.x + 3] = acct;  // no rotations: no mixed columns
      meta[MS * blockIdx.x + 4] = acct;
    }
    __syncthreads();
    const int c1 = tot_sh;
    int kpos = csum[threadIdx.x], tpos = ctop[threadIdx.x];
    for (int j = j0; j < j1; ++j) {
      if (!(rho * fabs(Z[j]) <= tol)) {
        NDC[kpos] = j;
        DL[kpos] = D[j];
        WV[kpos] = Z[j];
        // GEMM order: top-only columns first, then bottom-only
        pidx[o + kpos] = (P[j] < n1) ? tpos++ : c1 + (kpos - tpos);
        ++kpos;
      } else {
        const int dpos = j - kpos;  // deflated entries are already ascending (D sorted)
        DC[dpos] = j;
        DFV[dpos] = D[j];
      }
    }
    return;
  }
  if (threadIdx.x != 0) return;
  rho_out[blockIdx.x] = rho;
  // origin of each sorted column: 1 top child, 2 bottom child, 3 mixed by rotation (bits 0-1); bit 2:
  // the close-pair test against the original predecessor fired (a superset flag when chunk > 64)
  int* mask = prevnz;
  if (rho * zmax <= tol)
    for (int j = 0; j < n; ++j) mask[j] = (P[j] < n1) ? 1 : 2;
  int K = 0, nd = 0, nr = 0;
  if (rho * zmax <= tol) {
    for (int k = 0; k < n; ++k) {
      DC[nd] = k;
      DFV[nd] = D[k];
      ++nd;
    }
  } else {
    int pj = -1;
    bool pj_rot = false;  // Z[pj], D[pj] were changed by a rotation (the precomputed test does not apply)
    for (int j = 0; j < n; ++j) {
      if (rho * fabs(Z[j]) <= tol) {
        DC[nd] = j;
        DFV[nd] = D[j];
        ++nd;
        continue;
      }
      if (pj < 0) {
        pj = j;
        pj_rot = false;
        continue;
      }
      if (!pj_rot && !(mask[j] & 4)) {  // no deflation (same verdict as the test below)
        NDC[K] = pj;
        DL[K] = D[pj];
        WV[K] = Z[pj];
        ++K;
        pj = j;
        continue;
      }
      double s = Z[pj], c = Z[j];
      const double tau = hypot(c, s);
      double t = D[j] - D[pj];
      c /= tau;
      s = -s / tau;
      if (fabs(t * c * s) <= tol) {
        Z[j] = tau;
        Z[pj] = 0.0;
        mask[j] = (mask[j] & 3) | (mask[pj] & 3);
        RT[2 * nr] = pj;
        RT[2 * nr + 1] = j;
        RCS[2 * nr] = c;
        RCS[2 * nr + 1] = s;
        ++nr;
        t = D[pj] * c * c + D[j] * s * s;
        D[j] = D[pj] * s * s + D[j] * c * c;
        D[pj] = t;
        DC[nd] = pj;
        DFV[nd] = D[pj];
        ++nd;
        pj = j;
        pj_rot = true;
      } else {
        NDC[K] = pj;
        DL[K] = D[pj];
        WV[K] = Z[pj];
        ++K;
        pj = j;
        pj_rot = false;
      }
    }
    if (pj >= 0) {
      NDC[K] = pj;
      DL[K] = D[pj];
      WV[K] = Z[pj];
      ++K;
    }
  }
  // insertion-sort the deflated list by value (nearly sorted already)
  for (int i = 1; i < nd; ++i) {
    const double v = DFV[i];
    const int cidx = DC[i];
    int j = i - 1;
    while (j >= 0 && DFV[j] > v) {
      DFV[j + 1] = DFV[j];
      DC[j + 1] = DC[j];
      --j;
    }
    DFV[j + 1] = v;
    DC[j + 1] = cidx;
  }
  {  // GEMM order of the secular columns: top-only, mixed, bottom-only
    int c1 = 0, c2 = 0;
    for (int k = 0; k < K; ++k) {
      const int mk = mask[NDC[k]] & 3;
      c1 += (mk == 1);
      c2 += (mk == 3);
    }
    int i1 = 0, i2 = c1, i3 = c1 + c2;
    for (int k = 0; k < K; ++k) {
      const int mk = mask[NDC[k]] & 3;
      pidx[o + k] = (mk == 1) ? i1++ : (mk == 3) ? i2++ : i3++;
    }
    meta[MS * blockIdx.x + 3] = c1;
    meta[MS * blockIdx.x + 4] = c1 + c2;
  }
  meta[MS * blockIdx.x + 0] = K;
  meta[MS * blockIdx.x + 1] = nd;
  meta[MS * blockIdx.x + 2] = nr;
  (void)zs;
  (void)ds;
}

// One CTA per row of a merge block: gather the row into sorted column order in
// shared memory, apply the deflation rotations in order, then write the
// non-deflated part (Qnd, n × K) and the deflated part (Qdf, n × nd) with
// coalesced stores.
__global__ void dc_merge_vec_kernel(const MergeDesc* md, const double* Q, double* Qdf, double* Qnd, int ldq,
                                    const int* perm, const int* ndcol, const int* dcol, const int* rot,
                                    const double* rotcs, const int* meta, const int* pidx) {
  extern __shared__ double rowsm[];
  const MergeDesc m = md[blockIdx.y];
  const int o = m.o, n = m.n1 + m.n2;
  const int r = blockIdx.x;
  if (r >= n) return;
  const int K = meta[MS * blockIdx.y], nd = meta[MS * blockIdx.y + 1], nr = meta[MS * blockIdx.y + 2];
  const double* qrow = Q + (long)(o + r) * ldq + o;
  const int* P = perm + o;
  for (int j = threadIdx.x; j < n; j += blockDim.x) rowsm[j] = qrow[P[j]];
  __syncthreads();
  if (threadIdx.x == 0) {
    const int* RT = rot + 2 * o;
    const double* RCS = rotcs + 2 * o;
    for (int q = 0; q < nr; ++q) {
      const int pj = RT[2 * q], nj = RT[2 * q + 1];
      const double c = RCS[2 * q], s = RCS[2 * q + 1];
      const double x = rowsm[pj], y = rowsm[nj];
      rowsm[pj] = c * x + s * y;
      rowsm[nj] = c * y - s * x;
    }
  }
  __syncthreads();
  double* ndrow = Qnd + m.off + (long)r * (n + (n & 1));  // static even ld (K ≤ n), 16 B aligned
  for (int k = threadIdx.x; k < K; k += blockDim.x) ndrow[pidx[o + k]] = rowsm[ndcol[o + k]];
  double* dfrow = Qdf + m.off + (long)r * nd;
  for (int t = threadIdx.x; t < nd; t += blockDim.x) dfrow[t] = rowsm[dcol[o + t]];
}

struct RootRef {
  int merge, j;
};

// Secular equation 1 + ρ Σ w_i²/(d_i − λ) = 0, one warp per root.
// Stores λ_j and column j of Δ (Δ_ij = d_i − λ_j, computed from the origin pole).
__global__ void dc_secular_kernel(const MergeDesc* md, const int* meta, const double* dlam, const double* wv,
                                  const double* rho_arr, double* lam, double* Dl, int* err) {
  const int lane = threadIdx.x & 31;
  const int mi = blockIdx.y;
  const MergeDesc m = md[mi];
  const int K = meta[MS * mi];
  const int j = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (j >= K) return;
  const double* dl = dlam + m.o;
  const double* w = wv + m.o;
  const double rho = rho_arr[mi];
  double* delta = Dl + m.off + (long)j * K;
  if (K == 1) {
    if (lane == 0) {
      const double t = rho * w[0] * w[0];
      lam[m.o] = dl[0] + t;
      delta[0] = -t;
    }
    return;
  }
  int o;
  double lo, hi;
  if (j < K - 1) {
    const double gap = dl[j + 1] - dl[j];
    const double mid = 0.5 * gap;
    double f = 0.0;
    for (int i = lane; i < K; i += 32) f += w[i] * w[i] / ((dl[i] - dl[j]) - mid);
    f = 1.0 + rho * warp_sum(f);
    if (f >= 0.0) {
      o = j;
      lo = 0.0;
      hi = mid;
    } else {
      o = j + 1;
      lo = -(gap - mid);
      hi = 0.0;
    }
  } else {
    double s = 0.0;
    for (int i = lane; i < K; i += 32) s += w[i] * w[i];
    o = K - 1;
    lo = 0.0;
    hi = rho * warp_sum(s);
  }
  const double dor = dl[o];
  double tau = 0.5 * (lo + hi);
  bool ok = false;
  for (int it = 0; it < 200; ++it) {
    double psi = 0.0, dpsi = 0.0, phi = 0.0, dphi = 0.0;
    for (int i = lane; i < K; i += 32) {
      const double del = (dl[i] - dor) - tau;
      const double t = w[i] / del;
      if (i <= j) {
        psi += w[i] * t;
        dpsi += t * t;
      } else {
        phi += w[i] * t;
        dphi += t * t;
      }
    }
    psi = rho * warp_sum(psi);
    dpsi = rho * warp_sum(dpsi);
    phi = rho * warp_sum(phi);
    dphi = rho * warp_sum(dphi);
    const double f = 1.0 + psi + phi;
    const double ftol = 16.0 * DEPS * (1.0 + fabs(psi) + fabs(phi) + fabs(tau) * (dpsi + dphi));
    if (fabs(f) <= ftol) {
      ok = true;
      break;
    }
    if (f < 0.0)
      lo = tau;
    else
      hi = tau;
    if (hi - lo <= 4.0 * DEPS * fmax(fabs(lo), fabs(hi))) {
      ok = true;
      break;
    }
    // middle-way rational step (match ψ, ψ' and φ, φ' with the two nearest poles)
    const double dL = (dl[j] - dor) - tau;
    double eta = NAN;
    if (j < K - 1) {
      const double dR = (dl[j + 1] - dor) - tau;
      const double c = f - dL * dpsi - dR * dphi;
      const double s1 = dL * dL * dpsi, s2 = dR * dR * dphi;
      const double A = c, B = -(c * (dL + dR) + s1 + s2), C = c * dL * dR + s1 * dR + s2 * dL;
      if (A == 0.0) {
        eta = -C / B;
      } else {
        double disc = B * B - 4.0 * A * C;
        disc = disc > 0.0 ? sqrt(disc) : 0.0;
        const double q = -0.5 * (B + copysign(disc, B));
        const double r1 = q / A, r2 = (q != 0.0) ? C / q : NAN;
        if (r1 > dL && r1 < dR)
          eta = r1;
        else if (r2 > dL && r2 < dR)
          eta = r2;
      }
    } else {
      const double c = f - dL * dpsi;
      if (c > 0.0) eta = dL + dL * dL * dpsi / c;
    }
    double tn = tau + eta;
    if (!(tn > lo && tn < hi)) tn = 0.5 * (lo + hi);
    if (tn == tau) {
      ok = true;
      break;
    }
    tau = tn;
  }
  if (!ok && lane == 0) atomicExch(err, 2);
  for (int i = lane; i < K; i += 32) delta[i] = (dl[i] - dor) - tau;
  if (lane == 0) lam[m.o + j] = dor + tau;
}

// Gu–Eisenstat: ŵ_i = sign(w_i) sqrt(−Δ_ii Π_{j≠i} Δ_ij/(d_i − d_j)); warp per i.
__global__ void dc_what_kernel(const MergeDesc* md, const int* meta, const double* dlam, const double* wv,
                               const double* Dl, double* what) {
  const int lane = threadIdx.x & 31;
  const MergeDesc m = md[blockIdx.y];
  const int K = meta[MS * blockIdx.y];
  const int i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (i >= K) return;
  const double* dl = dlam + m.o;
  const double* D = Dl + m.off;
  double p = 1.0;
  for (int j = lane; j < K; j += 32) {
    const double dij = D[(long)j * K + i];
    p *= (j == i) ? dij : dij / (dl[i] - dl[j]);
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) p *= __shfl_xor_sync(0xffffffffu, p, s);
  if (lane == 0) what[m.o + i] = copysign(sqrt(fmax(-p, 0.0)), wv[m.o + i]);
}

// Column j of U: u_i = ŵ_i/Δ_ij normalised; written to Uw with its rows in the
// GEMM order π (top-only, mixed, bottom-only columns of Qnd); warp per column.
__global__ void dc_vec_kernel(const MergeDesc* md, const int* meta, const double* what, const double* Dl,
                              double* Uw, const int* pidx) {
  const int lane = threadIdx.x & 31;
  const MergeDesc m = md[blockIdx.y];
  const int K = meta[MS * blockIdx.y];
  const int j = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (j >= K) return;
  const int nm_ = m.n1 + m.n2;
  const double* col = Dl + m.off + (long)j * K;
  double* ucol = Uw + m.off + (long)j * (nm_ + (nm_ & 1));
  const double* wh = what + m.o;
  const int* pi = pidx + m.o;
  double s = 0.0;
  for (int i = lane; i < K; i += 32) {
    const double u = wh[i] / col[i];
    s += u * u;
  }
  s = warp_sum(s);
  const double inv = 1.0 / sqrt(s);
  for (int i = lane; i < K; i += 32) ucol[pi[i]] = (wh[i] / col[i]) * inv;
}

// Merge the ascending roots with the ascending deflated values (parallel
// ranks; roots go first on ties): eigenvalues into d[o..o+n) and the
// destination column of every eigenvector (non-deflated: colmap[o+k];
// deflated: colmap[o+K+t]).
__global__ void dc_order_kernel(const MergeDesc* md, const int* meta, const double* lam, const double* dfv, double* d,
                                int* colmap) {
  const MergeDesc m = md[blockIdx.x];
  const int o = m.o;
  const int K = meta[MS * blockIdx.x], nd = meta[MS * blockIdx.x + 1];
  const double* L = lam + o;
  const double* F = dfv + o;
  for (int a = threadIdx.x; a < K; a += blockDim.x) {
    const int pos = a + rank_lt(F, nd, L[a]);
    d[o + pos] = L[a];
    colmap[o + a] = pos;
  }
  for (int b = threadIdx.x; b < nd; b += blockDim.x) {
    const int pos = b + rank_le(L, K, F[b]);
    d[o + pos] = F[b];
    colmap[o + K + b] = pos;
  }
}

__global__ void dc_copy_deflated_kernel(const MergeDesc* md, const int* meta, const double* Qdf, double* Q, int ldq,
                                        const int* colmap) {
  const MergeDesc m = md[blockIdx.y];
  const int o = m.o, n = m.n1 + m.n2;
  const int K = meta[MS * blockIdx.y], nd = meta[MS * blockIdx.y + 1];
  const long total = (long)n * nd;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
    const int r = (int)(e / nd), t = (int)(e % nd);
    Q[(long)(o + r) * ldq + o + colmap[o + K + t]] = Qdf[m.off + e];
  }
}

struct EpiColMap {
  static constexpr bool kRowDot = false;
  double* Q;
  long ldq;
  int o, roff;
  const int* colmap;  // colmap[o + c]
  __device__ void store(int r, int c, double v) const { Q[(long)(o + roff + r) * ldq + o + colmap[o + c]] = v; }
  __device__ double rowdot_weight(int, int) const { return 0; }
  __device__ void rowdot_store(int, int, double) const {}
};

// All merges of one D&C level in ONE launch (grid.z = merge): the shape of each group — the top rows
// (M = n1, K = c12) or the bottom rows (M = n2, K range [c1, K)) of Qnd·U, N = K non-deflated
// columns — is read from the merge descriptor and the device meta, as the per-merge launches did.
struct EpiColMapGroup {
  static constexpr bool kRowDot = false;
  double* Q;
  long ldq;
  const int* colmap;
  const MergeDesc* md;
  const int* meta;
  const double* Qnd;
  const double* U;
  int bottom;
  int o = 0, roff = 0;
  __device__ void adapt(GemmShape& s, int z) {
    const MergeDesc m = md[z];
    const int nn = m.n1 + m.n2, ld = nn + (nn & 1);
    const int* mt = meta + MS * z;
    s.lda = s.ldb = ld;
    s.B = U + m.off;
    s.N = mt[0];
    o = m.o;
    if (!bottom) {
      s.A = Qnd + m.off;
      s.M = m.n1;
      s.K = mt[4];
      s.kstart = 0;
      roff = 0;
    } else {
      s.A = Qnd + m.off + (long)m.n1 * ld;
      s.M = m.n2;
      s.K = mt[0];
      s.kstart = mt[3];
      roff = m.n1;
    }
  }
  __device__ void store(int r, int c, double v) const { Q[(long)(o + roff + r) * ldq + o + colmap[o + c]] = v; }
  __device__ double rowdot_weight(int, int) const { return 0; }
  __device__ void rowdot_store(int, int, double) const {}
};

struct DcNode {
  int o, n, depth;
  bool leaf;
};

static void dc_build(int o, int n, int depth, std::vector<DcNode>& out) {
  if (n <= DC_LEAF) {
    out.push_back({o, n, depth, true});
    return;
  }
  const int n1 = n / 2;
  out.push_back({o, n, depth, false});
  dc_build(o, n1, depth + 1, out);
  dc_build(o + n1, n - n1, depth + 1, out);
}

// Eigen-decomposition of the symmetric tridiagonal (w.d, w.e): ascending
// eigenvalues in w.d, eigenvectors in w.Q (row-major, columns).
static void stedc(int n, EigWork& w, cudaStream_t st) {
  std::vector<DcNode> nodes;
  dc_build(0, n, 0, nodes);
  int* ib = w.ibuf;
  int* perm = ib;
  int* ndcol = ib + n;
  int* dcol = ib + 2L * n;
  int* rot = ib + 3L * n;     // 2n
  int* colmap = ib + 5L * n;  // n
  int* err = ib + 6L * n;     // 1
  int* pidx = ib + 7L * n;    // n: GEMM column order of the secular columns
  KOT_CUDA(cudaMemsetAsync(w.Q, 0, sizeof(double) * n * n, st));
  KOT_CUDA(cudaMemsetAsync(err, 0, sizeof(int), st));
  // host-pinned staging regions (distinct per purpose: copies are asynchronous)
  int* h_packed = w.hbuf;                                           // <= 2n + 8 ints
  char* h_desc = reinterpret_cast<char*>(w.hbuf + 2L * n + 64);      // <= n/16 descs
  char* d_desc_base = reinterpret_cast<char*>(w.dbuf);
  std::vector<int> splits, loff, llen;
  int maxdepth = 0;
  for (auto& nd : nodes) {
    maxdepth = std::max(maxdepth, nd.depth);
    if (nd.leaf) {
      loff.push_back(nd.o);
      llen.push_back(nd.n);
    } else {
      splits.push_back(nd.o + nd.n / 2 - 1);
    }
  }
  std::vector<int> packed;
  packed.insert(packed.end(), splits.begin(), splits.end());
  packed.insert(packed.end(), loff.begin(), loff.end());
  packed.insert(packed.end(), llen.begin(), llen.end());
  std::copy(packed.begin(), packed.end(), h_packed);
  int* d_packed = reinterpret_cast<int*>(d_desc_base);
  KOT_CUDA(cudaMemcpyAsync(d_packed, h_packed, sizeof(int) * packed.size(), cudaMemcpyHostToDevice, st));
  const int* dsplit = d_packed;
  const int* dloff = d_packed + splits.size();
  const int* dllen = dloff + loff.size();
  if (!splits.empty()) {
    dc_split_kernel<<<1, DC_SPLIT_THREADS, 0, st>>>(w.d, w.e, n, dsplit, (int)splits.size(), w.rho + n);
    KOT_LAUNCH_CHECK();
  }
  const int nleaves = (int)loff.size();
  ProfScope ps_leaf("dc.leaf", st);
  dc_leaf_kernel<<<ceil_div(nleaves, LEAF_WARPS), 32 * LEAF_WARPS, 0, st>>>(w.d, w.e, dloff, dllen, nleaves, w.Q, n, err);
  KOT_LAUNCH_CHECK();
  // all levels' merge descriptors uploaded once; each level gets its own meta region, so the
  // whole merge tree runs without a host round trip (kernels read K from device memory)
  const size_t packed_bytes = ((sizeof(int) * packed.size() + 63) / 64) * 64;
  std::vector<std::vector<MergeDesc>> levels;
  for (int depth = maxdepth; depth >= 0; --depth) {
    std::vector<MergeDesc> ms;
    long off = 0;
    for (auto& nd : nodes)
      if (!nd.leaf && nd.depth == depth) {
        ms.push_back({nd.o, nd.n / 2, nd.n - nd.n / 2, off});
        off += (long)nd.n * (nd.n + 1);  // room for an even leading dimension
        off += off & 1;                  // keep every region 16 B aligned
      }
    if (!ms.empty()) levels.push_back(ms);
  }
  size_t ndesc = 0;
  for (auto& l : levels) ndesc += l.size();
  MergeDesc* dms_all = reinterpret_cast<MergeDesc*>(d_desc_base + packed_bytes);
  int* dmeta_all = reinterpret_cast<int*>(dms_all + ndesc);
  {
    size_t k = 0;
    for (auto& l : levels)
      for (auto& m : l) reinterpret_cast<MergeDesc*>(h_desc)[k++] = m;
    KOT_CUDA(cudaMemcpyAsync(dms_all, h_desc, sizeof(MergeDesc) * ndesc, cudaMemcpyHostToDevice, st));
  }
  size_t base = 0;
  for (auto& ms : levels) {
    const int nm = (int)ms.size();
    MergeDesc* dms = dms_all + base;
    int* dmeta = dmeta_all + MS * base;
    base += nm;
    int maxm = 0;
    for (auto& mm : ms) maxm = std::max(maxm, mm.n1 + mm.n2);
    {
      ProfScope ps_prep("dc.prep", st);
      const size_t smem = (size_t)maxm * (3 * sizeof(double) + sizeof(int));
      ensure_smem_attr((const void*)dc_merge_prep_kernel, (int)smem);
      dc_merge_prep_kernel<<<nm, DC_PREP_THREADS, smem, st>>>(dms, w.Q, n, w.d, w.e, w.zs, w.ds, w.dlam, w.wv,
                                                              w.dfv, w.rotcs, w.rho, perm, ndcol, dcol, rot, dmeta,
                                                              pidx, w.rho + n);
      KOT_LAUNCH_CHECK();
    }
    {
      ProfScope ps_vec("dc.gather_rot", st);
      const size_t smem = (size_t)maxm * sizeof(double);
      ensure_smem_attr((const void*)dc_merge_vec_kernel, (int)smem);
      dc_merge_vec_kernel<<<dim3(maxm, nm), 256, smem, st>>>(dms, w.Q, w.Qw, w.Qnd, n, perm, ndcol, dcol, rot,
                                                             w.rotcs, dmeta, pidx);
      KOT_LAUNCH_CHECK();
    }
    {
      ProfScope ps_sec("dc.secular", st);
      const dim3 grid(ceil_div(maxm, 8), nm);
      dc_secular_kernel<<<grid, 256, 0, st>>>(dms, dmeta, w.dlam, w.wv, w.rho, w.lam, w.Dl, err);
      KOT_LAUNCH_CHECK();
      dc_what_kernel<<<grid, 256, 0, st>>>(dms, dmeta, w.dlam, w.wv, w.Dl, w.what);
      KOT_LAUNCH_CHECK();
      dc_vec_kernel<<<grid, 256, 0, st>>>(dms, dmeta, w.what, w.Dl, w.Uw, pidx);
      KOT_LAUNCH_CHECK();
    }
    ProfScope ps_ord("dc.order_gemm", st);
    dc_order_kernel<<<nm, 256, 0, st>>>(dms, dmeta, w.lam, w.dfv, w.d, colmap);
    KOT_LAUNCH_CHECK();
    dc_copy_deflated_kernel<<<dim3(64, nm), 256, 0, st>>>(dms, dmeta, w.Qw, w.Q, n, colmap);
    KOT_LAUNCH_CHECK();
    // Q_new = Qnd·U with Qnd's columns ordered (top-only | mixed | bottom-only): the top rows only
    // see the first c12 columns, the bottom rows only the last K − c1 (dlaed3 structure).  K, c1, c12
    // are read on the device; every merge of the level in one grouped launch per row half (the top-only
    // columns are exact zeros in the bottom rows, so an aligned K start is harmless there).
    {
      int mmax = 0, nnmax = 0;
      for (auto& mm : ms) {
        mmax = std::max(mmax, std::max(mm.n1, mm.n2));
        nnmax = std::max(nnmax, mm.n1 + mm.n2);
      }
      const int tiles = ceil_div(mmax, GB_M) * ceil_div(nnmax, GB_N);
      constexpr int smem = GTile<GB_M, GB_N>::SMEM;
      auto k = gemm_dmma_kernel<false, true, 2, EpiColMapGroup>;
      ensure_smem_attr((const void*)k, smem);
      for (int half = 0; half < 2; ++half) {
        GemmShape s = make_shape(mmax, nnmax, nnmax, w.Qnd, nnmax, w.Uw, nnmax);  // rewritten per group
        const int cap = gemm_cta_cap();
        const int ctas = cap > 0 ? std::max(1, std::min(tiles, cap / nm)) : tiles;
        k<<<dim3(ctas, 1, nm), G_THREADS, smem, st>>>(s, EpiColMapGroup{w.Q, n, colmap, dms, dmeta, w.Qnd, w.Uw,
                                                                       half}, tiles);
        KOT_LAUNCH_CHECK();
      }
    }
  }
  int herr = 0;
  KOT_CUDA(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, st));
  KOT_CUDA(cudaStreamSynchronize(st));
  if (herr)
    throw KotError(KOT_EEIG, herr == 1 ? "tridiagonal QL failed to converge"
                                       : "secular equation solver failed to converge");
}

// ====================================================== back-transform

// T factor of the forward block reflector (dlarft 'F','C').  Instead of the
// sequential recurrence T[0:i,i] = −τ_i T[0:i,0:i] S[0:i,i], use the identity
// T⁻¹ = diag(1/τ) + striu(VᵀV) (forward columnwise compact WY) and invert the
// upper triangle column-parallel: one warp per column, back substitution with
// warp-reduced dot products.  Reflectors with τ = 0 (H = I) were stored as a
// zero column of V by sytrd, which decouples them (T_ii = 1, no contribution).
constexpr int ORM_NB = 128;
constexpr int LARFT_THREADS = 512;
constexpr int LARFT_LDS = ORM_NB + 1;
constexpr int LARFT_SMEM = ORM_NB * LARFT_LDS * 8;  // S staged in shared memory

__global__ void __launch_bounds__(LARFT_THREADS) larft_kernel(const double* __restrict__ Sg, const double* tau,
                                                              int nb, double* T) {
  extern __shared__ double S_s[];  // [nb][LARFT_LDS]
  __shared__ double tcol[LARFT_THREADS / 32][ORM_NB];
  __shared__ double dinv[ORM_NB];  // 1/U_ii = τ_i (1 for τ_i = 0)
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) S_s[(e / nb) * LARFT_LDS + e % nb] = Sg[e];
  for (int i = threadIdx.x; i < nb; i += blockDim.x) dinv[i] = tau[i] != 0.0 ? tau[i] : 1.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int c = blockIdx.x * (LARFT_THREADS / 32) + wid;  // column of T
  if (c >= nb) return;
  double* t = tcol[wid];
  // Back substitution by columns: lane L keeps the running sums of rows L, L+32, L+64, L+96; once
  // t_j is known (computed by its owner lane and broadcast), every row i < j adds S_ij t_j.  One
  // shuffle + one FMA per step instead of a warp reduction per step.
  static_assert(ORM_NB <= 128, "4 rows per lane");
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  for (int j = c; j >= 0; --j) {
    const int q = j >> 5;
    const double sq = q == 0 ? s0 : (q == 1 ? s1 : (q == 2 ? s2 : s3));
    const double cand = (j == c) ? dinv[c] : -sq * dinv[j];
    const double tj = __shfl_sync(0xffffffffu, cand, j & 31);
    if (lane == (j & 31)) t[j] = tj;
    const int i0 = lane, i1 = lane + 32, i2 = lane + 64, i3 = lane + 96;
    if (i0 < j) s0 += S_s[j * LARFT_LDS + i0] * tj;  // S = VᵀV symmetric: row j, conflict-free
    if (i1 < j) s1 += S_s[j * LARFT_LDS + i1] * tj;  // S = VᵀV symmetric: row j, conflict-free
    if (i2 < j) s2 += S_s[j * LARFT_LDS + i2] * tj;  // S = VᵀV symmetric: row j, conflict-free
    if (i3 < j) s3 += S_s[j * LARFT_LDS + i3] * tj;  // S = VᵀV symmetric: row j, conflict-free
  }
  __syncwarp();
  for (int i = lane; i < nb; i += 32) T[(long)i * nb + c] = (i <= c) ? t[i] : 0.0;
}

__global__ void reverse_cols_kernel(const double* Q, const double* dasc, double* P, double* vals, int n) {
  const long total = (long)n * n;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
    const int r = (int)(e / n), c = (int)(e % n);
    P[e] = Q[(long)r * n + (n - 1 - c)];
  }
  if (blockIdx.x == 0)
    for (int i = threadIdx.x; i < n; i += blockDim.x) vals[i] = dasc[n - 1 - i];
}

__global__ void count_pos_kernel(const double* vals, int n, int* k) {
  __shared__ int cnt[32];
  int c = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) c += (vals[i] > 0.0) ? 1 : 0;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) cnt[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += cnt[w];
    *k = s;
  }
}

// Back-transform P ← H_0 H_1 ⋯ H_{n−2} P in compact-WY blocks of ORM_NB
// reflectors (I − V T Vᵀ), last block first: W1 = Vᵀ P (split-K), W2 = T W1,
// P −= V W2.
// dcols (nullable, device): only the first *dcols columns of P are transformed.
// T factor of every 128-reflector block (S = VᵀV, larft) on w.st_t: nothing here depends on the
// tridiagonal eigenvectors, so it runs beside stedc and ormtr only waits for w.ev_t1.
static void tfactors_async(int n, EigWork& w, cudaStream_t st) {
  w.ensure_tfactors();
  const int nref = n - 1;
  const int nblk = (nref + ORM_NB - 1) / ORM_NB;
  KOT_CUDA(cudaEventRecord(w.ev_t0, st));
  KOT_CUDA(cudaStreamWaitEvent(w.st_t, w.ev_t0, 0));
  for (int bi = 0; bi < nblk; ++bi) {
    const int p0 = bi * ORM_NB;
    const int nb = std::min(ORM_NB, nref - p0);
    const int r0 = p0 + 1;
    const double* Vp = w.Vall + (long)r0 * n + p0;
    GemmShape s = make_shape(nb, nb, n - r0, Vp, n, Vp, n);  // S = Vᵀ V (symmetric, one triangle mirrored)
    s.sym_tiles = 1;
    s.ws = w.ws_t;
    s.ksplit = choose_ksplit(s, 16L * 128 * 128);
    gemm_launch<true, false>(s, EpiSymMirror{w.Sside, nb, 1.0, nullptr, 0.0, 0.0}, w.st_t);
    ProfScope pl("orm.larft", w.st_t);
    ensure_smem_attr((const void*)larft_kernel, LARFT_SMEM);
    larft_kernel<<<ceil_div(nb, LARFT_THREADS / 32), LARFT_THREADS, LARFT_SMEM, w.st_t>>>(
        w.Sside, w.tau + p0, nb, w.Tall + (long)bi * ORM_NB * ORM_NB);
    KOT_LAUNCH_CHECK();
    // VT = V·T (T upper triangular, zero below the diagonal): the back-transform then needs two GEMMs
    // per block, P −= (V T)(Vᵀ P), instead of three
    double* VTp = w.VT + (long)r0 * n + p0;
    gemm_launch<false, false>(make_shape(n - r0, nb, nb, Vp, n, w.Tall + (long)bi * ORM_NB * ORM_NB, nb),
                              EpiAxpby{VTp, n, 1.0, 0.0}, w.st_t);
  }
  KOT_CUDA(cudaEventRecord(w.ev_t1, w.st_t));
}

static void ormtr(int n, EigWork& w, double* P, cudaStream_t st, const int* dcols = nullptr) {
  const int nref = n - 1;  // reflectors 0..n-2
  const int nblk = (nref + ORM_NB - 1) / ORM_NB;
  double* W1 = w.W1;
  KOT_CUDA(cudaStreamWaitEvent(st, w.ev_t1, 0));  // T factors and V·T (tfactors_async)
  for (int bi = nblk - 1; bi >= 0; --bi) {
    const int p0 = bi * ORM_NB;
    const int nb = std::min(ORM_NB, nref - p0);
    const int r0 = p0 + 1;
    const int mrows = n - r0;
    const double* Vp = w.Vall + (long)r0 * n + p0;  // mrows × nb (ld n), zero above each unit entry
    const double* VTp = w.VT + (long)r0 * n + p0;   // V·T of the block (tfactors_async)
    {  // W1 = Vᵀ P[r0:, :]
      GemmShape s = make_shape(nb, n, mrows, Vp, n, P + (long)r0 * n, n);
      s.dN = dcols;
      s.ws = w.splitws;
      s.ksplit = choose_ksplit(s, w.splitws_cap);
      gemm_launch<true, false>(s, EpiAxpby{W1, n, 1.0, 0.0}, st);
    }
    {  // P[r0:, :] −= (V T) W1
      GemmShape s = make_shape(mrows, n, nb, VTp, n, W1, n);
      s.dN = dcols;
      gemm_launch<false, false>(s, EpiAxpby{P + (long)r0 * n, n, -1.0, 1.0}, st);
    }
  }
}

__global__ void eig1_kernel(const double* Z, double* P, double* vals) {
  vals[0] = Z[0];
  P[0] = 1.0;
}

static int sytrd_per_sm(int n) {
  const size_t smem = sizeof(double) * (std::max(n, 1) + 3L * TRD_WARPS * TRD_RPW * TRD_NB);
  ensure_smem_attr((const void*)sytrd_panel_kernel, (int)smem);
  int per_sm = 0;
  KOT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sytrd_panel_kernel, TRD_THREADS, smem));
  return std::max(1, per_sm);
}

// Which tridiagonalisation an eigensolve uses (measured on B200, DESIGN.md §3/§5).
// Below ℓ ≈ 3000 the one-stage sytrd wins (ℓ = 2000: 35 vs 42 ms alone, 7.9 vs
// 5.2 it/s in the solver); from ℓ = 3000 on the two-stage path wins in the solver
// (3000: 3.39 vs 3.26 it/s; 4096: 1.60 vs 1.51; 8192: 0.435 vs 0.316 it/s): the
// one-stage panel streams the whole trailing matrix from HBM once per column,
// the two-stage path once per 16-column panel.  KOT_EIG_STAGES=1|2 (or
// kot_debug_eig_stages) forces either; 3 = two-stage for background eigensolves only.
constexpr int kTwoStageMinOrder = 3000;
static int g_eig_stages = -1;  // −1: read KOT_EIG_STAGES once (0 = automatic)
bool use_two_stage(int n, int lane) {
  if (g_eig_stages < 0) {
    const char* e = std::getenv("KOT_EIG_STAGES");
    g_eig_stages = e ? std::atoi(e) : 0;
  }
  if (n < 3) return false;
  switch (g_eig_stages) {
    case 1: return false;
    case 2: return true;
    case 3: return lane != 0;
    default: return n >= kTwoStageMinOrder;
  }
}

static void one_stage_tridiag(const double* Z, int n, EigWork& w, cudaStream_t st, int lane) {
  ProfScope ps("eig.sytrd", st, 4.0 / 3.0 * n * (double)n * n);
  const int total = sytrd_per_sm(n) * kNumSMs;
  CoopGate gate(total, trd_grid(n, lane), trd_grid(n, 0), lane);
  sytrd(Z, n, w, st, lane, &gate, total / kNumSMs);
  KOT_CUDA(cudaStreamSynchronize(st));  // the gate is held until the grids have retired
  if (w.mid_used) {
    w.mid_used = false;
    kot_require(*w.mid_err_host == 0, KOT_EEIG, "sytrd mid kernel: an exchange timed out (grid not co-resident)");
  }
}

void tridiag_device(const double* Z, int n, EigWork& w, cudaStream_t st, int stages) {
  kot_require(n >= 2, KOT_EINVAL, "order must be >= 2");
  if (stages == 2 && n >= 3)
    two_stage_tridiag(Z, n, w, st);
  else
    one_stage_tridiag(Z, n, w, st, 0);
}

void syevd_device(const double* Z, int n, double* P, double* vals, int* dk, EigWork& w, cudaStream_t st,
                  int lane, bool alpha_only) {
  if (n == 1) {
    eig1_kernel<<<1, 1, 0, st>>>(Z, P, vals);
    KOT_LAUNCH_CHECK();
  } else {
    const bool two = use_two_stage(n, lane);
    if (two)
      two_stage_tridiag(Z, n, w, st);
    else
      one_stage_tridiag(Z, n, w, st, lane);
    w.check_cancel(st);
    tfactors_async(n, w, st);
    {
      ProfScope ps("eig.stedc", st);
      stedc(n, w, st);
    }
    w.check_cancel(st);
    ProfScope ps("eig.ormtr", st, 2.0 * n * (double)n * n);
    reverse_cols_kernel<<<std::min(ceil_div((long)n * n, 256), 2048), 256, 0, st>>>(w.Q, w.d, P, vals, n);
    KOT_LAUNCH_CHECK();
    // α-only (PSD projection): the back-transforms act on the σ > 0 columns only (k read on device)
    const int* dcols = nullptr;
    if (alpha_only) {
      count_pos_kernel<<<1, 256, 0, st>>>(vals, n, dk);
      KOT_LAUNCH_CHECK();
      dcols = dk;
    }
    if (two) two_stage_q2_apply(n, w, P, st, dcols);
    ormtr(n, w, P, st, dcols);
  }
  count_pos_kernel<<<1, 256, 0, st>>>(vals, n, dk);
  KOT_LAUNCH_CHECK();
}

}  // namespace kot

extern "C" int kot_debug_tail_timing(int on, unsigned long long* out8) {
  using namespace kot;
  try {
    if (on) {
      if (!g_tail_dbg) KOT_CUDA(cudaMalloc(&g_tail_dbg, 8 * sizeof(unsigned long long)));
      KOT_CUDA(cudaMemset(g_tail_dbg, 0, 8 * sizeof(unsigned long long)));
    } else if (g_tail_dbg) {
      KOT_CUDA(cudaDeviceSynchronize());
      KOT_CUDA(cudaMemcpy(out8, g_tail_dbg, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
      cudaFree(g_tail_dbg);
      g_tail_dbg = nullptr;
    }
    return 0;
  } catch (const KotError& e) {
    return e.code;
  }
}

extern "C" int kot_debug_sytrd_timing(int on, unsigned long long* out8) {
  // on=1: allocate + zero the segment accumulators; on=0: copy them out and disable
  using namespace kot;
  try {
    if (on) {
      if (!g_trd_dbg) KOT_CUDA(cudaMalloc(&g_trd_dbg, 8 * sizeof(unsigned long long)));
      KOT_CUDA(cudaMemset(g_trd_dbg, 0, 8 * sizeof(unsigned long long)));
    } else if (g_trd_dbg) {
      KOT_CUDA(cudaDeviceSynchronize());
      KOT_CUDA(cudaMemcpy(out8, g_trd_dbg, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
      cudaFree(g_trd_dbg);
      g_trd_dbg = nullptr;
    }
    return 0;
  } catch (const KotError& e) {
    return e.code;
  }
}

// test hook: 0 = automatic, 1 = one-stage, 2 = two-stage, 3 = two-stage for background eigensolves
extern "C" int kot_debug_eig_stages(int stages) {
  kot::g_eig_stages = (stages >= 0 && stages <= 3) ? stages : 0;
  return 0;
}

// test hook: mode 0 off / 1 latency-critical eigensolves / 2 every eigensolve; tail = trailing columns
// handed to the cluster tail (0: the mid kernel runs to the last column); negative = leave unchanged
extern "C" int kot_debug_trd_mid(int mode, int tail) {
  kot::mid_mode();
  if (mode >= 0) kot::g_mid_mode = mode;
  if (tail >= 0) kot::g_mid_tail = tail;
  return 0;
}

extern "C" int kot_debug_mid_timing(int on, unsigned long long* out8) {
  using namespace kot;
  try {
    if (on) {
      if (!g_mid_dbg) KOT_CUDA(cudaMalloc(&g_mid_dbg, 8 * sizeof(unsigned long long)));
      KOT_CUDA(cudaMemset(g_mid_dbg, 0, 8 * sizeof(unsigned long long)));
    } else if (g_mid_dbg) {
      KOT_CUDA(cudaDeviceSynchronize());
      KOT_CUDA(cudaMemcpy(out8, g_mid_dbg, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
      cudaFree(g_mid_dbg);
      g_mid_dbg = nullptr;
    }
    return 0;
  } catch (const KotError& e) {
    return e.code;
  }
}

// clock64 stamps of the mid kernel: [8 columns from c0][16 warps][16 points] of CTA `cta` (on = 1 arms, 0 reads)
extern "C" int kot_debug_mid_trace(int on, int c0, int cta, long long* out) {
  using namespace kot;
  const size_t bytes = sizeof(long long) * MID_TRACE_COLS * MID_WARPS * MID_TRACE_PTS;
  try {
    if (on) {
      if (!g_mid_trace) KOT_CUDA(cudaMalloc(&g_mid_trace, bytes));
      KOT_CUDA(cudaMemset(g_mid_trace, 0, bytes));
      g_mid_trace_c0 = c0;
      g_mid_trace_cta = cta;
    } else if (g_mid_trace) {
      KOT_CUDA(cudaDeviceSynchronize());
      KOT_CUDA(cudaMemcpy(out, g_mid_trace, bytes, cudaMemcpyDeviceToHost));
      cudaFree(g_mid_trace);
      g_mid_trace = nullptr;
    }
    return 0;
  } catch (const KotError& e) {
    return e.code;
  }
}

// ---- host-only hooks (no GPU needed): shared-memory capacity rule and a gate self-test ----

// largest order of the mid kernel's resident block for a grid of G CTAs with smem_max bytes of dynamic
// shared memory per CTA
extern "C" int kot_debug_mid_capacity(int grid, long smem_max) {
  if (grid < 1 || smem_max < 0) return -1;
  return kot::mid_capacity(grid, (size_t)smem_max);
}

// Exercises the cooperative-grid gate for `ms` milliseconds with `nbg` background threads (panel loops
// that yield between panels) and one foreground thread that opens exclusive windows.  Returns the
// number of exclusive windows completed, or a negative code: −1 a background grid was in flight inside
// a window before its re-opening, −2 the slot accounting did not return to zero, −3 no window opened.
extern "C" int kot_debug_gate_selftest(int nbg, int ms) {
  using namespace kot;
  using clk = std::chrono::steady_clock;
  const int total = 2 * kNumSMs;
  std::atomic<bool> stop{false};
  std::atomic<int> in_panel{0}, bad{0}, windows{0};
  std::atomic<bool> window_closed{false};
  std::vector<std::thread> th;
  for (int t = 0; t < nbg; ++t)
    th.emplace_back([&, t] {
      while (!stop.load()) {
        CoopGate g(total, t % 2 ? 16 : 24, 96, 1 + t % 2);
        for (int p = 0; p < 40 && !stop.load(); ++p) {
          g.yield_to_exclusive(nullptr);
          ++in_panel;
          if (window_closed.load()) ++bad;  // admitted while a window was closed
          std::this_thread::sleep_for(std::chrono::microseconds(30));
          --in_panel;
        }
      }
    });
  std::thread fg([&] {
    while (!stop.load()) {
      CoopGate g(total, 96, 96, 0);
      std::this_thread::sleep_for(std::chrono::microseconds(200));  // its own panels
      g.exclusive_begin();
      // Background threads sample window_closed after their yield: give one that passed its yield
      // point just before the window its 30 µs panel, then nobody may be inside.
      window_closed = true;
      std::this_thread::sleep_for(std::chrono::microseconds(100));
      if (in_panel.load() != 0) ++bad;
      window_closed = false;
      g.exclusive_end(96, 2);
      std::this_thread::sleep_for(std::chrono::microseconds(300));  // the resident kernel, others beside it
      ++windows;
    }
  });
  std::this_thread::sleep_for(std::chrono::milliseconds(ms));
  stop = true;
  fg.join();
  for (auto& t : th) t.join();
  (void)clk::now();
  if (bad.load() != 0) return -1;
  {
    std::lock_guard<std::mutex> lk(g_coop_mu);
    if (g_coop_used != 0 || g_coop_fg != 0 || g_coop_excl) return -2;
  }
  return windows.load() > 0 ? windows.load() : -3;
}

// test hook: 0 no head launch, 1 beside an EG pipeline (default), 2 also for standalone eigensolves
extern "C" int kot_debug_trd_mid_head(int mode) {
  kot::g_mid_head = (mode >= 0 && mode <= 2) ? mode : 1;
  return 0;
}
