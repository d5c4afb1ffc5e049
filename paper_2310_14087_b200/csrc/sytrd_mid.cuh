// sytrd "mid" kernel: unblocked Householder tridiagonalisation (dsytd2, lower) of a trailing block
// that fits in the shared memory of the WHOLE grid (one CTA per SM, rows r ≡ blockIdx mod G, full
// symmetric rows), included by eig.cu.  Replaces the cooperative panel kernel (reference path:
// np.linalg.eigh in linalg.py:60-83) for every column whose trailing matrix is at most
// G × ~180 KB: 1776 columns of an ℓ = 2000 eigensolve on 148 SMs.
//
// Why: the panel kernel pays, per column, two grid barriers, the reduction of the panel corrections
// (Wᵀv, Vᵀv partials) and a symv that streams the trailing matrix through L2 — ≈ 12.5 µs per column.
// Here the matrix never leaves shared memory and a column needs ONE exchange:
//
//   with y = A v (column c's symv), w = τ y + α₂ v, α₂ = −½ τ² (yᵀv), and v_{c+1} = 1, the next
//   column after the rank-2 update is   x_{c+1} = A[:, c+1] − v w_{c+1} − w v_{c+1} = p − κ v,
//   p_r = A_{r,c+1} − τ y_r  (local to the owner of row r),   κ = τ y_{c+1} + 2 α₂  (a scalar).
//
// So every CTA publishes (y_r, p_r) for its rows and, after ONE all-gather, derives w, the next
// column, its norm and the Householder scalars redundantly — fixed-order sums, so all CTAs take
// bit-identical decisions.  The all-gather goes through TAGGED 32-byte sectors in global memory
// ({3 doubles, tag}: one 256-bit store, one 256-bit load — the sector is L2's access granule, the
// tag validates the payload, so a consumer polls the data itself; no grid barrier, no flag round
// trip).  A sector can be written to R replicas with a CTA reading replica blockIdx mod R
// (KOT_TRD_MID_REP); measured, one copy is fastest — the exchange costs the all-to-all skew of 148
// CTAs (≈ 2300–2800 cycles, tools/microbench/hop_bench.cu), not hot L2 lines — so R = 1 by default.
//
// The Householder scalars of a column stay off the critical path: the symv runs on the UNSCALED column
// (Â v = s (Â x̃ − β Â[:, c+1]), s = 1/(α − β)) while warp 15 derives β, τ, s, and x̃ is scaled into v
// while warp 0 publishes.  The column loop is kept small enough for the SM's instruction cache.
//
// The shared-memory copy runs ONE rank-2 update behind (dlatrd with a panel of one): column c's symv
// is a read-only pass over the stale rows, corrected per row with the two dot products w_{c−1}·v_c
// and v_{c−1}·v_c (every CTA has all vectors), and update c−1 is applied to the rows while the
// exchange of column c is in flight — off the critical path.
//
// Sector reuse is safe without barriers because of the data dependences: exchange c+2 (same parity
// buffer as exchange c) can only be published after exchange c+1 was gathered, which every CTA
// publishes after it finished gathering exchange c.  All CTAs must be co-resident (they spin on each
// other's sectors): launched cooperatively.
#pragma once

namespace kot {

constexpr int MID_THREADS = 512;
constexpr int MID_WARPS = MID_THREADS / 32;
constexpr int MID_MAX = 2048;                     // order of the resident block
constexpr int MID_RPC_MAX = 18;                   // rows per CTA
constexpr int MID_NTR_MAX = MID_RPC_MAX / 3;      // row triples per CTA
constexpr int MID_SPC = 2 * MID_NTR_MAX;          // sector stride per CTA (y triples, then p triples)
constexpr int MID_TPT = (kNumSMs * MID_NTR_MAX + MID_THREADS - 1) / MID_THREADS;  // polled row triples per thread
constexpr int MID_REP_MAX = 8;                    // replicas of every published sector
constexpr int MID_RG = 4;                         // rows per warp in the row passes
constexpr unsigned MID_SPIN_LIMIT = 1u << 21;     // polls before a gather gives up (error, no hang)

struct MidSector {  // 32 bytes, 32-byte aligned: L2's access granule
  unsigned long long a, b, c, tag;
};
static_assert(sizeof(MidSector) == 32, "sector layout");

struct MidArgs {
  double* A;        // n × n (ld n): trailing block at (c0, c0) fully updated and symmetric
  int n, c0, cend;  // local columns [0, cend) are reduced here, cend ≤ m0 − 1 (m0 = n − c0)
  double* d;
  double* e;
  double* tau;
  double* Vall;      // reflector c (global index) in column c, rows > c; v_{c+1} = 1
  MidSector* xchg;   // [2 parities][nrep][G][MID_SPC] tagged sectors
  int nrep;
  unsigned long long epoch0;  // launch sequence number << 12: tags = epoch0 + column + 2
  int* err;                 // set to 1 when a gather timed out
  unsigned* resident;       // host-mapped: CTA 0 stores epoch0 after its first gather (every CTA is resident)
  unsigned long long* dbg;  // nullable: per-segment ns accumulated by CTA 0 thread 0
  long long* trace;         // nullable: clock64 stamps [MID_TRACE_COLS][MID_WARPS][MID_TRACE_PTS] of CTA trace_cta
  int trace_c0, trace_cta;
};
constexpr int MID_TRACE_COLS = 8, MID_TRACE_PTS = 16;
unsigned long long* g_mid_dbg = nullptr;  // set by kot_debug_mid_timing
long long* g_mid_trace = nullptr;         // set by kot_debug_mid_trace
int g_mid_trace_c0 = 0, g_mid_trace_cta = 0;

__device__ __forceinline__ void mid_put(MidSector* s, double v0, double v1, double v2, unsigned long long tag) {
  asm volatile("st.relaxed.gpu.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(s), "l"(__double_as_longlong(v0)),
               "l"(__double_as_longlong(v1)), "l"(__double_as_longlong(v2)), "l"(tag)
               : "memory");
}
__device__ __forceinline__ bool mid_try(const MidSector* s, unsigned long long tag, double& v0, double& v1,
                                        double& v2) {
  unsigned long long a, b, c, t;
  asm volatile("ld.relaxed.gpu.global.v4.b64 {%0, %1, %2, %3}, [%4];"
               : "=l"(a), "=l"(b), "=l"(c), "=l"(t)
               : "l"(s)
               : "memory");
  if (t != tag) return false;
  v0 = __longlong_as_double((long long)a);
  v1 = __longlong_as_double((long long)b);
  v2 = __longlong_as_double((long long)c);
  return true;
}

// fixed-order tree sum of the 16 per-warp partials (the same code, hence the same bits, in every CTA)
__device__ __forceinline__ double mid_sum16(const double* r) {
  const double2* r2 = reinterpret_cast<const double2*>(r);
  const double2 a = r2[0], b = r2[1], c = r2[2], d = r2[3], e = r2[4], f = r2[5], g = r2[6], h = r2[7];
  return (((a.x + a.y) + (b.x + b.y)) + ((c.x + c.y) + (d.x + d.y))) +
         (((e.x + e.y) + (f.x + f.y)) + ((g.x + g.y) + (h.x + h.y)));
}

// three warp sums at once by a transposed butterfly (6 adds instead of 15): the totals of a, b, c end
// up in lanes 0, 8 and 16
__device__ __forceinline__ double mid_warp_sum3(double a, double b, double c, int lane) {
  const bool h16 = lane & 16, h8 = lane & 8;
  double k0 = h16 ? c : a, k1 = h16 ? 0.0 : b;
  k0 += __shfl_xor_sync(0xffffffffu, h16 ? a : c, 16);
  k1 += __shfl_xor_sync(0xffffffffu, h16 ? b : 0.0, 16);
  double t = (h8 ? k1 : k0) + __shfl_xor_sync(0xffffffffu, h8 ? k0 : k1, 8);
  t += __shfl_xor_sync(0xffffffffu, t, 4);
  t += __shfl_xor_sync(0xffffffffu, t, 2);
  t += __shfl_xor_sync(0xffffffffu, t, 1);
  return t;
}

// The row passes run on a 2-D warp grid: WR = ⌈live rows / 4⌉ row groups × WC = 15 / WR column chunks
// (warp 15 is kept out of them: it derives the Householder scalars beside the symv pass);
// warp (rg, cc) handles the 4 rows q0 … q0+3 (clamped to the last row; `nr` of them exist) on the
// double2 columns [i0, i1) counted from column `base` (even).
//
// symv: partial row-dots with x (read-only); the 4 × 32 lane partials are reduced by a transposed
// butterfly (12 shuffles instead of 40) and land in ypart[q − qlo][cc].
__device__ __forceinline__ void mid_symv_pass(const double* Aloc, int ld, int q0, int nr, int qlast, int qlo,
                                              int base, int i0, int i1, const double* x, int cchunk,
                                              double (*ypart)[MID_WARPS], int lane) {
  const double2* A2[MID_RG];
  double a0[MID_RG], a1[MID_RG];
#pragma unroll
  for (int j = 0; j < MID_RG; ++j) {
    A2[j] = reinterpret_cast<const double2*>(Aloc + (long)min(q0 + j, qlast) * ld + base);
    a0[j] = 0.0;
    a1[j] = 0.0;
  }
  const double2* x2 = reinterpret_cast<const double2*>(x + base);
#pragma unroll 2
  for (int i = i0 + lane; i < i1; i += 32) {
    const double2 xv = x2[i];
#pragma unroll
    for (int j = 0; j < MID_RG; ++j) {
      const double2 e = A2[j][i];
      a0[j] += e.x * xv.x;
      a1[j] += e.y * xv.y;
    }
  }
  double t0 = a0[0] + a1[0], t1 = a0[1] + a1[1], t2 = a0[2] + a1[2], t3 = a0[3] + a1[3];
  const bool h16 = lane & 16, h8 = lane & 8;
  const double s0 = h16 ? t0 : t2, s1 = h16 ? t1 : t3;
  double k0 = h16 ? t2 : t0, k1 = h16 ? t3 : t1;
  k0 += __shfl_xor_sync(0xffffffffu, s0, 16);
  k1 += __shfl_xor_sync(0xffffffffu, s1, 16);
  double b = (h8 ? k1 : k0) + __shfl_xor_sync(0xffffffffu, h8 ? k0 : k1, 8);
  b += __shfl_xor_sync(0xffffffffu, b, 4);
  b += __shfl_xor_sync(0xffffffffu, b, 2);
  b += __shfl_xor_sync(0xffffffffu, b, 1);
  const int j = lane >> 3;  // lanes 0, 8, 16, 24 hold rows 0 … 3
  if ((lane & 7) == 0 && j < nr) ypart[q0 + j - qlo][cchunk] = b;
}

// update: A_rs −= v_r w_s + w_r v_s for the warp's rows and columns
__device__ __forceinline__ void mid_update_pass(double* Aloc, int ld, int q0, int nr, int qlast, int g, int G,
                                                int base, int i0, int i1, const double* vp, const double* wp,
                                                int lane) {
  double2* A2[MID_RG];
  double vr[MID_RG], wr[MID_RG];
#pragma unroll
  for (int j = 0; j < MID_RG; ++j) {
    const int q = min(q0 + j, qlast);
    const int r = g + G * q;
    A2[j] = reinterpret_cast<double2*>(Aloc + (long)q * ld + base);
    vr[j] = vp[r];
    wr[j] = wp[r];
  }
  const double2* w2 = reinterpret_cast<const double2*>(wp + base);
  const double2* u2 = reinterpret_cast<const double2*>(vp + base);
#pragma unroll 2
  for (int i = i0 + lane; i < i1; i += 32) {
    const double2 ws = w2[i], us = u2[i];
#pragma unroll
    for (int j = 0; j < MID_RG; ++j) {
      double2 e = A2[j][i];
      e.x = e.x - vr[j] * ws.x - wr[j] * us.x;
      e.y = e.y - vr[j] * ws.y - wr[j] * us.y;
      if (j < nr) A2[j][i] = e;
    }
  }
}

// Segment timers / per-warp clock stamps (kot_debug_mid_timing, kot_debug_mid_trace) are compiled in
// only with -DKOT_MID_TRACE: the column loop has to stay inside the SM's instruction cache (≈ 32 KB
// measured, tools/microbench/icache_bench_gen.py — past it a lone warp runs at 17 cycles per
// instruction), and single-warp sections pay every instruction-fetch miss in full.
#ifdef KOT_MID_TRACE
#define MID_TR(k)                                                                                       \
  if (tracing && c >= a.trace_c0 && c < a.trace_c0 + MID_TRACE_COLS)                                    \
    a.trace[((long)(c - a.trace_c0) * MID_WARPS + wid) * MID_TRACE_PTS + (k)] = clock64();
#define MID_MARK(i)                         \
  if (timing) {                             \
    const unsigned long long t_ = gtimer(); \
    tseg[i] += t_ - tl;                     \
    tl = t_;                                \
  }
#else
#define MID_TR(k)
#define MID_MARK(i)
#endif

__global__ void __launch_bounds__(MID_THREADS, 1) sytrd_mid_kernel(MidArgs a) {
  extern __shared__ double msm[];
  const int G = gridDim.x, g = blockIdx.x;
  const int n = a.n, c0 = a.c0, m0 = n - c0, cend = a.cend;
  const int nrows = g < m0 ? (m0 - g + G - 1) / G : 0;  // own rows r = g + G q, q < nrows
  const int rpc = (m0 + G - 1) / G;
  const int ntr = (rpc + 2) / 3;  // row triples per CTA: sectors [0, ntr) carry y, [ntr, 2 ntr) carry p
  const int ld = m0 + (m0 & 1);
  double* Aloc = msm;                           // rpc × ld
  double* vwbuf = Aloc + (long)rpc * ld;        // by column parity: [v | w], 2 × 2 × ld
  __shared__ __align__(16) double red1[MID_WARPS], red2[3][MID_WARPS];
  __shared__ double scal[8];
  __shared__ __align__(16) double ypart[MID_RPC_MAX][MID_WARPS];
  __shared__ double ys[MID_RPC_MAX + 3], ps[MID_RPC_MAX + 3];
  __shared__ int dead;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

  if (tid == 0) dead = 0;
#pragma unroll 1
  for (int q = wid; q < nrows; q += MID_WARPS) {
    const double* src = a.A + (long)(c0 + g + G * q) * n + c0;
    double* dst = Aloc + (long)q * ld;
#pragma unroll 4
    for (int s = lane; s < ld; s += 32) dst[s] = (s < m0) ? src[s] : 0.0;
  }
#pragma unroll 1
  for (int s = tid; s < 4 * ld; s += MID_THREADS) vwbuf[s] = 0.0;
  if (tid < MID_RPC_MAX + 3) {
    ys[tid] = 0.0;
    ps[tid] = 0.0;
  }
  if (tid < 8) scal[tid] = 0.0;
  if (tid < MID_RPC_MAX * MID_WARPS) (&ypart[0][0])[tid] = 0.0;
  // the (up to two) row triples this thread polls: sector offset in a replica, first row, last existing
  // row (−1: none)
  int so0 = 0, so1 = 0, ra0 = 0, ra1 = 0, rl0 = -1, rl1 = -1;
#pragma unroll
  for (int u = 0; u < MID_TPT; ++u) {
    const int t = tid + u * MID_THREADS;
    if (t < G * ntr) {
      const int gg = t / ntr, j = t - gg * ntr;
      const int nrg = gg < m0 ? (m0 - gg + G - 1) / G : 0;
      const int qmax = min(3 * j + 2, nrg - 1);
      const int so = gg * MID_SPC + j, ra = gg + G * 3 * j, rl = qmax >= 3 * j ? gg + G * qmax : -1;
      if (u == 0) {
        so0 = so;
        ra0 = ra;
        rl0 = rl;
      } else {
        so1 = so;
        ra1 = ra;
        rl1 = rl;
      }
    }
  }
  static_assert(MID_TPT == 2, "two polled triples per thread");
  // the sector this lane of warp 0 publishes: k < ntr carries y of triple k, k ≥ ntr carries p
  const int pk = lane, pj = lane < ntr ? lane : lane - ntr;
  int prl = -1;
  if (lane < 2 * ntr) {
    const int qmax = min(3 * pj + 2, nrows - 1);
    prl = qmax >= 3 * pj ? g + G * qmax : -1;
  }
  const int rep = g % a.nrep;
  __syncthreads();

#ifdef KOT_MID_TRACE
  const bool timing = (a.dbg != nullptr) && g == 0 && tid == 0;
  unsigned long long tseg[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long tl = timing ? gtimer() : 0;
  const bool tracing = a.trace != nullptr && g == a.trace_cta && lane == 0;
#endif
  // Exchange c (c = −1 … cend−1) finishes column c (its w) and builds column c+1 (the unscaled x̃ and
  // the sums its Householder scalars need); c = −1 only distributes column 0 (τ = 0, v = 0).
  //
  // The scalars of column c (β, τ, 1/(α − β): a chain of ~100 dependent instructions) stay off the
  // critical path: the symv runs on the UNSCALED column, v = s (x̃ − β e_{c+1}) with s = 1/(α − β) gives
  // Â v = s (Â x̃ − β Â[:, c+1]), and warp 15 derives the scalars beside the pass; x̃ is scaled into v
  // (and the reflector stored) while warp 0 publishes.
  double tau = 0.0;  // τ of column c
  int qlo = 0;       // first live row of the CTA (r > c)
  // 2-D warp grid of the row passes, recomputed when the number of row groups changes
  int WR = -1, WC = MID_WARPS - 1, winv = 0, wrg = 0, wcc = 0;
#pragma unroll 1
  for (int c = -1; c < cend; ++c) {
    const int par = c & 1;
    double* vn = vwbuf + par * 2L * ld;  // x̃ then v of column c, and (w slot) its y then w
    double* wn = vn + ld;
    double* vq = vwbuf + (par ^ 1) * 2L * ld;  // column c−1's v and w (update in flight), then column c+1's x̃
    const double* wp = vq + ld;
    const unsigned long long tag = a.epoch0 + (unsigned)(c + 2);
    MidSector* xb = a.xchg + (long)par * a.nrep * G * MID_SPC;
    const bool pend = c >= 1;  // the rows still lack column c−1's rank-2 update
    MID_TR(0)
    if (qlo < nrows && g + G * qlo <= c) ++qlo;
    const int base = (c + 1) & ~1;
    const int n2 = (ld - base) >> 1;
    {
      const int nlive = nrows - qlo;
      const int wr = (nlive + MID_RG - 1) / MID_RG;
      if (wr != WR) {  // rare: a row group died
        WR = wr;
        WC = WR > 0 ? (MID_WARPS - 1) / WR : MID_WARPS - 1;  // column chunks (WR ≤ 5: at least 3)
        wrg = wid / WC;
        wcc = wid - wrg * WC;
        winv = 65536 / WC + 1;
      }
    }
    const bool wact = wrg < WR;
    const int chunk = ((n2 * winv) >> 16) + 1;  // ≥ ⌈n2 / WC⌉
    const int i0 = wcc * chunk, i1 = min(n2, i0 + chunk);
    const int wq0 = qlo + wrg * MID_RG, wnr = min(MID_RG, nrows - wq0);
    // (1) z_r = Σ_{s>c} Â_rs x̃_s over the stale rows (warps 0 … 14) ∥ dlarfg of column c (warp 15)
    if (c >= 0) {
      if (wact) mid_symv_pass(Aloc, ld, wq0, wnr, nrows - 1, qlo, base, i0, i1, vn, wcc, ypart, lane);
      if (wid == MID_WARPS - 1) {
        // lanes 0..2 reduce the three sums; lane 0: β = −sign(α)‖(α, x)‖, τ = (β − α)/β = 1 + |α|/‖·‖,
        // 1/(α − β) = sign(α)/(|α| + ‖·‖) with one rsqrt and one reciprocal
        const double s = lane < 3 ? mid_sum16(red2[lane]) : 0.0;
        const double xn2 = __shfl_sync(0xffffffffu, s, 0);
        const double swx = __shfl_sync(0xffffffffu, s, 1), svx = __shfl_sync(0xffffffffu, s, 2);
        if (lane == 0) {
          const double alpha = vn[c + 1];
          double beta, tn, scale;
          dlarfg_scalars(alpha, xn2, beta, tn, scale);
          scal[0] = tn;
          scal[1] = scale;
          scal[2] = beta;
          scal[6] = pend ? wp[c + 1] + scale * swx : 0.0;  // w_{c−1}·v_c over the rows > c
          scal[7] = pend ? vq[c + 1] + scale * svx : 0.0;  // v_{c−1}·v_c
          if (g == 0) {
            a.e[c0 + c] = beta;
            a.tau[c0 + c] = tn;
          }
        }
      }
      MID_TR(1)
      __syncthreads();
      tau = scal[0];
    }
    MID_TR(2)
    MID_MARK(0)
    // (2) warp 0 publishes y_r = s (z_r − β Â_{r,c+1}) − v'_r t1 − w'_r t2 and p_r = A_{r,c+1} − τ y_r
    // (update c−1 applied on the fly; v', w' = column c−1's) as row triples packed into sectors; the
    // other warps scale x̃ into v and store the reflector
    if (wid == 0) {
      if (lane < nrows) {
        double y = 0.0, pv = 0.0;
        if (lane >= qlo) {
          const int r = g + G * lane;
          double ac = Aloc[(long)lane * ld + c + 1];
          if (c >= 0) {  // fixed-order sum of the column-chunk partials (unused entries are zero)
            const double2* yp = reinterpret_cast<const double2*>(ypart[lane - qlo]);
            double y0 = 0.0, y1 = 0.0, y2 = 0.0, y3 = 0.0;
#pragma unroll
            for (int k = 0; k < MID_WARPS / 4; ++k) {
              const double2 pa = yp[2 * k], pb = yp[2 * k + 1];
              y0 += pa.x;
              y1 += pa.y;
              y2 += pb.x;
              y3 += pb.y;
            }
            y = scal[1] * (((y0 + y1) + (y2 + y3)) - scal[2] * ac);
          }
          if (pend) {
            const double vr = vq[r], wr = wp[r];
            y = y - vr * scal[6] - wr * scal[7];
            ac = ac - vr * wp[c + 1] - wr * vq[c + 1];
          }
          pv = ac - tau * y;
        }
        ys[lane] = y;
        ps[lane] = pv;
      }
      __syncwarp();
      if (prl >= c + 1) {  // the sector holds a live row
        const double* src = pk < ntr ? ys : ps;
        const double v0 = src[3 * pj], v1 = src[3 * pj + 1], v2 = src[3 * pj + 2];
        for (int rp = 0; rp < a.nrep; ++rp) mid_put(xb + ((long)rp * G + g) * MID_SPC + pk, v0, v1, v2, tag);
      }
    } else if (c >= 0) {
      const double scale = scal[1];
#pragma unroll 1
      for (int r = c + 1 + tid - 32; r < m0; r += MID_THREADS - 32) vn[r] = (r == c + 1) ? 1.0 : vn[r] * scale;
    }
    MID_TR(3)
    __syncthreads();
    if (c >= 0 && tid < nrows) {
      const int r = g + G * tid;
      if (r > c) a.Vall[(long)(c0 + r) * n + c0 + c] = (tau == 0.0) ? 0.0 : vn[r];
    }
    // (3) while the exchange is in flight: the rows catch up with column c−1's update
    if (pend) {
      if (wact) mid_update_pass(Aloc, ld, wq0, wnr, nrows - 1, g, G, base, i0, i1, vq, wp, lane);
      MID_TR(4)
      __syncthreads();  // vq (column c−1's v) is free from here on
    }
    MID_MARK(1)
    // (4) gather: every thread polls the (y, p) sectors of its row triples and scatters y into wn, p into vq
    {
      const MidSector* rb = xb + (long)rep * G * MID_SPC;
      int need = (rl0 >= c + 1 ? 3 : 0) | (rl1 >= c + 1 ? 12 : 0);  // bit 2u + h: sector h (y / p) of triple u
      unsigned spins = 0;
      while (need) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (need & (1 << k)) {
            const int so = k < 2 ? so0 : so1, ra = k < 2 ? ra0 : ra1;
            double v0, v1, v2;
            if (mid_try(rb + so + (k & 1) * ntr, tag, v0, v1, v2)) {
              need &= ~(1 << k);
              double* dst = (k & 1) ? vq : wn;
              dst[ra] = v0;  // ra < m0: the triple's first row exists
              if (ra + G < m0) dst[ra + G] = v1;
              if (ra + 2 * G < m0) dst[ra + 2 * G] = v2;
            }
          }
        }
        if (need) {
          if (*(volatile int*)&dead) break;
          if (++spins > MID_SPIN_LIMIT) {
            dead = 1;
            atomicExch(a.err, 1);
            break;
          }
        }
      }
    }
    MID_TR(5)
    __syncthreads();
    if (c == -1 && g == 0 && tid == 0) {  // every producer has published: the whole grid is resident
      *reinterpret_cast<volatile unsigned*>(a.resident) = (unsigned)a.epoch0;
      __threadfence_system();
    }
    // (5) w = τ y + α₂ v (α₂ = −½ τ² yᵀv) finishes column c; x̃_{c+1} = p − κ v, κ = τ y_{c+1} + 2 α₂.
    // Thread t takes rows cc + t, cc + t + 512, …; y sits in wn, p in vq, and both are rewritten in place.
    const int cc = c + 1;
    double pyv = 0.0;
#pragma unroll 1
    for (int r = cc + tid; r < m0; r += MID_THREADS) pyv += wn[r] * vn[r];
    const double ycc = wn[cc];
    pyv = warp_sum(pyv);
    if (lane == 0) red1[wid] = pyv;
    __syncthreads();
    MID_TR(6)
    const double yv = mid_sum16(red1);
    const double alpha2 = -0.5 * tau * (tau * yv);
    const double kappa = tau * ycc + 2.0 * alpha2;
    double pn = 0.0, pwx = 0.0, pvx = 0.0;
#pragma unroll 1
    for (int r = cc + tid; r < m0; r += MID_THREADS) {
      const double v = vn[r];
      const double w = tau * wn[r] + alpha2 * v;
      const double x = vq[r] - kappa * v;
      wn[r] = w;
      if (r == cc) {  // the diagonal entry; the symv pass may start on it (even column): it must not count
        if (g == 0) a.d[c0 + cc] = x;
        vq[r] = 0.0;
      } else {
        vq[r] = x;
      }
      if (r >= cc + 2) {
        pn += x * x;
        pwx += w * x;
        pvx += v * x;
      }
    }
    const double t3 = mid_warp_sum3(pn, pwx, pvx, lane);
    if ((lane & 7) == 0 && lane < 24) red2[lane >> 3][wid] = t3;
    __syncthreads();
    MID_TR(7)
    MID_TR(9)
    MID_MARK(2)
  }
#ifdef KOT_MID_TRACE
  if (timing)
    for (int i = 0; i < 8; ++i) a.dbg[i] += tseg[i];
#endif
#undef MID_MARK
#undef MID_TR
  // hand-over: the still unreduced block (rows/columns ≥ cend) goes back to global memory with the
  // last column's update applied (with cend = m0 − 1 nothing is left: d[n−1] came out of the last exchange)
  if (cend < m0 - 1) {
    const double* vp = vwbuf + ((cend - 1) & 1) * 2L * ld;
    const double* wp = vp + ld;
    const bool pd = cend >= 1;
    const int ql = (cend > g) ? (cend - g + G - 1) / G : 0;  // rows r ≥ cend
#pragma unroll 1
    for (int q = ql + wid; q < nrows; q += MID_WARPS) {
      const int r = g + G * q;
      const double* Ar = Aloc + (long)q * ld;
      double* dst = a.A + (long)(c0 + r) * n + c0;
      const double vr = pd ? vp[r] : 0.0, wr = pd ? wp[r] : 0.0;
#pragma unroll 2
      for (int s = cend + lane; s < m0; s += 32) dst[s] = Ar[s] - vr * wp[s] - wr * vp[s];
    }
  }
}

// largest order of the resident block for a grid of G CTAs (shared memory: rows + 4 vectors)
static int mid_capacity(int G, size_t smem_max) {
  int best = 0;
  for (int m0 = 2; m0 <= MID_MAX; ++m0) {
    const int rpc = (m0 + G - 1) / G;
    const int ld = m0 + (m0 & 1);
    if (rpc > MID_RPC_MAX) break;
    if (sizeof(double) * ((size_t)rpc * ld + 4L * ld) <= smem_max) best = m0;
  }
  return best;
}

}  // namespace kot
