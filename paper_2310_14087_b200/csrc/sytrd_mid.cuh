// sytrd "mid" kernel: unblocked Householder tridiagonalisation (dsytd2, lower) of a trailing block
// that fits in the shared memory of the WHOLE grid (one CTA per SM, rows r ≡ blockIdx mod G, full
// symmetric rows), included by eig.cu.  Replaces the cooperative panel kernel (reference path:
// np.linalg.eigh in linalg.py:60-83) for every column whose trailing matrix is at most
// G × ~180 KB: 1776 columns of an ℓ = 2000 eigensolve on 148 SMs.
//
// Why: the panel kernel pays, per column, two grid barriers, the reduction of the panel corrections
// (Wᵀv, Vᵀv partials) and a symv that streams the trailing matrix through L2 — ≈ 12.5 µs per column.
// Here the matrix never leaves shared memory (the rank-2 update of column c is fused into column
// c+1's symv pass, as in the cluster tail) and a column needs ONE exchange:
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
// trip).  Every sector is written to R replicas and a CTA reads replica blockIdx mod R, otherwise
// 148 SMs would poll the same cache lines of a few L2 slices.
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
constexpr int MID_XPT = MID_MAX / MID_THREADS;    // vector entries per thread
constexpr int MID_RPC_MAX = 24;                   // rows per CTA
constexpr int MID_NTR_MAX = MID_RPC_MAX / 3;      // row triples per CTA
constexpr int MID_SPC = 2 * MID_NTR_MAX;          // sector stride per CTA (y triples, then p triples)
constexpr int MID_SPT = (kNumSMs * MID_SPC + MID_THREADS - 1) / MID_THREADS;  // polled sectors per thread
constexpr int MID_REP_MAX = 8;                    // replicas of every published sector
constexpr int MID_RG = 4;                         // rows per register group in the fused pass
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
  unsigned epoch0;
  int* err;                 // set to 1 when a gather timed out
  unsigned long long* dbg;  // nullable: per-segment ns accumulated by CTA 0 thread 0
};
unsigned long long* g_mid_dbg = nullptr;  // set by kot_debug_mid_timing

__device__ __forceinline__ void mid_put(MidSector* s, double v0, double v1, double v2, unsigned long long tag) {
  asm volatile("st.volatile.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(s), "l"(__double_as_longlong(v0)),
               "l"(__double_as_longlong(v1)), "l"(__double_as_longlong(v2)), "l"(tag)
               : "memory");
}
__device__ __forceinline__ bool mid_try(const MidSector* s, unsigned long long tag, double& v0, double& v1,
                                        double& v2) {
  unsigned long long a, b, c, t;
  asm volatile("ld.volatile.global.v4.b64 {%0, %1, %2, %3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(t) : "l"(s) : "memory");
  if (t != tag) return false;
  v0 = __longlong_as_double((long long)a);
  v1 = __longlong_as_double((long long)b);
  v2 = __longlong_as_double((long long)c);
  return true;
}

// R live rows of the CTA (consecutive q from q0), double2 columns [i0, i1) counted from column `base`
// (even): the pending rank-2 update applied in place (if pend) fused with the partial row-dot with vn.
// Partial sums land in ypart[q − qlo][warp].
template <int R>
__device__ __forceinline__ void mid_rows_pass(double* Aloc, int ld, int q0, int qlo, int g, int G, int base, int i0,
                                              int i1, bool pend, const double* vp, const double* wp,
                                              const double* vn, double (*ypart)[MID_WARPS + 1], int lane, int wid) {
  double2* A2[R];
  double vr[R], wr[R], a0[R], a1[R];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const int q = q0 + j;
    const int r = g + G * q;
    A2[j] = reinterpret_cast<double2*>(Aloc + (long)q * ld + base);
    vr[j] = pend ? vp[r] : 0.0;
    wr[j] = pend ? wp[r] : 0.0;
    a0[j] = 0.0;
    a1[j] = 0.0;
  }
  const double2* x2 = reinterpret_cast<const double2*>(vn + base);
  if (pend) {
    const double2* w2 = reinterpret_cast<const double2*>(wp + base);
    const double2* u2 = reinterpret_cast<const double2*>(vp + base);
    for (int i = i0 + lane; i < i1; i += 32) {
      const double2 x = x2[i], ws = w2[i], us = u2[i];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        double2 e = A2[j][i];
        e.x = e.x - vr[j] * ws.x - wr[j] * us.x;
        e.y = e.y - vr[j] * ws.y - wr[j] * us.y;
        A2[j][i] = e;
        a0[j] += e.x * x.x;
        a1[j] += e.y * x.y;
      }
    }
  } else {
    for (int i = i0 + lane; i < i1; i += 32) {
      const double2 x = x2[i];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const double2 e = A2[j][i];
        a0[j] += e.x * x.x;
        a1[j] += e.y * x.y;
      }
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
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < R; ++j) ypart[q0 + j - qlo][wid] = t[j];
  }
}

__global__ void __launch_bounds__(MID_THREADS, 1) sytrd_mid_kernel(MidArgs a) {
  extern __shared__ double msm[];
  const int G = gridDim.x, g = blockIdx.x;
  const int n = a.n, c0 = a.c0, m0 = n - c0, cend = a.cend;
  const int nrows = g < m0 ? (m0 - g + G - 1) / G : 0;  // own rows r = g + G q, q < nrows
  const int rpc = (m0 + G - 1) / G;
  const int ntr = (rpc + 2) / 3;  // row triples per CTA: sectors [0, ntr) carry y, [ntr, 2 ntr) carry p
  const int spc = 2 * ntr;
  const int nsec = G * spc;
  const int ld = m0 + (m0 & 1);
  double* Aloc = msm;                           // rpc × ld
  double* vwbuf = Aloc + (long)rpc * ld;        // by column parity: [v | w], 2 × 2 × ld
  __shared__ double red1[MID_WARPS], red2[MID_WARPS];
  __shared__ double scal[4];
  __shared__ double ypart[MID_RPC_MAX][MID_WARPS + 1];
  __shared__ double ys[MID_RPC_MAX + 3], ps[MID_RPC_MAX + 3];
  __shared__ int dead;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int rep = g % a.nrep;

  if (tid == 0) dead = 0;
  for (int q = wid; q < nrows; q += MID_WARPS) {
    const double* src = a.A + (long)(c0 + g + G * q) * n + c0;
    double* dst = Aloc + (long)q * ld;
    for (int s = lane; s < ld; s += 32) dst[s] = (s < m0) ? src[s] : 0.0;
  }
  for (int s = tid; s < 4 * ld; s += MID_THREADS) vwbuf[s] = 0.0;
  if (tid < MID_RPC_MAX + 3) {
    ys[tid] = 0.0;
    ps[tid] = 0.0;
  }
  __syncthreads();

  const bool timing = (a.dbg != nullptr) && g == 0 && tid == 0;
  unsigned long long tseg[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long tl = timing ? gtimer() : 0;
#define MID_MARK(i)                         \
  if (timing) {                             \
    const unsigned long long t_ = gtimer(); \
    tseg[i] += t_ - tl;                     \
    tl = t_;                                \
  }
  // Exchange c (c = −1 … cend−1) finishes column c (its w) and builds column c+1 (x, Householder
  // scalars, v); c = −1 only distributes column 0 (τ = 0, v = 0).
  double tau = 0.0;  // τ of column c
  for (int c = -1; c < cend; ++c) {
    const int par = c & 1;
    double* vn = vwbuf + par * 2L * ld;  // v of column c, its y and then its w
    double* wn = vn + ld;
    double* vq = vwbuf + (par ^ 1) * 2L * ld;  // column c−1's v and w (pending update), then column c+1's v
    const double* wp = vq + ld;
    const unsigned long long tag = (unsigned long long)a.epoch0 + (unsigned)(c + 2);
    MidSector* xb = a.xchg + (long)par * a.nrep * G * MID_SPC;
    const bool pend = c >= 1;  // column c−1's rank-2 update is still to be applied
    // (C) pending update fused with y_r = Σ_{s>c} A_rs v_s: warp w takes the w-th column chunk of
    // every live row, MID_RG rows at a time (the vectors are loaded once per row group)
    const int qlo = (c + 1 > g) ? (c + 1 - g + G - 1) / G : 0;  // first live row (r > c)
    if (c >= 0) {
      const int base = (c + 1) & ~1;
      const int n2 = (ld - base) >> 1;
      const int chunk = (n2 + MID_WARPS - 1) / MID_WARPS;
      const int i0 = wid * chunk, i1 = min(n2, i0 + chunk);
      for (int q0 = qlo; q0 < nrows; q0 += MID_RG) {
        const int nr = min(MID_RG, nrows - q0);
        if (nr == 4)
          mid_rows_pass<4>(Aloc, ld, q0, qlo, g, G, base, i0, i1, pend, vq, wp, vn, ypart, lane, wid);
        else if (nr == 3)
          mid_rows_pass<3>(Aloc, ld, q0, qlo, g, G, base, i0, i1, pend, vq, wp, vn, ypart, lane, wid);
        else if (nr == 2)
          mid_rows_pass<2>(Aloc, ld, q0, qlo, g, G, base, i0, i1, pend, vq, wp, vn, ypart, lane, wid);
        else
          mid_rows_pass<1>(Aloc, ld, q0, qlo, g, G, base, i0, i1, pend, vq, wp, vn, ypart, lane, wid);
      }
      __syncthreads();
    }
    MID_MARK(0)
    // publish (y_r, p_r = A_{r,c+1} − τ y_r) for the live rows: warp 0 packs row triples into sectors
    if (wid == 0) {
      if (lane < nrows) {
        double y = 0.0, pv = 0.0;
        if (lane >= qlo) {
          if (c >= 0) {
#pragma unroll
            for (int w = 0; w < MID_WARPS; ++w) y += ypart[lane - qlo][w];
          }
          pv = Aloc[(long)lane * ld + c + 1] - tau * y;
        }
        ys[lane] = y;
        ps[lane] = pv;
      }
      __syncwarp();
      for (int l = lane; l < spc * a.nrep; l += 32) {
        const int k = l % spc, rp = l / spc;
        const int j = k < ntr ? k : k - ntr;
        const int qmax = min(3 * j + 2, nrows - 1);
        if (qmax >= 3 * j && g + G * qmax >= c + 1) {  // the sector holds a live row
          const double* src = k < ntr ? ys : ps;
          mid_put(xb + ((long)rp * G + g) * MID_SPC + k, src[3 * j], src[3 * j + 1], src[3 * j + 2], tag);
        }
      }
    }
    MID_MARK(1)
    // gather: every thread polls its sectors of the CTA's replica and scatters y into wn, p into vq
    {
      const MidSector* rb = xb + (long)rep * G * MID_SPC;
      bool have[MID_SPT];
      int gs[MID_SPT], ks[MID_SPT];
#pragma unroll
      for (int u = 0; u < MID_SPT; ++u) {
        const int sid = tid + u * MID_THREADS;
        have[u] = true;
        gs[u] = 0;
        ks[u] = 0;
        if (sid < nsec) {
          const int gg = sid / spc, k = sid - gg * spc;
          const int j = k < ntr ? k : k - ntr;
          const int nrg = gg < m0 ? (m0 - gg + G - 1) / G : 0;
          const int qmax = min(3 * j + 2, nrg - 1);
          have[u] = !(qmax >= 3 * j && gg + G * qmax >= c + 1);
          gs[u] = gg;
          ks[u] = k;
        }
      }
      unsigned spins = 0;
      while (true) {
        bool all = true;
#pragma unroll
        for (int u = 0; u < MID_SPT; ++u) {
          if (!have[u]) {
            double v0, v1, v2;
            if (mid_try(rb + (long)gs[u] * MID_SPC + ks[u], tag, v0, v1, v2)) {
              have[u] = true;
              const int k = ks[u];
              const int j = k < ntr ? k : k - ntr;
              double* dst = k < ntr ? wn : vq;
              const int r0 = gs[u] + G * 3 * j;
              if (r0 >= c + 1 && r0 < m0) dst[r0] = v0;
              if (r0 + G >= c + 1 && r0 + G < m0) dst[r0 + G] = v1;
              if (r0 + 2 * G >= c + 1 && r0 + 2 * G < m0) dst[r0 + 2 * G] = v2;
            } else {
              all = false;
            }
          }
        }
        if (all) break;
        if (*(volatile int*)&dead) break;
        if (++spins > MID_SPIN_LIMIT) {
          dead = 1;
          atomicExch(a.err, 1);
          break;
        }
      }
    }
    __syncthreads();
    MID_MARK(2)
    // w = τ y + α₂ v (α₂ = −½ τ² yᵀv) finishes column c; x_{c+1} = p − κ v, κ = τ y_{c+1} + 2 α₂
    const int cc = c + 1;
    double yr[MID_XPT], vr[MID_XPT], pr[MID_XPT];
    double pyv = 0.0;
#pragma unroll
    for (int u = 0; u < MID_XPT; ++u) {
      const int r = cc + tid + u * MID_THREADS;
      const bool in = r < m0;
      yr[u] = in ? wn[r] : 0.0;
      vr[u] = in ? vn[r] : 0.0;
      pr[u] = in ? vq[r] : 0.0;
      pyv += yr[u] * vr[u];
    }
    const double ycc = wn[cc];
    pyv = warp_sum(pyv);
    if (lane == 0) red1[wid] = pyv;
    __syncthreads();
    double yv = 0.0;
#pragma unroll
    for (int w = 0; w < MID_WARPS; ++w) yv += red1[w];
    const double alpha2 = -0.5 * tau * (tau * yv);
    const double kappa = tau * ycc + 2.0 * alpha2;
    double xr[MID_XPT];
    double pn = 0.0;
#pragma unroll
    for (int u = 0; u < MID_XPT; ++u) {
      const int r = cc + tid + u * MID_THREADS;
      if (r < m0) {
        wn[r] = tau * yr[u] + alpha2 * vr[u];
        xr[u] = pr[u] - kappa * vr[u];
        if (r >= cc + 2) pn += xr[u] * xr[u];
      } else {
        xr[u] = 0.0;
      }
    }
    if (tid == 0 && g == 0) a.d[c0 + cc] = xr[0];
    if (tid == 1) scal[2] = xr[0];  // α = x_{cc+1}
    pn = warp_sum(pn);
    if (lane == 0) red2[wid] = pn;
    __syncthreads();
    if (tid == 0) {
      double xn2 = 0.0;
#pragma unroll
      for (int w = 0; w < MID_WARPS; ++w) xn2 += red2[w];
      const double alpha = scal[2];
      double beta, tn, scale;
      if (xn2 == 0.0 || cc + 1 >= m0) {  // dlarfg: H = I
        tn = 0.0;
        beta = alpha;
        scale = 1.0;
      } else {
        beta = -copysign(hypot(alpha, sqrt(xn2)), alpha);
        tn = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      scal[0] = tn;
      scal[1] = scale;
      if (g == 0 && cc < cend) {
        a.e[c0 + cc] = beta;
        a.tau[c0 + cc] = tn;
      }
    }
    __syncthreads();
    tau = scal[0];
    const double scale = scal[1];
#pragma unroll
    for (int u = 0; u < MID_XPT; ++u) {
      const int r = cc + tid + u * MID_THREADS;
      if (r < m0) vq[r] = (r == cc) ? 0.0 : (r == cc + 1) ? 1.0 : xr[u] * scale;  // entry cc masks the even start
    }
    __syncthreads();
    if (tid < nrows && cc < cend) {
      const int r = g + G * tid;
      if (r > cc) a.Vall[(long)(c0 + r) * n + c0 + cc] = (tau == 0.0) ? 0.0 : vq[r];
    }
    MID_MARK(3)
  }
  if (timing)
    for (int i = 0; i < 8; ++i) a.dbg[i] += tseg[i];
#undef MID_MARK
  // hand-over: the still unreduced block (rows/columns ≥ cend) goes back to global memory with the
  // last column's update applied (with cend = m0 − 1 nothing is left: d[n−1] came out of the last exchange)
  if (cend < m0 - 1) {
    const double* vp = vwbuf + ((cend - 1) & 1) * 2L * ld;
    const double* wp = vp + ld;
    const bool pd = cend >= 1;
    const int qlo = (cend > g) ? (cend - g + G - 1) / G : 0;  // rows r ≥ cend
    for (int q = qlo + wid; q < nrows; q += MID_WARPS) {
      const int r = g + G * q;
      const double* Ar = Aloc + (long)q * ld;
      double* dst = a.A + (long)(c0 + r) * n + c0;
      const double vr = pd ? vp[r] : 0.0, wr = pd ? wp[r] : 0.0;
      for (int s = cend + lane; s < m0; s += 32) dst[s] = pd ? Ar[s] - vr * wp[s] - wr * vp[s] : Ar[s];
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
