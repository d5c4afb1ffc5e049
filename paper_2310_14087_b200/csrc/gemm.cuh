// FP64 tensor-core GEMM core for sm_100a.
//
// tcgen05 has no FP64 kind (ptxas rejects .kind::f64), so the
// FP64 tensor path on B200 is the warp-level DMMA (`mma.sync.m8n8k4.f64`,
// SASS DMMA.8x8x4).  This core stages op(A)/op(B) tiles global→shared with a
// 3-stage cp.async (LDGSTS) pipeline into bank-conflict-free padded layouts,
// each warp owns a 32×32 C sub-tile (16 DMMA per k4 step), and a pluggable
// epilogue consumes the accumulators:
//   * plain / axpby stores,
//   * symmetric "compute one triangle and mirror" stores (keeps symmetric
//     iterates bitwise symmetric),
//   * fused row-dot partials  out[r] = Σ_c acc(r,c)·E(r,c)  (Φ and the
//     structure-reduced CG matvec), reduced deterministically afterwards.
// Structural zeros of triangular operands (R is upper triangular) are skipped
// by restricting the K range per output tile.
#pragma once
#include <algorithm>
#include <type_traits>
#include "common.cuh"
#include "prof.cuh"

namespace kot {

#ifndef KOT_GEMM_STAGES
#define KOT_GEMM_STAGES 4
#endif
#ifndef KOT_GEMM_BK
#define KOT_GEMM_BK 8
#endif
// CTAs a GEMM launch from the calling host thread may use (0 = one per tile).  The solver's background
// chains (EG pipeline threads) set a cap so that their GEMMs never fill every SM slot: the Newton
// chain's CG kernels, launched one after another, then find free slots instead of queueing behind
// a background GEMM's waves.
// The calling host thread runs a background chain (the EG pipeline): its GEMMs and panels bring SMs up
// with the maximum shared-memory carveout (per launch), so the Newton chain's kernels fit beside them.
inline bool& background_thread() {
  static thread_local bool bg = false;
  return bg;
}

inline int& gemm_cta_cap() {
  static thread_local int cap = 0;
  return cap;
}

constexpr int GB_M = 64, GB_N = 64, GB_K = KOT_GEMM_BK, G_STAGES = KOT_GEMM_STAGES, G_THREADS = 128;
constexpr int G_PADK = GB_K + 4;  // stride ≡ 4 (mod 16) doubles → conflict-free fragment loads
// CTA tile BM×BN, 4 warps as 2×2, each (BM/2)×(BN/2).  64×64 is used everywhere: 64×128 / 128×64
// are 17 % faster on the CG matvec shapes in isolation (tools/gemmbench/gemm_big.cu) but slower
// inside the solver, where the concurrent chains leave fewer SMs free (matvec 1.05 → 1.23 ms).
template <int BM, int BN>
struct GTile {
  static constexpr int PADM = BM + 4, PADN = BN + 4;
  static constexpr int ATILE = (BM * G_PADK > GB_K * PADM) ? BM * G_PADK : GB_K * PADM;
  static constexpr int BTILE = (BN * G_PADK > GB_K * PADN) ? BN * G_PADK : GB_K * PADN;
  static constexpr int SMEM = G_STAGES * (ATILE + BTILE + GB_K) * 8;
  static constexpr int WM = BM / 2, WN = BN / 2, MI = WM / 8, NJ = WN / 8;
};
constexpr int G_PADM = GB_M + 4;
constexpr int G_PADN = GB_N + 4;
constexpr int G_SMEM_BYTES = GTile<GB_M, GB_N>::SMEM;

// C(M×N) = op(A)(M×K) · diag(kscale) · op(B)(K×N), all row-major.
//   op(A)[m][k] = TA ? A[k*lda+m] : A[m*lda+k]
//   op(B)[k][n] = TB ? B[n*ldb+k] : B[k*ldb+n]
struct GemmShape {
  int M, N, K;
  const double* A;
  long lda;
  const double* B;
  long ldb;
  const double* kscale;  // nullable
  // K-range restriction per output tile (structural zeros of triangular R):
  //   k_begin = max(kb_m ? m0 : 0, kb_n ? n0 : 0)
  //   k_end   = min(K, ke_m ? m0+BM : K, ke_n ? n0+BN : K)
  int kb_m, kb_n, ke_m, ke_n;
  int kstart;     // K range starts at max(..., kstart), rounded down to the k-tile
  // device-side overrides (nullable), read at kernel start: the grid is sized for the static
  // N/K (upper bounds) and tiles beyond the actual size exit (no host round trip needed)
  const int* dN;
  const int* dK;
  const int* dKstart;
  const double* skipf = nullptr;  // nullable: the launch is a no-op when *skipf != 0 (batched CG)
  int sym_tiles;  // enumerate only tiles with tm <= tn (symmetric outputs)
  // split-K: grid.y = ksplit partial products written to ws[split][M][N] (ld N),
  // then reduced in fixed order by splitk_reduce_kernel (deterministic).
  int ksplit;
  double* ws;
};

__device__ __forceinline__ void cp_async_16(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_8(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Load a (rows × cols) tile whose global rows are contiguous (row-major, ld),
// into smem with padded stride `pad`.  Rows [r0, r0+ROWS), cols [c0, c0+COLS);
// elements outside [0,rmax)×[0,cmax) are zero-filled.
template <int ROWS, int COLS, int VEC>
__device__ __forceinline__ void load_tile(double* sm, int pad, const double* g, long ld, int r0, int c0,
                                          int rmax, int cmax) {
  constexpr int CPR = COLS / VEC;  // chunks per row
  constexpr int TOTAL = ROWS * CPR;
#pragma unroll
  for (int i = threadIdx.x; i < TOTAL; i += G_THREADS) {
    const int r = i / CPR, c = (i % CPR) * VEC;
    const int gr = r0 + r, gc = c0 + c;
    int valid = 0;
    if (gr < rmax) valid = min(max(cmax - gc, 0), VEC);
    const double* src = valid ? (g + (long)gr * ld + gc) : g;
    double* dst = sm + r * pad + c;
    if (VEC == 2)
      cp_async_16(dst, src, valid * 8);
    else
      cp_async_8(dst, src, valid * 8);
  }
}

template <class E, class = void>
struct EpiHasAdapt : std::false_type {};
template <class E>
struct EpiHasAdapt<E, std::void_t<decltype(&E::adapt)>> : std::true_type {};

// Epilogue interface:
//   static constexpr bool kRowDot;            // use the fused row-dot path
//   __device__ void store(int r, int c, double v) const;          (kRowDot == false)
//   __device__ double rowdot_weight(int r, int c) const;          (kRowDot == true)
//   __device__ void rowdot_store(int tn, int r, double partial) const;
template <bool TA, bool TB, int VEC, class Epi, int BM = GB_M, int BN = GB_N>
__global__ void __launch_bounds__(G_THREADS) gemm_dmma_kernel(GemmShape s, Epi epi, int ntiles) {
  using T = GTile<BM, BN>;
  static_assert(!Epi::kRowDot || BN == GB_N, "row-dot partials are per 64-column tile");
  extern __shared__ __align__(16) double gsm[];
  if (s.skipf != nullptr && *s.skipf != 0.0) return;
  const int tiles_n_grid = (s.N + BN - 1) / BN;  // grid layout uses the static bound
  const int n_static = s.N;                        // … and so does the split-K partial layout
  if (s.dN) s.N = *s.dN;
  if (s.dK) s.K = *s.dK;
  if (s.dKstart) s.kstart = *s.dKstart;
  // grouped launches: the epilogue rewrites the shape (and itself) for group blockIdx.z
  if constexpr (EpiHasAdapt<Epi>::value) epi.adapt(s, blockIdx.z);
  double* As = gsm;
  double* Bs = gsm + G_STAGES * T::ATILE;
  double* Ks = gsm + G_STAGES * (T::ATILE + T::BTILE);

  // tiles in a loop: a launch may use fewer CTAs than tiles (gemm_cta_cap)
  for (int bx = blockIdx.x; bx < ntiles; bx += gridDim.x) {
  __syncthreads();  // the previous tile's epilogue may still read the staging buffers
    const int tiles_m = (s.M + BM - 1) / BM;
    const int tiles_n = (s.N + BN - 1) / BN;
    int tm, tn;
    if (s.sym_tiles) {
      int t = bx;
      tm = 0;
      while (t >= tiles_n_grid - tm) {
        t -= tiles_n_grid - tm;
        ++tm;
      }
      tn = tm + t;
    } else {
      tm = bx % tiles_m;
      tn = bx / tiles_m;
    }
    if (tm >= tiles_m || tn >= tiles_n) continue;
    const int m0 = tm * BM, n0 = tn * BN;

    int kbeg = 0, kend = s.K;
    if (s.kb_m) kbeg = max(kbeg, m0);
    if (s.kb_n) kbeg = max(kbeg, n0);
    kbeg = max(kbeg, s.kstart);
    if (s.ke_m) kend = min(kend, m0 + BM);
    if (s.ke_n) kend = min(kend, n0 + BN);
    kbeg = (kbeg / GB_K) * GB_K;
    int nkt = kend > kbeg ? (kend - kbeg + GB_K - 1) / GB_K : 0;
    if (s.ksplit > 1) {  // this CTA's share of the K tiles
      const int per = (nkt + s.ksplit - 1) / s.ksplit;
      const int t0 = blockIdx.y * per;
      kbeg += t0 * GB_K;
      nkt = max(0, min(per, nkt - t0));
    }

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int wm = (warp >> 1) * T::WM, wn = (warp & 1) * T::WN;

    double acc[T::MI][T::NJ][2];
  #pragma unroll
    for (int i = 0; i < T::MI; i++)
  #pragma unroll
      for (int j = 0; j < T::NJ; j++) acc[i][j][0] = acc[i][j][1] = 0.0;

    auto issue = [&](int kt, int stage) {
      const int k0 = kbeg + kt * GB_K;
      double* as = As + stage * T::ATILE;
      double* bs = Bs + stage * T::BTILE;
      if (TA)  // A stored K×M: tile rows k, cols m
        load_tile<GB_K, BM, VEC>(as, T::PADM, s.A, s.lda, k0, m0, s.K, s.M);
      else
        load_tile<BM, GB_K, VEC>(as, G_PADK, s.A, s.lda, m0, k0, s.M, s.K);
      if (TB)  // B stored N×K
        load_tile<BN, GB_K, VEC>(bs, G_PADK, s.B, s.ldb, n0, k0, s.N, s.K);
      else
        load_tile<GB_K, BN, VEC>(bs, T::PADN, s.B, s.ldb, k0, n0, s.K, s.N);
      if (s.kscale != nullptr && threadIdx.x < GB_K) {
        const int k = k0 + threadIdx.x;
        cp_async_8(Ks + stage * GB_K + threadIdx.x, k < s.K ? s.kscale + k : s.kscale, k < s.K ? 8 : 0);
      }
    };

  #pragma unroll
    for (int st = 0; st < G_STAGES - 1; ++st) {
      if (st < nkt) issue(st, st);
      cp_async_commit();
    }

    for (int kt = 0; kt < nkt; ++kt) {
      cp_async_wait<G_STAGES - 2>();
      __syncthreads();
      {
        const int nk = kt + G_STAGES - 1;
        if (nk < nkt) issue(nk, nk % G_STAGES);
        cp_async_commit();
      }
      const int stage = kt % G_STAGES;
      const double* as = As + stage * T::ATILE;
      const double* bs = Bs + stage * T::BTILE;
      const double* ks = Ks + stage * GB_K;
      // the K-scaling multiply only exists in the instantiation that needs it (uniform branch)
      auto mma_stage = [&](auto has_kscale) {
        constexpr bool kKS = decltype(has_kscale)::value;
  #pragma unroll
        for (int kk = 0; kk < GB_K; kk += 4) {
          double a[T::MI], b[T::NJ];
          double kscl = 1.0;
          if constexpr (kKS) kscl = ks[kk + t];
  #pragma unroll
          for (int i = 0; i < T::MI; i++) {
            const int m = wm + i * 8 + g;
            const double av = TA ? as[(kk + t) * T::PADM + m] : as[m * G_PADK + kk + t];
            if constexpr (kKS)
              a[i] = av * kscl;
            else
              a[i] = av;
          }
  #pragma unroll
          for (int j = 0; j < T::NJ; j++) {
            const int n = wn + j * 8 + g;
            b[j] = TB ? bs[n * G_PADK + kk + t] : bs[(kk + t) * T::PADN + n];
          }
  #pragma unroll
          for (int i = 0; i < T::MI; i++)
  #pragma unroll
            for (int j = 0; j < T::NJ; j++) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
        }
      };
      if (s.kscale != nullptr)
        mma_stage(std::true_type{});
      else
        mma_stage(std::false_type{});
    }
    cp_async_wait<0>();

    if constexpr (Epi::kRowDot) {
      // partial[r] = Σ_{c in this tile} acc(r,c)·E(r,c): 4-lane shuffle + 2-warp smem combine.
      __syncthreads();
      double* red = gsm;  // reuse: [2][BM]
  #pragma unroll
      for (int i = 0; i < T::MI; i++) {
        const int r = m0 + wm + i * 8 + g;
        double p = 0.0;
  #pragma unroll
        for (int j = 0; j < T::NJ; j++)
  #pragma unroll
          for (int h = 0; h < 2; h++) {
            const int c = n0 + wn + j * 8 + 2 * t + h;
            if (r < s.M && c < s.N) p += acc[i][j][h] * epi.rowdot_weight(r, c);
          }
        p += __shfl_xor_sync(0xffffffffu, p, 1);
        p += __shfl_xor_sync(0xffffffffu, p, 2);
        if (t == 0) red[(warp & 1) * BM + wm + i * 8 + g] = p;
      }
      __syncthreads();
      for (int q = threadIdx.x; q < BM; q += G_THREADS) {
        const int r = m0 + q;
        // split-K: every K share writes its own partial row block (row-dots are linear in the product)
        if (r < s.M) epi.rowdot_store(tn + (int)blockIdx.y * tiles_n_grid, r, red[q] + red[BM + q]);
      }
    } else if (s.ksplit > 1) {
      double* ws = s.ws + (long)blockIdx.y * s.M * n_static;
  #pragma unroll
      for (int i = 0; i < T::MI; i++) {
        const int r = m0 + wm + i * 8 + g;
        if (r >= s.M) continue;
  #pragma unroll
        for (int j = 0; j < T::NJ; j++)
  #pragma unroll
          for (int h = 0; h < 2; h++) {
            const int c = n0 + wn + j * 8 + 2 * t + h;
            if (c < s.N) ws[(long)r * n_static + c] = acc[i][j][h];
          }
      }
    } else {
  #pragma unroll
      for (int i = 0; i < T::MI; i++) {
        const int r = m0 + wm + i * 8 + g;
        if (r >= s.M) continue;
  #pragma unroll
        for (int j = 0; j < T::NJ; j++)
  #pragma unroll
          for (int h = 0; h < 2; h++) {
            const int c = n0 + wn + j * 8 + 2 * t + h;
            if (c < s.N) epi.store(r, c, acc[i][j][h]);
          }
      }
    }
  }
}

template <class Epi>
__global__ void splitk_reduce_kernel(int M, int N, int splits, int sym_tiles, const double* __restrict__ ws,
                                     Epi epi, const int* __restrict__ dN, const double* skipf) {
  if (skipf != nullptr && *skipf != 0.0) return;
  // ws layout [split][M][N] with the static N; columns ≥ *dN (device-side N) were not computed
  const int n_act = dN ? *dN : N;
  const long total = (long)M * N;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
    const int r = (int)(e / N), c = (int)(e % N);
    if (c >= n_act) continue;
    if (sym_tiles && r / GB_M > c / GB_N) continue;
    double v = 0.0;
    for (int sp = 0; sp < splits; ++sp) v += ws[(long)sp * total + e];
    epi.store(r, c, v);
  }
}

inline int gemm_grid(const GemmShape& s, int bm = GB_M, int bn = GB_N) {
  const int tm = (s.M + bm - 1) / bm, tn = (s.N + bn - 1) / bn;
  if (s.sym_tiles) return tm * (tm + 1) / 2;
  return tm * tn;
}

inline bool gemm_vec2_ok(const GemmShape& s) {
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  return al(s.A) && al(s.B) && (s.lda % 2 == 0) && (s.ldb % 2 == 0);
}

// Algorithmic FLOPs of one launch: per computed tile, 2·rows·cols·(true K range),
// excluding zero padding and the structurally-zero tiles that are skipped.
inline double gemm_alg_flops(const GemmShape& s, int bm = GB_M, int bn = GB_N) {
  const int tm_n = (s.M + bm - 1) / bm, tn_n = (s.N + bn - 1) / bn;
  double f = 0.0;
  for (int tm = 0; tm < tm_n; ++tm)
    for (int tn = s.sym_tiles ? tm : 0; tn < tn_n; ++tn) {
      const int m0 = tm * bm, n0 = tn * bn;
      int kb = 0, ke = s.K;
      if (s.kb_m) kb = std::max(kb, m0);
      if (s.kb_n) kb = std::max(kb, n0);
      kb = std::max(kb, s.kstart);
      if (s.ke_m) ke = std::min(ke, m0 + bm);
      if (s.ke_n) ke = std::min(ke, n0 + bn);
      if (ke > kb) f += 2.0 * std::min(bm, s.M - m0) * std::min(bn, s.N - n0) * (double)(ke - kb);
    }
  return f;
}

// Launch with a BM×BN CTA tile (64×64: every GEMM; 64×128 / 128×64: long-thin products).
template <bool TA, bool TB, int BM, int BN, class Epi>
void gemm_launch_tiled(const GemmShape& s, const Epi& epi, cudaStream_t st) {
  if (s.M <= 0 || s.N <= 0) return;
  if (BM != BN) kot_require(!s.sym_tiles, KOT_EINVAL, "symmetric tiling needs square CTA tiles");
  constexpr int smem = GTile<BM, BN>::SMEM;
  ProfScope prof("gemm_dmma", st);
  if (prof.tok >= 0) prof.flops = gemm_alg_flops(s, BM, BN);  // only for recorded (sampled) launches
  const int tiles = gemm_grid(s, BM, BN);
  const int cap = gemm_cta_cap();
  const int ctas = cap > 0 ? std::max(1, std::min(tiles, cap / std::max(s.ksplit, 1))) : tiles;
  const dim3 grid(ctas, s.ksplit > 1 ? s.ksplit : 1);
  auto launch = [&](auto k) {
    ensure_smem_attr((const void*)k, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(G_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    if (background_thread() && carveout_preferred()) {
      at[0].id = cudaLaunchAttributePreferredSharedMemoryCarveout;
      at[0].val.sharedMemCarveout = cudaSharedmemCarveoutMaxShared;
      cfg.attrs = at;
      cfg.numAttrs = 1;
    }
    KOT_CUDA(cudaLaunchKernelEx(&cfg, k, s, epi, tiles));
  };
  if (gemm_vec2_ok(s))
    launch(gemm_dmma_kernel<TA, TB, 2, Epi, BM, BN>);
  else
    launch(gemm_dmma_kernel<TA, TB, 1, Epi, BM, BN>);
  KOT_LAUNCH_CHECK();
  if constexpr (!Epi::kRowDot) {
    if (s.ksplit > 1) {
      const long total = (long)s.M * s.N;
      splitk_reduce_kernel<Epi><<<(int)std::min<long>((total + 255) / 256, 4L * 148 * 8), 256, 0, st>>>(
          s.M, s.N, s.ksplit, s.sym_tiles, s.ws, epi, s.dN, s.skipf);
      KOT_LAUNCH_CHECK();
    }
  }
}

}  // namespace kot
#include "gemm_tma.cuh"
namespace kot {

// TMA path on/off (KOT_GEMM_TMA=0 forces the cp.async core; kot_debug_gemm_tma switches at run time)
inline std::atomic<int>& gemm_tma_mode() {
  static std::atomic<int> mode{[] {
    const char* e = std::getenv("KOT_GEMM_TMA");
    return e ? std::atoi(e) : 1;
  }()};
  return mode;
}

template <bool TA, bool TB, class Epi>
void gemm_launch(const GemmShape& s, const Epi& epi, cudaStream_t st) {
  const int mode = gemm_tma_mode().load(std::memory_order_relaxed);
  // the TMA core from a tile's worth of K on; small / device-sized launches keep the cp.async core
  // (measured on B200, tools/gemmbench/gemm_tma_bench.cu: 64×64 CTA tiles of four 32×32 warps for
  // everything — NN 2000³ 32.7 TF/s vs 27.2 on the cp.async core, cuBLAS 33.0 — except the row-dot
  // products, whose tall M×(k) shapes prefer 128×64 with eight warps: CG matvec GEMM2 27.8 vs 22.5)
  if (mode > 0 && s.K >= 2 * TMA_BK && (long)s.M * s.N >= 64L * 64) {
    // 128×64 CTAs hold one SM each (288 threads × 122 registers): only when there are enough of them
    const long tiles128 = (long)((s.M + 127) / 128) * ((s.N + 63) / 64) * std::max(s.ksplit, 1);
    const bool tall = Epi::kRowDot && !s.sym_tiles && s.M >= 1024 && tiles128 >= 200;
    if (tall ? gemm_launch_tma<TA, TB, 128, 64, 32, 32, 4>(s, epi, st)
             : gemm_launch_tma<TA, TB, 64, 64, 32, 32, 4>(s, epi, st))
      return;
  }
  gemm_launch_tiled<TA, TB, GB_M, GB_N>(s, epi, st);
}

// Pick a split-K factor so that skinny / few-tile GEMMs fill the 148 SMs.
// ws must hold ksplit·M·N doubles; returns 1 when splitting does not pay.
inline int choose_ksplit(const GemmShape& s, long ws_capacity) {
  const int tiles = gemm_grid(s);
  if (tiles >= 120 || s.K < 512 || s.ws == nullptr) return 1;
  int ks = std::min((2 * 148 + tiles - 1) / tiles, s.K / 256);
  ks = std::min(ks, 16);
  while (ks > 1 && (long)ks * s.M * s.N > ws_capacity) --ks;
  return std::max(ks, 1);
}

inline GemmShape make_shape(int M, int N, int K, const double* A, long lda, const double* B, long ldb) {
  GemmShape s{};
  s.M = M;
  s.N = N;
  s.K = K;
  s.A = A;
  s.lda = lda;
  s.B = B;
  s.ldb = ldb;
  s.ksplit = 1;
  s.ws = nullptr;
  s.dN = s.dK = s.dKstart = nullptr;
  return s;
}

// ------------------------------------------------------------------ epilogues

// C = alpha*acc + beta*C
struct EpiAxpby {
  static constexpr bool kRowDot = false;
  double* C;
  long ldc;
  double alpha, beta;
  __device__ void store(int r, int c, double v) const {
    double* p = C + (long)r * ldc + c;
    *p = (beta == 0.0) ? alpha * v : alpha * v + beta * (*p);
  }
  __device__ double rowdot_weight(int, int) const { return 0; }
  __device__ void rowdot_store(int, int, double) const {}
};

// Symmetric output: only tiles tm<=tn are computed; value written to (r,c) and (c,r).
// out = beta*X(r,c) + alpha*(acc + diag*δ_rc)   (X must itself be symmetric; beta ignored if X null)
struct EpiSymMirror {
  static constexpr bool kRowDot = false;
  double* C;
  long ldc;
  double alpha;
  const double* X;  // nullable
  double beta;
  double diag;
  __device__ void store(int r, int c, double v) const {
    if (r > c) return;  // the diagonal tile computes both halves; keep one
    double o = v;
    if (r == c) o = __dadd_rn(o, diag);
    o = __dmul_rn(alpha, o);
    if (X != nullptr) o = __dadd_rn(__dmul_rn(beta, X[(long)r * ldc + c]), o);
    C[(long)r * ldc + c] = o;
    C[(long)c * ldc + r] = o;
  }
  __device__ double rowdot_weight(int, int) const { return 0; }
  __device__ void rowdot_store(int, int, double) const {}
};

// partial[tn][r] = Σ_c acc(r,c)·E[r][c]
struct EpiRowDot {
  static constexpr bool kRowDot = true;
  const double* E;
  long lde;
  double* partial;  // [tiles_n][ldp]
  long ldp;
  __device__ void store(int, int, double) const {}
  __device__ double rowdot_weight(int r, int c) const { return E[(long)r * lde + c]; }
  __device__ void rowdot_store(int tn, int r, double p) const { partial[(long)tn * ldp + r] = p; }
};

}  // namespace kot
