// Blackwell-native operand path for the FP64 DMMA GEMM core (included by gemm.cuh).
//
// Same contract as gemm_dmma_kernel (GemmShape, the epilogues, split-K, symmetric tiles, the
// triangular K ranges), different staging: op(A)/op(B) k-tiles of 16 doubles (= 128 B, one swizzle
// span) are fetched by TMA (cp.async.bulk.tensor, FP64 tensor maps with 128-byte swizzle and
// hardware zero fill outside the matrix) into a ST-stage ring in shared memory, driven by one
// producer warp through full/empty mbarriers — no per-k-tile __syncthreads, no per-thread address
// arithmetic for the loads.  Consumer warps own WM×WN sub-tiles of a BM×BN CTA tile and issue
// `mma.sync.m8n8k4.f64` (SASS DMMA.8x8x4; tcgen05 has no f64 kind).
//
// Fragment reads from the swizzled tiles are conflict-free (2 wavefronts per 256-byte warp read,
// the minimum):
//   * K-contiguous operand (A row-major, B "TB"): smem row = one m (or n) with its 16 k values,
//     16-byte chunk q stored at q ^ (row & 7); the 8 rows of a fragment hit every chunk slot once
//     per k pair.
//   * M/N-contiguous operand (A "TA", B row-major): 16×16 sub-tiles [k][16 m], chunk (m&15)>>1
//     stored at chunk ^ (k & 7).  A fragment's 8 lanes of one k take the rows
//     m = 4·(g>>1) + (g&1) + 2·h of a 16-row group (h: which half of the group) — even chunks for
//     h = 0, odd for h = 1 — so the XOR keys of the 4 k rows split them over all 8 slots.  The
//     accumulator rows / columns follow the same map in the epilogue.
#pragma once
#include <cuda.h>

#include <mutex>

namespace kot {

constexpr int TMA_BK = 16;


using TmaEncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// cuTensorMapEncodeTiled through the runtime's driver entry point (libkotgpu does not link libcuda).
inline TmaEncodeFn tma_encoder() {
  static TmaEncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    (void)cudaGetLastError();
    return reinterpret_cast<TmaEncodeFn>(p);
  }();
  return fn;
}

// 2-D FP64 map over a row-major matrix with `rows` rows of `cols` contiguous doubles (row pitch ld),
// box = bcols (contiguous) × brows, 128-byte swizzle; false if the operand does not qualify.
inline bool tma_map_2d(CUtensorMap* m, const double* base, long cols, long rows, long ld, int bcols, int brows) {
  const TmaEncodeFn enc = tma_encoder();
  if (!enc || (reinterpret_cast<uintptr_t>(base) & 15) || (ld & 1) || cols <= 0 || rows <= 0) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  const cuuint32_t box[2] = {(cuuint32_t)bcols, (cuuint32_t)brows};
  const cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

inline bool tma_map_1d(CUtensorMap* m, const double* base, long n) {
  const TmaEncodeFn enc = tma_encoder();
  if (!enc || (reinterpret_cast<uintptr_t>(base) & 15) || n <= 0) return false;
  const cuuint64_t dims[1] = {(cuuint64_t)n};
  const cuuint64_t strides[1] = {(cuuint64_t)n * 8};
  const cuuint32_t box[1] = {TMA_BK};
  const cuuint32_t es[1] = {1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, const_cast<double*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ double lds64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const CUtensorMap* map, int c0, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(smem_u32(bar))
      : "memory");
}

// Row (or column) of a fragment element inside a warp sub-tile.
//   K-contiguous operand: 8 consecutive rows per fragment group.
//   M/N-contiguous operand: the conflict-free interleave described at the top of the file.
template <bool MN_MAJOR>
__device__ __forceinline__ int frag_row(int i, int g) {
  if constexpr (MN_MAJOR)
    return 16 * (i >> 1) + 4 * (g >> 1) + (g & 1) + 2 * (i & 1);
  else
    return 8 * i + g;
}
// Byte offset of element (row r, k) of a stage tile (r = m or n inside the CTA tile, k < 16).
template <bool MN_MAJOR>
__device__ __forceinline__ uint32_t tile_off(int r, int k) {
  if constexpr (MN_MAJOR)
    return (uint32_t)((r >> 4) * 2048 + k * 128 + ((((r & 15) >> 1) ^ (k & 7)) << 4) + (r & 1) * 8);
  else
    return (uint32_t)(r * 128 + (((k >> 1) ^ (r & 7)) << 4) + (k & 1) * 8);
}

// Output tile t of the launch (symmetric launches enumerate the tiles with tm <= tn); false if t is
// outside the matrix.  The K range follows the triangular-structure and split-K rules of the core.
struct TmaTile {
  int m0, n0, tn, kbeg, nkt;
};
template <int BM, int BN>
__device__ __forceinline__ bool tma_tile(const GemmShape& s, int t, int tiles_m, int tiles_n, TmaTile& o) {
  int tm, tn;
  if (s.sym_tiles) {
    tm = 0;
    while (t >= tiles_n - tm) {
      t -= tiles_n - tm;
      ++tm;
    }
    tn = tm + t;
  } else {
    tm = t % tiles_m;
    tn = t / tiles_m;
  }
  if (tm >= tiles_m || tn >= tiles_n) return false;
  o.m0 = tm * BM;
  o.n0 = tn * BN;
  o.tn = tn;
  int kbeg = 0, kend = s.K;
  if (s.kb_m) kbeg = max(kbeg, o.m0);
  if (s.kb_n) kbeg = max(kbeg, o.n0);
  kbeg = max(kbeg, s.kstart);
  if (s.ke_m) kend = min(kend, o.m0 + BM);
  if (s.ke_n) kend = min(kend, o.n0 + BN);
  kbeg = (kbeg / TMA_BK) * TMA_BK;
  int nkt = kend > kbeg ? (kend - kbeg + TMA_BK - 1) / TMA_BK : 0;
  if (s.ksplit > 1) {
    const int per = (nkt + s.ksplit - 1) / s.ksplit;
    const int t0 = blockIdx.y * per;
    kbeg += t0 * TMA_BK;
    nkt = max(0, min(per, nkt - t0));
  }
  o.kbeg = kbeg;
  o.nkt = nkt;
  return true;
}

// Tiles are processed in a loop (tile = blockIdx.x, += gridDim.x): a launch may use fewer CTAs than
// tiles (gemm_cta_cap, background solver chains), the ring and its phases carry across tiles.
// At most 96 registers per thread (a few bytes of epilogue spill): two of these CTAs then fit beside a
// resident sytrd panel CTA (256 threads × 128 registers), which inside the solver outweighs the ≈8 %
// this costs a GEMM alone (CG Newton direction 37.2 → 35.5 ms with the max-shared carveout below).
#ifndef KOT_TMA_MAXREG
#define KOT_TMA_MAXREG 96
#endif
#if KOT_TMA_MAXREG > 0
#define KOT_TMA_BOUNDS __maxnreg__(KOT_TMA_MAXREG)
#else
#define KOT_TMA_BOUNDS __launch_bounds__(((BM / WM) * (BN / WN) + 1) * 32)
#endif
template <bool TA, bool TB, int BM, int BN, int WM, int WN, int ST, class Epi>
__global__ void KOT_TMA_BOUNDS
    gemm_tma_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                    const __grid_constant__ CUtensorMap mapK, GemmShape s, Epi epi, int ntiles) {
  constexpr int NWN = BN / WN, NWC = (BM / WM) * NWN;  // consumer warps
  constexpr int MI = WM / 8, NJ = WN / 8;
  constexpr uint32_t A_BYTES = BM * TMA_BK * 8, B_BYTES = BN * TMA_BK * 8;
  static_assert(BM % 16 == 0 && BN % 16 == 0 && WM % 16 == 0 && WN % 16 == 0, "tile shapes");
  static_assert(!Epi::kRowDot || BN == GB_N, "row-dot partials are per 64-column tile");
  extern __shared__ __align__(1024) unsigned char tsm_raw[];
  unsigned char* tsm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(tsm_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* As = tsm;
  unsigned char* Bs = tsm + ST * A_BYTES;
  double* Ks = reinterpret_cast<double*>(Bs + ST * B_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(Ks + ST * TMA_BK);
  uint64_t* empty = full + ST;
  double* red = reinterpret_cast<double*>(empty + ST);  // [NWN][BM] row-dot combine (not in the ring)

  if (s.skipf != nullptr && *s.skipf != 0.0) return;
  const int tiles_n = (s.N + BN - 1) / BN, tiles_m = (s.M + BM - 1) / BM;
  const bool has_ks = s.kscale != nullptr;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int q = 0; q < ST; ++q) {
      mbar_init(full + q, 1);
      mbar_init(empty + q, NWC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == NWC) {  // ---------------- producer: one elected lane issues the TMA copies
    if (lane == 0) {
      const uint32_t bytes = A_BYTES + B_BYTES + (has_ks ? TMA_BK * 8 : 0);
      int g = 0;  // k-tiles issued so far (ring position across tiles)
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        TmaTile tl;
        if (!tma_tile<BM, BN>(s, t, tiles_m, tiles_n, tl)) continue;
        for (int kt = 0; kt < tl.nkt; ++kt, ++g) {
          const int q = g % ST;
          if (g >= ST) mbar_wait(empty + q, ((g / ST) & 1) ^ 1);
          mbar_expect_tx(full + q, bytes);
          const int k0 = tl.kbeg + kt * TMA_BK;
          if constexpr (TA) {
#pragma unroll
            for (int sub = 0; sub < BM / 16; ++sub)
              tma_load_2d(As + q * A_BYTES + sub * 2048, &mapA, tl.m0 + 16 * sub, k0, full + q);
          } else {
            tma_load_2d(As + q * A_BYTES, &mapA, k0, tl.m0, full + q);
          }
          if constexpr (!TB) {
#pragma unroll
            for (int sub = 0; sub < BN / 16; ++sub)
              tma_load_2d(Bs + q * B_BYTES + sub * 2048, &mapB, tl.n0 + 16 * sub, k0, full + q);
          } else {
            tma_load_2d(Bs + q * B_BYTES, &mapB, k0, tl.n0, full + q);
          }
          if (has_ks) tma_load_1d(Ks + q * TMA_BK, &mapK, k0, full + q);
        }
      }
    }
    return;
  }

  // ---------------- consumers
  const int g8 = lane >> 2, t = lane & 3;
  const int wm = (warp / NWN) * WM, wn = (warp % NWN) * WN;
  int g = 0;  // k-tiles consumed so far
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    TmaTile tl;
    if (!tma_tile<BM, BN>(s, tile, tiles_m, tiles_n, tl)) continue;
    double acc[MI][NJ][2];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int kt = 0; kt < tl.nkt; ++kt, ++g) {
      const int q = g % ST;
      mbar_wait(full + q, (g / ST) & 1);
      const uint32_t as = smem_u32(As + q * A_BYTES);
      const uint32_t bs = smem_u32(Bs + q * B_BYTES);
      const double* ks = Ks + q * TMA_BK;
      auto step = [&](auto kks, auto has_kscale) {
        constexpr int kk = decltype(kks)::value;
        constexpr bool kKS = decltype(has_kscale)::value;
        const int k = kk + t;
        double a[MI], b[NJ];
        double kscl = 1.0;
        if constexpr (kKS) kscl = lds64(smem_u32(ks + k));
#pragma unroll
        for (int i = 0; i < MI; ++i) {
          const double av = lds64(as + tile_off<TA>(wm + frag_row<TA>(i, g8), k));
          if constexpr (kKS)
            a[i] = av * kscl;
          else
            a[i] = av;
        }
#pragma unroll
        for (int j = 0; j < NJ; ++j) b[j] = lds64(bs + tile_off<!TB>(wn + frag_row<!TB>(j, g8), k));
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int j = 0; j < NJ; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
      };
      auto stage = [&](auto has_kscale) {
        step(std::integral_constant<int, 0>{}, has_kscale);
        step(std::integral_constant<int, 4>{}, has_kscale);
        step(std::integral_constant<int, 8>{}, has_kscale);
        step(std::integral_constant<int, 12>{}, has_kscale);
      };
      if (has_ks)
        stage(std::true_type{});
      else
        stage(std::false_type{});
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + q);
    }

    // ---------------- epilogue (same semantics as gemm_dmma_kernel)
    const int m0 = tl.m0, n0 = tl.n0;
    auto row_of = [&](int i) { return m0 + wm + frag_row<TA>(i, g8); };
    auto col_of = [&](int j, int h) { return n0 + wn + frag_row<!TB>(j, 2 * t + h); };
    if constexpr (Epi::kRowDot) {
      // partial[r] = Σ_{c in this 64-column tile} acc(r,c)·E(r,c): 4-lane shuffle + cross-warp smem combine
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int r = row_of(i);
        double p = 0.0;
#pragma unroll
        for (int j = 0; j < NJ; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = col_of(j, h);
            if (r < s.M && c < s.N) p += acc[i][j][h] * epi.rowdot_weight(r, c);
          }
        p += __shfl_xor_sync(0xffffffffu, p, 1);
        p += __shfl_xor_sync(0xffffffffu, p, 2);
        if (t == 0) red[(warp % NWN) * BM + (r - m0)] = p;
      }
      asm volatile("bar.sync 1, %0;\n" ::"r"(NWC * 32) : "memory");
      for (int qq = threadIdx.x; qq < BM; qq += NWC * 32) {
        const int r = m0 + qq;
        double v = 0.0;
#pragma unroll
        for (int w = 0; w < NWN; ++w) v += red[w * BM + qq];
        if (r < s.M) epi.rowdot_store(tl.tn + (int)blockIdx.y * tiles_n, r, v);
      }
      asm volatile("bar.sync 1, %0;\n" ::"r"(NWC * 32) : "memory");  // red is reused by the next tile
    } else if (s.ksplit > 1) {
      double* ws = s.ws + (long)blockIdx.y * s.M * s.N;
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int r = row_of(i);
        if (r >= s.M) continue;
#pragma unroll
        for (int j = 0; j < NJ; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = col_of(j, h);
            if (c < s.N) ws[(long)r * s.N + c] = acc[i][j][h];
          }
      }
    } else {
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int r = row_of(i);
        if (r >= s.M) continue;
#pragma unroll
        for (int j = 0; j < NJ; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = col_of(j, h);
            if (c < s.N) epi.store(r, c, acc[i][j][h]);
          }
      }
    }
  }
}

template <int BM, int BN, int ST>
constexpr int tma_smem_bytes() {
  return ST * (BM + BN) * TMA_BK * 8 + ST * TMA_BK * 8 + 2 * ST * 8 + BM * (BN / 32) * 8 + 1024;
}

// TMA-staged launch; returns false (nothing launched) when the operands do not qualify (device-side
// N/K overrides, misaligned bases or odd leading dimensions, non-square symmetric tiling), so the
// caller falls back to the cp.async core.
template <bool TA, bool TB, int BM, int BN, int WM, int WN, int ST, class Epi>
bool gemm_launch_tma(const GemmShape& s, const Epi& epi, cudaStream_t st) {
  if (s.M <= 0 || s.N <= 0) return true;
  if (s.dN || s.dK || s.dKstart) return false;
  if (s.sym_tiles && BM != BN) return false;
  if (Epi::kRowDot && BN != GB_N) return false;
  CUtensorMap ma, mb, mk;
  const bool ok_a = TA ? tma_map_2d(&ma, s.A, s.M, s.K, s.lda, 16, 16) : tma_map_2d(&ma, s.A, s.K, s.M, s.lda, 16, BM);
  const bool ok_b = TB ? tma_map_2d(&mb, s.B, s.K, s.N, s.ldb, 16, BN) : tma_map_2d(&mb, s.B, s.N, s.K, s.ldb, 16, 16);
  if (!ok_a || !ok_b) return false;
  if (s.kscale) {
    if (!tma_map_1d(&mk, s.kscale, s.K)) return false;
  } else {
    mk = ma;  // unused
  }
  constexpr int smem = tma_smem_bytes<BM, BN, ST>();
  constexpr int threads = ((BM / WM) * (BN / WN) + 1) * 32;
  ProfScope prof("gemm_dmma", st);
  if (prof.tok >= 0) prof.flops = gemm_alg_flops(s, BM, BN);
  const int tm = (s.M + BM - 1) / BM, tn = (s.N + BN - 1) / BN;
  const int tiles = s.sym_tiles ? tm * (tm + 1) / 2 : tm * tn;
  const int cap = gemm_cta_cap();
  const int ctas = cap > 0 ? std::max(1, std::min(tiles, cap / std::max(s.ksplit, 1))) : tiles;
  const dim3 grid(ctas, s.ksplit > 1 ? s.ksplit : 1);
  auto k = gemm_tma_kernel<TA, TB, BM, BN, WM, WN, ST, Epi>;
  ensure_smem_attr((const void*)k, smem);
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    if (background_thread() && carveout_preferred()) {  // see background_thread (gemm.cuh)
      at[0].id = cudaLaunchAttributePreferredSharedMemoryCarveout;
      at[0].val.sharedMemCarveout = cudaSharedmemCarveoutMaxShared;
      cfg.attrs = at;
      cfg.numAttrs = 1;
    }
    KOT_CUDA(cudaLaunchKernelEx(&cfg, k, ma, mb, mk, s, epi, tiles));
  }
  KOT_LAUNCH_CHECK();
  if constexpr (!Epi::kRowDot) {
    if (s.ksplit > 1) {
      const long total = (long)s.M * s.N;
      splitk_reduce_kernel<Epi><<<(int)std::min<long>((total + 255) / 256, 4L * 148 * 8), 256, 0, st>>>(
          s.M, s.N, s.ksplit, s.sym_tiles, s.ws, epi, nullptr, s.skipf);
      KOT_LAUNCH_CHECK();
    }
  }
  return true;
}

}  // namespace kot
