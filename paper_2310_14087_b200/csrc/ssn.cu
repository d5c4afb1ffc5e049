// SSN operators on device (north-star items 3, 5, 6).
//
// Reference map (pkg/src/kot/...):
//   phi_forward  problem.py:172-177  → DMMA GEMM R·X (triangular K-skip) with a
//                                       fused row-dot epilogue against R
//   phi_adjoint  problem.py:180-185  → DMMA Rᵀdiag(γ)R, one triangle + mirror,
//                                       with the Z / EG argument fused in
//   proj         psdcone.py:52-59    → DMMA P_α diag(σ_α) P_αᵀ + mirror, X − Π fused
//   𝒯 / M        psdcone.py:94-151   → low-rank 4-GEMM chain, ξ/η computed from σ
//                                       in the epilogue (no k×(ℓ−k) coefficient matrix)
//   residual     problem.py:204-214,  eg_step eg.py:34-41
//   CG           linalg.py:117-162   → fused single-CTA update kernel
//   newton       newton.py:116-195
#include <mutex>
#include <thread>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <string>

#include "gemm.cuh"
#include "ssn.cuh"

namespace kot {

// ---------------------------------------------------------------- Problem

double* Problem::alloc(long count) {
  double* p = static_cast<double*>(dev_alloc(std::max(count, 1L) * sizeof(double)));
  owned.push_back(p);
  return p;
}

void Problem::init_scratch() {
  const long nn = (long)n * n;
  const int tiles = ceil_div(n, GB_N);
  partial = alloc((long)tiles * n);
  M1 = alloc(nn);
  M2 = alloc(nn);
  M3 = alloc(nn);
  M4 = alloc(nn);
  M5 = alloc(nn);
  red = alloc(512 * 16);
  splitws_cap = 16L * 256 * n;
  splitws = alloc(splitws_cap);
  dsc = alloc(64);
  hsc = static_cast<double*>(host_alloc_pinned(64 * sizeof(double)));
  dk = static_cast<int*>(dev_alloc(16 * sizeof(int)));
  dflag = dk + 8;
  hk = static_cast<int*>(host_alloc_pinned(16 * sizeof(int)));
  if (with_eig) eig.reset(new EigWork(n));
}

Problem::~Problem() {
  if (st) cudaStreamSynchronize(st);
  if (nccl_comm || host_comm) {
    try {
      problem_unshard(*this);
    } catch (...) {
    }
  }
  aux_.reset();
  aux2_.reset();
  aux3_.reset();
  crit_.reset();
  if (crit_done) cudaEventDestroy(crit_done);
  if (crit_after) cudaEventDestroy(crit_after);
  if (crit_dx_done) cudaEventDestroy(crit_dx_done);
  if (ev_half) cudaEventDestroy(ev_half);
  if (ev_mv0) cudaEventDestroy(ev_mv0);
  if (ev_mv1) cudaEventDestroy(ev_mv1);
  if (ev_rhs) cudaEventDestroy(ev_rhs);
  if (cg_graph.exec) cudaGraphExecDestroy(cg_graph.exec);
  eig.reset();
  for (double* p : owned) dev_free(p);
  host_free_pinned(hsc, 64 * sizeof(double));
  if (host_comm_buf) host_free_pinned(host_comm_buf, sizeof(double) * host_comm_cap);
  dev_free(dk);
  host_free_pinned(hk, 16 * sizeof(int));
  if (st) cudaStreamDestroy(st);
}

namespace {
std::mutex g_pool_mu;
// idle problems (streams synchronised); never destroyed at process exit (the CUDA runtime and the
// allocator's own statics may already be gone by then)
auto& g_pool = *new std::vector<std::unique_ptr<Problem>>();
constexpr int kPoolPerOrder = 2;
}  // namespace

void problem_release(std::unique_ptr<Problem> p) {
  if (!p) return;
  if (p->sharded() || p->emul_world > 1) return;  // destroyed (unique_ptr goes out of scope)
  for (Problem* c : {p.get(), p->aux_.get(), p->aux2_.get(), p->aux3_.get(), p->crit_.get()})
    if (c && c->st) KOT_CUDA(cudaStreamSynchronize(c->st));
  std::lock_guard<std::mutex> lk(g_pool_mu);
  int same = 0;
  for (auto& q : g_pool) same += (q->n == p->n && q->device == p->device);
  if (same < kPoolPerOrder) g_pool.push_back(std::move(p));
}

static void refresh_children(Problem& p) {
  for (Problem* c : {p.aux_.get(), p.aux2_.get(), p.aux3_.get(), p.crit_.get()}) {
    if (!c) continue;
    c->l1 = p.l1;
    c->l2 = p.l2;
    c->q_sq = p.q_sq;
    c->jitter = p.jitter;
    c->has_embed = p.has_embed;
    c->g2_valid = false;
  }
}

static std::unique_ptr<Problem> make_problem(int n, int device) {
  kot_require(n >= 1, KOT_EINVAL, "problem order must be >= 1");
  KOT_CUDA(cudaSetDevice(device));
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    for (auto it = g_pool.begin(); it != g_pool.end(); ++it)
      if ((*it)->n == n && (*it)->device == device) {
        std::unique_ptr<Problem> p = std::move(*it);
        g_pool.erase(it);
        p->Kmat = nullptr;
        p->g2_valid = false;
        p->has_embed = false;
        return p;
      }
  }
  std::unique_ptr<Problem> p(new Problem());
  p->n = n;
  p->device = device;
  {  // the Newton chain (critical path) gets the highest stream priority
    int lo = 0, hi = 0;
    KOT_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    KOT_CUDA(cudaStreamCreateWithPriority(&p->st, cudaStreamNonBlocking, hi));
  }
  const long nn = (long)n * n;
  p->Q = p->alloc(nn);
  p->z = p->alloc(n);
  p->R = p->alloc(nn);
  p->embed = p->alloc(n);
  p->init_scratch();
  p->row1 = n;
  return p;
}

__global__ void sym_copy_kernel(const double* __restrict__ a, double* __restrict__ out, int n) {
  const long total = (long)n * n;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    const int r = (int)(i / n), c = (int)(i % n);
    out[i] = 0.5 * (a[i] + a[(long)c * n + r]);  // problem.py:112 q_mat = symmetrize(q)
  }
}

int ew_grid(long count) { return (int)std::min<long>(ceil_div(count, 256), 4L * kNumSMs * 8); }

std::unique_ptr<Problem> problem_from_host(const double* q, const double* z, double q_sq, const double* r,
                                           const double* embed, int n, double l1, double l2, double jitter,
                                           int device) {
  kot_require(l1 > 0.0 && l2 > 0.0, KOT_EINVAL, "regularization parameters must be positive");
  auto p = make_problem(n, device);
  const long nn = (long)n * n;
  p->l1 = l1;
  p->l2 = l2;
  p->q_sq = q_sq;
  p->jitter = jitter;
  KOT_CUDA(cudaMemcpyAsync(p->M1, q, nn * sizeof(double), cudaMemcpyHostToDevice, p->st));
  sym_copy_kernel<<<ew_grid(nn), 256, 0, p->st>>>(p->M1, p->Q, n);
  KOT_LAUNCH_CHECK();
  KOT_CUDA(cudaMemcpyAsync(p->z, z, n * sizeof(double), cudaMemcpyHostToDevice, p->st));
  KOT_CUDA(cudaMemcpyAsync(p->R, r, nn * sizeof(double), cudaMemcpyHostToDevice, p->st));
  if (embed) {
    KOT_CUDA(cudaMemcpyAsync(p->embed, embed, n * sizeof(double), cudaMemcpyHostToDevice, p->st));
    p->has_embed = true;
  }
  KOT_CUDA(cudaStreamSynchronize(p->st));
  refresh_children(*p);
  return p;
}

std::unique_ptr<Problem> problem_assemble(const double* xs, int nx, const double* ys, int ny, const double* xt,
                                          const double* yt, int l, int d, double bw_x, double bw_y, double bw_xy,
                                          double l1, double l2, int device) {
  kot_require(l1 > 0.0 && l2 > 0.0, KOT_EINVAL, "lambda1 and lambda2 must be positive");
  kot_require(bw_x > 0.0 && bw_y > 0.0 && bw_xy > 0.0, KOT_EINVAL, "bandwidth_sq must be positive");
  kot_require(nx >= 1 && ny >= 1, KOT_EINVAL, "sample set is empty");
  auto p = make_problem(l, device);
  p->l1 = l1;
  p->l2 = l2;
  const long nn = (long)l * l;
  // host → device staging of the raw points (temporaries, freed once the instance is built)
  struct Tmp {
    double* p;
    explicit Tmp(long cnt) : p(static_cast<double*>(dev_alloc(std::max(cnt, 1L) * sizeof(double)))) {}
    ~Tmp() { dev_free(p); }
  };
  Tmp txs((long)nx * d), tys((long)ny * d), txt((long)l * d), tyt((long)l * d), tscratch(nx + ny + 8);
  double *dxs = txs.p, *dys = tys.p, *dxt = txt.p, *dyt = tyt.p;
  KOT_CUDA(cudaMemcpyAsync(dxs, xs, sizeof(double) * nx * d, cudaMemcpyHostToDevice, p->st));
  KOT_CUDA(cudaMemcpyAsync(dys, ys, sizeof(double) * ny * d, cudaMemcpyHostToDevice, p->st));
  KOT_CUDA(cudaMemcpyAsync(dxt, xt, sizeof(double) * l * d, cudaMemcpyHostToDevice, p->st));
  KOT_CUDA(cudaMemcpyAsync(dyt, yt, sizeof(double) * l * d, cudaMemcpyHostToDevice, p->st));
  if (!p->kmat_buf) p->kmat_buf = p->alloc(nn);
  p->Kmat = p->kmat_buf;
  double* scratch = tscratch.p;
  assemble_device(dxs, nx, dys, ny, dxt, dyt, l, d, bw_x, bw_y, bw_xy, l2, p->Q, p->Kmat, p->embed, p->z, p->dsc, scratch, p->st);
  KOT_CUDA(cudaMemcpyAsync(p->hsc, p->dsc, sizeof(double), cudaMemcpyDeviceToHost, p->st));
  KOT_CUDA(cudaStreamSynchronize(p->st));
  p->q_sq = p->hsc[0];
  p->has_embed = true;
  p->jitter = cholesky_psd_device(p->Kmat, l, p->R, p->M1, p->dsc + 32, p->dflag, p->st);
  KOT_CUDA(cudaStreamSynchronize(p->st));
  refresh_children(*p);
  return p;
}

void symmetrize(Problem& p, const double* a, double* out) {
  sym_copy_kernel<<<ew_grid((long)p.n * p.n), 256, 0, p.st>>>(a, out, p.n);
  KOT_LAUNCH_CHECK();
}

// ------------------------------------------------------------- reductions

__global__ void dot_partial_kernel(const double* __restrict__ a, const double* __restrict__ b, long count,
                                   double* __restrict__ part) {
  __shared__ double sh[32];
  double s = 0.0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < count; i += (long)gridDim.x * blockDim.x)
    s += b ? a[i] * b[i] : a[i] * a[i];
  s = block_sum(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void sum_partials_kernel(const double* __restrict__ part, int np, double* __restrict__ out, int do_sqrt) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) s += part[i];
  s = block_sum(s, sh);
  if (threadIdx.x == 0) out[0] = do_sqrt ? sqrt(s) : s;
}

static int red_grid(long count) { return (int)std::min<long>(std::max<long>(ceil_div(count, 4096), 1), 512); }

// writes into p.dsc[slot] asynchronously
void dev_reduce(Problem& p, const double* a, const double* b, long count, int slot, bool sq) {
  const int G = red_grid(count);
  dot_partial_kernel<<<G, 256, 0, p.st>>>(a, b, count, p.red + 512 * slot);
  KOT_LAUNCH_CHECK();
  sum_partials_kernel<<<1, 256, 0, p.st>>>(p.red + 512 * slot, G, p.dsc + slot, sq ? 1 : 0);
  KOT_LAUNCH_CHECK();
}

void fetch(Problem& p, int count) {
  KOT_CUDA(cudaMemcpyAsync(p.hsc, p.dsc, sizeof(double) * count, cudaMemcpyDeviceToHost, p.st));
  KOT_CUDA(cudaStreamSynchronize(p.st));
}

double dev_norm(Problem& p, const double* x, long count) {
  dev_reduce(p, x, nullptr, count, 0, true);
  fetch(p, 1);
  return p.hsc[0];
}

double dev_dot(Problem& p, const double* x, const double* y, long count) {
  dev_reduce(p, x, y, count, 0, false);
  fetch(p, 1);
  return p.hsc[0];
}

// ------------------------------------------------------------ elementwise

__global__ void axpby_kernel(long count, double a, const double* __restrict__ x, double b,
                             const double* __restrict__ y, double* __restrict__ out) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < count; i += (long)gridDim.x * blockDim.x) {
    const double xv = (a == 1.0) ? x[i] : __dmul_rn(a, x[i]);
    const double yv = y ? ((b == 1.0) ? y[i] : __dmul_rn(b, y[i])) : 0.0;
    out[i] = __dadd_rn(xv, yv);
  }
}
void axpby(Problem& p, long count, double a, const double* x, double b, const double* y, double* out) {
  axpby_kernel<<<ew_grid(count), 256, 0, p.st>>>(count, a, x, b, y, out);
  KOT_LAUNCH_CHECK();
}

// out = -(x / c)
__global__ void neg_div_kernel(long count, const double* __restrict__ x, double c, double* __restrict__ out) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < count; i += (long)gridDim.x * blockDim.x)
    out[i] = -(x[i] / c);
}

// POS:   out = G + Gᵀ
// NONPOS: out = S/μ − (G + Gᵀ)   (mode 0, eliminator)   |  S − (G + Gᵀ)  (mode 1, Jacobian)
__global__ void symadd_kernel(int n, const double* __restrict__ G, const double* S, int nonpos, int mode, double mu,
                              double* out) {
  const long total = (long)n * n;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    const int r = (int)(i / n), c = (int)(i % n);
    const double g = __dadd_rn(G[i], G[(long)c * n + r]);
    if (!nonpos)
      out[i] = g;
    else
      out[i] = __dsub_rn(mode == 0 ? S[i] / mu : S[i], g);
  }
}

// out = (a + (1+μ)·b) + c    (Jacobian bottom block + r2)
__global__ void jac_bottom_kernel(long count, const double* __restrict__ a, const double* __restrict__ b, double mu,
                                  const double* __restrict__ c, double* __restrict__ out) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < count; i += (long)gridDim.x * blockDim.x)
    out[i] = __dadd_rn(__dadd_rn(a[i], __dmul_rn(1.0 + mu, b[i])), c[i]);
}

void neg_div(Problem& p, long count, const double* x, double c, double* out) {
  neg_div_kernel<<<ew_grid(count), 256, 0, p.st>>>(count, x, c, out);
  KOT_LAUNCH_CHECK();
}

void jac_bottom(Problem& p, long count, const double* a, const double* b, double mu, const double* c, double* out) {
  jac_bottom_kernel<<<ew_grid(count), 256, 0, p.st>>>(count, a, b, mu, c, out);
  KOT_LAUNCH_CHECK();
}

// ------------------------------------------------------------- Φ finalize


struct FinArgs {
  int n, mode, tiles, tri;
  int r0, r1;  // rows computed (row sharding); default [0, n)
  const double* Q;
  const double* G2;  // nullable: + (G2·u)/μ  (structure-reduced NONPOS matvec)
  const double* u;
  const double* partial;
  const double* z;
  const double* r1v;
  double l2, mu, phsign;
  double* out;
  const double* skipf = nullptr;  // nullable: no-op when *skipf != 0 (batched CG)
  // split H form: only the rows in [own0, own1) ∪ [own2, own3) take the Q / H GEMVs and μv (this
  // rank's share); the other rows get the mixed-block partials alone (summed over ranks afterwards)
  int split_rows = 0, own0 = 0, own1 = 0, own2 = 0, own3 = 0;
};

// warp per row: GEMV row of Q (coalesced) + fixed-order sum of the Φ partials.
__global__ void finalize_kernel(FinArgs f) {
  if (f.skipf != nullptr && *f.skipf != 0.0) return;
  const int warps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  for (int r = f.r0 + blockIdx.x * warps + (threadIdx.x >> 5); r < f.r1; r += gridDim.x * warps) {
    double qv = 0.0, ph = 0.0, gv = 0.0;
    const bool own = !f.split_rows || (r >= f.own0 && r < f.own1) || (r >= f.own2 && r < f.own3);
    if (!own) {  // split H form, another rank's row: the mixed-block partials only
      if (f.partial) {
        for (int tn = lane; tn < f.tiles; tn += 32) ph += f.partial[(long)tn * f.n + r];
        ph = warp_sum(ph);
      }
      if (lane == 0) f.out[r] = ph;
      continue;
    }
    if (f.Q) {
      const double* qr = f.Q + (long)r * f.n;
      for (int c = lane; c < f.n; c += 32) qv += qr[c] * f.u[c];
      qv = warp_sum(qv);
    }
    if (f.G2) {
      const double* gr = f.G2 + (long)r * f.n;
      for (int c = lane; c < f.n; c += 32) gv += gr[c] * f.u[c];
      gv = warp_sum(gv);
    }
    if (f.partial) {
      for (int tn = (f.tri ? r / GB_N : 0) + lane; tn < f.tiles; tn += 32) ph += f.partial[(long)tn * f.n + r];
      ph = warp_sum(ph);
    }
    if (lane) continue;
    const double two_l2 = 2.0 * f.l2;
    double o;
    switch (f.mode) {
      case FIN_RES: o = __dsub_rn(__dsub_rn(qv, f.z[r]) / two_l2, ph); break;
      case FIN_MATVEC: o = __dadd_rn(__dadd_rn(qv / two_l2, __dmul_rn(f.mu, f.u[r])), ph); break;
      case FIN_MATVEC_B: {
        const double mid = f.G2 ? __dadd_rn(gv / f.mu, f.phsign * ph) : ph;
        o = __dadd_rn(__dadd_rn(qv / two_l2, __dmul_rn(f.mu, f.u[r])), mid);
        break;
      }
      case FIN_A1: o = __dsub_rn(-f.r1v[r], ph / (f.mu + 1.0)); break;
      case FIN_JTOP:
        o = __dadd_rn(__dsub_rn(__dadd_rn(qv / two_l2, __dmul_rn(f.mu, f.u[r])), ph), f.r1v[r]);
        break;
      case FIN_PHI: o = ph; break;
      case FIN_GRAD: o = __dsub_rn(qv, f.z[r]) / two_l2; break;
      default: o = qv; break;
    }
    f.out[r] = o;
  }
}

void finalize(Problem& p, int mode, const double* u, bool with_phi, const double* r1, double mu,
                     double* out) {
  FinArgs f;
  f.n = p.n;
  f.mode = mode;
  f.tiles = ceil_div(p.n, GB_N);
  f.tri = 1;
  f.r0 = 0;
  f.r1 = p.n;
  f.G2 = nullptr;
  f.phsign = 1.0;
  const bool need_q = (mode == FIN_RES || mode == FIN_MATVEC || mode == FIN_JTOP || mode == FIN_GRAD || mode == FIN_QV);
  f.Q = need_q ? p.Q : nullptr;
  f.u = u;
  f.partial = with_phi ? p.partial : nullptr;
  f.z = p.z;
  f.r1v = r1;
  f.l2 = p.l2;
  f.mu = mu;
  f.out = out;
  finalize_kernel<<<std::min(ceil_div(p.n, 8), 8 * kNumSMs), 256, 0, p.st>>>(f);
  KOT_LAUNCH_CHECK();
}

// ------------------------------------------- structure-reduced middle operator
//
// With B = R·P (once per outer iteration), Φ(𝒯[Φ*(v)])_i = b_i T̂ b_iᵀ where
// T̂ = W∘(Bᵀ diag(v) B) and W is the eliminator's coefficient matrix in the
// eigenbasis (W_αα = 1/μ, W_αᾱ = ξ, W_ᾱᾱ = 0; psdcone.py:113-121).  Only the
// rows of the smaller sign block are needed:
//   POS    (k ≤ ℓ−k): C = B_αᵀ D B (k×ℓ); T̃ = W∘C with ᾱ columns doubled;
//                     y_i = Σ_a (B T̃ᵀ)_ia B_ia
//   NONPOS (k > ℓ−k): W = (1/μ)·1 − W', W' supported on ᾱ rows/cols:
//                     y = (G2 v)/μ − rowquad(B, W'∘C'),  G2 = (RRᵀ)∘(RRᵀ)
// 4·min(k, ℓ−k)·ℓ² FLOPs per matvec instead of ℓ³ + 8kℓ² (two DMMA GEMMs).
struct EpiMvCoef {
  static constexpr bool kRowDot = false;
  double* C;
  long ldc;
  const double* vals;
  int k, pos;
  double mu;
  __device__ void store(int r, int c, double v) const {
    double o;
    if (pos) {  // row r = eigen index a ∈ α
      if (c < k) {
        o = v / mu;
      } else {
        const double sa = vals[r], sb = vals[c];
        const double eta = sa / (sa - sb);
        o = 2.0 * ((eta / (mu + 1.0 - eta)) * v);
      }
    } else {  // row r ↔ eigen index k + r ∈ ᾱ
      if (c >= k) {
        o = v / mu;
      } else {
        const double sa = vals[c], sb = vals[k + r];
        const double eta = sa / (sa - sb);
        o = 2.0 * ((1.0 / mu - eta / (mu + 1.0 - eta)) * v);
      }
    }
    C[(long)r * ldc + c] = o;
  }
  __device__ double rowdot_weight(int, int) const { return 0; }
  __device__ void rowdot_store(int, int, double) const {}
};

// B's columns regrouped as [smaller sign block | pad | other block | pad] (even widths, ld even).
__global__ void pack_blocks_kernel(const double* __restrict__ B, int n, int k, int pos, int ksp, int ldp,
                                   double* __restrict__ out) {
  const long total = (long)n * ldp;
  const int ks = pos ? k : n - k;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    const int r = (int)(i / ldp), c = (int)(i % ldp);
    int src = -1;
    if (c < ks)
      src = pos ? c : k + c;
    else if (c >= ksp && c - ksp < n - ks)
      src = pos ? k + (c - ksp) : c - ksp;
    out[i] = src >= 0 ? B[(long)r * n + src] : 0.0;
  }
}

// Mixed-sign block only (H form): T̃ = 2ξ∘C on α×ᾱ.  pos: row r = a ∈ α, column c ↔ k + c ∈ ᾱ;
// else row r ↔ k + r ∈ ᾱ, column c = a ∈ α.  ξ = η/(μ+1−η), η = σ_a/(σ_a − σ_b) (psdcone.py:35-49).
struct EpiMvOff {
  static constexpr bool kRowDot = false;
  double* C;
  long ldc;
  const double* vals;
  int k, pos;
  double mu;
  int coff = 0;  // column offset of this launch inside the mixed block (split H form); C is pre-offset
  __device__ void store(int r, int c, double v) const {
    const int cg = c + coff;
    const double sa = pos ? vals[r] : vals[cg], sb = pos ? vals[k + cg] : vals[k + r];
    const double eta = sa / (sa - sb);
    C[(long)r * ldc + c] = 2.0 * ((eta / (mu + 1.0 - eta)) * v);
  }
  __device__ double rowdot_weight(int, int) const { return 0; }
  __device__ void rowdot_store(int, int, double) const {}
};

// G2 = (R Rᵀ) ∘ (R Rᵀ), once per problem (one triangle, mirrored).
struct EpiSquareMirror {
  static constexpr bool kRowDot = false;
  double* C;
  long ldc;
  __device__ void store(int r, int c, double v) const {
    if (r > c) return;
    const double o = v * v;
    C[(long)r * ldc + c] = o;
    C[(long)c * ldc + r] = o;
  }
  __device__ double rowdot_weight(int, int) const { return 0; }
  __device__ void rowdot_store(int, int, double) const {}
};

// Rows [r0, r0 + M) of H = G_α∘G_α (split H form: this rank's rows only).
struct EpiSquareRows {
  static constexpr bool kRowDot = false;
  double* C;  // row r0 of H
  long ldc;
  __device__ void store(int r, int c, double v) const { C[(long)r * ldc + c] = v * v; }
  __device__ double rowdot_weight(int, int) const { return 0; }
  __device__ void rowdot_store(int, int, double) const {}
};

// Row blocks of B this process computes: its own block under NCCL sharding, every
// block in turn under the single-device emulation hook (emul_world > 1), else [0, n).
static std::vector<std::pair<int, int>> row_blocks(const Problem& p) {
  std::vector<std::pair<int, int>> v;
  if (p.sharded()) {
    v.emplace_back(p.row0, p.row1);
  } else if (p.emul_world > 1) {
    const int blk = (p.n + p.emul_world - 1) / p.emul_world;
    for (int g = 0; g < p.emul_world; ++g) v.emplace_back(std::min(p.n, g * blk), std::min(p.n, (g + 1) * blk));
  } else {
    v.emplace_back(0, p.n);
  }
  return v;
}

void matvec_prepare(Problem& p, const Decomp& dc, double mu, MvCtx& m, bool allow_hform,
                    cudaStream_t stream) {
  const cudaStream_t st = stream ? stream : p.st;
  const int n = p.n;
  Bufs& b = p.bufs();
  m.dc = dc;
  m.mu = mu;
  static const bool direct = [] {
    const char* e = std::getenv("KOT_MATVEC");
    return e != nullptr && std::string(e) == "direct";
  }();
  m.direct = direct;
  if (direct) return;
  m.pos = dc.k <= n - dc.k;
  m.B = b.Bm;
  static const bool full = [] {
    const char* e = std::getenv("KOT_MATVEC");
    return e != nullptr && std::string(e) == "full";
  }();
  const int world = p.sharded() ? p.shard_world : p.emul_world;
  m.hform = allow_hform && !full;
  m.split = m.hform && world > 1;
  m.world = m.split ? world : 1;
  m.H = b.Hm;
  // B = R P; R upper triangular: a row block's K range starts at its first row
  auto b_rows = [&](int r0, int r1, double* dst) {
    if (r1 <= r0) return;
    GemmShape s = make_shape(r1 - r0, n, n, p.R + (long)r0 * n, n, dc.P, n);
    s.kb_m = 1;
    s.kstart = r0;
    gemm_launch<false, false>(s, EpiAxpby{dst, n, 1.0, 0.0}, st);
  };
  if (m.split && p.sharded()) {
    // every rank needs all of B (both GEMMs contract over all rows): each computes its two folded row
    // blocks (equal shares of R's triangle) into its slots of the gather-order staging (slot g: block
    // g, slot N+g: block 2N−1−g), two all-gathers, then B in natural row order
    const int N = world, g = p.shard_rank;
    const FoldedRows f = folded_rows(n, g, N);
    const long slot = (long)f.blk * n;
    if (p.shard_stage_cap < 2L * N * slot) {
      p.shard_stage = p.alloc(2L * N * slot);
      p.shard_stage_cap = 2L * N * slot;
    }
    double* S = p.shard_stage;
    b_rows(f.a0, f.a1, S + g * slot);
    b_rows(f.b0, f.b1, S + (long)(N + g) * slot);
    shard_allgather(p, S, slot, st);
    shard_allgather(p, S + (long)N * slot, slot, st);
    const long first = std::min<long>(n, (long)N * f.blk);  // blocks 0..N−1 are contiguous in both
    KOT_CUDA(cudaMemcpyAsync(b.Bm, S, sizeof(double) * first * n, cudaMemcpyDeviceToDevice, st));
    for (int h = 0; h < N; ++h) {
      const FoldedRows fh = folded_rows(n, h, N);
      if (fh.b1 > fh.b0)
        KOT_CUDA(cudaMemcpyAsync(b.Bm + (long)fh.b0 * n, S + (long)(N + h) * slot,
                                 sizeof(double) * (fh.b1 - fh.b0) * n, cudaMemcpyDeviceToDevice, st));
    }
  } else {
    for (const auto& [r0, r1] : row_blocks(p)) b_rows(r0, r1, b.Bm + (long)r0 * n);
  }
  if (m.hform) {
    // The sign blocks of B packed side by side with even widths, so that every operand of the
    // matvec GEMMs is 16-byte aligned (16-byte cp.async) whatever the parity of k.
    const int k = dc.k, ks = m.pos ? k : n - k, ns = n - ks;
    const int ksp = ks + (ks & 1), nsp = ns + (ns & 1);
    m.ldp = ksp + nsp;
    pack_blocks_kernel<<<ew_grid((long)n * m.ldp), 256, 0, st>>>(b.Bm, n, k, m.pos ? 1 : 0, ksp, m.ldp, b.Bp);
    KOT_LAUNCH_CHECK();
    m.Bs = b.Bp;
    m.Bo = b.Bp + ksp;
    // H = G_α∘G_α, G_α = B_α B_αᵀ (one triangle + mirror, once per Newton step): the α×α block of
    // W∘(Bᵀdiag(v)B) is the constant 1/μ, so its share of Φ(𝒯[Φ*(v)])_i = Σ_j v_j (b_iα·b_jα)²/μ
    // is the GEMV (H v)/μ, and only the α×ᾱ block remains for the two GEMMs of every matvec.
    if (k == 0) {
      KOT_CUDA(cudaMemsetAsync(m.H, 0, sizeof(double) * n * n, st));
    } else if (m.split) {  // only the rows of this rank's folded blocks (every block under emulation)
      const double* Ba = m.pos ? m.Bs : m.Bo;
      for (int g = 0; g < world; ++g) {
        if (p.sharded() && g != p.shard_rank) continue;
        const FoldedRows f = folded_rows(n, g, world);
        for (const auto& [r0, r1] : {std::make_pair(f.a0, f.a1), std::make_pair(f.b0, f.b1)}) {
          if (r1 <= r0) continue;
          GemmShape s = make_shape(r1 - r0, n, k, Ba + (long)r0 * m.ldp, m.ldp, Ba, m.ldp);
          gemm_launch<false, true>(s, EpiSquareRows{m.H + (long)r0 * n, n}, st);
        }
      }
    } else {
      const double* Ba = m.pos ? m.Bs : m.Bo;
      GemmShape s = make_shape(n, n, k, Ba, m.ldp, Ba, m.ldp);
      s.sym_tiles = 1;
      gemm_launch<false, true>(s, EpiSquareMirror{m.H, n}, st);
    }
    return;
  }
  if (!m.pos && !p.g2_valid) {
    if (p.G2 == nullptr) p.G2 = p.alloc((long)n * n);
    p.g2_valid = true;
    GemmShape s = make_shape(n, n, n, p.R, n, p.R, n);  // (R Rᵀ)_ij = Σ_{k ≥ max(i,j)} R_ik R_jk
    s.kb_m = 1;
    s.kb_n = 1;
    s.sym_tiles = 1;
    gemm_launch<false, true>(s, EpiSquareMirror{p.G2, n}, st);
  }
}

// CTAs a CG-matvec GEMM should have to fill every SM (KOT_MV_CTAS, default 2.5 per SM)
static int mv_target_ctas() {
  static const int v = [] {
    const char* e = std::getenv("KOT_MV_CTAS");
    return e ? std::max(1, std::atoi(e)) : (5 * kNumSMs) / 2;
  }();
  return v;
}

// y = Qv/(2λ₂) + μv + (Hv)/μ + Σ_{a∈α, b∈ᾱ} 2ξ_ab (B_{:,a}∘B_{:,b})·C_ab,  C = Bᵀdiag(v)B
// (one process, no row blocks): two DMMA GEMMs of 2·k(ℓ−k)·ℓ FLOPs each + two GEMVs.
// Split H form, rank g of N: the columns [c0, c1) of the mixed block (both GEMMs; even bounds keep
// every operand 16-byte aligned) — the y partials over all ℓ rows — plus the Q / H GEMVs and μv on the
// rows of g's folded blocks; the ranks' vectors add up to the unsplit matvec.
static void split_cols(int ns, int g, int world, int& c0, int& c1) {
  c0 = (int)(((long)ns * g / world) & ~1L);
  c1 = g == world - 1 ? ns : (int)(((long)ns * (g + 1) / world) & ~1L);
}

static void middle_operator_hform(Problem& p, const MvCtx& m, const double* v, double* out,
                                  const double* skipf, int part = 0) {
  const int n = p.n, k = m.dc.k;
  const int ks = m.pos ? k : n - k;  // rows of T̃ (the smaller sign block)
  int c0 = 0, c1 = n - ks;
  if (m.split) split_cols(n - ks, part, m.world, c0, c1);
  const int ns = c1 - c0;  // this launch's columns of the other block
  const double nn = n;
  ProfScope ps("matvec", p.st, 4.0 * ks * (double)ns * nn + 4.0 * nn * nn / m.world);
  double* Ct = p.mv_ct ? p.mv_ct : p.bufs().Ct;
  const double* Bs = m.Bs;       // columns of the T̃-row block (the smaller sign block)
  const double* Bo = m.Bo + c0;  // this launch's columns of the other block
  const long ld = m.ldp;
  int rd_tiles = 0;
  if (ks > 0 && ns > 0) {
    GemmShape s = make_shape(ks, ns, n, Bs, ld, Bo, ld);
    s.kscale = v;
    s.skipf = skipf;
    s.ws = p.splitws;
    s.ksplit = choose_ksplit(s, p.splitws_cap);
    // split-K so that the launch has enough CTAs to spread over every SM: the sign-block split k
    // moves every iteration, and e.g. 162 tiles on 148 SMs leave 14 SMs with twice the work (ncu:
    // tensor pipe 61 % active); KOT_MV_SPLIT forces a factor
    static const int mv_split = [] {
      const char* e = std::getenv("KOT_MV_SPLIT");
      return e ? std::atoi(e) : 0;
    }();
    const int t1 = ceil_div(ks, GB_M) * ceil_div(ns, GB_N);
    const int sp1 = mv_split > 0 ? mv_split : std::min(4, std::max(1, ceil_div(mv_target_ctas(), t1)));
    if (sp1 > 1 && (long)sp1 * s.M * s.N <= p.splitws_cap) s.ksplit = sp1;
    gemm_launch<true, false>(s, EpiMvOff{Ct + c0, n, m.dc.vals, k, m.pos ? 1 : 0, m.mu, c0}, p.st);
    GemmShape s2 = make_shape(n, ks, ns, Bo, ld, Ct + c0, n);
    s2.skipf = skipf;
    // optional split-K on the row-dot GEMM (each K share adds its own partial rows, summed in fixed
    // order by finalize); KOT_MV2_SPLIT=2 measured neutral inside the solver (12.66 vs 12.68 it/s)
    static const int mv2_split = [] {
      const char* e = std::getenv("KOT_MV2_SPLIT");
      return e ? std::max(0, std::atoi(e)) : 0;
    }();
    const int t2 = ceil_div(n, GB_M) * ceil_div(ks, GB_N);
    const int sp2 = mv2_split > 0 ? mv2_split : std::min(2, std::max(1, ceil_div(mv_target_ctas(), t2)));
    s2.ksplit = (sp2 > 1 && (long)sp2 * ceil_div(ks, GB_N) <= ceil_div(n, GB_N) && ns >= 256 * sp2) ? sp2 : 1;
    gemm_launch<false, true>(s2, EpiRowDot{Bs, ld, p.partial, n}, p.st);
    rd_tiles = ceil_div(ks, GB_N) * s2.ksplit;
  }
  FinArgs f;
  f.n = n;
  f.mode = FIN_MATVEC_B;
  f.tiles = (ks > 0 && ns > 0) ? rd_tiles : 0;
  f.tri = 0;
  f.Q = p.Q;
  f.G2 = m.H;
  f.skipf = skipf;
  f.u = v;
  f.partial = f.tiles > 0 ? p.partial : nullptr;
  f.z = p.z;
  f.r1v = nullptr;
  f.l2 = p.l2;
  f.mu = m.mu;
  f.phsign = 1.0;
  f.out = out;
  f.r0 = 0;
  f.r1 = n;
  if (m.split) {
    const FoldedRows fr = folded_rows(n, part, m.world);
    f.split_rows = 1;
    f.own0 = fr.a0;
    f.own1 = fr.a1;
    f.own2 = fr.b0;
    f.own3 = fr.b1;
  }
  finalize_kernel<<<std::min(ceil_div(n, 8), 8 * kNumSMs), 256, 0, p.st>>>(f);
  KOT_LAUNCH_CHECK();
}

void middle_operator_fast(Problem& p, const MvCtx& m, const double* v, double* out, const double* skipf) {
  const int n = p.n, k = m.dc.k;
  const int ks = m.pos ? k : n - k;
  const bool nccl = p.sharded();  // NCCL or the caller's host data plane
  const auto blocks = row_blocks(p);
  const double nn = n, own = nccl ? p.row1 - p.row0 : n;
  Bufs& b = p.bufs();
  if (m.hform && m.split) {
    kot_require(skipf == nullptr, KOT_EINVAL, "the split H form runs the CG without batching");
    if (nccl) {  // this rank's share, then Σ over ranks (ℓ doubles)
      middle_operator_hform(p, m, v, out, nullptr, p.shard_rank);
      shard_allreduce_sum(p, out, n, p.st);
    } else {  // emulation: every rank's share in turn, summed in rank order
      if (!p.mv_y) p.mv_y = p.alloc(n);
      middle_operator_hform(p, m, v, out, nullptr, 0);
      for (int g = 1; g < m.world; ++g) {
        middle_operator_hform(p, m, v, p.mv_y, nullptr, g);
        axpby(p, n, 1.0, out, 1.0, p.mv_y, out);
      }
    }
    return;
  }
  if (m.hform) {
    middle_operator_hform(p, m, v, out, skipf);
    return;
  }
  kot_require(skipf == nullptr, KOT_EINVAL, "batched CG needs the H-form matvec");
  ProfScope ps("matvec", p.st, 4.0 * ks * nn * own + 2.0 * nn * own);
  const double* Bsub = m.pos ? m.B : m.B + k;
  if (ks > 0) {
    // C = B_subᵀ diag(v) B summed over row blocks, coefficients in the epilogue → T̃ (ks × n).
    // W∘ is linear in C, so the coefficient-scaled block partials simply add.
    bool first = true;
    for (const auto& [r0, r1] : blocks) {
      if (r1 <= r0) continue;
      double* dst = first ? b.Ct : p.shard_tmp;
      GemmShape s = make_shape(ks, n, r1 - r0, Bsub + (long)r0 * n, n, m.B + (long)r0 * n, n);
      s.kscale = v + r0;
      s.ws = p.splitws;
      s.ksplit = choose_ksplit(s, p.splitws_cap);
      // split-K 3 even when the tile count would not need it: inside the concurrent solver the
      // extra CTAs fill SMs left between the other chains' kernels (probe cfg3: matvec 1.06 →
      // 0.94–1.0 ms, 7.8 → 8.0 it/s; 2/4/6 measured worse).  KOT_MV_SPLIT overrides.
      static const int mv_split = [] {
        const char* e = std::getenv("KOT_MV_SPLIT");
        return e ? std::atoi(e) : 3;
      }();
      if (mv_split > 1 && (long)mv_split * s.M * s.N <= p.splitws_cap) s.ksplit = mv_split;
      gemm_launch<true, false>(s, EpiMvCoef{dst, n, m.dc.vals, k, m.pos ? 1 : 0, m.mu}, p.st);
      if (!first) axpby(p, (long)ks * n, 1.0, b.Ct, 1.0, p.shard_tmp, b.Ct);
      first = false;
    }
    if (first) KOT_CUDA(cudaMemsetAsync(b.Ct, 0, sizeof(double) * ks * n, p.st));
    if (nccl) shard_allreduce_sum(p, b.Ct, (long)ks * n);  // Σ over ranks
    for (const auto& [r0, r1] : blocks) {  // y_i = Σ_a (B T̃ᵀ)_ia B_sub[i][a] for the block's rows
      if (r1 <= r0) continue;
      GemmShape s = make_shape(r1 - r0, ks, n, m.B + (long)r0 * n, n, b.Ct, n);
      gemm_launch<false, true>(s, EpiRowDot{Bsub + (long)r0 * n, n, p.partial + r0, n}, p.st);
    }
  }
  FinArgs f;
  f.n = n;
  f.mode = FIN_MATVEC_B;
  f.tiles = ks > 0 ? ceil_div(ks, GB_N) : 0;
  f.tri = 0;
  f.Q = p.Q;
  f.G2 = m.pos ? nullptr : p.G2;
  f.u = v;
  f.partial = ks > 0 ? p.partial : nullptr;
  f.z = p.z;
  f.r1v = nullptr;
  f.l2 = p.l2;
  f.mu = m.mu;
  f.phsign = -1.0;  // complement form: (G2·v)/μ − ph
  f.out = nccl ? p.ygather : out;  // r0 = rank·block: own rows land at ygather[r0 …]
  f.r0 = blocks.front().first;
  f.r1 = blocks.back().second;
  if (f.r1 > f.r0) {
    finalize_kernel<<<std::min(ceil_div(f.r1 - f.r0, 8), 8 * kNumSMs), 256, 0, p.st>>>(f);
    KOT_LAUNCH_CHECK();
  }
  if (nccl) {
    shard_allgather(p, p.ygather, p.shard_block);
    KOT_CUDA(cudaMemcpyAsync(out, p.ygather, sizeof(double) * n, cudaMemcpyDeviceToDevice, p.st));
  }
}

// Φ(X) row-dot partials: tile (tm, tn>=tm) of R·X contracted against R.
void phi_partials(Problem& p, const double* X) {
  const int n = p.n;
  GemmShape s = make_shape(n, n, n, p.R, n, X, n);
  s.kb_m = 1;       // R[m][k] = 0 for k < m
  s.sym_tiles = 1;  // R[r][c] = 0 for c < r ⇒ tiles tn < tm contribute nothing
  EpiRowDot epi{p.R, n, p.partial, n};
  gemm_launch<false, false>(s, epi, p.st);
}

void phi_forward(Problem& p, const double* X, double* out) {
  phi_partials(p, X);
  finalize(p, FIN_PHI, nullptr, true, nullptr, 0.0, out);
}

// out = beta·X + alpha·(Rᵀdiag(γ)R + diag·I), one triangle + mirror.
void phi_adjoint_ex(Problem& p, const double* g, double* out, double alpha, const double* X, double beta,
                           double diag) {
  const int n = p.n;
  GemmShape s = make_shape(n, n, n, p.R, n, p.R, n);
  s.kscale = g;
  s.ke_m = 1;
  s.ke_n = 1;
  s.sym_tiles = 1;
  EpiSymMirror epi{out, n, alpha, X, beta, diag};
  gemm_launch<true, false>(s, epi, p.st);
}

void phi_adjoint(Problem& p, const double* g, double* out) { phi_adjoint_ex(p, g, out, 1.0, nullptr, 0.0, 0.0); }

void eigh(Problem& p, const double* Z, Decomp& dc, bool alpha_only) {
  ProfScope ps("eigh", p.st, 14.0 / 3.0 * p.n * (double)p.n * p.n);
  syevd_device(Z, p.n, dc.P, dc.vals, p.dk, *p.eig, p.st, p.lane, alpha_only);
  KOT_CUDA(cudaMemcpyAsync(p.hk, p.dk, sizeof(int), cudaMemcpyDeviceToHost, p.st));
  KOT_CUDA(cudaStreamSynchronize(p.st));
  dc.k = p.hk[0];
}

void proj(Problem& p, const Decomp& dc, const double* X, double* out) {
  const int n = p.n;
  GemmShape s = make_shape(n, n, dc.k, dc.P, n, dc.P, n);
  s.kscale = dc.vals;
  s.sym_tiles = 1;
  EpiSymMirror epi = X ? EpiSymMirror{out, n, -1.0, X, 1.0, 0.0} : EpiSymMirror{out, n, 1.0, nullptr, 0.0, 0.0};
  gemm_launch<false, true>(s, epi, p.st);
}

// Ĉ = W∘C on the α (pos) or ᾱ rows; ξ/η computed from σ (psdcone.py:67-80,103-110).
struct EpiSpectral {
  static constexpr bool kRowDot = false;
  double* C;
  long ldc;
  const double* vals;
  int k, pos, mode;
  double mu;
  __device__ void store(int r, int c, double v) const {
    double o;
    if (pos) {
      if (c < k) {
        o = (mode == 0) ? v / (2.0 * mu) : v * 0.5;
      } else {
        const double sa = vals[r], sb = vals[c];
        const double eta = sa / (sa - sb);
        o = (mode == 0) ? (eta / (mu + 1.0 - eta)) * v : eta * v;
      }
    } else {
      if (c >= k) {
        o = (mode == 0) ? v / (2.0 * mu) : v * 0.5;
      } else {
        const double sa = vals[c], sb = vals[k + r];
        const double eta = sa / (sa - sb);
        o = (mode == 0) ? (1.0 / mu - eta / (mu + 1.0 - eta)) * v : (1.0 - eta) * v;
      }
    }
    C[(long)r * ldc + c] = o;
  }
  __device__ double rowdot_weight(int, int) const { return 0; }
  __device__ void rowdot_store(int, int, double) const {}
};

void spectral_filter(Problem& p, const Decomp& dc, const double* S, double* out, double mu, int mode,
                     int force_path) {
  const int n = p.n, k = dc.k;
  const bool pos = (force_path < 0) ? (k <= n - k) : (force_path == 0);
  const int ks = pos ? k : n - k;
  const double* Psub = pos ? dc.P : dc.P + k;
  double* U = p.M3;
  double* C = p.M4;
  double* H = p.M3;
  double* G = p.M5;
  static const int sf_split = [] {
    const char* e = std::getenv("KOT_SF_SPLIT");  // diagnostic: split-K of the ks×ℓ×ℓ products
    return e ? std::atoi(e) : 1;
  }();
  auto split = [&](GemmShape& s) {
    if (sf_split > 1 && (long)sf_split * s.M * s.N <= p.splitws_cap) {
      s.ws = p.splitws;
      s.ksplit = sf_split;
    }
  };
  if (ks > 0) {
    {  // U = P_subᵀ S
      GemmShape s = make_shape(ks, n, n, Psub, n, S, n);
      split(s);
      gemm_launch<true, false>(s, EpiAxpby{U, n, 1.0, 0.0}, p.st);
    }
    {  // Ĉ = W ∘ (U P)
      GemmShape s = make_shape(ks, n, n, U, n, dc.P, n);
      split(s);
      gemm_launch<false, false>(s, EpiSpectral{C, n, dc.vals, k, pos ? 1 : 0, mode, mu}, p.st);
    }
    {  // H = Ĉ Pᵀ
      GemmShape s = make_shape(ks, n, n, C, n, dc.P, n);
      split(s);
      gemm_launch<false, true>(s, EpiAxpby{H, n, 1.0, 0.0}, p.st);
    }
  }
  {  // G = P_sub H   (zeros when ks == 0)
    GemmShape s = make_shape(n, n, ks, Psub, n, H, n);
    gemm_launch<false, false>(s, EpiAxpby{G, n, 1.0, 0.0}, p.st);
  }
  symadd_kernel<<<ew_grid((long)n * n), 256, 0, p.st>>>(n, G, S, pos ? 0 : 1, mode, mu, out);
  KOT_LAUNCH_CHECK();
}

double residual_parts(Problem& p, const double* g, const double* X, double* r1, double* r2, Decomp& dc,
                      bool alpha_only) {
  ProfScope ps("residual", p.st);
  const int n = p.n;
  const long nn = (long)n * n;
  phi_partials(p, X);
  finalize(p, FIN_RES, g, true, nullptr, 0.0, r1);
  // Z = X − (Φ*(γ) + λ₁ I)
  phi_adjoint_ex(p, g, p.M1, -1.0, X, 1.0, p.l1);
  eigh(p, p.M1, dc, alpha_only);
  proj(p, dc, X, r2);
  dev_reduce(p, r1, nullptr, n, 0, true);
  dev_reduce(p, r2, nullptr, nn, 1, true);
  fetch(p, 2);
  return p.hsc[0] + p.hsc[1];
}

__global__ void scaled_identity_decomp_kernel(int n, double c, double* P, double* vals) {
  const long total = (long)n * n;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    const long r = i / n, col = i % n;
    P[i] = (r == col) ? 1.0 : 0.0;
    if (r == col) vals[r] = c;
  }
}

// The residual at the starting pair (γ, X) = (0, 0) (solver.py:129-139): Z = −(Φ*(0) + λ₁I) = −λ₁I
// exactly, whose eigendecomposition is known (σ = −λ₁ for every column, P = I, k = 0) — the same
// values LAPACK returns for a scaled identity; the eigensolve is skipped.
double residual_parts_origin(Problem& p, const double* g, const double* X, double* r1, double* r2, Decomp& dc) {
  ProfScope ps("residual", p.st);
  const int n = p.n;
  const long nn = (long)n * n;
  phi_partials(p, X);
  finalize(p, FIN_RES, g, true, nullptr, 0.0, r1);
  scaled_identity_decomp_kernel<<<ew_grid(nn), 256, 0, p.st>>>(n, -p.l1, dc.P, dc.vals);
  KOT_LAUNCH_CHECK();
  dc.k = 0;  // λ₁ > 0
  proj(p, dc, X, r2);
  dev_reduce(p, r1, nullptr, n, 0, true);
  dev_reduce(p, r2, nullptr, nn, 1, true);
  fetch(p, 2);
  return p.hsc[0] + p.hsc[1];
}

void middle_operator(Problem& p, const Decomp& dc, double mu, const double* v, double* out) {
  // F_mv = ℓ³ + 8kℓ² + 2ℓ², k = min(|α|, |ᾱ|)
  const double n = p.n, kk = std::min(dc.k, p.n - dc.k);
  ProfScope ps("matvec", p.st, n * n * n + 8.0 * kk * n * n + 2.0 * n * n);
  phi_adjoint(p, v, p.M1);
  spectral_filter(p, dc, p.M1, p.M2, mu, 0);
  phi_partials(p, p.M2);
  finalize(p, FIN_MATVEC, v, true, nullptr, mu, out);
}

void eg_step(Problem& p, const double* g, const double* X, double s, double* g_out, double* X_out) {
  ProfScope ps("eg_step", p.st);
  Bufs& b = p.bufs();
  const int n = p.n;
  Decomp dc{b.Pe, b.vale, 0};
  // field at v: g_vec = ∇f(γ) − Φ(X); g_mat = Φ*(γ) + λ₁I   (eg.py:27-31)
  phi_partials(p, X);
  finalize(p, FIN_RES, g, true, nullptr, 0.0, b.e1);
  axpby(p, n, 1.0, g, -s, b.e1, b.e2);            // γ½ = γ − s g_vec
  phi_adjoint_ex(p, g, p.M1, -s, X, 1.0, p.l1);     // X − s (Φ*(γ) + λ₁I)
  eigh(p, p.M1, dc, true);                          // projection only: α eigenvectors suffice
  if (p.eig) p.eig->check_cancel(p.st);
  proj(p, dc, nullptr, b.Xh);                       // X½ = Π(·)
  phi_partials(p, b.Xh);
  finalize(p, FIN_RES, b.e2, true, nullptr, 0.0, b.e1);
  phi_adjoint_ex(p, b.e2, p.M1, -s, X, 1.0, p.l1);  // X − s (Φ*(γ½) + λ₁I)
  axpby(p, n, 1.0, g, -s, b.e1, g_out);             // γ − s g_vec(½)
  eigh(p, p.M1, dc, true);
  proj(p, dc, nullptr, X_out);
}

void eg_step_parallel(Problem& p, Problem& c, const double* g, const double* X, double s, double* g_out,
                      double* X_out) {
  ProfScope ps("eg_step", p.st);
  Bufs& b = p.bufs();
  const int n = p.n;
  Decomp dc{b.Pe, b.vale, 0};
  // field at v: g_vec = ∇f(γ) − Φ(X)   (eg.py:27-31);  γ½ = γ − s g_vec
  phi_partials(p, X);
  finalize(p, FIN_RES, g, true, nullptr, 0.0, b.e1);
  axpby(p, n, 1.0, g, -s, b.e1, b.e2);
  if (!p.ev_half) KOT_CUDA(cudaEventCreateWithFlags(&p.ev_half, cudaEventDisableTiming));
  KOT_CUDA(cudaEventRecord(p.ev_half, p.st));
  // second projection on c:  X_out = Π(X − s (Φ*(γ½) + λ₁I))
  std::exception_ptr err = nullptr;
  const int cta_cap = gemm_cta_cap();  // a background caller's GEMM cap applies to its helper too
  const bool bg = background_thread();
  std::thread helper([&] {
    try {
      gemm_cta_cap() = cta_cap;
      background_thread() = bg;
      KOT_CUDA(cudaSetDevice(c.device));
      KOT_CUDA(cudaStreamWaitEvent(c.st, p.ev_half, 0));
      Decomp dc2{c.M2, c.M3, 0};
      phi_adjoint_ex(c, b.e2, c.M1, -s, X, 1.0, c.l1);
      eigh(c, c.M1, dc2, true);
      if (c.eig) c.eig->check_cancel(c.st);
      proj(c, dc2, nullptr, X_out);
      KOT_CUDA(cudaStreamSynchronize(c.st));
    } catch (...) {
      err = std::current_exception();
    }
  });
  try {
    // first projection on p:  X½ = Π(X − s (Φ*(γ) + λ₁I)), then g_out = γ − s (∇f(γ½) − Φ(X½))
    phi_adjoint_ex(p, g, p.M1, -s, X, 1.0, p.l1);
    eigh(p, p.M1, dc, true);
    if (p.eig) p.eig->check_cancel(p.st);
    proj(p, dc, nullptr, b.Xh);
    phi_partials(p, b.Xh);
    finalize(p, FIN_RES, b.e2, true, nullptr, 0.0, b.e1);
    axpby(p, n, 1.0, g, -s, b.e1, g_out);
    KOT_CUDA(cudaStreamSynchronize(p.st));
  } catch (...) {
    helper.join();
    throw;
  }
  helper.join();
  if (err) std::rethrow_exception(err);
}

static void make_context(Problem& src, std::unique_ptr<Problem>& dst, bool high_priority = false,
                         bool with_eig = true) {
  KOT_CUDA(cudaSetDevice(src.device));
  dst.reset(new Problem());
  Problem& a = *dst;
  a.with_eig = with_eig;
  a.n = src.n;
  a.device = src.device;
  a.l1 = src.l1;
  a.l2 = src.l2;
  a.q_sq = src.q_sq;
  a.jitter = src.jitter;
  a.has_embed = src.has_embed;
  a.Q = src.Q;  // shared, not owned
  a.z = src.z;
  a.R = src.R;
  a.embed = src.embed;
  a.lane = high_priority ? 0 : 1;
  int lo = 0, hi = 0;
  KOT_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  KOT_CUDA(cudaStreamCreateWithPriority(&a.st, cudaStreamNonBlocking, high_priority ? hi : lo));
  a.init_scratch();
}

Problem& Problem::crit() {
  if (!crit_) {
    make_context(*this, crit_, true, false);
    Problem& c = *crit_;
    c.crit_dg = c.alloc(n);
    c.crit_dX = c.alloc((long)n * n);
    c.crit_e1 = c.alloc(n);
    KOT_CUDA(cudaEventCreateWithFlags(&c.crit_done, cudaEventDisableTiming));
    KOT_CUDA(cudaEventCreateWithFlags(&c.crit_after, cudaEventDisableTiming));
    KOT_CUDA(cudaEventCreateWithFlags(&c.crit_dx_done, cudaEventDisableTiming));
  }
  return *crit_;
}

// Background (EG pipeline) contexts: lowest stream priority at moderate ℓ, where the Newton chain
// is the critical path (cfg3: 8.30 vs 8.12 it/s); highest from ℓ = 4096, where the pipeline's two
// sequential eigensolves per EG step are (cfg4: 0.453 vs 0.437 it/s).  KOT_EG_PRIORITY=low|high.
static bool eg_high_priority(int n) {
  static const int v = [] {
    const char* e = std::getenv("KOT_EG_PRIORITY");
    if (!e) return -1;
    return std::string(e) == "high" ? 1 : 0;
  }();
  return v < 0 ? n >= 4096 : v == 1;
}

Problem& Problem::aux2() {
  if (!aux2_) {
    make_context(*this, aux2_, eg_high_priority(n));
    aux2_->lane = 2;  // residual thread of the EG pipeline
  }
  return *aux2_;
}

Problem& Problem::aux3() {
  if (!aux3_) {
    make_context(*this, aux3_, eg_high_priority(n));
    aux3_->lane = 1;  // EG step, second projection
  }
  return *aux3_;
}

Problem& Problem::aux() {
  if (!aux_) {
    make_context(*this, aux_, eg_high_priority(n));
    aux_->lane = 1;
  }
  return *aux_;
}

Bufs& Problem::bufs() {
  if (!bufs_) {
    bufs_.reset(new Bufs());
    Bufs& b = *bufs_;
    const long nn = (long)n * n;
    for (double** m : {&b.Xw, &b.Xv, &b.Xt, &b.r2w, &b.r2v, &b.r2t, &b.Pw, &b.Pv, &b.Pt, &b.Pe, &b.Xh, &b.dX,
                       &b.filt, &b.a2t, &b.Bm, &b.Ct, &b.Hm})
      *m = alloc(nn);
    b.Bp = alloc((long)n * (n + 2));
    for (double** v : {&b.gw, &b.gv, &b.gt, &b.r1w, &b.r1v, &b.r1t, &b.valw, &b.valv, &b.valt, &b.vale, &b.dg,
                       &b.a1, &b.rhs, &b.sol, &b.corr, &b.cx, &b.cr, &b.cp, &b.cap, &b.e1, &b.e2, &b.e3})
      *v = alloc(n);
  }
  return *bufs_;
}

}  // namespace kot
