// Algorithm 1 (inexact regularized Newton direction with CG) and Algorithm 2
// (EG-safeguarded SSN loop) on device-resident state.
//
// Reference: newton.py:144-211 (newton_direction, theta_update),
// linalg.py:117-162 (cg_solve), solver.py:114-289 (solve, solve_pure_eg).
// Control flow, tie-breaking and error conditions follow the reference line
// by line; all vectors/matrices stay in HBM and only the scalars that steer
// the control flow (norms, pAp, flags) cross to the host.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <exception>
#include <functional>
#include <mutex>
#include <memory>
#include <thread>
#include <utility>
#include <vector>

#include "gemm.cuh"
#include "ssn.cuh"

namespace kot {

using clk = std::chrono::steady_clock;
static double ms_since(clk::time_point t0) {
  return std::chrono::duration<double, std::milli>(clk::now() - t0).count();
}

// ------------------------------------------------------------------- CG

// 256, not 1024: the single-CTA update must fit beside the resident panel and GEMM CTAs of the other
// chains (a 1024-thread CTA needs a nearly empty SM and waited for one inside the solver)
constexpr int CG_THREADS = 256;
// scalar slots in p.dsc used by CG
constexpr int SC_RR = 8, SC_BN = 9, SC_PAP = 10, SC_RES = 11, SC_FLAG = 12;
// batched CG (device-side stopping): done flag, completed steps, target residual, step limit
constexpr int SC_DONE = 13, SC_IT = 14, SC_TARGET = 15, SC_MAXIT = 16;

__global__ void __launch_bounds__(CG_THREADS) cg_init_kernel(int n, const double* __restrict__ b, double* x,
                                                             double* r, double* pv, double* sc) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double bi = b[i];
    x[i] = 0.0;
    r[i] = bi;
    pv[i] = bi;
    s += bi * bi;
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) {
    sc[SC_RR] = s;
    sc[SC_BN] = sqrt(s);
  }
}

// one CG update after ap = A p (linalg.py:142-161)
__global__ void __launch_bounds__(CG_THREADS) cg_step_kernel(int n, double* x, double* r, double* pv,
                                                             const double* __restrict__ ap, double* sc,
                                                             int batched) {
  __shared__ double sh[32];
  // batched mode: the stopping test of cg_solve runs here (same arithmetic, same order); once it
  // fires, this and every later launch of the batch (matvec kernels included) is a no-op
  if (batched && sc[SC_DONE] != 0.0) return;
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += pv[i] * ap[i];
  const double pap = block_sum(s, sh);
  const double rr = sc[SC_RR];
  __syncthreads();
  if (threadIdx.x == 0) sc[SC_PAP] = pap;
  if (!isfinite(pap)) {
    if (threadIdx.x == 0) {
      sc[SC_FLAG] = 1.0;
      sc[SC_DONE] = 1.0;
    }
    return;
  }
  if (pap <= 0.0) {
    if (threadIdx.x == 0) {
      sc[SC_FLAG] = 2.0;
      sc[SC_DONE] = 1.0;
    }
    return;
  }
  const double alpha = rr / pap;
  double s2 = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    x[i] = __dadd_rn(x[i], __dmul_rn(alpha, pv[i]));
    const double ri = __dsub_rn(r[i], __dmul_rn(alpha, ap[i]));
    r[i] = ri;
    s2 += ri * ri;
  }
  const double rrn = block_sum(s2, sh);
  const double res = sqrt(rrn);
  const double beta = rrn / rr;
  for (int i = threadIdx.x; i < n; i += blockDim.x) pv[i] = __dadd_rn(r[i], __dmul_rn(beta, pv[i]));
  __syncthreads();
  if (threadIdx.x == 0) {
    sc[SC_RES] = res;
    sc[SC_RR] = rrn;
    sc[SC_FLAG] = isfinite(res) ? 0.0 : 3.0;
    if (batched) {
      const double it = sc[SC_IT] + 1.0;
      sc[SC_IT] = it;
      if (!isfinite(res) || res <= sc[SC_TARGET] || it >= sc[SC_MAXIT]) sc[SC_DONE] = 1.0;
    }
  }
}

__global__ void cg_arm_kernel(double* sc, double target, int max_iter) {
  sc[SC_DONE] = 0.0;
  sc[SC_IT] = 0.0;
  sc[SC_TARGET] = target;
  sc[SC_MAXIT] = (double)max_iter;
}

// CG iterations enqueued per host check (KOT_CG_BATCH, test hook kot_debug_cg_batch; 1 = a host
// check after every iteration) and whether the EG step runs its two projections side by side
// (KOT_EG_PARALLEL, kot_debug_eg_parallel)
static std::atomic<int> g_cg_batch{-1}, g_eg_parallel{-1};
static int cg_batch() {
  int v = g_cg_batch.load();
  if (v < 0) {
    const char* e = std::getenv("KOT_CG_BATCH");
    v = e ? std::max(1, std::atoi(e)) : 4;
    g_cg_batch = v;
  }
  return v;
}
static bool eg_parallel() {
  int v = g_eg_parallel.load();
  if (v < 0) {
    const char* e = std::getenv("KOT_EG_PARALLEL");
    v = (e && std::atoi(e) == 0) ? 0 : 1;
    g_eg_parallel = v;
  }
  return v != 0;
}

// Experimental (KOT_L2_PERSIST=<MB>): keep the CG matvec's packed sign blocks of B resident in L2
// (access-policy window on the Newton stream) while the EG chain's eigensolves stream through L2.
struct L2Window {
  cudaStream_t st = nullptr;
  L2Window(Problem& p, const MvCtx& mv) {
    static const long mb = [] {
      const char* e = std::getenv("KOT_L2_PERSIST");
      return e ? std::atol(e) : 0L;
    }();
    if (mb <= 0 || !mv.hform) return;
    static std::once_flag once;
    std::call_once(once, [] { cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)mb << 20); });
    cudaStreamAttrValue a{};
    a.accessPolicyWindow.base_ptr = const_cast<double*>(mv.Bs);
    a.accessPolicyWindow.num_bytes = std::min<size_t>((size_t)mb << 20, sizeof(double) * (size_t)p.n * mv.ldp);
    a.accessPolicyWindow.hitRatio = 1.0f;
    a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    if (cudaStreamSetAttribute(p.st, cudaStreamAttributeAccessPolicyWindow, &a) == cudaSuccess) st = p.st;
    (void)cudaGetLastError();
  }
  ~L2Window() {
    if (!st) return;
    cudaStreamAttrValue a{};
    a.accessPolicyWindow.num_bytes = 0;
    cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &a);
    cudaCtxResetPersistingL2Cache();
    (void)cudaGetLastError();
  }
};

// CUDA-graph replay of the batched CG steps (KOT_CG_GRAPH=0: direct launches).
static bool cg_graphs() {
  static const bool v = [] {
    const char* e = std::getenv("KOT_CG_GRAPH");
    return !(e && std::atoi(e) == 0);
  }();
  return v;
}

// The graph of one batch for the current matvec context; re-captured when the context changes (one
// Newton step: new decomposition, μ, sign blocks), updated in place when the topology allows it.
template <class F>
static void cg_graph_launch(Problem& p, const MvCtx& mv, int batch, F&& enqueue) {
  CgGraph& g = p.cg_graph;
  const CgGraphKey key{mv.Bs, mv.Bo, mv.ldp, mv.H, mv.dc.vals, mv.dc.k, mv.pos, mv.mu, batch};
  if (!g.exec || !(g.key == key)) {
    const long long l0 = thread_launches();
    cudaGraph_t graph = nullptr;
    prof_capturing() = true;
    KOT_CUDA(cudaStreamBeginCapture(p.st, cudaStreamCaptureModeThreadLocal));
    try {
      enqueue();
    } catch (...) {
      cudaStreamEndCapture(p.st, &graph);
      if (graph) cudaGraphDestroy(graph);
      prof_capturing() = false;
      throw;
    }
    KOT_CUDA(cudaStreamEndCapture(p.st, &graph));
    prof_capturing() = false;
    g.kernels = thread_launches() - l0;  // this thread's captured kernels (other threads keep launching)
    g_kot_launches -= g.kernels;        // counted when the graph runs
    bool updated = false;
    if (g.exec) {
      cudaGraphExecUpdateResultInfo info{};
      updated = cudaGraphExecUpdate(g.exec, graph, &info) == cudaSuccess;
      if (!updated) {
        (void)cudaGetLastError();
        cudaGraphExecDestroy(g.exec);
        g.exec = nullptr;
      }
    }
    if (!updated) KOT_CUDA(cudaGraphInstantiate(&g.exec, graph, 0));
    KOT_CUDA(cudaGraphDestroy(graph));
    g.key = key;
  }
  KOT_CUDA(cudaGraphLaunch(g.exec, p.st));
  g_kot_launches += g.kernels;
}

struct CgOut {
  int iters;
  double res;
  bool aborted = false;
};

// x (= b.cx) solves A x = rhs to tol·‖rhs‖ with A = middle operator.  `abort` (nullable) is polled
// after every iteration; when it returns true the solve stops early (speculative attempt discarded).
static CgOut cg_solve(Problem& p, const MvCtx& mv, const double* rhs, double tol, int max_iter,
                      const std::function<bool()>* abort = nullptr) {
  Bufs& b = p.bufs();
  const int n = p.n;
  kot_require(max_iter >= 1, KOT_EINVAL, "max_iter must be >= 1");
  cg_init_kernel<<<1, CG_THREADS, 0, p.st>>>(n, rhs, b.cx, b.cr, b.cp, p.dsc);
  KOT_LAUNCH_CHECK();
  fetch(p, 16);
  const double target = tol * p.hsc[SC_BN];
  double res = p.hsc[SC_BN];
  if (res <= target) return {0, res};
  // Batched stopping (H-form matvec): B iterations are enqueued per host check and the device applies
  // the stopping rule (cg_step_kernel, batched mode) — the launches after the stop are no-ops — so
  // the host waits once per B steps instead of after every step; identical arithmetic and results.
  const int kBatch = cg_batch();
  if (!mv.direct && mv.hform && !mv.split && kBatch > 1) {
    cg_arm_kernel<<<1, 1, 0, p.st>>>(p.dsc, target, max_iter);
    KOT_LAUNCH_CHECK();
    const double* done = p.dsc + SC_DONE;
    auto enqueue_batch = [&]() {
      for (int bq = 0; bq < kBatch; ++bq) {
        middle_operator_fast(p, mv, b.cp, b.cap, done);
        cg_step_kernel<<<1, CG_THREADS, 0, p.st>>>(n, b.cx, b.cr, b.cp, b.cap, p.dsc, 1);
        KOT_LAUNCH_CHECK();
      }
    };
    int launched = 0;
    for (;;) {
      // The device applies the stopping rule (launches after the stop are no-ops, the step limit is
      // SC_MAXIT), so every batch is the same kernel sequence: after the first batch (which also
      // sets every kernel attribute) it is replayed as one CUDA graph per Newton step.
      if (launched == 0 || !cg_graphs())
        enqueue_batch();
      else
        cg_graph_launch(p, mv, kBatch, enqueue_batch);
      launched += kBatch;
      fetch(p, SC_MAXIT + 1);
      const bool stop = p.hsc[SC_DONE] != 0.0 || launched >= max_iter;
      const int it = (int)p.hsc[SC_IT];
      if (stop) {
        const int flag = (int)p.hsc[SC_FLAG];
        if (flag == 1) throw KotError(KOT_ECG, "non-finite curvature in conjugate gradient");
        if (flag == 3) throw KotError(KOT_ECG, "non-finite residual in conjugate gradient");
        return {it, it > 0 ? p.hsc[SC_RES] : res};  // flag 2: the last completed step's residual
      }
      res = p.hsc[SC_RES];
      if (abort && (*abort)()) return {it, res, true};
    }
  }
  int it = 0;
  for (it = 1; it <= max_iter; ++it) {
    if (mv.direct)
      middle_operator(p, mv.dc, mv.mu, b.cp, b.cap);
    else
      middle_operator_fast(p, mv, b.cp, b.cap);
    cg_step_kernel<<<1, CG_THREADS, 0, p.st>>>(n, b.cx, b.cr, b.cp, b.cap, p.dsc, 0);
    KOT_LAUNCH_CHECK();
    fetch(p, 16);
    const int flag = (int)p.hsc[SC_FLAG];
    if (flag == 1) throw KotError(KOT_ECG, "non-finite curvature in conjugate gradient");
    if (flag == 2) {  // p collapsed to numerical zero on an SPD operator
      it -= 1;
      break;
    }
    res = p.hsc[SC_RES];
    if (flag == 3) throw KotError(KOT_ECG, "non-finite residual in conjugate gradient");
    if (res <= target) return {it, res};
    if (abort && (*abort)()) return {it, res, true};
  }
  if (it > max_iter) it = max_iter;
  return {it, res};
}

// linalg.cg_solve (linalg.py:117-162) for any operator `apply(p_dev, ap_dev)` on p's stream: the same
// recurrence, stopping rule and error conditions as the solver's CG (cg_init/cg_step kernels).
CgResult cg_solve_op(Problem& p, const double* rhs, double tol, int max_iter,
                     const std::function<void(const double*, double*)>& apply, double* x_out) {
  Bufs& b = p.bufs();
  const int n = p.n;
  kot_require(max_iter >= 1, KOT_EINVAL, "max_iter must be >= 1");
  cg_init_kernel<<<1, CG_THREADS, 0, p.st>>>(n, rhs, b.cx, b.cr, b.cp, p.dsc);
  KOT_LAUNCH_CHECK();
  fetch(p, 16);
  const double target = tol * p.hsc[SC_BN];
  double res = p.hsc[SC_BN];
  int it = 0;
  if (res > target) {
    for (it = 1; it <= max_iter; ++it) {
      apply(b.cp, b.cap);
      cg_step_kernel<<<1, CG_THREADS, 0, p.st>>>(n, b.cx, b.cr, b.cp, b.cap, p.dsc, 0);
      KOT_LAUNCH_CHECK();
      fetch(p, 16);
      const int flag = (int)p.hsc[SC_FLAG];
      if (flag == 1) throw KotError(KOT_ECG, "non-finite curvature in conjugate gradient");
      if (flag == 2) {  // p collapsed to numerical zero on an SPD operator
        it -= 1;
        break;
      }
      res = p.hsc[SC_RES];
      if (flag == 3) throw KotError(KOT_ECG, "non-finite residual in conjugate gradient");
      if (res <= target) break;
    }
    if (it > max_iter) it = max_iter;
  }
  KOT_CUDA(cudaMemcpyAsync(x_out, b.cx, sizeof(double) * n, cudaMemcpyDeviceToDevice, p.st));
  return {it, res};
}

// --------------------------------------------------------------- Newton

// Criterion ‖(J+μI)dw + r‖ ≤ τ min(1, κ‖r‖‖dw‖) for dw = (sol, ã2 − 𝒯[Φ*(sol)]) (newton.py:131-141,
// problem.py:222-236).  With that dw the two blocks of (J+μI)dw + r are, exactly (Lemma 1):
//   top    = Q sol/(2λ₂) + μ sol − Φ(ã2 − 𝒯Φ*(sol)) + r1 = A·sol − a1   (A: the middle operator,
//            a1 = −r1 + Φ(ã2)), i.e. minus the true residual of the reduced system;
//   bottom = M[Φ*(sol) − dX] + (1+μ)dX + r2 = 0, because dX = −((1+μ)I − M)⁻¹(r2 + MΦ*(sol)) and
//            ã2 = −((1+μ)I − M)⁻¹ r2 (M, 𝒯 share the eigenbasis, 𝒯 = M((1+μ)I − M)⁻¹).
// So lhs = ‖a1 − A·sol‖₂: the next attempt's right-hand side, which the main stream computes anyway
// (`rhs_next`), or one matvec on the criterion context after the last attempt.  The reference
// evaluates the same quantity through apply_jacobian (Φ, Φ*, a dense M, four GEMM chains); the two
// differ by rounding only.  dw itself (needed for ‖dw‖ and as the step) is built here as before.
// Enqueued on the criterion context q after `crit_after` (recorded on p's stream): dw into
// q.crit_dg / q.crit_dX, the norms into q.hsc[0..3], completion = q.crit_done.
static void criterion_enqueue(Problem& p, Problem& q, const Decomp& dc, double mu, const MvCtx& mv,
                              const double* rhs_next, cudaEvent_t rhs_ready) {
  Bufs& b = p.bufs();
  const int n = p.n;
  const long nn = (long)n * n;
  KOT_CUDA(cudaEventRecord(q.crit_after, p.st));
  KOT_CUDA(cudaStreamWaitEvent(q.st, q.crit_after, 0));
  ProfScope pcrit("newton.criterion", q.st);
  KOT_CUDA(cudaMemcpyAsync(q.crit_dg, b.sol, sizeof(double) * n, cudaMemcpyDeviceToDevice, q.st));
  phi_adjoint(q, b.sol, q.M1);
  spectral_filter(q, dc, q.M1, q.M2, mu, 0);
  axpby(q, nn, 1.0, b.a2t, -1.0, q.M2, q.crit_dX);
  KOT_CUDA(cudaEventRecord(q.crit_dx_done, q.st));  // dw is complete; the norms below feed the record
  const double* top;
  if (rhs_next) {  // a1 − A·sol, from the main stream
    KOT_CUDA(cudaStreamWaitEvent(q.st, rhs_ready, 0));
    top = rhs_next;
  } else {  // after the last attempt: the (H-form) matvec here, off the critical path
    if (!q.mv_ct) q.mv_ct = q.alloc(nn);
    middle_operator_fast(q, mv, q.crit_dg, q.crit_e1);
    axpby(q, n, 1.0, b.a1, -1.0, q.crit_e1, q.crit_e1);
    top = q.crit_e1;
  }
  dev_reduce(q, top, nullptr, n, 0, true);
  KOT_CUDA(cudaMemsetAsync(q.dsc + 1, 0, sizeof(double), q.st));  // bottom block: identically zero
  dev_reduce(q, q.crit_dg, nullptr, n, 2, true);
  dev_reduce(q, q.crit_dX, nullptr, nn, 3, true);
  KOT_CUDA(cudaMemcpyAsync(q.hsc, q.dsc, sizeof(double) * 4, cudaMemcpyDeviceToHost, q.st));
  KOT_CUDA(cudaEventRecord(q.crit_done, q.st));
}

// Algorithm 1 (newton.py:144-195).  Attempt a+1 only runs when attempt a's criterion fails, and its
// right-hand side a1 − M(sol) does not depend on that criterion: so the criterion of attempt a runs
// on the criterion context while attempt a+1 already starts on the main stream.  If the criterion
// turns out met, the speculative attempt is discarded before it touches `sol` — same arithmetic,
// same results, the criterion's latency off the critical path whenever it fails.
NewtonOut newton_direction(Problem& p, const double* r1, const double* r2, double rn, const Decomp& dc, double mu,
                           const SolverCfg& cfg, double* dg, double* dX) {
  Bufs& b = p.bufs();
  const int n = p.n;
  const long nn = (long)n * n;
  kot_require(rn > 0.0, KOT_EINVAL, "direction requires a nonzero residual");
  ProfScope ps("newton", p.st);
  // filt = r2 + 𝒯[r2];  a1 = −r1 − Φ(filt)/(μ+1);  ã2 = −filt/(μ+1)   (newton.py:161-163)
  auto ppre = std::make_unique<ProfScope>("newton.prologue", p.st);
  // B = R·P, its packed sign blocks and H depend only on the decomposition: built on the criterion
  // context's (idle) stream beside 𝒯[r2] and the right-hand side, joined before the first matvec
  Problem& q = p.crit();
  if (!p.ev_mv0) {
    KOT_CUDA(cudaEventCreateWithFlags(&p.ev_mv0, cudaEventDisableTiming));
    KOT_CUDA(cudaEventCreateWithFlags(&p.ev_mv1, cudaEventDisableTiming));
    KOT_CUDA(cudaEventCreateWithFlags(&p.ev_rhs, cudaEventDisableTiming));
  }
  KOT_CUDA(cudaEventRecord(p.ev_mv0, p.st));
  KOT_CUDA(cudaStreamWaitEvent(q.st, p.ev_mv0, 0));
  MvCtx mv;
  matvec_prepare(p, dc, mu, mv, true, q.st);
  KOT_CUDA(cudaEventRecord(p.ev_mv1, q.st));
  spectral_filter(p, dc, r2, p.M2, mu, 0);
  axpby(p, nn, 1.0, r2, 1.0, p.M2, b.filt);
  phi_partials(p, b.filt);
  finalize(p, FIN_A1, nullptr, true, r1, mu, b.a1);
  neg_div(p, nn, b.filt, mu + 1.0, b.a2t);
  double rel = cfg.has_cg_tol ? cfg.cg_tol : cfg.tau * std::min(1.0, cfg.kappa * rn);
  const double a1n = dev_norm(p, b.a1, n);
  KOT_CUDA(cudaMemsetAsync(b.sol, 0, sizeof(double) * n, p.st));
  KOT_CUDA(cudaStreamWaitEvent(p.st, p.ev_mv1, 0));
  ppre.reset();
  L2Window l2w(p, mv);
  NewtonOut out{0, 0, 0, INFINITY, 0.0, 0.0};
  const auto t0 = clk::now();
  bool pending = false;  // criterion of attempt `att − 1` in flight on q
  bool pending_met = false;
  auto read_crit = [&]() {
    out.lhs = q.hsc[0] + q.hsc[1];
    const double dwn = q.hsc[2] + q.hsc[3];
    out.rhs = cfg.tau * std::min(1.0, cfg.kappa * rn * dwn);
    out.met = out.lhs <= out.rhs;
  };
  auto resolve = [&](bool wait) {  // true once the pending criterion is known
    if (!pending) return true;
    if (wait) {
      KOT_CUDA(cudaEventSynchronize(q.crit_done));
    } else if (cudaEventQuery(q.crit_done) != cudaSuccess) {
      (void)cudaGetLastError();
      return false;
    }
    read_crit();
    pending = false;
    pending_met = out.met;
    return true;
  };
  auto finish = [&]() {  // the accepted attempt's dw (in q's outputs) → caller's buffers
    KOT_CUDA(cudaStreamWaitEvent(p.st, q.crit_done, 0));
    KOT_CUDA(cudaMemcpyAsync(dg, q.crit_dg, sizeof(double) * n, cudaMemcpyDeviceToDevice, p.st));
    KOT_CUDA(cudaMemcpyAsync(dX, q.crit_dX, sizeof(double) * nn, cudaMemcpyDeviceToDevice, p.st));
    out.cg_ms = ms_since(t0);
  };
  const std::function<bool()> abort_if_met = [&]() { return resolve(false) && pending_met; };
  // Row-sharded problems: each CG matvec is a collective, so every rank must run the same number of
  // them.  The speculative abort polls the criterion's completion (timing-dependent per rank), hence
  // no speculation there: attempt a+1 starts only after attempt a's criterion is known (same result);
  // and the last attempt's lhs matvec (a collective) runs on the main stream, in program order.
  const bool may_speculate = !p.sharded();
  // right-hand sides of attempts ≥ 1 (a1 − A·sol), alternating so that attempt a+2 never overwrites
  // the vector attempt a's criterion still reads (that criterion is resolved before a+2 starts)
  double* rhs_buf[2] = {b.rhs, b.corr};
  for (int att = 0; att <= cfg.cg_restarts; ++att) {
    if (pending && !may_speculate) {
      resolve(true);
      if (pending_met) {
        finish();
        return out;
      }
    }
    const bool speculative = pending;
    CgOut c{0, 0.0};
    bool ran = false;
    try {
      const double* rhs = att ? rhs_buf[att & 1] : b.a1;
      const double bn = dev_norm(p, rhs, n);
      if (bn > 0.0 && a1n > 0.0) {
        c = cg_solve(p, mv, rhs, rel * a1n / bn, cfg.cg_max, speculative ? &abort_if_met : nullptr);
        ran = true;
      }
    } catch (...) {
      // a speculative attempt's failure only counts if its predecessor's criterion failed
      if (speculative && resolve(true) && pending_met) {
        finish();
        return out;
      }
      throw;
    }
    if (speculative) {  // attempt att−1's criterion decides whether this attempt happened at all
      resolve(true);
      if (pending_met) {
        finish();
        return out;
      }
    }
    out.attempts = att + 1;
    if (ran) {
      axpby(p, n, 1.0, b.sol, 1.0, b.cx, b.sol);
      out.cg_iters += c.iters;
    }
    const bool last = att == cfg.cg_restarts;
    const double* rhs_next = nullptr;
    if (!last || !may_speculate || !mv.hform) {  // a1 − A·sol: attempt att+1's rhs and this criterion's lhs
      double* rn_buf = rhs_buf[(att + 1) & 1];
      if (mv.direct)
        middle_operator(p, dc, mu, b.sol, b.e3);
      else
        middle_operator_fast(p, mv, b.sol, b.e3);
      axpby(p, n, 1.0, b.a1, -1.0, b.e3, rn_buf);
      KOT_CUDA(cudaEventRecord(p.ev_rhs, p.st));
      rhs_next = rn_buf;
    }
    criterion_enqueue(p, q, dc, mu, mv, rhs_next, p.ev_rhs);
    pending = true;
    if (last) break;
    rel /= 10.0;
  }
  // The last attempt's criterion only feeds the record (met, lhs, rhs): dw is taken as soon as it is
  // ready and the norms are resolved by the caller (newton_resolve), off the critical path.
  KOT_CUDA(cudaStreamWaitEvent(p.st, q.crit_dx_done, 0));
  KOT_CUDA(cudaMemcpyAsync(dg, q.crit_dg, sizeof(double) * n, cudaMemcpyDeviceToDevice, p.st));
  KOT_CUDA(cudaMemcpyAsync(dX, q.crit_dX, sizeof(double) * nn, cudaMemcpyDeviceToDevice, p.st));
  out.cg_ms = ms_since(t0);
  out.crit_pending = true;
  return out;
}

void newton_resolve(Problem& p, double rn, const SolverCfg& cfg, NewtonOut& out) {
  if (!out.crit_pending) return;
  Problem& q = p.crit();
  KOT_CUDA(cudaEventSynchronize(q.crit_done));
  out.lhs = q.hsc[0] + q.hsc[1];
  const double dwn = q.hsc[2] + q.hsc[3];
  out.rhs = cfg.tau * std::min(1.0, cfg.kappa * rn * dwn);
  out.met = out.lhs <= out.rhs;
  out.crit_pending = false;
}

static double theta_update(double theta, double rho, double dw_sq, const SolverCfg& c) {
  double t;
  if (rho >= c.alpha2 * dw_sq)
    t = std::max(c.theta_min, c.beta0 * theta);
  else if (rho >= c.alpha1 * dw_sq)
    t = c.beta1 * theta;
  else
    t = std::min(c.theta_max, c.beta2 * theta);
  return std::min(std::max(t, c.theta_min), c.theta_max);
}

// ----------------------------------------------------------------- solve

struct HostProbe {
  std::vector<double> wg, wx, rg, rx, dg, dx;
};

static void copy_state(Problem& p, Bufs& b, Decomp& dw, const Decomp& dv) {
  const int n = p.n;
  const long nn = (long)n * n;
  KOT_CUDA(cudaMemcpyAsync(b.gw, b.gv, sizeof(double) * n, cudaMemcpyDeviceToDevice, p.st));
  KOT_CUDA(cudaMemcpyAsync(b.Xw, b.Xv, sizeof(double) * nn, cudaMemcpyDeviceToDevice, p.st));
  KOT_CUDA(cudaMemcpyAsync(b.r1w, b.r1v, sizeof(double) * n, cudaMemcpyDeviceToDevice, p.st));
  KOT_CUDA(cudaMemcpyAsync(b.r2w, b.r2v, sizeof(double) * nn, cudaMemcpyDeviceToDevice, p.st));
  KOT_CUDA(cudaMemcpyAsync(dw.P, dv.P, sizeof(double) * nn, cudaMemcpyDeviceToDevice, p.st));
  KOT_CUDA(cudaMemcpyAsync(dw.vals, dv.vals, sizeof(double) * n, cudaMemcpyDeviceToDevice, p.st));
  dw.k = dv.k;
}

// ------------------------------------------------------------ EG pipeline
//
// The safeguard sequence v_{j+1} = eg_step(v_j) (eg.py:34-41) never depends on
// the Newton iterate: solver.py:186-192 copies v into w on an EG acceptance but
// never the other way.  So v_1, v_2, … and their residuals are produced ahead
// of the Newton chain by two host threads on their own streams (thread A: EG
// steps, thread B: residual at v_j), and the solve loop consumes slot j at the
// iteration whose safeguard step produces v_j.  Same operations, same values,
// same acceptance logic; only the schedule changes (3 concurrent chains).
// CTAs per GEMM launch on the EG-chain threads (KOT_BG_GEMM_CTAS; 0 = uncapped): see gemm_cta_cap.
static int bg_gemm_ctas() {
  static const int v = [] {
    const char* e = std::getenv("KOT_BG_GEMM_CTAS");
    return e ? std::max(0, std::atoi(e)) : 0;
  }();
  return v;
}

struct EgSlot {
  double *g = nullptr, *X = nullptr, *r1 = nullptr, *r2 = nullptr, *P = nullptr, *vals = nullptr;
  int k = 0;
  bool alpha_only = false;  // P holds only the σ > 0 eigenvectors
  double res = 0.0, eg_ms = 0.0, resid_ms = 0.0;
  std::exception_ptr err = nullptr;
};

class EgPipeline {
 public:
  EgPipeline(Problem& p, double stepsize) : p_(p), s_(stepsize) {
    const int n = p.n;
    const long nn = (long)n * n;
    // slot buffers are allocated once per problem and reused by every later solve on it
    if (p.pipe_bufs.empty()) {
      for (int i = 0; i < kDepth; ++i)
        for (long cnt : {(long)n, nn, (long)n, nn, nn, (long)n}) p.pipe_bufs.push_back(p.alloc(cnt));
      p.pipe_bufs.push_back(p.alloc(n));
      p.pipe_bufs.push_back(p.alloc(nn));
    }
    int b = 0;
    for (auto& sl : slots_) {
      sl.g = p.pipe_bufs[b++];
      sl.X = p.pipe_bufs[b++];
      sl.r1 = p.pipe_bufs[b++];
      sl.r2 = p.pipe_bufs[b++];
      sl.P = p.pipe_bufs[b++];
      sl.vals = p.pipe_bufs[b++];
    }
    Problem& a = p.aux();
    Problem& bb = p.aux2();
    Problem& a3 = p.aux3();
    KOT_CUDA(cudaMemsetAsync(v0g_ = p.pipe_bufs[b++], 0, sizeof(double) * n, p.st));
    KOT_CUDA(cudaMemsetAsync(v0X_ = p.pipe_bufs[b++], 0, sizeof(double) * nn, p.st));
    KOT_CUDA(cudaStreamSynchronize(p.st));
    a.eig->cancel = &cancel_;
    bb.eig->cancel = &cancel_;
    a3.eig->cancel = &cancel_;
    eig_pipeline_active(+1);
    ta_ = std::thread([this, &a] { run_steps(a); });
    tb_ = std::thread([this, &bb] { run_residuals(bb); });
  }
  ~EgPipeline() {
    // the steps still running are speculative (v_j beyond the last iteration): cancel them at the
    // next eigensolve panel instead of waiting up to one EG step
    cancel_ = true;
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    ta_.join();
    tb_.join();
    p_.aux().eig->cancel = nullptr;
    p_.aux2().eig->cancel = nullptr;
    p_.aux3().eig->cancel = nullptr;
    eig_pipeline_active(-1);
  }
  // Slot of v_j (j >= 1) once its residual is evaluated.  Also releases v_{j-2}.
  EgSlot& acquire(int j) {
    std::unique_lock<std::mutex> lk(mu_);
    consumed_ = std::max(consumed_, j - 2);  // v_{j-1} stays valid (stale r_v / decomp_v reuse)
    cv_.notify_all();
    cv_.wait(lk, [&] { return evaluated_ >= j || failed_at_ == j; });
    return slots_[j % kDepth];
  }

 private:
  static constexpr int kDepth = 4;
  Problem& p_;
  double s_;
  EgSlot slots_[kDepth];
  double *v0g_ = nullptr, *v0X_ = nullptr;
  std::mutex mu_;
  std::condition_variable cv_;
  bool stop_ = false;
  std::atomic<bool> cancel_{false};
  int produced_ = 0, evaluated_ = 0, consumed_ = 0, failed_at_ = -1;
  std::thread ta_, tb_;

  void run_steps(Problem& a) {
    gemm_cta_cap() = bg_gemm_ctas();
    background_thread() = true;
    for (int j = 1;; ++j) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        // slot j%D is reusable once v_{j-D} was consumed (released) by the solve loop
        cv_.wait(lk, [&] { return stop_ || (j - kDepth <= consumed_ && failed_at_ < 0); });
        if (stop_ || failed_at_ >= 0) return;
      }
      EgSlot& out = slots_[j % kDepth];
      const double* gin = (j == 1) ? v0g_ : slots_[(j - 1) % kDepth].g;
      const double* Xin = (j == 1) ? v0X_ : slots_[(j - 1) % kDepth].X;
      try {
        KOT_CUDA(cudaSetDevice(a.device));
        const auto t0 = clk::now();
        // the step's two projections side by side (default) or in sequence (KOT_EG_PARALLEL=0: fewer
        // concurrent cooperative grids, for many solves sharing one GPU)
        if (eg_parallel()) {
          eg_step_parallel(a, p_.aux3(), gin, Xin, s_, out.g, out.X);
        } else {
          eg_step(a, gin, Xin, s_, out.g, out.X);
          KOT_CUDA(cudaStreamSynchronize(a.st));
        }
        out.eg_ms = ms_since(t0);
        prof_host("host.pipe_eg", out.eg_ms);
      } catch (const Cancelled&) {
        return;
      } catch (...) {
        std::lock_guard<std::mutex> lk(mu_);
        out.err = std::current_exception();
        failed_at_ = j;
        cv_.notify_all();
        return;
      }
      std::lock_guard<std::mutex> lk(mu_);
      produced_ = j;
      cv_.notify_all();
    }
  }

  void run_residuals(Problem& b) {
    gemm_cta_cap() = bg_gemm_ctas();
    background_thread() = true;
    for (int j = 1;; ++j) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || produced_ >= j || failed_at_ >= 0; });
        if (stop_ || (produced_ < j)) return;
      }
      EgSlot& sl = slots_[j % kDepth];
      try {
        KOT_CUDA(cudaSetDevice(b.device));
        const auto t0 = clk::now();
        Decomp dc{sl.P, sl.vals, 0};
        // The decomposition at v is only needed if the EG step is accepted (w ← v), which the
        // trajectories practically never do: compute the σ > 0 part only and
        // redo the full decomposition on acceptance (same kernels, same input → same result).
        static const bool kAlpha = [] {
          const char* e = std::getenv("KOT_PIPE_ALPHA");
          return !(e && std::atoi(e) == 0);
        }();
        sl.res = residual_parts(b, sl.g, sl.X, sl.r1, sl.r2, dc, kAlpha);
        sl.alpha_only = kAlpha;
        sl.k = dc.k;
        sl.resid_ms = ms_since(t0);
        prof_host("host.pipe_resid", sl.resid_ms);
      } catch (const Cancelled&) {
        return;
      } catch (...) {
        std::lock_guard<std::mutex> lk(mu_);
        sl.err = std::current_exception();
        failed_at_ = j;
        cv_.notify_all();
        return;
      }
      std::lock_guard<std::mutex> lk(mu_);
      evaluated_ = j;
      cv_.notify_all();
    }
  }
};

// One pass of the solver.py:142-222 loop body on the current buffers.
// Returns false if a non-finite residual was met (SolverNumericsError).
struct LoopState {
  double res_w, res_v, theta;
  Decomp dw, dv, dt;
  EgPipeline* pipe = nullptr;  // when set, v comes from the pipeline (slot vj)
  int vj = 0;
  EgSlot* vslot = nullptr;     // slot of the current v (for EG acceptance)
};

static bool loop_body(Problem& p, const SolverCfg& cfg, LoopState& s, int k, IterRecord& rec, IterCallback cb,
                      void* user, HostProbe* hp) {
  if (canary_check_all(("before iteration " + std::to_string(k)).c_str()) > 0)
    throw KotError(KOT_ECUDA, "device canary overwritten (KOT_CANARY)");
  Bufs& b = p.bufs();
  const int n = p.n;
  const long nn = (long)n * n;
  const auto t_it = clk::now();
  ProfScope ps("ssn_iteration", p.st);
  double eg_ms = 0.0, resid_ms = 0.0;
  // EG safeguard chain (eg.py:34-41 + residual at v) on the auxiliary stream,
  // concurrently with the Newton chain below: the two only meet at acceptance
  // (solver.py:186-192), so the arithmetic is unchanged.
  const bool do_eg = (k % cfg.safeguard_every == 0);
  std::exception_ptr eg_err = nullptr;
  double eg_resid_ms = 0.0;
  std::thread eg_thread;
  if (do_eg && !s.pipe) {
    Problem& a = p.aux();
    eg_thread = std::thread([&]() {
      try {
        gemm_cta_cap() = bg_gemm_ctas();
        background_thread() = true;
        KOT_CUDA(cudaSetDevice(a.device));
        auto t0 = clk::now();
        eg_step(a, b.gv, b.Xv, cfg.eg_stepsize, b.gv, b.Xv);
        KOT_CUDA(cudaStreamSynchronize(a.st));
        eg_ms = ms_since(t0);
        t0 = clk::now();
        s.res_v = residual_parts(a, b.gv, b.Xv, b.r1v, b.r2v, s.dv);
        eg_resid_ms = ms_since(t0);
      } catch (...) {
        eg_err = std::current_exception();
      }
    });
  }
  auto t0 = clk::now();
  NewtonOut st{};
  double mu = 0.0, res_t = 0.0;
  std::exception_ptr nt_err = nullptr;
  double newton_ms = 0.0;
  try {
    kot_require(s.res_w > 0.0, KOT_EINVAL, "context requires a nonzero residual");
    mu = s.theta * s.res_w;
    kot_require(mu > 0.0, KOT_EINVAL, "regularization mu must be positive");
    st = newton_direction(p, b.r1w, b.r2w, s.res_w, s.dw, mu, cfg, b.dg, b.dX);
    KOT_CUDA(cudaStreamSynchronize(p.st));
    newton_ms = ms_since(t0);
    prof_host("host.newton", newton_ms);
    axpby(p, n, 1.0, b.gw, 1.0, b.dg, b.gt);
    axpby(p, nn, 1.0, b.Xw, 1.0, b.dX, b.Xt);
    t0 = clk::now();
    res_t = residual_parts(p, b.gt, b.Xt, b.r1t, b.r2t, s.dt);
    resid_ms += ms_since(t0);
    prof_host("host.trial_resid", resid_ms);
    newton_resolve(p, s.res_w, cfg, st);
  } catch (...) {
    nt_err = std::current_exception();
  }
  if (eg_thread.joinable()) eg_thread.join();
  if (do_eg && s.pipe) {
    const auto tw = clk::now();
    EgSlot& sl = s.pipe->acquire(++s.vj);
    prof_host("host.eg_wait", ms_since(tw));
    if (sl.err) eg_err = sl.err;
    s.vslot = &sl;
    s.res_v = sl.res;
    s.dv = Decomp{sl.P, sl.vals, sl.k};
    eg_ms = sl.eg_ms;
    eg_resid_ms = sl.resid_ms;
  }
  if (eg_err) std::rethrow_exception(eg_err);
  if (nt_err) std::rethrow_exception(nt_err);
  resid_ms += eg_resid_ms;
  if (do_eg && !std::isfinite(s.res_v)) return false;
  if (!std::isfinite(res_t)) return false;
  if (cb) {
    hp->wg.resize(n);
    hp->wx.resize(nn);
    hp->rg.resize(n);
    hp->rx.resize(nn);
    hp->dg.resize(n);
    hp->dx.resize(nn);
    KOT_CUDA(cudaMemcpyAsync(hp->wg.data(), b.gw, sizeof(double) * n, cudaMemcpyDeviceToHost, p.st));
    KOT_CUDA(cudaMemcpyAsync(hp->wx.data(), b.Xw, sizeof(double) * nn, cudaMemcpyDeviceToHost, p.st));
    KOT_CUDA(cudaMemcpyAsync(hp->rg.data(), b.r1w, sizeof(double) * n, cudaMemcpyDeviceToHost, p.st));
    KOT_CUDA(cudaMemcpyAsync(hp->rx.data(), b.r2w, sizeof(double) * nn, cudaMemcpyDeviceToHost, p.st));
    KOT_CUDA(cudaMemcpyAsync(hp->dg.data(), b.dg, sizeof(double) * n, cudaMemcpyDeviceToHost, p.st));
    KOT_CUDA(cudaMemcpyAsync(hp->dx.data(), b.dX, sizeof(double) * nn, cudaMemcpyDeviceToHost, p.st));
    KOT_CUDA(cudaStreamSynchronize(p.st));
    if (cb(user, k, hp->wg.data(), hp->wx.data(), hp->rg.data(), hp->rx.data(), mu, s.theta, hp->dg.data(),
           hp->dx.data(), st.met) != 0)
      throw KotError(KOT_ECALLBACK, "on_iteration observer raised");
  }
  // damping update from the trial point, whether or not it is kept (solver.py:224-226)
  dev_reduce(p, b.r1t, b.dg, n, 0, false);
  dev_reduce(p, b.r2t, b.dX, nn, 1, false);
  dev_reduce(p, b.dg, nullptr, n, 2, true);
  dev_reduce(p, b.dX, nullptr, nn, 3, true);
  fetch(p, 4);
  const double rho = -(p.hsc[0] + p.hsc[1]);
  const double dwn = p.hsc[2] + p.hsc[3];
  const double theta_next = theta_update(s.theta, rho, dwn * dwn, cfg);
  int acc_ssn;
  if (res_t <= s.res_v) {
    acc_ssn = 1;
    std::swap(b.gw, b.gt);
    std::swap(b.Xw, b.Xt);
    std::swap(b.r1w, b.r1t);
    std::swap(b.r2w, b.r2t);
    std::swap(s.dw, s.dt);
    s.res_w = res_t;
  } else {
    acc_ssn = 0;
    if (s.pipe) {  // w ← v.copy() from the pipeline slot of the current v
      EgSlot& sl = *s.vslot;
      KOT_CUDA(cudaMemcpyAsync(b.gw, sl.g, sizeof(double) * n, cudaMemcpyDeviceToDevice, p.st));
      KOT_CUDA(cudaMemcpyAsync(b.Xw, sl.X, sizeof(double) * nn, cudaMemcpyDeviceToDevice, p.st));
      if (sl.alpha_only) {  // full decomposition at v for the next Newton step
        (void)residual_parts(p, b.gw, b.Xw, b.r1w, b.r2w, s.dw);
      } else {
        KOT_CUDA(cudaMemcpyAsync(b.r1w, sl.r1, sizeof(double) * n, cudaMemcpyDeviceToDevice, p.st));
        KOT_CUDA(cudaMemcpyAsync(b.r2w, sl.r2, sizeof(double) * nn, cudaMemcpyDeviceToDevice, p.st));
        KOT_CUDA(cudaMemcpyAsync(s.dw.P, sl.P, sizeof(double) * nn, cudaMemcpyDeviceToDevice, p.st));
        KOT_CUDA(cudaMemcpyAsync(s.dw.vals, sl.vals, sizeof(double) * n, cudaMemcpyDeviceToDevice, p.st));
        s.dw.k = sl.k;
      }
    } else {
      copy_state(p, b, s.dw, s.dv);
    }
    s.res_w = s.res_v;
  }
  rec.iteration = k;
  rec.res_accepted = s.res_w;
  rec.res_ssn = res_t;
  rec.res_eg = s.res_v;
  rec.accepted_ssn = acc_ssn;
  rec.theta = s.theta;
  rec.mu = mu;
  rec.cg_iters = st.cg_iters;
  rec.criterion_met = st.met;
  rec.crit_lhs = st.lhs;
  rec.crit_rhs = st.rhs;
  rec.eg_ms = eg_ms;
  rec.newton_ms = newton_ms;
  rec.cg_ms = st.cg_ms;
  rec.resid_ms = resid_ms;
  KOT_CUDA(cudaStreamSynchronize(p.st));
  rec.step_ms = ms_since(t_it);
  rec.n_pos = s.dw.k;
  rec.attempts = st.attempts;
  s.theta = theta_next;
  return true;
}

static void init_state(Problem& p, LoopState& s) {
  Bufs& b = p.bufs();
  const int n = p.n;
  const long nn = (long)n * n;
  s.dw = Decomp{b.Pw, b.valw, 0};
  s.dv = Decomp{b.Pv, b.valv, 0};
  s.dt = Decomp{b.Pt, b.valt, 0};
  for (double* v : {b.gw, b.gv}) KOT_CUDA(cudaMemsetAsync(v, 0, sizeof(double) * n, p.st));
  for (double* m : {b.Xw, b.Xv}) KOT_CUDA(cudaMemsetAsync(m, 0, sizeof(double) * nn, p.st));
}

SolveResult solve(Problem& p, const SolverCfg& cfg, IterCallback cb, void* user, double* gamma_out, double* x_out,
                  IterRecord* trace, int trace_cap, bool pure_eg) {
  kot_require(cfg.residual_tol > 0.0, KOT_EINVAL, "residual_tol must be positive");
  kot_require(cfg.max_iter >= 1, KOT_EINVAL, "max_iter must be >= 1");
  kot_require(cfg.safeguard_every >= 1, KOT_EINVAL, "safeguard_every must be >= 1");
  kot_require(cfg.eg_stepsize > 0.0, KOT_EINVAL, "stepsize must be positive");
  const auto t_start = clk::now();
  Bufs& b = p.bufs();
  const int n = p.n;
  const long nn = (long)n * n;
  LoopState s;
  init_state(p, s);
  SolveResult out{KOT_OK, 0, 0, 0.0, NAN, 0.0};
  HostProbe hp;
  prof_host("solve.setup", ms_since(t_start));
  // initial residual at the zero pair (solver.py:129-139)
  const auto t_res0 = clk::now();
  double res0 = pure_eg ? residual_parts_origin(p, b.gv, b.Xv, b.r1v, b.r2v, s.dv)
                        : residual_parts_origin(p, b.gw, b.Xw, b.r1w, b.r2w, s.dw);
  prof_host("solve.res0", ms_since(t_res0));
  s.res_w = s.res_v = res0;
  s.theta = cfg.theta0;
  int k = 0;
  bool conv = res0 <= cfg.residual_tol;
  bool finite = std::isfinite(res0);
  std::unique_ptr<EgPipeline> pipe;
  static const bool no_pipe = [] {  // diagnostic: EG chain per iteration on a helper thread
    const char* e = std::getenv("KOT_NO_PIPE");
    return e && std::atoi(e) > 0;
  }();
  if (!pure_eg && finite && !conv && !no_pipe) {
    const auto t_pipe = clk::now();
    pipe.reset(new EgPipeline(p, cfg.eg_stepsize));
    s.pipe = pipe.get();
    prof_host("solve.pipe_start", ms_since(t_pipe));
  }
  while (finite && !conv && k < cfg.max_iter) {
    IterRecord rec{};
    if (pure_eg) {
      const auto t_it = clk::now();
      auto t0 = clk::now();
      eg_step(p, b.gv, b.Xv, cfg.eg_stepsize, b.gv, b.Xv);
      KOT_CUDA(cudaStreamSynchronize(p.st));
      const double eg_ms = ms_since(t0);
      t0 = clk::now();
      s.res_v = residual_parts(p, b.gv, b.Xv, b.r1v, b.r2v, s.dv);
      const double resid_ms = ms_since(t0);
      if (!std::isfinite(s.res_v)) {
        finite = false;
        break;
      }
      rec = IterRecord{k, s.res_v, NAN, s.res_v, 0, NAN, NAN, 0, 0, NAN, NAN, eg_ms, 0.0, 0.0, resid_ms,
                       ms_since(t_it), s.dv.k, 0};
      s.res_w = s.res_v;
    } else if (!loop_body(p, cfg, s, k, rec, cb, user, &hp)) {
      finite = false;
      break;
    }
    if (trace && k < trace_cap) trace[k] = rec;
    ++k;
    conv = s.res_w <= cfg.residual_tol;
  }
  out.iterations = k;
  out.converged = conv ? 1 : 0;
  out.residual_norm = s.res_w;
  if (!finite) {
    out.status = KOT_ENUMERICS;
    return out;
  }
  const auto t_fin = clk::now();
  const double* gfin = pure_eg ? b.gv : b.gw;
  const double* xfin = pure_eg ? b.Xv : b.Xw;
  if (p.has_embed) out.ot_estimate = (p.q_sq - dev_dot(p, gfin, p.embed, n)) / (2.0 * p.l2);
  if (gamma_out) KOT_CUDA(cudaMemcpyAsync(gamma_out, gfin, sizeof(double) * n, cudaMemcpyDeviceToHost, p.st));
  if (x_out) KOT_CUDA(cudaMemcpyAsync(x_out, xfin, sizeof(double) * nn, cudaMemcpyDeviceToHost, p.st));
  KOT_CUDA(cudaStreamSynchronize(p.st));
  prof_host("solve.download", ms_since(t_fin));
  out.total_ms = ms_since(t_start);
  return out;
}

// ---------------------------------------------------------------- sessions
// A solve whose iterations are driven in chunks by the caller (bench.py times
// W warm-up + K measured iterations of one continuous trajectory).
struct Session {
  Problem* p;
  SolverCfg cfg;
  LoopState s;
  HostProbe hp;
  int k = 0;
  bool conv = false;
  std::unique_ptr<EgPipeline> pipe;
};

Session* session_begin(Problem& p, const SolverCfg& cfg) {
  kot_require(cfg.residual_tol > 0.0 && cfg.max_iter >= 1 && cfg.safeguard_every >= 1 && cfg.eg_stepsize > 0.0,
              KOT_EINVAL, "invalid solver configuration");
  Bufs& b = p.bufs();
  auto* se = new Session();
  se->p = &p;
  se->cfg = cfg;
  init_state(p, se->s);
  const double res0 = residual_parts_origin(p, b.gw, b.Xw, b.r1w, b.r2w, se->s.dw);
  se->s.res_w = se->s.res_v = res0;
  se->s.theta = cfg.theta0;
  se->conv = res0 <= cfg.residual_tol;
  if (!std::isfinite(res0)) {
    delete se;
    throw KotError(KOT_ENUMERICS, "non-finite residual in solver iterate");
  }
  se->pipe.reset(new EgPipeline(p, cfg.eg_stepsize));
  se->s.pipe = se->pipe.get();
  return se;
}

int session_step(Session& se, int iters, IterRecord* recs) {
  int done = 0;
  for (int i = 0; i < iters && !se.conv && se.k < se.cfg.max_iter; ++i) {
    IterRecord rec{};
    if (!loop_body(*se.p, se.cfg, se.s, se.k, rec, nullptr, nullptr, &se.hp))
      throw KotError(KOT_ENUMERICS, "non-finite residual in solver iterate");
    if (recs) recs[done] = rec;
    ++done;
    ++se.k;
    se.conv = se.s.res_w <= se.cfg.residual_tol;
  }
  return done;
}

void session_result(Session& se, double* gamma, double* x, SolveResult& out) {
  Problem& p = *se.p;
  Bufs& b = p.bufs();
  out.status = KOT_OK;
  out.converged = se.conv ? 1 : 0;
  out.iterations = se.k;
  out.residual_norm = se.s.res_w;
  out.ot_estimate = p.has_embed ? (p.q_sq - dev_dot(p, b.gw, p.embed, p.n)) / (2.0 * p.l2) : NAN;
  if (gamma) KOT_CUDA(cudaMemcpyAsync(gamma, b.gw, sizeof(double) * p.n, cudaMemcpyDeviceToHost, p.st));
  if (x) KOT_CUDA(cudaMemcpyAsync(x, b.Xw, sizeof(double) * (long)p.n * p.n, cudaMemcpyDeviceToHost, p.st));
  KOT_CUDA(cudaStreamSynchronize(p.st));
  out.total_ms = 0.0;
}

// Loop state between two iterations: w, the current safeguard iterate v (the slot consumed by the
// last iteration; (0, 0) before the first) and θ — the oracle's State(w, v, θ) for a CPU replay.
void session_state(Session& se, double* wg, double* wx, double* vg, double* vx, double* theta) {
  Problem& p = *se.p;
  Bufs& b = p.bufs();
  const int n = p.n;
  const long nn = (long)n * n;
  if (wg) KOT_CUDA(cudaMemcpyAsync(wg, b.gw, sizeof(double) * n, cudaMemcpyDeviceToHost, p.st));
  if (wx) KOT_CUDA(cudaMemcpyAsync(wx, b.Xw, sizeof(double) * nn, cudaMemcpyDeviceToHost, p.st));
  const EgSlot* v = se.s.vslot;
  if (v) {
    if (vg) KOT_CUDA(cudaMemcpyAsync(vg, v->g, sizeof(double) * n, cudaMemcpyDeviceToHost, p.st));
    if (vx) KOT_CUDA(cudaMemcpyAsync(vx, v->X, sizeof(double) * nn, cudaMemcpyDeviceToHost, p.st));
  } else {
    if (vg) std::fill(vg, vg + n, 0.0);
    if (vx) std::fill(vx, vx + nn, 0.0);
  }
  KOT_CUDA(cudaStreamSynchronize(p.st));
  if (theta) *theta = se.s.theta;
}

void session_end(Session* se) { delete se; }

IterRecord iterate_once(Problem& p, const SolverCfg& cfg, const ReplayIn& in, ReplayOut& out) {
  Bufs& b = p.bufs();
  const int n = p.n;
  const long nn = (long)n * n;
  LoopState s;
  init_state(p, s);
  KOT_CUDA(cudaMemcpyAsync(b.gw, in.wg, sizeof(double) * n, cudaMemcpyHostToDevice, p.st));
  KOT_CUDA(cudaMemcpyAsync(b.Xw, in.wx, sizeof(double) * nn, cudaMemcpyHostToDevice, p.st));
  KOT_CUDA(cudaMemcpyAsync(b.gv, in.vg, sizeof(double) * n, cudaMemcpyHostToDevice, p.st));
  KOT_CUDA(cudaMemcpyAsync(b.Xv, in.vx, sizeof(double) * nn, cudaMemcpyHostToDevice, p.st));
  s.res_w = residual_parts(p, b.gw, b.Xw, b.r1w, b.r2w, s.dw);
  s.res_v = s.res_w;
  if (in.k % cfg.safeguard_every != 0) s.res_v = residual_parts(p, b.gv, b.Xv, b.r1v, b.r2v, s.dv);
  s.theta = in.theta;
  IterRecord rec{};
  HostProbe hp;
  if (!loop_body(p, cfg, s, in.k, rec, nullptr, nullptr, &hp))
    throw KotError(KOT_ENUMERICS, "non-finite residual in solver iterate");
  KOT_CUDA(cudaMemcpyAsync(out.wg, b.gw, sizeof(double) * n, cudaMemcpyDeviceToHost, p.st));
  KOT_CUDA(cudaMemcpyAsync(out.wx, b.Xw, sizeof(double) * nn, cudaMemcpyDeviceToHost, p.st));
  KOT_CUDA(cudaMemcpyAsync(out.vg, b.gv, sizeof(double) * n, cudaMemcpyDeviceToHost, p.st));
  KOT_CUDA(cudaMemcpyAsync(out.vx, b.Xv, sizeof(double) * nn, cudaMemcpyDeviceToHost, p.st));
  KOT_CUDA(cudaStreamSynchronize(p.st));
  out.theta = s.theta;
  return rec;
}

}  // namespace kot

namespace kot {
void set_panel_grid_cap(int cap);
}
extern "C" int kot_set_panel_grid_cap(int cap) {  // 0: default (all SMs)
  kot::set_panel_grid_cap(cap);
  return 0;
}

extern "C" int kot_debug_gemm_tma(int mode) {  // test hook: 1 TMA-staged GEMM core (default), 0 cp.async core
  kot::gemm_tma_mode().store(mode);
  return 0;
}

extern "C" int kot_debug_cg_batch(int batch) {  // test hook: CG iterations per host check (≥ 1)
  kot::g_cg_batch = batch >= 1 ? batch : 1;
  return 0;
}

extern "C" int kot_debug_eg_parallel(int on) {  // test hook: EG projections side by side (1) or in sequence
  kot::g_eg_parallel = on ? 1 : 0;
  return 0;
}
