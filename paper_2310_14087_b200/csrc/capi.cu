// extern "C" boundary of libkotgpu (declared in include/kotgpu.h).
// Every entry point maps kot::KotError onto a status code and stores the
// message in a thread-local buffer (kot_last_error).
#include <cstring>
#include <string>
#include <vector>

#include "../../include/kotgpu.h"
#include "ssn.cuh"

namespace kot {
std::atomic<long long> g_kot_launches{0};
}

struct kot_problem {
  std::unique_ptr<kot::Problem> p;
};

static thread_local std::string g_last_error;

template <class F>
static int guarded(F&& f) {
  try {
    f();
    return kot::KOT_OK;
  } catch (const kot::KotError& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return kot::KOT_ECUDA;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return kot::KOT_ECUDA;
  }
}

static kot::SolverCfg to_cfg(const kot_solver_cfg* c) {
  kot::SolverCfg s;
  static_assert(sizeof(kot::SolverCfg) == sizeof(kot_solver_cfg), "cfg layout");
  std::memcpy(&s, c, sizeof(s));
  return s;
}

static void check_cfg(const kot::SolverCfg& c) {
  using kot::kot_require;
  kot_require(c.tau > 0.0 && c.tau < 1.0 && c.kappa > 0.0 && c.kappa < 1.0, kot::KOT_EINVAL,
              "tau and kappa must lie in (0, 1)");
  kot_require(c.alpha1 > 0.0 && c.alpha1 <= c.alpha2, kot::KOT_EINVAL, "need 0 < alpha1 <= alpha2");
  kot_require(c.beta0 < 1.0 && 1.0 < c.beta2, kot::KOT_EINVAL, "need beta0 < 1 < beta2");
  kot_require(c.theta_min > 0.0 && c.theta_min <= c.theta_max, kot::KOT_EINVAL, "need 0 < theta_min <= theta_max");
  kot_require(c.cg_max >= 1 && c.cg_restarts >= 0, kot::KOT_EINVAL, "invalid CG budget");
}

static_assert(sizeof(kot::IterRecord) == sizeof(kot_iter_record), "record layout");

extern "C" {

const char* kot_last_error(void) { return g_last_error.c_str(); }

long long kot_launch_count(void) { return kot::g_kot_launches.load(); }

int kot_reserve(int device, unsigned long long bytes) {
  return guarded([&] {
    KOT_CUDA(cudaSetDevice(device));
    kot::dev_reserve((size_t)bytes);
  });
}

int kot_problem_create(const double* q, const double* z, double q_sq, const double* r_upper, const double* embed,
                       int l, double lambda1, double lambda2, double jitter, int device, kot_problem** out) {
  return guarded([&] {
    auto h = new kot_problem();
    try {
      h->p = kot::problem_from_host(q, z, q_sq, r_upper, embed, l, lambda1, lambda2, jitter, device);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int kot_assemble(const double* xs, int n_mu, const double* ys, int n_nu, const double* xt, const double* yt, int l,
                 int d, double bw_x, double bw_y, double bw_xy, double lambda1, double lambda2, int device,
                 kot_problem** out) {
  return guarded([&] {
    auto h = new kot_problem();
    try {
      h->p = kot::problem_assemble(xs, n_mu, ys, n_nu, xt, yt, l, d, bw_x, bw_y, bw_xy, lambda1, lambda2, device);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int kot_problem_info(const kot_problem* h, int* l, double* q_sq, double* jitter, double* lambda1, double* lambda2,
                     int* has_embed) {
  return guarded([&] {
    const kot::Problem& p = *h->p;
    if (l) *l = p.n;
    if (q_sq) *q_sq = p.q_sq;
    if (jitter) *jitter = p.jitter;
    if (lambda1) *lambda1 = p.l1;
    if (lambda2) *lambda2 = p.l2;
    if (has_embed) *has_embed = p.has_embed ? 1 : 0;
  });
}

int kot_problem_download(kot_problem* h, double* q, double* z, double* r_upper, double* embed, double* kmat) {
  return guarded([&] {
    kot::Problem& p = *h->p;
    KOT_CUDA(cudaSetDevice(p.device));
    const long nn = (long)p.n * p.n;
    if (q) KOT_CUDA(cudaMemcpyAsync(q, p.Q, nn * 8, cudaMemcpyDeviceToHost, p.st));
    if (z) KOT_CUDA(cudaMemcpyAsync(z, p.z, p.n * 8, cudaMemcpyDeviceToHost, p.st));
    if (r_upper) KOT_CUDA(cudaMemcpyAsync(r_upper, p.R, nn * 8, cudaMemcpyDeviceToHost, p.st));
    if (embed && p.has_embed) KOT_CUDA(cudaMemcpyAsync(embed, p.embed, p.n * 8, cudaMemcpyDeviceToHost, p.st));
    if (kmat) {
      kot::kot_require(p.Kmat != nullptr, kot::KOT_EINVAL, "pair Gram only available for assembled problems");
      KOT_CUDA(cudaMemcpyAsync(kmat, p.Kmat, nn * 8, cudaMemcpyDeviceToHost, p.st));
    }
    KOT_CUDA(cudaStreamSynchronize(p.st));
  });
}

void kot_problem_destroy(kot_problem* h) {
  if (!h) return;
  try {
    kot::problem_release(std::move(h->p));  // idle problems are pooled for reuse (bounded)
  } catch (...) {
  }
  delete h;
}

int kot_solve(kot_problem* h, const kot_solver_cfg* cfg, kot_iter_cb cb, void* user, double* gamma_out,
              double* x_out, kot_iter_record* trace, int trace_cap, kot_report* out) {
  int status = guarded([&] {
    kot::Problem& p = *h->p;
    KOT_CUDA(cudaSetDevice(p.device));
    const kot::SolverCfg c = to_cfg(cfg);
    check_cfg(c);
    const kot::SolveResult r = kot::solve(p, c, (kot::IterCallback)cb, user, gamma_out, x_out,
                                          reinterpret_cast<kot::IterRecord*>(trace), trace_cap, false);
    out->converged = r.converged;
    out->iterations = r.iterations;
    out->residual_norm = r.residual_norm;
    out->ot_estimate = r.ot_estimate;
    out->total_ms = r.total_ms;
    if (r.status != kot::KOT_OK) throw kot::KotError(r.status, "non-finite residual in solver iterate");
  });
  return status;
}

int kot_solve_pure_eg(kot_problem* h, const kot_solver_cfg* cfg, double* gamma_out, double* x_out,
                      kot_iter_record* trace, int trace_cap, kot_report* out) {
  return guarded([&] {
    kot::Problem& p = *h->p;
    KOT_CUDA(cudaSetDevice(p.device));
    const kot::SolverCfg c = to_cfg(cfg);
    const kot::SolveResult r = kot::solve(p, c, nullptr, nullptr, gamma_out, x_out,
                                          reinterpret_cast<kot::IterRecord*>(trace), trace_cap, true);
    out->converged = r.converged;
    out->iterations = r.iterations;
    out->residual_norm = r.residual_norm;
    out->ot_estimate = r.ot_estimate;
    out->total_ms = r.total_ms;
    if (r.status != kot::KOT_OK) throw kot::KotError(r.status, "non-finite residual in solver iterate");
  });
}

int kot_iterate(kot_problem* h, const kot_solver_cfg* cfg, const double* w_gamma, const double* w_x,
                const double* v_gamma, const double* v_x, double theta, int k, double* w_gamma_out, double* w_x_out,
                double* v_gamma_out, double* v_x_out, double* theta_out, kot_iter_record* rec) {
  return guarded([&] {
    kot::Problem& p = *h->p;
    KOT_CUDA(cudaSetDevice(p.device));
    const kot::SolverCfg c = to_cfg(cfg);
    check_cfg(c);
    kot::ReplayIn in{w_gamma, w_x, v_gamma, v_x, theta, k};
    kot::ReplayOut o{w_gamma_out, w_x_out, v_gamma_out, v_x_out, 0.0};
    const kot::IterRecord r = kot::iterate_once(p, c, in, o);
    *theta_out = o.theta;
    if (rec) std::memcpy(rec, &r, sizeof(r));
  });
}

struct kot_session {
  kot::Session* s;
  kot_problem* h;
};

int kot_session_begin(kot_problem* h, const kot_solver_cfg* cfg, kot_session** out) {
  return guarded([&] {
    kot::Problem& p = *h->p;
    KOT_CUDA(cudaSetDevice(p.device));
    const kot::SolverCfg c = to_cfg(cfg);
    check_cfg(c);
    *out = new kot_session{kot::session_begin(p, c), h};
  });
}

int kot_session_step(kot_session* s, int iters, kot_iter_record* recs, int* done) {
  return guarded([&] {
    KOT_CUDA(cudaSetDevice(s->h->p->device));
    *done = kot::session_step(*s->s, iters, reinterpret_cast<kot::IterRecord*>(recs));
  });
}

int kot_session_result(kot_session* s, double* gamma_out, double* x_out, kot_report* out) {
  return guarded([&] {
    KOT_CUDA(cudaSetDevice(s->h->p->device));
    kot::SolveResult r{};
    kot::session_result(*s->s, gamma_out, x_out, r);
    out->converged = r.converged;
    out->iterations = r.iterations;
    out->residual_norm = r.residual_norm;
    out->ot_estimate = r.ot_estimate;
    out->total_ms = r.total_ms;
  });
}

int kot_session_state(kot_session* s, double* w_gamma, double* w_x, double* v_gamma, double* v_x, double* theta) {
  return guarded([&] {
    KOT_CUDA(cudaSetDevice(s->h->p->device));
    kot::session_state(*s->s, w_gamma, w_x, v_gamma, v_x, theta);
  });
}

void kot_session_end(kot_session* s) {
  if (!s) return;
  kot::session_end(s->s);
  delete s;
}

void* kot_problem_stream(kot_problem* h) { return (void*)h->p->st; }

int kot_nccl_unique_id(char* out128) {
  return guarded([&] { kot::nccl_unique_id(out128); });
}

int kot_problem_shard(kot_problem* h, const char* id128, int rank, int world) {
  return guarded([&] {
    if (world <= 1)
      kot::problem_unshard(*h->p);
    else if (id128 == nullptr)
      kot::problem_shard_emulate(*h->p, world);
    else
      kot::problem_shard(*h->p, id128, rank, world);
  });
}

int kot_problem_shard_host(kot_problem* h, kot_comm_fn fn, void* user, int rank, int world) {
  return guarded([&] {
    if (world <= 1)
      kot::problem_unshard(*h->p);
    else
      kot::problem_shard_host(*h->p, fn, user, rank, world);
  });
}

int kot_problem_shard_info(const kot_problem* h, int* rank, int* world, int* row0, int* row1) {
  return guarded([&] {
    const kot::Problem& p = *h->p;
    if (rank) *rank = p.shard_rank;
    if (world) *world = p.shard_world;
    if (row0) *row0 = p.shard_world > 1 ? p.row0 : 0;
    if (row1) *row1 = p.shard_world > 1 ? p.row1 : p.n;
  });
}

// ------------------------------------------------------------ operators

namespace {
struct DevBuf {
  double* p = nullptr;
  explicit DevBuf(long count) : p(static_cast<double*>(kot::dev_alloc(std::max(count, 1L) * sizeof(double)))) {}
  ~DevBuf() { kot::dev_free(p); }
};
}  // namespace

static void up(kot::Problem& p, double* d, const double* h, long count) {
  KOT_CUDA(cudaMemcpyAsync(d, h, count * 8, cudaMemcpyHostToDevice, p.st));
}
static void down(kot::Problem& p, double* h, const double* d, long count) {
  KOT_CUDA(cudaMemcpyAsync(h, d, count * 8, cudaMemcpyDeviceToHost, p.st));
}

// Upload a host SpectralDecomp into p's (Pw, valw).
static kot::Decomp up_decomp(kot::Problem& p, const double* vecs, const double* vals, int n_pos) {
  kot::kot_require(n_pos >= 0 && n_pos <= p.n, kot::KOT_EINVAL, "invalid decomposition");
  kot::Bufs& b = p.bufs();
  up(p, b.Pw, vecs, (long)p.n * p.n);
  up(p, b.valw, vals, p.n);
  return kot::Decomp{b.Pw, b.valw, n_pos};
}

// A scratch problem for the matrix-only entry points (no instance data needed).
static std::unique_ptr<kot::Problem> scratch_problem(int n, int device) {
  std::vector<double> zeros(1, 0.0);
  std::vector<double> q((long)n * n, 0.0), r((long)n * n, 0.0), z(n, 0.0);
  for (int i = 0; i < n; ++i) q[(long)i * n + i] = r[(long)i * n + i] = 1.0;
  return kot::problem_from_host(q.data(), z.data(), 0.0, r.data(), nullptr, n, 1.0, 1.0, 0.0, device);
}

int kot_gram(const double* pts, int n, int d, double bandwidth_sq, int device, double* out) {
  return guarded([&] {
    kot::kot_require(bandwidth_sq > 0.0, kot::KOT_EINVAL, "bandwidth_sq must be positive");
    KOT_CUDA(cudaSetDevice(device));
    cudaStream_t st;
    KOT_CUDA(cudaStreamCreate(&st));
    DevBuf dp((long)n * d), dout((long)n * n);
    KOT_CUDA(cudaMemcpyAsync(dp.p, pts, (long)n * d * 8, cudaMemcpyHostToDevice, st));
    kot::gram_square(dp.p, dp.p, n, d, bandwidth_sq, bandwidth_sq, 1, false, dout.p, st);
    KOT_CUDA(cudaMemcpyAsync(out, dout.p, (long)n * n * 8, cudaMemcpyDeviceToHost, st));
    KOT_CUDA(cudaStreamSynchronize(st));
    cudaStreamDestroy(st);
  });
}

int kot_gram_rect(const double* a, int m, const double* b, int p, int d, double bandwidth_sq, int device,
                  double* out) {
  return guarded([&] {
    kot::kot_require(bandwidth_sq > 0.0, kot::KOT_EINVAL, "bandwidth_sq must be positive");
    kot::kot_require(m >= 0 && p >= 0 && d >= 1, kot::KOT_EINVAL, "invalid shapes");
    KOT_CUDA(cudaSetDevice(device));
    if (m == 0 || p == 0) return;
    cudaStream_t st;
    KOT_CUDA(cudaStreamCreate(&st));
    DevBuf da((long)m * d), db((long)p * d), dout((long)m * p);
    KOT_CUDA(cudaMemcpyAsync(da.p, a, (long)m * d * 8, cudaMemcpyHostToDevice, st));
    KOT_CUDA(cudaMemcpyAsync(db.p, b, (long)p * d * 8, cudaMemcpyHostToDevice, st));
    kot::gram_rect(da.p, m, db.p, p, d, bandwidth_sq, dout.p, st);
    KOT_CUDA(cudaMemcpyAsync(out, dout.p, (long)m * p * 8, cudaMemcpyDeviceToHost, st));
    KOT_CUDA(cudaStreamSynchronize(st));
    cudaStreamDestroy(st);
  });
}

int kot_sobol_points(const unsigned long long* dirnums, int dim, int bits, long first, int count,
                     const double* lower, const double* upper, int device, double* out) {
  return guarded([&] {
    kot::kot_require(dim >= 1 && bits >= 1 && bits <= 64 && count >= 0 && first >= 0, kot::KOT_EINVAL,
                     "invalid Sobol request");
    KOT_CUDA(cudaSetDevice(device));
    if (count == 0) return;
    cudaStream_t st;
    KOT_CUDA(cudaStreamCreate(&st));
    DevBuf dv((long)dim * bits), dlo(dim), dhi(dim), dout((long)count * dim);
    KOT_CUDA(cudaMemcpyAsync(dv.p, dirnums, 8L * dim * bits, cudaMemcpyHostToDevice, st));
    KOT_CUDA(cudaMemcpyAsync(dlo.p, lower, 8L * dim, cudaMemcpyHostToDevice, st));
    KOT_CUDA(cudaMemcpyAsync(dhi.p, upper, 8L * dim, cudaMemcpyHostToDevice, st));
    kot::sobol_points_device(reinterpret_cast<const unsigned long long*>(dv.p), dim, bits, first, count, dlo.p, dhi.p,
                             dout.p, st);
    KOT_CUDA(cudaMemcpyAsync(out, dout.p, 8L * count * dim, cudaMemcpyDeviceToHost, st));
    KOT_CUDA(cudaStreamSynchronize(st));
    cudaStreamDestroy(st);
  });
}

int kot_mean_embedding(const double* samples, int n, const double* queries, int m, int d, double bandwidth_sq,
                       int device, double* out) {
  return guarded([&] {
    kot::kot_require(bandwidth_sq > 0.0, kot::KOT_EINVAL, "bandwidth_sq must be positive");
    kot::kot_require(n >= 1, kot::KOT_EINVAL, "sample set is empty");
    KOT_CUDA(cudaSetDevice(device));
    if (m == 0) return;
    cudaStream_t st;
    KOT_CUDA(cudaStreamCreate(&st));
    DevBuf ds((long)n * d), dq((long)m * d), dout(m);
    KOT_CUDA(cudaMemcpyAsync(ds.p, samples, (long)n * d * 8, cudaMemcpyHostToDevice, st));
    KOT_CUDA(cudaMemcpyAsync(dq.p, queries, (long)m * d * 8, cudaMemcpyHostToDevice, st));
    kot::mean_embedding_device(ds.p, n, dq.p, m, d, bandwidth_sq, dout.p, st);
    KOT_CUDA(cudaMemcpyAsync(out, dout.p, (long)m * 8, cudaMemcpyDeviceToHost, st));
    KOT_CUDA(cudaStreamSynchronize(st));
    cudaStreamDestroy(st);
  });
}

int kot_embedding_norm_sq(const double* samples, int n, int d, double bandwidth_sq, int device, double* out) {
  return guarded([&] {
    kot::kot_require(bandwidth_sq > 0.0, kot::KOT_EINVAL, "bandwidth_sq must be positive");
    kot::kot_require(n >= 1, kot::KOT_EINVAL, "sample set is empty");
    KOT_CUDA(cudaSetDevice(device));
    cudaStream_t st;
    KOT_CUDA(cudaStreamCreate(&st));
    DevBuf ds((long)n * d), scratch(n + 1), dout(1);
    KOT_CUDA(cudaMemcpyAsync(ds.p, samples, (long)n * d * 8, cudaMemcpyHostToDevice, st));
    kot::embedding_norm_sq_device(ds.p, n, d, bandwidth_sq, scratch.p, dout.p, st);
    KOT_CUDA(cudaMemcpyAsync(out, dout.p, 8, cudaMemcpyDeviceToHost, st));
    KOT_CUDA(cudaStreamSynchronize(st));
    cudaStreamDestroy(st);
  });
}

int kot_evaluate_map(const double* xs, int n, const double* xt, const double* gamma, int l, const double* queries,
                     int m, int d, double bandwidth_sq, double lambda2, int device, double* u_out, double* t_out) {
  return guarded([&] {
    kot::kot_require(bandwidth_sq > 0.0 && lambda2 > 0.0, kot::KOT_EINVAL, "bandwidth_sq and lambda2 must be positive");
    kot::kot_require(n >= 1 && l >= 1 && m >= 0, kot::KOT_EINVAL, "empty sample or filling set");
    KOT_CUDA(cudaSetDevice(device));
    if (m == 0) return;
    cudaStream_t st;
    KOT_CUDA(cudaStreamCreate(&st));
    DevBuf dxs((long)n * d), dxt((long)l * d), dg(l), dq((long)m * d), du(m), dt((long)m * d);
    KOT_CUDA(cudaMemcpyAsync(dxs.p, xs, (long)n * d * 8, cudaMemcpyHostToDevice, st));
    KOT_CUDA(cudaMemcpyAsync(dxt.p, xt, (long)l * d * 8, cudaMemcpyHostToDevice, st));
    KOT_CUDA(cudaMemcpyAsync(dg.p, gamma, (long)l * 8, cudaMemcpyHostToDevice, st));
    KOT_CUDA(cudaMemcpyAsync(dq.p, queries, (long)m * d * 8, cudaMemcpyHostToDevice, st));
    kot::evaluate_map_device(dxs.p, n, dxt.p, dg.p, l, dq.p, m, d, bandwidth_sq, lambda2, du.p, dt.p, st);
    KOT_CUDA(cudaMemcpyAsync(u_out, du.p, (long)m * 8, cudaMemcpyDeviceToHost, st));
    KOT_CUDA(cudaMemcpyAsync(t_out, dt.p, (long)m * d * 8, cudaMemcpyDeviceToHost, st));
    KOT_CUDA(cudaStreamSynchronize(st));
    cudaStreamDestroy(st);
  });
}

int kot_cholesky_psd(const double* k, int n, int device, double* r_upper, double* jitter) {
  return guarded([&] {
    kot::kot_require(n >= 1, kot::KOT_EINVAL, "order must be >= 1");
    KOT_CUDA(cudaSetDevice(device));
    cudaStream_t st;
    KOT_CUDA(cudaStreamCreate(&st));
    DevBuf dk((long)n * n), dr((long)n * n), work((long)n * n + 8);
    int* flag;
    KOT_CUDA(cudaMalloc(&flag, sizeof(int)));
    KOT_CUDA(cudaMemcpyAsync(dk.p, k, (long)n * n * 8, cudaMemcpyHostToDevice, st));
    try {
      *jitter = kot::cholesky_psd_device(dk.p, n, dr.p, work.p, work.p + (long)n * n, flag, st);
    } catch (...) {
      cudaFree(flag);
      cudaStreamDestroy(st);
      throw;
    }
    KOT_CUDA(cudaMemcpyAsync(r_upper, dr.p, (long)n * n * 8, cudaMemcpyDeviceToHost, st));
    KOT_CUDA(cudaStreamSynchronize(st));
    cudaFree(flag);
    cudaStreamDestroy(st);
  });
}

int kot_sym_eig(const double* z, int n, int device, double* vecs, double* vals, int* n_pos) {
  return guarded([&] {
    auto p = scratch_problem(n, device);
    const long nn = (long)n * n;
    up(*p, p->M1, z, nn);
    kot::symmetrize(*p, p->M1, p->M2);  // sym(z), linalg.py:66
    kot::Decomp dc{p->M3, p->M4, 0};
    kot::eigh(*p, p->M2, dc);
    down(*p, vecs, dc.P, nn);
    down(*p, vals, dc.vals, n);
    KOT_CUDA(cudaStreamSynchronize(p->st));
    *n_pos = dc.k;
  });
}

int kot_debug_tridiag(const double* z, int n, int device, int stages, double* d_out, double* e_out) {
  return guarded([&] {
    auto p = scratch_problem(n, device);
    const long nn = (long)n * n;
    up(*p, p->M1, z, nn);
    kot::symmetrize(*p, p->M1, p->M2);
    kot::tridiag_device(p->M2, n, *p->eig, p->st, stages);
    down(*p, d_out, p->eig->d, n);
    down(*p, e_out, p->eig->e, n - 1);
    KOT_CUDA(cudaStreamSynchronize(p->st));
  });
}

int kot_proj_psd(const double* z, int n, int device, double* out) {
  return guarded([&] {
    auto p = scratch_problem(n, device);
    const long nn = (long)n * n;
    up(*p, p->M1, z, nn);
    kot::symmetrize(*p, p->M1, p->M2);
    kot::Decomp dc{p->M3, p->M4, 0};
    kot::eigh(*p, p->M2, dc);
    kot::proj(*p, dc, nullptr, p->M5);
    down(*p, out, p->M5, nn);
    KOT_CUDA(cudaStreamSynchronize(p->st));
  });
}

int kot_spectral_apply(const double* z, int n, int device, int mode, double mu, int path, const double* s,
                       double* out) {
  return guarded([&] {
    if (mode == 0) kot::kot_require(mu > 0.0, kot::KOT_EINVAL, "regularization mu must be positive");
    auto p = scratch_problem(n, device);
    kot::Bufs& b = p->bufs();
    const long nn = (long)n * n;
    up(*p, p->M1, z, nn);
    kot::symmetrize(*p, p->M1, p->M2);
    kot::Decomp dc{b.Pw, b.valw, 0};
    kot::eigh(*p, p->M2, dc);
    up(*p, b.Xw, s, nn);
    kot::spectral_filter(*p, dc, b.Xw, b.Xv, mu, mode, path);
    down(*p, out, b.Xv, nn);
    KOT_CUDA(cudaStreamSynchronize(p->st));
  });
}

int kot_spectral_apply_decomp(const double* vecs, const double* vals, int n, int n_pos, int device, int mode,
                              double mu, int path, const double* s, double* out) {
  return guarded([&] {
    kot::kot_require(n >= 1 && n_pos >= 0 && n_pos <= n, kot::KOT_EINVAL, "invalid decomposition");
    kot::kot_require(mode >= 0 && mode <= 2, kot::KOT_EINVAL, "invalid mode");
    if (mode == 0) kot::kot_require(mu > 0.0, kot::KOT_EINVAL, "regularization mu must be positive");
    auto p = scratch_problem(n, device);
    kot::Bufs& b = p->bufs();
    const long nn = (long)n * n;
    up(*p, b.Pw, vecs, nn);
    up(*p, b.valw, vals, n);
    const kot::Decomp dc{b.Pw, b.valw, n_pos};
    if (mode == 2) {
      if (n_pos == 0)
        KOT_CUDA(cudaMemsetAsync(b.Xv, 0, sizeof(double) * nn, p->st));
      else
        kot::proj(*p, dc, nullptr, b.Xv);
    } else {
      up(*p, b.Xw, s, nn);
      kot::spectral_filter(*p, dc, b.Xw, b.Xv, mu, mode, path);
    }
    down(*p, out, b.Xv, nn);
    KOT_CUDA(cudaStreamSynchronize(p->st));
  });
}

int kot_apply_jacobian(kot_problem* h, const double* vecs, const double* vals, int n_pos, double mu,
                       const double* dgamma, const double* dx, double* top, double* bottom) {
  return guarded([&] {
    kot::Problem& p = *h->p;
    const int n = p.n;
    kot::kot_require(n_pos >= 0 && n_pos <= n, kot::KOT_EINVAL, "invalid decomposition");
    KOT_CUDA(cudaSetDevice(p.device));
    kot::Bufs& b = p.bufs();
    const long nn = (long)n * n;
    const kot::Decomp dc = up_decomp(p, vecs, vals, n_pos);
    up(p, b.dg, dgamma, n);
    up(p, b.dX, dx, nn);
    KOT_CUDA(cudaMemsetAsync(b.e3, 0, sizeof(double) * n, p.st));
    KOT_CUDA(cudaMemsetAsync(b.Xv, 0, sizeof(double) * nn, p.st));
    // top = Qdγ/(2λ₂) + μdγ − Φ(dX);  bottom = M[Φ*(dγ) − dX] + (1+μ)dX   (problem.py:222-236)
    kot::phi_partials(p, b.dX);
    kot::finalize(p, kot::FIN_JTOP, b.dg, true, b.e3, mu, b.e1);
    kot::phi_adjoint_ex(p, b.dg, p.M1, 1.0, b.dX, -1.0, 0.0);
    kot::spectral_filter(p, dc, p.M1, p.M2, mu, 1);
    kot::jac_bottom(p, nn, p.M2, b.dX, mu, b.Xv, p.M1);
    down(p, top, b.e1, n);
    down(p, bottom, p.M1, nn);
    KOT_CUDA(cudaStreamSynchronize(p.st));
  });
}

int kot_cg_solve(kot_matvec_fn fn, void* user, const double* rhs, int n, double tol, int max_iter, int device,
                 double* x_out, int* iters, double* res) {
  return guarded([&] {
    kot::kot_require(fn != nullptr && n >= 1, kot::KOT_EINVAL, "invalid operator");
    kot::kot_require(max_iter >= 1, kot::KOT_EINVAL, "max_iter must be >= 1");
    auto p = scratch_problem(n, device);
    kot::Bufs& b = p->bufs();
    std::vector<double> hp(n), hap(n);
    up(*p, b.e1, rhs, n);
    const kot::CgResult r = kot::cg_solve_op(*p, b.e1, tol, max_iter, [&](const double* pv, double* ap) {
      down(*p, hp.data(), pv, n);
      KOT_CUDA(cudaStreamSynchronize(p->st));
      kot::kot_require(fn(user, hp.data(), hap.data()) == 0, kot::KOT_ECALLBACK, "matvec callback raised");
      up(*p, ap, hap.data(), n);
    }, b.e2);
    down(*p, x_out, b.e2, n);
    KOT_CUDA(cudaStreamSynchronize(p->st));
    *iters = r.iters;
    *res = r.res;
  });
}

int kot_cg_solve_middle(kot_problem* h, const double* vecs, const double* vals, int n_pos, double mu,
                        const double* rhs, double tol, int max_iter, double* x_out, int* iters, double* res) {
  return guarded([&] {
    kot::Problem& p = *h->p;
    KOT_CUDA(cudaSetDevice(p.device));
    kot::kot_require(mu > 0.0, kot::KOT_EINVAL, "regularization mu must be positive");
    kot::Bufs& b = p.bufs();
    const kot::Decomp dc = up_decomp(p, vecs, vals, n_pos);
    kot::MvCtx mv;
    kot::matvec_prepare(p, dc, mu, mv, true);
    up(p, b.e1, rhs, p.n);
    const kot::CgResult r = kot::cg_solve_op(p, b.e1, tol, max_iter, [&](const double* pv, double* ap) {
      kot::middle_operator_fast(p, mv, pv, ap);
    }, b.e2);
    down(p, x_out, b.e2, p.n);
    KOT_CUDA(cudaStreamSynchronize(p.st));
    *iters = r.iters;
    *res = r.res;
  });
}

int kot_middle_operator_decomp(kot_problem* h, const double* vecs, const double* vals, int n_pos, double mu,
                               const double* v, double* out) {
  return guarded([&] {
    kot::Problem& p = *h->p;
    KOT_CUDA(cudaSetDevice(p.device));
    kot::kot_require(mu > 0.0, kot::KOT_EINVAL, "regularization mu must be positive");
    kot::Bufs& b = p.bufs();
    const kot::Decomp dc = up_decomp(p, vecs, vals, n_pos);
    kot::MvCtx mv;
    kot::matvec_prepare(p, dc, mu, mv, true);
    up(p, b.e2, v, p.n);
    kot::middle_operator_fast(p, mv, b.e2, b.e1);
    down(p, out, b.e1, p.n);
    KOT_CUDA(cudaStreamSynchronize(p.st));
  });
}

int kot_newton_direction_decomp(kot_problem* h, const kot_solver_cfg* cfg, const double* r1, const double* r2,
                                const double* vecs, const double* vals, int n_pos, double mu, double* dgamma,
                                double* dx, int* cg_iters, int* criterion_met, double* crit_lhs, double* crit_rhs) {
  return guarded([&] {
    kot::Problem& p = *h->p;
    KOT_CUDA(cudaSetDevice(p.device));
    const kot::SolverCfg c = to_cfg(cfg);
    check_cfg(c);
    kot::kot_require(mu > 0.0, kot::KOT_EINVAL, "regularization mu must be positive");
    kot::Bufs& b = p.bufs();
    const long nn = (long)p.n * p.n;
    const kot::Decomp dc = up_decomp(p, vecs, vals, n_pos);
    up(p, b.r1w, r1, p.n);
    up(p, b.r2w, r2, nn);
    // r.norm() = ‖r1‖₂ + ‖r2‖_F (problem.py:56-57)
    const double rn = kot::dev_norm(p, b.r1w, p.n) + kot::dev_norm(p, b.r2w, nn);
    kot::kot_require(rn > 0.0, kot::KOT_EINVAL, "direction requires a nonzero residual");
    kot::NewtonOut o = kot::newton_direction(p, b.r1w, b.r2w, rn, dc, mu, c, b.dg, b.dX);
    kot::newton_resolve(p, rn, c, o);
    down(p, dgamma, b.dg, p.n);
    down(p, dx, b.dX, nn);
    KOT_CUDA(cudaStreamSynchronize(p.st));
    *cg_iters = o.cg_iters;
    *criterion_met = o.met;
    *crit_lhs = o.lhs;
    *crit_rhs = o.rhs;
  });
}

int kot_phi_forward(kot_problem* h, const double* x, double* out) {
  return guarded([&] {
    kot::Problem& p = *h->p;
    KOT_CUDA(cudaSetDevice(p.device));
    kot::Bufs& b = p.bufs();
    const long nn = (long)p.n * p.n;
    up(p, b.Xh, x, nn);
    kot::phi_forward(p, b.Xh, b.e1);
    down(p, out, b.e1, p.n);
    KOT_CUDA(cudaStreamSynchronize(p.st));
  });
}

int kot_phi_adjoint(kot_problem* h, const double* gamma, double* out) {
  return guarded([&] {
    kot::Problem& p = *h->p;
    KOT_CUDA(cudaSetDevice(p.device));
    kot::Bufs& b = p.bufs();
    const long nn = (long)p.n * p.n;
    up(p, b.e1, gamma, p.n);
    kot::phi_adjoint(p, b.e1, b.Xh);
    down(p, out, b.Xh, nn);
    KOT_CUDA(cudaStreamSynchronize(p.st));
  });
}

// objective_grad (problem.py:188-189): (Qγ − z)/(2λ₂);  mode 1 objective_grad_dir (:239-241): Qd/(2λ₂)
int kot_objective_grad(kot_problem* h, const double* gamma, int dir, double* out) {
  return guarded([&] {
    kot::Problem& p = *h->p;
    KOT_CUDA(cudaSetDevice(p.device));
    kot::Bufs& b = p.bufs();
    up(p, b.e1, gamma, p.n);
    if (dir) {
      KOT_CUDA(cudaMemsetAsync(b.e3, 0, sizeof(double) * p.n, p.st));
      kot::finalize(p, kot::FIN_JTOP, b.e1, false, b.e3, 0.0, b.e2);  // Qd/(2λ₂) + 0·d − 0 + 0
    } else {
      kot::finalize(p, kot::FIN_GRAD, b.e1, false, nullptr, 0.0, b.e2);
    }
    down(p, out, b.e2, p.n);
    KOT_CUDA(cudaStreamSynchronize(p.st));
  });
}

// constraint_matrix (problem.py:199-201): Φ*(γ) + λ₁I
int kot_constraint_matrix(kot_problem* h, const double* gamma, double* out) {
  return guarded([&] {
    kot::Problem& p = *h->p;
    KOT_CUDA(cudaSetDevice(p.device));
    kot::Bufs& b = p.bufs();
    const long nn = (long)p.n * p.n;
    up(p, b.e1, gamma, p.n);
    kot::phi_adjoint_ex(p, b.e1, b.Xh, 1.0, nullptr, 0.0, p.l1);
    down(p, out, b.Xh, nn);
    KOT_CUDA(cudaStreamSynchronize(p.st));
  });
}

int kot_residual_parts(kot_problem* h, const double* gamma, const double* x, double* r1, double* r2, double* eigvals,
                       int* n_pos, double* res_norm, double* eigvecs) {
  return guarded([&] {
    kot::Problem& p = *h->p;
    KOT_CUDA(cudaSetDevice(p.device));
    kot::Bufs& b = p.bufs();
    const long nn = (long)p.n * p.n;
    up(p, b.gw, gamma, p.n);
    up(p, b.Xw, x, nn);
    kot::Decomp dc{b.Pw, b.valw, 0};
    const double res = kot::residual_parts(p, b.gw, b.Xw, b.r1w, b.r2w, dc);
    if (r1) down(p, r1, b.r1w, p.n);
    if (r2) down(p, r2, b.r2w, nn);
    if (eigvals) down(p, eigvals, dc.vals, p.n);
    if (eigvecs) down(p, eigvecs, dc.P, nn);
    KOT_CUDA(cudaStreamSynchronize(p.st));
    if (n_pos) *n_pos = dc.k;
    if (res_norm) *res_norm = res;
  });
}

int kot_middle_operator(kot_problem* h, const double* gamma, const double* x, double theta, const double* v,
                        int form, double* out, double* mu_out) {
  return guarded([&] {
    kot::Problem& p = *h->p;
    KOT_CUDA(cudaSetDevice(p.device));
    kot::Bufs& b = p.bufs();
    const long nn = (long)p.n * p.n;
    up(p, b.gw, gamma, p.n);
    up(p, b.Xw, x, nn);
    kot::Decomp dc{b.Pw, b.valw, 0};
    const double res = kot::residual_parts(p, b.gw, b.Xw, b.r1w, b.r2w, dc);
    kot::kot_require(res > 0.0, kot::KOT_EINVAL, "context requires a nonzero residual");
    const double mu = theta * res;
    up(p, b.e2, v, p.n);
    if (form == 1) {
      kot::middle_operator(p, dc, mu, b.e2, b.e1);  // reference form Φ(𝒯[Φ*(v)])
    } else {
      kot::MvCtx mv;  // structure-reduced form: 0 the solver's, 2 the row-sharding layout
      kot::matvec_prepare(p, dc, mu, mv, form != 2);
      kot::middle_operator_fast(p, mv, b.e2, b.e1);
    }
    down(p, out, b.e1, p.n);
    KOT_CUDA(cudaStreamSynchronize(p.st));
    if (mu_out) *mu_out = mu;
  });
}

int kot_newton_direction(kot_problem* h, const kot_solver_cfg* cfg, const double* gamma, const double* x,
                         double theta, double* dgamma, double* dx, int* cg_iters, int* criterion_met,
                         double* crit_lhs, double* crit_rhs) {
  return guarded([&] {
    kot::Problem& p = *h->p;
    KOT_CUDA(cudaSetDevice(p.device));
    const kot::SolverCfg c = to_cfg(cfg);
    check_cfg(c);
    kot::Bufs& b = p.bufs();
    const long nn = (long)p.n * p.n;
    up(p, b.gw, gamma, p.n);
    up(p, b.Xw, x, nn);
    kot::Decomp dc{b.Pw, b.valw, 0};
    const double res = kot::residual_parts(p, b.gw, b.Xw, b.r1w, b.r2w, dc);
    kot::kot_require(res > 0.0, kot::KOT_EINVAL, "context requires a nonzero residual");
    kot::NewtonOut o = kot::newton_direction(p, b.r1w, b.r2w, res, dc, theta * res, c, b.dg, b.dX);
    kot::newton_resolve(p, res, c, o);
    down(p, dgamma, b.dg, p.n);
    down(p, dx, b.dX, nn);
    KOT_CUDA(cudaStreamSynchronize(p.st));
    *cg_iters = o.cg_iters;
    *criterion_met = o.met;
    *crit_lhs = o.lhs;
    *crit_rhs = o.rhs;
  });
}

int kot_eg_step(kot_problem* h, const double* gamma, const double* x, double stepsize, double* gamma_out,
                double* x_out) {
  return guarded([&] {
    kot::kot_require(stepsize > 0.0, kot::KOT_EINVAL, "stepsize must be positive");
    kot::Problem& p = *h->p;
    KOT_CUDA(cudaSetDevice(p.device));
    kot::Bufs& b = p.bufs();
    const long nn = (long)p.n * p.n;
    up(p, b.gv, gamma, p.n);
    up(p, b.Xv, x, nn);
    kot::eg_step_parallel(p, p.aux3(), b.gv, b.Xv, stepsize, b.gt, b.Xt);  // the solver's EG step
    down(p, gamma_out, b.gt, p.n);
    down(p, x_out, b.Xt, nn);
    KOT_CUDA(cudaStreamSynchronize(p.st));
  });
}

int kot_objective(kot_problem* h, const double* gamma, double* out) {
  return guarded([&] {
    kot::Problem& p = *h->p;
    KOT_CUDA(cudaSetDevice(p.device));
    kot::Bufs& b = p.bufs();
    up(p, b.e1, gamma, p.n);
    kot::finalize(p, kot::FIN_QV, b.e1, false, nullptr, 0.0, b.e2);  // Qγ
    const double quad = kot::dev_dot(p, b.e1, b.e2, p.n) / (4.0 * p.l2);
    const double lin = kot::dev_dot(p, b.e1, p.z, p.n) / (2.0 * p.l2);
    *out = quad - lin + p.q_sq / (4.0 * p.l2);
  });
}

int kot_ot_estimate(kot_problem* h, const double* gamma, double* out) {
  return guarded([&] {
    kot::Problem& p = *h->p;
    KOT_CUDA(cudaSetDevice(p.device));
    kot::kot_require(p.has_embed, kot::KOT_EINVAL, "instance carries no embedding sums; assemble() provides them");
    kot::Bufs& b = p.bufs();
    up(p, b.e1, gamma, p.n);
    *out = (p.q_sq - kot::dev_dot(p, b.e1, p.embed, p.n)) / (2.0 * p.l2);
  });
}

}  // extern "C"
