/* libkotgpu — C ABI of the B200-native semismooth-Newton kernel-OT solver.
 *
 * Drop-in boundary for the reference package `kot` (pure Python;
 * /root/reference/pkg/src/kot).  The reference exposes no native ABI, so each
 * entry point below replaces the Python call it cites; the Python host layer
 * (paper_2310_14087_b200/) binds them with ctypes exactly as INTEGRATION.md
 * shows.  Conventions:
 *   - all arrays are caller-owned, C-contiguous (row-major) float64; inputs
 *     are read-only and copied to the device, outputs are caller-allocated;
 *   - every function returns a status (0 = ok) that maps 1:1 onto the
 *     reference's exception classes; kot_last_error() gives the message
 *     (thread-local);
 *   - one handle per problem, each with its own CUDA stream; handles may be
 *     used from different host threads concurrently; no global mutable state.
 */
#ifndef KOTGPU_H_
#define KOTGPU_H_

#ifdef __cplusplus
extern "C" {
#endif

enum {
  KOT_OK = 0,
  KOT_EINVAL = 1,       /* ValueError                 problem.py:116-119, newton.py:61-71, solver.py:45-51 */
  KOT_EINDEFINITE = 2,  /* IndefiniteKernelError      linalg.py:114 */
  KOT_EEIG = 3,         /* EigenSolveError            linalg.py:70 */
  KOT_ENUMERICS = 4,    /* SolverNumericsError        solver.py:28-33 (partial trace returned) */
  KOT_ECG = 5,          /* FloatingPointError         linalg.py:146,156 */
  KOT_ECUDA = 6,        /* CUDA runtime failure */
  KOT_EASSERT = 7,      /* AssertionError             psdcone.py:77 */
  KOT_ECALLBACK = 8     /* the on_iteration callback returned nonzero (solver.py:170-181: an observer
                           exception propagates and ends the solve) */
};

typedef struct kot_problem kot_problem;

/* SolverConfig + NewtonConfig + EgConfig flattened (solver.py:36-51,
 * newton.py:36-71, eg.py:18-24). */
typedef struct {
  double tau, kappa, alpha1, alpha2, beta0, beta1, beta2, theta_min, theta_max, theta0;
  int cg_max, cg_restarts;
  double cg_tol;
  int has_cg_tol;
  double eg_stepsize, residual_tol;
  int max_iter, safeguard_every;
} kot_solver_cfg;

/* IterationRecord (solver.py:54-73) + n_pos and CG attempts. */
typedef struct {
  int iteration;
  double res_accepted, res_ssn, res_eg;
  int accepted_ssn;
  double theta, mu;
  int cg_iters, criterion_met;
  double crit_lhs, crit_rhs, eg_ms, newton_ms, cg_ms, resid_ms, step_ms;
  int n_pos, attempts;
} kot_iter_record;

/* SolverReport scalars (solver.py:89-101). */
typedef struct {
  int converged;     /* termination == "converged" (else "max_iter") */
  int iterations;    /* len(trace) */
  double residual_norm;
  double ot_estimate; /* NaN if the instance carries no embedding sums */
  double total_ms;
} kot_report;

/* on_iteration observer (solver.py:76-86, 170-181); host copies of w, r, dw.  A nonzero return
 * stops the solve with KOT_ECALLBACK (the Python shim re-raises the observer's exception). */
typedef int (*kot_iter_cb)(void* user, int iteration, const double* w_gamma, const double* w_x,
                            const double* r_gamma, const double* r_x, double mu, double theta,
                            const double* dw_gamma, const double* dw_x, int criterion_met);

/* ---- problem construction --------------------------------------------- */

/* Upload a host ProblemData (problem.py:86-123; q is symmetrised as in :112). */
int kot_problem_create(const double* q, const double* z, double q_sq, const double* r_upper,
                       const double* embed /* nullable */, int l, double lambda1, double lambda2,
                       double jitter, int device, kot_problem** out);

/* assemble() on device (problem.py:135-169): Gaussian Grams, mean embeddings,
 * embedding norms, pair Gram K and its jittered Cholesky factor.  bw_x / bw_y / bw_xy are
 * spec_x / spec_y / spec_xy.bandwidth_sq (equal under build_kernel_specs, problem.py:126-132). */
int kot_assemble(const double* xs, int n_mu, const double* ys, int n_nu, const double* xt,
                 const double* yt, int l, int d, double bw_x, double bw_y, double bw_xy, double lambda1,
                 double lambda2, int device, kot_problem** out);

int kot_problem_info(const kot_problem* p, int* l, double* q_sq, double* jitter, double* lambda1,
                     double* lambda2, int* has_embed);

/* Download ProblemData fields (any pointer may be NULL). */
int kot_problem_download(kot_problem* p, double* q, double* z, double* r_upper, double* embed,
                         double* kmat);

void kot_problem_destroy(kot_problem* p);

const char* kot_last_error(void);

/* ---- solve (solver.py:114-233, 236-289) -------------------------------- */

int kot_solve(kot_problem* p, const kot_solver_cfg* cfg, kot_iter_cb cb, void* user,
              double* gamma_out /* l */, double* x_out /* l*l, nullable */,
              kot_iter_record* trace /* trace_cap */, int trace_cap, kot_report* out);

int kot_solve_pure_eg(kot_problem* p, const kot_solver_cfg* cfg, double* gamma_out, double* x_out,
                      kot_iter_record* trace, int trace_cap, kot_report* out);

/* One loop body from host state (w, v, theta) at iteration k: the lock-step
 * replay unit of the parity protocol. */
int kot_iterate(kot_problem* p, const kot_solver_cfg* cfg, const double* w_gamma, const double* w_x,
                const double* v_gamma, const double* v_x, double theta, int k, double* w_gamma_out,
                double* w_x_out, double* v_gamma_out, double* v_x_out, double* theta_out,
                kot_iter_record* rec);

/* ---- sessions: a solve driven in chunks (bench.py: warm-up + timed
 * iterations of one continuous trajectory, timed with CUDA events on the
 * problem's stream) ---------------------------------------------------- */
typedef struct kot_session kot_session;
int kot_session_begin(kot_problem* p, const kot_solver_cfg* cfg, kot_session** out);
/* run up to `iters` loop bodies; *done = how many ran (stops at convergence/max_iter) */
int kot_session_step(kot_session* s, int iters, kot_iter_record* recs /* nullable */, int* done);
int kot_session_result(kot_session* s, double* gamma_out, double* x_out, kot_report* out);
void kot_session_end(kot_session* s);
/* loop state between two iterations (any pointer may be NULL): w, the safeguard iterate v, theta */
int kot_session_state(kot_session* s, double* w_gamma, double* w_x, double* v_gamma, double* v_x, double* theta);
/* the cudaStream_t (as void*) every kernel of this problem is launched on */
void* kot_problem_stream(kot_problem* p);

/* ---- row sharding of the CG matvec over NCCL (BASELINE config 4) ----------
 * Replaces nothing in the reference (kot is single-process); the sharded solve
 * is the same kot.solver.solve (solver.py:114) with its structure-reduced
 * middle operator (newton.py:70-95) split by rows of B = R·P across `world`
 * processes, one GPU each.  Every rank calls the same entry points on the same
 * problem; results are identical on all ranks.
 *   kot_nccl_unique_id: rank 0 creates the 128-byte ncclUniqueId, the caller
 *                       broadcasts it (torch.distributed / MPI / files).
 *   kot_problem_shard:  collective over `world` ranks; world <= 1 unshards.
 *                       id128 == NULL with world > 1 is a single-device test hook:
 *                       every row block is computed in turn, no communication.
 * NCCL (libnccl.so.2) is dlopen'ed on first use. */
int kot_nccl_unique_id(char* out128);
int kot_problem_shard(kot_problem* p, const char* id128, int rank, int world);
/* Same row sharding over a caller-supplied host data plane (gloo, MPI, …) instead of NCCL: the
 * library stages the exchanged device buffers through pinned host memory and calls fn on the thread
 * that called kot_solve.  op 0: in-place sum over ranks of `count` doubles; op 1: in-place
 * all-gather, rank g's `block` doubles at buf + g·block (count = block·world).  fn returns 0 on
 * success.  Used where ranks share a GPU (tests) or NCCL is unavailable. */
typedef int (*kot_comm_fn)(void* user, int op, double* buf, long count, long block, int rank, int world);
int kot_problem_shard_host(kot_problem* p, kot_comm_fn fn, void* user, int rank, int world);
int kot_problem_shard_info(const kot_problem* p, int* rank, int* world, int* row0, int* row1);

/* ---- phase profiler (CUDA events around library phases; off by default) --- */
typedef struct {
  char name[32];
  long long calls;
  double ms;      /* summed event time */
  double flops;   /* algorithmic FLOPs (0 where not applicable) */
  double bytes;   /* algorithmic HBM/L2 bytes (0 where not applicable) */
} kot_prof_entry;
int kot_profile_enable(int on);  /* 0 off, 1 every scope, 2 roofline scopes only (cheap); resets the counters */
int kot_profile_read(kot_prof_entry* out, int cap);  /* returns #entries */

/* Process-wide cap on the CTAs of every tridiagonalisation panel grid (0 = all SMs): several concurrent
 * solves sharing one GPU (batches of independent problems) run faster on thin grids. */
int kot_set_panel_grid_cap(int cap);

/* Process set-up of a long-running service: grows the library's device memory pool by `bytes` once (the
 * bytes go straight back to the pool, which never trims).  Without it the first solve of a process pays the
 * driver's mapping of the pool (4 … 300 ms for the ≈ 3.5 GB of an l = 2000 problem, depending on what ran on
 * the GPU before); every problem, workspace and context is still allocated by the calls that need them. */
int kot_reserve(int device, unsigned long long bytes);

/* ---- test / diagnostic hooks (process-wide; not part of the drop-in surface) ---- */
int kot_debug_eig_stages(int stages);   /* 0 automatic, 1 one-stage, 2 two-stage, 3 two-stage in background */
int kot_debug_cg_batch(int batch);      /* CG iterations enqueued per host check (>= 1; default 4) */
int kot_debug_gemm_tma(int mode);       /* 1: TMA-staged DMMA GEMM core (default), 0: the cp.async core */
int kot_debug_eg_parallel(int on);      /* EG-step projections side by side (1, default) or in sequence */
int kot_debug_sytrd_timing(int on, unsigned long long* out8);  /* panel-kernel segment timers (ns) */
int kot_debug_tail_timing(int on, unsigned long long* out8);   /* cluster-tail segment timers (ns) */
int kot_debug_mid_timing(int on, unsigned long long* out8);    /* grid-resident mid-kernel segment timers (ns) */
/* grid-resident sytrd mid kernel: mode 0 off, 1 latency-critical eigensolves (default), 2 every eigensolve;
 * tail = trailing columns handed to the cluster tail (0: none); a negative value leaves a setting unchanged */
int kot_debug_trd_mid(int mode, int tail);
/* the mid kernel's head launch (the columns only every SM together can hold, before the launch that leaves
 * SMs to the other chains): 0 off, 1 beside an EG pipeline (default), 2 also for standalone eigensolves */
int kot_debug_trd_mid_head(int mode);
/* clock64 stamps of the mid kernel, [8 columns from c0][16 warps][16 points] of CTA cta (on = 1 arms, 0 reads) */
int kot_debug_mid_trace(int on, int c0, int cta, long long* out);
/* host-only (no GPU): largest order of the mid kernel's resident block for `grid` CTAs with smem_max bytes
 * of dynamic shared memory each; a self-test of the cooperative-grid gate (background panel loops that
 * yield, a foreground thread opening exclusive windows): windows completed, or < 0 on a violation */
int kot_debug_mid_capacity(int grid, long smem_max);
int kot_debug_gate_selftest(int nbg, int ms);

/* ---- operators (host buffers in/out; per-kernel parity) ----------------- */

/* gram_matrix (kernels.py:61-73), square form: out = exp(-|a_i-a_j|^2/(2 bw)), unit diag. */
int kot_gram(const double* pts, int n, int d, double bandwidth_sq, int device, double* out);
/* gram_matrix (kernels.py:61-73), rectangular form: out[i][j] = exp(-|a_i-b_j|^2/(2 bw)), m × p. */
int kot_gram_rect(const double* a, int m, const double* b, int p, int d, double bandwidth_sq, int device,
                  double* out);
/* mean_embedding (kernels.py:83-87): out[j] = mean_i k(s_i, q_j), the n × m Gram never stored. */
int kot_mean_embedding(const double* samples, int n, const double* queries, int m, int d, double bandwidth_sq,
                       int device, double* out);
/* sobol_natural / sobol_points (datagen.py:77-132): unscrambled Sobol points with natural indices
 * first … first+count−1 (the reference's `index + 1`), each coordinate mapped into [lower, upper]:
 * out[j][k] = lower[k] + (XOR_{b: bit b of first+j} dirnums[k][b]) / 2^bits · (upper[k] − lower[k]).
 * dirnums: dim × bits direction numbers (the reference's SciPy generator's table). */
int kot_sobol_points(const unsigned long long* dirnums, int dim, int bits, long first, int count,
                     const double* lower, const double* upper, int device, double* out);
/* embedding_norm_sq (kernels.py:90-94): mean of the n × n sample Gram. */
int kot_embedding_norm_sq(const double* samples, int n, int d, double bandwidth_sq, int device, double* out);
/* cholesky_psd (linalg.py:91-114). */
int kot_cholesky_psd(const double* k, int n, int device, double* r_upper, double* jitter);
/* sym_eig (linalg.py:60-83): descending eigenvalues, eigvecs in columns, n_pos. */
int kot_sym_eig(const double* z, int n, int device, double* vecs, double* vals, int* n_pos);
/* proj_psd (psdcone.py:62-64). */
int kot_proj_psd(const double* z, int n, int device, double* out);
/* apply_eliminator / apply_proj_jacobian at the decomposition of z (psdcone.py:94-151).
 * mode 0: eliminator with mu; mode 1: projection Jacobian.  path: -1 auto, 0 POS, 1 NONPOS. */
int kot_spectral_apply(const double* z, int n, int device, int mode, double mu, int path,
                       const double* s, double* out);
/* The same operators at a GIVEN decomposition (eigvecs in columns, eigenvalues descending, the first
 * n_pos strictly positive — a SpectralDecomp): mode 0 apply_eliminator(make_eliminator(coeffs, mu), s)
 * (psdcone.py:103-151), 1 apply_proj_jacobian(coeffs, s) (:94-100), 2 proj_from_decomp (:52-59; s unused). */
int kot_spectral_apply_decomp(const double* vecs, const double* vals, int n, int n_pos, int device, int mode,
                              double mu, int path, const double* s, double* out);
/* apply_jacobian (problem.py:222-236) at a decomposition: top = Qdγ/(2λ₂) + μdγ − Φ(dX),
 * bottom = M[Φ*(dγ) − dX] + (1+μ)dX. */
int kot_apply_jacobian(kot_problem* p, const double* vecs, const double* vals, int n_pos, double mu,
                       const double* dgamma, const double* dx, double* top, double* bottom);
/* cg_solve (linalg.py:117-162) for a host matvec callable: the CG recurrence runs on the device, each
 * matvec calls fn(user, p, ap) on host copies (nonzero return → KOT_ECALLBACK).  Same stopping rule
 * (‖r‖ ≤ tol·‖rhs‖), pᵀAp ≤ 0 → iters−1, non-finite → KOT_ECG. */
typedef int (*kot_matvec_fn)(void* user, const double* p, double* ap);
int kot_cg_solve(kot_matvec_fn fn, void* user, const double* rhs, int n, double tol, int max_iter, int device,
                 double* x_out, int* iters, double* res);
/* middle_operator(pd, make_eliminator(proj_jacobian_coeffs(decomp), mu), mu) (newton.py:116-128)
 * applied to v, at a given decomposition (the solver's structure-reduced evaluation). */
int kot_middle_operator_decomp(kot_problem* p, const double* vecs, const double* vals, int n_pos, double mu,
                               const double* v, double* out);
/* cg_solve on that middle operator, entirely on the device (the fused CG of the Newton step). */
int kot_cg_solve_middle(kot_problem* p, const double* vecs, const double* vals, int n_pos, double mu,
                        const double* rhs, double tol, int max_iter, double* x_out, int* iters, double* res);
/* newton_direction(pd, r, ctx, cfg) (newton.py:144-195) with ctx = newton_context(decomp, r.norm(),
 * theta), mu = theta·r.norm(). */
int kot_newton_direction_decomp(kot_problem* p, const kot_solver_cfg* cfg, const double* r1, const double* r2,
                                const double* vecs, const double* vals, int n_pos, double mu, double* dgamma,
                                double* dx, int* cg_iters, int* criterion_met, double* crit_lhs,
                                double* crit_rhs);
int kot_phi_forward(kot_problem* p, const double* x, double* out);      /* problem.py:172-177 */
int kot_phi_adjoint(kot_problem* p, const double* gamma, double* out);  /* problem.py:180-185 */
/* objective_grad (problem.py:188-189): (Qγ − z)/(2λ₂); dir = 1: objective_grad_dir (:239-241), Qd/(2λ₂). */
int kot_objective_grad(kot_problem* p, const double* gamma, int dir, double* out);
/* constraint_matrix (problem.py:199-201): Φ*(γ) + λ₁I. */
int kot_constraint_matrix(kot_problem* p, const double* gamma, double* out);
/* residual_parts (problem.py:204-214): r1, r2, eigenvalues of Z (descending), n_pos, ||r||, and
 * the eigenvectors (nullable: the SpectralDecomp's host copy). */
int kot_residual_parts(kot_problem* p, const double* gamma, const double* x, double* r1, double* r2,
                       double* eigvals, int* n_pos, double* res_norm, double* eigvecs);
/* middle_operator (newton.py:116-128) at the context of w with damping theta.
 * form 0: structure-reduced B = R·P form used by the solver (same-sign block as (G_a∘G_a)v/mu);
 * 1: reference form Φ(𝒯[Φ*(v)]); 2: structure-reduced, whole sign block in the GEMMs (row-sharded layout). */
int kot_middle_operator(kot_problem* p, const double* gamma, const double* x, double theta,
                        const double* v, int form, double* out, double* mu_out);
/* newton_direction (newton.py:144-195) at w with damping theta. */
int kot_newton_direction(kot_problem* p, const kot_solver_cfg* cfg, const double* gamma,
                         const double* x, double theta, double* dgamma, double* dx, int* cg_iters,
                         int* criterion_met, double* crit_lhs, double* crit_rhs);
/* eg_step (eg.py:34-41). */
int kot_eg_step(kot_problem* p, const double* gamma, const double* x, double stepsize,
                double* gamma_out, double* x_out);
/* evaluate_map (problem.py:254-284): potential u(q_j) and Monge map T(q_j) = q_j − ∇u(q_j). */
int kot_evaluate_map(const double* xs, int n, const double* x_tilde, const double* gamma_hat, int l,
                     const double* queries, int m, int d, double bandwidth_sq, double lambda2, int device,
                     double* u_out, double* t_out);
/* objective (problem.py:192-196) and ot_estimate (problem.py:244-251). */
int kot_objective(kot_problem* p, const double* gamma, double* out);
int kot_ot_estimate(kot_problem* p, const double* gamma, double* out);

/* Diagnostics: number of kernels libkotgpu launched since load (all handles). */
long long kot_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* KOTGPU_H_ */
