// Device-resident SSN problem and operators (reference problem.py, psdcone.py,
// newton.py, eg.py, solver.py).
#pragma once
#include <functional>
#include <memory>
#include <vector>

#include "kernels.cuh"

namespace kot {

struct Decomp {
  double* P = nullptr;     // n×n, columns = eigenvectors (descending)
  double* vals = nullptr;  // n
  int k = 0;               // #(σ > 0)
};

struct SolverCfg {
  double tau, kappa, alpha1, alpha2, beta0, beta1, beta2, theta_min, theta_max, theta0;
  int cg_max, cg_restarts;
  double cg_tol;
  int has_cg_tol;
  double eg_stepsize, residual_tol;
  int max_iter, safeguard_every;
};

struct IterRecord {
  int iteration;
  double res_accepted, res_ssn, res_eg;
  int accepted_ssn;
  double theta, mu;
  int cg_iters, criterion_met;
  double crit_lhs, crit_rhs, eg_ms, newton_ms, cg_ms, resid_ms, step_ms;
  int n_pos, attempts;
};

// Solver-owned device buffers (allocated on first use).
struct Bufs {
  double *Xw, *Xv, *Xt, *r2w, *r2v, *r2t, *Pw, *Pv, *Pt, *Pe, *Xh, *dX, *filt, *a2t;  // n×n
  double *gw, *gv, *gt, *r1w, *r1v, *r1t, *valw, *valv, *valt, *vale, *dg, *a1, *rhs, *sol, *corr;  // n
  double *cx, *cr, *cp, *cap, *e1, *e2, *e3;  // n
  double *Bm, *Ct, *Hm;  // n×n: B = R·P, T̃, H = G_α∘G_α (structure-reduced matvec)
  double* Bp;            // n×(n+2): B's sign blocks packed [smaller | other], 16-B aligned
};

// CUDA graph of one batch of CG steps (solver.cu) and the matvec context it was captured for.
struct CgGraphKey {
  const double *Bs = nullptr, *Bo = nullptr;
  long ldp = 0;
  const double *H = nullptr, *vals = nullptr;
  int k = -1;
  bool pos = false;
  double mu = 0.0;
  int batch = 0;
  bool operator==(const CgGraphKey& o) const {
    return Bs == o.Bs && Bo == o.Bo && ldp == o.ldp && H == o.H && vals == o.vals && k == o.k && pos == o.pos &&
           mu == o.mu && batch == o.batch;
  }
};
struct CgGraph {
  cudaGraphExec_t exec = nullptr;
  CgGraphKey key;
  long long kernels = 0;
};

struct Problem {
  int n = 0;
  int device = 0;
  int lane = 0;  // 0: Newton chain (priority), 1: EG pipeline contexts
  double l1 = 0, l2 = 0, q_sq = 0, jitter = 0;
  bool has_embed = false;
  cudaStream_t st = nullptr;
  // instance data (device)
  double *Q = nullptr, *z = nullptr, *R = nullptr, *embed = nullptr, *Kmat = nullptr;
  double* G2 = nullptr;  // (RRᵀ)∘(RRᵀ), lazily
  bool g2_valid = false;   // G2 holds the current R's product (reset when a pooled problem is reused)
  double* kmat_buf = nullptr;  // pair Gram storage (Kmat points here for assembled instances)
  std::vector<double*> pipe_bufs;  // EG pipeline slots, allocated once per problem (solver.cu)
  // scratch
  std::unique_ptr<EigWork> eig;
  std::vector<double*> owned;
  double* partial = nullptr;  // rowdot partials [tiles][n]
  double *M1 = nullptr, *M2 = nullptr, *M3 = nullptr, *M4 = nullptr, *M5 = nullptr;  // n×n temps
  double* red = nullptr;   // reduction partials
  double* splitws = nullptr;  // split-K partials
  long splitws_cap = 0;
  double* dsc = nullptr;   // device scalars
  double* hsc = nullptr;   // pinned host scalars
  int* dk = nullptr;
  int* dflag = nullptr;
  int* hk = nullptr;       // pinned

  std::unique_ptr<Bufs> bufs_;
  Bufs& bufs();
  // second execution context (own stream + scratch, shared instance data) on
  // which the EG safeguard chain runs concurrently with the Newton chain
  // row sharding of the CG matvec (config 4): NCCL communicator and this rank's row block
  void* nccl_comm = nullptr;
  // host data plane (kot_problem_shard_host): the caller's collectives on host buffers (gloo, MPI…)
  int (*host_comm)(void* user, int op, double* buf, long count, long block, int rank, int world) = nullptr;
  void* host_comm_user = nullptr;
  double* host_comm_buf = nullptr;  // pinned staging, max(k·ℓ, block·world) doubles
  long host_comm_cap = 0;
  bool sharded() const { return nccl_comm != nullptr || host_comm != nullptr; }
  int shard_rank = 0, shard_world = 1, shard_block = 0, row0 = 0, row1 = -1;
  double* ygather = nullptr;  // shard_block·world doubles
  int emul_world = 1;          // test hook: all row blocks in turn on one device, no NCCL
  double* shard_tmp = nullptr;  // (⌊ℓ/2⌋+1)·ℓ block partial of T̃ (emulation only)
  double* shard_stage = nullptr;  // 2N·⌈ℓ/2N⌉ rows of B in gather order (split H form, sharded)
  long shard_stage_cap = 0;
  double* mv_y = nullptr;         // ℓ: one emulated rank's partial y (split H form, emulation)
  std::unique_ptr<Problem> aux_, aux2_, aux3_, crit_;
  Problem& aux();
  Problem& aux2();
  Problem& aux3();  // second EG-step context: the step's second projection runs beside the first
  // high-priority context for the speculative Newton criterion (no eigensolver workspace):
  // its stream, scratch, outputs (crit_dg, crit_dX, crit_e1) and completion event
  Problem& crit();
  double *crit_dg = nullptr, *crit_dX = nullptr, *crit_e1 = nullptr;
  double* mv_ct = nullptr;  // criterion context: its own T̃ (ℓ×ℓ) for the H-form matvec (no full Bufs)
  cudaEvent_t crit_done = nullptr, crit_after = nullptr, crit_dx_done = nullptr;
  cudaEvent_t ev_half = nullptr;  // eg_step_parallel: γ½ ready
  cudaEvent_t ev_mv0 = nullptr, ev_mv1 = nullptr;  // newton_direction: matvec_prepare on the crit stream
  cudaEvent_t ev_rhs = nullptr;
  CgGraph cg_graph;                    // newton_direction: next attempt's rhs ready
  bool with_eig = true;
  double* alloc(long count);
  void init_scratch();
  ~Problem();
};

// Destroyed handles go to a small per-(order, device) pool of idle problems with all their workspace
// (contexts, eigensolver, solver buffers); a new instance of the same order reuses one and only
// uploads / assembles its data.  Sharded problems are never pooled.
void problem_release(std::unique_ptr<Problem> p);
std::unique_ptr<Problem> problem_from_host(const double* q, const double* z, double q_sq, const double* r,
                                           const double* embed, int n, double l1, double l2, double jitter, int device);
std::unique_ptr<Problem> problem_assemble(const double* xs, int nx, const double* ys, int ny, const double* xt,
                                          const double* yt, int l, int d, double bw_x, double bw_y, double bw_xy,
                                          double l1, double l2, int device);

// ---- operators (device pointers in/out, all on p.st)
void phi_forward(Problem& p, const double* X, double* out);
void phi_adjoint(Problem& p, const double* g, double* out);
void eigh(Problem& p, const double* Z, Decomp& dc, bool alpha_only = false);
void proj(Problem& p, const Decomp& dc, const double* X, double* out);  // out = X − Π (X!=null) or Π
// mode 0: eliminator 𝒯 with μ; mode 1: projection Jacobian M. force_path: -1 auto, 0 POS, 1 NONPOS.
void spectral_filter(Problem& p, const Decomp& dc, const double* S, double* out, double mu, int mode,
                     int force_path = -1);
// alpha_only: the decomposition holds only the σ > 0 eigenvectors (enough for r2 and the norm)
double residual_parts(Problem& p, const double* g, const double* X, double* r1, double* r2, Decomp& dc,
                      bool alpha_only = false);
// residual_parts at (γ, X) = (0, 0) (the solver's starting pair): no eigensolve needed
double residual_parts_origin(Problem& p, const double* g, const double* X, double* r1, double* r2, Decomp& dc);
void middle_operator(Problem& p, const Decomp& dc, double mu, const double* v, double* out);
void eg_step(Problem& p, const double* g, const double* X, double s, double* g_out, double* X_out);
// Same values as eg_step; the second projection Π(X − s(Φ*(γ½) + λ₁I)) needs γ½ but not X½
// (eg.py:34-41), so it runs on context c (its own host thread) concurrently with the first one.
void eg_step_parallel(Problem& p, Problem& c, const double* g, const double* X, double s, double* g_out,
                      double* X_out);

// structure-reduced middle operator (the CG matvec of the solver)
struct MvCtx {
  Decomp dc;
  double mu = 0.0;
  bool pos = true;
  bool direct = false;  // diagnostic: KOT_MATVEC=direct uses the reference Φ*→𝒯→Φ chain
  bool hform = false;   // same-sign block as a GEMV with H = G_α∘G_α (KOT_MATVEC=full: off)
  // H form split over ranks (row-sharded problems, or the single-device emulation hook): rank g owns
  // the columns [c0_g, c1_g) of the mixed sign block (both GEMMs), the rows of its folded row blocks for
  // the H/Q GEMVs, and the ranks' partial y vectors are summed (one all-reduce of ℓ doubles per matvec)
  bool split = false;
  int world = 1;
  double* B = nullptr;
  double* H = nullptr;
  const double *Bs = nullptr, *Bo = nullptr;  // H form: packed smaller / other sign block of B
  long ldp = 0;
};
// stream (nullable): where B, its packed sign blocks and H are built (default p.st)
void matvec_prepare(Problem& p, const Decomp& dc, double mu, MvCtx& m, bool allow_hform = true,
                    cudaStream_t stream = nullptr);
// shard.cu
void nccl_unique_id(char* out128);
void problem_shard(Problem& p, const char* id128, int rank, int world);
void problem_unshard(Problem& p);
void problem_shard_emulate(Problem& p, int world);
void problem_shard_host(Problem& p, int (*fn)(void*, int, double*, long, long, int, int), void* user, int rank,
                        int world);
// collectives of a sharded problem on stream st (NCCL, or the host data plane)
void shard_allreduce_sum(Problem& p, double* buf, long count, cudaStream_t st);
void shard_allgather(Problem& p, double* buf, long block, cudaStream_t st);
// folded row blocks of rank g of N: [a0,a1) = block g and [b0,b1) = block 2N−1−g of ⌈ℓ/2N⌉ rows each,
// so that every rank gets the same share of R's upper triangle (row i costs ℓ − i in B = R·P)
struct FoldedRows {
  int blk, a0, a1, b0, b1;
};
FoldedRows folded_rows(int n, int g, int world);
void shard_allreduce_sum(Problem& p, double* buf, long count);
void shard_allgather(Problem& p, double* buf, long block);
// skipf (nullable): every launch is a no-op once *skipf != 0 (batched CG, H form only)
void middle_operator_fast(Problem& p, const MvCtx& m, const double* v, double* out,
                          const double* skipf = nullptr);

struct NewtonOut {
  int cg_iters, met, attempts;
  double lhs, rhs, cg_ms;
  bool crit_pending = false;  // met/lhs/rhs of the last attempt still in flight: newton_resolve
};
struct CgResult {
  int iters;
  double res;
};
CgResult cg_solve_op(Problem& p, const double* rhs, double tol, int max_iter,
                     const std::function<void(const double*, double*)>& apply, double* x_out);
NewtonOut newton_direction(Problem& p, const double* r1, const double* r2, double res_norm, const Decomp& dc,
                           double mu, const SolverCfg& cfg, double* dg, double* dX);
// completes met / lhs / rhs of a direction whose last criterion was left running (res_norm as passed
// to newton_direction)
void newton_resolve(Problem& p, double res_norm, const SolverCfg& cfg, NewtonOut& out);

// internal helpers shared with solver.cu
enum FinMode { FIN_RES = 0, FIN_MATVEC = 1, FIN_A1 = 2, FIN_JTOP = 3, FIN_PHI = 4, FIN_GRAD = 5, FIN_QV = 6,
               FIN_MATVEC_B = 7 };
void dev_reduce(Problem& p, const double* a, const double* b, long count, int slot, bool sq);
void fetch(Problem& p, int count);
void axpby(Problem& p, long count, double a, const double* x, double b, const double* y, double* out);
void finalize(Problem& p, int mode, const double* u, bool with_phi, const double* r1, double mu, double* out);
void phi_partials(Problem& p, const double* X);
void phi_adjoint_ex(Problem& p, const double* g, double* out, double alpha, const double* X, double beta, double diag);
int ew_grid(long count);
void symmetrize(Problem& p, const double* a, double* out);  // 0.5 (a + aᵀ)
void neg_div(Problem& p, long count, const double* x, double c, double* out);               // out = −(x/c)
void jac_bottom(Problem& p, long count, const double* a, const double* b, double mu, const double* c,
                double* out);                                                                 // (a + (1+μ)b) + c

// host-side reductions (synchronising)
double dev_norm(Problem& p, const double* x, long count);
double dev_dot(Problem& p, const double* x, const double* y, long count);

// ---- solver
typedef int (*IterCallback)(void* user, int iteration, const double* w_gamma, const double* w_x,
                             const double* r_gamma, const double* r_x, double mu, double theta,
                             const double* dw_gamma, const double* dw_x, int criterion_met);
struct SolveResult {
  int status;  // KOT_OK or KOT_ENUMERICS
  int converged;
  int iterations;
  double residual_norm;
  double ot_estimate;
  double total_ms;
};
SolveResult solve(Problem& p, const SolverCfg& cfg, IterCallback cb, void* user, double* gamma_out, double* x_out,
                  IterRecord* trace, int trace_cap, bool pure_eg);

struct ReplayIn {
  const double *wg, *wx, *vg, *vx;
  double theta;
  int k;
};
struct ReplayOut {
  double *wg, *wx, *vg, *vx;
  double theta;
};
IterRecord iterate_once(Problem& p, const SolverCfg& cfg, const ReplayIn& in, ReplayOut& out);

struct Session;
Session* session_begin(Problem& p, const SolverCfg& cfg);
int session_step(Session& se, int iters, IterRecord* recs);
void session_result(Session& se, double* gamma, double* x, SolveResult& out);
void session_end(Session* se);
void session_state(Session& se, double* wg, double* wx, double* vg, double* vx, double* theta);

}  // namespace kot
