#include <atomic>
// Internal (C++) interface of libkotgpu: device-level building blocks.
#pragma once
#include "common.cuh"

namespace kot {

// ---------------------------------------------------------------- gram.cu
void gram_square(const double* P0, const double* P1, int n, int d, double bw0, double bw1, int nsets, bool pair,
                 double* out, cudaStream_t st);
void assemble_device(const double* xs, int nx, const double* ys, int ny, const double* xt, const double* yt, int l,
                     int d, double bw_x, double bw_y, double bw_xy, double lambda2, double* Q, double* Kmat,
                     double* embed, double* z, double* q_sq, double* scratch, cudaStream_t st);
// rectangular Gram out[i][j] = k(a_i, b_j) (m × p); column means of the n × m sample/query Gram;
// mean of the n × n sample Gram (unit diagonal) — kernels.py:61-94
void sobol_points_device(const unsigned long long* V, int dim, int bits, long first, int count,
                         const double* lower, const double* upper, double* out, cudaStream_t st);
void gram_rect(const double* A, int m, const double* B, int p, int d, double bw, double* out, cudaStream_t st);
void mean_embedding_device(const double* S, int n, const double* F, int m, int d, double bw, double* out,
                           cudaStream_t st);
void embedding_norm_sq_device(const double* S, int n, int d, double bw, double* scratch, double* out,
                              cudaStream_t st);

void evaluate_map_device(const double* xs, int n, const double* xt, const double* gamma, int l, const double* qs,
                         int m, int d, double bw, double lambda2, double* u, double* tmap, cudaStream_t st);

// ---------------------------------------------------------------- chol.cu
// Upper R with RᵀR = sym(K) + jitter·I (row-major).  work: n*n doubles; dscal: 1 device double.
double cholesky_psd_device(const double* K, int n, double* R, double* work, double* dscal, int* dflag,
                           cudaStream_t st);

// ----------------------------------------------------------------- eig.cu
struct EigWork {
  int n;
  double *A = nullptr, *Vall = nullptr, *X = nullptr, *d = nullptr, *e = nullptr, *tau = nullptr;
  double *xv = nullptr, *yv = nullptr, *part = nullptr, *partn = nullptr, *Tf = nullptr, *W1 = nullptr;
  double *Q = nullptr, *Qw = nullptr, *Qnd = nullptr, *Dl = nullptr, *Uw = nullptr;
  double *zs = nullptr, *ds = nullptr, *dlam = nullptr, *wv = nullptr, *what = nullptr, *lam = nullptr;
  double *dfv = nullptr, *rotcs = nullptr, *rho = nullptr, *splitws = nullptr, *gpart = nullptr;
  int* gcnt = nullptr;
  double *Vq2 = nullptr, *tq2 = nullptr, *Tq2 = nullptr;  // two-stage: stage-2 reflectors, τ, group T
  cudaStream_t st2 = nullptr;  // two-stage: look-ahead stream
  // back-transform T factors, computed on st_t beside the tridiagonal eigensolve (ormtr only waits)
  double *Tall = nullptr, *Sside = nullptr, *ws_t = nullptr, *VT = nullptr;  // VT = V·T per block (ormtr layout)
  cudaStream_t st_t = nullptr;
  cudaEvent_t ev_t0 = nullptr, ev_t1 = nullptr;
  void ensure_tfactors();
  // grid-resident sytrd mid kernel: tagged exchange slots, launch sequence number, error flag
  void* mid_x = nullptr;
  int *mid_err = nullptr, *mid_err_host = nullptr;
  unsigned* mid_resident = nullptr;  // host-mapped: the kernel's epoch once every CTA is resident
  unsigned long long mid_seq = 0;
  bool mid_used = false;
  void ensure_mid();
  cudaEvent_t ev_panel[8] = {};  // panel-loop throttle of the background chains
  void ensure_panel_events();
  cudaEvent_t ev_w = nullptr, ev_rest = nullptr;
  long splitws_cap = 0;
  const std::atomic<bool>* cancel = nullptr;  // set: throw Cancelled at the next panel boundary
  void check_cancel(cudaStream_t st) const {
    if (cancel && cancel->load(std::memory_order_relaxed)) {
      cudaStreamSynchronize(st);  // in-flight grids retire before any gate slot is released
      if (st2) cudaStreamSynchronize(st2);
      if (st_t) cudaStreamSynchronize(st_t);
      throw Cancelled{};
    }
  }
  int* ibuf = nullptr;
  void* dbuf = nullptr;
  int* hbuf = nullptr;
  explicit EigWork(int n);
  void ensure_two_stage();
  ~EigWork();
  EigWork(const EigWork&) = delete;
  EigWork& operator=(const EigWork&) = delete;
};
// Z symmetric (n×n, row-major, device).  Outputs: P (columns = eigenvectors,
// descending eigenvalues), vals (descending), *dk = #(vals > 0).
// lane: 0 = latency-critical caller (always keeps a co-residency slot), 1 = background.
// two-stage tridiagonalisation (eig2.cu): Z → (w.d, w.e), stage-1 reflectors in
// w.Vall/w.tau (ormtr layout), stage-2 reflectors in w.Vq2/w.tq2
long two_stage_q2_size(int n);
long two_stage_t_size(int n);
void two_stage_tridiag(const double* Z, int n, EigWork& w, cudaStream_t st);
void two_stage_q2_apply(int n, EigWork& w, double* P, cudaStream_t st,
                        const int* dcols = nullptr);  // P ← Q2 P (first *dcols columns if set)
bool use_two_stage(int n, int lane);
// +1 / −1 when an EG pipeline starts / stops (panel grid sizing for three concurrent chains)
void eig_pipeline_active(int delta);
// tridiagonal form only (debug/tests): stages = 1 (one-stage sytrd) or 2
void tridiag_device(const double* Z, int n, EigWork& w, cudaStream_t st, int stages);
// alpha_only: only the eigenvectors of σ > 0 (the first *dk columns) are back-transformed — enough
// for the PSD projection; the other columns of P are left unspecified.
void syevd_device(const double* Z, int n, double* P, double* vals, int* dk, EigWork& w, cudaStream_t st,
                  int lane = 0, bool alpha_only = false);

}  // namespace kot
