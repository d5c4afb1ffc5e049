// Phase profiler: CUDA events recorded around library phases on the launching
// stream (enabled by kot_profile_enable; zero cost when off).  Backs the
// live per-kernel timing and roofline numbers of bench.py.
#pragma once
#include "common.cuh"

namespace kot {

bool prof_enabled();
// the calling thread is capturing a CUDA graph: scopes are skipped (their events would be graph nodes)
inline bool& prof_capturing() {
  static thread_local bool c = false;
  return c;
}
// open a scope: returns a token (or -1 when disabled)
int prof_begin(const char* name, cudaStream_t st);
void prof_end(int token, cudaStream_t st, double flops, double bytes = 0.0);
// host-side wall time (e.g. the solve loop waiting for the EG pipeline)
void prof_host(const char* name, double ms);

struct ProfScope {
  int tok;
  cudaStream_t st;
  double flops, bytes;
  ProfScope(const char* name, cudaStream_t s, double f = 0.0, double b = 0.0)
      : tok(prof_enabled() && !prof_capturing() ? prof_begin(name, s) : -1), st(s), flops(f), bytes(b) {}
  ~ProfScope() {
    if (tok >= 0) prof_end(tok, st, flops, bytes);
  }
};

}  // namespace kot
