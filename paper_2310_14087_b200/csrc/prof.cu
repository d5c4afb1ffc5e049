#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/kotgpu.h"
#include "prof.cuh"

namespace kot {

namespace {
struct Entry {
  std::string name;
  long long calls = 0;
  double ms = 0.0, flops = 0.0, bytes = 0.0;
};
struct Pending {
  cudaEvent_t a, b;
  int entry;
  double flops, bytes;
};
std::mutex g_mu;
bool g_on = false;
std::vector<Entry> g_entries;
std::vector<Pending> g_open;     // indexed by token
std::vector<Pending> g_pending;  // closed, not yet resolved

int entry_of(const char* name) {
  for (size_t i = 0; i < g_entries.size(); ++i)
    if (g_entries[i].name == name) return (int)i;
  g_entries.push_back(Entry{name});
  return (int)g_entries.size() - 1;
}

void resolve_locked() {
  for (auto& p : g_pending) {
    cudaEventSynchronize(p.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p.a, p.b);
    g_entries[p.entry].ms += ms;
    g_entries[p.entry].flops += p.flops;
    g_entries[p.entry].bytes += p.bytes;
    g_entries[p.entry].calls += 1;
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  g_pending.clear();
}
}  // namespace

bool prof_enabled() { return g_on; }

int prof_begin(const char* name, cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_mu);
  Pending p{};
  p.entry = entry_of(name);
  cudaEventCreate(&p.a);
  cudaEventCreate(&p.b);
  cudaEventRecord(p.a, st);
  g_open.push_back(p);
  return (int)g_open.size() - 1;
}

void prof_end(int tok, cudaStream_t st, double flops, double bytes) {
  std::lock_guard<std::mutex> lk(g_mu);
  Pending p = g_open[tok];
  p.flops = flops;
  p.bytes = bytes;
  cudaEventRecord(p.b, st);
  g_pending.push_back(p);
  if (g_pending.size() > 4096) resolve_locked();
}

void prof_host(const char* name, double ms) {
  if (!g_on) return;
  std::lock_guard<std::mutex> lk(g_mu);
  Entry& e = g_entries[entry_of(name)];
  e.ms += ms;
  e.calls += 1;
}

}  // namespace kot

extern "C" int kot_profile_enable(int on) {
  std::lock_guard<std::mutex> lk(kot::g_mu);
  kot::resolve_locked();
  kot::g_entries.clear();
  kot::g_open.clear();
  kot::g_on = on != 0;
  return 0;
}

extern "C" int kot_profile_read(kot_prof_entry* out, int cap) {
  std::lock_guard<std::mutex> lk(kot::g_mu);
  kot::resolve_locked();
  int n = 0;
  for (auto& e : kot::g_entries) {
    if (n >= cap) break;
    std::memset(&out[n], 0, sizeof(kot_prof_entry));
    std::strncpy(out[n].name, e.name.c_str(), sizeof(out[n].name) - 1);
    out[n].calls = e.calls;
    out[n].ms = e.ms;
    out[n].flops = e.flops;
    out[n].bytes = e.bytes;
    ++n;
  }
  return n;
}
