// Row-sharded structure-reduced CG matvec over NCCL (BASELINE config 4, ℓ=8192;
// SURVEY.md §8(e)): rank g owns the row block [r0, r1) of B = R·P.
//   T̃ = W∘(B_αᵀ diag(v) B) = Σ_g W∘(B_{g,α}ᵀ diag(v_g) B_g)   → ncclAllReduce (k×ℓ doubles)
//   y_i = Σ_a (B T̃ᵀ)_ia B_ia   for own rows i                 → ncclAllGather  (ℓ doubles)
// CG vectors stay replicated, so every rank takes identical control decisions.
// NCCL is dlopen'ed (after torch.distributed has loaded its own libnccl), never linked.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

#include "ssn.cuh"

namespace kot {

namespace {
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};
NcclApi g_nccl;
std::once_flag g_nccl_once;

const NcclApi& nccl() {
  std::call_once(g_nccl_once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))dlsym(h, "ncclCommInitRank");
    g_nccl.AllReduce = (decltype(g_nccl.AllReduce))dlsym(h, "ncclAllReduce");
    g_nccl.AllGather = (decltype(g_nccl.AllGather))dlsym(h, "ncclAllGather");
    g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))dlsym(h, "ncclCommDestroy");
    g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))dlsym(h, "ncclGetErrorString");
    g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.AllReduce && g_nccl.AllGather &&
                g_nccl.CommDestroy && g_nccl.GetErrorString;
  });
  kot_require(g_nccl.ok, KOT_ECUDA, "libnccl.so.2 could not be loaded (row sharding needs NCCL)");
  return g_nccl;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw KotError(KOT_ECUDA, std::string(what) + ": " + nccl().GetErrorString(r));
}
}  // namespace

void nccl_unique_id(char* out128) {
  ncclUniqueId id;
  nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  memcpy(out128, &id, 128);
}

void problem_shard(Problem& p, const char* id128, int rank, int world) {
  kot_require(world >= 1 && rank >= 0 && rank < world, KOT_EINVAL, "invalid rank/world");
  KOT_CUDA(cudaSetDevice(p.device));
  ncclUniqueId id;
  memcpy(&id, id128, 128);
  ncclComm_t comm;
  nccl_check(nccl().CommInitRank(&comm, world, id, rank), "ncclCommInitRank");
  p.nccl_comm = comm;
  p.shard_rank = rank;
  p.shard_world = world;
  p.shard_block = (p.n + world - 1) / world;
  p.row0 = std::min(p.n, rank * p.shard_block);
  p.row1 = std::min(p.n, p.row0 + p.shard_block);
  if (!p.ygather) p.ygather = p.alloc((long)p.shard_block * world);
}

void problem_shard_emulate(Problem& p, int world) {
  kot_require(world >= 1, KOT_EINVAL, "invalid world");
  problem_unshard(p);
  p.emul_world = world;
  if (world > 1 && !p.shard_tmp) p.shard_tmp = p.alloc((long)(p.n / 2 + 1) * p.n);
}

// Host data plane: the caller supplies the two collectives on host buffers (op 0: in-place sum over
// ranks of `count` doubles; op 1: in-place all-gather, rank g's `block` doubles at buf + g·block).
// Same row blocks and arithmetic as the NCCL path; the device data is staged through pinned memory.
void problem_shard_host(Problem& p, int (*fn)(void*, int, double*, long, long, int, int), void* user, int rank,
                        int world) {
  kot_require(fn != nullptr && world >= 1 && rank >= 0 && rank < world, KOT_EINVAL, "invalid rank/world");
  problem_unshard(p);
  p.host_comm = fn;
  p.host_comm_user = user;
  p.shard_rank = rank;
  p.shard_world = world;
  p.shard_block = (p.n + world - 1) / world;
  p.row0 = std::min(p.n, rank * p.shard_block);
  p.row1 = std::min(p.n, p.row0 + p.shard_block);
  if (!p.ygather) p.ygather = p.alloc((long)p.shard_block * world);
  const long cap = std::max((long)p.n * p.n, (long)p.shard_block * world);
  if (p.host_comm_cap < cap) {
    if (p.host_comm_buf) host_free_pinned(p.host_comm_buf, sizeof(double) * p.host_comm_cap);
    p.host_comm_buf = static_cast<double*>(host_alloc_pinned(sizeof(double) * cap));
    p.host_comm_cap = cap;
  }
}

static void host_collective(Problem& p, int op, double* buf, long count, long block, cudaStream_t st) {
  if (p.host_comm_cap < count) {  // the split H form gathers whole row blocks of B
    if (p.host_comm_buf) host_free_pinned(p.host_comm_buf, sizeof(double) * p.host_comm_cap);
    p.host_comm_buf = static_cast<double*>(host_alloc_pinned(sizeof(double) * count));
    p.host_comm_cap = count;
  }
  KOT_CUDA(cudaMemcpyAsync(p.host_comm_buf, buf, sizeof(double) * count, cudaMemcpyDeviceToHost, st));
  KOT_CUDA(cudaStreamSynchronize(st));
  const int rc = p.host_comm(p.host_comm_user, op, p.host_comm_buf, count, block, p.shard_rank, p.shard_world);
  kot_require(rc == 0, KOT_ECUDA, "host data-plane collective failed");
  KOT_CUDA(cudaMemcpyAsync(buf, p.host_comm_buf, sizeof(double) * count, cudaMemcpyHostToDevice, st));
}

void problem_unshard(Problem& p) {
  if (p.nccl_comm) {
    nccl().CommDestroy((ncclComm_t)p.nccl_comm);
    p.nccl_comm = nullptr;
  }
  p.host_comm = nullptr;
  p.host_comm_user = nullptr;
  p.shard_world = 1;
  p.shard_rank = 0;
  p.emul_world = 1;
  p.row0 = 0;
  p.row1 = p.n;
}

// Every rank receives the same sum (NCCL's ring / tree and the host collectives return one result to
// all ranks), so the ranks keep taking identical control decisions.
void shard_allreduce_sum(Problem& p, double* buf, long count, cudaStream_t st) {
  if (p.host_comm) return host_collective(p, 0, buf, count, 0, st);
  nccl_check(nccl().AllReduce(buf, buf, (size_t)count, ncclDouble, ncclSum, (ncclComm_t)p.nccl_comm, st),
             "ncclAllReduce");
}
void shard_allreduce_sum(Problem& p, double* buf, long count) { shard_allreduce_sum(p, buf, count, p.st); }

// in place: rank g's block sits at buf + g·block; afterwards every rank holds all blocks
void shard_allgather(Problem& p, double* buf, long block, cudaStream_t st) {
  if (p.host_comm) return host_collective(p, 1, buf, block * p.shard_world, block, st);
  nccl_check(nccl().AllGather(buf + (long)p.shard_rank * block, buf, (size_t)block, ncclDouble,
                              (ncclComm_t)p.nccl_comm, st),
             "ncclAllGather");
}
void shard_allgather(Problem& p, double* buf, long block) { shard_allgather(p, buf, block, p.st); }

FoldedRows folded_rows(int n, int g, int world) {
  FoldedRows f;
  f.blk = (n + 2 * world - 1) / (2 * world);
  f.a0 = std::min(n, g * f.blk);
  f.a1 = std::min(n, f.a0 + f.blk);
  f.b0 = std::min(n, (2 * world - 1 - g) * f.blk);
  f.b1 = std::min(n, f.b0 + f.blk);
  return f;
}

}  // namespace kot
