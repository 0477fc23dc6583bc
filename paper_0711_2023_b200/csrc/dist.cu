// dist.cu -- multi-GPU plumbing for the sharded sweep:
// NCCL loaded on demand (dlopen of libnccl.so.2: the one torch already loaded
// when the caller imported it; a single-GPU process never needs it), the
// collectives the sweep uses, and the contiguous work-balanced shard bounds.
//
// Exchange steps (one per mode, all sums of disjoint or partial terms):
//   HOOI, Y Y^T route: rows of Y_(n) are disjoint across ranks -> allgatherv Y
//   HOOI, Y^T Y route: partial Gram over the rank's K range -> allreduce S (fp64);
//                      rows of U = Y V Theta^{-1/2} disjoint -> allgatherv U
//   HOOI core:         G = U_N^T Y_(N) partial when Y was not gathered -> allreduce G
//   MP:                partial M_n over the rank's slices -> allreduce M_n (fp64)
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <string>

#include "internal.cuh"

namespace tk {
namespace {

struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& api() {
  static NcclApi a;
  if (!a.lib) {
    // an NCCL already in the process (e.g. torch's) is reused through its soname;
    // TUCKER_NCCL_LIB names a specific library otherwise
    const char* path = std::getenv("TUCKER_NCCL_LIB");
    void* l = dlopen(path && *path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!l) fail(TUCKER_E_NCCL, std::string("cannot load NCCL: ") + dlerror());
    auto sym = [&](const char* n) {
      void* p = dlsym(l, n);
      if (!p) fail(TUCKER_E_NCCL, std::string("libnccl.so.2 lacks ") + n);
      return p;
    };
    a.GetUniqueId = (decltype(a.GetUniqueId))sym("ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))sym("ncclCommInitRank");
    a.AllReduce = (decltype(a.AllReduce))sym("ncclAllReduce");
    a.Broadcast = (decltype(a.Broadcast))sym("ncclBroadcast");
    a.GroupStart = (decltype(a.GroupStart))sym("ncclGroupStart");
    a.GroupEnd = (decltype(a.GroupEnd))sym("ncclGroupEnd");
    a.CommDestroy = (decltype(a.CommDestroy))sym("ncclCommDestroy");
    a.GetErrorString = (decltype(a.GetErrorString))sym("ncclGetErrorString");
    a.lib = l;
  }
  return a;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(TUCKER_E_NCCL, std::string(what) + ": " + api().GetErrorString(r));
}

}  // namespace

// A handle's communicator: NCCL, or (TUCKER_HOST_COLLECTIVES) a host callback
// int fn(void* dev_buf, int64_t count, int dtype, void* stream, void* user)
// that sums dev_buf over the ranks in place (dtype 0 = fp32, 1 = fp64), called
// after the library's stream is synchronised.
struct DistComm {
  ncclComm_t nccl = nullptr;
  int (*cb)(void*, int64_t, int, void*, void*) = nullptr;
  void* user = nullptr;
};

void* dist_comm_init(const void* unique_id, int world, int rank) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  auto* c = new DistComm;
  try {
    check(api().CommInitRank(&c->nccl, world, id, rank), "ncclCommInitRank");
  } catch (...) {
    delete c;
    throw;
  }
  return c;
}

void* dist_comm_host() { return new DistComm; }

void dist_comm_set_callback(void* comm, void* fn, void* user) {
  auto* c = static_cast<DistComm*>(comm);
  c->cb = reinterpret_cast<int (*)(void*, int64_t, int, void*, void*)>(fn);
  c->user = user;
}

void dist_comm_destroy(void* comm) {
  auto* c = static_cast<DistComm*>(comm);
  if (!c) return;
  if (c->nccl) api().CommDestroy(c->nccl);
  delete c;
}

static void allreduce(void* comm, void* p, int64_t n, int dtype, cudaStream_t st) {
  auto* c = static_cast<DistComm*>(comm);
  if (n <= 0) return;
  if (c->nccl) {
    check(api().AllReduce(p, p, (size_t)n, dtype ? ncclFloat64 : ncclFloat32, ncclSum, c->nccl, st),
          "ncclAllReduce");
    return;
  }
  if (!c->cb) fail(TUCKER_E_STATE, "host collectives: no allreduce callback (tucker_set_allreduce)");
  TK_CUDA(cudaStreamSynchronize(st));
  if (c->cb(p, n, dtype, (void*)st, c->user) != 0) fail(TUCKER_E_NCCL, "host allreduce callback failed");
  // the callback may write the result back on any stream (e.g. a pageable
  // cudaMemcpy, whose DMA can still be in flight when it returns): wait for the
  // whole device before the handle's stream reads the buffer
  TK_CUDA(cudaDeviceSynchronize());
}

// Every rank owns the contiguous element range [off[r], off[r + 1]) of `base` and
// receives everybody's: one ncclBroadcast per rank, rooted at the owner, in place, in
// one NCCL group (an allgather with unequal counts; each byte crosses the fabric once,
// half of what an allreduce of the zero-padded buffer moves).  Host collectives: the
// other ranks' ranges are zero in this rank's buffer, so the allreduce callback is the
// same gather.
static void allgatherv(void* comm, void* base, const int64_t* off, int world, int dtype, cudaStream_t st) {
  auto* c = static_cast<DistComm*>(comm);
  if (!c->nccl) {
    allreduce(comm, (char*)base + off[0] * (dtype ? 8 : 4), off[world] - off[0], dtype, st);
    return;
  }
  const size_t es = dtype ? 8 : 4;
  check(api().GroupStart(), "ncclGroupStart");
  for (int r = 0; r < world; ++r) {
    const int64_t n = off[r + 1] - off[r];
    if (n <= 0) continue;
    void* p = (char*)base + off[r] * es;
    check(api().Broadcast(p, p, (size_t)n, dtype ? ncclFloat64 : ncclFloat32, r, c->nccl, st), "ncclBroadcast");
  }
  check(api().GroupEnd(), "ncclGroupEnd");
}
void dist_allgatherv_f32(void* comm, float* base, const int64_t* off, int world, cudaStream_t st) {
  allgatherv(comm, base, off, world, 0, st);
}
void dist_allgatherv_f64(void* comm, double* base, const int64_t* off, int world, cudaStream_t st) {
  allgatherv(comm, base, off, world, 1, st);
}

void dist_allreduce_f32(void* comm, float* p, int64_t n, cudaStream_t st) { allreduce(comm, p, n, 0, st); }
void dist_allreduce_f64(void* comm, double* p, int64_t n, cudaStream_t st) { allreduce(comm, p, n, 1, st); }

void dist_unique_id(void* out) {
  ncclUniqueId id;
  check(api().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof(id));
}

// Contiguous shard bounds over n items with nonnegative work w: bounds[0] = 0,
// bounds[world] = n, bounds[r] = the first index whose work prefix reaches
// r / world of the total (ties and zero work go to the lower rank); empty
// shards are allowed (more ranks than items, or one item heavier than a share).
void shard_bounds(const double* w, int64_t n, int world, int64_t* bounds) {
  double total = 0;
  for (int64_t i = 0; i < n; ++i) total += w[i];
  bounds[0] = 0;
  int64_t i = 0;
  double prefix = 0;
  for (int r = 1; r < world; ++r) {
    const double target = total * (double)r / (double)world;
    while (i < n && prefix + 0.5 * w[i] < target) prefix += w[i++];
    bounds[r] = i;
  }
  bounds[world] = n;
}

}  // namespace tk
