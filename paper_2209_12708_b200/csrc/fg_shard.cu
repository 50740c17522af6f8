// fg_shard.cu -- the all-reduce behind the column-sharded pass.
//
//   * NCCL: ncclAllReduce of the concretization partials over NVLink/NVSwitch, stream-ordered
//     on the pass stream (CUDA-graph capturable).  libnccl.so.2 is loaded on first use, so the
//     library has no link-time NCCL dependency (torch's copy is reused when already loaded).
//   * loopback: `nranks` models on ONE device driven by one host thread each; the reduction
//     is a rank-ordered kernel between CUDA events (deterministic, identical on every rank).
//     It exercises the sharded pass on a single GPU; it is not a throughput path.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "fg_host.h"

using fgh::DBuf;
using fgh::fail;

// ---- NCCL (run-time loaded) ------------------------------------------------------------------
namespace {

typedef struct {
  char internal[128];
} NcclUid;
typedef void* NcclComm;
enum { kNcclDouble = 8, kNcclSum = 0, kNcclMax = 2 };

struct NcclApi {
  void* h = nullptr;
  int (*get_unique_id)(NcclUid*) = nullptr;
  int (*comm_init_rank)(NcclComm*, int, NcclUid, int) = nullptr;
  int (*all_reduce)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
  int (*comm_destroy)(NcclComm) = nullptr;
  const char* (*error_string)(int) = nullptr;
  bool ok() const { return all_reduce != nullptr; }
};

NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    // RTLD_LOCAL: when torch has already loaded its bundled NCCL this resolves to that same
    // library (matched by soname); otherwise the copy found here must not export its symbols
    // globally, or a later `import torch` binds libtorch_cuda against it (a different NCCL
    // version: missing symbols at import time).
    const char* path = std::getenv("FG_NCCL_LIB");  // an explicit libnccl (e.g. the one torch bundles)
    if (path && path[0]) a.h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
    if (!a.h) a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!a.h) return a;
    a.get_unique_id = (int (*)(NcclUid*))dlsym(a.h, "ncclGetUniqueId");
    a.comm_init_rank = (int (*)(NcclComm*, int, NcclUid, int))dlsym(a.h, "ncclCommInitRank");
    a.comm_destroy = (int (*)(NcclComm))dlsym(a.h, "ncclCommDestroy");
    a.error_string = (const char* (*)(int))dlsym(a.h, "ncclGetErrorString");
    a.all_reduce = (int (*)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t))dlsym(a.h, "ncclAllReduce");
    if (!a.get_unique_id || !a.comm_init_rank || !a.comm_destroy) a.all_reduce = nullptr;
    return a;
  }();
  return api;
}

struct NcclEndpoint {
  NcclComm comm = nullptr;
  ~NcclEndpoint() {
    if (comm) nccl().comm_destroy(comm);
  }
};

int nccl_allreduce(void* user, double* buf, size_t count, int op, void* stream) {
  auto* ep = static_cast<NcclEndpoint*>(user);
  return nccl().all_reduce(buf, buf, count, kNcclDouble, op == FG_REDUCE_MAX ? kNcclMax : kNcclSum, ep->comm,
                           (cudaStream_t)stream);
}

}  // namespace

namespace fgh {

fg_status nccl_unique_id(unsigned char id[128], std::string& err) {
  if (!nccl().ok()) {
    err = "libnccl.so.2 not loadable";
    return FG_ECUDA;
  }
  NcclUid u;
  int r = nccl().get_unique_id(&u);
  if (r != 0) {
    err = std::string("ncclGetUniqueId: ") + nccl().error_string(r);
    return FG_ECUDA;
  }
  std::memcpy(id, u.internal, 128);
  return FG_OK;
}

fg_status nccl_exchange(int rank, int nranks, const unsigned char id[128], ShardState& out, std::string& err) {
  if (!nccl().ok()) {
    err = "libnccl.so.2 not loadable";
    return FG_ECUDA;
  }
  auto ep = std::make_shared<NcclEndpoint>();
  NcclUid u;
  std::memcpy(u.internal, id, 128);
  int r = nccl().comm_init_rank(&ep->comm, nranks, u, rank);
  if (r != 0) {
    ep->comm = nullptr;
    err = std::string("ncclCommInitRank: ") + nccl().error_string(r);
    return FG_ECUDA;
  }
  out.rank = rank;
  out.nranks = nranks;
  out.fn = nccl_allreduce;
  out.user = ep.get();
  out.capturable = true;
  out.owned = ep;
  return FG_OK;
}

}  // namespace fgh

// ---- loopback group ------------------------------------------------------------------------
namespace {

constexpr int kMaxLoop = 16;
struct Ptrs {
  const double* p[kMaxLoop];
};

__global__ void combine_kernel(Ptrs in, int n, size_t count, int op, double* out) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double v = in.p[0][i];
  for (int q = 1; q < n; ++q) v = op == FG_REDUCE_MAX ? fmax(v, in.p[q][i]) : v + in.p[q][i];
  out[i] = v;
}

}  // namespace

struct fg_loopback {
  int n = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long generation = 0;
  std::vector<double*> bufs;
  std::vector<cudaEvent_t> ev1, ev2;
  std::vector<DBuf> tmp;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    long long gen = generation;
    if (++arrived == n) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

namespace {

struct LoopRank {
  fg_loopback* g;
  int rank;
};

int loop_allreduce(void* user, double* buf, size_t count, int op, void* stream_) {
  auto* lr = static_cast<LoopRank*>(user);
  fg_loopback* g = lr->g;
  const int r = lr->rank;
  cudaStream_t st = (cudaStream_t)stream_;
  g->bufs[r] = buf;
  if (cudaEventRecord(g->ev1[r], st) != cudaSuccess) return 1;
  g->barrier();
  for (int q = 0; q < g->n; ++q)
    if (q != r) cudaStreamWaitEvent(st, g->ev1[q], 0);
  if (g->tmp[r].bytes < count * sizeof(double) && g->tmp[r].alloc(count * sizeof(double)) != cudaSuccess) return 1;
  Ptrs p{};
  for (int q = 0; q < g->n; ++q) p.p[q] = g->bufs[q];
  if (count) combine_kernel<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(p, g->n, count, op, g->tmp[r].as<double>());
  cudaEventRecord(g->ev2[r], st);
  g->barrier();  // every rank's combine has been enqueued behind its inputs
  for (int q = 0; q < g->n; ++q)
    if (q != r) cudaStreamWaitEvent(st, g->ev2[q], 0);
  if (count) cudaMemcpyAsync(buf, g->tmp[r].p, count * sizeof(double), cudaMemcpyDeviceToDevice, st);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace

extern "C" {

fg_status fg_nccl_unique_id(unsigned char id[128]) {
  std::string err;
  return fgh::nccl_unique_id(id, err);
}

fg_status fg_loopback_create(int nranks, fg_loopback** out) {
  *out = nullptr;
  if (nranks < 1 || nranks > kMaxLoop) return FG_EINVAL;
  auto g = new fg_loopback();
  g->n = nranks;
  g->bufs.assign(nranks, nullptr);
  g->ev1.resize(nranks);
  g->ev2.resize(nranks);
  g->tmp.resize(nranks);
  for (int q = 0; q < nranks; ++q) {
    if (cudaEventCreateWithFlags(&g->ev1[q], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&g->ev2[q], cudaEventDisableTiming) != cudaSuccess) {
      delete g;
      return FG_ECUDA;
    }
  }
  *out = g;
  return FG_OK;
}

void fg_loopback_destroy(fg_loopback* g) {
  if (!g) return;
  for (auto e : g->ev1) cudaEventDestroy(e);
  for (auto e : g->ev2) cudaEventDestroy(e);
  delete g;
}

}  // extern "C"

namespace fgh {

fg_status loopback_exchange(fg_loopback* g, int rank, ShardState& out) {
  if (!g || rank < 0 || rank >= g->n) return FG_EINVAL;
  auto lr = std::make_shared<LoopRank>(LoopRank{g, rank});
  out.rank = rank;
  out.nranks = g->n;
  out.fn = loop_allreduce;
  out.user = lr.get();
  out.capturable = false;  // host barriers between the enqueues
  out.ranks_per_device = g->n;
  out.owned = lr;
  return FG_OK;
}

}  // namespace fgh
