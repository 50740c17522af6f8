// fg_host.h -- host-side internals shared by the C-ABI translation units (fg_host.cu,
// fg_ops64.cu): the context object, error plumbing and an RAII device buffer.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "../../include/faith_gpu.h"

struct fg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  uint64_t launches = 0;
  int precision = FG_PRECISION_F32;  // operator-level arithmetic (fg_ctx_set_precision)
};

namespace fgh {

// Column (perturbation-dimension) sharding of a model's passes (fg_model_set_column_shard):
// this rank owns columns [rank*D/nranks, (rank+1)*D/nranks) of every Λ; concretization
// partials are all-reduced through `fn` (stream-ordered on the pass stream).
struct ShardState {
  int rank = 0, nranks = 1;
  fg_allreduce_fn fn = nullptr;
  void* user = nullptr;
  bool capturable = true;       // fn may be captured into a CUDA graph (NCCL: yes)
  int ranks_per_device = 1;     // loopback: all ranks share one device's HBM
  std::shared_ptr<void> owned;  // communicator / loopback endpoint kept alive with the model
  bool active() const { return fn != nullptr; }
};

// built-in exchanges (fg_shard.cu)
fg_status nccl_exchange(int rank, int nranks, const unsigned char id[128], ShardState& out, std::string& err);
fg_status nccl_unique_id(unsigned char id[128], std::string& err);
fg_status loopback_exchange(fg_loopback* group, int rank, ShardState& out);

inline fg_status fail(fg_ctx* ctx, fg_status code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

// RAII device allocation.  alloc(): cudaMalloc.  alloc_async(): stream-ordered from the
// device's default memory pool (cudaMallocAsync / cudaFreeAsync on that stream): no device-wide
// synchronisation on free, so the exact-mode paths (many short-lived f64 tensors) do not stall.
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t stream = nullptr;
  bool pooled = false;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), bytes(o.bytes), stream(o.stream), pooled(o.pooled) {
    o.p = nullptr;
    o.bytes = 0;
    o.pooled = false;
  }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      reset();
      p = o.p;
      bytes = o.bytes;
      stream = o.stream;
      pooled = o.pooled;
      o.p = nullptr;
      o.bytes = 0;
      o.pooled = false;
    }
    return *this;
  }
  ~DBuf() { reset(); }
  void reset() {
    if (p) {
      if (pooled) cudaFreeAsync(p, stream);
      else cudaFree(p);
    }
    p = nullptr;
    bytes = 0;
    pooled = false;
  }
  cudaError_t alloc(size_t b) {
    reset();
    bytes = b ? b : 16;
    return cudaMalloc(&p, bytes);
  }
  cudaError_t alloc_async(size_t b, cudaStream_t st) {
    reset();
    bytes = b ? b : 16;
    stream = st;
    cudaError_t e = cudaMallocAsync(&p, bytes, st);
    pooled = e == cudaSuccess;
    return e;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// f64 operator level of the exact precision mode (fg_ops64.cu); same contracts as the
// extern "C" entries that dispatch to them.
fg_status x64_concretize(fg_ctx* ctx, size_t n, size_t d, const double* lw, const double* lb, const double* uw,
                         const double* ub, int norm, double eps, double* lo, double* hi);
fg_status x64_affine(fg_ctx* ctx, size_t rows, size_t c, size_t o, size_t d, const double* xlw, const double* xlb,
                     const double* xuw, const double* xub, const double* w, const double* bias, double* ylw,
                     double* ylb, double* yuw, double* yub);
fg_status x64_compose(fg_ctx* ctx, size_t n, size_t d, const double* xlw, const double* xlb, const double* xuw,
                      const double* xub, const double* a_low, const double* b_low, const double* a_up,
                      const double* b_up, double* ylw, double* ylb, double* yuw, double* yub);
fg_status x64_elementwise_verify(fg_ctx* ctx, int kind, size_t n, size_t d, const double* xlw, const double* xlb,
                                 const double* xuw, const double* xub, int norm, double eps, double* ylw,
                                 double* ylb, double* yuw, double* yub);
fg_status x64_dot(fg_ctx* ctx, int layout, size_t batch, size_t len, size_t embed, size_t heads, size_t d,
                  const double* alw, const double* alb, const double* auw, const double* aub, const double* blw,
                  const double* blb, const double* buw, const double* bub, int norm, double eps, double* ylw,
                  double* ylb, double* yuw, double* yub);
fg_status x64_softmax(fg_ctx* ctx, size_t outer, size_t n, size_t inner, size_t d, const double* xlw,
                      const double* xlb, const double* xuw, const double* xub, int norm, double eps, double* ylw,
                      double* ylb, double* yuw, double* yub);
fg_status x64_add(fg_ctx* ctx, size_t n, size_t d, const double* alw, const double* alb, const double* auw,
                  const double* aub, const double* blw, const double* blb, const double* buw, const double* bub,
                  double* ylw, double* ylb, double* yuw, double* yub);
fg_status x64_scale(fg_ctx* ctx, size_t n, size_t d, const double* xlw, const double* xlb, const double* xuw,
                    const double* xub, double s, double* ylw, double* ylb, double* yuw, double* yub);

// An exact pass running asynchronously on a side stream (fg_maxeps' re-decisions overlap the
// fused passes): results land in pinned host memory, `done` is recorded after them.
struct ExactJob {
  double* host = nullptr;  // logits lo [classes], hi [classes]
  int* hstat = nullptr;    // relaxation-site status words [nsites], then the non-finite flag
  int nsites = 0, classes = 0;
  cudaEvent_t start = nullptr, done = nullptr;
  int sentence = -1;
  double eps = 0.0;
  bool busy = false;
  std::vector<double> lo32, hi32;  // the fused pass's logits bounds of the probe (calibration)
};

// The word-level pass of one sentence in the exact precision mode (fg_exact_pass.cu).  With
// `job`, nothing is waited for: the results and statuses are copied into the job's pinned
// buffers on ctx->stream and `job->done` is recorded (`status` / `logits_*` unused).
fg_status exact_pass(fg_ctx* ctx, const fg_config& c, const double* params_dev, const double* x_host,
                     const int* pos_host, int words, int norm, double eps, double* logits_lo, double* logits_hi,
                     double* node_lo, double* node_hi, int* status, ExactJob* job = nullptr);

}  // namespace fgh

#define CK(expr)                                                                             \
  do {                                                                                       \
    cudaError_t e_ = (expr);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      return fgh::fail(ctx, FG_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));   \
  } while (0)
