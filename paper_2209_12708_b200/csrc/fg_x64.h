// fg_x64.h -- device-resident f64 bound tensors in the reference layout and the exact-mode
// building blocks shared by the operator entries (fg_ops64.cu) and the graph executor
// (fg_graph.cu).  Internal to the library.
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <string>

#include "fg_host.h"
#include "fg_internal.cuh"

namespace fgx {

using namespace fg;
using fgh::DBuf;
using fgh::fail;

#define XL(expr)                                                                         \
  do {                                                                                   \
    ctx->launches += (uint64_t)(expr);                                                   \
    cudaError_t e_ = cudaGetLastError();                                                 \
    if (e_ != cudaSuccess)                                                               \
      return fail(ctx, FG_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));    \
  } while (0)

inline bool eps_ok(double eps) { return eps >= 0.0 && std::isfinite(eps); }  // bounds.cpp:38-44

// One bound tensor in the reference layout on the device.
struct XB {
  DBuf lw, lb, uw, ub;
  size_t n = 0, d = 0;
  double* plw() const { return lw.as<double>(); }
  double* plb() const { return lb.as<double>(); }
  double* puw() const { return uw.as<double>(); }
  double* pub() const { return ub.as<double>(); }
};

inline fg_status xb_alloc(fg_ctx* ctx, XB& b, size_t n, size_t d) {
  b.n = n;
  b.d = d;
  CK(b.lw.alloc_async(sizeof(double) * n * d, ctx->stream));
  CK(b.uw.alloc_async(sizeof(double) * n * d, ctx->stream));
  CK(b.lb.alloc_async(sizeof(double) * n, ctx->stream));
  CK(b.ub.alloc_async(sizeof(double) * n, ctx->stream));
  return FG_OK;
}

inline fg_status xb_upload(fg_ctx* ctx, XB& b, size_t n, size_t d, const double* lw, const double* lb, const double* uw,
                    const double* ub) {
  if (fg_status s = xb_alloc(ctx, b, n, d)) return s;
  if (n * d) {
    CK(cudaMemcpyAsync(b.lw.p, lw, sizeof(double) * n * d, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(b.uw.p, uw, sizeof(double) * n * d, cudaMemcpyHostToDevice, ctx->stream));
  }
  if (n) {
    CK(cudaMemcpyAsync(b.lb.p, lb, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(b.ub.p, ub, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  }
  return FG_OK;
}

inline fg_status xb_download(fg_ctx* ctx, const XB& b, double* lw, double* lb, double* uw, double* ub) {
  if (b.n * b.d) {
    CK(cudaMemcpyAsync(lw, b.lw.p, sizeof(double) * b.n * b.d, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(uw, b.uw.p, sizeof(double) * b.n * b.d, cudaMemcpyDeviceToHost, ctx->stream));
  }
  if (b.n) {
    CK(cudaMemcpyAsync(lb, b.lb.p, sizeof(double) * b.n, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(ub, b.ub.p, sizeof(double) * b.n, cudaMemcpyDeviceToHost, ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return FG_OK;
}

// Device status word for envelope checks (kStatusClear / site<<4|code, fg_internal.cuh).
inline fg_status x_status(fg_ctx* ctx, int* dstatus, const char* what) {
  int v = kStatusClear;
  CK(cudaMemcpyAsync(&v, dstatus, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (v == kStatusClear) return FG_OK;
  if ((v & 15) == kCodeInval) return fail(ctx, FG_EINVAL, std::string(what) + ": lo > hi (ConcreteBounds::validate)");
  return fail(ctx, FG_EDOMAIN, std::string(what) + ": relaxation domain / overflow");
}

// concretize on the device, result stays on the device
inline fg_status x_conc(fg_ctx* ctx, const XB& x, int norm, double eps, DBuf& lo, DBuf& hi) {
  CK(lo.alloc_async(sizeof(double) * x.n, ctx->stream));
  CK(hi.alloc_async(sizeof(double) * x.n, ctx->stream));
  XL(launch_x_concretize(x.plw(), x.plb(), x.puw(), x.pub(), (long long)x.n, (int)x.d, norm, eps,
                         lo.as<double>(), hi.as<double>(), ctx->stream));
  return FG_OK;
}

// relax_<kind> + compose_elementwise on device-resident operands (graph.cpp:484-501 order)
inline fg_status x_relax_compose(fg_ctx* ctx, int kind, const XB& x, const DBuf& lo, const DBuf& hi, XB& y,
                          const char* what) {
  DBuf lines, st;
  CK(lines.alloc_async(sizeof(double) * 4 * x.n, ctx->stream));
  CK(st.alloc_async(sizeof(int), ctx->stream));
  XL(launch_fill_int(st.as<int>(), kStatusClear, 1, ctx->stream));
  double* l = lines.as<double>();
  XL(launch_relax(kind, lo.as<double>(), hi.as<double>(), (long long)x.n, l, l + x.n, l + 2 * x.n, l + 3 * x.n,
                  st.as<int>(), ctx->stream));
  if (fg_status s = x_status(ctx, st.as<int>(), what)) return s;
  if (fg_status s = xb_alloc(ctx, y, x.n, x.d)) return s;
  XL(launch_x_compose(x.plw(), x.plb(), x.puw(), x.pub(), l, l + x.n, l + 2 * x.n, l + 3 * x.n, y.plw(), y.plb(),
                      y.puw(), y.pub(), (long long)x.n, (int)x.d, ctx->stream));
  return FG_OK;
}

inline fg_status x_sum_axis(fg_ctx* ctx, const XB& x, size_t outer, size_t n, size_t inner, XB& y) {
  if (fg_status s = xb_alloc(ctx, y, outer * inner, x.d)) return s;
  XL(launch_x_sum_axis(x.plw(), x.plb(), x.puw(), x.pub(), y.plw(), y.plb(), y.puw(), y.pub(), (long long)outer,
                       (int)n, (long long)inner, (int)x.d, ctx->stream));
  return FG_OK;
}

inline fg_status x_mul_broadcast(fg_ctx* ctx, const XB& x, const XB& r, size_t outer, size_t n, size_t inner, int norm,
                          double eps, XB& y) {
  DBuf xlo, xhi, rlo, rhi;
  if (fg_status s = x_conc(ctx, x, norm, eps, xlo, xhi)) return s;
  if (fg_status s = x_conc(ctx, r, norm, eps, rlo, rhi)) return s;
  if (fg_status s = xb_alloc(ctx, y, x.n, x.d)) return s;
  XDotArgs a{x.plw(), x.plb(), x.puw(), x.pub(), xlo.as<double>(),
             r.plw(), r.plb(), r.puw(), r.pub(), rlo.as<double>(), rhi.as<double>(),
             y.plw(), y.plb(), y.puw(), y.pub(), 0, 1, 0, 0, 1, (int)x.d};
  XL(launch_x_mul_broadcast(a, (long long)outer, (int)n, (long long)inner, ctx->stream));
  return FG_OK;
}


}  // namespace fgx
