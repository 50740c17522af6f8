// fg_ops64.cu -- operator level of the exact precision mode (FG_PRECISION_F64) and the
// operator entries that exist only in f64 (sum_axis, mul_broadcast, bilinear, general-axis
// softmax).  Host f64 buffers in the reference layout are uploaded as-is, run through the
// f64 kernels of fg_exact.cu (reference operation order) and downloaded: value semantics of
// proj/src/relax.cpp and proj/src/bounds.cpp, with their exception taxonomy as fg_status.
#include <cuda_runtime.h>

#include <cmath>
#include <string>
#include <vector>

#include "fg_host.h"
#include "fg_internal.cuh"
#include "fg_x64.h"

using namespace fg;
using fgh::DBuf;
using fgh::fail;

using namespace fgx;

namespace fgh {

fg_status x64_concretize(fg_ctx* ctx, size_t n, size_t d, const double* lw, const double* lb, const double* uw,
                         const double* ub, int norm, double eps, double* lo, double* hi) {
  XB x;
  if (fg_status s = xb_upload(ctx, x, n, d, lw, lb, uw, ub)) return s;
  DBuf dlo, dhi;
  if (fg_status s = x_conc(ctx, x, norm, eps, dlo, dhi)) return s;
  CK(cudaMemcpyAsync(lo, dlo.p, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(hi, dhi.p, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return FG_OK;
}

fg_status x64_affine(fg_ctx* ctx, size_t rows, size_t c, size_t o, size_t d, const double* xlw, const double* xlb,
                     const double* xuw, const double* xub, const double* w, const double* bias, double* ylw,
                     double* ylb, double* yuw, double* yub) {
  XB x, y;
  if (fg_status s = xb_upload(ctx, x, rows * c, d, xlw, xlb, xuw, xub)) return s;
  if (fg_status s = xb_alloc(ctx, y, rows * o, d)) return s;
  DBuf dw, db;
  CK(dw.alloc(sizeof(double) * c * o));
  CK(cudaMemcpyAsync(dw.p, w, sizeof(double) * c * o, cudaMemcpyHostToDevice, ctx->stream));
  if (bias) {
    CK(db.alloc(sizeof(double) * o));
    CK(cudaMemcpyAsync(db.p, bias, sizeof(double) * o, cudaMemcpyHostToDevice, ctx->stream));
  }
  XL(launch_x_affine(x.plw(), x.plb(), x.puw(), x.pub(), dw.as<double>(), bias ? db.as<double>() : nullptr,
                     y.plw(), y.plb(), y.puw(), y.pub(), (long long)rows, (int)c, (int)o, (int)d, ctx->stream));
  return xb_download(ctx, y, ylw, ylb, yuw, yub);
}

fg_status x64_compose(fg_ctx* ctx, size_t n, size_t d, const double* xlw, const double* xlb, const double* xuw,
                      const double* xub, const double* a_low, const double* b_low, const double* a_up,
                      const double* b_up, double* ylw, double* ylb, double* yuw, double* yub) {
  XB x, y;
  if (fg_status s = xb_upload(ctx, x, n, d, xlw, xlb, xuw, xub)) return s;
  if (fg_status s = xb_alloc(ctx, y, n, d)) return s;
  DBuf rel;
  CK(rel.alloc(sizeof(double) * 4 * n));
  double* r = rel.as<double>();
  if (n) {
    CK(cudaMemcpyAsync(r, a_low, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(r + n, b_low, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(r + 2 * n, a_up, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(r + 3 * n, b_up, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  }
  XL(launch_x_compose(x.plw(), x.plb(), x.puw(), x.pub(), r, r + n, r + 2 * n, r + 3 * n, y.plw(), y.plb(),
                      y.puw(), y.pub(), (long long)n, (int)d, ctx->stream));
  return xb_download(ctx, y, ylw, ylb, yuw, yub);
}

fg_status x64_elementwise_verify(fg_ctx* ctx, int kind, size_t n, size_t d, const double* xlw, const double* xlb,
                                 const double* xuw, const double* xub, int norm, double eps, double* ylw,
                                 double* ylb, double* yuw, double* yub) {
  XB x, y;
  if (fg_status s = xb_upload(ctx, x, n, d, xlw, xlb, xuw, xub)) return s;
  DBuf lo, hi;
  if (fg_status s = x_conc(ctx, x, norm, eps, lo, hi)) return s;
  if (fg_status s = x_relax_compose(ctx, kind, x, lo, hi, y, "elementwise_verify")) return s;
  return xb_download(ctx, y, ylw, ylb, yuw, yub);
}

fg_status x64_dot(fg_ctx* ctx, int layout, size_t batch, size_t len, size_t embed, size_t heads, size_t d,
                  const double* alw, const double* alb, const double* auw, const double* aub, const double* blw,
                  const double* blb, const double* buw, const double* bub, int norm, double eps, double* ylw,
                  double* ylb, double* yuw, double* yub) {
  const bool sim = layout == FG_DOT_SIMILARITY;
  const size_t na = sim ? batch * len * embed : batch * heads * len * len;
  const size_t nb = batch * len * embed;
  const size_t ny = sim ? batch * heads * len * len : batch * len * embed;
  XB a, b, y;
  if (fg_status s = xb_upload(ctx, a, na, d, alw, alb, auw, aub)) return s;
  if (fg_status s = xb_upload(ctx, b, nb, d, blw, blb, buw, bub)) return s;
  DBuf alo, ahi, blo, bhi;  // both operands concretized first (relax.cpp:583-584)
  if (fg_status s = x_conc(ctx, a, norm, eps, alo, ahi)) return s;
  if (fg_status s = x_conc(ctx, b, norm, eps, blo, bhi)) return s;
  if (fg_status s = xb_alloc(ctx, y, ny, d)) return s;
  XDotArgs args{a.plw(), a.plb(), a.puw(), a.pub(), alo.as<double>(),
                b.plw(), b.plb(), b.puw(), b.pub(), blo.as<double>(), bhi.as<double>(),
                y.plw(), y.plb(), y.puw(), y.pub(), sim ? 0 : 1, (long long)batch, (int)len, (int)embed,
                (int)heads, (int)d};
  XL(launch_x_dot(args, ctx->stream));
  return xb_download(ctx, y, ylw, ylb, yuw, yub);
}

// propagate_softmax (relax.cpp:777-790): exp -> sum -> recip -> McCormick multiply.
fg_status x64_softmax(fg_ctx* ctx, size_t outer, size_t n, size_t inner, size_t d, const double* xlw,
                      const double* xlb, const double* xuw, const double* xub, int norm, double eps, double* ylw,
                      double* ylb, double* yuw, double* yub) {
  XB x, e, s, r, y;
  if (fg_status st = xb_upload(ctx, x, outer * n * inner, d, xlw, xlb, xuw, xub)) return st;
  DBuf lo, hi;
  if (fg_status st = x_conc(ctx, x, norm, eps, lo, hi)) return st;
  if (fg_status st = x_relax_compose(ctx, FG_RELAX_EXP, x, lo, hi, e, "relax_exp")) return st;
  if (fg_status st = x_sum_axis(ctx, e, outer, n, inner, s)) return st;
  DBuf slo, shi;
  if (fg_status st = x_conc(ctx, s, norm, eps, slo, shi)) return st;
  if (fg_status st = x_relax_compose(ctx, FG_RELAX_RECIP, s, slo, shi, r, "relax_recip")) return st;
  if (fg_status st = x_mul_broadcast(ctx, e, r, outer, n, inner, norm, eps, y)) return st;
  return xb_download(ctx, y, ylw, ylb, yuw, yub);
}

fg_status x64_add(fg_ctx* ctx, size_t n, size_t d, const double* alw, const double* alb, const double* auw,
                  const double* aub, const double* blw, const double* blb, const double* buw, const double* bub,
                  double* ylw, double* ylb, double* yuw, double* yub) {
  XB a, b, y;
  if (fg_status s = xb_upload(ctx, a, n, d, alw, alb, auw, aub)) return s;
  if (fg_status s = xb_upload(ctx, b, n, d, blw, blb, buw, bub)) return s;
  if (fg_status s = xb_alloc(ctx, y, n, d)) return s;
  XL(launch_x_add(a.plb(), b.plb(), y.plb(), (long long)n, ctx->stream));
  XL(launch_x_add(a.pub(), b.pub(), y.pub(), (long long)n, ctx->stream));
  XL(launch_x_add(a.plw(), b.plw(), y.plw(), (long long)(n * d), ctx->stream));
  XL(launch_x_add(a.puw(), b.puw(), y.puw(), (long long)(n * d), ctx->stream));
  return xb_download(ctx, y, ylw, ylb, yuw, yub);
}

fg_status x64_scale(fg_ctx* ctx, size_t n, size_t d, const double* xlw, const double* xlb, const double* xuw,
                    const double* xub, double sv, double* ylw, double* ylb, double* yuw, double* yub) {
  XB x, y;
  if (fg_status s = xb_upload(ctx, x, n, d, xlw, xlb, xuw, xub)) return s;
  if (fg_status s = xb_alloc(ctx, y, n, d)) return s;
  XL(launch_x_scale(x.plb(), x.pub(), sv, y.plb(), y.pub(), (long long)n, ctx->stream));
  XL(launch_x_scale(x.plw(), x.puw(), sv, y.plw(), y.puw(), (long long)(n * d), ctx->stream));
  return xb_download(ctx, y, ylw, ylb, yuw, yub);
}

}  // namespace fgh

extern "C" {

fg_status fg_ctx_set_precision(fg_ctx* ctx, int precision) {
  if (!ctx) return FG_EINVAL;
  if (precision != FG_PRECISION_F32 && precision != FG_PRECISION_F64)
    return fail(ctx, FG_EINVAL, "fg_ctx_set_precision: unknown precision");
  ctx->precision = precision;
  return FG_OK;
}

int fg_ctx_precision(const fg_ctx* ctx) { return ctx ? ctx->precision : -1; }

fg_status fg_sum_axis(fg_ctx* ctx, size_t outer, size_t n, size_t inner, size_t d, const double* xlw,
                      const double* xlb, const double* xuw, const double* xub, double* ylw, double* ylb,
                      double* yuw, double* yub) {
  cudaSetDevice(ctx->device);
  XB x, y;
  if (fg_status s = xb_upload(ctx, x, outer * n * inner, d, xlw, xlb, xuw, xub)) return s;
  if (fg_status s = x_sum_axis(ctx, x, outer, n, inner, y)) return s;
  return xb_download(ctx, y, ylw, ylb, yuw, yub);
}

fg_status fg_mul_broadcast(fg_ctx* ctx, size_t outer, size_t n, size_t inner, size_t d, const double* xlw,
                           const double* xlb, const double* xuw, const double* xub, const double* rlw,
                           const double* rlb, const double* ruw, const double* rub, int norm, double eps,
                           double* ylw, double* ylb, double* yuw, double* yub) {
  if (!eps_ok(eps)) return fail(ctx, FG_EINVAL, "PerturbationSpec: epsilon must be finite and >= 0");
  cudaSetDevice(ctx->device);
  XB x, r, y;
  if (fg_status s = xb_upload(ctx, x, outer * n * inner, d, xlw, xlb, xuw, xub)) return s;
  if (fg_status s = xb_upload(ctx, r, outer * inner, d, rlw, rlb, ruw, rub)) return s;
  if (fg_status s = x_mul_broadcast(ctx, x, r, outer, n, inner, norm, eps, y)) return s;
  return xb_download(ctx, y, ylw, ylb, yuw, yub);
}

fg_status fg_bilinear(fg_ctx* ctx, size_t n, const double* xlo, const double* xhi, const double* ylo,
                      const double* yhi, double* lo_x, double* lo_y, double* lo_c, double* up_x, double* up_y,
                      double* up_c) {
  cudaSetDevice(ctx->device);
  DBuf in, out, st;
  CK(in.alloc(sizeof(double) * 4 * n));
  CK(out.alloc(sizeof(double) * 6 * n));
  CK(st.alloc(sizeof(int)));
  double* p = in.as<double>();
  if (n) {
    CK(cudaMemcpyAsync(p, xlo, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(p + n, xhi, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(p + 2 * n, ylo, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(p + 3 * n, yhi, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  }
  XL(launch_fill_int(st.as<int>(), kStatusClear, 1, ctx->stream));
  XL(launch_x_bilinear(p, p + n, p + 2 * n, p + 3 * n, out.as<double>(), (long long)n, st.as<int>(), ctx->stream));
  if (fg_status s = x_status(ctx, st.as<int>(), "relax_bilinear")) return s;
  std::vector<double> h(6 * n);
  if (n) CK(cudaMemcpy(h.data(), out.p, sizeof(double) * 6 * n, cudaMemcpyDeviceToHost));
  double* dst[6] = {lo_x, lo_y, lo_c, up_x, up_y, up_c};
  for (int k = 0; k < 6; ++k)
    for (size_t i = 0; i < n; ++i) dst[k][i] = h[k * n + i];
  return FG_OK;
}

}  // extern "C"
