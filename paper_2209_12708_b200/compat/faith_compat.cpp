// faith_compat.cpp -- C++ drop-in layer: the faith:: bounds operators (proj/include/faith/
// bounds.hpp:12-69) and every faith::relax:: function (proj/include/faith/relax.hpp:36-115),
// with byte-identical signatures, executed on the B200 through the C ABI of
// include/faith_gpu.h.  Linking this library instead of proj/src/bounds.cpp + relax.cpp lets
// the reference's own callers -- graph::evaluate (graph.cpp:505-673), cli::cmd_verify /
// cmd_maxeps (cli.cpp:64-193), the machine executors and the acceptance suite -- run
// unchanged with every bound operator on the GPU.
//
// Value semantics are kept (const& in, fresh value out).  Precision: FG_PRECISION_F64 by
// default, i.e. f64 kernels in the reference's operation order (bit-identical arithmetic
// operators); FAITH_GPU_PRECISION=f32 selects the f32-Λ arithmetic of the fused pass.
// FAITH_GPU_DEVICE picks the device (default 0).  Exceptions follow the reference taxonomy:
// FG_EINVAL -> std::invalid_argument, FG_EDOMAIN -> std::domain_error, FG_ERANGE ->
// std::out_of_range.  There is no CPU fallback: without an sm_100 device every bound operator
// throws std::runtime_error.  Host-side pieces are the ones the reference itself keeps on the
// host next to the operators: shape validation, the identity input binding, norm naming, the
// scalar helpers (silu_scalar, tanh_tangent_residual) and the exact forward oracle forward_*.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "faith/bounds.hpp"
#include "faith/relax.hpp"
#include "faith_gpu.h"

namespace faith {

namespace {

struct CtxHolder {
  fg_ctx* c = nullptr;
  ~CtxHolder() {
    if (c) fg_ctx_destroy(c);
  }
};

fg_ctx* gpu() {
  thread_local CtxHolder h;
  if (!h.c) {
    const char* dev = std::getenv("FAITH_GPU_DEVICE");
    if (fg_ctx_create(dev ? std::atoi(dev) : 0, &h.c) != FG_OK || !h.c)
      throw std::runtime_error("faith-gpu: no usable sm_100 device (there is no CPU fallback)");
    const char* prec = std::getenv("FAITH_GPU_PRECISION");
    const bool f32 = prec && std::string(prec) == "f32";
    fg_ctx_set_precision(h.c, f32 ? FG_PRECISION_F32 : FG_PRECISION_F64);
  }
  return h.c;
}

void check(fg_status s, const std::string& what) {
  if (s == FG_OK) return;
  const std::string msg = what + ": " + fg_last_error(gpu());
  switch (s) {
    case FG_EINVAL:
      throw std::invalid_argument(msg);
    case FG_EDOMAIN:
      throw std::domain_error(msg);
    case FG_ERANGE:
      throw std::out_of_range(msg);
    default:
      throw std::runtime_error(msg);
  }
}

int norm_code(Norm p) {
  switch (p) {
    case Norm::L1:
      return FG_NORM_L1;
    case Norm::L2:
      return FG_NORM_L2;
    case Norm::LInf:
      return FG_NORM_LINF;
  }
  throw std::invalid_argument("unknown norm");
}

// Output bounds with the given neuron shape and perturbation width (zero-filled, so an
// empty operator result is already correct).
LinearBounds make_bounds(const std::vector<std::size_t>& nshape, std::size_t d) {
  std::vector<std::size_t> wshape = nshape;
  wshape.push_back(d);
  LinearBounds y;
  y.lb = Tensor::zeros(nshape);
  y.ub = Tensor::zeros(nshape);
  y.lw = Tensor::zeros(wshape);
  y.uw = Tensor::zeros(wshape);
  return y;
}

// axis split [outer, n, inner] of a neuron shape
void axis_split(const Tensor& t, std::size_t axis, std::size_t& outer, std::size_t& n, std::size_t& inner) {
  n = t.extent(axis);
  inner = t.trailing(axis + 1);
  outer = n * inner ? t.numel() / (n * inner) : 0;
}

}  // namespace

// ---- bounds.hpp ----------------------------------------------------------------------------
Norm dual(Norm p) {
  switch (p) {
    case Norm::L1:
      return Norm::LInf;
    case Norm::L2:
      return Norm::L2;
    case Norm::LInf:
      return Norm::L1;
  }
  throw std::invalid_argument("dual: unknown norm");
}

std::string norm_name(Norm p) {
  return p == Norm::L1 ? "l1" : p == Norm::L2 ? "l2" : p == Norm::LInf ? "linf" : "?";
}

Norm norm_from_name(const std::string& name) {
  for (Norm p : {Norm::L1, Norm::L2, Norm::LInf})
    if (norm_name(p) == name) return p;
  throw std::invalid_argument("norm_from_name: unknown norm '" + name + "'");
}

PerturbationSpec::PerturbationSpec(Norm p_, double epsilon_, std::size_t dim_) : p(p_), epsilon(epsilon_), dim(dim_) {
  if (!(epsilon >= 0.0) || !std::isfinite(epsilon))
    throw std::invalid_argument("PerturbationSpec: epsilon must be finite and >= 0");
  if (dim < 1) throw std::invalid_argument("PerturbationSpec: dim must be >= 1");
}

void LinearBounds::validate(const std::string& context) const {
  if (!lw.same_shape(uw))
    throw std::invalid_argument(context + ": lw/uw shape mismatch " + lw.shape_str() + " vs " + uw.shape_str());
  if (!lb.same_shape(ub)) throw std::invalid_argument(context + ": lb/ub shape mismatch");
  if (lw.rank() != lb.rank() + 1) throw std::invalid_argument(context + ": lw rank must be lb rank + 1");
  for (std::size_t a = 0; a < lb.rank(); ++a)
    if (lw.extent(a) != lb.extent(a))
      throw std::invalid_argument(context + ": lw " + lw.shape_str() + " does not extend lb " + lb.shape_str());
}

void ConcreteBounds::validate(const std::string& context) const {
  if (!lo.same_shape(hi)) throw std::invalid_argument(context + ": lo/hi shape mismatch");
  for (std::size_t i = 0; i < lo.numel(); ++i)
    if (lo[i] > hi[i]) throw std::invalid_argument(context + ": lo > hi at neuron " + std::to_string(i));
}

double row_norm(std::span<const double> row, Norm q) {  // one row: a host scalar utility
  double s = 0.0;
  for (double v : row) {
    if (q == Norm::L1) s += std::fabs(v);
    else if (q == Norm::L2) s += v * v;
    else s = std::max(s, std::fabs(v));
  }
  return q == Norm::L2 ? std::sqrt(s) : s;
}

LinearBounds input_bounds(const Tensor& x, const PerturbationSpec& spec) {
  if (x.numel() != spec.dim)
    throw std::invalid_argument("input_bounds: input has " + std::to_string(x.numel()) + " elements, spec.dim is " +
                                std::to_string(spec.dim));
  const std::size_t n = x.numel();
  LinearBounds out = make_bounds(x.shape(), spec.dim);
  out.lb = x;
  out.ub = x;
  for (std::size_t i = 0; i < n; ++i) {
    out.lw[i * n + i] = 1.0;
    out.uw[i * n + i] = 1.0;
  }
  return out;
}

ConcreteBounds concretize(const LinearBounds& b, const PerturbationSpec& spec) {
  b.validate("concretize");
  ConcreteBounds out;
  out.lo = Tensor::zeros(b.lb.shape());
  out.hi = Tensor::zeros(b.ub.shape());
  const std::size_t n = b.neuron_count();
  if (n == 0) return out;
  check(fg_concretize(gpu(), n, b.pert_dim(), b.lw.data(), b.lb.data(), b.uw.data(), b.ub.data(),
                      norm_code(spec.p), spec.epsilon, out.lo.data(), out.hi.data()),
        "concretize");
  return out;
}

bool check_robust(const ConcreteBounds& pred_bounds, std::size_t true_class, double margin) {
  const std::size_t n = pred_bounds.lo.numel();
  if (true_class >= n)
    throw std::out_of_range("check_robust: true_class " + std::to_string(true_class) + " out of range for " +
                            std::to_string(n) + " classes");
  if (margin < 0.0) throw std::invalid_argument("check_robust: margin must be >= 0");
  int verified = 0;
  check(fg_check_robust(n, pred_bounds.lo.data(), pred_bounds.hi.data(), true_class, margin, &verified),
        "check_robust");
  return verified != 0;
}

namespace relax {

// ---- scalar helpers and the exact forward oracle (host, as in the reference) --------------
double silu_scalar(double x) { return x * (1.0 / (1.0 + std::exp(-x))); }

double silu_derivative(double x) {
  const double s = 1.0 / (1.0 + std::exp(-x));
  return s * (1.0 + x * (1.0 - s));
}

double tanh_tangent_residual(double anchor, double tangent_point) {
  const double t = std::tanh(tangent_point);
  return t + (1.0 - t * t) * (anchor - tangent_point) - std::tanh(anchor);
}

namespace {
template <class F>
Tensor map_elements(const Tensor& x, F f) {
  Tensor out = Tensor::zeros(x.shape());
  for (std::size_t i = 0; i < x.numel(); ++i) out[i] = f(x[i]);
  return out;
}
}  // namespace

Tensor forward_relu(const Tensor& x) {
  return map_elements(x, [](double v) { return v > 0.0 ? v : 0.0; });
}
Tensor forward_tanh(const Tensor& x) {
  return map_elements(x, [](double v) { return std::tanh(v); });
}
Tensor forward_silu(const Tensor& x) { return map_elements(x, silu_scalar); }
Tensor forward_exp(const Tensor& x) {
  return map_elements(x, [](double v) { return std::exp(v); });
}
Tensor forward_recip(const Tensor& x) {
  for (std::size_t i = 0; i < x.numel(); ++i)
    if (x[i] <= 0.0) throw std::domain_error("forward_recip: non-positive input");
  return map_elements(x, [](double v) { return 1.0 / v; });
}

Tensor forward_matmul(const Tensor& x, const Tensor& w, const Tensor* bias) {
  if (w.rank() != 2) throw std::invalid_argument("forward_matmul: weight must be rank 2");
  const std::size_t c = w.extent(0), o = w.extent(1);
  if (x.rank() == 0 || x.shape().back() != c)
    throw std::invalid_argument("forward_matmul: inner dimensions do not conform: x " + x.shape_str() + " vs W " +
                                w.shape_str());
  if (bias && bias->numel() != o) throw std::invalid_argument("forward_matmul: bias length mismatch");
  std::vector<std::size_t> oshape = x.shape();
  oshape.back() = o;
  Tensor out = Tensor::zeros(oshape);
  const std::size_t rows = x.numel() / c;
  for (std::size_t r = 0; r < rows; ++r)
    for (std::size_t j = 0; j < o; ++j) {
      double acc = 0.0;
      for (std::size_t i = 0; i < c; ++i) acc += x[r * c + i] * w[i * o + j];
      out[r * o + j] = acc + (bias ? (*bias)[j] : 0.0);
    }
  return out;
}

Tensor forward_pairwise_dot(const Tensor& a, const Tensor& b) {
  if (a.rank() != 3 || !a.same_shape(b))
    throw std::invalid_argument("forward_pairwise_dot: expects two tensors of shape [B, L, D]");
  const std::size_t batch = a.extent(0), len = a.extent(1), d = a.extent(2);
  Tensor out = Tensor::zeros({batch, len, len});
  for (std::size_t bi = 0; bi < batch; ++bi)
    for (std::size_t i = 0; i < len; ++i)
      for (std::size_t j = 0; j < len; ++j) {
        double acc = 0.0;
        for (std::size_t k = 0; k < d; ++k) acc += a[(bi * len + i) * d + k] * b[(bi * len + j) * d + k];
        out[(bi * len + i) * len + j] = acc;
      }
  return out;
}

Tensor forward_softmax(const Tensor& x, std::size_t axis) {
  if (axis >= x.rank()) throw std::invalid_argument("forward_softmax: axis out of range");
  std::size_t outer, n, inner;
  axis_split(x, axis, outer, n, inner);
  Tensor out = Tensor::zeros(x.shape());
  for (std::size_t oi = 0; oi < outer; ++oi)
    for (std::size_t ii = 0; ii < inner; ++ii) {
      auto at = [&](std::size_t j) { return (oi * n + j) * inner + ii; };
      double mx = -HUGE_VAL;
      for (std::size_t j = 0; j < n; ++j) mx = std::max(mx, x[at(j)]);
      double sum = 0.0;
      for (std::size_t j = 0; j < n; ++j) sum += std::exp(x[at(j)] - mx);
      for (std::size_t j = 0; j < n; ++j) out[at(j)] = std::exp(x[at(j)] - mx) / sum;
    }
  return out;
}

// ---- bound propagation rules on the GPU -----------------------------------------------------
LinearBounds propagate_affine(const LinearBounds& x, const Tensor& w, const Tensor* bias) {
  x.validate("propagate_affine");
  if (w.rank() != 2) throw std::invalid_argument("propagate_affine: weight must be rank 2");
  const std::size_t c = w.extent(0), o = w.extent(1);
  if (x.lb.rank() == 0 || x.lb.shape().back() != c)
    throw std::invalid_argument("propagate_affine: inner dimensions do not conform: x " + x.lb.shape_str() +
                                " vs W " + w.shape_str());
  if (bias && bias->numel() != o) throw std::invalid_argument("propagate_affine: bias length mismatch");
  std::vector<std::size_t> oshape = x.lb.shape();
  oshape.back() = o;
  LinearBounds y = make_bounds(oshape, x.pert_dim());
  const std::size_t rows = c ? x.lb.numel() / c : 0;
  if (rows == 0 || o == 0) return y;
  if (c == 0) {  // empty contraction: y = bias
    for (std::size_t r = 0; r < rows; ++r)
      for (std::size_t j = 0; j < o; ++j) y.lb[r * o + j] = y.ub[r * o + j] = bias ? (*bias)[j] : 0.0;
    return y;
  }
  check(fg_affine(gpu(), rows, c, o, x.pert_dim(), x.lw.data(), x.lb.data(), x.uw.data(), x.ub.data(), w.data(),
                  bias ? bias->data() : nullptr, y.lw.data(), y.lb.data(), y.uw.data(), y.ub.data()),
        "propagate_affine");
  return y;
}

namespace {
ElementwiseLinearRelaxation relax_kind(const ConcreteBounds& c, int kind, const char* name) {
  c.validate(name);
  ElementwiseLinearRelaxation r;
  r.a_low = Tensor::zeros(c.lo.shape());
  r.b_low = Tensor::zeros(c.lo.shape());
  r.a_up = Tensor::zeros(c.lo.shape());
  r.b_up = Tensor::zeros(c.lo.shape());
  if (c.lo.numel() == 0) return r;
  check(fg_relax(gpu(), kind, c.lo.numel(), c.lo.data(), c.hi.data(), r.a_low.data(), r.b_low.data(),
                 r.a_up.data(), r.b_up.data()),
        name);
  for (const Tensor* t : {&r.a_low, &r.b_low, &r.a_up, &r.b_up}) t->check_finite(name);
  return r;
}
}  // namespace

ElementwiseLinearRelaxation relax_relu(const ConcreteBounds& c) { return relax_kind(c, FG_RELAX_RELU, "relax_relu"); }
ElementwiseLinearRelaxation relax_tanh(const ConcreteBounds& c) { return relax_kind(c, FG_RELAX_TANH, "relax_tanh"); }
ElementwiseLinearRelaxation relax_exp(const ConcreteBounds& c) { return relax_kind(c, FG_RELAX_EXP, "relax_exp"); }
ElementwiseLinearRelaxation relax_recip(const ConcreteBounds& c) {
  return relax_kind(c, FG_RELAX_RECIP, "relax_recip");
}
ElementwiseLinearRelaxation relax_silu(const ConcreteBounds& c) { return relax_kind(c, FG_RELAX_SILU, "relax_silu"); }

LinearBounds compose_elementwise(const LinearBounds& x, const ElementwiseLinearRelaxation& r) {
  x.validate("compose_elementwise");
  if (!r.a_low.same_shape(x.lb))
    throw std::invalid_argument("compose_elementwise: relaxation shape " + r.a_low.shape_str() +
                                " does not match bounds " + x.lb.shape_str());
  LinearBounds y = make_bounds(x.lb.shape(), x.pert_dim());
  if (x.neuron_count() == 0) return y;
  check(fg_compose(gpu(), x.neuron_count(), x.pert_dim(), x.lw.data(), x.lb.data(), x.uw.data(), x.ub.data(),
                   r.a_low.data(), r.b_low.data(), r.a_up.data(), r.b_up.data(), y.lw.data(), y.lb.data(),
                   y.uw.data(), y.ub.data()),
        "compose_elementwise");
  return y;
}

BilinearRelaxation relax_bilinear(const ConcreteBounds& cx, const ConcreteBounds& cy) {
  cx.validate("relax_bilinear");
  cy.validate("relax_bilinear");
  if (!cx.lo.same_shape(cy.lo)) throw std::invalid_argument("relax_bilinear: operand shape mismatch");
  BilinearRelaxation r;
  for (Tensor* t : {&r.lo_x, &r.lo_y, &r.lo_c, &r.up_x, &r.up_y, &r.up_c}) *t = Tensor::zeros(cx.lo.shape());
  if (cx.lo.numel() == 0) return r;
  check(fg_bilinear(gpu(), cx.lo.numel(), cx.lo.data(), cx.hi.data(), cy.lo.data(), cy.hi.data(), r.lo_x.data(),
                    r.lo_y.data(), r.lo_c.data(), r.up_x.data(), r.up_y.data(), r.up_c.data()),
        "relax_bilinear");
  return r;
}

LinearBounds propagate_dot_product(const LinearBounds& a, const LinearBounds& b, const PerturbationSpec& spec,
                                   DotLayout layout, std::size_t num_heads) {
  a.validate("propagate_dot_product");
  b.validate("propagate_dot_product");
  if (num_heads == 0) throw std::invalid_argument("propagate_dot_product: num_heads must be >= 1");
  const std::size_t d = a.pert_dim();
  if (d != b.pert_dim()) throw std::invalid_argument("propagate_dot_product: perturbation dims differ");
  std::size_t batch, len, e;
  LinearBounds y;
  if (layout == DotLayout::PairwiseSimilarity) {
    if (a.lb.rank() != 3 || !a.lb.same_shape(b.lb))
      throw std::invalid_argument("propagate_dot_product: similarity expects two [B, L, E] inputs");
    batch = a.lb.extent(0), len = a.lb.extent(1), e = a.lb.extent(2);
    if (e % num_heads != 0)
      throw std::invalid_argument("propagate_dot_product: feature dim not divisible by heads");
    y = make_bounds({batch, num_heads, len, len}, d);
  } else {
    if (a.lb.rank() != 4 || b.lb.rank() != 3)
      throw std::invalid_argument("propagate_dot_product: weighted-values expects [B, H, L, L] and [B, L, E]");
    batch = a.lb.extent(0), len = a.lb.extent(2), e = b.lb.extent(2);
    const std::size_t heads = a.lb.extent(1);
    if (heads != num_heads || a.lb.extent(3) != len || b.lb.extent(0) != batch || b.lb.extent(1) != len ||
        e % num_heads != 0)
      throw std::invalid_argument("propagate_dot_product: weighted-values shape mismatch");
    y = make_bounds({batch, len, e}, d);
  }
  if (y.neuron_count() == 0) return y;
  if (e == 0 || len == 0) return y;
  check(fg_dot_batched(gpu(), layout == DotLayout::PairwiseSimilarity ? FG_DOT_SIMILARITY : FG_DOT_WEIGHTED_VALUES,
                       batch, len, e, num_heads, d, a.lw.data(), a.lb.data(), a.uw.data(), a.ub.data(), b.lw.data(),
                       b.lb.data(), b.uw.data(), b.ub.data(), norm_code(spec.p), spec.epsilon, y.lw.data(),
                       y.lb.data(), y.uw.data(), y.ub.data()),
        "propagate_dot_product");
  return y;
}

LinearBounds propagate_add(const LinearBounds& a, const LinearBounds& b) {
  a.validate("propagate_add");
  b.validate("propagate_add");
  if (!a.lb.same_shape(b.lb) || !a.lw.same_shape(b.lw))
    throw std::invalid_argument("propagate_add: operand shape mismatch " + a.lb.shape_str() + " vs " +
                                b.lb.shape_str());
  LinearBounds y = make_bounds(a.lb.shape(), a.pert_dim());
  if (a.neuron_count() == 0) return y;
  check(fg_add(gpu(), a.neuron_count(), a.pert_dim(), a.lw.data(), a.lb.data(), a.uw.data(), a.ub.data(),
               b.lw.data(), b.lb.data(), b.uw.data(), b.ub.data(), y.lw.data(), y.lb.data(), y.uw.data(),
               y.ub.data()),
        "propagate_add");
  return y;
}

LinearBounds propagate_scale(const LinearBounds& x, double s) {
  x.validate("propagate_scale");
  LinearBounds y = make_bounds(x.lb.shape(), x.pert_dim());
  if (x.neuron_count() == 0) return y;
  check(fg_scale(gpu(), x.neuron_count(), x.pert_dim(), x.lw.data(), x.lb.data(), x.uw.data(), x.ub.data(), s,
                 y.lw.data(), y.lb.data(), y.uw.data(), y.ub.data()),
        "propagate_scale");
  return y;
}

LinearBounds propagate_sum_axis(const LinearBounds& x, std::size_t axis) {
  x.validate("propagate_sum_axis");
  if (axis >= x.lb.rank()) throw std::invalid_argument("propagate_sum_axis: axis out of range");
  std::size_t outer, n, inner;
  axis_split(x.lb, axis, outer, n, inner);
  std::vector<std::size_t> oshape = x.lb.shape();
  oshape[axis] = 1;
  LinearBounds y = make_bounds(oshape, x.pert_dim());
  if (outer * inner == 0 || n == 0) return y;
  check(fg_sum_axis(gpu(), outer, n, inner, x.pert_dim(), x.lw.data(), x.lb.data(), x.uw.data(), x.ub.data(),
                    y.lw.data(), y.lb.data(), y.uw.data(), y.ub.data()),
        "propagate_sum_axis");
  return y;
}

LinearBounds propagate_mul_broadcast(const LinearBounds& x, const LinearBounds& r, std::size_t axis,
                                     const PerturbationSpec& spec) {
  x.validate("propagate_mul_broadcast");
  r.validate("propagate_mul_broadcast");
  if (axis >= x.lb.rank() || r.lb.rank() != x.lb.rank() || r.lb.extent(axis) != 1)
    throw std::invalid_argument("propagate_mul_broadcast: operand shapes incompatible");
  std::size_t outer, n, inner;
  axis_split(x.lb, axis, outer, n, inner);
  LinearBounds y = make_bounds(x.lb.shape(), x.pert_dim());
  if (x.neuron_count() == 0) return y;
  check(fg_mul_broadcast(gpu(), outer, n, inner, x.pert_dim(), x.lw.data(), x.lb.data(), x.uw.data(), x.ub.data(),
                         r.lw.data(), r.lb.data(), r.uw.data(), r.ub.data(), norm_code(spec.p), spec.epsilon,
                         y.lw.data(), y.lb.data(), y.uw.data(), y.ub.data()),
        "propagate_mul_broadcast");
  return y;
}

LinearBounds propagate_softmax(const LinearBounds& x, std::size_t axis, const PerturbationSpec& spec) {
  x.validate("propagate_softmax");
  if (axis >= x.lb.rank()) throw std::invalid_argument("propagate_softmax: axis out of range");
  std::size_t outer, n, inner;
  axis_split(x.lb, axis, outer, n, inner);
  LinearBounds y = make_bounds(x.lb.shape(), x.pert_dim());
  if (x.neuron_count() == 0) return y;
  check(fg_softmax_axis(gpu(), outer, n, inner, x.pert_dim(), x.lw.data(), x.lb.data(), x.uw.data(), x.ub.data(),
                        norm_code(spec.p), spec.epsilon, y.lw.data(), y.lb.data(), y.uw.data(), y.ub.data()),
        "propagate_softmax");
  return y;
}

}  // namespace relax
}  // namespace faith
