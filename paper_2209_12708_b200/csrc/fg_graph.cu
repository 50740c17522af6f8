// fg_graph.cu -- device-resident executor of faith-graph/v1 verification graphs
// (graph::evaluate, proj/src/graph.cpp:505-673).
//
// Every node value lives in HBM: LinearBounds / PartialBounds as f64 tensors in the reference
// layout (lb/ub [n], lw/uw [n, d]), weights and their sign halves as f64 matrices, per-side
// halves as (b, w).  Values are released after their last consumer (graph.cpp:655-660).  All
// arithmetic is the exact f64 mode of fg_exact.cu (reference operation order, no FMA), so a
// graph evaluates to the same values as the reference's host walk:
//   * MatmulPair runs the propagate_affine kernel on the half matrix: the other half's sums
//     are sums of exact zeros, so every partial equals matmul_half's (graph.cpp:427-472);
//   * CombineHalves: (a + b) + bias (graph.cpp:557-575), bias 0.0 when absent;
//   * AffineBound: propagate_affine, one side kept (graph.cpp:474-481).
// Operator shapes follow the VALUES flowing through the graph (as the reference does), not the
// nodes' recorded out_shape.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <optional>
#include <string>
#include <vector>

#include "fg_host.h"
#include "fg_internal.cuh"
#include "fg_x64.h"

using namespace fgx;

namespace {

using Shape = std::vector<size_t>;

size_t numel(const Shape& s) {
  size_t n = 1;
  for (size_t e : s) n *= e;
  return n;
}

std::string shape_str(const Shape& s) {
  std::string r = "[";
  for (size_t i = 0; i < s.size(); ++i) r += (i ? ", " : "") + std::to_string(s[i]);
  return r + "]";
}

// ---- kernels ---------------------------------------------------------------------------------
__global__ void identity_rows_kernel(double* lw, double* uw, long long n) {  // bounds.cpp:112-116
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * n) return;
  const double v = (t / n == t % n) ? 1.0 : 0.0;
  lw[t] = v;
  uw[t] = v;
}

__global__ void split_signs_kernel(const double* w, double* pos, double* neg, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double v = w[i];
  pos[i] = (v < 0.0) ? 0.0 : v;  // std::max(w, 0.0)
  neg[i] = (0.0 < v) ? 0.0 : v;  // std::min(w, 0.0)
}

__global__ void combine_bias_kernel(const double* a, const double* b, const double* bias, long long o,
                                    double* y, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double bv = bias ? bias[i % o] : 0.0;
  y[i] = a[i] + b[i] + bv;
}

__global__ void count_nonfinite_kernel(const double* v, long long n, int* flag) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && !isfinite(v[i])) atomicExch(flag, 1);
}

unsigned blocks(long long n, int t) { return (unsigned)std::max<long long>(1, (n + t - 1) / t); }

// ---- values --------------------------------------------------------------------------------
enum VKind { V_NONE, V_TENSOR, V_HALVES, V_BOUNDS, V_PARTIAL, V_HALF };

struct Value {
  VKind kind = V_NONE;
  Shape shape;      // tensor shape, or the lb shape of a bounds-like value
  XB xb;            // V_BOUNDS / V_PARTIAL
  DBuf t0, t1;      // V_TENSOR: t0; V_HALVES: pos, neg; V_HALF: b, w
  int side = 0;     // V_HALF
  size_t d = 0;     // V_HALF pert dim
  const double* tensor = nullptr;  // V_TENSOR data (a constant or t0)
};

}  // namespace

struct fg_graph {
  fg_ctx* ctx = nullptr;
  std::vector<fg_node> nodes;
  std::vector<Shape> const_shape;
  std::vector<DBuf> const_data;
  int sink = -1;
  Value result;
};

namespace {

fg_status need(fg_ctx* ctx, bool ok, const std::string& msg, fg_status code = FG_EINVAL) {
  return ok ? FG_OK : fail(ctx, code, msg);
}

const Value* bounds_in(const std::vector<std::optional<Value>>& v, const fg_node& n, int k) {
  const Value& x = *v[n.inputs[k]];
  return x.kind == V_BOUNDS ? &x : nullptr;
}

#define REQ(cond, msg) \
  if (fg_status s_ = need(ctx, (cond), (msg))) return s_

fg_status make_bounds(fg_ctx* ctx, Value& y, const Shape& shape, size_t d) {
  y.kind = V_BOUNDS;
  y.shape = shape;
  return xb_alloc(ctx, y.xb, numel(shape), d);
}

// propagate_affine (relax.cpp:237-307) on device values; w rank 2 [C, O]
fg_status affine(fg_ctx* ctx, const Value& x, const double* w, const Shape& ws, const Value* bias, Value& y,
                 const char* what) {
  REQ(ws.size() == 2, std::string(what) + ": weight must be rank 2");
  const size_t c = ws[0], o = ws[1];
  REQ(!x.shape.empty() && x.shape.back() == c, std::string(what) + ": inner dimensions do not conform");
  if (bias) REQ(bias->kind == V_TENSOR && numel(bias->shape) == o, std::string(what) + ": bias size mismatch");
  Shape os = x.shape;
  os.back() = o;
  if (fg_status s = make_bounds(ctx, y, os, x.xb.d)) return s;
  const size_t rows = x.xb.n / c;
  XL(launch_x_affine(x.xb.plw(), x.xb.plb(), x.xb.puw(), x.xb.pub(), w, bias ? bias->tensor : nullptr, y.xb.plw(),
                     y.xb.plb(), y.xb.puw(), y.xb.pub(), (long long)rows, (int)c, (int)o, (int)x.xb.d, ctx->stream));
  return FG_OK;
}

fg_status elementwise(fg_ctx* ctx, int relax, const Value& x, int norm, double eps, Value& y, const char* what) {
  DBuf lo, hi;
  if (fg_status s = x_conc(ctx, x.xb, norm, eps, lo, hi)) return s;
  y.kind = V_BOUNDS;
  y.shape = x.shape;
  return x_relax_compose(ctx, relax, x.xb, lo, hi, y.xb, what);
}

void axis_split(const Shape& s, size_t axis, size_t& outer, size_t& n, size_t& inner) {
  n = s[axis];
  inner = 1;
  for (size_t i = axis + 1; i < s.size(); ++i) inner *= s[i];
  outer = numel(s) / std::max<size_t>(1, n * inner);
}

fg_status sum_axis(fg_ctx* ctx, const Value& x, size_t axis, Value& y, const char* what) {
  REQ(axis < x.shape.size(), std::string(what) + ": axis out of range");
  size_t outer, n, inner;
  axis_split(x.shape, axis, outer, n, inner);
  y.kind = V_BOUNDS;
  y.shape = x.shape;
  y.shape[axis] = 1;
  return x_sum_axis(ctx, x.xb, outer, n, inner, y.xb);
}

fg_status scale(fg_ctx* ctx, const Value& x, double s, Value& y) {
  if (fg_status st = make_bounds(ctx, y, x.shape, x.xb.d)) return st;
  XL(launch_x_scale(x.xb.plb(), x.xb.pub(), s, y.xb.plb(), y.xb.pub(), (long long)x.xb.n, ctx->stream));
  XL(launch_x_scale(x.xb.plw(), x.xb.puw(), s, y.xb.plw(), y.xb.puw(), (long long)(x.xb.n * x.xb.d), ctx->stream));
  return FG_OK;
}

fg_status mul_broadcast(fg_ctx* ctx, const Value& x, const Value& r, size_t axis, int norm, double eps, Value& y) {
  REQ(axis < x.shape.size() && r.shape.size() == x.shape.size() && r.shape[axis] == 1,
      "propagate_mul_broadcast: operand shapes incompatible");
  REQ(r.xb.d == x.xb.d, "propagate_mul_broadcast: perturbation dims differ");
  size_t outer, n, inner;
  axis_split(x.shape, axis, outer, n, inner);
  REQ(r.xb.n == outer * inner, "propagate_mul_broadcast: operand shapes incompatible");
  y.kind = V_BOUNDS;
  y.shape = x.shape;
  return x_mul_broadcast(ctx, x.xb, r.xb, outer, n, inner, norm, eps, y.xb);
}

fg_status softmax(fg_ctx* ctx, const Value& x, size_t axis, int norm, double eps, Value& y) {  // relax.cpp:777-790
  REQ(axis < x.shape.size(), "propagate_softmax: axis out of range");
  Value e, s, r;
  if (fg_status st = elementwise(ctx, FG_RELAX_EXP, x, norm, eps, e, "relax_exp")) return st;
  if (fg_status st = sum_axis(ctx, e, axis, s, "propagate_sum_axis")) return st;
  if (fg_status st = elementwise(ctx, FG_RELAX_RECIP, s, norm, eps, r, "relax_recip")) return st;
  return mul_broadcast(ctx, e, r, axis, norm, eps, y);
}

fg_status dot(fg_ctx* ctx, const fg_node& nd, const Value& a, const Value& b, int norm, double eps, Value& y) {
  REQ(nd.heads >= 1, "propagate_dot_product: num_heads must be >= 1");
  REQ(a.xb.d == b.xb.d, "propagate_dot_product: perturbation dims differ");
  const size_t H = (size_t)nd.heads;
  size_t batch, len, e;
  Shape os;
  if (nd.layout == FG_DOT_SIMILARITY) {
    REQ(a.shape.size() == 3 && a.shape == b.shape, "propagate_dot_product: similarity expects two [B, L, E] inputs");
    batch = a.shape[0];
    len = a.shape[1];
    e = a.shape[2];
    REQ(e % H == 0, "propagate_dot_product: feature dim not divisible by heads");
    os = {batch, H, len, len};
  } else {
    REQ(a.shape.size() == 4 && b.shape.size() == 3,
        "propagate_dot_product: weighted-values expects [B, H, L, L] and [B, L, E]");
    batch = a.shape[0];
    len = a.shape[2];
    e = b.shape[2];
    REQ(a.shape[1] == H && a.shape[3] == len && b.shape[0] == batch && b.shape[1] == len && e % H == 0,
        "propagate_dot_product: weighted-values shape mismatch");
    os = {batch, len, e};
  }
  DBuf alo, ahi, blo, bhi;  // both operands concretized first (relax.cpp:583-584)
  if (fg_status s = x_conc(ctx, a.xb, norm, eps, alo, ahi)) return s;
  if (fg_status s = x_conc(ctx, b.xb, norm, eps, blo, bhi)) return s;
  if (fg_status s = make_bounds(ctx, y, os, a.xb.d)) return s;
  XDotArgs args{a.xb.plw(), a.xb.plb(), a.xb.puw(), a.xb.pub(), alo.as<double>(),
                b.xb.plw(), b.xb.plb(), b.xb.puw(), b.xb.pub(), blo.as<double>(), bhi.as<double>(),
                y.xb.plw(), y.xb.plb(), y.xb.puw(), y.xb.pub(), nd.layout == FG_DOT_SIMILARITY ? 0 : 1,
                (long long)batch, (int)len, (int)e, (int)H, (int)a.xb.d};
  XL(launch_x_dot(args, ctx->stream));
  return FG_OK;
}

fg_status evaluate(fg_graph* g, size_t n_inputs, const size_t* in_rank, const size_t* in_shape,
                   const double* const* in_data, int norm, double eps, size_t dim) {
  fg_ctx* ctx = g->ctx;
  REQ(eps_ok(eps), "PerturbationSpec: epsilon must be finite and >= 0");
  REQ(dim >= 1, "PerturbationSpec: dim must be >= 1");
  REQ(norm == FG_NORM_L1 || norm == FG_NORM_L2 || norm == FG_NORM_LINF, "PerturbationSpec: unknown norm");
  const size_t N = g->nodes.size();
  std::vector<size_t> remaining(N, 0);
  for (const fg_node& n : g->nodes)
    for (int k = 0; k < n.n_inputs; ++k) ++remaining[n.inputs[k]];
  int sink = -1;
  for (size_t i = 0; i < N; ++i) {
    const int kd = g->nodes[i].kind;
    if (kd != FG_NODE_INPUT && kd != FG_NODE_WEIGHT && remaining[i] == 0) {
      REQ(sink < 0, "evaluate: graph has multiple sinks");
      sink = (int)i;
    }
  }
  REQ(sink >= 0, "evaluate: graph has no operator sink");
  g->result = Value();
  std::vector<std::optional<Value>> v(N);
  for (size_t id = 0; id < N; ++id) {
    const fg_node& nd = g->nodes[id];
    Value y;
    switch (nd.kind) {
      case FG_NODE_INPUT: {  // input_bounds (bounds.cpp:101-120)
        REQ(nd.input >= 0 && (size_t)nd.input < n_inputs, "evaluate: missing input binding for node " +
                                                               std::to_string(id));
        const size_t r = in_rank[nd.input];
        REQ(r >= 1 && r <= FG_GRAPH_MAX_RANK, "input_bounds: bad input rank");
        Shape s(in_shape + (size_t)nd.input * FG_GRAPH_MAX_RANK, in_shape + (size_t)nd.input * FG_GRAPH_MAX_RANK + r);
        const size_t n = numel(s);
        REQ(n == dim, "input_bounds: x.numel() " + std::to_string(n) + " != spec.dim " + std::to_string(dim));
        if (fg_status st = make_bounds(ctx, y, s, dim)) return st;
        CK(cudaMemcpyAsync(y.xb.lb.p, in_data[nd.input], sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(y.xb.ub.p, in_data[nd.input], sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
        identity_rows_kernel<<<blocks((long long)(n * n), 256), 256, 0, ctx->stream>>>(y.xb.plw(), y.xb.puw(),
                                                                                       (long long)n);
        XL(1);
        break;
      }
      case FG_NODE_WEIGHT:
        y.kind = V_TENSOR;
        y.shape = g->const_shape[nd.constant];
        y.tensor = g->const_data[nd.constant].as<double>();
        break;
      case FG_NODE_SPLIT_SIGNS: {
        const Value& w = *v[nd.inputs[0]];
        REQ(w.kind == V_TENSOR, "split_signs: expected a tensor value");
        const size_t n = numel(w.shape);
        y.kind = V_HALVES;
        y.shape = w.shape;
        CK(y.t0.alloc(sizeof(double) * n));
        CK(y.t1.alloc(sizeof(double) * n));
        split_signs_kernel<<<blocks((long long)n, 256), 256, 0, ctx->stream>>>(w.tensor, y.t0.as<double>(),
                                                                               y.t1.as<double>(), (long long)n);
        XL(1);
        break;
      }
      case FG_NODE_MATMUL_PAIR: {
        const Value* x = bounds_in(v, nd, 0);
        REQ(x, "matmul_pair: expected a bounds value");
        const Value& h = *v[nd.inputs[1]];
        REQ(h.kind == V_HALVES, "matmul_pair: expected split halves input");
        REQ(h.shape.size() == 2 && x->shape.back() == h.shape[0], "matmul_pair: inner dimensions do not conform");
        if (fg_status st = affine(ctx, *x, (nd.sign == 0 ? h.t0 : h.t1).as<double>(), h.shape, nullptr, y,
                                  "matmul_pair"))
          return st;
        y.kind = V_PARTIAL;
        break;
      }
      case FG_NODE_COMBINE_HALVES: {
        const Value& a = *v[nd.inputs[0]];
        const Value& b = *v[nd.inputs[1]];
        REQ(a.kind == V_PARTIAL && b.kind == V_PARTIAL, "combine_halves: expected partial products");
        REQ(a.shape == b.shape && a.xb.d == b.xb.d, "combine_halves: partial shapes differ");
        const Value* bias = nd.n_inputs > 2 ? &*v[nd.inputs[2]] : nullptr;
        if (bias) REQ(bias->kind == V_TENSOR, "combine_halves: expected a tensor value");
        const size_t o = a.shape.back();
        if (bias) REQ(numel(bias->shape) >= o, "combine_halves: bias size mismatch");
        if (fg_status st = make_bounds(ctx, y, a.shape, a.xb.d)) return st;
        const long long n = (long long)a.xb.n, nd_ = (long long)(a.xb.n * a.xb.d);
        const double* bp = bias ? bias->tensor : nullptr;
        combine_bias_kernel<<<blocks(n, 256), 256, 0, ctx->stream>>>(a.xb.plb(), b.xb.plb(), bp, (long long)o,
                                                                     y.xb.plb(), n);
        combine_bias_kernel<<<blocks(n, 256), 256, 0, ctx->stream>>>(a.xb.pub(), b.xb.pub(), bp, (long long)o,
                                                                     y.xb.pub(), n);
        XL(2);
        XL(launch_x_add(a.xb.plw(), b.xb.plw(), y.xb.plw(), nd_, ctx->stream));
        XL(launch_x_add(a.xb.puw(), b.xb.puw(), y.xb.puw(), nd_, ctx->stream));
        break;
      }
      case FG_NODE_AFFINE_BOUND:
      case FG_NODE_AFFINE_VERIFY: {
        const char* what = nd.kind == FG_NODE_AFFINE_BOUND ? "affine_bound" : "affine_verify";
        const Value* x = bounds_in(v, nd, 0);
        REQ(x, std::string(what) + ": expected a bounds value");
        const Value& w = *v[nd.inputs[1]];
        REQ(w.kind == V_TENSOR, std::string(what) + ": expected a tensor value");
        const Value* bias = nd.n_inputs > 2 ? &*v[nd.inputs[2]] : nullptr;
        if (fg_status st = affine(ctx, *x, w.tensor, w.shape, bias, y, what)) return st;
        if (nd.kind == FG_NODE_AFFINE_BOUND) {  // affine_one_side (graph.cpp:474-481)
          Value h;
          h.kind = V_HALF;
          h.side = nd.side;
          h.shape = y.shape;
          h.d = y.xb.d;
          h.t0 = std::move(nd.side == 0 ? y.xb.lb : y.xb.ub);
          h.t1 = std::move(nd.side == 0 ? y.xb.lw : y.xb.uw);
          y = std::move(h);
        }
        break;
      }
      case FG_NODE_MERGE_SIDES: {
        Value& a = *v[nd.inputs[0]];
        Value& b = *v[nd.inputs[1]];
        REQ(a.kind == V_HALF && b.kind == V_HALF, "merge_sides: expected half bounds");
        Value* lower = a.side == 0 ? &a : &b;
        Value* upper = a.side == 1 ? &a : &b;
        REQ(lower->side == 0 && upper->side == 1, "merge_sides: need one lower and one upper half");
        REQ(lower->shape == upper->shape && lower->d == upper->d, "merge_sides: half shapes differ");
        if (fg_status st = make_bounds(ctx, y, lower->shape, lower->d)) return st;
        const size_t n = y.xb.n, nd_ = n * y.xb.d;
        CK(cudaMemcpyAsync(y.xb.lb.p, lower->t0.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream));
        CK(cudaMemcpyAsync(y.xb.lw.p, lower->t1.p, sizeof(double) * nd_, cudaMemcpyDeviceToDevice, ctx->stream));
        CK(cudaMemcpyAsync(y.xb.ub.p, upper->t0.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream));
        CK(cudaMemcpyAsync(y.xb.uw.p, upper->t1.p, sizeof(double) * nd_, cudaMemcpyDeviceToDevice, ctx->stream));
        break;
      }
      case FG_NODE_DOT_PRODUCT: {
        const Value* a = bounds_in(v, nd, 0);
        const Value* b = bounds_in(v, nd, 1);
        REQ(a && b, "dot_product: expected a bounds value");
        if (fg_status st = dot(ctx, nd, *a, *b, norm, eps, y)) return st;
        break;
      }
      case FG_NODE_SCALE: {
        const Value* x = bounds_in(v, nd, 0);
        REQ(x, "scale: expected a bounds value");
        if (fg_status st = scale(ctx, *x, nd.scale, y)) return st;
        break;
      }
      case FG_NODE_ADD: {  // propagate_add (relax.cpp:656-674)
        const Value* a = bounds_in(v, nd, 0);
        const Value* b = bounds_in(v, nd, 1);
        REQ(a && b, "add: expected a bounds value");
        REQ(a->xb.n == b->xb.n && a->xb.d == b->xb.d, "propagate_add: operand shape mismatch");
        if (fg_status st = make_bounds(ctx, y, a->shape, a->xb.d)) return st;
        const long long n = (long long)a->xb.n, nd_ = (long long)(a->xb.n * a->xb.d);
        XL(launch_x_add(a->xb.plb(), b->xb.plb(), y.xb.plb(), n, ctx->stream));
        XL(launch_x_add(a->xb.pub(), b->xb.pub(), y.xb.pub(), n, ctx->stream));
        XL(launch_x_add(a->xb.plw(), b->xb.plw(), y.xb.plw(), nd_, ctx->stream));
        XL(launch_x_add(a->xb.puw(), b->xb.puw(), y.xb.puw(), nd_, ctx->stream));
        break;
      }
      case FG_NODE_MEAN_POOL: {  // scale(sum_axis(x, axis), 1/extent) (graph.cpp:628-634)
        const Value* x = bounds_in(v, nd, 0);
        REQ(x, "mean_pool: expected a bounds value");
        REQ((size_t)nd.axis < x->shape.size(), "propagate_sum_axis: axis out of range");
        const size_t extent = x->shape[nd.axis];
        Value s;
        if (fg_status st = sum_axis(ctx, *x, (size_t)nd.axis, s, "propagate_sum_axis")) return st;
        if (fg_status st = scale(ctx, s, 1.0 / (double)extent, y)) return st;
        break;
      }
      case FG_NODE_RELU_VERIFY:
      case FG_NODE_TANH_VERIFY:
      case FG_NODE_SILU_VERIFY:
      case FG_NODE_EXP_VERIFY:
      case FG_NODE_RECIP_VERIFY: {  // graph.cpp:484-501
        const Value* x = bounds_in(v, nd, 0);
        REQ(x, "elementwise: expected a bounds value");
        const int relax = nd.kind == FG_NODE_RELU_VERIFY   ? FG_RELAX_RELU
                          : nd.kind == FG_NODE_TANH_VERIFY ? FG_RELAX_TANH
                          : nd.kind == FG_NODE_SILU_VERIFY ? FG_RELAX_SILU
                          : nd.kind == FG_NODE_EXP_VERIFY  ? FG_RELAX_EXP
                                                           : FG_RELAX_RECIP;
        if (fg_status st = elementwise(ctx, relax, *x, norm, eps, y, "elementwise_verify")) return st;
        break;
      }
      case FG_NODE_SOFTMAX: {
        const Value* x = bounds_in(v, nd, 0);
        REQ(x, "softmax: expected a bounds value");
        if (fg_status st = softmax(ctx, *x, (size_t)nd.axis, norm, eps, y)) return st;
        break;
      }
      case FG_NODE_SUM_REDUCE: {
        const Value* x = bounds_in(v, nd, 0);
        REQ(x, "sum_reduce: expected a bounds value");
        if (fg_status st = sum_axis(ctx, *x, (size_t)nd.axis, y, "propagate_sum_axis")) return st;
        break;
      }
      case FG_NODE_MUL_BROADCAST: {
        const Value* x = bounds_in(v, nd, 0);
        const Value* r = bounds_in(v, nd, 1);
        REQ(x && r, "mul_broadcast: expected a bounds value");
        if (fg_status st = mul_broadcast(ctx, *x, *r, (size_t)nd.axis, norm, eps, y)) return st;
        break;
      }
      default:
        return fail(ctx, FG_EINVAL, "evaluate: unknown node kind " + std::to_string(nd.kind));
    }
    v[id] = std::move(y);
    for (int k = 0; k < nd.n_inputs; ++k) {  // release values with no further consumers
      const int in = nd.inputs[k];
      if (--remaining[in] == 0 && in != sink) v[in].reset();
    }
  }
  Value& res = *v[sink];
  REQ(res.kind == V_BOUNDS, "evaluate: expected a bounds value");
  DBuf flag;
  CK(flag.alloc(sizeof(int)));
  CK(cudaMemsetAsync(flag.p, 0, sizeof(int), ctx->stream));
  const double* parts[4] = {res.xb.plb(), res.xb.pub(), res.xb.plw(), res.xb.puw()};
  const size_t counts[4] = {res.xb.n, res.xb.n, res.xb.n * res.xb.d, res.xb.n * res.xb.d};
  for (int k = 0; k < 4; ++k)
    if (counts[k])
      count_nonfinite_kernel<<<blocks((long long)counts[k], 256), 256, 0, ctx->stream>>>(
          parts[k], (long long)counts[k], flag.as<int>());
  XL(4);
  int h = 0;
  CK(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (h) return fail(ctx, FG_EDOMAIN, "evaluate: bounds overflowed at this radius");  // graph.cpp:663-671
  g->sink = sink;
  g->result = std::move(res);
  return FG_OK;
}

}  // namespace

extern "C" {

fg_status fg_graph_create(fg_ctx* ctx, size_t n_nodes, const fg_node* nodes, size_t n_constants,
                          const size_t* const_rank, const size_t* const_shape, const double* const* const_data,
                          fg_graph** out) {
  if (!ctx || !out) return FG_EINVAL;
  *out = nullptr;
  cudaSetDevice(ctx->device);
  // VerGraph::validate (graph.cpp:133-144)
  for (size_t i = 0; i < n_nodes; ++i) {
    const fg_node& n = nodes[i];
    if (n.kind < FG_NODE_INPUT || n.kind > FG_NODE_MUL_BROADCAST)
      return fail(ctx, FG_EINVAL, "node_kind_from_name: unknown kind " + std::to_string(n.kind));
    if (n.n_inputs < 0 || n.n_inputs > 3) return fail(ctx, FG_EINVAL, "VerGraph: bad input count");
    for (int k = 0; k < n.n_inputs; ++k)
      if (n.inputs[k] < 0 || (size_t)n.inputs[k] >= i) return fail(ctx, FG_EINVAL, "VerGraph: cycle or forward edge");
    if (n.kind == FG_NODE_WEIGHT && (n.constant < 0 || (size_t)n.constant >= n_constants))
      return fail(ctx, FG_EINVAL, "VerGraph: weight node without constant");
    static const int want[] = {0, 0, 1, 2, -1, -1, 2, -1, 2, 1, 2, 1, 1, 1, 1, 1, 1, 1, 1, 2};
    const int w = want[n.kind];
    const bool ok = w >= 0 ? n.n_inputs == w
                           : (n.kind == FG_NODE_COMBINE_HALVES ? (n.n_inputs == 2 || n.n_inputs == 3)
                                                               : (n.n_inputs == 2 || n.n_inputs == 3));
    if (!ok) return fail(ctx, FG_EINVAL, "VerGraph: node " + std::to_string(i) + " has the wrong number of inputs");
  }
  auto g = new fg_graph();
  g->ctx = ctx;
  g->nodes.assign(nodes, nodes + n_nodes);
  g->const_shape.resize(n_constants);
  g->const_data.resize(n_constants);
  for (size_t c = 0; c < n_constants; ++c) {
    if (const_rank[c] > FG_GRAPH_MAX_RANK) {
      delete g;
      return fail(ctx, FG_EINVAL, "graph constant rank too large");
    }
    g->const_shape[c].assign(const_shape + c * FG_GRAPH_MAX_RANK, const_shape + c * FG_GRAPH_MAX_RANK + const_rank[c]);
    const size_t n = numel(g->const_shape[c]);
    if (g->const_data[c].alloc(sizeof(double) * n) != cudaSuccess ||
        (n && cudaMemcpy(g->const_data[c].p, const_data[c], sizeof(double) * n, cudaMemcpyHostToDevice) !=
                  cudaSuccess)) {
      delete g;
      return fail(ctx, FG_ECUDA, "fg_graph_create: constant upload failed");
    }
  }
  if (cudaStreamSynchronize(0) != cudaSuccess) {  // legacy-stream uploads done before the context stream reads
    delete g;
    return fail(ctx, FG_ECUDA, "fg_graph_create: constant upload failed");
  }
  *out = g;
  return FG_OK;
}

void fg_graph_destroy(fg_graph* g) { delete g; }

fg_status fg_graph_evaluate(fg_graph* g, size_t n_inputs, const size_t* in_rank, const size_t* in_shape,
                            const double* const* in_data, int norm, double eps, size_t dim) {
  if (!g) return FG_EINVAL;
  cudaSetDevice(g->ctx->device);
  return evaluate(g, n_inputs, in_rank, in_shape, in_data, norm, eps, dim);
}

fg_status fg_graph_result_shape(const fg_graph* g, size_t* rank, size_t* shape, size_t* d) {
  if (!g || g->result.kind != V_BOUNDS) return FG_EINVAL;
  *rank = g->result.shape.size();
  for (size_t i = 0; i < g->result.shape.size(); ++i) shape[i] = g->result.shape[i];
  *d = g->result.xb.d;
  return FG_OK;
}

fg_status fg_graph_result(fg_graph* g, double* lw, double* lb, double* uw, double* ub) {
  if (!g || g->result.kind != V_BOUNDS) return FG_EINVAL;
  cudaSetDevice(g->ctx->device);
  return xb_download(g->ctx, g->result.xb, lw, lb, uw, ub);
}

}  // extern "C"
