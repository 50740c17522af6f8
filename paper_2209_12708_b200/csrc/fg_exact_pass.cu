// fg_exact_pass.cu -- the word-level bound pass in the exact precision mode, on the device.
//
// One sentence walks the same node sequence as graph::evaluate over fuse_all(build_graph(spec))
// (proj/src/graph.cpp:531-661, proj/src/model.cpp:393-448): Q/K/V propagate_affine ->
// similarity dot -> Scale 1/sqrt(hd) -> ExpVerify -> SumReduce -> RecipVerify -> MulBroadcast ->
// weighted-values dot -> Wo affine -> Add -> W1 affine -> activation verify -> W2 affine -> Add,
// then MeanPool and the classifier, the sink finiteness check (graph.cpp:663-671) and the final
// concretize (cli.cpp:90).  Every value is an f64 tensor in the reference layout in HBM and
// every operator is one of fg_exact.cu's reference-order kernels (compiled -fmad=false), so the
// arithmetic operators reproduce proj/src/relax.cpp / bounds.cpp bit for bit; the exp / tanh /
// SiLU envelopes agree to the last ulp or two of the device libm.
//
// Used by the fused pass's ε search (fg_maxeps, fg_certify) to settle the verdict of a probe
// whose f32-Λ margin lies within its error estimate of zero (see fg_host.cu `Ambiguity`), and
// exported as fg_bound_pass_exact(_dump) for parity checks against the reference's golden
// vectors.  Input binding is the word-level one of SURVEY G1 (oracle/faith_oracle.c
// bound_pass): lb = ub = x, the rows of the perturbed positions one-hot into D = words*E.
#include <cuda_runtime.h>

#include <cmath>
#include <string>
#include <vector>

#include "fg_host.h"
#include "fg_internal.cuh"
#include "fg_x64.h"

using namespace fgx;

namespace {

__global__ void x_bind_input_kernel(const double* __restrict__ x, const int* __restrict__ pos, int words,
                                    long long L, int E, double* lb, double* ub, double* lw, double* uw) {
  const long long D = (long long)words * E;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < L * E) {
    lb[t] = x[t];
    ub[t] = x[t];
  }
  if (t < (long long)words * E) {  // row (pos[w], e) -> column w*E + e
    const int w = (int)(t / E), e = (int)(t % E);
    const long long row = (long long)pos[w] * E + e;
    lw[row * D + t] = 1.0;
    uw[row * D + t] = 1.0;
  }
}

__global__ void x_finite_kernel(const double* __restrict__ v, long long n, int* flag) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && !isfinite(v[i])) atomicExch(flag, 1);
}

inline unsigned nblocks(long long n, int t) { return (unsigned)((n + t - 1) / t); }

struct Walk {
  fg_ctx* ctx;
  const fg_config& c;
  int norm;
  double eps;
  double* node_lo;
  double* node_hi;
  int* dstat = nullptr;  // asynchronous walk: one device status word per relaxation site
  int site = 0;
  size_t off = 0;

  // concretize one node into the host dump (fo_bound_pass order)
  fg_status dump(const XB& b) {
    if (node_lo) {
      DBuf lo, hi;
      if (fg_status s = x_conc(ctx, b, norm, eps, lo, hi)) return s;
      CK(cudaMemcpyAsync(node_lo + off, lo.p, sizeof(double) * b.n, cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaMemcpyAsync(node_hi + off, hi.p, sizeof(double) * b.n, cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
    }
    off += b.n;
    return FG_OK;
  }

  fg_status affine(const XB& x, size_t rows, size_t cin, size_t o, const double* w, const double* b, XB& y) {
    if (fg_status s = xb_alloc(ctx, y, rows * o, x.d)) return s;
    XL(launch_x_affine(x.plw(), x.plb(), x.puw(), x.pub(), w, b, y.plw(), y.plb(), y.puw(), y.pub(),
                       (long long)rows, (int)cin, (int)o, (int)x.d, ctx->stream));
    return FG_OK;
  }

  fg_status dot(int layout, const XB& a, const XB& b, XB& y) {
    const size_t L = c.length, E = c.embed, H = c.heads;
    DBuf alo, ahi, blo, bhi;  // both operands concretized first (relax.cpp:583-584)
    if (fg_status s = x_conc(ctx, a, norm, eps, alo, ahi)) return s;
    if (fg_status s = x_conc(ctx, b, norm, eps, blo, bhi)) return s;
    const size_t ny = layout == FG_DOT_SIMILARITY ? H * L * L : L * E;
    if (fg_status s = xb_alloc(ctx, y, ny, a.d)) return s;
    XDotArgs args{a.plw(), a.plb(), a.puw(), a.pub(), alo.as<double>(),
                  b.plw(), b.plb(), b.puw(), b.pub(), blo.as<double>(), bhi.as<double>(),
                  y.plw(), y.plb(), y.puw(), y.pub(), layout == FG_DOT_SIMILARITY ? 0 : 1, 1LL, (int)L, (int)E,
                  (int)H, (int)a.d};
    XL(launch_x_dot(args, ctx->stream));
    return FG_OK;
  }

  fg_status add(const XB& a, const XB& b, XB& y) {
    if (fg_status s = xb_alloc(ctx, y, a.n, a.d)) return s;
    XL(launch_x_add(a.plb(), b.plb(), y.plb(), (long long)a.n, ctx->stream));
    XL(launch_x_add(a.pub(), b.pub(), y.pub(), (long long)a.n, ctx->stream));
    XL(launch_x_add(a.plw(), b.plw(), y.plw(), (long long)(a.n * a.d), ctx->stream));
    XL(launch_x_add(a.puw(), b.puw(), y.puw(), (long long)(a.n * a.d), ctx->stream));
    return FG_OK;
  }

  fg_status scale(const XB& x, double sv, XB& y) {
    if (fg_status s = xb_alloc(ctx, y, x.n, x.d)) return s;
    XL(launch_x_scale(x.plb(), x.pub(), sv, y.plb(), y.pub(), (long long)x.n, ctx->stream));
    XL(launch_x_scale(x.plw(), x.puw(), sv, y.plw(), y.puw(), (long long)(x.n * x.d), ctx->stream));
    return FG_OK;
  }

  // elementwise_verify (graph.cpp:484-501): concretize -> relax (validate, domain) -> compose.
  // Asynchronous walks do not stop at a failing relaxation: its status word is kept on the device
  // and the first failing site decides the sentence's status when the walk has finished.
  fg_status verify(int kind, const XB& x, XB& y, const char* what) {
    DBuf lo, hi;
    if (fg_status s = x_conc(ctx, x, norm, eps, lo, hi)) return s;
    if (!dstat) return x_relax_compose(ctx, kind, x, lo, hi, y, what);
    DBuf lines;
    CK(lines.alloc_async(sizeof(double) * 4 * x.n, ctx->stream));
    double* l = lines.as<double>();
    XL(launch_relax(kind, lo.as<double>(), hi.as<double>(), (long long)x.n, l, l + x.n, l + 2 * x.n, l + 3 * x.n,
                    dstat + site++, ctx->stream));
    if (fg_status s = xb_alloc(ctx, y, x.n, x.d)) return s;
    XL(launch_x_compose(x.plw(), x.plb(), x.puw(), x.pub(), l, l + x.n, l + 2 * x.n, l + 3 * x.n, y.plw(), y.plb(),
                        y.puw(), y.pub(), (long long)x.n, (int)x.d, ctx->stream));
    return FG_OK;
  }
};

}  // namespace

namespace fgh {

// The exact pass for one sentence.  `params` are the model's f64 weights on the device
// (gen_synthetic order).  Returns FG_OK with *status = FG_OK / FG_EINVAL / FG_EDOMAIN for the
// sentence (the reference's exceptions, graph.cpp / relax.cpp), or an error code for a failure
// of the call itself.
fg_status exact_pass(fg_ctx* ctx, const fg_config& c, const double* params, const double* x_host,
                     const int* pos_host, int words, int norm, double eps, double* logits_lo, double* logits_hi,
                     double* node_lo, double* node_hi, int* status, ExactJob* job) {
  const size_t L = c.length, E = c.embed, H = c.heads, F = c.ffn, C = c.classes, D = (size_t)words * E;
  Walk wk{ctx, c, norm, eps, node_lo, node_hi};
  if (status) *status = FG_OK;
  DBuf dstat;
  const int nsites = 3 * c.layers;  // exp, recip, activation per layer
  if (job) {
    CK(dstat.alloc_async(sizeof(int) * nsites, ctx->stream));
    XL(launch_fill_int(dstat.as<int>(), kStatusClear, nsites, ctx->stream));
    wk.dstat = dstat.as<int>();
  }
  XB cur;
  if (fg_status s = xb_alloc(ctx, cur, L * E, D)) return s;
  CK(cudaMemsetAsync(cur.lw.p, 0, sizeof(double) * L * E * D, ctx->stream));
  CK(cudaMemsetAsync(cur.uw.p, 0, sizeof(double) * L * E * D, ctx->stream));
  DBuf dx, dpos;
  CK(dx.alloc_async(sizeof(double) * L * E, ctx->stream));
  CK(dpos.alloc_async(sizeof(int) * words, ctx->stream));
  CK(cudaMemcpyAsync(dx.p, x_host, sizeof(double) * L * E, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(dpos.p, pos_host, sizeof(int) * words, cudaMemcpyHostToDevice, ctx->stream));
  x_bind_input_kernel<<<nblocks((long long)L * E, 256), 256, 0, ctx->stream>>>(
      dx.as<double>(), dpos.as<int>(), words, (long long)L, (int)E, cur.plb(), cur.pub(), cur.plw(), cur.puw());
  ++ctx->launches;

  // a relaxation's domain / validation error ends the pass with that status (not a call failure)
  auto sentence_error = [&](fg_status s) { return s == FG_EINVAL || s == FG_EDOMAIN; };
  const double inv_sqrt_hd = 1.0 / std::sqrt((double)(E / H));  // model.cpp:417
  const size_t per_layer = 4 * (E * E + E) + E * F + F + F * E + E;
  for (int l = 0; l < c.layers; ++l) {
    const double* p = params + (size_t)l * per_layer;
    const double *wq = p, *bq = wq + E * E, *wkk = bq + E, *bk = wkk + E * E, *wv = bk + E, *bv = wv + E * E,
                 *wo = bv + E, *bo = wo + E * E, *w1 = bo + E, *b1 = w1 + E * F, *w2 = b1 + F, *b2 = w2 + F * E;
    XB q, k, v, sc, scl, e, s, r, pr, cx, attn, res1, f1, act, f2, nxt;
    if (fg_status st = wk.affine(cur, L, E, E, wq, bq, q)) return st;
    if (fg_status st = wk.dump(q)) return st;
    if (fg_status st = wk.affine(cur, L, E, E, wkk, bk, k)) return st;
    if (fg_status st = wk.dump(k)) return st;
    if (fg_status st = wk.affine(cur, L, E, E, wv, bv, v)) return st;
    if (fg_status st = wk.dump(v)) return st;
    if (fg_status st = wk.dot(FG_DOT_SIMILARITY, q, k, sc)) return st;
    if (fg_status st = wk.dump(sc)) return st;
    q = XB();
    k = XB();
    if (fg_status st = wk.scale(sc, inv_sqrt_hd, scl)) return st;
    if (fg_status st = wk.dump(scl)) return st;
    sc = XB();
    // softmax as the fused graph evaluates it (graph.cpp:237-240)
    if (fg_status st = wk.verify(FG_RELAX_EXP, scl, e, "relax_exp")) {
      if (sentence_error(st)) { *status = st; return FG_OK; }
      return st;
    }
    if (fg_status st = wk.dump(e)) return st;
    if (fg_status st = x_sum_axis(ctx, e, H * L, L, 1, s)) return st;
    if (fg_status st = wk.dump(s)) return st;
    if (fg_status st = wk.verify(FG_RELAX_RECIP, s, r, "relax_recip")) {
      if (sentence_error(st)) { *status = st; return FG_OK; }
      return st;
    }
    if (fg_status st = wk.dump(r)) return st;
    if (fg_status st = x_mul_broadcast(ctx, e, r, H * L, L, 1, norm, eps, pr)) return st;
    if (fg_status st = wk.dump(pr)) return st;
    scl = XB();
    e = XB();
    s = XB();
    r = XB();
    if (fg_status st = wk.dot(FG_DOT_WEIGHTED_VALUES, pr, v, cx)) return st;
    if (fg_status st = wk.dump(cx)) return st;
    pr = XB();
    v = XB();
    if (fg_status st = wk.affine(cx, L, E, E, wo, bo, attn)) return st;
    if (fg_status st = wk.dump(attn)) return st;
    cx = XB();
    if (fg_status st = wk.add(cur, attn, res1)) return st;
    if (fg_status st = wk.dump(res1)) return st;
    cur = XB();
    attn = XB();
    if (fg_status st = wk.affine(res1, L, E, F, w1, b1, f1)) return st;
    if (fg_status st = wk.dump(f1)) return st;
    const int kind = c.activation;  // FG_RELAX_RELU / TANH / SILU
    if (fg_status st = wk.verify(kind, f1, act, "elementwise_verify")) {
      if (sentence_error(st)) { *status = st; return FG_OK; }
      return st;
    }
    if (fg_status st = wk.dump(act)) return st;
    f1 = XB();
    if (fg_status st = wk.affine(act, L, F, E, w2, b2, f2)) return st;
    if (fg_status st = wk.dump(f2)) return st;
    act = XB();
    if (fg_status st = wk.add(res1, f2, nxt)) return st;
    if (fg_status st = wk.dump(nxt)) return st;
    cur = std::move(nxt);
  }
  // MeanPool (graph.cpp:628-634): sum over positions, then scale 1/L; then the classifier head
  XB sum, pooled, logits;
  if (fg_status st = x_sum_axis(ctx, cur, 1, L, E, sum)) return st;
  if (fg_status st = wk.scale(sum, 1.0 / (double)L, pooled)) return st;
  if (fg_status st = wk.dump(pooled)) return st;
  const double* wc = params + (size_t)c.layers * per_layer;
  if (fg_status st = wk.affine(pooled, 1, E, C, wc, wc + E * C, logits)) return st;
  if (fg_status st = wk.dump(logits)) return st;
  // sink finiteness (graph.cpp:663-671) over lb, ub, lw, uw
  DBuf flag;
  CK(flag.alloc_async(sizeof(int), ctx->stream));
  CK(cudaMemsetAsync(flag.p, 0, sizeof(int), ctx->stream));
  x_finite_kernel<<<1, 64, 0, ctx->stream>>>(logits.plb(), (long long)C, flag.as<int>());
  x_finite_kernel<<<1, 64, 0, ctx->stream>>>(logits.pub(), (long long)C, flag.as<int>());
  x_finite_kernel<<<nblocks((long long)(C * D), 256), 256, 0, ctx->stream>>>(logits.plw(), (long long)(C * D),
                                                                               flag.as<int>());
  x_finite_kernel<<<nblocks((long long)(C * D), 256), 256, 0, ctx->stream>>>(logits.puw(), (long long)(C * D),
                                                                               flag.as<int>());
  ctx->launches += 4;
  DBuf lo, hi;
  if (fg_status st = x_conc(ctx, logits, norm, eps, lo, hi)) return st;
  if (job) {  // results land in the job's pinned buffer; the caller waits on job->done
    double* h = job->host;
    CK(cudaMemcpyAsync(h, lo.p, sizeof(double) * C, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(h + C, hi.p, sizeof(double) * C, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(job->hstat, dstat.p, sizeof(int) * nsites, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(job->hstat + nsites, flag.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaEventRecord(job->done, ctx->stream));
    job->nsites = nsites;
    job->classes = (int)C;
    return FG_OK;
  }
  int nonfinite = 0;
  CK(cudaMemcpyAsync(&nonfinite, flag.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(logits_lo, lo.p, sizeof(double) * C, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(logits_hi, hi.p, sizeof(double) * C, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaGetLastError());
  if (nonfinite) *status = FG_EDOMAIN;
  return FG_OK;
}

}  // namespace fgh
