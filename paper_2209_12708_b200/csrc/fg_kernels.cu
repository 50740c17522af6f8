// fg_kernels.cu -- memory-bound and f64 kernels of the B200 bound pass.
//
// Compiled with -fmad=false: the O(N) f64 scalar paths (biases, envelopes,
// softmax chain) then round exactly like the reference's host arithmetic
// (no FMA contraction), so on identical inputs they are bit-identical to
// proj/src/relax.cpp.  The dense Λ contractions live in fg_gemm.cu.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <cooperative_groups.h>

#include "fg_internal.cuh"

namespace fg {

namespace {

constexpr int kWarp = 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Dual norm q of the perturbation norm p (bounds.cpp:9-19).
__host__ __device__ __forceinline__ int dual_norm(int p) {
  return p == NORM_L1 ? NORM_LINF : (p == NORM_L2 ? NORM_L2 : NORM_L1);
}

constexpr double kNormPad = 1.0 + 0x1p-22;

// Accumulates the q-norm partials of the upper (u = c + r) and lower (l = c - r) rows.
template <int Q>
struct NormAcc {
  double u = 0.0, l = 0.0;
  __device__ __forceinline__ void add(float c, float r) {
    double dc = c, dr = r;
    double uu = dc + dr, ll = dc - dr;
    if (Q == NORM_L1) {
      u += fabs(uu);
      l += fabs(ll);
    } else if (Q == NORM_L2) {
      u += uu * uu;
      l += ll * ll;
    } else {
      u = fmax(u, fabs(uu));
      l = fmax(l, fabs(ll));
    }
  }
  __device__ __forceinline__ void add4(float4 c, float4 r) {
    add(c.x, r.x);
    add(c.y, r.y);
    add(c.z, r.z);
    add(c.w, r.w);
  }
  __device__ __forceinline__ void warp_reduce() {
    if (Q == NORM_LINF) {
      u = warp_max(u);
      l = warp_max(l);
    } else {
      u = warp_sum(u);
      l = warp_sum(l);
    }
  }
  // The finished norm carries an outward pad of 2^-22 (four f32 ulps), so every
  // concretization widens [lo, hi] by 2^-22 * eps * ||Λ|| beyond what the f32 Λ planes give: the
  // f32 storage rounding of the planes cannot pull a bound inside the exact one.
  __device__ __forceinline__ double fin(double v) const { return (Q == NORM_L2 ? sqrt(v) : v) * kNormPad; }
};

template <int Q>
__device__ __forceinline__ double qcombine(double a, double b) {
  return Q == NORM_LINF ? fmax(a, b) : a + b;
}

__device__ __forceinline__ void set_status(int* status, int s, int site, int code) {
  atomicMin(status + s, (site << 4) | code);
}

// Early exit (enqueue_pass' `skip`): this slot's pass already failed, its later results are unused.
__device__ __forceinline__ bool slot_failed(const int* skip, long long s) {
  return skip != nullptr && skip[s] != kStatusClear;
}

// ---------------------------------------------------------------------------
// Envelope lines in f64 (relax.cpp:12-108, 313-468).  Return 0, kCodeInval or
// kCodeDomain exactly where the reference throws.
// ---------------------------------------------------------------------------
struct Lines {
  double al, bl, au, bu;
};

__device__ __forceinline__ double sech2(double x) {
  double t = tanh(x);
  return 1.0 - t * t;
}

__device__ void chord(double lo, double hi, double flo, double fhi, double& a, double& b) {
  double s = (fhi - flo) / (hi - lo);
  a = s;
  b = flo - s * lo;
}

__device__ double bisect_tanh_tangent(double anchor, double blo, double bhi) {  // relax.cpp:33
  double fa = tanh(anchor);
  double a = blo, b = bhi;
  for (int it = 0; it < 60 && (b - a) > 1e-9; ++it) {
    double mid = 0.5 * (a + b);
    double g = tanh(mid) + sech2(mid) * (anchor - mid) - fa;
    if (g >= 0.0) b = mid;
    else a = mid;
  }
  return b;
}

__device__ void tanh_nonneg(double lo, double hi, double& la, double& lb, double& ua,
                            double& ub) {  // relax.cpp:56-62
  chord(lo, hi, tanh(lo), tanh(hi), la, lb);
  double m = 0.5 * (lo + hi);
  double a = sech2(m);
  ua = a;
  ub = tanh(m) - a * m;
}

__device__ Lines tanh_lines(double lo, double hi) {  // relax.cpp:64-108
  Lines r;
  if (lo == hi) {
    double a = sech2(lo);
    double b = tanh(lo) - a * lo;
    r.al = a; r.bl = b; r.au = a; r.bu = b;
    return r;
  }
  if (lo >= 0.0) {
    tanh_nonneg(lo, hi, r.al, r.bl, r.au, r.bu);
    return r;
  }
  if (hi <= 0.0) {
    double mla, mlb, mua, mub;
    tanh_nonneg(-hi, -lo, mla, mlb, mua, mub);
    r.al = mua; r.bl = -mub;
    r.au = mla; r.bu = -mlb;
    return r;
  }
  double flo = tanh(lo);
  double gap_hi = tanh(hi) + sech2(hi) * (lo - hi) - flo;
  if (gap_hi < 0.0) {
    chord(lo, hi, flo, tanh(hi), r.au, r.bu);
  } else {
    double d = bisect_tanh_tangent(lo, 0.0, hi);
    double a = sech2(d);
    r.au = a;
    r.bu = tanh(d) - a * d;
  }
  double mua, mub;
  double mflo = tanh(-hi);
  double mgap = tanh(-lo) + sech2(-lo) * (-hi + lo) - mflo;
  if (mgap < 0.0) {
    chord(-hi, -lo, mflo, tanh(-lo), mua, mub);
  } else {
    double d = bisect_tanh_tangent(-hi, 0.0, -lo);
    double a = sech2(d);
    mua = a;
    mub = tanh(d) - a * d;
  }
  r.al = mua;
  r.bl = -mub;
  return r;
}

__device__ __forceinline__ double silu_scalar(double x) { return x * (1.0 / (1.0 + exp(-x))); }
__device__ __forceinline__ double silu_derivative(double x) {
  double s = 1.0 / (1.0 + exp(-x));
  return s * (1.0 + x * (1.0 - s));
}

// ExpVerify envelope alone (relax.cpp:363-394), inlined where it sits on a per-key dependency
// chain (the three exponentials are independent and overlap).  Same arithmetic as envelope().
__device__ __forceinline__ int exp_envelope(double lo, double hi, Lines& r) {
  r.al = r.bl = r.au = r.bu = 0.0;
  if (lo > hi) return kCodeInval;
  const double m = 0.5 * (lo + hi), c2 = lo + 15.0 / 16.0;
  const double d = (c2 < m) ? c2 : m;
  const double ed = exp(d), elo = exp(lo), ehi = exp(hi);
  r.al = ed;
  r.bl = ed - ed * d;
  if (lo == hi) {
    r.au = ed;
    r.bu = ed - ed * d;
  } else {
    const double sl = (ehi - elo) / (hi - lo);
    r.au = sl;
    r.bu = elo - sl * lo;
  }
  if (!isfinite(r.bl) || !isfinite(r.au) || !isfinite(r.bu)) return kCodeDomain;
  return 0;
}

// Envelope of `kind` on [lo, hi].  For SiLU the 257-point grid (relax.cpp:452-460) is
// spread over the lanes of a warp when `lane`/`lanes` say so (min/max are exact, so the
// result does not depend on the split).
__device__ int envelope(int kind, double lo, double hi, Lines& r, int lane = 0, int lanes = 1) {
  r.al = r.bl = r.au = r.bu = 0.0;
  if (lo > hi) return kCodeInval;  // ConcreteBounds::validate (bounds.cpp:69-78)
  switch (kind) {
    case RELAX_RELU:  // relax.cpp:313-337
      if (lo >= 0.0) {
        r.al = 1.0;
        r.au = 1.0;
      } else if (hi <= 0.0) {
      } else {
        double s = hi / (hi - lo);
        r.au = s;
        r.bu = -s * lo;
        r.al = (fabs(lo) > fabs(hi)) ? 0.0 : 1.0;
      }
      return 0;
    case RELAX_TANH:
      r = tanh_lines(lo, hi);
      return 0;
    case RELAX_EXP: {  // relax.cpp:363-394
      double m = 0.5 * (lo + hi), c2 = lo + 15.0 / 16.0;
      double d = (c2 < m) ? c2 : m;
      double ed = exp(d);
      r.al = ed;
      r.bl = ed - ed * d;
      if (lo == hi) {
        r.au = ed;
        r.bu = ed - ed * d;
      } else {
        chord(lo, hi, exp(lo), exp(hi), r.au, r.bu);
      }
      if (!isfinite(r.bl) || !isfinite(r.au) || !isfinite(r.bu)) return kCodeDomain;
      return 0;
    }
    case RELAX_RECIP: {  // relax.cpp:396-424
      if (lo <= 0.0) return kCodeDomain;
      double m = 0.5 * (lo + hi);
      double am = -1.0 / (m * m);
      r.al = am;
      r.bl = 2.0 / m;
      if (lo == hi) {
        r.au = am;
        r.bu = 2.0 / m;
      } else {
        chord(lo, hi, 1.0 / lo, 1.0 / hi, r.au, r.bu);
      }
      return 0;
    }
    case RELAX_SQRT: {  // extension: concave on [0, inf) -> lower chord, upper tangent at the midpoint
      if (lo < 0.0) return kCodeDomain;
      const double m = 0.5 * (lo + hi);
      if (m == 0.0) return 0;  // lo = hi = 0: the zero lines are exact
      const double sm = sqrt(m);
      r.au = 0.5 / sm;
      r.bu = 0.5 * sm;  // sqrt(m) - m / (2 sqrt(m))
      if (lo == hi) {
        r.al = r.au;
        r.bl = r.bu;
      } else {
        chord(lo, hi, sqrt(lo), sqrt(hi), r.al, r.bl);
      }
      if (!isfinite(r.au) || !isfinite(r.bu) || !isfinite(r.al) || !isfinite(r.bl)) return kCodeDomain;
      return 0;
    }
    case RELAX_SQUARE: {  // extension: convex -> lower tangent at the midpoint, upper chord
      const double m = 0.5 * (lo + hi);
      r.al = 2.0 * m;
      r.bl = -m * m;
      if (lo == hi) {
        r.au = r.al;
        r.bu = r.bl;
      } else {
        r.au = lo + hi;  // chord of x^2: slope (hi^2 - lo^2) / (hi - lo), intercept -lo * hi
        r.bu = -lo * hi;
      }
      if (!isfinite(r.al) || !isfinite(r.bl) || !isfinite(r.au) || !isfinite(r.bu)) return kCodeDomain;
      return 0;
    }
    case RELAX_SILU: {  // relax.cpp:426-468
      if (lo == hi) {
        double a = silu_derivative(lo);
        r.al = a;
        r.au = a;
        r.bl = silu_scalar(lo) - a * lo;
        r.bu = r.bl;
        return 0;
      }
      double s = (silu_scalar(hi) - silu_scalar(lo)) / (hi - lo);
      double step = (hi - lo) / 256;
      double gmin = HUGE_VAL, gmax = -HUGE_VAL;
      for (int k = lane; k <= 256; k += lanes) {
        double x = (k == 256) ? hi : lo + step * k;
        double g = silu_scalar(x) - s * x;
        gmin = fmin(gmin, g);
        gmax = fmax(gmax, g);
      }
      if (lanes > 1) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          gmin = fmin(gmin, __shfl_xor_sync(0xffffffffu, gmin, o));
          gmax = fmax(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
        }
      }
      double margin = 0.6 * step * step / 8.0 + 1e-12;
      r.al = s;
      r.au = s;
      r.bl = gmin - margin;
      r.bu = gmax + margin;
      return 0;
    }
  }
  return kCodeInval;
}

// Rows whose relaxation keeps (al = au = 1: a stably active ReLU) or zeroes (al = au = 0: stably
// inactive) the row's Λ need no compose sweep when the consumer is told which rows are zero:
// keep[row] = 0 for a zero row (its stale Λ is masked by the consumer), 1 otherwise.  Near a
// sentence's certified radius almost every ReLU neuron is stable (c3: 99 %, about half each way).
__device__ __forceinline__ bool lines_identity(const Lines& e) { return e.al == 1.0 && e.au == 1.0; }
__device__ __forceinline__ bool lines_zero(const Lines& e) { return e.al == 0.0 && e.au == 0.0; }

// compose_elementwise on one element (relax.cpp:484-494) in center/radius form.
__device__ __forceinline__ void compose_cr(const Lines& e, float c, float r, float& oc,
                                           float& orr) {
  double dc = c, dr = r;
  double u = dc + dr, l = dc - dr;
  double yu = e.au * (e.au >= 0.0 ? u : l);
  double yl = e.al * (e.al >= 0.0 ? l : u);
  oc = (float)(0.5 * (yu + yl));
  orr = (float)(0.5 * (yu - yl));
}

// ---------------------------------------------------------------------------
// concretize (bounds.cpp:122-140): one warp per neuron row.
// ---------------------------------------------------------------------------
template <int Q>
__global__ void __launch_bounds__(256) concretize_kernel(const float* __restrict__ lam, long long cr,
                                                         const double* __restrict__ lb,
                                                         const double* __restrict__ ub,
                                                         long long rows_per_s, long long nrows, int D,
                                                         const double* __restrict__ eps,
                                                         double* __restrict__ lo,
                                                         double* __restrict__ hi, const int* __restrict__ skip) {
  long long row = (long long)blockIdx.x * (blockDim.x / kWarp) + threadIdx.x / kWarp;
  int lane = threadIdx.x & (kWarp - 1);
  if (row >= nrows || slot_failed(skip, row / rows_per_s)) return;
  const float* c = lam + row * D;
  const float* r = c + cr;
  NormAcc<Q> acc;
  for (int d = lane * 4; d < D; d += 4 * kWarp)
    acc.add4(*reinterpret_cast<const float4*>(c + d), *reinterpret_cast<const float4*>(r + d));
  acc.warp_reduce();
  if (lane == 0) {
    double e = eps[row / rows_per_s];
    lo[row] = lb[row] - e * acc.fin(acc.l);
    hi[row] = ub[row] + e * acc.fin(acc.u);
  }
}

// concretize of a token-row tensor whose Λ rows are zero outside the perturbed tokens (the
// first layer's Q/K/V under the one-hot binding): unperturbed rows get lo = lb, hi = ub
// (eps * ||0|| = 0 exactly) without reading Λ.  row = (s, token, f), f < width.
template <int Q>
__global__ void __launch_bounds__(256) concretize_tokens_kernel(
    const float* __restrict__ lam, long long cr, const double* __restrict__ lb, const double* __restrict__ ub,
    long long rows_per_s, long long nrows, int D, const double* __restrict__ eps, double* __restrict__ lo,
    double* __restrict__ hi, const int* __restrict__ positions, const int* __restrict__ slot_map, int W, int width) {
  long long row = (long long)blockIdx.x * (blockDim.x / kWarp) + threadIdx.x / kWarp;
  int lane = threadIdx.x & (kWarp - 1);
  if (row >= nrows) return;
  const long long s = row / rows_per_s;
  const int tok = (int)((row % rows_per_s) / width);
  const int src = slot_map[s];
  bool hot = false;
  for (int q = 0; q < W; ++q) hot |= positions[src * W + q] == tok;
  if (!hot) {
    if (lane == 0) {
      lo[row] = lb[row];
      hi[row] = ub[row];
    }
    return;
  }
  const float* c = lam + row * D;
  const float* r = c + cr;
  NormAcc<Q> acc;
  for (int d = lane * 4; d < D; d += 4 * kWarp)
    acc.add4(*reinterpret_cast<const float4*>(c + d), *reinterpret_cast<const float4*>(r + d));
  acc.warp_reduce();
  if (lane == 0) {
    double e = eps[s];
    lo[row] = lb[row] - e * acc.fin(acc.l);
    hi[row] = ub[row] + e * acc.fin(acc.u);
  }
}

// The same in two launches: unperturbed rows copied one thread per row, perturbed rows (W per
// sentence and feature) reduced one warp per row -- instead of a warp per row for all of them,
// most of which only copy two doubles.
__global__ void __launch_bounds__(256) concretize_cold_kernel(const double* __restrict__ lb,
                                                              const double* __restrict__ ub, long long rows_per_s,
                                                              long long nrows, double* __restrict__ lo,
                                                              double* __restrict__ hi, const int* __restrict__ positions,
                                                              const int* __restrict__ slot_map, int W, int width) {
  const long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= nrows) return;
  const long long s = row / rows_per_s;
  const int tok = (int)((row % rows_per_s) / width);
  const int src = slot_map[s];
  bool hot = false;
  for (int q = 0; q < W; ++q) hot |= positions[src * W + q] == tok;
  if (!hot) {
    lo[row] = lb[row];
    hi[row] = ub[row];
  }
}

template <int Q>
__global__ void __launch_bounds__(256) concretize_hot_kernel(
    const float* __restrict__ lam, long long cr, const double* __restrict__ lb, const double* __restrict__ ub,
    long long rows_per_s, int S, int D, const double* __restrict__ eps, double* __restrict__ lo,
    double* __restrict__ hi, const int* __restrict__ positions, const int* __restrict__ slot_map, int W, int width) {
  const long long hid = (long long)blockIdx.x * (blockDim.x / kWarp) + threadIdx.x / kWarp;  // (s, q, f)
  const int lane = threadIdx.x & (kWarp - 1);
  if (hid >= (long long)S * W * width) return;
  const int f = (int)(hid % width), q = (int)((hid / width) % W);
  const long long s = hid / ((long long)W * width);
  const int tok = positions[slot_map[s] * W + q];
  const long long row = s * rows_per_s + (long long)tok * width + f;
  const float* c = lam + row * D;
  const float* r = c + cr;
  NormAcc<Q> acc;
  for (int d = lane * 4; d < D; d += 4 * kWarp)
    acc.add4(*reinterpret_cast<const float4*>(c + d), *reinterpret_cast<const float4*>(r + d));
  acc.warp_reduce();
  if (lane == 0) {
    const double e = eps[s];
    lo[row] = lb[row] - e * acc.fin(acc.l);
    hi[row] = ub[row] + e * acc.fin(acc.u);
  }
}

// ---------------------------------------------------------------------------
// elementwise_verify (graph.cpp:484-501) fused: concretize -> envelope -> compose,
// in place, one warp per neuron row.  Λ is read from HBM once (the second sweep
// re-reads the warp's own row from L1/L2) and written once.
// ---------------------------------------------------------------------------
template <int Q>
__global__ void __launch_bounds__(256) elementwise_verify_kernel(
    int kind, float* __restrict__ lam, long long cr, double* __restrict__ lb, double* __restrict__ ub,
    long long rows_per_s, long long nrows, int D, const double* __restrict__ eps,
    int* __restrict__ status, int site, double* __restrict__ lo_out, double* __restrict__ hi_out,
    const double* __restrict__ lo_in, const double* __restrict__ hi_in, const int* __restrict__ skip,
    unsigned char* __restrict__ keep) {
  long long row = (long long)blockIdx.x * (blockDim.x / kWarp) + threadIdx.x / kWarp;
  int lane = threadIdx.x & (kWarp - 1);
  if (row >= nrows || slot_failed(skip, row / rows_per_s)) return;
  float* c = lam + row * D;
  float* r = c + cr;
  long long s = row / rows_per_s;
  double xlb = lb[row], xub = ub[row];
  double lo, hi;
  if (lo_in) {  // concretized elsewhere (column-sharded pass: norms all-reduced across ranks)
    lo = lo_in[row];
    hi = hi_in[row];
  } else {
    NormAcc<Q> acc;
    for (int d = lane * 4; d < D; d += 4 * kWarp)
      acc.add4(*reinterpret_cast<const float4*>(c + d), *reinterpret_cast<const float4*>(r + d));
    acc.warp_reduce();
    double e = eps[s];
    lo = xlb - e * acc.fin(acc.l);
    hi = xub + e * acc.fin(acc.u);
  }
  Lines ln;
  int code = envelope(kind, lo, hi, ln, lane, kind == RELAX_SILU ? kWarp : 1);
  if (lane == 0) {
    if (code) set_status(status, (int)s, site, code);
    if (lo_out) {
      lo_out[row] = lo;
      hi_out[row] = hi;
    }
    ub[row] = ln.au * (ln.au >= 0.0 ? xub : xlb) + ln.bu;
    lb[row] = ln.al * (ln.al >= 0.0 ? xlb : xub) + ln.bl;
  }
  if (keep) {  // warp-uniform: every lane holds the same lines
    const bool zero = lines_zero(ln);
    if (lane == 0) keep[row] = zero ? 0 : 1;
    if (zero || lines_identity(ln)) return;
  }
  for (int d = lane * 4; d < D; d += 4 * kWarp) {
    float4 cv = *reinterpret_cast<const float4*>(c + d);
    float4 rv = *reinterpret_cast<const float4*>(r + d);
    float4 oc, orr;
    compose_cr(ln, cv.x, rv.x, oc.x, orr.x);
    compose_cr(ln, cv.y, rv.y, oc.y, orr.y);
    compose_cr(ln, cv.z, rv.z, oc.z, orr.z);
    compose_cr(ln, cv.w, rv.w, oc.w, orr.w);
    *reinterpret_cast<float4*>(c + d) = oc;
    *reinterpret_cast<float4*>(r + d) = orr;
  }
}

// Narrow rows (D <= 256: one or two float4 per lane and plane): two rows per warp, their loads
// issued together so each warp keeps twice the bytes in flight through the reductions and the
// f64 envelope.  Per row the arithmetic (lane partial order, butterfly, envelope) is that of
// concretize_kernel / elementwise_verify_kernel, so results are bit-identical.
template <int Q>
__global__ void __launch_bounds__(256) concretize_rows2_kernel(const float* __restrict__ lam, long long cr,
                                                               const double* __restrict__ lb,
                                                               const double* __restrict__ ub, long long rows_per_s,
                                                               long long nrows, int D, const double* __restrict__ eps,
                                                               double* __restrict__ lo, double* __restrict__ hi,
                                                               const int* __restrict__ skip) {
  const long long row0 = 2 * ((long long)blockIdx.x * (blockDim.x / kWarp) + threadIdx.x / kWarp);
  const int lane = threadIdx.x & (kWarp - 1);
  if (row0 >= nrows) return;
  const bool two = row0 + 1 < nrows;
  if (slot_failed(skip, row0 / rows_per_s) && (!two || slot_failed(skip, (row0 + 1) / rows_per_s))) return;
  NormAcc<Q> acc[2];
  for (int d = lane * 4; d < D; d += 4 * kWarp) {
    const float* c0 = lam + row0 * D + d;
    const float4 c0v = *reinterpret_cast<const float4*>(c0), r0v = *reinterpret_cast<const float4*>(c0 + cr);
    float4 c1v = make_float4(0.f, 0.f, 0.f, 0.f), r1v = c1v;
    if (two) {
      c1v = *reinterpret_cast<const float4*>(c0 + D);
      r1v = *reinterpret_cast<const float4*>(c0 + D + cr);
    }
    acc[0].add4(c0v, r0v);
    acc[1].add4(c1v, r1v);
  }
  acc[0].warp_reduce();
  acc[1].warp_reduce();
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const long long row = row0 + q;
      if (row >= nrows) break;
      const double e = eps[row / rows_per_s];
      lo[row] = lb[row] - e * acc[q].fin(acc[q].l);
      hi[row] = ub[row] + e * acc[q].fin(acc[q].u);
    }
  }
}

template <int Q>
__global__ void __launch_bounds__(256) elementwise_verify_rows2_kernel(
    int kind, float* __restrict__ lam, long long cr, double* __restrict__ lb, double* __restrict__ ub,
    long long rows_per_s, long long nrows, int D, const double* __restrict__ eps, int* __restrict__ status, int site,
    double* __restrict__ lo_out, double* __restrict__ hi_out, const int* __restrict__ skip,
    unsigned char* __restrict__ keep) {
  const long long row0 = 2 * ((long long)blockIdx.x * (blockDim.x / kWarp) + threadIdx.x / kWarp);
  const int lane = threadIdx.x & (kWarp - 1);
  if (row0 >= nrows) return;
  const int nr = row0 + 1 < nrows ? 2 : 1;
  if (slot_failed(skip, row0 / rows_per_s) && (nr == 1 || slot_failed(skip, (row0 + 1) / rows_per_s))) return;
  NormAcc<Q> acc[2];
  for (int d = lane * 4; d < D; d += 4 * kWarp) {
    const float* c0 = lam + row0 * D + d;
    const float4 c0v = *reinterpret_cast<const float4*>(c0), r0v = *reinterpret_cast<const float4*>(c0 + cr);
    float4 c1v = make_float4(0.f, 0.f, 0.f, 0.f), r1v = c1v;
    if (nr == 2) {
      c1v = *reinterpret_cast<const float4*>(c0 + D);
      r1v = *reinterpret_cast<const float4*>(c0 + D + cr);
    }
    acc[0].add4(c0v, r0v);
    acc[1].add4(c1v, r1v);
  }
  acc[0].warp_reduce();
  acc[1].warp_reduce();
  Lines ln[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    if (q >= nr) break;
    const long long row = row0 + q;
    const long long s = row / rows_per_s;
    const double xlb = lb[row], xub = ub[row];
    const double e = eps[s];
    const double lo = xlb - e * acc[q].fin(acc[q].l);
    const double hi = xub + e * acc[q].fin(acc[q].u);
    const int code = envelope(kind, lo, hi, ln[q], lane, kind == RELAX_SILU ? kWarp : 1);
    if (lane == 0) {
      if (code) set_status(status, (int)s, site, code);
      if (lo_out) {
        lo_out[row] = lo;
        hi_out[row] = hi;
      }
      ub[row] = ln[q].au * (ln[q].au >= 0.0 ? xub : xlb) + ln[q].bu;
      lb[row] = ln[q].al * (ln[q].al >= 0.0 ? xlb : xub) + ln[q].bl;
    }
  }
  bool sweep[2] = {true, true};
  if (keep) {  // LamGemm::kmask consumer: zero rows flagged, identity / zero rows not rewritten
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (q >= nr) break;
      const bool zero = lines_zero(ln[q]);
      if (lane == 0) keep[row0 + q] = zero ? 0 : 1;
      sweep[q] = !(zero || lines_identity(ln[q]));
    }
    if (!sweep[0] && (nr == 1 || !sweep[1])) return;
  }
  for (int d = lane * 4; d < D; d += 4 * kWarp) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (q >= nr || !sweep[q]) continue;
      float* c = lam + (row0 + q) * D + d;
      const float4 cv = *reinterpret_cast<const float4*>(c), rv = *reinterpret_cast<const float4*>(c + cr);
      float4 oc, orr;
      compose_cr(ln[q], cv.x, rv.x, oc.x, orr.x);
      compose_cr(ln[q], cv.y, rv.y, oc.y, orr.y);
      compose_cr(ln[q], cv.z, rv.z, oc.z, orr.z);
      compose_cr(ln[q], cv.w, rv.w, oc.w, orr.w);
      *reinterpret_cast<float4*>(c) = oc;
      *reinterpret_cast<float4*>(c + cr) = orr;
    }
  }
}

__global__ void relax_kernel(int kind, const double* lo, const double* hi, long long n,
                             double* al, double* bl, double* au, double* bu, int* status) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  Lines ln;
  int code = envelope(kind, lo[i], hi[i], ln);
  if (code) set_status(status, 0, 0, code);
  al[i] = ln.al; bl[i] = ln.bl; au[i] = ln.au; bu[i] = ln.bu;
}

__global__ void compose_kernel(const float* __restrict__ lin, long long crin, const double* lbin,
                               const double* ubin, const double* al, const double* bl,
                               const double* au, const double* bu, float* __restrict__ lout,
                               long long crout, double* lbout, double* ubout, long long n, int D) {
  long long row = (long long)blockIdx.x * (blockDim.x / kWarp) + threadIdx.x / kWarp;
  int lane = threadIdx.x & (kWarp - 1);
  if (row >= n) return;
  Lines ln{al[row], bl[row], au[row], bu[row]};
  if (lane == 0) {
    double xlb = lbin[row], xub = ubin[row];
    ubout[row] = ln.au * (ln.au >= 0.0 ? xub : xlb) + ln.bu;
    lbout[row] = ln.al * (ln.al >= 0.0 ? xlb : xub) + ln.bl;
  }
  const float* c = lin + row * D;
  float* oc = lout + row * D;
  for (int d = lane; d < D; d += kWarp) compose_cr(ln, c[d], c[d + crin], oc[d], oc[d + crout]);
}

// ---------------------------------------------------------------------------
// Affine bias path (relax.cpp:273-299) in f64: one thread per output neuron,
// i accumulated in the reference's order; optional residual propagate_add(res, y).
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// Affine bias in f64 (relax.cpp:280-303 on the O(N) part): per token row r and output j
//   ub' = sum_i (W > 0 ? W ub : W lb) + b,   lb' = sum_i (W > 0 ? W lb : W ub) + b  (+ residual)
// as the two FP64 products  m = W . mid,  q = |W| . rad  (mid = (lb + ub) / 2, rad = (ub - lb) / 2,
// ub' = m + q + b, lb' = m - q + b): the same sums without a per-term sign select, so the kernel
// is a register-tiled DFMA GEMM (rows x outputs, K = inputs).  CTA tile 64 rows x 64 outputs,
// 16-deep K chunks staged in shared memory (W and |W|, mid and rad), thread tile 4 x 4 with rows
// {2ty, 2ty + 1, 32 + 2ty, 33 + 2ty} and outputs likewise in tx (double2 loads, conflict-free).
// Rounding differs from the reference's four sign-half sums by f64 ulps, far inside the fused
// pass's f32 error band (the exact mode keeps the reference's order, fg_exact.cu).
// ---------------------------------------------------------------------------
constexpr int kBgR = 64, kBgJ = 64, kBgK = 16;
constexpr int kBgS = 68;  // padded SMEM row (doubles): conflict-free DMMA fragment loads (68 = 4 mod 16)

// f64 tensor-core version (DMMA m8n8k4): CTA tile 64 rows x 64 outputs, 8 warps as 2 x 4, warp
// tile 32 x 16 = 4 x 2 MMA tiles of 8 x 8 per product; K chunks of 16 staged k-major in shared
// memory (mid, rad rows; W, |W| columns), the next chunk prefetched into registers.
// Fragments (PTX mma.m8n8k4 .f64): A[r][k] with r = lane >> 2, k = lane & 3; B[k][n] with
// k = lane & 3, n = lane >> 2; C[r][2 (lane & 3) + i].
__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(256) affine_bias_kernel(
    const double* __restrict__ lb_in, const double* __restrict__ ub_in, const double* __restrict__ w,
    const double* __restrict__ bias, const double* __restrict__ res_lb, const double* __restrict__ res_ub,
    double* __restrict__ lb_out, double* __restrict__ ub_out, long long nrows, int C, int O,
    const int* __restrict__ skip, int rows_per_slot) {
  __shared__ __align__(16) double sM[kBgK][kBgS];
  __shared__ __align__(16) double sR[kBgK][kBgS];
  __shared__ __align__(16) double sW[kBgK][kBgS];
  __shared__ __align__(16) double sA[kBgK][kBgS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wr = warp >> 2, wc = warp & 3;  // warp tile rows 32 wr.., outputs 16 wc..
  const long long r0 = (long long)blockIdx.y * kBgR;
  const int j0 = blockIdx.x * kBgJ;
  // every row of the CTA in failed slots (block-uniform test)
  if (skip && slot_failed(skip, r0 / rows_per_slot) &&
      slot_failed(skip, (min(r0 + kBgR, nrows) - 1) / rows_per_slot))
    return;
  double am[4][2][2], aq[4][2][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) am[a][b][0] = am[a][b][1] = aq[a][b][0] = aq[a][b][1] = 0.0;
  // staging: element e = threadIdx.x + 256 p (p < 4) of the chunk; (lb, ub) with K fastest
  // (k = e % 16, row = e / 16: coalesced 128 B row segments), W with outputs fastest
  double pl[4], pu[4], pw[4];
  auto load = [&](int k0) {
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int e = threadIdx.x + 256 * p;
      const int k = e % kBgK, r = e / kBgK;
      const bool ok = r0 + r < nrows && k0 + k < C;
      pl[p] = ok ? lb_in[(r0 + r) * C + k0 + k] : 0.0;
      pu[p] = ok ? ub_in[(r0 + r) * C + k0 + k] : 0.0;
      const int j = e % kBgJ, kw = e / kBgJ;
      pw[p] = (k0 + kw < C && j0 + j < O) ? w[(long long)(k0 + kw) * O + j0 + j] : 0.0;
    }
  };
  load(0);
  const int fr = lane >> 2, fk = lane & 3;
  for (int k0 = 0; k0 < C; k0 += kBgK) {
    __syncthreads();
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int e = threadIdx.x + 256 * p;
      sM[e % kBgK][e / kBgK] = 0.5 * (pl[p] + pu[p]);
      sR[e % kBgK][e / kBgK] = 0.5 * (pu[p] - pl[p]);
      sW[e / kBgJ][e % kBgJ] = pw[p];
      sA[e / kBgJ][e % kBgJ] = fabs(pw[p]);
    }
    __syncthreads();
    if (k0 + kBgK < C) load(k0 + kBgK);
#pragma unroll
    for (int ks = 0; ks < kBgK; ks += 4) {
      double fm[4], fq[4], fw[2], fa[2];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        fm[a] = sM[ks + fk][wr * 32 + a * 8 + fr];
        fq[a] = sR[ks + fk][wr * 32 + a * 8 + fr];
      }
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        fw[b] = sW[ks + fk][wc * 16 + b * 8 + fr];
        fa[b] = sA[ks + fk][wc * 16 + b * 8 + fr];
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          dmma884(am[a][b], fm[a], fw[b]);
          dmma884(aq[a][b], fq[a], fa[b]);
        }
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const long long row = r0 + wr * 32 + a * 8 + fr;
    if (row >= nrows) continue;
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int j = j0 + wc * 16 + b * 8 + 2 * fk + i;
        if (j >= O) continue;
        const double bv = bias ? bias[j] : 0.0;
        const long long t = row * O + j;
        double yub = (am[a][b][i] + aq[a][b][i]) + bv;
        double ylb = (am[a][b][i] - aq[a][b][i]) + bv;
        if (res_lb) {  // propagate_add(res, y) (relax.cpp:666-667)
          yub = res_ub[t] + yub;
          ylb = res_lb[t] + ylb;
        }
        ub_out[t] = yub;
        lb_out[t] = ylb;
      }
  }
}

// ---------------------------------------------------------------------------
// McCormick dot products (relax.cpp:533-654).
// In center/radius form the Λ part of each product term splits into dense
// contractions: with (lx, ly, uy) = (lo x, lo y, hi y),
//   x-side:  c += ((ly+uy)/2) xc + ((|uy|-|ly|)/2) xr,   r += ((uy-ly)/2) xc + ((|uy|+|ly|)/2) xr
//   y-side:  c += lx yc,                                  r += |lx| yr
// The coefficient matrices are built here (f32) and contracted by launch_gemm.
// ---------------------------------------------------------------------------
__device__ __forceinline__ long long nidx(const NView& v, long long s, long long row, int f) {
  return s * v.s_stride + row * v.row_stride + v.col0 + f;
}

// per (s,h): A1 [2][2hd][L] (x-side coefficients for K rows j), A2 [2][hd][L] (lx for Q rows i)
__global__ void sim_coef_kernel(NView q, NView k, int H, int L, int hd, float* ws) {
  int sh = blockIdx.x;
  int s = sh / H, h = sh % H;
  float* a1 = ws + (long long)sh * 6 * hd * L;
  float* a2 = a1 + 4LL * hd * L;
  for (int t = threadIdx.x; t < hd * L; t += blockDim.x) {
    int kk = t / L, m = t % L;  // m: key row j for A1, query row i for A2
    long long yi = nidx(k, s, m, h * hd + kk);
    double ly = k.lo[yi], uy = k.hi[yi];
    a1[(0 * 2 * hd + kk) * L + m] = (float)(0.5 * (ly + uy));
    a1[(0 * 2 * hd + hd + kk) * L + m] = (float)(0.5 * (fabs(uy) - fabs(ly)));
    a1[(1 * 2 * hd + kk) * L + m] = (float)(0.5 * (uy - ly));
    a1[(1 * 2 * hd + hd + kk) * L + m] = (float)(0.5 * (fabs(uy) + fabs(ly)));
    double lx = q.lo[nidx(q, s, m, h * hd + kk)];
    a2[(0 * hd + kk) * L + m] = (float)lx;
    a2[(1 * hd + kk) * L + m] = (float)fabs(lx);
  }
}

// per (s,h): B1 [2][2L][hd] (x-side coefficients from V rows), B2 [2][L][L] (lx of P)
__global__ void wv_coef_kernel(NView p, NView v, int H, int L, int hd, float* ws) {
  int sh = blockIdx.x;
  int s = sh / H, h = sh % H;
  long long per = 4LL * L * hd + 2LL * L * L;
  float* b1 = ws + (long long)sh * per;
  float* b2 = b1 + 4LL * L * hd;
  for (int t = threadIdx.x; t < L * hd; t += blockDim.x) {
    int j = t / hd, kk = t % hd;
    long long yi = nidx(v, s, j, h * hd + kk);
    double ly = v.lo[yi], uy = v.hi[yi];
    b1[(0 * 2 * L + j) * hd + kk] = (float)(0.5 * (ly + uy));
    b1[(0 * 2 * L + L + j) * hd + kk] = (float)(0.5 * (fabs(uy) - fabs(ly)));
    b1[(1 * 2 * L + j) * hd + kk] = (float)(0.5 * (uy - ly));
    b1[(1 * 2 * L + L + j) * hd + kk] = (float)(0.5 * (fabs(uy) + fabs(ly)));
  }
  for (int t = threadIdx.x; t < L * L; t += blockDim.x) {
    int j = t / L, i = t % L;
    double lx = p.lo[nidx(p, s, (long long)h * L + i, j)];
    b2[(0 * L + j) * L + i] = (float)lx;
    b2[(1 * L + j) * L + i] = (float)fabs(lx);
  }
}

// One McCormick product term's bias contribution (relax.cpp:546-547, 560-561).
__device__ __forceinline__ void term_bias(double lx, double ly, double uy, double xlb, double xub,
                                          double ylb, double yub, double& olb, double& oub) {
  {
    double cx = ly, cy = lx;
    olb += cx * ((cx >= 0.0) ? xlb : xub) + cy * ((cy >= 0.0) ? ylb : yub) - lx * ly;
  }
  {
    double cx = uy, cy = lx;
    oub += cx * ((cx >= 0.0) ? xub : xlb) + cy * ((cy >= 0.0) ? yub : ylb) - lx * uy;
  }
}

// McCormick product biases as a tiled f64 kernel (relax.cpp:546-547, 560-561, 635-651):
//   out[a, b] = scale * sum_c term(X[a, c], Y[b, c])     c ascending (the reference order)
// similarity: a = query row i, b = key row j, c = head feature kk   (X = Q, Y = K)
// weighted:   a = query row i, b = head feature kk, c = key row j   (X = P, Y = V)
// One CTA per (sentence, head, 32 a x 64 b tile); c is staged through shared memory in chunks
// of 16, so every Y element is read from HBM/L2 once per tile and reused by 32 outputs.
struct McBias {
  const double *xlo, *xlb, *xub, *ylo, *yhi, *ylb, *yub;
  double *olb, *oub;
  long long xs, ys, os;  // per-sentence strides
  long long xh, yh, oh;  // per-head offsets
  long long xa, xc, yb, yc, oa, ob;
  int H, A, B, C;
  double scale;
};

constexpr int kMbA = 32, kMbB = 64, kMbC = 16, kMbThreads = 256, kMbR = kMbA / (kMbThreads / kMbB);

__global__ void __launch_bounds__(kMbThreads) mc_bias_kernel(McBias p) {
  __shared__ double ys[4][kMbC][kMbB];
  __shared__ double xs[3][kMbC][kMbA];
  const int ta = (p.A + kMbA - 1) / kMbA, tb = (p.B + kMbB - 1) / kMbB;
  long long blk = blockIdx.x;
  const int bt = (int)(blk % tb);
  blk /= tb;
  const int at = (int)(blk % ta);
  blk /= ta;
  const int h = (int)(blk % p.H);
  const long long s = blk / p.H;
  const int a0 = at * kMbA, b0 = bt * kMbB;
  const long long xbase = s * p.xs + h * p.xh, ybase = s * p.ys + h * p.yh;
  const int tid = threadIdx.x, bl = tid % kMbB, ag = tid / kMbB;
  double olb[kMbR], oub[kMbR];
#pragma unroll
  for (int r = 0; r < kMbR; ++r) olb[r] = oub[r] = 0.0;
  for (int c0 = 0; c0 < p.C; c0 += kMbC) {
    const int nc = min(kMbC, p.C - c0);
    __syncthreads();
    for (int idx = tid; idx < kMbC * kMbB; idx += kMbThreads) {
      int b, c;
      if (p.yc == 1) c = idx % kMbC, b = idx / kMbC;
      else b = idx % kMbB, c = idx / kMbB;
      if (c < nc && b0 + b < p.B) {
        const long long g = ybase + (long long)(b0 + b) * p.yb + (long long)(c0 + c) * p.yc;
        ys[0][c][b] = p.ylo[g];
        ys[1][c][b] = p.yhi[g];
        ys[2][c][b] = p.ylb[g];
        ys[3][c][b] = p.yub[g];
      }
    }
    for (int idx = tid; idx < kMbC * kMbA; idx += kMbThreads) {
      const int c = idx % kMbC, a = idx / kMbC;
      if (c < nc && a0 + a < p.A) {
        const long long g = xbase + (long long)(a0 + a) * p.xa + (long long)(c0 + c) * p.xc;
        xs[0][c][a] = p.xlo[g];
        xs[1][c][a] = p.xlb[g];
        xs[2][c][a] = p.xub[g];
      }
    }
    __syncthreads();
    for (int c = 0; c < nc; ++c) {
      const double ly = ys[0][c][bl], uy = ys[1][c][bl], ylb = ys[2][c][bl], yub = ys[3][c][bl];
#pragma unroll
      for (int r = 0; r < kMbR; ++r) {
        const int a = ag * kMbR + r;
        term_bias(xs[0][c][a], ly, uy, xs[1][c][a], xs[2][c][a], ylb, yub, olb[r], oub[r]);
      }
    }
  }
  if (b0 + bl >= p.B) return;
#pragma unroll
  for (int r = 0; r < kMbR; ++r) {
    const int a = a0 + ag * kMbR + r;
    if (a >= p.A) break;
    const long long o = s * p.os + h * p.oh + (long long)a * p.oa + (long long)(b0 + bl) * p.ob;
    p.olb[o] = p.scale * olb[r];
    p.oub[o] = p.scale * oub[r];
  }
}

// scores bias for (s,h,i,j), then the Scale node (propagate_scale, relax.cpp:683-687)
void sim_bias(const NView& q, const NView& k, const NView& out, int S, int H, int L, int hd, double scale,
              cudaStream_t st) {
  McBias p{q.lo, q.lb, q.ub, k.lo, k.hi, k.lb, k.ub, out.lb, out.ub};
  p.xs = q.s_stride; p.ys = k.s_stride; p.os = out.s_stride;
  p.xh = hd; p.yh = hd; p.oh = (long long)L * out.row_stride;
  p.xlo += q.col0; p.xlb += q.col0; p.xub += q.col0;
  p.ylo += k.col0; p.yhi += k.col0; p.ylb += k.col0; p.yub += k.col0;
  p.olb += out.col0; p.oub += out.col0;
  p.xa = q.row_stride; p.xc = 1; p.yb = k.row_stride; p.yc = 1; p.oa = out.row_stride; p.ob = 1;
  p.H = H; p.A = L; p.B = L; p.C = hd; p.scale = scale;
  const long long blocks = (long long)S * H * ((L + kMbA - 1) / kMbA) * ((L + kMbB - 1) / kMbB);
  mc_bias_kernel<<<(unsigned)blocks, kMbThreads, 0, st>>>(p);
}

// context bias for (s,i,h,k): sum over key rows j (relax.cpp:635-651)
void wv_bias(const NView& pv, const NView& v, const NView& out, int S, int H, int L, int hd, cudaStream_t st) {
  McBias p{pv.lo, pv.lb, pv.ub, v.lo, v.hi, v.lb, v.ub, out.lb, out.ub};
  p.xs = pv.s_stride; p.ys = v.s_stride; p.os = out.s_stride;
  p.xh = (long long)L * pv.row_stride; p.yh = hd; p.oh = hd;
  p.xlo += pv.col0; p.xlb += pv.col0; p.xub += pv.col0;
  p.ylo += v.col0; p.yhi += v.col0; p.ylb += v.col0; p.yub += v.col0;
  p.olb += out.col0; p.oub += out.col0;
  p.xa = pv.row_stride; p.xc = 1; p.yb = 1; p.yc = v.row_stride; p.oa = out.row_stride; p.ob = 1;
  p.H = H; p.A = L; p.B = hd; p.C = L; p.scale = 1.0;
  const long long blocks = (long long)S * H * ((L + kMbA - 1) / kMbA) * ((hd + kMbB - 1) / kMbB);
  mc_bias_kernel<<<(unsigned)blocks, kMbThreads, 0, st>>>(p);
}

// ---------------------------------------------------------------------------
// Softmax chain (graph.cpp:237-240 -> relax.cpp:363-394, 705-742, 396-424, 744-775),
// per (sentence, score row), in place: exp envelope per key -> Σ_j e_j -> recip envelope ->
// McCormick e_j * r written back as probs with their lo/hi.  Kernels: softmax2 (general D),
// softmax3 (D split over a CTA cluster), softmax4 / softmax5 / softmax6 (streaming at full
// width; launch_softmax picks by shape).
// ---------------------------------------------------------------------------

template <int Q>
__device__ __forceinline__ double block_reduce(double v, double* scratch) {
  // scratch: >= 32 doubles
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = (Q == NORM_LINF) ? warp_max(v) : warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[w] = v;
  __syncthreads();
  double r = scratch[0];
  for (int i = 1; i < nw; ++i) r = qcombine<Q>(r, scratch[i]);
  return r;
}

// Softmax chain, two-read version (the pass uses this one):
//   phase 1 (warp per key row j): row norms -> exp envelope (ExpVerify) -> e bounds/norms, and the
//            composed row a*sel(row) accumulated into the warp's Σ slab in SMEM (SumReduce);
//   phase 2 (column-owned): Σ over the warp slabs -> norms -> recip envelope (RecipVerify) -> r;
//   phase 3 (warp per key row): McCormick e_j * r (MulBroadcast) written in place, row norms by
//            warp reduction -> probs lb/ub/lo/hi.
// Scores Λ is read twice and written once; occupancy is capped so that the second read of a
// CTA's rows (L*D*8 bytes) is served by L2.
template <int Q>
__global__ void __launch_bounds__(512) softmax2_kernel(NView sc, int rows_per_s, int n, int D,
                                                       const double* __restrict__ eps, int* __restrict__ status,
                                                       int site_exp, int site_recip) {
  extern __shared__ double sm2[];
  const int nw = blockDim.x >> 5;
  double* a_lo = sm2;
  double* a_up = a_lo + n;
  double* e_lb = a_up + n;
  double* e_ub = e_lb + n;
  double* e_lo = e_ub + n;
  double* e_hi = e_lo + n;
  double* ru = e_hi + n;  // Σ_u, then r_u  [D]
  double* rl = ru + D;    // Σ_l, then r_l  [D]
  double* red = rl + D;   // 32
  double* scal = red + 32;
  float* part = reinterpret_cast<float*>(scal + 8);  // [nw][2][D]

  const int s = blockIdx.x / rows_per_s;
  const int row = blockIdx.x % rows_per_s;
  const long long nb = (long long)s * sc.s_stride + (long long)row * n;
  float* cb = sc.lam + nb * D;
  float* rb = cb + sc.cr;
  const double e = eps[s];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  for (int t = threadIdx.x; t < nw * 2 * D; t += blockDim.x) part[t] = 0.f;
  __syncthreads();
  float* pu = part + (size_t)warp * 2 * D;
  float* pl = pu + D;

  // ---- phase 1: ExpVerify per key + SumReduce into the warp slab
  int err_exp = 0;
  for (int j = warp; j < n; j += nw) {
    const float* c = cb + (long long)j * D;
    const float* r = rb + (long long)j * D;
    NormAcc<Q> acc;
    for (int d = lane * 4; d < D; d += 128)
      acc.add4(*reinterpret_cast<const float4*>(c + d), *reinterpret_cast<const float4*>(r + d));
    acc.warp_reduce();
    const double nl = acc.fin(acc.l), nu = acc.fin(acc.u);
    const double xlb = sc.lb[nb + j], xub = sc.ub[nb + j];
    Lines ln;
    const int code = envelope(RELAX_EXP, xlb - e * nl, xub + e * nu, ln);
    if (code) err_exp = err_exp ? min(err_exp, code) : code;
    const double au = ln.au, al = ln.al;
    if (lane == 0) {
      a_lo[j] = al;
      a_up[j] = au;
      const double ub2 = au * (au >= 0.0 ? xub : xlb) + ln.bu;
      const double lb2 = al * (al >= 0.0 ? xlb : xub) + ln.bl;
      e_ub[j] = ub2;
      e_lb[j] = lb2;
      // ||a v||_q = |a| ||v||_q: norms of the composed rows without re-reading them
      e_lo[j] = lb2 - e * fabs(al) * (al >= 0.0 ? nl : nu);
      e_hi[j] = ub2 + e * fabs(au) * (au >= 0.0 ? nu : nl);
    }
    for (int d = lane * 4; d < D; d += 128) {  // second touch of the row: L1
      const float4 cv = *reinterpret_cast<const float4*>(c + d);
      const float4 rv = *reinterpret_cast<const float4*>(r + d);
      const float cc[4] = {cv.x, cv.y, cv.z, cv.w}, rr[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const double u = (double)cc[t] + (double)rr[t], l = (double)cc[t] - (double)rr[t];
        pu[d + t] += (float)(au * (au >= 0.0 ? u : l));
        pl[d + t] += (float)(al * (al >= 0.0 ? l : u));
      }
    }
  }
  if (lane == 0 && err_exp) set_status(status, s, site_exp, err_exp);
  __syncthreads();

  // ---- phase 2: Σ rows, RecipVerify, r rows
  double pnu = 0.0, pnl = 0.0;
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    double su = 0.0, sl = 0.0;
    for (int w = 0; w < nw; ++w) {
      su += part[(size_t)(2 * w) * D + d];
      sl += part[(size_t)(2 * w + 1) * D + d];
    }
    ru[d] = su;
    rl[d] = sl;
    if (Q == NORM_L1) { pnu += fabs(su); pnl += fabs(sl); }
    else if (Q == NORM_L2) { pnu += su * su; pnl += sl * sl; }
    else { pnu = fmax(pnu, fabs(su)); pnl = fmax(pnl, fabs(sl)); }
  }
  const double nsu = block_reduce<Q>(pnu, red);
  const double nsl = block_reduce<Q>(pnl, red);
  NormAcc<Q> fin;
  if (threadIdx.x == 0) {
    double slb = 0.0, sub = 0.0;  // propagate_sum_axis order (relax.cpp:728-731)
    for (int j = 0; j < n; ++j) {
      slb += e_lb[j];
      sub += e_ub[j];
    }
    Lines ln;
    const int code = envelope(RELAX_RECIP, slb - e * fin.fin(nsl), sub + e * fin.fin(nsu), ln);
    if (code) set_status(status, s, site_recip, code);
    scal[0] = ln.al;
    scal[1] = ln.au;
    scal[2] = ln.al * (ln.al >= 0.0 ? slb : sub) + ln.bl;
    scal[3] = ln.au * (ln.au >= 0.0 ? sub : slb) + ln.bu;
  }
  __syncthreads();
  const double r_al = scal[0], r_au = scal[1], r_lb = scal[2], r_ub = scal[3];
  pnu = pnl = 0.0;
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    const double u = ru[d], l = rl[d];
    const double yu = r_au * (r_au >= 0.0 ? u : l), yl = r_al * (r_al >= 0.0 ? l : u);
    ru[d] = yu;
    rl[d] = yl;
    if (Q == NORM_L1) { pnu += fabs(yu); pnl += fabs(yl); }
    else if (Q == NORM_L2) { pnu += yu * yu; pnl += yl * yl; }
    else { pnu = fmax(pnu, fabs(yu)); pnl = fmax(pnl, fabs(yl)); }
  }
  const double r_lo = r_lb - e * fin.fin(block_reduce<Q>(pnl, red));
  const double r_hi = r_ub + e * fin.fin(block_reduce<Q>(pnu, red));
  __syncthreads();

  // ---- phase 3: MulBroadcast per key row (warp per row)
  for (int j = warp; j < n; j += nw) {
    float* c = cb + (long long)j * D;
    float* r = rb + (long long)j * D;
    const double au = a_up[j], al = a_lo[j];
    const double lx = e_lo[j], ly = r_lo, uy = r_hi;
    double gu = 0.0, gl = 0.0;
    for (int d = lane * 4; d < D; d += 128) {
      const float4 cv = *reinterpret_cast<const float4*>(c + d);
      const float4 rv = *reinterpret_cast<const float4*>(r + d);
      const float cc[4] = {cv.x, cv.y, cv.z, cv.w}, rr[4] = {rv.x, rv.y, rv.z, rv.w};
      float oc[4], orr[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const double u = (double)cc[t] + (double)rr[t], l = (double)cc[t] - (double)rr[t];
        const double eu = au * (au >= 0.0 ? u : l), el = al * (al >= 0.0 ? l : u);
        const double su = ru[d + t], sl = rl[d + t];
        double p_l = 0.0, p_u = 0.0;
        if (ly != 0.0) p_l += ly * (ly >= 0.0 ? el : eu);  // relax.cpp:542-553
        if (lx != 0.0) p_l += lx * (lx >= 0.0 ? sl : su);
        if (uy != 0.0) p_u += uy * (uy >= 0.0 ? eu : el);  // relax.cpp:556-567
        if (lx != 0.0) p_u += lx * (lx >= 0.0 ? su : sl);
        oc[t] = (float)(0.5 * (p_u + p_l));
        orr[t] = (float)(0.5 * (p_u - p_l));
        if (Q == NORM_L1) { gu += fabs(p_u); gl += fabs(p_l); }
        else if (Q == NORM_L2) { gu += p_u * p_u; gl += p_l * p_l; }
        else { gu = fmax(gu, fabs(p_u)); gl = fmax(gl, fabs(p_l)); }
      }
      *reinterpret_cast<float4*>(c + d) = make_float4(oc[0], oc[1], oc[2], oc[3]);
      *reinterpret_cast<float4*>(r + d) = make_float4(orr[0], orr[1], orr[2], orr[3]);
    }
    if (Q == NORM_LINF) { gu = warp_max(gu); gl = warp_max(gl); }
    else { gu = warp_sum(gu); gl = warp_sum(gl); }
    if (lane == 0) {
      double olb = 0.0, oub = 0.0;
      term_bias(lx, ly, uy, e_lb[j], e_ub[j], r_lb, r_ub, olb, oub);
      const long long o = nb + j;
      sc.lb[o] = olb;
      sc.ub[o] = oub;
      if (sc.lo) {
        sc.lo[o] = olb - e * fin.fin(gl);
        sc.hi[o] = oub + e * fin.fin(gu);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Softmax chain, single-read cluster version (the pass uses this one).
//
// Persistent kernel: a thread-block CLUSTER of CS CTAs walks (sentence, head, query) score
// rows; CTA `rank` owns the perturbation columns [rank*Dc, (rank+1)*Dc) of all n key rows.
// The chunk of the NEXT row is bulk-loaded (cp.async.bulk + mbarriers, double-buffered)
// while the current row is processed, so every SM keeps HBM reads in flight through the
// serial parts of the chain.  Everything that couples columns is a q-norm over D: each CTA
// reduces its chunk and PUSHES the partials into every CTA's exchange slot for its rank
// (st.shared::cluster, slots double-buffered by row parity); after one cluster barrier each
// CTA combines the CS slots in rank order 0..CS-1, so every CTA holds bit-identical norms and
// takes identical envelope decisions.  Exchanges per row:
//   x1  exp-input norms per key      -> ExpVerify envelopes (relax.cpp:363-394)
//   x2  Σ_j e_j row norms             -> RecipVerify envelope (relax.cpp:396-424)
//   x3  r = recip(Σ) row norms         -> McCormick y-interval of MulBroadcast
//   x4  output row norms per key (to rank 0) -> probs lb/ub/lo/hi (relax.cpp:744-775)
// Key rows are reduced by groups of `lpk` lanes (32/lpk keys per warp step).  Element math
// is f32 (Λ is stored in f32); per-lane partials are combined in f64.
// Scores Λ is read from HBM once and written once (in place).
constexpr int kSm3Threads = 256;
constexpr int kSm3MaxBars = 16;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int Q>
__device__ __forceinline__ float qacc_f(float acc, float v) {  // f32 q-norm partial
  return Q == NORM_L2 ? __fmaf_rn(v, v, acc) : (Q == NORM_L1 ? acc + fabsf(v) : fmaxf(acc, fabsf(v)));
}

template <int Q>
__device__ __forceinline__ double qpart(double v) {  // one element's contribution to a q-norm
  return Q == NORM_L2 ? v * v : fabs(v);
}

// q-combine across the `lpk` lanes of a key group (lanes lpk-aligned within the warp)
template <int Q>
__device__ __forceinline__ double group_reduce(double v, int lpk) {
  for (int o = lpk >> 1; o > 0; o >>= 1) v = qcombine<Q>(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Cluster barrier split into arrive (release) / wait (acquire) halves.
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Asynchronous remote store of two doubles into CTA `rank`'s copy of `slot`, completing
// `bytes` on that CTA's copy of `bar` (st.async ... mbarrier::complete_tx): the receiver
// waits on its own mbarrier, so no cluster-wide barrier (and no release fence over the
// CTA's global stores) is needed for the exchange.
__device__ __forceinline__ void push2(double* slot, uint64_t* bar, int rank, double a, double b) {
  uint32_t ra, rb;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_addr(slot)), "r"(rank));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(smem_addr(bar)), "r"(rank));
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(ra),
               "d"(a), "d"(b), "r"(rb)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_par(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WP_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WP_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}

template <int Q>
__global__ void __launch_bounds__(kSm3Threads) softmax3_kernel(NView sc, int rows_per_s, int nrows, int n,
                                                               int D, int CS, int lpk, int nbuf,
                                                               const double* __restrict__ eps,
                                                               int* __restrict__ status, int site_exp,
                                                               int site_recip) {
  extern __shared__ __align__(16) unsigned char sm3[];
  const int Dc = D / CS;
  uint32_t rank_u;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank_u));
  const int rank = (int)rank_u;
  const size_t tile = (size_t)n * Dc;
  float* tbuf = reinterpret_cast<float*>(sm3);           // [nbuf buffers][c|r][n][Dc]
  float* ru_f = tbuf + 2 * nbuf * tile;                  // [Dc] r_u rows (phase 3 operand)
  float* rl_f = ru_f + Dc;                               // [Dc] r_l
  double* su = reinterpret_cast<double*>(rl_f + Dc);     // [Dc] Σ_u
  double* sl = su + Dc;                                  // [Dc] Σ_l
  double* a_lo = sl + Dc;                                // per key [n] x 6
  double* a_up = a_lo + n;
  double* e_lb = a_up + n;
  double* e_ub = e_lb + n;
  double* e_lo = e_ub + n;
  double* e_hi = e_lo + n;
  double* xk0 = e_hi + n;                      // [2 parities][CS][n][2] per-key exchange (x1, x4)
  double* xs0 = xk0 + (size_t)2 * CS * 2 * n;  // [2 parities][2][CS][2] row exchanges x2, x3
  double* red = xs0 + 8 * CS;                  // [32]
  double* scal = red + 32;                     // [8]
  double* hs = scal + 8;                       // [kSm3Threads][8] key-range partial sums
  uint64_t* bars = reinterpret_cast<uint64_t*>(hs + 8 * kSm3Threads);  // [2][kSm3MaxBars] loads
  uint64_t* xbar = bars + 2 * kSm3MaxBars;                              // [2 parities][x1..x4]
  float* a_lo_f = reinterpret_cast<float*>(xbar + 8);                   // [n]
  float* a_up_f = a_lo_f + n;                                           // [n]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int kpw = 32 / lpk;                  // keys per warp step
  const int kstep = nw * kpw;                // keys per block step
  const int nsteps = (n + kstep - 1) / kstep;
  const int spb = (nsteps + kSm3MaxBars - 1) / kSm3MaxBars;  // block steps per mbarrier
  const int nbars = (nsteps + spb - 1) / spb;
  const int kpb = spb * kstep;               // keys per mbarrier
  const int sub = lane % lpk;                // lane within the key group
  const int kofs = warp * kpw + lane / lpk;  // key offset within a block step
  const int D4 = Dc / 4;
  const int cluster_id = blockIdx.x / CS, nclusters = gridDim.x / CS;
  NormAcc<Q> fin;

  if (tid == 0) {
    for (int b = 0; b < 2 * kSm3MaxBars + 8; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bars + b)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cluster_arrive();  // "this CTA has started": waited on before the first DSMEM store

  // issue the bulk loads of row `rid` into buffer `buf` (warp 0)
  auto issue = [&](int rid, int buf) {
    if (warp != 0 || rid >= nrows) return;
    const int s = rid / rows_per_s, row = rid % rows_per_s;
    const long long nb = (long long)s * sc.s_stride + (long long)row * n;
    const float* cb = sc.lam + nb * D + (long long)rank * Dc;
    const float* rb = cb + sc.cr;
    float* tc = tbuf + (size_t)buf * 2 * tile;
    float* tr = tc + tile;
    uint64_t* bb = bars + buf * kSm3MaxBars;
    const uint32_t row_bytes = (uint32_t)Dc * 4u;
    if (lane == 0) {
      // the previous row's generic-proxy reads of this buffer precede the async-proxy writes
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      for (int b = 0; b < nbars; ++b) {
        const int j0 = b * kpb, j1 = min(n, j0 + kpb);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bb + b)),
                     "r"(2u * row_bytes * (uint32_t)(j1 - j0))
                     : "memory");
      }
    }
    __syncwarp();
    for (int j = lane; j < n; j += 32) {
      const uint32_t bar = smem_addr(bb + j / kpb);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_addr(tc + (size_t)j * Dc)),
          "l"(cb + (long long)j * D), "r"(row_bytes), "r"(bar)
          : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_addr(tr + (size_t)j * Dc)),
          "l"(rb + (long long)j * D), "r"(row_bytes), "r"(bar)
          : "memory");
    }
  };

  issue(cluster_id, 0);
  bool started = false;
  int it_row = 0;
  for (int rid = cluster_id; rid < nrows; rid += nclusters, ++it_row) {
    const int buf = nbuf == 2 ? (it_row & 1) : 0, par = it_row & 1;
    const uint32_t use_parity = (uint32_t)((it_row >> 1) & 1);
    const uint32_t load_parity = nbuf == 2 ? use_parity : (uint32_t)(it_row & 1);
    if (nbuf == 2) issue(rid + nclusters, buf ^ 1);  // prefetch the next row of this cluster
    else if (it_row > 0) issue(rid, 0);              // single buffer: load after the last row's reads
    const int s = rid / rows_per_s, row = rid % rows_per_s;
    const long long nb = (long long)s * sc.s_stride + (long long)row * n;  // first neuron of the row
    float* cb = sc.lam + nb * D + (long long)rank * Dc;
    float* rb = cb + sc.cr;
    const float* tc = tbuf + (size_t)buf * 2 * tile;
    const float* tr = tc + tile;
    uint64_t* bb = bars + buf * kSm3MaxBars;
    double* xk = xk0 + (size_t)par * CS * 2 * n;
    double* xs = xs0 + (size_t)par * 4 * CS;
    uint64_t* xb = xbar + 4 * par;
    const uint32_t xpar = use_parity;
    if (tid == 0) {  // bytes each exchange delivers to this CTA (tx-count may run ahead)
      mbar_expect(xb + 0, (uint32_t)(CS * n * 16));
      mbar_expect(xb + 1, (uint32_t)(CS * 16));
      mbar_expect(xb + 2, (uint32_t)(CS * 16));
      if (rank == 0) mbar_expect(xb + 3, (uint32_t)(CS * n * 16));
    }
    const double e = eps[s];

    for (int j = tid; j < n; j += blockDim.x) {  // scores lb/ub, consumed by phase 1b
      e_lb[j] = sc.lb[nb + j];
      e_ub[j] = sc.ub[nb + j];
    }
    // ---- phase 1a: partial norms of the exp inputs (lpk lanes per key)
    for (int it = 0; it < nsteps; ++it) {
      if (it % spb == 0) {
        const uint32_t bar = smem_addr(bb + it / spb);
        asm volatile(
            "{\n\t.reg .pred p;\n"
            "W3_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
            "@!p bra W3_%=;\n}" ::"r"(bar),
            "r"(load_parity)
            : "memory");
      }
      const int j = it * kstep + kofs;
      float fu = 0.f, fl = 0.f;
      if (j < n) {
        const float4* c = reinterpret_cast<const float4*>(tc + (size_t)j * Dc);
        const float4* r = reinterpret_cast<const float4*>(tr + (size_t)j * Dc);
        for (int f = sub; f < D4; f += lpk) {
          const float4 cv = c[f], rv = r[f];
          fu = qacc_f<Q>(fu, cv.x + rv.x); fl = qacc_f<Q>(fl, cv.x - rv.x);
          fu = qacc_f<Q>(fu, cv.y + rv.y); fl = qacc_f<Q>(fl, cv.y - rv.y);
          fu = qacc_f<Q>(fu, cv.z + rv.z); fl = qacc_f<Q>(fl, cv.z - rv.z);
          fu = qacc_f<Q>(fu, cv.w + rv.w); fl = qacc_f<Q>(fl, cv.w - rv.w);
        }
      }
      const double gu = group_reduce<Q>((double)fu, lpk), gl = group_reduce<Q>((double)fl, lpk);
      if (!started) {
        cluster_wait();
        started = true;
      }
      if (j < n)  // push to every rank's slot [rank]
        for (int q = sub; q < CS; q += lpk) push2(xk + ((size_t)rank * n + j) * 2, xb + 0, q, gu, gl);
    }
    mbar_wait_par(xb + 0, xpar);  // x1 from every rank

    // ---- phase 1b: ExpVerify envelopes per key (every rank computes the same values)
    int err_exp = 0;
    for (int j = tid; j < n; j += blockDim.x) {
      double pu = 0.0, pl = 0.0;
      for (int q = 0; q < CS; ++q) {
        pu = qcombine<Q>(pu, xk[((size_t)q * n + j) * 2]);
        pl = qcombine<Q>(pl, xk[((size_t)q * n + j) * 2 + 1]);
      }
      const double nu = fin.fin(pu), nl = fin.fin(pl);
      const double xlb = e_lb[j], xub = e_ub[j];  // prefetched scores lb/ub
      Lines ln;
      const int code = envelope(RELAX_EXP, xlb - e * nl, xub + e * nu, ln);
      if (code) err_exp = err_exp ? min(err_exp, code) : code;
      a_lo[j] = ln.al;
      a_up[j] = ln.au;
      a_lo_f[j] = (float)ln.al;
      a_up_f[j] = (float)ln.au;
      const double ub2 = ln.au * (ln.au >= 0.0 ? xub : xlb) + ln.bu;
      const double lb2 = ln.al * (ln.al >= 0.0 ? xlb : xub) + ln.bl;
      e_ub[j] = ub2;
      e_lb[j] = lb2;
      // ||a v||_q = |a| ||v||_q: norms of the composed rows without another sweep
      e_lo[j] = lb2 - e * fabs(ln.al) * (ln.al >= 0.0 ? nl : nu);
      e_hi[j] = ub2 + e * fabs(ln.au) * (ln.au >= 0.0 ? nu : nl);
    }
    if (err_exp && rank == 0) set_status(status, s, site_exp, err_exp);
    __syncthreads();
    if (warp == nw - 1) {  // Σ_j e_lb / e_ub (SumReduce bias) while the other warps start phase 2
      double a = 0.0, b = 0.0;
      for (int j = lane; j < n; j += 32) {
        a += e_lb[j];
        b += e_ub[j];
      }
      a = warp_sum(a);
      b = warp_sum(b);
      if (lane == 0) {
        scal[4] = a;
        scal[5] = b;
      }
    }

    // ---- phase 2: SumReduce over keys.  Thread = (float4 column group, key range); 8
    // independent f64 accumulators per thread (f32 products), key ranges combined in order.
    const int gpt = D4 <= (int)blockDim.x ? D4 : (int)blockDim.x;  // column groups per sweep
    const int nh = (int)blockDim.x / gpt;
    {
      const int h = tid / gpt;
      if (h < nh) {
        const int j0 = (int)((long long)n * h / nh), j1 = (int)((long long)n * (h + 1) / nh);
        for (int g = tid % gpt; g < D4; g += gpt) {
          double au_s[4] = {0.0, 0.0, 0.0, 0.0}, al_s[4] = {0.0, 0.0, 0.0, 0.0};
          for (int j = j0; j < j1; ++j) {
            const float au = a_up_f[j], al = a_lo_f[j];
            const float4 cv = reinterpret_cast<const float4*>(tc + (size_t)j * Dc)[g];
            const float4 rv = reinterpret_cast<const float4*>(tr + (size_t)j * Dc)[g];
            const float cc[4] = {cv.x, cv.y, cv.z, cv.w}, rr[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const float u = cc[t] + rr[t], l = cc[t] - rr[t];
              au_s[t] += (double)(au * (au >= 0.f ? u : l));
              al_s[t] += (double)(al * (al >= 0.f ? l : u));
            }
          }
          double* dst = nh > 1 ? hs + ((size_t)h * D4 + g) * 8 : nullptr;
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            if (nh > 1) {
              dst[t] = au_s[t];
              dst[4 + t] = al_s[t];
            } else {
              su[4 * g + t] = au_s[t];
              sl[4 * g + t] = al_s[t];
            }
          }
        }
      }
    }
    __syncthreads();
    double pnu = 0.0, pnl = 0.0;
    for (int d = tid; d < Dc; d += blockDim.x) {
      if (nh > 1) {
        double a = 0.0, b = 0.0;
        for (int h = 0; h < nh; ++h) {
          a += hs[((size_t)h * D4 + d / 4) * 8 + (d & 3)];
          b += hs[((size_t)h * D4 + d / 4) * 8 + 4 + (d & 3)];
        }
        su[d] = a;
        sl[d] = b;
      }
      pnu = qcombine<Q>(pnu, qpart<Q>(su[d]));
      pnl = qcombine<Q>(pnl, qpart<Q>(sl[d]));
    }
    pnu = block_reduce<Q>(pnu, red);
    pnl = block_reduce<Q>(pnl, red);
    if (tid < CS) push2(xs + 2 * rank, xb + 1, tid, pnu, pnl);
    mbar_wait_par(xb + 1, xpar);
    if (tid == 0) {
      double nsu = 0.0, nsl = 0.0;
      for (int q = 0; q < CS; ++q) {
        nsu = qcombine<Q>(nsu, xs[2 * q]);
        nsl = qcombine<Q>(nsl, xs[2 * q + 1]);
      }
      const double slb = scal[4], sub_ = scal[5];  // propagate_sum_axis (relax.cpp:728-731)
      Lines ln;
      const int code = envelope(RELAX_RECIP, slb - e * fin.fin(nsl), sub_ + e * fin.fin(nsu), ln);
      if (code && rank == 0) set_status(status, s, site_recip, code);
      scal[0] = ln.al;
      scal[1] = ln.au;
      scal[2] = ln.al * (ln.al >= 0.0 ? slb : sub_) + ln.bl;
      scal[3] = ln.au * (ln.au >= 0.0 ? sub_ : slb) + ln.bu;
    }
    __syncthreads();
    const double r_al = scal[0], r_au = scal[1], r_lb = scal[2], r_ub = scal[3];
    pnu = pnl = 0.0;
    for (int d = tid; d < Dc; d += blockDim.x) {
      const double u = su[d], l = sl[d];
      const double yu = r_au * (r_au >= 0.0 ? u : l), yl = r_al * (r_al >= 0.0 ? l : u);
      ru_f[d] = (float)yu;
      rl_f[d] = (float)yl;
      pnu = qcombine<Q>(pnu, qpart<Q>(yu));
      pnl = qcombine<Q>(pnl, qpart<Q>(yl));
    }
    pnu = block_reduce<Q>(pnu, red);
    pnl = block_reduce<Q>(pnl, red);
    if (tid < CS) push2(xs + 2 * CS + 2 * rank, xb + 2, tid, pnu, pnl);
    mbar_wait_par(xb + 2, xpar);
    double nru = 0.0, nrl = 0.0;
    for (int q = 0; q < CS; ++q) {
      nru = qcombine<Q>(nru, xs[2 * CS + 2 * q]);
      nrl = qcombine<Q>(nrl, xs[2 * CS + 2 * q + 1]);
    }
    const double r_lo = r_lb - e * fin.fin(nrl);
    const double r_hi = r_ub + e * fin.fin(nru);

    // ---- phase 3: MulBroadcast (McCormick e_j * r) per key, written to HBM
    const float ly = (float)r_lo, uy = (float)r_hi;
    const bool ly_p = ly >= 0.f, uy_p = uy >= 0.f;
    for (int it = 0; it < nsteps; ++it) {
      const int j = it * kstep + kofs;
      float fu = 0.f, fl = 0.f;
      if (j < n) {
        const float4* c = reinterpret_cast<const float4*>(tc + (size_t)j * Dc);
        const float4* r = reinterpret_cast<const float4*>(tr + (size_t)j * Dc);
        float4* gc = reinterpret_cast<float4*>(cb + (long long)j * D);
        float4* gr = reinterpret_cast<float4*>(rb + (long long)j * D);
        const float au = a_up_f[j], al = a_lo_f[j], lx = (float)e_lo[j];
        const bool au_p = au >= 0.f, al_p = al >= 0.f, lx_p = lx >= 0.f;
        for (int f = sub; f < D4; f += lpk) {
          const float4 cv = c[f], rv = r[f];
          const float4 yuv = reinterpret_cast<const float4*>(ru_f)[f];
          const float4 ylv = reinterpret_cast<const float4*>(rl_f)[f];
          const float cc[4] = {cv.x, cv.y, cv.z, cv.w}, rr[4] = {rv.x, rv.y, rv.z, rv.w};
          const float yuu[4] = {yuv.x, yuv.y, yuv.z, yuv.w}, yll[4] = {ylv.x, ylv.y, ylv.z, ylv.w};
          float oc[4], orr[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const float u = cc[t] + rr[t], l = cc[t] - rr[t];
            const float eu = au * (au_p ? u : l), el = al * (al_p ? l : u);
            // relax.cpp:542-567: lower plane (cx = ly, cy = lx), upper plane (cx = uy, cy = lx)
            const float p_l = __fmaf_rn(ly, ly_p ? el : eu, lx * (lx_p ? yll[t] : yuu[t]));
            const float p_u = __fmaf_rn(uy, uy_p ? eu : el, lx * (lx_p ? yuu[t] : yll[t]));
            oc[t] = 0.5f * (p_u + p_l);
            orr[t] = 0.5f * (p_u - p_l);
            fu = qacc_f<Q>(fu, p_u);
            fl = qacc_f<Q>(fl, p_l);
          }
          gc[f] = make_float4(oc[0], oc[1], oc[2], oc[3]);
          gr[f] = make_float4(orr[0], orr[1], orr[2], orr[3]);
        }
      }
      const double gu = group_reduce<Q>((double)fu, lpk), gl = group_reduce<Q>((double)fl, lpk);
      if (j < n && sub == 0) push2(xk + ((size_t)rank * n + j) * 2, xb + 3, 0, gu, gl);  // to rank 0
    }
    if (rank == 0) {
      mbar_wait_par(xb + 3, xpar);
      for (int j = tid; j < n; j += blockDim.x) {
        double gu = 0.0, gl = 0.0;
        for (int q = 0; q < CS; ++q) {
          gu = qcombine<Q>(gu, xk[((size_t)q * n + j) * 2]);
          gl = qcombine<Q>(gl, xk[((size_t)q * n + j) * 2 + 1]);
        }
        double olb = 0.0, oub = 0.0;
        term_bias(e_lo[j], r_lo, r_hi, e_lb[j], e_ub[j], r_lb, r_ub, olb, oub);
        const long long o = nb + j;
        sc.lb[o] = olb;
        sc.ub[o] = oub;
        if (sc.lo) {
          sc.lo[o] = olb - e * fin.fin(gl);
          sc.hi[o] = oub + e * fin.fin(gu);
        }
      }
    }
    __syncthreads();  // e_* / a_* / buffers are rewritten by the next row
  }
  if (!started) cluster_wait();
  cluster_arrive();  // no CTA leaves while a peer may still address its SMEM
  cluster_wait();
}

// ---------------------------------------------------------------------------
// Softmax chain, streaming version (D <= 512, D % 128 == 0; the pass uses it when it applies).
//
// Persistent CTAs (4 per SM), one score row (s, h, i) at a time with the FULL perturbation
// width, so no norm ever crosses a CTA: one producer warp streams key rows (c and r planes,
// 8·D bytes) through a 2·NC-stage shared-memory ring with cp.async.bulk + mbarriers, and NC = 4
// consumer warps take one key row each (stage s always belongs to warp s mod NC):
//   pass 1  per key: q-norms of the exp input (warp reduction) -> ExpVerify envelope
//           (relax.cpp:363-394) -> Σ_j e_j accumulated in the warp's registers;
//   then    Σ rows combined over the warps in a fixed order -> RecipVerify (relax.cpp:396-424)
//           -> r rows and their norms (block reduction among the consumers);
//   pass 2  per key: McCormick e_j * r (relax.cpp:744-775) written to HBM, probs lb/ub/lo/hi.
// Every row is streamed twice -- pass 2 in reverse key order, so it starts on the keys the CTA
// read last, which are still in L2 -- and written once.  The producer warp stays resident to
// the end (lanes of a warp exiting early while others still issue bulk copies lost mbarrier
// arrivals on the B200 when two CTAs shared an SM).  The producer never waits on the consumers' reductions: it prefetches pass 2
// of the row and pass 1 of the next row while Σ / recip / r are being formed, so HBM traffic
// stays in flight through the serial part of the chain.  Element math f32, norms and O(N)
// state f64, as softmax3_kernel.
// A stage count that is a multiple of the consumer count: the items of one stage are then always
// taken by the same warp, so a warp never waits on a stage whose previous fill (issued earlier,
// but possibly completing later -- bulk copies complete out of order) is still pending, which
// would let the parity wait succeed one phase early.
template <int NC, int KG>
struct Sm4 {
  // 8·D-byte key rows; 32 KB of ring per CTA whatever D is (more, smaller stages for small D)
  static constexpr int kStages = NC * (8 / KG);
  static constexpr int kThreads = (NC + 1) * 32;
  static_assert(kStages % NC == 0, "stage ownership must be per warp");
};

template <int NC>
__device__ __forceinline__ void sm4_sync() {  // consumer warps only
  asm volatile("bar.sync 1, %0;" ::"r"(NC * 32) : "memory");
}
__device__ __forceinline__ void mbar_arrive1(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n}"
               : "=r"(ok) : "r"(smem_addr(bar)), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void sm4_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try(bar, parity)) {
  }
}

// consumer-block q-combine of two values at once (red: >= 2*NC doubles)
template <int Q, int NC>
__device__ __forceinline__ void sm4_reduce2(double& a, double& b, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (Q == NORM_LINF) {
    a = warp_max(a);
    b = warp_max(b);
  } else {
    a = warp_sum(a);
    b = warp_sum(b);
  }
  sm4_sync<NC>();
  if (lane == 0) {
    red[w] = a;
    red[NC + w] = b;
  }
  sm4_sync<NC>();
  a = red[0];
  b = red[NC];
  for (int i = 1; i < NC; ++i) {
    a = qcombine<Q>(a, red[i]);
    b = qcombine<Q>(b, red[NC + i]);
  }
}

size_t softmax4_smem(int n, int D, int NC) {
  return (size_t)NC * (8 / (D / 128)) * 8 * D    // ring
         + (size_t)NC * 2 * D * 4                // Σ partials per warp
         + (size_t)2 * D * 4                     // r rows (f32)
         + (size_t)(n + 1) * (2 * 4 + 3 * 8)     // a_lo_f, a_up_f, e_lb, e_ub, e_lo
         + 64 * 8                                // red + scal
         + 2 * (size_t)NC * (8 / (D / 128)) * 8 + 64;  // barriers + alignment
}

template <int Q, int KG, int NC>  // KG = D / 128 float4 groups per lane per plane; NC consumer warps
__global__ void __launch_bounds__(Sm4<NC, KG>::kThreads, NC <= 4 ? 4 : 2) softmax4_kernel(NView sc, int rows_per_s, int nrows, int n,
                                                                  const double* __restrict__ eps,
                                                                  int* __restrict__ status, int site_exp,
                                                                  int site_recip) {
  constexpr int D = KG * 128;
  extern __shared__ __align__(16) unsigned char sm4[];
  float* ring = reinterpret_cast<float*>(sm4);                          // [NS][c|r][D]
  float* part = ring + (size_t)Sm4<NC, KG>::kStages * 2 * D;                      // [NC][u|l][D]
  float* ru_f = part + (size_t)NC * 2 * D;                   // [D]
  float* rl_f = ru_f + D;                                               // [D]
  const int n2 = (n + 1) & ~1;                                          // keeps the f64 arrays aligned
  float* a_lo_f = rl_f + D;                                             // [n]
  float* a_up_f = a_lo_f + n2;                                          // [n]
  double* e_lb = reinterpret_cast<double*>(a_up_f + n2);                // [n]
  double* e_ub = e_lb + n;
  double* e_lo = e_ub + n;
  double* red = e_lo + n;    // [32]
  double* scal = red + 32;   // [32]
  uint64_t* full = reinterpret_cast<uint64_t*>(scal + 32);
  uint64_t* empty = full + Sm4<NC, KG>::kStages;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int b = 0; b < Sm4<NC, KG>::kStages; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(full + b)) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(empty + b)) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == NC) {  // ---- producer
    if (lane == 0) {
      long long t = 0;
      for (int rid = blockIdx.x; rid < nrows; rid += gridDim.x) {
        const int s = rid / rows_per_s, row = rid % rows_per_s;
        const long long nb = (long long)s * sc.s_stride + (long long)row * n;
        const float* cb = sc.lam + nb * D;
        const float* rb = cb + sc.cr;
        for (int p = 0; p < 2; ++p)
          for (int j = 0; j < n; ++j, ++t) {
            const int st = (int)(t % Sm4<NC, KG>::kStages);
            const uint32_t ph = (uint32_t)((t / Sm4<NC, KG>::kStages) & 1);
            if (t >= Sm4<NC, KG>::kStages) sm4_wait(empty + st, ph ^ 1u);
            float* dst = ring + (size_t)st * 2 * D;
            const int key = p == 0 ? j : n - 1 - j;  // pass 2 in reverse: the latest keys are still in L2
            mbar_expect(full + st, 8u * D);
            asm volatile(
                "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_addr(dst)),
                "l"(cb + (long long)key * D), "r"(4u * D), "r"(smem_addr(full + st))
                : "memory");
            asm volatile(
                "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_addr(dst + D)),
                "l"(rb + (long long)key * D), "r"(4u * D), "r"(smem_addr(full + st))
                : "memory");
          }
      }
    }
    __syncwarp();
  } else {  // ---- consumers
  NormAcc<Q> fin;
  long long t0 = 0;
  for (int rid = blockIdx.x; rid < nrows; rid += gridDim.x, t0 += 2LL * n) {
    const int s = rid / rows_per_s, row = rid % rows_per_s;
    const long long nb = (long long)s * sc.s_stride + (long long)row * n;
    float* cbw = sc.lam + nb * D;
    float* rbw = cbw + sc.cr;
    const double e = eps[s];

    // pass 1: exp envelopes per key, Σ_j e_j in registers
    float su[KG * 4], sl[KG * 4];
#pragma unroll
    for (int k = 0; k < KG * 4; ++k) su[k] = sl[k] = 0.f;
    int err_exp = 0;
    for (int j = warp; j < n; j += NC) {
      const long long ti = t0 + j;
      const int st = (int)(ti % Sm4<NC, KG>::kStages);
      const double xlb = sc.lb[nb + j], xub = sc.ub[nb + j];  // issued before the wait
      sm4_wait(full + st, (uint32_t)((ti / Sm4<NC, KG>::kStages) & 1));
      const float4* c4 = reinterpret_cast<const float4*>(ring + (size_t)st * 2 * D);
      const float4* r4 = c4 + D / 4;
      float fu = 0.f, fl = 0.f;
#pragma unroll
      for (int k = 0; k < KG; ++k) {
        const float4 cv = c4[lane + 32 * k], rv = r4[lane + 32 * k];
        fu = qacc_f<Q>(fu, cv.x + rv.x); fl = qacc_f<Q>(fl, cv.x - rv.x);
        fu = qacc_f<Q>(fu, cv.y + rv.y); fl = qacc_f<Q>(fl, cv.y - rv.y);
        fu = qacc_f<Q>(fu, cv.z + rv.z); fl = qacc_f<Q>(fl, cv.z - rv.z);
        fu = qacc_f<Q>(fu, cv.w + rv.w); fl = qacc_f<Q>(fl, cv.w - rv.w);
      }
      const double nu = fin.fin(group_reduce<Q>((double)fu, 32)), nl = fin.fin(group_reduce<Q>((double)fl, 32));
      Lines ln;
      const int code = exp_envelope(xlb - e * nl, xub + e * nu, ln);
      if (code) err_exp = err_exp ? min(err_exp, code) : code;
      const float au = (float)ln.au, al = (float)ln.al;
      if (lane == 0) {
        a_lo_f[j] = al;
        a_up_f[j] = au;
        const double ub2 = ln.au * (ln.au >= 0.0 ? xub : xlb) + ln.bu;
        const double lb2 = ln.al * (ln.al >= 0.0 ? xlb : xub) + ln.bl;
        e_ub[j] = ub2;
        e_lb[j] = lb2;
        e_lo[j] = lb2 - e * fabs(ln.al) * (ln.al >= 0.0 ? nl : nu);  // ||a v||_q = |a| ||v||_q
      }
#pragma unroll
      for (int k = 0; k < KG; ++k) {  // second read of the stage (SMEM): no row data live across the envelope
        const float4 cv = c4[lane + 32 * k], rv = r4[lane + 32 * k];
        const float cc[4] = {cv.x, cv.y, cv.z, cv.w}, rr[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float u = cc[q] + rr[q], l = cc[q] - rr[q];
          su[4 * k + q] += au * (au >= 0.f ? u : l);
          sl[4 * k + q] += al * (al >= 0.f ? l : u);
        }
      }
      // generic-proxy reads of the stage precede the producer's next async-proxy (TMA) write
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive1(empty + st);
    }
    if (err_exp && lane == 0) set_status(status, s, site_exp, err_exp);
    {
      float4* pu = reinterpret_cast<float4*>(part + (size_t)warp * 2 * D);
      float4* pl = pu + D / 4;
#pragma unroll
      for (int k = 0; k < KG; ++k) {
        pu[lane + 32 * k] = make_float4(su[4 * k], su[4 * k + 1], su[4 * k + 2], su[4 * k + 3]);
        pl[lane + 32 * k] = make_float4(sl[4 * k], sl[4 * k + 1], sl[4 * k + 2], sl[4 * k + 3]);
      }
    }
    sm4_sync<NC>();
    // Σ rows (warp partials combined in warp order, f64), their norms, the SumReduce bias
    double pnu = 0.0, pnl = 0.0;
    constexpr int kPer = D / (NC * 32) > 0 ? D / (NC * 32) : 1;  // columns per consumer thread
    double sud[kPer], sld[kPer];  // fully unrolled: registers
#pragma unroll
    for (int m = 0; m < kPer; ++m) {
      const int d = tid + m * NC * 32;
      double a = 0.0, b = 0.0;
      if (d < D) {
        for (int w = 0; w < NC; ++w) {
          a += (double)part[(size_t)w * 2 * D + d];
          b += (double)part[(size_t)w * 2 * D + D + d];
        }
        pnu = qcombine<Q>(pnu, qpart<Q>(a));
        pnl = qcombine<Q>(pnl, qpart<Q>(b));
      }
      sud[m] = a;
      sld[m] = b;
    }
    if (warp == 0) {  // propagate_sum_axis bias (relax.cpp:728-731)
      double a = 0.0, b = 0.0;
      for (int j = lane; j < n; j += 32) {
        a += e_lb[j];
        b += e_ub[j];
      }
      a = warp_sum(a);
      b = warp_sum(b);
      if (lane == 0) {
        scal[4] = a;
        scal[5] = b;
      }
    }
    sm4_reduce2<Q, NC>(pnu, pnl, red);
    const double nsu = pnu, nsl = pnl;
    if (tid == 0) {
      const double slb = scal[4], sub_ = scal[5];
      Lines ln;
      const int code = envelope(RELAX_RECIP, slb - e * fin.fin(nsl), sub_ + e * fin.fin(nsu), ln);
      if (code) set_status(status, s, site_recip, code);
      scal[0] = ln.al;
      scal[1] = ln.au;
      scal[2] = ln.al * (ln.al >= 0.0 ? slb : sub_) + ln.bl;
      scal[3] = ln.au * (ln.au >= 0.0 ? sub_ : slb) + ln.bu;
    }
    sm4_sync<NC>();
    const double r_al = scal[0], r_au = scal[1], r_lb = scal[2], r_ub = scal[3];
    pnu = pnl = 0.0;
#pragma unroll
    for (int m = 0; m < kPer; ++m) {
      const int d = tid + m * NC * 32;
      if (d >= D) continue;
      const double u = sud[m], l = sld[m];
      const double yu = r_au * (r_au >= 0.0 ? u : l), yl = r_al * (r_al >= 0.0 ? l : u);
      ru_f[d] = (float)yu;
      rl_f[d] = (float)yl;
      pnu = qcombine<Q>(pnu, qpart<Q>(yu));
      pnl = qcombine<Q>(pnl, qpart<Q>(yl));
    }
    sm4_reduce2<Q, NC>(pnu, pnl, red);  // (its barriers also publish ru_f / rl_f)
    const double nru = pnu, nrl = pnl;
    const double r_lo = r_lb - e * fin.fin(nrl);
    const double r_hi = r_ub + e * fin.fin(nru);

    // pass 2: MulBroadcast per key, written to HBM
    const float ly = (float)r_lo, uy = (float)r_hi;
    const bool ly_p = ly >= 0.f, uy_p = uy >= 0.f;
    const float4* yu4 = reinterpret_cast<const float4*>(ru_f);  // r rows: re-read from SMEM per key
    const float4* yl4 = reinterpret_cast<const float4*>(rl_f);  // (keeps pass 2 free of spills)
    for (int m = warp; m < n; m += NC) {
      const int j = n - 1 - m;  // the producer streams pass 2 in reverse key order
      const long long ti = t0 + n + m;
      const int st = (int)(ti % Sm4<NC, KG>::kStages);
      const float au = a_up_f[j], al = a_lo_f[j], lx = (float)e_lo[j];
      const bool au_p = au >= 0.f, al_p = al >= 0.f, lx_p = lx >= 0.f;
      sm4_wait(full + st, (uint32_t)((ti / Sm4<NC, KG>::kStages) & 1));
      const float4* c4 = reinterpret_cast<const float4*>(ring + (size_t)st * 2 * D);
      const float4* r4 = c4 + D / 4;
      float4 cv[KG], rv[KG];
#pragma unroll
      for (int k = 0; k < KG; ++k) {
        cv[k] = c4[lane + 32 * k];
        rv[k] = r4[lane + 32 * k];
      }
      // generic-proxy reads of the stage precede the producer's next async-proxy (TMA) write
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive1(empty + st);
      float4* gc = reinterpret_cast<float4*>(cbw + (long long)j * D);
      float4* gr = reinterpret_cast<float4*>(rbw + (long long)j * D);
      float fu = 0.f, fl = 0.f;
#pragma unroll
      for (int k = 0; k < KG; ++k) {
        const float cc[4] = {cv[k].x, cv[k].y, cv[k].z, cv[k].w}, rr[4] = {rv[k].x, rv[k].y, rv[k].z, rv[k].w};
        const float4 yuv = yu4[lane + 32 * k], ylv = yl4[lane + 32 * k];
        const float yuu[4] = {yuv.x, yuv.y, yuv.z, yuv.w};
        const float yll[4] = {ylv.x, ylv.y, ylv.z, ylv.w};
        float oc[4], orr[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float u = cc[q] + rr[q], l = cc[q] - rr[q];
          const float eu = au * (au_p ? u : l), el = al * (al_p ? l : u);
          // relax.cpp:542-567: lower plane (cx = ly, cy = lx), upper plane (cx = uy, cy = lx)
          const float p_l = __fmaf_rn(ly, ly_p ? el : eu, lx * (lx_p ? yll[q] : yuu[q]));
          const float p_u = __fmaf_rn(uy, uy_p ? eu : el, lx * (lx_p ? yuu[q] : yll[q]));
          oc[q] = 0.5f * (p_u + p_l);
          orr[q] = 0.5f * (p_u - p_l);
          fu = qacc_f<Q>(fu, p_u);
          fl = qacc_f<Q>(fl, p_l);
        }
        gc[lane + 32 * k] = make_float4(oc[0], oc[1], oc[2], oc[3]);
        gr[lane + 32 * k] = make_float4(orr[0], orr[1], orr[2], orr[3]);
      }
      const double gu = group_reduce<Q>((double)fu, 32), gl = group_reduce<Q>((double)fl, 32);
      if (lane == 0) {
        double olb = 0.0, oub = 0.0;
        term_bias(e_lo[j], r_lo, r_hi, e_lb[j], e_ub[j], r_lb, r_ub, olb, oub);
        const long long o = nb + j;
        sc.lb[o] = olb;
        sc.ub[o] = oub;
        if (sc.lo) {
          sc.lo[o] = olb - e * fin.fin(gl);
          sc.hi[o] = oub + e * fin.fin(gu);
        }
      }
    }
    sm4_sync<NC>();  // per-key arrays / partials are rewritten by the next row
  }
  }
  __syncthreads();  // the producer warp stays resident until every stage has been consumed
}

// Streaming softmax for any D % 128 == 0 (the wide rows of c5, D = 1536): softmax4_kernel's
// structure with runtime D -- the warps' Σ partials accumulate in SHARED memory (read-modify-
// write per key) instead of registers, and nothing per column is held in registers across a
// key, so the register budget does not grow with D.  ns stages (a multiple of NC).
template <int Q, int NC>
__global__ void __launch_bounds__((NC + 1) * 32) softmax5_kernel(NView sc, int rows_per_s, int nrows, int n, int D,
                                                                 int ns, const double* __restrict__ eps,
                                                                 int* __restrict__ status, int site_exp,
                                                                 int site_recip) {
  extern __shared__ __align__(16) unsigned char sm5[];
  const int KG = D / 128;
  float* ring = reinterpret_cast<float*>(sm5);        // [ns][c|r][D]
  float* part = ring + (size_t)ns * 2 * D;            // [NC][u|l][D]
  float* ru_f = part + (size_t)NC * 2 * D;            // [D]
  float* rl_f = ru_f + D;                             // [D]
  const int n2 = (n + 1) & ~1;
  float* a_lo_f = rl_f + D;
  float* a_up_f = a_lo_f + n2;
  double* e_lb = reinterpret_cast<double*>(a_up_f + n2);
  double* e_ub = e_lb + n;
  double* e_lo = e_ub + n;
  double* red = e_lo + n;   // [32]
  double* scal = red + 32;  // [32]
  uint64_t* full = reinterpret_cast<uint64_t*>(scal + 32);
  uint64_t* empty = full + ns;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int b = 0; b < ns; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(full + b)) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(empty + b)) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == NC) {  // ---- producer (stays resident to the end, see softmax4_kernel)
    if (lane == 0) {
      long long t = 0;
      for (int rid = blockIdx.x; rid < nrows; rid += gridDim.x) {
        const int s = rid / rows_per_s, row = rid % rows_per_s;
        const long long nb = (long long)s * sc.s_stride + (long long)row * n;
        const float* cb = sc.lam + nb * D;
        const float* rb = cb + sc.cr;
        for (int p = 0; p < 2; ++p)
          for (int j = 0; j < n; ++j, ++t) {
            const int st = (int)(t % ns);
            const uint32_t ph = (uint32_t)((t / ns) & 1);
            if (t >= ns) sm4_wait(empty + st, ph ^ 1u);
            float* dst = ring + (size_t)st * 2 * D;
            const int key = p == 0 ? j : n - 1 - j;
            mbar_expect(full + st, 8u * D);
            asm volatile(
                "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_addr(dst)),
                "l"(cb + (long long)key * D), "r"(4u * D), "r"(smem_addr(full + st))
                : "memory");
            asm volatile(
                "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_addr(dst + D)),
                "l"(rb + (long long)key * D), "r"(4u * D), "r"(smem_addr(full + st))
                : "memory");
          }
      }
    }
    __syncwarp();
  } else {  // ---- consumers
    NormAcc<Q> fin;
    float4* pu = reinterpret_cast<float4*>(part + (size_t)warp * 2 * D);
    float4* pl = pu + D / 4;
    long long t0 = 0;
    for (int rid = blockIdx.x; rid < nrows; rid += gridDim.x, t0 += 2LL * n) {
      const int s = rid / rows_per_s, row = rid % rows_per_s;
      const long long nb = (long long)s * sc.s_stride + (long long)row * n;
      float* cbw = sc.lam + nb * D;
      float* rbw = cbw + sc.cr;
      const double e = eps[s];
      for (int k = 0; k < KG; ++k) {
        pu[lane + 32 * k] = make_float4(0.f, 0.f, 0.f, 0.f);
        pl[lane + 32 * k] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      // pass 1: exp envelopes per key; Σ_j e_j accumulated into the warp's SMEM partial
      int err_exp = 0;
      for (int j = warp; j < n; j += NC) {
        const long long ti = t0 + j;
        const int st = (int)(ti % ns);
        const double xlb = sc.lb[nb + j], xub = sc.ub[nb + j];
        sm4_wait(full + st, (uint32_t)((ti / ns) & 1));
        const float4* c4 = reinterpret_cast<const float4*>(ring + (size_t)st * 2 * D);
        const float4* r4 = c4 + D / 4;
        float fu = 0.f, fl = 0.f;
        for (int k = 0; k < KG; ++k) {
          const float4 cv = c4[lane + 32 * k], rv = r4[lane + 32 * k];
          fu = qacc_f<Q>(fu, cv.x + rv.x); fl = qacc_f<Q>(fl, cv.x - rv.x);
          fu = qacc_f<Q>(fu, cv.y + rv.y); fl = qacc_f<Q>(fl, cv.y - rv.y);
          fu = qacc_f<Q>(fu, cv.z + rv.z); fl = qacc_f<Q>(fl, cv.z - rv.z);
          fu = qacc_f<Q>(fu, cv.w + rv.w); fl = qacc_f<Q>(fl, cv.w - rv.w);
        }
        const double nu = fin.fin(group_reduce<Q>((double)fu, 32)), nl = fin.fin(group_reduce<Q>((double)fl, 32));
        Lines ln;
        const int code = exp_envelope(xlb - e * nl, xub + e * nu, ln);
        if (code) err_exp = err_exp ? min(err_exp, code) : code;
        const float au = (float)ln.au, al = (float)ln.al;
        if (lane == 0) {
          a_lo_f[j] = al;
          a_up_f[j] = au;
          const double ub2 = ln.au * (ln.au >= 0.0 ? xub : xlb) + ln.bu;
          const double lb2 = ln.al * (ln.al >= 0.0 ? xlb : xub) + ln.bl;
          e_ub[j] = ub2;
          e_lb[j] = lb2;
          e_lo[j] = lb2 - e * fabs(ln.al) * (ln.al >= 0.0 ? nl : nu);
        }
        for (int k = 0; k < KG; ++k) {
          const float4 cv = c4[lane + 32 * k], rv = r4[lane + 32 * k];
          float4 a = pu[lane + 32 * k], b = pl[lane + 32 * k];
          const float cc[4] = {cv.x, cv.y, cv.z, cv.w}, rr[4] = {rv.x, rv.y, rv.z, rv.w};
          float* ap = &a.x;
          float* bp = &b.x;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float uu = cc[q] + rr[q], ll = cc[q] - rr[q];
            ap[q] += au * (au >= 0.f ? uu : ll);
            bp[q] += al * (al >= 0.f ? ll : uu);
          }
          pu[lane + 32 * k] = a;
          pl[lane + 32 * k] = b;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive1(empty + st);
      }
      if (err_exp && lane == 0) set_status(status, s, site_exp, err_exp);
      sm4_sync<NC>();
      // Σ rows: warp partials combined in warp order (f64) -- recomputed below for r
      double pnu = 0.0, pnl = 0.0;
      for (int d = tid; d < D; d += NC * 32) {
        double a = 0.0, b = 0.0;
        for (int w = 0; w < NC; ++w) {
          a += (double)part[(size_t)w * 2 * D + d];
          b += (double)part[(size_t)w * 2 * D + D + d];
        }
        pnu = qcombine<Q>(pnu, qpart<Q>(a));
        pnl = qcombine<Q>(pnl, qpart<Q>(b));
      }
      if (warp == 0) {  // propagate_sum_axis bias (relax.cpp:728-731)
        double a = 0.0, b = 0.0;
        for (int j = lane; j < n; j += 32) {
          a += e_lb[j];
          b += e_ub[j];
        }
        a = warp_sum(a);
        b = warp_sum(b);
        if (lane == 0) {
          scal[4] = a;
          scal[5] = b;
        }
      }
      sm4_reduce2<Q, NC>(pnu, pnl, red);
      if (tid == 0) {
        const double slb = scal[4], sub_ = scal[5];
        Lines ln;
        const int code = envelope(RELAX_RECIP, slb - e * fin.fin(pnl), sub_ + e * fin.fin(pnu), ln);
        if (code) set_status(status, s, site_recip, code);
        scal[0] = ln.al;
        scal[1] = ln.au;
        scal[2] = ln.al * (ln.al >= 0.0 ? slb : sub_) + ln.bl;
        scal[3] = ln.au * (ln.au >= 0.0 ? sub_ : slb) + ln.bu;
      }
      sm4_sync<NC>();
      const double r_al = scal[0], r_au = scal[1], r_lb = scal[2], r_ub = scal[3];
      pnu = pnl = 0.0;
      for (int d = tid; d < D; d += NC * 32) {
        double u = 0.0, l = 0.0;
        for (int w = 0; w < NC; ++w) {
          u += (double)part[(size_t)w * 2 * D + d];
          l += (double)part[(size_t)w * 2 * D + D + d];
        }
        const double yu = r_au * (r_au >= 0.0 ? u : l), yl = r_al * (r_al >= 0.0 ? l : u);
        ru_f[d] = (float)yu;
        rl_f[d] = (float)yl;
        pnu = qcombine<Q>(pnu, qpart<Q>(yu));
        pnl = qcombine<Q>(pnl, qpart<Q>(yl));
      }
      sm4_reduce2<Q, NC>(pnu, pnl, red);  // (its barriers also publish ru_f / rl_f)
      const double r_lo = r_lb - e * fin.fin(pnl);
      const double r_hi = r_ub + e * fin.fin(pnu);

      // pass 2: MulBroadcast per key (reverse key order), written to HBM
      const float ly = (float)r_lo, uy = (float)r_hi;
      const bool ly_p = ly >= 0.f, uy_p = uy >= 0.f;
      const float4* yu4 = reinterpret_cast<const float4*>(ru_f);
      const float4* yl4 = reinterpret_cast<const float4*>(rl_f);
      for (int m = warp; m < n; m += NC) {
        const int j = n - 1 - m;
        const long long ti = t0 + n + m;
        const int st = (int)(ti % ns);
        const float au = a_up_f[j], al = a_lo_f[j], lx = (float)e_lo[j];
        const bool au_p = au >= 0.f, al_p = al >= 0.f, lx_p = lx >= 0.f;
        sm4_wait(full + st, (uint32_t)((ti / ns) & 1));
        const float4* c4 = reinterpret_cast<const float4*>(ring + (size_t)st * 2 * D);
        const float4* r4 = c4 + D / 4;
        float4* gc = reinterpret_cast<float4*>(cbw + (long long)j * D);
        float4* gr = reinterpret_cast<float4*>(rbw + (long long)j * D);
        float fu = 0.f, fl = 0.f;
        for (int k = 0; k < KG; ++k) {
          const float4 cv = c4[lane + 32 * k], rv = r4[lane + 32 * k];
          const float4 yuv = yu4[lane + 32 * k], ylv = yl4[lane + 32 * k];
          const float cc[4] = {cv.x, cv.y, cv.z, cv.w}, rr[4] = {rv.x, rv.y, rv.z, rv.w};
          const float yuu[4] = {yuv.x, yuv.y, yuv.z, yuv.w}, yll[4] = {ylv.x, ylv.y, ylv.z, ylv.w};
          float oc[4], orr[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float u = cc[q] + rr[q], l = cc[q] - rr[q];
            const float eu = au * (au_p ? u : l), el = al * (al_p ? l : u);
            const float p_l = __fmaf_rn(ly, ly_p ? el : eu, lx * (lx_p ? yll[q] : yuu[q]));
            const float p_u = __fmaf_rn(uy, uy_p ? eu : el, lx * (lx_p ? yuu[q] : yll[q]));
            oc[q] = 0.5f * (p_u + p_l);
            orr[q] = 0.5f * (p_u - p_l);
            fu = qacc_f<Q>(fu, p_u);
            fl = qacc_f<Q>(fl, p_l);
          }
          gc[lane + 32 * k] = make_float4(oc[0], oc[1], oc[2], oc[3]);
          gr[lane + 32 * k] = make_float4(orr[0], orr[1], orr[2], orr[3]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive1(empty + st);
        const double gu = group_reduce<Q>((double)fu, 32), gl = group_reduce<Q>((double)fl, 32);
        if (lane == 0) {
          double olb = 0.0, oub = 0.0;
          term_bias(e_lo[j], r_lo, r_hi, e_lb[j], e_ub[j], r_lb, r_ub, olb, oub);
          const long long o = nb + j;
          sc.lb[o] = olb;
          sc.ub[o] = oub;
          if (sc.lo) {
            sc.lo[o] = olb - e * fin.fin(gl);
            sc.hi[o] = oub + e * fin.fin(gu);
          }
        }
      }
      sm4_sync<NC>();
    }
  }
  __syncthreads();
}

size_t softmax5_smem(int n, int D, int NC, int ns) {
  return (size_t)ns * 8 * D + (size_t)NC * 2 * D * 4 + (size_t)2 * D * 4 + (size_t)(n + 1) * (2 * 4 + 3 * 8) +
         64 * 8 + 2 * (size_t)ns * 8 + 64;
}

// Streaming softmax for narrow rows (D = 64 / 128: c1, c2).  A key row is only 0.5-1 KB, so a
// stage carries G = 512 / D consecutive keys (4 KB, one pair of bulk copies) and a consumer warp
// works on all G of them at once: LPK = 32 / G lanes per key, 16 columns per lane.  The per-key
// scalar work (norm reductions over LPK lanes, the exp envelope, the output bounds) then runs on
// G keys in parallel instead of one after the other; Σ partials of the G lane groups are
// combined with two shuffles at the end of pass 1.  Otherwise softmax4_kernel.
template <int Q, int NC, int G>
__global__ void __launch_bounds__((NC + 1) * 32, 4) softmax6_kernel(NView sc, int rows_per_s, int nrows, int n,
                                                                    const double* __restrict__ eps,
                                                                    int* __restrict__ status, int site_exp,
                                                                    int site_recip) {
  constexpr int D = 512 / G, LPK = 32 / G, NS = 2 * NC;  // 4 float4 groups per lane
  extern __shared__ __align__(16) unsigned char sm6[];
  float* ring = reinterpret_cast<float*>(sm6);  // [NS][c(G rows)|r(G rows)][D]
  float* part = ring + (size_t)NS * 2 * G * D;  // [NC][u|l][D]
  float* ru_f = part + (size_t)NC * 2 * D;
  float* rl_f = ru_f + D;
  const int n2 = (n + 1) & ~1;
  float* a_lo_f = rl_f + D;
  float* a_up_f = a_lo_f + n2;
  double* e_lb = reinterpret_cast<double*>(a_up_f + n2);
  double* e_ub = e_lb + n;
  double* e_lo = e_ub + n;
  double* red = e_lo + n;
  double* scal = red + 32;
  uint64_t* full = reinterpret_cast<uint64_t*>(scal + 32);
  uint64_t* empty = full + NS;
  const int ng = n / G;  // key groups per row

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kg = lane / LPK, sub = lane % LPK;  // key within the group, lane within the key
  if (tid == 0) {
    for (int b = 0; b < NS; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(full + b)) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(empty + b)) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == NC) {  // ---- producer: one stage = G consecutive keys (contiguous rows)
    if (lane == 0) {
      long long t = 0;
      for (int rid = blockIdx.x; rid < nrows; rid += gridDim.x) {
        const int s = rid / rows_per_s, row = rid % rows_per_s;
        const long long nb = (long long)s * sc.s_stride + (long long)row * n;
        const float* cb = sc.lam + nb * D;
        const float* rb = cb + sc.cr;
        for (int p = 0; p < 2; ++p)
          for (int gi = 0; gi < ng; ++gi, ++t) {
            const int st = (int)(t % NS);
            const uint32_t ph = (uint32_t)((t / NS) & 1);
            if (t >= NS) sm4_wait(empty + st, ph ^ 1u);
            float* dst = ring + (size_t)st * 2 * G * D;
            const int grp = p == 0 ? gi : ng - 1 - gi;  // pass 2 in reverse (L2 reuse)
            mbar_expect(full + st, 8u * G * D);
            asm volatile(
                "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_addr(dst)),
                "l"(cb + (long long)grp * G * D), "r"(4u * G * D), "r"(smem_addr(full + st))
                : "memory");
            asm volatile(
                "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_addr(dst + G * D)),
                "l"(rb + (long long)grp * G * D), "r"(4u * G * D), "r"(smem_addr(full + st))
                : "memory");
          }
      }
    }
    __syncwarp();
  } else {  // ---- consumers
    NormAcc<Q> fin;
    long long t0 = 0;
    for (int rid = blockIdx.x; rid < nrows; rid += gridDim.x, t0 += 2LL * ng) {
      const int s = rid / rows_per_s, row = rid % rows_per_s;
      const long long nb = (long long)s * sc.s_stride + (long long)row * n;
      float* cbw = sc.lam + nb * D;
      float* rbw = cbw + sc.cr;
      const double e = eps[s];
      float su[16], sl[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) su[k] = sl[k] = 0.f;
      int err_exp = 0;
      for (int gi = warp; gi < ng; gi += NC) {
        const long long ti = t0 + gi;
        const int st = (int)(ti % NS);
        const int j = gi * G + kg;
        const double xlb = sc.lb[nb + j], xub = sc.ub[nb + j];
        sm4_wait(full + st, (uint32_t)((ti / NS) & 1));
        const float4* c4 = reinterpret_cast<const float4*>(ring + (size_t)st * 2 * G * D + (size_t)kg * D);
        const float4* r4 = c4 + G * D / 4;
        float fu = 0.f, fl = 0.f;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float4 cv = c4[sub + LPK * k], rv = r4[sub + LPK * k];
          fu = qacc_f<Q>(fu, cv.x + rv.x); fl = qacc_f<Q>(fl, cv.x - rv.x);
          fu = qacc_f<Q>(fu, cv.y + rv.y); fl = qacc_f<Q>(fl, cv.y - rv.y);
          fu = qacc_f<Q>(fu, cv.z + rv.z); fl = qacc_f<Q>(fl, cv.z - rv.z);
          fu = qacc_f<Q>(fu, cv.w + rv.w); fl = qacc_f<Q>(fl, cv.w - rv.w);
        }
        const double nu = fin.fin(group_reduce<Q>((double)fu, LPK)), nl = fin.fin(group_reduce<Q>((double)fl, LPK));
        Lines ln;
        const int code = exp_envelope(xlb - e * nl, xub + e * nu, ln);
        if (code) err_exp = err_exp ? min(err_exp, code) : code;
        const float au = (float)ln.au, al = (float)ln.al;
        if (sub == 0) {
          a_lo_f[j] = al;
          a_up_f[j] = au;
          const double ub2 = ln.au * (ln.au >= 0.0 ? xub : xlb) + ln.bu;
          const double lb2 = ln.al * (ln.al >= 0.0 ? xlb : xub) + ln.bl;
          e_ub[j] = ub2;
          e_lb[j] = lb2;
          e_lo[j] = lb2 - e * fabs(ln.al) * (ln.al >= 0.0 ? nl : nu);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float4 cv = c4[sub + LPK * k], rv = r4[sub + LPK * k];
          const float cc[4] = {cv.x, cv.y, cv.z, cv.w}, rr[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float uu = cc[q] + rr[q], ll = cc[q] - rr[q];
            su[4 * k + q] += au * (au >= 0.f ? uu : ll);
            sl[4 * k + q] += al * (al >= 0.f ? ll : uu);
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive1(empty + st);
      }
      if (err_exp) set_status(status, s, site_exp, err_exp);
      // combine the G lane groups (same columns, different keys) in a fixed order
#pragma unroll
      for (int k = 0; k < 16; ++k)
        for (int o = LPK; o < 32; o <<= 1) {
          su[k] += __shfl_xor_sync(0xffffffffu, su[k], o);
          sl[k] += __shfl_xor_sync(0xffffffffu, sl[k], o);
        }
      if (kg == 0) {
        float4* pu = reinterpret_cast<float4*>(part + (size_t)warp * 2 * D);
        float4* pl = pu + D / 4;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          pu[sub + LPK * k] = make_float4(su[4 * k], su[4 * k + 1], su[4 * k + 2], su[4 * k + 3]);
          pl[sub + LPK * k] = make_float4(sl[4 * k], sl[4 * k + 1], sl[4 * k + 2], sl[4 * k + 3]);
        }
      }
      sm4_sync<NC>();
      double pnu = 0.0, pnl = 0.0;
      for (int d = tid; d < D; d += NC * 32) {
        double a = 0.0, b = 0.0;
        for (int w = 0; w < NC; ++w) {
          a += (double)part[(size_t)w * 2 * D + d];
          b += (double)part[(size_t)w * 2 * D + D + d];
        }
        pnu = qcombine<Q>(pnu, qpart<Q>(a));
        pnl = qcombine<Q>(pnl, qpart<Q>(b));
      }
      if (warp == 0) {
        double a = 0.0, b = 0.0;
        for (int j = lane; j < n; j += 32) {
          a += e_lb[j];
          b += e_ub[j];
        }
        a = warp_sum(a);
        b = warp_sum(b);
        if (lane == 0) {
          scal[4] = a;
          scal[5] = b;
        }
      }
      sm4_reduce2<Q, NC>(pnu, pnl, red);
      if (tid == 0) {
        const double slb = scal[4], sub_ = scal[5];
        Lines ln;
        const int code = envelope(RELAX_RECIP, slb - e * fin.fin(pnl), sub_ + e * fin.fin(pnu), ln);
        if (code) set_status(status, s, site_recip, code);
        scal[0] = ln.al;
        scal[1] = ln.au;
        scal[2] = ln.al * (ln.al >= 0.0 ? slb : sub_) + ln.bl;
        scal[3] = ln.au * (ln.au >= 0.0 ? sub_ : slb) + ln.bu;
      }
      sm4_sync<NC>();
      const double r_al = scal[0], r_au = scal[1], r_lb = scal[2], r_ub = scal[3];
      pnu = pnl = 0.0;
      for (int d = tid; d < D; d += NC * 32) {
        double u = 0.0, l = 0.0;
        for (int w = 0; w < NC; ++w) {
          u += (double)part[(size_t)w * 2 * D + d];
          l += (double)part[(size_t)w * 2 * D + D + d];
        }
        const double yu = r_au * (r_au >= 0.0 ? u : l), yl = r_al * (r_al >= 0.0 ? l : u);
        ru_f[d] = (float)yu;
        rl_f[d] = (float)yl;
        pnu = qcombine<Q>(pnu, qpart<Q>(yu));
        pnl = qcombine<Q>(pnl, qpart<Q>(yl));
      }
      sm4_reduce2<Q, NC>(pnu, pnl, red);
      const double r_lo = r_lb - e * fin.fin(pnl);
      const double r_hi = r_ub + e * fin.fin(pnu);

      const float ly = (float)r_lo, uy = (float)r_hi;
      const bool ly_p = ly >= 0.f, uy_p = uy >= 0.f;
      const float4* yu4 = reinterpret_cast<const float4*>(ru_f);
      const float4* yl4 = reinterpret_cast<const float4*>(rl_f);
      for (int m = warp; m < ng; m += NC) {
        const int grp = ng - 1 - m;  // the producer streams pass 2 in reverse group order
        const int j = grp * G + kg;
        const long long ti = t0 + ng + m;
        const int st = (int)(ti % NS);
        const float au = a_up_f[j], al = a_lo_f[j], lx = (float)e_lo[j];
        const bool au_p = au >= 0.f, al_p = al >= 0.f, lx_p = lx >= 0.f;
        sm4_wait(full + st, (uint32_t)((ti / NS) & 1));
        const float4* c4 = reinterpret_cast<const float4*>(ring + (size_t)st * 2 * G * D + (size_t)kg * D);
        const float4* r4 = c4 + G * D / 4;
        float4* gc = reinterpret_cast<float4*>(cbw + (long long)j * D);
        float4* gr = reinterpret_cast<float4*>(rbw + (long long)j * D);
        float fu = 0.f, fl = 0.f;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float4 cv = c4[sub + LPK * k], rv = r4[sub + LPK * k];
          const float4 yuv = yu4[sub + LPK * k], ylv = yl4[sub + LPK * k];
          const float cc[4] = {cv.x, cv.y, cv.z, cv.w}, rr[4] = {rv.x, rv.y, rv.z, rv.w};
          const float yuu[4] = {yuv.x, yuv.y, yuv.z, yuv.w}, yll[4] = {ylv.x, ylv.y, ylv.z, ylv.w};
          float oc[4], orr[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float u = cc[q] + rr[q], l = cc[q] - rr[q];
            const float eu = au * (au_p ? u : l), el = al * (al_p ? l : u);
            const float p_l = __fmaf_rn(ly, ly_p ? el : eu, lx * (lx_p ? yll[q] : yuu[q]));
            const float p_u = __fmaf_rn(uy, uy_p ? eu : el, lx * (lx_p ? yuu[q] : yll[q]));
            oc[q] = 0.5f * (p_u + p_l);
            orr[q] = 0.5f * (p_u - p_l);
            fu = qacc_f<Q>(fu, p_u);
            fl = qacc_f<Q>(fl, p_l);
          }
          gc[sub + LPK * k] = make_float4(oc[0], oc[1], oc[2], oc[3]);
          gr[sub + LPK * k] = make_float4(orr[0], orr[1], orr[2], orr[3]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive1(empty + st);
        const double gu = group_reduce<Q>((double)fu, LPK), gl = group_reduce<Q>((double)fl, LPK);
        if (sub == 0) {
          double olb = 0.0, oub = 0.0;
          term_bias(e_lo[j], r_lo, r_hi, e_lb[j], e_ub[j], r_lb, r_ub, olb, oub);
          const long long o = nb + j;
          sc.lb[o] = olb;
          sc.ub[o] = oub;
          if (sc.lo) {
            sc.lo[o] = olb - e * fin.fin(gl);
            sc.hi[o] = oub + e * fin.fin(gu);
          }
        }
      }
      sm4_sync<NC>();
    }
  }
  __syncthreads();
}

size_t softmax6_smem(int n, int D, int NC) {
  const int G = 512 / D;
  return (size_t)2 * NC * 8 * G * D + (size_t)NC * 2 * D * 4 + (size_t)2 * D * 4 +
         (size_t)(n + 1) * (2 * 4 + 3 * 8) + 64 * 8 + 2 * (size_t)2 * NC * 8 + 64;
}

size_t softmax3_smem(int n, int Dc, int CS, int nbuf) {
  return (size_t)nbuf * n * Dc * 8 + (size_t)Dc * 8 + (size_t)Dc * 16 + (size_t)n * 6 * 8 +
         (size_t)2 * CS * 2 * n * 8 + (size_t)8 * CS * 8 + (32 + 8) * 8 + (size_t)8 * kSm3Threads * 8 +
         (2 * kSm3MaxBars + 8) * 8 + (size_t)n * 8;
}

// Lanes per key row: about 16 columns per lane, a power of two in [1, 32].
int softmax3_lpk(int Dc) {
  int l = 1;
  while (l < 32 && l * 16 < Dc) l *= 2;
  return l;
}

// Cluster size for the single-read softmax: the smallest power of two (<= 16) that divides
// D/4 and brings the CTA's row tile (n*Dc*8 bytes) to <= `tile_kb`; else the smallest one
// that fits SMEM at all; 0 when none does.
int softmax3_cluster(int n, int D, int nbuf, int tile_kb) {
  if (D % 4) return 0;
  int best = 0;
  for (int cs = 1; cs <= 16; cs *= 2) {
    if ((D / 4) % cs) break;
    const size_t sm = softmax3_smem(n, D / cs, cs, nbuf);
    if (sm <= 227 * 1024 && best == 0) best = cs;
    if ((size_t)n * (D / cs) * 8 <= (size_t)tile_kb * 1024) return sm <= 227 * 1024 ? cs : best;
  }
  return best;
}


// ---------------------------------------------------------------------------
// Input binding, mean pooling, classifier head
// ---------------------------------------------------------------------------
// Word-level binding: slot s holds sentence slot_map[s]; rows of the
// W perturbed positions are one-hot into columns w*E + e, all other rows zero.
__global__ void init_input_kernel(float* lam, long long cr, double* lb, double* ub, const double* x,
                                  const int* positions, const int* slot_map, int S, int L, int E,
                                  int W, int D, int col0) {
  long long row = (long long)blockIdx.x * (blockDim.x / kWarp) + threadIdx.x / kWarp;
  int lane = threadIdx.x & (kWarp - 1);
  long long nrows = (long long)S * L * E;
  if (row >= nrows) return;
  int e = (int)(row % E);
  int tok = (int)((row / E) % L);
  int s = (int)(row / ((long long)L * E));
  int src = slot_map ? slot_map[s] : s;
  if (lane == 0) {
    long long xi = ((long long)src * L + tok) * E + e;
    lb[row] = x[xi];
    ub[row] = x[xi];
  }
  if (!lam) return;  // bias-only binding (the first layer consumes Λ0 analytically)
  float* c = lam + row * D;
  float* r = c + cr;
  int hot = -1;
  for (int w = 0; w < W; ++w)
    if (positions[src * W + w] == tok) hot = w * E + e - col0;  // local column of this shard
  for (int d = lane * 4; d < D; d += 4 * kWarp) {
    float v[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int t = 0; t < 4; ++t) v[t] = (hot == d + t) ? 1.0f : 0.0f;
    *reinterpret_cast<float4*>(c + d) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4*>(r + d) = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// First-layer Q/K/V Λ without a GEMM.  Λ0 is one-hot (centre plane 1 at column w*E + e of the
// perturbed token pos[w], radius 0), so propagate_affine's Λ output is W itself scattered:
//   out_c[s, t, o, d] = W[e][o] if t == pos[w] and d == w*E + e (global column), else 0;
//   out_r = |W| . 0 = 0.
// Exact (no TF32 splitting of a product with 1).  Row (s, t, o) per warp, float4 stores.
// Rows of neurons o < skip_o at unperturbed tokens are not written (skip_o = 2E when every
// layer-1 reader of Q/K Λ gathers the perturbed tokens only: concretize_tokens and the gathered
// McCormick GEMMs); V rows (and everything at skip_o = 0) are written, zeros included.
__global__ void onehot_affine_kernel(float* lam, long long cr, const float* __restrict__ w, const int* positions,
                                     const int* slot_map, int S, int L, int E, int O, int W, int D, int col0,
                                     int skip_o) {
  long long row = (long long)blockIdx.x * (blockDim.x / kWarp) + threadIdx.x / kWarp;
  int lane = threadIdx.x & (kWarp - 1);
  long long nrows = (long long)S * L * O;
  if (row >= nrows) return;
  const int o = (int)(row % O);
  const int tok = (int)((row / O) % L);
  const int s = (int)(row / ((long long)L * O));
  const int src = slot_map ? slot_map[s] : s;
  int word = -1;
  for (int q = 0; q < W; ++q)
    if (positions[src * W + q] == tok) word = q;
  if (word < 0 && o < skip_o) return;
  float* c = lam + row * D;
  float* r = c + cr;
  for (int d = lane * 4; d < D; d += 4 * kWarp) {
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    if (word >= 0) {
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int e = col0 + d + t - word * E;  // embedding index of this (global) column
        if (e >= 0 && e < E) v[t] = w[(long long)e * O + o];
      }
    }
    *reinterpret_cast<float4*>(c + d) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4*>(r + d) = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// Residual add of Λ0 (propagate_add(x, .), relax.cpp:656-674) without reading it: +1 on the
// centre plane at (s, pos[w], e, column w*E + e).
__global__ void add_onehot_kernel(float* lam, const int* positions, const int* slot_map, int S, int L, int E, int W,
                                  int D, int col0) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)S * W * E) return;
  const int e = (int)(t % E);
  const int q = (int)((t / E) % W);
  const int s = (int)(t / ((long long)W * E));
  const int src = slot_map ? slot_map[s] : s;
  const int col = q * E + e - col0;
  if (col < 0 || col >= D) return;
  const int tok = positions[src * W + q];
  lam[(((long long)s * L + tok) * E + e) * D + col] += 1.0f;
}

__global__ void meanpool_kernel(const float* lam, long long cr, const double* lb, const double* ub,
                                double* pc, double* pr, double* plb, double* pub, int S, int L,
                                int E, int D) {
  int d = blockIdx.x * blockDim.x + threadIdx.x;
  int e = blockIdx.y, s = blockIdx.z;
  double inv = 1.0 / (double)L;
  if (d < D) {
    double ac = 0.0, ar = 0.0;
    for (int t = 0; t < L; ++t) {
      const float* c = lam + (((long long)s * L + t) * E + e) * D;
      ac += (double)c[d];
      ar += (double)c[d + cr];
    }
    pc[((long long)s * E + e) * D + d] = inv * ac;
    pr[((long long)s * E + e) * D + d] = inv * ar;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // sum_axis then scale (graph.cpp:628-634)
    double slb = 0.0, sub = 0.0;
    for (int t = 0; t < L; ++t) {
      slb += lb[((long long)s * L + t) * E + e];
      sub += ub[((long long)s * L + t) * E + e];
    }
    plb[(long long)s * E + e] = inv * slb;
    pub[(long long)s * E + e] = inv * sub;
  }
}

// meanpool_kernel with four columns per thread (float4 loads, D % 4 == 0): per column the same
// t-ascending f64 sums, so results are bit-identical; 4x fewer load instructions per byte.
__global__ void meanpool4_kernel(const float* lam, long long cr, const double* lb, const double* ub, double* pc,
                                 double* pr, double* plb, double* pub, int S, int L, int E, int D) {
  const int d = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
  const int e = blockIdx.y, s = blockIdx.z;
  const double inv = 1.0 / (double)L;
  if (d < D) {
    double ac[4] = {0.0, 0.0, 0.0, 0.0}, ar[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 4
    for (int t = 0; t < L; ++t) {
      const float* c = lam + (((long long)s * L + t) * E + e) * D + d;
      const float4 cv = *reinterpret_cast<const float4*>(c), rv = *reinterpret_cast<const float4*>(c + cr);
      ac[0] += (double)cv.x; ac[1] += (double)cv.y; ac[2] += (double)cv.z; ac[3] += (double)cv.w;
      ar[0] += (double)rv.x; ar[1] += (double)rv.y; ar[2] += (double)rv.z; ar[3] += (double)rv.w;
    }
    double* oc = pc + ((long long)s * E + e) * D + d;
    double* orr = pr + ((long long)s * E + e) * D + d;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      oc[q] = inv * ac[q];
      orr[q] = inv * ar[q];
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // sum_axis then scale (graph.cpp:628-634)
    double slb = 0.0, sub = 0.0;
    for (int t = 0; t < L; ++t) {
      slb += lb[((long long)s * L + t) * E + e];
      sub += ub[((long long)s * L + t) * E + e];
    }
    plb[(long long)s * E + e] = inv * slb;
    pub[(long long)s * E + e] = inv * sub;
  }
}

template <int Q>
__global__ void head_kernel(const double* pc, const double* pr, const double* plb, const double* pub,
                            const double* wc, const double* bc, int E, int C, int D,
                            const double* eps, double* out_lo, double* out_hi, int* status,
                            int site) {
  __shared__ double red[32];
  int s = blockIdx.x / C, cls = blockIdx.x % C;
  double nu = 0.0, nl = 0.0;
  int finite = 1;
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    double ac = 0.0, ar = 0.0;
    for (int e = 0; e < E; ++e) {
      double w = wc[e * C + cls];
      ac += w * pc[((long long)s * E + e) * D + d];
      ar += fabs(w) * pr[((long long)s * E + e) * D + d];
    }
    double u = ac + ar, l = ac - ar;
    finite &= (isfinite(u) && isfinite(l));
    if (Q == NORM_L1) { nu += fabs(u); nl += fabs(l); }
    else if (Q == NORM_L2) { nu += u * u; nl += l * l; }
    else { nu = fmax(nu, fabs(u)); nl = fmax(nl, fabs(l)); }
  }
  finite = __syncthreads_and(finite);
  nu = block_reduce<Q>(nu, red);
  nl = block_reduce<Q>(nl, red);
  if (threadIdx.x == 0) {
    double ub_pos = 0.0, ub_neg = 0.0, lb_pos = 0.0, lb_neg = 0.0;  // relax.cpp:280-299
    for (int i = 0; i < E; ++i) {
      double wv = wc[i * C + cls];
      double wp = (wv < 0.0) ? 0.0 : wv, wn = (0.0 < wv) ? 0.0 : wv;
      double xu = pub[(long long)s * E + i], xl = plb[(long long)s * E + i];
      ub_pos += wp * xu;
      ub_neg += wn * xl;
      lb_pos += wp * xl;
      lb_neg += wn * xu;
    }
    double yub = ub_pos + ub_neg + bc[cls];
    double ylb = lb_pos + lb_neg + bc[cls];
    if (!finite || !isfinite(yub) || !isfinite(ylb)) set_status(status, s, site, kCodeDomain);
    NormAcc<Q> fin;
    double e = eps[s];
    out_lo[(long long)s * C + cls] = ylb - e * fin.fin(nl);
    out_hi[(long long)s * C + cls] = yub + e * fin.fin(nu);
  }
}

// The same classifier head, one CTA per sentence for all classes at once (C <= kHeadMaxC): each
// pooled Λ element is loaded once for every class, and a CTA's 512 threads cover D, so the
// whole head is one short wave instead of S*C single CTAs walking E serially.  Per (s, class, d)
// the accumulation is the same (e ascending, same operations) as head_kernel.
constexpr int kHeadMaxC = 8;
constexpr int kHeadThreads = 512;

template <int Q>
__global__ void __launch_bounds__(kHeadThreads) head_all_kernel(const double* pc, const double* pr,
                                                                const double* plb, const double* pub,
                                                                const double* wc, const double* bc, int E, int C,
                                                                int D, const double* eps, double* out_lo,
                                                                double* out_hi, int* status, int site) {
  __shared__ double red[32];
  const int s = blockIdx.x;
  double nu[kHeadMaxC], nl[kHeadMaxC];
#pragma unroll
  for (int c = 0; c < kHeadMaxC; ++c) nu[c] = nl[c] = 0.0;
  int finite = 1;
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    double ac[kHeadMaxC], ar[kHeadMaxC];
#pragma unroll
    for (int c = 0; c < kHeadMaxC; ++c) ac[c] = ar[c] = 0.0;
    for (int e = 0; e < E; ++e) {
      const double vc = pc[((long long)s * E + e) * D + d], vr = pr[((long long)s * E + e) * D + d];
#pragma unroll
      for (int c = 0; c < kHeadMaxC; ++c) {
        if (c >= C) break;
        const double w = wc[e * C + c];
        ac[c] += w * vc;
        ar[c] += fabs(w) * vr;
      }
    }
#pragma unroll
    for (int c = 0; c < kHeadMaxC; ++c) {
      if (c >= C) break;
      const double u = ac[c] + ar[c], l = ac[c] - ar[c];
      finite &= (isfinite(u) && isfinite(l));
      if (Q == NORM_L1) { nu[c] += fabs(u); nl[c] += fabs(l); }
      else if (Q == NORM_L2) { nu[c] += u * u; nl[c] += l * l; }
      else { nu[c] = fmax(nu[c], fabs(u)); nl[c] = fmax(nl[c], fabs(l)); }
    }
  }
  finite = __syncthreads_and(finite);
  for (int c = 0; c < C; ++c) {
    const double gu = block_reduce<Q>(nu[c], red);
    const double gl = block_reduce<Q>(nl[c], red);
    if (threadIdx.x == 0) {
      double ub_pos = 0.0, ub_neg = 0.0, lb_pos = 0.0, lb_neg = 0.0;  // relax.cpp:280-299
      for (int i = 0; i < E; ++i) {
        const double wv = wc[i * C + c];
        const double wp = (wv < 0.0) ? 0.0 : wv, wn = (0.0 < wv) ? 0.0 : wv;
        const double xu = pub[(long long)s * E + i], xl = plb[(long long)s * E + i];
        ub_pos += wp * xu;
        ub_neg += wn * xl;
        lb_pos += wp * xl;
        lb_neg += wn * xu;
      }
      const double yub = ub_pos + ub_neg + bc[c];
      const double ylb = lb_pos + lb_neg + bc[c];
      if (!finite || !isfinite(yub) || !isfinite(ylb)) set_status(status, s, site, kCodeDomain);
      NormAcc<Q> fin;
      const double e = eps[s];
      out_lo[(long long)s * C + c] = ylb - e * fin.fin(gl);
      out_hi[(long long)s * C + c] = yub + e * fin.fin(gu);
    }
  }
}

template <int Q>
__global__ void concretize_f64_kernel(const double* pc, const double* pr, const double* lb,
                                      const double* ub, long long rows_per_s, long long nrows,
                                      int D, const double* eps, double* lo, double* hi) {
  long long row = (long long)blockIdx.x * (blockDim.x / kWarp) + threadIdx.x / kWarp;
  int lane = threadIdx.x & (kWarp - 1);
  if (row >= nrows) return;
  double nu = 0.0, nl = 0.0;
  for (int d = lane; d < D; d += kWarp) {
    double u = pc[row * D + d] + pr[row * D + d], l = pc[row * D + d] - pr[row * D + d];
    if (Q == NORM_L1) { nu += fabs(u); nl += fabs(l); }
    else if (Q == NORM_L2) { nu += u * u; nl += l * l; }
    else { nu = fmax(nu, fabs(u)); nl = fmax(nl, fabs(l)); }
  }
  if (Q == NORM_LINF) { nu = warp_max(nu); nl = warp_max(nl); }
  else { nu = warp_sum(nu); nl = warp_sum(nl); }
  if (lane == 0) {
    NormAcc<Q> fin;
    double e = eps[row / rows_per_s];
    lo[row] = lb[row] - e * fin.fin(nl);
    hi[row] = ub[row] + e * fin.fin(nu);
  }
}

// ---------------------------------------------------------------------------
// Operator-level helpers
// ---------------------------------------------------------------------------
// Reference layout [n, d] f64 (lw, uw) <-> padded center/radius planes [n, Dp] f32.
__global__ void ul_to_cr_kernel(const double* lw, const double* uw, float* lam, long long cr,
                                long long n, int d, int Dp) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * Dp) return;
  long long row = i / Dp;
  int col = (int)(i % Dp);
  double u = 0.0, l = 0.0;
  if (col < d) {
    u = uw[row * d + col];
    l = lw[row * d + col];
  }
  lam[i] = (float)(0.5 * (u + l));
  lam[i + cr] = (float)(0.5 * (u - l));
}

__global__ void cr_to_ul_kernel(const float* lam, long long cr, double* lw, double* uw,
                                long long n, int d, int Dp) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * d) return;
  long long row = i / d;
  int col = (int)(i % d);
  double c = lam[row * Dp + col], r = lam[row * Dp + col + cr];
  uw[i] = c + r;
  lw[i] = c - r;
}

__global__ void add_kernel(const float* a, long long acr, const double* alb, const double* aub,
                           const float* b, long long bcr, const double* blb, const double* bub,
                           float* y, long long ycr, double* ylb, double* yub, long long n, int D) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n * D) {
    // u/l sums in f64 (relax.cpp:669-672), then back to center/radius
    double au = (double)a[i] + a[i + acr], al = (double)a[i] - a[i + acr];
    double bu = (double)b[i] + b[i + bcr], bl = (double)b[i] - b[i + bcr];
    double u = au + bu, l = al + bl;
    y[i] = (float)(0.5 * (u + l));
    y[i + ycr] = (float)(0.5 * (u - l));
  }
  if (i < n) {
    ylb[i] = alb[i] + blb[i];
    yub[i] = aub[i] + bub[i];
  }
}

__global__ void scale_kernel(const float* x, long long xcr, const double* xlb, const double* xub,
                             double s, float* y, long long ycr, double* ylb, double* yub,
                             long long n, int D) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n * D) {  // relax.cpp:683-701: c' = s c, r' = |s| r
    y[i] = (float)(s * (double)x[i]);
    y[i + ycr] = (float)(fabs(s) * (double)x[i + xcr]);
  }
  if (i < n) {
    if (s >= 0.0) {
      ylb[i] = s * xlb[i];
      yub[i] = s * xub[i];
    } else {
      ylb[i] = s * xub[i];
      yub[i] = s * xlb[i];
    }
  }
}

__global__ void fill_int_kernel(int* p, int v, long long n) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

// TF32 split of a coefficient: hi = rna_tf32(v), lo = v - hi (exact).
__device__ __forceinline__ void split_store(float* hi, float* lo, long long i, double v) {
  float f = (float)v;
  uint32_t hb;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(f));
  float h = __uint_as_float(hb);
  hi[i] = h;
  lo[i] = f - h;
}

// McCormick coefficients of Q.K^T for the tcgen05 engine (K-major, see fg_internal.cuh).
// The contraction index k runs over kp >= hd (hd rounded up to the engine's 32-deep K steps);
// coefficients of the padding k in [hd, kp) are zero, so the Λ rows the padded K reads past the
// head (the next head's, finite) contribute exactly nothing.
__global__ void sim_coef_split_kernel(NView q, NView k, int H, int L, int hd, int kp, float* xh, float* xl,
                                      float* yh, float* yl) {
  const int sh = blockIdx.x;
  const int s = sh / H, h = sh % H;
  for (int t = threadIdx.x; t < L * kp; t += blockDim.x) {
    const int j = t / kp, kk = t % kp;
    const long long x0 = ((long long)(sh * 2 + 0) * L + j) * 2 * kp, x1 = ((long long)(sh * 2 + 1) * L + j) * 2 * kp;
    const long long y0 = ((long long)(sh * 2 + 0) * L + j) * kp + kk, y1 = ((long long)(sh * 2 + 1) * L + j) * kp + kk;
    if (kk >= hd) {  // padding: zero coefficients
      xh[x0 + kk] = xl[x0 + kk] = 0.f;
      xh[x0 + kp + kk] = xl[x0 + kp + kk] = 0.f;
      xh[x1 + kk] = xl[x1 + kk] = 0.f;
      xh[x1 + kp + kk] = xl[x1 + kp + kk] = 0.f;
      yh[y0] = yl[y0] = 0.f;
      yh[y1] = yl[y1] = 0.f;
      continue;
    }
    const long long yi = nidx(k, s, j, h * hd + kk);
    const double ly = k.lo[yi], uy = k.hi[yi];
    split_store(xh, xl, x0 + kk, 0.5 * (ly + uy));
    split_store(xh, xl, x0 + kp + kk, 0.5 * (fabs(uy) - fabs(ly)));
    split_store(xh, xl, x1 + kk, 0.5 * (uy - ly));
    split_store(xh, xl, x1 + kp + kk, 0.5 * (fabs(uy) + fabs(ly)));
    const double lx = q.lo[nidx(q, s, j, h * hd + kk)];  // row i = j of Q
    split_store(yh, yl, y0, lx);
    split_store(yh, yl, y1, fabs(lx));
  }
}

// McCormick coefficients of P.V for the tcgen05 engine.
__global__ void wv_coef_split_kernel(NView p, NView v, int H, int L, int hd, float* xh, float* xl, float* yh,
                                     float* yl) {
  const int sh = blockIdx.x;
  const int s = sh / H, h = sh % H;
  for (int t = threadIdx.x; t < hd * L; t += blockDim.x) {
    const int kk = t / L, j = t % L;
    const long long yi = nidx(v, s, j, h * hd + kk);
    const double ly = v.lo[yi], uy = v.hi[yi];
    const long long x0 = ((long long)(sh * 2 + 0) * hd + kk) * 2 * L, x1 = ((long long)(sh * 2 + 1) * hd + kk) * 2 * L;
    split_store(xh, xl, x0 + j, 0.5 * (ly + uy));
    split_store(xh, xl, x0 + L + j, 0.5 * (fabs(uy) - fabs(ly)));
    split_store(xh, xl, x1 + j, 0.5 * (uy - ly));
    split_store(xh, xl, x1 + L + j, 0.5 * (fabs(uy) + fabs(ly)));
  }
  for (int t = threadIdx.x; t < L * L; t += blockDim.x) {
    const int i = t / L, j = t % L;
    const double lx = p.lo[nidx(p, s, (long long)h * L + i, j)];
    split_store(yh, yl, ((long long)(sh * 2 + 0) * L + i) * L + j, lx);
    split_store(yh, yl, ((long long)(sh * 2 + 1) * L + i) * L + j, fabs(lx));
  }
}

inline unsigned blocks_for(long long n, int per_block) {
  return (unsigned)((n + per_block - 1) / per_block);
}

}  // namespace

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
bool rows2_enabled() {  // comparison runs: FG_NO_ROWS2=1 keeps one row per warp for narrow rows
  static const bool v = getenv("FG_NO_ROWS2") == nullptr;
  return v;
}

#define DISPATCH_Q(q, KERNEL, ...)                        \
  switch (q) {                                            \
    case NORM_L1: KERNEL<NORM_L1> __VA_ARGS__; break;     \
    case NORM_L2: KERNEL<NORM_L2> __VA_ARGS__; break;     \
    default: KERNEL<NORM_LINF> __VA_ARGS__; break;        \
  }

int launch_concretize(const float* lam, long long cr, const double* lb, const double* ub,
                      long long rows_per_s, long long nrows, int D, int norm, const double* eps,
                      double* lo, double* hi, cudaStream_t st, const int* skip) {
  if (nrows <= 0) return 0;
  if (rows2_enabled() && D % 4 == 0 && D <= 256) {
    DISPATCH_Q(dual_norm(norm), concretize_rows2_kernel,
               <<<blocks_for((nrows + 1) / 2, 8), 256, 0, st>>>(lam, cr, lb, ub, rows_per_s, nrows, D, eps, lo, hi,
                                                                 skip));
    return 1;
  }
  dim3 grid(blocks_for(nrows, 8)), block(256);
  DISPATCH_Q(dual_norm(norm), concretize_kernel,
             <<<grid, block, 0, st>>>(lam, cr, lb, ub, rows_per_s, nrows, D, eps, lo, hi, skip));
  return 1;
}

int launch_concretize_tokens(const float* lam, long long cr, const double* lb, const double* ub,
                             long long rows_per_s, long long nrows, int D, int norm, const double* eps,
                             double* lo, double* hi, const int* positions, const int* slot_map, int W, int width,
                             cudaStream_t st) {
  if (nrows <= 0) return 0;
  if (D % 4 == 0 && getenv("FG_TOKENS_ONEPASS") == nullptr) {  // env: comparison runs
    concretize_cold_kernel<<<blocks_for(nrows, 256), 256, 0, st>>>(lb, ub, rows_per_s, nrows, lo, hi, positions,
                                                                   slot_map, W, width);
    const int S = (int)(nrows / rows_per_s);
    DISPATCH_Q(dual_norm(norm), concretize_hot_kernel,
               <<<blocks_for((long long)S * W * width, 8), 256, 0, st>>>(lam, cr, lb, ub, rows_per_s, S, D, eps, lo,
                                                                          hi, positions, slot_map, W, width));
    return 2;
  }
  DISPATCH_Q(dual_norm(norm), concretize_tokens_kernel,
             <<<blocks_for(nrows, 8), 256, 0, st>>>(lam, cr, lb, ub, rows_per_s, nrows, D, eps, lo, hi, positions,
                                                     slot_map, W, width));
  return 1;
}

int launch_elementwise_verify(int kind, float* lam, long long cr, double* lb, double* ub,
                              long long rows_per_s, long long nrows, int D, int norm,
                              const double* eps, int* status, int site, double* lo_out,
                              double* hi_out, cudaStream_t st, const double* lo_in, const double* hi_in,
                              const int* skip, unsigned char* keep) {
  if (nrows <= 0) return 0;
  if (rows2_enabled() && !lo_in && D % 4 == 0 && D <= 256) {
    DISPATCH_Q(dual_norm(norm), elementwise_verify_rows2_kernel,
               <<<blocks_for((nrows + 1) / 2, 8), 256, 0, st>>>(kind, lam, cr, lb, ub, rows_per_s, nrows, D, eps,
                                                                 status, site, lo_out, hi_out, skip, keep));
    return 1;
  }
  dim3 grid(blocks_for(nrows, 8)), block(256);
  DISPATCH_Q(dual_norm(norm), elementwise_verify_kernel,
             <<<grid, block, 0, st>>>(kind, lam, cr, lb, ub, rows_per_s, nrows, D, eps, status,
                                      site, lo_out, hi_out, lo_in, hi_in, skip, keep));
  return 1;
}

int launch_relax(int kind, const double* lo, const double* hi, long long n, double* a_low,
                 double* b_low, double* a_up, double* b_up, int* status, cudaStream_t st) {
  if (n <= 0) return 0;
  relax_kernel<<<blocks_for(n, 128), 128, 0, st>>>(kind, lo, hi, n, a_low, b_low, a_up, b_up,
                                                   status);
  return 1;
}

int launch_compose(float* lam_in, long long cr_in, const double* lb_in, const double* ub_in,
                   const double* a_low, const double* b_low, const double* a_up,
                   const double* b_up, float* lam_out, long long cr_out, double* lb_out,
                   double* ub_out, long long n, int D, cudaStream_t st) {
  if (n <= 0) return 0;
  compose_kernel<<<blocks_for(n, 8), 256, 0, st>>>(lam_in, cr_in, lb_in, ub_in, a_low, b_low, a_up,
                                                   b_up, lam_out, cr_out, lb_out, ub_out, n, D);
  return 1;
}

int launch_affine_bias(const double* lb_in, const double* ub_in, const double* w64,
                       const double* bias, const double* res_lb, const double* res_ub,
                       double* lb_out, double* ub_out, int S, int rows, int C, int O,
                       cudaStream_t st, const int* skip) {
  long long nrows = (long long)S * rows;
  long long total = nrows * O;
  if (total <= 0) return 0;
  dim3 grid(blocks_for(O, kBgJ), blocks_for(nrows, kBgR));
  affine_bias_kernel<<<grid, 256, 0, st>>>(lb_in, ub_in, w64, bias, res_lb, res_ub, lb_out, ub_out, nrows,
                                                 C, O, skip, rows);
  return 1;
}

int launch_dot_similarity(const NView& q, const NView& k, const NView& out, int S, int L, int H,
                          int hd, int D, float* ws, float scale, cudaStream_t st) {
  int n = 0;
  sim_coef_kernel<<<S * H, 256, 0, st>>>(q, k, H, L, hd, ws);
  ++n;
  sim_bias(q, k, out, S, H, L, hd, (double)scale, st);
  ++n;
  const long long per = 6LL * hd * L;
  // x-side (Q rows scaled by K-derived coefficients): batch (s, h, i, out plane)
  GemmArgs g{};
  g.M = L; g.N = D; g.K = 2 * hd; g.K0 = hd;
  g.A = ws; g.lda = L;
  g.B = q.lam + (long long)(q.col0) * D; g.ldb = D; g.b_off1 = q.cr;
  g.C = out.lam + (long long)out.col0 * D; g.ldc = D;
  g.alpha = scale; g.accumulate = 0;
  g.nb[0] = S; g.nb[1] = H; g.nb[2] = L; g.nb[3] = 2;
  g.sA[0] = H * per; g.sA[1] = per; g.sA[2] = 0; g.sA[3] = 2LL * hd * L;
  g.sB[0] = q.s_stride * D; g.sB[1] = (long long)hd * D; g.sB[2] = (long long)q.row_stride * D; g.sB[3] = 0;
  g.sC[0] = out.s_stride * D; g.sC[1] = (long long)L * L * D; g.sC[2] = (long long)L * D; g.sC[3] = out.cr;
  {
    const int r = launch_gemm(g, st);
    if (r < 0) return r;  // unsupported shape: reported by the caller, never silently skipped
    n += r;
  }
  // y-side (K rows scaled by lx of Q): batch (s, h, j, plane), accumulate
  GemmArgs t{};
  t.M = L; t.N = D; t.K = hd; t.K0 = hd;
  t.A = ws + 4LL * hd * L; t.lda = L;
  t.B = k.lam + (long long)k.col0 * D; t.ldb = D; t.b_off1 = 0;
  t.C = out.lam + (long long)out.col0 * D; t.ldc = (long long)L * D;
  t.alpha = scale; t.accumulate = 1;
  t.nb[0] = S; t.nb[1] = H; t.nb[2] = L; t.nb[3] = 2;
  t.sA[0] = H * per; t.sA[1] = per; t.sA[2] = 0; t.sA[3] = (long long)hd * L;
  t.sB[0] = k.s_stride * D; t.sB[1] = (long long)hd * D; t.sB[2] = (long long)k.row_stride * D; t.sB[3] = k.cr;
  t.sC[0] = out.s_stride * D; t.sC[1] = (long long)L * L * D; t.sC[2] = D; t.sC[3] = out.cr;
  {
    const int r = launch_gemm(t, st);
    if (r < 0) return r;  // unsupported shape: reported by the caller, never silently skipped
    n += r;
  }
  return n;
}

int launch_dot_weighted(const NView& p, const NView& v, const NView& out, int S, int L, int H,
                        int hd, int D, float* ws, cudaStream_t st) {
  int n = 0;
  wv_coef_kernel<<<S * H, 256, 0, st>>>(p, v, H, L, hd, ws);
  ++n;
  wv_bias(p, v, out, S, H, L, hd, st);
  ++n;
  const long long per = 4LL * L * hd + 2LL * L * L;
  // x-side (P rows scaled by V-derived coefficients): batch (s, h, i, out plane)
  GemmArgs g{};
  g.M = hd; g.N = D; g.K = 2 * L; g.K0 = L;
  g.A = ws; g.lda = hd;
  g.B = p.lam + (long long)p.col0 * D; g.ldb = D; g.b_off1 = p.cr;
  g.C = out.lam + (long long)out.col0 * D; g.ldc = D;
  g.alpha = 1.0f; g.accumulate = 0;
  g.nb[0] = S; g.nb[1] = H; g.nb[2] = L; g.nb[3] = 2;
  g.sA[0] = H * per; g.sA[1] = per; g.sA[2] = 0; g.sA[3] = 2LL * L * hd;
  g.sB[0] = p.s_stride * D; g.sB[1] = (long long)L * L * D; g.sB[2] = (long long)L * D; g.sB[3] = 0;
  g.sC[0] = out.s_stride * D; g.sC[1] = (long long)hd * D; g.sC[2] = (long long)out.row_stride * D; g.sC[3] = out.cr;
  {
    const int r = launch_gemm(g, st);
    if (r < 0) return r;  // unsupported shape: reported by the caller, never silently skipped
    n += r;
  }
  // y-side (V rows scaled by lx of P): batch (s, h, plane); N spans (k, d) of the head
  GemmArgs t{};
  t.M = L; t.N = hd * D; t.K = L; t.K0 = L;
  t.A = ws + 4LL * L * hd; t.lda = L;
  t.B = v.lam + (long long)v.col0 * D; t.ldb = (long long)v.row_stride * D; t.b_off1 = 0;
  t.C = out.lam + (long long)out.col0 * D; t.ldc = (long long)out.row_stride * D;
  t.alpha = 1.0f; t.accumulate = 1;
  t.nb[0] = S; t.nb[1] = H; t.nb[2] = 2; t.nb[3] = 1;
  t.sA[0] = H * per; t.sA[1] = per; t.sA[2] = (long long)L * L; t.sA[3] = 0;
  t.sB[0] = v.s_stride * D; t.sB[1] = (long long)hd * D; t.sB[2] = v.cr; t.sB[3] = 0;
  t.sC[0] = out.s_stride * D; t.sC[1] = (long long)hd * D; t.sC[2] = out.cr; t.sC[3] = 0;
  {
    const int r = launch_gemm(t, st);
    if (r < 0) return r;  // unsupported shape: reported by the caller, never silently skipped
    n += r;
  }
  return n;
}

int launch_softmax(const NView& sc, int S, int rows_per_s, int n, int D, int norm,
                   const double* eps, int* status, int site_exp, int site_recip,
                   cudaStream_t st) {
  // Shape-based choice (each measured best for its shapes): narrow rows (D 64 / 128)
  // -> softmax6, several keys per warp step; D 256 / 512 -> softmax4, streaming at full width;
  // wide rows (D > 512, multiple of 128) -> softmax5, Σ partials in SMEM; any other D that fits
  // a cluster -> softmax3 (columns split over a CTA cluster); otherwise softmax2.
  constexpr int nbuf = 1;
  if ((D == 64 || D == 128) && n % (512 / D) == 0) {  // narrow rows: G keys per warp step
    constexpr int NC6 = 4;
    const size_t smem = softmax6_smem(n, D, NC6);
    static size_t attr6[2][3] = {};
    static int grid6[2][3] = {};
    const int q = dual_norm(norm), gi = D == 64 ? 0 : 1;
    const int nrows = S * rows_per_s;
    auto launch = [&](auto kern) {
      if (attr6[gi][q] < smem) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr6[gi][q] = smem;
        int per_sm = 0, dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, (NC6 + 1) * 32, smem) != cudaSuccess ||
            per_sm < 1)
          per_sm = 1;
        grid6[gi][q] = per_sm * sms;
      }
      const int grid = nrows < grid6[gi][q] ? nrows : grid6[gi][q];
      kern<<<grid, (NC6 + 1) * 32, smem, st>>>(sc, rows_per_s, nrows, n, eps, status, site_exp, site_recip);
    };
#define SM6(QQ)                                                \
  if (D == 64) launch(softmax6_kernel<QQ, NC6, 8>);            \
  else launch(softmax6_kernel<QQ, NC6, 4>);
    if (q == NORM_L1) { SM6(NORM_L1) }
    else if (q == NORM_L2) { SM6(NORM_L2) }
    else { SM6(NORM_LINF) }
#undef SM6
    return 1;
  }
  if (D % 128 == 0 && D > 512) {  // wide rows (c5): streaming kernel, Σ partials in SMEM
    constexpr int NC5 = 2;
    // one stage per consumer warp and three CTAs per SM measured best on c5 (40 ms per pass vs 50 ms
    // with two stages per warp at two CTAs per SM, 148 ms for the cluster kernel)
    const int ns = NC5;
    const size_t smem = softmax5_smem(n, D, NC5, ns);
    if (smem <= 227 * 1024) {
      static size_t attr5[2][3] = {};
      static int grid5[2][3] = {};
      const int q = dual_norm(norm);
      const int nrows = S * rows_per_s;
      auto launch = [&](auto kern) {
        if (attr5[NC5 - 1][q] < smem) {
          cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
          attr5[NC5 - 1][q] = smem;
          int per_sm = 0, dev = 0, sms = 0;
          cudaGetDevice(&dev);
          cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
          if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, (NC5 + 1) * 32, smem) != cudaSuccess ||
              per_sm < 1)
            per_sm = 1;
          grid5[NC5 - 1][q] = per_sm * sms;
        }
        const int grid = nrows < grid5[NC5 - 1][q] ? nrows : grid5[NC5 - 1][q];
        kern<<<grid, (NC5 + 1) * 32, smem, st>>>(sc, rows_per_s, nrows, n, D, ns, eps, status, site_exp, site_recip);
      };
      if (q == NORM_L1) launch(softmax5_kernel<NORM_L1, NC5>);
      else if (q == NORM_L2) launch(softmax5_kernel<NORM_L2, NC5>);
      else launch(softmax5_kernel<NORM_LINF, NC5>);
      return 1;
    }
  }
  // streaming kernel (full D per CTA) where a key row is wide enough to amortise its per-key
  // envelope and reductions (measured: D = 512 3.3 vs 7.2 ms per c3 pass; D = 128 2.06 vs 1.98 ms
  // per c2 pass for the cluster kernel, which stays the choice there)
  if (D == 256 || D == 512) {
    const int NCsel = 4;  // 4 consumer warps, 4 CTAs per SM (8 warps measured slower)
    const size_t smem = softmax4_smem(n, D, NCsel);
    static size_t attr4[3][3][3] = {};
    static int grid4[3][3][3] = {};
    const int q = dual_norm(norm), kg = D == 128 ? 0 : (D == 256 ? 1 : 2), ci = NCsel == 4 ? 0 : 1;
    const int nrows = S * rows_per_s;
    auto launch = [&](auto kern, int threads) {
      if (attr4[ci][q][kg] < smem) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr4[ci][q][kg] = smem;
        int per_sm = 0, dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem) != cudaSuccess || per_sm < 1)
          per_sm = 1;
        grid4[ci][q][kg] = per_sm * sms;
      }
      const int grid = nrows < grid4[ci][q][kg] ? nrows : grid4[ci][q][kg];
      kern<<<grid, threads, smem, st>>>(sc, rows_per_s, nrows, n, eps, status, site_exp, site_recip);
    };
#define SM4(QQ, NCC)                                                                  \
  if (kg == 0) launch(softmax4_kernel<QQ, 1, NCC>, Sm4<NCC, 1>::kThreads);               \
  else if (kg == 1) launch(softmax4_kernel<QQ, 2, NCC>, Sm4<NCC, 2>::kThreads);          \
  else launch(softmax4_kernel<QQ, 4, NCC>, Sm4<NCC, 4>::kThreads);
    if (NCsel == 4) {
      if (q == NORM_L1) { SM4(NORM_L1, 4) }
      else if (q == NORM_L2) { SM4(NORM_L2, 4) }
      else { SM4(NORM_LINF, 4) }
    } else {
      if (q == NORM_L1) { SM4(NORM_L1, 8) }
      else if (q == NORM_L2) { SM4(NORM_L2, 8) }
      else { SM4(NORM_LINF, 8) }
    }
#undef SM4
    return 1;
  }
  const int cs = softmax3_cluster(n, D, nbuf, 64);
  if (cs > 0) {
    const size_t smem = softmax3_smem(n, D / cs, cs, nbuf);
    const int lpk = softmax3_lpk(D / cs);
    static size_t attr_set[3] = {0, 0, 0};
    const int q = dual_norm(norm);
    auto launch = [&](auto kern) {
      if (attr_set[q] < smem) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        attr_set[q] = smem;
      }
      const int nrows = S * rows_per_s;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)(nrows * cs));
      cfg.blockDim = dim3(kSm3Threads);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = cs;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, kern, sc, rows_per_s, nrows, n, D, cs, lpk, nbuf, eps, status, site_exp, site_recip);
    };
    if (q == NORM_L1) launch(softmax3_kernel<NORM_L1>);
    else if (q == NORM_L2) launch(softmax3_kernel<NORM_L2>);
    else launch(softmax3_kernel<NORM_LINF>);
    return 1;
  }
  {
    const int nw = D <= 512 ? 16 : 8;
    size_t smem = (6 * (size_t)n + 2 * (size_t)D + 40) * sizeof(double) + (size_t)nw * 2 * D * sizeof(float);
    // at most two CTAs per SM: their rows (n*D*8 bytes each) stay in L2 between phases 1 and 3
    const size_t cap = 110 * 1024;
    if (smem < cap && (size_t)n * D * 8 > 64 * 1024) smem = cap;
    if (smem > 227 * 1024) return -1;
    static size_t attr_set[3] = {0, 0, 0};
    const int q = dual_norm(norm);
    auto launch = [&](auto kern) {
      if (attr_set[q] < smem) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr_set[q] = smem;
      }
      kern<<<S * rows_per_s, nw * 32, smem, st>>>(sc, rows_per_s, n, D, eps, status, site_exp, site_recip);
    };
    if (q == NORM_L1) launch(softmax2_kernel<NORM_L1>);
    else if (q == NORM_L2) launch(softmax2_kernel<NORM_L2>);
    else launch(softmax2_kernel<NORM_LINF>);
    return 1;
  }
}

int launch_init_input(float* lam, long long cr, double* lb, double* ub, const double* x,
                      const int* positions, const int* slot_map, int S, int L, int E, int W,
                      cudaStream_t st, int D, int col0) {
  long long nrows = (long long)S * L * E;
  if (D <= 0) D = W * E;
  init_input_kernel<<<blocks_for(nrows, 8), 256, 0, st>>>(lam, cr, lb, ub, x, positions, slot_map, S,
                                                          L, E, W, D, col0);
  return 1;
}

int launch_onehot_affine(float* lam, long long cr, const float* w, const int* positions, const int* slot_map, int S,
                         int L, int E, int O, int W, int D, int col0, cudaStream_t st, int skip_o) {
  const long long nrows = (long long)S * L * O;
  onehot_affine_kernel<<<blocks_for(nrows, 8), 256, 0, st>>>(lam, cr, w, positions, slot_map, S, L, E, O, W, D,
                                                             col0, skip_o);
  return 1;
}

int launch_add_onehot(float* lam, const int* positions, const int* slot_map, int S, int L, int E, int W, int D,
                      int col0, cudaStream_t st) {
  const long long n = (long long)S * W * E;
  add_onehot_kernel<<<blocks_for(n, 256), 256, 0, st>>>(lam, positions, slot_map, S, L, E, W, D, col0);
  return 1;
}

int launch_meanpool(const float* lam, long long cr, const double* lb, const double* ub,
                    double* pc, double* pr, double* plb, double* pub, int S, int L, int E, int D,
                    cudaStream_t st) {
  if (D % 4 == 0 && getenv("FG_MEANPOOL_SCALAR") == nullptr) {  // env: comparison runs
    const int threads = D / 4 >= 128 ? 128 : (D / 4 + 31) / 32 * 32;
    dim3 grid(blocks_for(D / 4, threads), E, S);
    meanpool4_kernel<<<grid, threads, 0, st>>>(lam, cr, lb, ub, pc, pr, plb, pub, S, L, E, D);
    return 1;
  }
  dim3 grid(blocks_for(D, 128), E, S);
  meanpool_kernel<<<grid, 128, 0, st>>>(lam, cr, lb, ub, pc, pr, plb, pub, S, L, E, D);
  return 1;
}

int launch_head(const double* pc, const double* pr, const double* plb, const double* pub,
                const double* wc, const double* bc, int S, int E, int C, int D, int norm,
                const double* eps, double* out_lo, double* out_hi, int* status, int site,
                double* pooled_lo, double* pooled_hi, cudaStream_t st) {
  int q = dual_norm(norm);
  if (C <= kHeadMaxC) {
    DISPATCH_Q(q, head_all_kernel,
               <<<S, kHeadThreads, 0, st>>>(pc, pr, plb, pub, wc, bc, E, C, D, eps, out_lo, out_hi, status,
                                            site));
  } else {
    DISPATCH_Q(q, head_kernel,
               <<<S * C, 256, 0, st>>>(pc, pr, plb, pub, wc, bc, E, C, D, eps, out_lo, out_hi,
                                       status, site));
  }
  int n = 1;
  if (pooled_lo) {
    long long nrows = (long long)S * E;
    DISPATCH_Q(q, concretize_f64_kernel,
               <<<blocks_for(nrows, 8), 256, 0, st>>>(pc, pr, plb, pub, E, nrows, D, eps,
                                                       pooled_lo, pooled_hi));
    ++n;
  }
  return n;
}

int launch_ul_to_cr(const double* lw, const double* uw, float* lam, long long cr, long long n,
                    int d, int Dp, cudaStream_t st) {
  if (n <= 0) return 0;
  ul_to_cr_kernel<<<blocks_for(n * Dp, 256), 256, 0, st>>>(lw, uw, lam, cr, n, d, Dp);
  return 1;
}

int launch_cr_to_ul(const float* lam, long long cr, double* lw, double* uw, long long n, int d,
                    int Dp, cudaStream_t st) {
  if (n <= 0 || d <= 0) return 0;
  cr_to_ul_kernel<<<blocks_for(n * d, 256), 256, 0, st>>>(lam, cr, lw, uw, n, d, Dp);
  return 1;
}

int launch_add(const float* a, long long acr, const double* alb, const double* aub,
               const float* b, long long bcr, const double* blb, const double* bub, float* y,
               long long ycr, double* ylb, double* yub, long long n, int D, cudaStream_t st) {
  long long total = n * (long long)(D > 0 ? D : 1);
  if (total < n) total = n;
  add_kernel<<<blocks_for(total, 256), 256, 0, st>>>(a, acr, alb, aub, b, bcr, blb, bub, y, ycr,
                                                     ylb, yub, n, D);
  return 1;
}

int launch_scale(const float* x, long long xcr, const double* xlb, const double* xub, double s,
                 float* y, long long ycr, double* ylb, double* yub, long long n, int D,
                 cudaStream_t st) {
  long long total = n * (long long)(D > 0 ? D : 1);
  if (total < n) total = n;
  scale_kernel<<<blocks_for(total, 256), 256, 0, st>>>(x, xcr, xlb, xub, s, y, ycr, ylb, yub, n, D);
  return 1;
}

int launch_sim_coef_split(const NView& q, const NView& k, int S, int H, int L, int hd, int kp, float* x_hi,
                          float* x_lo, float* y_hi, float* y_lo, cudaStream_t st) {
  sim_coef_split_kernel<<<S * H, 256, 0, st>>>(q, k, H, L, hd, kp, x_hi, x_lo, y_hi, y_lo);
  return 1;
}

int launch_wv_coef_split(const NView& p, const NView& v, int S, int H, int L, int hd, float* x_hi,
                         float* x_lo, float* y_hi, float* y_lo, cudaStream_t st) {
  wv_coef_split_kernel<<<S * H, 256, 0, st>>>(p, v, H, L, hd, x_hi, x_lo, y_hi, y_lo);
  return 1;
}

int launch_sim_bias(const NView& q, const NView& k, const NView& out, int S, int H, int L, int hd,
                    double scale, cudaStream_t st) {
  sim_bias(q, k, out, S, H, L, hd, scale, st);
  return 1;
}

int launch_wv_bias(const NView& p, const NView& v, const NView& out, int S, int H, int L, int hd,
                   cudaStream_t st) {
  wv_bias(p, v, out, S, H, L, hd, st);
  return 1;
}

int launch_fill_int(int* p, int v, long long n, cudaStream_t st) {
  fill_int_kernel<<<blocks_for(n, 256), 256, 0, st>>>(p, v, n);
  return 1;
}

__global__ void init_status_kernel(int* status, const int* active, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) status[i] = active[i] ? kStatusClear : kStatusIdle;
}

int launch_init_status(int* status, const int* active, int n, cudaStream_t st) {
  init_status_kernel<<<(n + 255) / 256, 256, 0, st>>>(status, active, n);
  return 1;
}

// ===========================================================================
// Column-sharded pass: rank r owns perturbation columns [col0, col0 + D)
// of every Λ.  Every column-separable op is unchanged; each concretization becomes
//   local partial q-norm  ->  all-reduce across ranks (SUM; MAX for the l-inf dual)  ->  finish,
// "partial" meaning the raw accumulation before the l2 square root.  The softmax chain, which
// holds four dependent concretizations, runs as five kernels around four all-reduces.
// ===========================================================================
namespace {

// raw q-norm partials of the upper / lower rows: pu[row], pl[row] (pl = pu + nrows)
template <int Q>
__global__ void __launch_bounds__(256) partial_norm_kernel(const float* __restrict__ lam, long long cr,
                                                           long long nrows, int D, double* __restrict__ part) {
  long long row = (long long)blockIdx.x * (blockDim.x / kWarp) + threadIdx.x / kWarp;
  int lane = threadIdx.x & (kWarp - 1);
  if (row >= nrows) return;
  const float* c = lam + row * D;
  const float* r = c + cr;
  NormAcc<Q> acc;
  for (int d = lane * 4; d < D; d += 4 * kWarp)
    acc.add4(*reinterpret_cast<const float4*>(c + d), *reinterpret_cast<const float4*>(r + d));
  acc.warp_reduce();
  if (lane == 0) {
    part[row] = acc.u;
    part[nrows + row] = acc.l;
  }
}

template <int Q>
__global__ void finish_concretize_kernel(const double* __restrict__ part, const double* __restrict__ lb,
                                         const double* __restrict__ ub, long long rows_per_s, long long nrows,
                                         const double* __restrict__ eps, double* __restrict__ lo,
                                         double* __restrict__ hi) {
  long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= nrows) return;
  NormAcc<Q> fin;
  const double e = eps[row / rows_per_s];
  lo[row] = lb[row] - e * fin.fin(part[nrows + row]);
  hi[row] = ub[row] + e * fin.fin(part[row]);
}

// softmax chain, phase B: one CTA per score row (s, h, i).  Exp envelopes per key from the
// all-reduced input norms; Σ_j e_j rows (local columns, f64) and their partial norms; Σ_j e_lb,
// Σ_j e_ub.  ex: [5][nSC] a_lo, a_up, e_lb, e_ub, e_lo; sig: [rows][2][D]; p2: [2][rows];
// sb: [2][rows].
template <int Q>
__global__ void __launch_bounds__(256) sm_shard_b_kernel(NView sc, int rows_per_s, int n, int D,
                                                         const double* __restrict__ p1, long long nsc,
                                                         const double* __restrict__ eps, int* __restrict__ status,
                                                         int site_exp, double* __restrict__ ex,
                                                         double* __restrict__ sig, double* __restrict__ p2,
                                                         double* __restrict__ sb, long long nrows) {
  extern __shared__ double smb[];
  double* a_lo = smb;
  double* a_up = smb + n;
  double* red = smb + 2 * n;
  const long long rid = blockIdx.x;
  const int s = (int)(rid / rows_per_s);
  const long long nb = (long long)s * sc.s_stride + (rid % rows_per_s) * n;  // first key neuron
  const double e = eps[s];
  NormAcc<Q> fin;
  int err = 0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const long long o = nb + j;
    const double nu = fin.fin(p1[o]), nl = fin.fin(p1[nsc + o]);
    const double xlb = sc.lb[o], xub = sc.ub[o];
    Lines ln;
    const int code = envelope(RELAX_EXP, xlb - e * nl, xub + e * nu, ln);
    if (code) err = err ? min(err, code) : code;
    a_lo[j] = ln.al;
    a_up[j] = ln.au;
    const double ub2 = ln.au * (ln.au >= 0.0 ? xub : xlb) + ln.bu;
    const double lb2 = ln.al * (ln.al >= 0.0 ? xlb : xub) + ln.bl;
    ex[o] = ln.al;
    ex[nsc + o] = ln.au;
    ex[2 * nsc + o] = lb2;
    ex[3 * nsc + o] = ub2;
    ex[4 * nsc + o] = lb2 - e * fabs(ln.al) * (ln.al >= 0.0 ? nl : nu);
  }
  if (err) set_status(status, s, site_exp, err);
  __syncthreads();
  const float* cb = sc.lam + nb * D;
  const float* rb = cb + sc.cr;
  double* sg = sig + rid * 2 * D;
  double pnu = 0.0, pnl = 0.0;
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    double su = 0.0, sl = 0.0;
    for (int j = 0; j < n; ++j) {
      const double c = cb[(long long)j * D + d], r = rb[(long long)j * D + d];
      const double u = c + r, l = c - r;
      su += a_up[j] * (a_up[j] >= 0.0 ? u : l);
      sl += a_lo[j] * (a_lo[j] >= 0.0 ? l : u);
    }
    sg[d] = su;
    sg[D + d] = sl;
    pnu = qcombine<Q>(pnu, Q == NORM_L2 ? su * su : fabs(su));
    pnl = qcombine<Q>(pnl, Q == NORM_L2 ? sl * sl : fabs(sl));
  }
  pnu = block_reduce<Q>(pnu, red);
  pnl = block_reduce<Q>(pnl, red);
  if (threadIdx.x == 0) {
    p2[rid] = pnu;
    p2[nrows + rid] = pnl;
    double slb = 0.0, sub = 0.0;  // propagate_sum_axis order (relax.cpp:728-731)
    for (int j = 0; j < n; ++j) {
      slb += ex[2 * nsc + nb + j];
      sub += ex[3 * nsc + nb + j];
    }
    sb[rid] = slb;
    sb[nrows + rid] = sub;
  }
}

// phase C: RecipVerify of the all-reduced Σ norms; r rows (in place in sig) and partial norms.
// rb4: [4][rows] r_al, r_au, r_lb, r_ub.
template <int Q>
__global__ void __launch_bounds__(256) sm_shard_c_kernel(int rows_per_s, int D, const double* __restrict__ p2,
                                                         const double* __restrict__ sb, long long nrows,
                                                         const double* __restrict__ eps, int* __restrict__ status,
                                                         int site_recip, double* __restrict__ sig,
                                                         double* __restrict__ p3, double* __restrict__ rb4) {
  __shared__ double red[40];
  const long long rid = blockIdx.x;
  const int s = (int)(rid / rows_per_s);
  const double e = eps[s];
  NormAcc<Q> fin;
  if (threadIdx.x == 0) {
    const double slb = sb[rid], sub = sb[nrows + rid];
    Lines ln;
    const int code = envelope(RELAX_RECIP, slb - e * fin.fin(p2[nrows + rid]), sub + e * fin.fin(p2[rid]), ln);
    if (code) set_status(status, s, site_recip, code);
    red[32] = ln.al;
    red[33] = ln.au;
    red[34] = ln.al * (ln.al >= 0.0 ? slb : sub) + ln.bl;
    red[35] = ln.au * (ln.au >= 0.0 ? sub : slb) + ln.bu;
  }
  __syncthreads();
  const double r_al = red[32], r_au = red[33];
  if (threadIdx.x == 0) {
    rb4[rid] = r_al;
    rb4[nrows + rid] = r_au;
    rb4[2 * nrows + rid] = red[34];
    rb4[3 * nrows + rid] = red[35];
  }
  double* sg = sig + rid * 2 * D;
  double pnu = 0.0, pnl = 0.0;
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    const double u = sg[d], l = sg[D + d];
    const double yu = r_au * (r_au >= 0.0 ? u : l), yl = r_al * (r_al >= 0.0 ? l : u);
    sg[d] = yu;
    sg[D + d] = yl;
    pnu = qcombine<Q>(pnu, Q == NORM_L2 ? yu * yu : fabs(yu));
    pnl = qcombine<Q>(pnl, Q == NORM_L2 ? yl * yl : fabs(yl));
  }
  pnu = block_reduce<Q>(pnu, red);
  pnl = block_reduce<Q>(pnl, red);
  if (threadIdx.x == 0) {
    p3[rid] = pnu;
    p3[nrows + rid] = pnl;
  }
}

// phase D: McCormick e_j * r per key (warp per key), in place, with per-key partial norms
// (p4 [2][nSC]); r_lo / r_hi per row appended to rb4 rows 4, 5.
template <int Q>
__global__ void __launch_bounds__(256) sm_shard_d_kernel(NView sc, int rows_per_s, int n, int D,
                                                         const double* __restrict__ p3, long long nrows,
                                                         const double* __restrict__ eps,
                                                         const double* __restrict__ ex, long long nsc,
                                                         const double* __restrict__ sig, double* __restrict__ rb4,
                                                         double* __restrict__ p4) {
  const long long rid = blockIdx.x;
  const int s = (int)(rid / rows_per_s);
  const long long nb = (long long)s * sc.s_stride + (rid % rows_per_s) * n;
  const double e = eps[s];
  NormAcc<Q> fin;
  const double r_lo = rb4[2 * nrows + rid] - e * fin.fin(p3[nrows + rid]);
  const double r_hi = rb4[3 * nrows + rid] + e * fin.fin(p3[rid]);
  if (threadIdx.x == 0) {
    rb4[4 * nrows + rid] = r_lo;
    rb4[5 * nrows + rid] = r_hi;
  }
  const double* sg = sig + rid * 2 * D;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = warp; j < n; j += nw) {
    const long long o = nb + j;
    float* c = sc.lam + o * D;
    float* r = c + sc.cr;
    const double al = ex[o], au = ex[nsc + o], lx = ex[4 * nsc + o], ly = r_lo, uy = r_hi;
    double gu = 0.0, gl = 0.0;
    for (int d = lane; d < D; d += 32) {
      const double cv = c[d], rv = r[d];
      const double u = cv + rv, l = cv - rv;
      const double eu = au * (au >= 0.0 ? u : l), el = al * (al >= 0.0 ? l : u);
      const double yu = sg[d], yl = sg[D + d];
      double p_l = 0.0, p_u = 0.0;
      if (ly != 0.0) p_l += ly * (ly >= 0.0 ? el : eu);  // relax.cpp:542-553
      if (lx != 0.0) p_l += lx * (lx >= 0.0 ? yl : yu);
      if (uy != 0.0) p_u += uy * (uy >= 0.0 ? eu : el);  // relax.cpp:556-567
      if (lx != 0.0) p_u += lx * (lx >= 0.0 ? yu : yl);
      c[d] = (float)(0.5 * (p_u + p_l));
      r[d] = (float)(0.5 * (p_u - p_l));
      gu = qcombine<Q>(gu, Q == NORM_L2 ? p_u * p_u : fabs(p_u));
      gl = qcombine<Q>(gl, Q == NORM_L2 ? p_l * p_l : fabs(p_l));
    }
    if (Q == NORM_LINF) { gu = warp_max(gu); gl = warp_max(gl); }
    else { gu = warp_sum(gu); gl = warp_sum(gl); }
    if (lane == 0) {
      p4[o] = gu;
      p4[nsc + o] = gl;
    }
  }
}

// phase E: probs lb/ub (term_bias) and lo/hi per key from the all-reduced output norms.
template <int Q>
__global__ void sm_shard_e_kernel(NView sc, int rows_per_s, int n, long long nrows_total,
                                  const double* __restrict__ ex, long long nsc, const double* __restrict__ rb4,
                                  long long nrows, const double* __restrict__ p4, const double* __restrict__ eps) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nrows_total * n) return;
  const long long rid = t / n;
  const int j = (int)(t % n);
  const int s = (int)(rid / rows_per_s);
  const long long o = (long long)s * sc.s_stride + (rid % rows_per_s) * n + j;
  double olb = 0.0, oub = 0.0;
  term_bias(ex[4 * nsc + o], rb4[4 * nrows + rid], rb4[5 * nrows + rid], ex[2 * nsc + o], ex[3 * nsc + o],
            rb4[2 * nrows + rid], rb4[3 * nrows + rid], olb, oub);
  sc.lb[o] = olb;
  sc.ub[o] = oub;
  if (sc.lo) {
    NormAcc<Q> fin;
    const double e = eps[s];
    sc.lo[o] = olb - e * fin.fin(p4[nsc + o]);
    sc.hi[o] = oub + e * fin.fin(p4[o]);
  }
}

// classifier head, partial: logits Λ over the local columns, raw norms + f64 biases.
// part: [2][S*C] (u, l raw partials; +inf when a local element is non-finite); bias: [2][S*C]
template <int Q>
__global__ void head_partial_kernel(const double* pc, const double* pr, const double* plb, const double* pub,
                                    const double* wc, const double* bc, int S, int E, int C, int D, double* part,
                                    double* bias) {
  __shared__ double red[32];
  const int s = blockIdx.x / C, cls = blockIdx.x % C;
  double nu = 0.0, nl = 0.0;
  int finite = 1;
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    double ac = 0.0, ar = 0.0;
    for (int e = 0; e < E; ++e) {
      const double w = wc[e * C + cls];
      ac += w * pc[((long long)s * E + e) * D + d];
      ar += fabs(w) * pr[((long long)s * E + e) * D + d];
    }
    const double u = ac + ar, l = ac - ar;
    finite &= (isfinite(u) && isfinite(l));
    nu = qcombine<Q>(nu, Q == NORM_L2 ? u * u : fabs(u));
    nl = qcombine<Q>(nl, Q == NORM_L2 ? l * l : fabs(l));
  }
  finite = __syncthreads_and(finite);
  nu = block_reduce<Q>(nu, red);
  nl = block_reduce<Q>(nl, red);
  if (threadIdx.x == 0) {
    double ub_pos = 0.0, ub_neg = 0.0, lb_pos = 0.0, lb_neg = 0.0;  // relax.cpp:280-299
    for (int i = 0; i < E; ++i) {
      const double wv = wc[i * C + cls];
      const double wp = (wv < 0.0) ? 0.0 : wv, wn = (0.0 < wv) ? 0.0 : wv;
      const double xu = pub[(long long)s * E + i], xl = plb[(long long)s * E + i];
      ub_pos += wp * xu;
      ub_neg += wn * xl;
      lb_pos += wp * xl;
      lb_neg += wn * xu;
    }
    const int k = s * C + cls, SC = S * C;
    part[k] = finite ? nu : HUGE_VAL;
    part[SC + k] = finite ? nl : HUGE_VAL;
    bias[k] = ub_pos + ub_neg + bc[cls];
    bias[SC + k] = lb_pos + lb_neg + bc[cls];
  }
}

template <int Q>
__global__ void head_finish_kernel(const double* part, const double* bias, int S, int C, const double* eps,
                                   double* out_lo, double* out_hi, int* status, int site) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= S * C) return;
  const int s = k / C, SC = S * C;
  const double yub = bias[k], ylb = bias[SC + k], nu = part[k], nl = part[SC + k];
  if (!isfinite(yub) || !isfinite(ylb) || !isfinite(nu) || !isfinite(nl))  // graph.cpp:663-671
    set_status(status, s, site, kCodeDomain);
  NormAcc<Q> fin;
  const double e = eps[s];
  out_lo[k] = ylb - e * fin.fin(nl);
  out_hi[k] = yub + e * fin.fin(nu);
}

}  // namespace

int launch_partial_norms(const float* lam, long long cr, long long nrows, int D, int norm, double* part,
                         cudaStream_t st) {
  if (nrows <= 0) return 0;
  DISPATCH_Q(dual_norm(norm), partial_norm_kernel, <<<blocks_for(nrows, 8), 256, 0, st>>>(lam, cr, nrows, D, part));
  return 1;
}

int launch_finish_concretize(const double* part, const double* lb, const double* ub, long long rows_per_s,
                             long long nrows, int norm, const double* eps, double* lo, double* hi, cudaStream_t st) {
  if (nrows <= 0) return 0;
  DISPATCH_Q(dual_norm(norm), finish_concretize_kernel,
             <<<blocks_for(nrows, 256), 256, 0, st>>>(part, lb, ub, rows_per_s, nrows, eps, lo, hi));
  return 1;
}

int reduce_op_for_norm(int norm) { return dual_norm(norm) == NORM_LINF ? 1 : 0; }  // 0 SUM, 1 MAX

int launch_sm_shard(int phase, const NView& sc, int S, int rows_per_s, int n, int D, int norm, const double* eps,
                    int* status, int site_exp, int site_recip, SmShardBufs b, cudaStream_t st) {
  const long long nrows = (long long)S * rows_per_s, nsc = nrows * n;
  const int q = dual_norm(norm);
  switch (phase) {
    case 0:  // exp-input partial norms per key
      return launch_partial_norms(sc.lam, sc.cr, nsc, D, norm, b.p_key, st);
    case 1:
      DISPATCH_Q(q, sm_shard_b_kernel, <<<(unsigned)nrows, 256, (2 * n + 32) * sizeof(double), st>>>(
          sc, rows_per_s, n, D, b.p_key, nsc, eps, status, site_exp, b.ex, b.sig, b.p_row, b.sb, nrows));
      return 1;
    case 2:
      DISPATCH_Q(q, sm_shard_c_kernel, <<<(unsigned)nrows, 256, 0, st>>>(
          rows_per_s, D, b.p_row, b.sb, nrows, eps, status, site_recip, b.sig, b.p_row2, b.rb));
      return 1;
    case 3:
      DISPATCH_Q(q, sm_shard_d_kernel, <<<(unsigned)nrows, 256, 0, st>>>(
          sc, rows_per_s, n, D, b.p_row2, nrows, eps, b.ex, nsc, b.sig, b.rb, b.p_key));
      return 1;
    default:
      DISPATCH_Q(q, sm_shard_e_kernel, <<<blocks_for(nsc, 256), 256, 0, st>>>(
          sc, rows_per_s, n, nrows, b.ex, nsc, b.rb, nrows, b.p_key, eps));
      return 1;
  }
}

int launch_head_partial(const double* pc, const double* pr, const double* plb, const double* pub, const double* wc,
                        const double* bc, int S, int E, int C, int D, int norm, double* part, double* bias,
                        cudaStream_t st) {
  DISPATCH_Q(dual_norm(norm), head_partial_kernel,
             <<<S * C, 256, 0, st>>>(pc, pr, plb, pub, wc, bc, S, E, C, D, part, bias));
  return 1;
}

int launch_head_finish(const double* part, const double* bias, int S, int C, int norm, const double* eps,
                       double* out_lo, double* out_hi, int* status, int site, cudaStream_t st) {
  DISPATCH_Q(dual_norm(norm), head_finish_kernel,
             <<<blocks_for((long long)S * C, 128), 128, 0, st>>>(part, bias, S, C, eps, out_lo, out_hi, status, site));
  return 1;
}

}  // namespace fg
