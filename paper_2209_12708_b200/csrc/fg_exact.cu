// fg_exact.cu -- f64 operator kernels of the exact precision mode (FG_PRECISION_F64).
//
// The operator-level C ABI (fg_affine, fg_concretize, fg_compose, fg_dot, ...) runs these
// when a context is switched to FG_PRECISION_F64: bounds stay in the reference layout
// (lw/uw [n, d] row-major f64, lb/ub [n] f64) and every output element is produced by one
// thread that walks the reduction in the reference's order with separate multiplies and
// adds (this file is compiled with -fmad=false).  The arithmetic operators are therefore
// bit-identical to proj/src/relax.cpp and proj/src/bounds.cpp; the transcendental envelopes
// (exp/tanh, fg_kernels.cu) agree to the last ulp or two of the device libm.
// This is the path the C++ drop-in layer (paper_2209_12708_b200/compat) uses by default,
// so the reference's own graph::evaluate / cmd_verify / cmd_maxeps and its acceptance
// suite run unchanged on the GPU.  The fused batched pass stays f32 Λ + f64 O(N) state.
#include <math.h>

#include "fg_internal.cuh"

namespace fg {

namespace {

constexpr int kXThreads = 128;

// std::max(v, 0.0) / std::min(v, 0.0) exactly (signed zeros included).
__device__ __forceinline__ double pos_part(double v) { return (v < 0.0) ? 0.0 : v; }
__device__ __forceinline__ double neg_part(double v) { return (0.0 < v) ? 0.0 : v; }

// propagate_affine Λ rows (relax.cpp:268-303): thread = (row r, output j, column k).
__global__ void x_affine_lam_kernel(const double* __restrict__ xlw, const double* __restrict__ xuw,
                                    const double* __restrict__ w, double* __restrict__ ylw,
                                    double* __restrict__ yuw, long long rows, int c, int o, int d) {
  const int kb = d > 0 ? (d + kXThreads - 1) / kXThreads : 1;
  const long long blk = blockIdx.x;
  const long long rj = blk / kb;
  const int k = (int)(blk % kb) * kXThreads + threadIdx.x;
  if (rj >= rows * o || k >= d) return;
  const long long r = rj / o;
  const int j = (int)(rj % o);
  double yu = 0.0, un = 0.0, yl = 0.0, ln = 0.0;
  for (int i = 0; i < c; ++i) {
    const double wv = w[(long long)i * o + j];
    const double wp = pos_part(wv), wn = neg_part(wv);
    const double xu = xuw[((r * c + i) * d) + k], xl = xlw[((r * c + i) * d) + k];
    yu += wp * xu;
    un += wn * xl;
    yl += wp * xl;
    ln += wn * xu;
  }
  yuw[rj * d + k] = yu + un;
  ylw[rj * d + k] = yl + ln;
}

// The same Λ rows, JT outputs per thread: thread = (row r, outputs j0..j0+JT-1, column k).
// Every output still accumulates its four partial sums over i = 0..c-1 in order, so the
// result is bit-identical to x_affine_lam_kernel; the block stages kIC input rows of both Λ
// planes (its 128 columns) and the matching kIC x JT weights in shared memory per step, so
// the loads are issued together and each x value feeds JT outputs (the one-output kernel
// re-reads each Λ row from L2 once per output).  Terms with w == 0 are skipped: both of their
// products are signed zeros, and adding a signed zero never changes a partial sum here (a sum
// that starts at +0.0 can never become -0.0 in round-to-nearest), so skipping them is exact.
// The sign tests read shared memory and are warp-uniform (all threads share j).
constexpr int kIC = 16;
template <int JT>
__global__ void __launch_bounds__(kXThreads) x_affine_lam_tiled_kernel(
    const double* __restrict__ xlw, const double* __restrict__ xuw, const double* __restrict__ w,
    double* __restrict__ ylw, double* __restrict__ yuw, long long rows, int c, int o, int d) {
  __shared__ double su[kIC][kXThreads], sl[kIC][kXThreads], sw[kIC][JT];
  // per staged input row: bit t = (w_t > 0), bit 8 + t = (w_t < 0), so the inner loop branches on
  // integer bits instead of two f64 compares per weight on the FP64 pipe (NaN / ±0: neither bit)
  __shared__ uint32_t sgn[kIC];
  static_assert(JT <= 8, "sign mask holds 8 weights per row");
  const int kb = (d + kXThreads - 1) / kXThreads;
  const int jtiles = o / JT;
  const long long blk = blockIdx.x;
  const int kc = (int)(blk % kb);
  const long long rjt = blk / kb;
  const int jt = (int)(rjt % jtiles);
  const long long r = rjt / jtiles;
  const int k = kc * kXThreads + threadIdx.x;
  if (r >= rows) return;
  const bool live = k < d;
  const int j0 = jt * JT;
  double yu[JT], un[JT], yl[JT], ln[JT];
#pragma unroll
  for (int t = 0; t < JT; ++t) yu[t] = un[t] = yl[t] = ln[t] = 0.0;
  const double* xu_p = xuw + r * c * (long long)d + k;
  const double* xl_p = xlw + r * c * (long long)d + k;
  for (int i0 = 0; i0 < c; i0 += kIC) {
    const int ni = min(kIC, c - i0);
    __syncthreads();
#pragma unroll
    for (int ii = 0; ii < kIC; ++ii) {
      const bool in = live && ii < ni;
      su[ii][threadIdx.x] = in ? xu_p[(long long)(i0 + ii) * d] : 0.0;
      sl[ii][threadIdx.x] = in ? xl_p[(long long)(i0 + ii) * d] : 0.0;
    }
    for (int e = threadIdx.x; e < kIC * JT; e += kXThreads) {
      const int ii = e / JT, t = e % JT;
      sw[ii][t] = ii < ni ? w[(long long)(i0 + ii) * o + j0 + t] : 0.0;
    }
    __syncthreads();
    if (threadIdx.x < kIC) {
      uint32_t m = 0;
#pragma unroll
      for (int t = 0; t < JT; ++t) {
        const double v = sw[threadIdx.x][t];
        m |= (v > 0.0 ? 1u : 0u) << t;
        m |= (v < 0.0 ? 1u : 0u) << (8 + t);
      }
      sgn[threadIdx.x] = m;
    }
    __syncthreads();
    for (int ii = 0; ii < ni; ++ii) {
      const double xu = su[ii][threadIdx.x], xl = sl[ii][threadIdx.x];
      const uint32_t m = sgn[ii];
      double wv[JT];
#pragma unroll
      for (int t = 0; t < JT; ++t) wv[t] = sw[ii][t];
#pragma unroll
      for (int t = 0; t < JT; ++t) {
        if ((m >> t) & 1u) {  // w > 0: wp = w, wn = 0
          yu[t] += wv[t] * xu;
          yl[t] += wv[t] * xl;
        } else if ((m >> (8 + t)) & 1u) {  // w < 0: wp = 0, wn = w
          un[t] += wv[t] * xl;
          ln[t] += wv[t] * xu;
        }
      }
    }
  }
  if (!live) return;
#pragma unroll
  for (int t = 0; t < JT; ++t) {
    const long long rj = r * o + j0 + t;
    yuw[rj * d + k] = yu[t] + un[t];
    ylw[rj * d + k] = yl[t] + ln[t];
  }
}

// propagate_affine biases: y_ub = (ub_pos + ub_neg) + b, y_lb likewise.
__global__ void x_affine_bias_kernel(const double* __restrict__ xlb, const double* __restrict__ xub,
                                     const double* __restrict__ w, const double* __restrict__ bias,
                                     double* __restrict__ ylb, double* __restrict__ yub, long long rows, int c,
                                     int o) {
  const long long rj = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (rj >= rows * o) return;
  const long long r = rj / o;
  const int j = (int)(rj % o);
  double up = 0.0, un = 0.0, lp = 0.0, ln = 0.0;
  for (int i = 0; i < c; ++i) {
    const double wv = w[(long long)i * o + j];
    const double wp = pos_part(wv), wn = neg_part(wv);
    up += wp * xub[r * c + i];
    un += wn * xlb[r * c + i];
    lp += wp * xlb[r * c + i];
    ln += wn * xub[r * c + i];
  }
  const double bv = bias ? bias[j] : 0.0;
  yub[rj] = up + un + bv;
  ylb[rj] = lp + ln + bv;
}

// concretize / row_norm (bounds.cpp:80-140): thread per neuron, sequential over d.
__global__ void x_concretize_kernel(const double* __restrict__ lw, const double* __restrict__ lb,
                                    const double* __restrict__ uw, const double* __restrict__ ub,
                                    long long n, int d, int q, double eps, double* __restrict__ lo,
                                    double* __restrict__ hi) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* l = lw + i * d;
  const double* u = uw + i * d;
  double sl = 0.0, su = 0.0;
  if (q == NORM_L1) {
    for (int k = 0; k < d; ++k) sl += fabs(l[k]);
    for (int k = 0; k < d; ++k) su += fabs(u[k]);
  } else if (q == NORM_L2) {
    for (int k = 0; k < d; ++k) sl += l[k] * l[k];
    for (int k = 0; k < d; ++k) su += u[k] * u[k];
    sl = sqrt(sl);
    su = sqrt(su);
  } else {
    for (int k = 0; k < d; ++k) {
      const double a = fabs(l[k]);
      sl = (sl < a) ? a : sl;  // std::max(m, |v|)
    }
    for (int k = 0; k < d; ++k) {
      const double a = fabs(u[k]);
      su = (su < a) ? a : su;
    }
  }
  lo[i] = lb[i] - eps * sl;
  hi[i] = ub[i] + eps * su;
}

// The same reduction with coalesced loads: a block of kXThreads neurons stages its rows
// kCC columns at a time through shared memory (each warp loads whole column chunks of
// consecutive rows), then every thread continues its own row's sum in order k = 0..d-1.
constexpr int kCC = 16;
__global__ void __launch_bounds__(kXThreads) x_concretize_staged_kernel(
    const double* __restrict__ lw, const double* __restrict__ lb, const double* __restrict__ uw,
    const double* __restrict__ ub, long long n, int d, int q, double eps, double* __restrict__ lo,
    double* __restrict__ hi) {
  __shared__ double tl[kXThreads][kCC + 1], tu[kXThreads][kCC + 1];
  const long long i0 = (long long)blockIdx.x * kXThreads;
  const long long i = i0 + threadIdx.x;
  double sl = 0.0, su = 0.0;
  for (int k0 = 0; k0 < d; k0 += kCC) {
    const int kw = min(kCC, d - k0);
    for (int e = threadIdx.x; e < kXThreads * kCC; e += kXThreads) {
      const int rr = e / kCC, cc = e % kCC;
      const long long row = i0 + rr;
      const bool in = row < n && cc < kw;
      tl[rr][cc] = in ? lw[row * d + k0 + cc] : 0.0;
      tu[rr][cc] = in ? uw[row * d + k0 + cc] : 0.0;
    }
    __syncthreads();
    if (q == NORM_L1) {
      for (int cc = 0; cc < kw; ++cc) sl += fabs(tl[threadIdx.x][cc]);
      for (int cc = 0; cc < kw; ++cc) su += fabs(tu[threadIdx.x][cc]);
    } else if (q == NORM_L2) {
      for (int cc = 0; cc < kw; ++cc) sl += tl[threadIdx.x][cc] * tl[threadIdx.x][cc];
      for (int cc = 0; cc < kw; ++cc) su += tu[threadIdx.x][cc] * tu[threadIdx.x][cc];
    } else {
      for (int cc = 0; cc < kw; ++cc) {
        const double a = fabs(tl[threadIdx.x][cc]);
        sl = (sl < a) ? a : sl;
      }
      for (int cc = 0; cc < kw; ++cc) {
        const double a = fabs(tu[threadIdx.x][cc]);
        su = (su < a) ? a : su;
      }
    }
    __syncthreads();
  }
  if (i >= n) return;
  if (q == NORM_L2) {
    sl = sqrt(sl);
    su = sqrt(su);
  }
  lo[i] = lb[i] - eps * sl;
  hi[i] = ub[i] + eps * su;
}

// compose_elementwise (relax.cpp:470-497): thread = (neuron i, column k); k == 0 does biases.
__global__ void x_compose_kernel(const double* __restrict__ xlw, const double* __restrict__ xlb,
                                 const double* __restrict__ xuw, const double* __restrict__ xub,
                                 const double* __restrict__ a_low, const double* __restrict__ b_low,
                                 const double* __restrict__ a_up, const double* __restrict__ b_up,
                                 double* __restrict__ ylw, double* __restrict__ ylb, double* __restrict__ yuw,
                                 double* __restrict__ yub, long long n, int d) {
  const int kb = d > 0 ? (d + kXThreads - 1) / kXThreads : 1;
  const long long i = blockIdx.x / kb;
  const int k = (int)(blockIdx.x % kb) * kXThreads + threadIdx.x;
  if (i >= n) return;
  const double au = a_up[i], al = a_low[i];
  if (k == 0) {
    yub[i] = au * ((au >= 0.0) ? xub[i] : xlb[i]) + b_up[i];
    ylb[i] = al * ((al >= 0.0) ? xlb[i] : xub[i]) + b_low[i];
  }
  if (k < d) {
    yuw[i * d + k] = au * ((au >= 0.0) ? xuw[i * d + k] : xlw[i * d + k]);
    ylw[i * d + k] = al * ((al >= 0.0) ? xlw[i * d + k] : xuw[i * d + k]);
  }
}

// One McCormick-bounded product term (accumulate_product_term, relax.cpp:533-569) for column
// k (k < 0: biases only).  lx = ca.lo[xi], ly = cb.lo[yi], uy = cb.hi[yi].
__device__ __forceinline__ void x_term(const double* alw, const double* alb, const double* auw,
                                       const double* aub, const double* blw, const double* blb,
                                       const double* buw, const double* bub, long long xi, long long yi,
                                       double lx, double ly, double uy, int d, int k, bool bias,
                                       double& olb, double& oub, double& olw, double& ouw) {
  {  // lower plane: z >= ly*x + lx*y - lx*ly
    const double cx = ly, cy = lx;
    if (bias)
      olb += cx * ((cx >= 0.0) ? alb[xi] : aub[xi]) + cy * ((cy >= 0.0) ? blb[yi] : bub[yi]) - lx * ly;
    if (k >= 0) {
      if (cx != 0.0) olw += cx * ((cx >= 0.0) ? alw[xi * d + k] : auw[xi * d + k]);
      if (cy != 0.0) olw += cy * ((cy >= 0.0) ? blw[yi * d + k] : buw[yi * d + k]);
    }
  }
  {  // upper plane: z <= uy*x + lx*y - lx*uy
    const double cx = uy, cy = lx;
    if (bias)
      oub += cx * ((cx >= 0.0) ? aub[xi] : alb[xi]) + cy * ((cy >= 0.0) ? bub[yi] : blb[yi]) - lx * uy;
    if (k >= 0) {
      if (cx != 0.0) ouw += cx * ((cx >= 0.0) ? auw[xi * d + k] : alw[xi * d + k]);
      if (cy != 0.0) ouw += cy * ((cy >= 0.0) ? buw[yi * d + k] : blw[yi * d + k]);
    }
  }
}

struct XOps {  // device pointers of two operands, their concretizations and the output
  const double *alw, *alb, *auw, *aub, *alo;
  const double *blw, *blb, *buw, *bub, *blo, *bhi;
  double *ylw, *ylb, *yuw, *yub;
};

// propagate_dot_product (relax.cpp:573-654), batch b: thread = (output neuron, column k).
// Λ part of one McCormick term (x_term's row additions) with the operand rows already loaded:
// the same additions in the same order, with the "skip when the coefficient is 0" of
// relax.cpp:545-566 as a select, so all loads can be issued before any coefficient is known.
__device__ __forceinline__ void x_term_rows(double lx, double ly, double uy, double xl, double xu, double yl,
                                            double yu, double& olw, double& ouw) {
  const double a = ly * ((ly >= 0.0) ? xl : xu);  // lower plane: cx = ly, cy = lx
  olw = (ly != 0.0) ? olw + a : olw;
  const double b = lx * ((lx >= 0.0) ? yl : yu);
  olw = (lx != 0.0) ? olw + b : olw;
  const double c = uy * ((uy >= 0.0) ? xu : xl);  // upper plane: cx = uy, cy = lx
  ouw = (uy != 0.0) ? ouw + c : ouw;
  const double e = lx * ((lx >= 0.0) ? yu : yl);
  ouw = (lx != 0.0) ? ouw + e : ouw;
}

// propagate_dot_product (relax.cpp:573-654): thread = (output neuron, column k); the k == 0
// thread of each output also accumulates the biases (in a second loop: same per-output order).
// Both candidate rows of every operand are loaded unconditionally and the term loop is unrolled,
// so the row loads of several terms are in flight together.
__global__ void x_dot_kernel(XOps p, int layout, long long batch, int len, int e, int heads, int d) {
  const int kb = d > 0 ? (d + kXThreads - 1) / kXThreads : 1;
  const long long oidx = blockIdx.x / kb;
  const int kk = (int)(blockIdx.x % kb) * kXThreads + threadIdx.x;
  const int hd = e / heads;
  const bool sim = layout == 0;
  const long long nout = sim ? batch * heads * len * len : batch * len * e;
  if (oidx >= nout) return;
  const bool bias = kk == 0;
  const int k = kk < d ? kk : -1;
  if (k < 0 && !bias) return;
  // term t: x row xi0 + t*xs, y row yi0 + t*ys
  long long xi0, yi0, xs, ys;
  int nt;
  if (sim) {  // scores[b, h, i, j] = sum_t q[b, i, h*hd + t] k[b, j, h*hd + t]
    const int j = (int)(oidx % len);
    const int i = (int)((oidx / len) % len);
    const int h = (int)((oidx / ((long long)len * len)) % heads);
    const long long bi = oidx / ((long long)heads * len * len);
    xi0 = (bi * len + i) * e + (long long)h * hd;
    yi0 = (bi * len + j) * e + (long long)h * hd;
    xs = ys = 1;
    nt = hd;
  } else {  // ctx[b, i, h*hd + t] = sum_j s[b, h, i, j] v[b, j, h*hd + t]
    const int f = (int)(oidx % e);
    const int i = (int)((oidx / e) % len);
    const long long bi = oidx / ((long long)len * e);
    const int h = f / hd;
    xi0 = ((bi * heads + h) * len + i) * len;
    yi0 = (bi * len) * e + f;
    xs = 1;
    ys = e;
    nt = len;
  }
  if (k >= 0) {
    double olw = 0.0, ouw = 0.0;
#pragma unroll 4
    for (int t = 0; t < nt; ++t) {
      const long long xi = xi0 + t * xs, yi = yi0 + t * ys;
      x_term_rows(p.alo[xi], p.blo[yi], p.bhi[yi], p.alw[xi * d + k], p.auw[xi * d + k], p.blw[yi * d + k],
                  p.buw[yi * d + k], olw, ouw);
    }
    p.ylw[oidx * d + k] = olw;
    p.yuw[oidx * d + k] = ouw;
  }
  if (bias) {
    double olb = 0.0, oub = 0.0, dl = 0.0, du = 0.0;
    for (int t = 0; t < nt; ++t) {
      const long long xi = xi0 + t * xs, yi = yi0 + t * ys;
      x_term(p.alw, p.alb, p.auw, p.aub, p.blw, p.blb, p.buw, p.bub, xi, yi, p.alo[xi], p.blo[yi], p.bhi[yi], d,
             -1, true, olb, oub, dl, du);
    }
    p.ylb[oidx] = olb;
    p.yub[oidx] = oub;
  }
}

// propagate_mul_broadcast (relax.cpp:744-775): x [outer, n, inner], r [outer, 1, inner].
__global__ void x_mul_broadcast_kernel(XOps p, long long outer, int n, long long inner, int d) {
  const int kb = d > 0 ? (d + kXThreads - 1) / kXThreads : 1;
  const long long idx = blockIdx.x / kb;
  const int kk = (int)(blockIdx.x % kb) * kXThreads + threadIdx.x;
  if (idx >= outer * n * inner) return;
  const bool bias = kk == 0;
  const int k = kk < d ? kk : -1;
  if (k < 0 && !bias) return;
  const long long ii = idx % inner;
  const long long oi = idx / ((long long)n * inner);
  const long long ridx = oi * inner + ii;
  double olb = 0.0, oub = 0.0, olw = 0.0, ouw = 0.0;
  x_term(p.alw, p.alb, p.auw, p.aub, p.blw, p.blb, p.buw, p.bub, idx, ridx, p.alo[idx], p.blo[ridx],
         p.bhi[ridx], d, k, bias, olb, oub, olw, ouw);
  if (bias) {
    p.ylb[idx] = olb;
    p.yub[idx] = oub;
  }
  if (k >= 0) {
    p.ylw[idx * d + k] = olw;
    p.yuw[idx * d + k] = ouw;
  }
}

// propagate_sum_axis (relax.cpp:705-742): x [outer, n, inner] -> y [outer, 1, inner].
__global__ void x_sum_axis_kernel(const double* __restrict__ xlw, const double* __restrict__ xlb,
                                  const double* __restrict__ xuw, const double* __restrict__ xub,
                                  double* __restrict__ ylw, double* __restrict__ ylb, double* __restrict__ yuw,
                                  double* __restrict__ yub, long long outer, int n, long long inner, int d) {
  const int kb = d > 0 ? (d + kXThreads - 1) / kXThreads : 1;
  const long long oidx = blockIdx.x / kb;
  const int k = (int)(blockIdx.x % kb) * kXThreads + threadIdx.x;
  if (oidx >= outer * inner) return;
  const long long oi = oidx / inner, ii = oidx % inner;
  if (k == 0) {
    double l = 0.0, u = 0.0;
    for (int j = 0; j < n; ++j) {
      const long long idx = (oi * n + j) * inner + ii;
      l += xlb[idx];
      u += xub[idx];
    }
    ylb[oidx] = l;
    yub[oidx] = u;
  }
  if (k < d) {
    double l = 0.0, u = 0.0;
    for (int j = 0; j < n; ++j) {
      const long long idx = (oi * n + j) * inner + ii;
      l += xlw[idx * d + k];
      u += xuw[idx * d + k];
    }
    ylw[oidx * d + k] = l;
    yuw[oidx * d + k] = u;
  }
}

// propagate_add / propagate_scale (relax.cpp:656-703), flat over lw (and lb) elements.
__global__ void x_add_kernel(const double* a, const double* b, double* y, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = a[i] + b[i];
}
__global__ void x_scale_kernel(const double* xl, const double* xu, double s, double* yl, double* yu,
                               long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (s >= 0.0) {
    yl[i] = s * xl[i];
    yu[i] = s * xu[i];
  } else {
    yl[i] = s * xu[i];
    yu[i] = s * xl[i];
  }
}

// relax_bilinear (relax.cpp:499-523) with ConcreteBounds::validate of both operands.
__global__ void x_bilinear_kernel(const double* xlo, const double* xhi, const double* ylo, const double* yhi,
                                  double* lo_x, double* lo_y, double* lo_c, double* up_x, double* up_y,
                                  double* up_c, long long n, int* status) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (xlo[i] > xhi[i] || ylo[i] > yhi[i]) atomicMin(status, kCodeInval);
  const double lx = xlo[i], ly = ylo[i], uy = yhi[i];
  lo_x[i] = ly;
  lo_y[i] = lx;
  lo_c[i] = -lx * ly;
  up_x[i] = uy;
  up_y[i] = lx;
  up_c[i] = -lx * uy;
}

inline unsigned blocks_for(long long n, int t) { return (unsigned)((n + t - 1) / t); }
inline unsigned row_blocks(long long rows, int d) {
  const long long kb = (d + kXThreads - 1) / kXThreads;
  return (unsigned)(rows * (kb > 0 ? kb : 1));
}

}  // namespace

int launch_x_affine(const double* xlw, const double* xlb, const double* xuw, const double* xub, const double* w,
                    const double* bias, double* ylw, double* ylb, double* yuw, double* yub, long long rows, int c,
                    int o, int d, cudaStream_t st) {
  int n = 0;
  if (rows * o <= 0) return 0;
  if (d > 0) {
    if (o % 8 == 0)
      x_affine_lam_tiled_kernel<8><<<row_blocks(rows * (o / 8), d), kXThreads, 0, st>>>(xlw, xuw, w, ylw, yuw, rows,
                                                                                         c, o, d);
    else
      x_affine_lam_kernel<<<row_blocks(rows * o, d), kXThreads, 0, st>>>(xlw, xuw, w, ylw, yuw, rows, c, o, d);
    ++n;
  }
  x_affine_bias_kernel<<<blocks_for(rows * o, 128), 128, 0, st>>>(xlb, xub, w, bias, ylb, yub, rows, c, o);
  return n + 1;
}

int launch_x_concretize(const double* lw, const double* lb, const double* uw, const double* ub, long long n,
                        int d, int norm, double eps, double* lo, double* hi, cudaStream_t st) {
  const int q = norm == NORM_L1 ? NORM_LINF : (norm == NORM_L2 ? NORM_L2 : NORM_L1);  // dual (bounds.cpp:9-19)
  if (n <= 0) return 0;
  if (d >= kCC)
    x_concretize_staged_kernel<<<blocks_for(n, kXThreads), kXThreads, 0, st>>>(lw, lb, uw, ub, n, d, q, eps, lo, hi);
  else
    x_concretize_kernel<<<blocks_for(n, 128), 128, 0, st>>>(lw, lb, uw, ub, n, d, q, eps, lo, hi);
  return 1;
}

int launch_x_compose(const double* xlw, const double* xlb, const double* xuw, const double* xub,
                     const double* a_low, const double* b_low, const double* a_up, const double* b_up, double* ylw,
                     double* ylb, double* yuw, double* yub, long long n, int d, cudaStream_t st) {
  if (n <= 0) return 0;
  x_compose_kernel<<<row_blocks(n, d), kXThreads, 0, st>>>(xlw, xlb, xuw, xub, a_low, b_low, a_up, b_up, ylw, ylb,
                                                          yuw, yub, n, d);
  return 1;
}

int launch_x_dot(const XDotArgs& a, cudaStream_t st) {
  XOps p{a.alw, a.alb, a.auw, a.aub, a.alo, a.blw, a.blb, a.buw, a.bub, a.blo, a.bhi, a.ylw, a.ylb, a.yuw, a.yub};
  const long long nout = a.layout == 0 ? a.batch * a.heads * a.len * (long long)a.len
                                       : a.batch * a.len * (long long)a.e;
  if (nout <= 0) return 0;
  x_dot_kernel<<<row_blocks(nout, a.d), kXThreads, 0, st>>>(p, a.layout, a.batch, a.len, a.e, a.heads, a.d);
  return 1;
}

int launch_x_mul_broadcast(const XDotArgs& a, long long outer, int n, long long inner, cudaStream_t st) {
  if (outer * n * inner <= 0) return 0;
  XOps p{a.alw, a.alb, a.auw, a.aub, a.alo, a.blw, a.blb, a.buw, a.bub, a.blo, a.bhi, a.ylw, a.ylb, a.yuw, a.yub};
  x_mul_broadcast_kernel<<<row_blocks(outer * n * inner, a.d), kXThreads, 0, st>>>(p, outer, n, inner, a.d);
  return 1;
}

int launch_x_sum_axis(const double* xlw, const double* xlb, const double* xuw, const double* xub, double* ylw,
                      double* ylb, double* yuw, double* yub, long long outer, int n, long long inner, int d,
                      cudaStream_t st) {
  if (outer * inner <= 0) return 0;
  x_sum_axis_kernel<<<row_blocks(outer * inner, d), kXThreads, 0, st>>>(xlw, xlb, xuw, xub, ylw, ylb, yuw, yub,
                                                                       outer, n, inner, d);
  return 1;
}

int launch_x_add(const double* a, const double* b, double* y, long long n, cudaStream_t st) {
  if (n <= 0) return 0;
  x_add_kernel<<<blocks_for(n, 256), 256, 0, st>>>(a, b, y, n);
  return 1;
}

int launch_x_scale(const double* xl, const double* xu, double s, double* yl, double* yu, long long n,
                   cudaStream_t st) {
  if (n <= 0) return 0;
  x_scale_kernel<<<blocks_for(n, 256), 256, 0, st>>>(xl, xu, s, yl, yu, n);
  return 1;
}

int launch_x_bilinear(const double* xlo, const double* xhi, const double* ylo, const double* yhi, double* out6,
                      long long n, int* status, cudaStream_t st) {
  if (n <= 0) return 0;
  x_bilinear_kernel<<<blocks_for(n, 256), 256, 0, st>>>(xlo, xhi, ylo, yhi, out6, out6 + n, out6 + 2 * n,
                                                         out6 + 3 * n, out6 + 4 * n, out6 + 5 * n, n, status);
  return 1;
}

}  // namespace fg
