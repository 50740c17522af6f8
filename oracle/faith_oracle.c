/*
 * faith_oracle.c -- TEST INFRASTRUCTURE ONLY.  Plain-C restatement of the
 * reference verifier's bound-propagation hot path (Faith, arXiv 2209.12708,
 * C++ reproduction under /root/reference/proj).  Used by tests/ as the
 * parity checker for the CUDA path and by bench.py as the CPU baseline
 * ("port"); never linked into the product library.
 *
 * Every function cites the reference code it restates.  Operation order is
 * kept identical to the reference (same accumulation order, same branch
 * rules), so on the same inputs the results are bit-identical to the
 * reference compiled with the same flags (checked in tests/test_oracle.py
 * against oracle/_ref/libfaith_ref.so and the golden vectors in
 * tests/golden/).  Compile WITHOUT -march=native / -ffast-math: FMA
 * contraction would change the rounding.
 */
#include "faith_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* Rng: std::mt19937_64 + faith::Rng draws (include/faith/rng.hpp:11-54)    */
/* ------------------------------------------------------------------------ */
typedef struct {
  uint64_t mt[312];
  int mti;
} mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->mti = 312;
}

static uint64_t mt64_next(mt64* s) {
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
  uint64_t x;
  if (s->mti >= 312) {
    int i;
    for (i = 0; i < 156; ++i) {
      x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + 156] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
    }
    for (; i < 311; ++i) {
      x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i - 156] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
    }
    x = (s->mt[311] & UM) | (s->mt[0] & LM);
    s->mt[311] = s->mt[155] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
    s->mti = 0;
  }
  x = s->mt[s->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* Rng::uniform() (rng.hpp:18) */
static double rng_uniform(mt64* s) { return (double)(mt64_next(s) >> 11) * 0x1.0p-53; }
/* Rng::uniform(lo, hi) (rng.hpp:21) */
static double rng_uniform_range(mt64* s, double lo, double hi) {
  return lo + (hi - lo) * rng_uniform(s);
}
/* Rng::uniform_index (rng.hpp:24-32) */
static uint64_t rng_uniform_index(mt64* s, uint64_t n) {
  uint64_t limit = UINT64_MAX - UINT64_MAX % n;
  uint64_t v;
  do {
    v = mt64_next(s);
  } while (v >= limit);
  return v % n;
}

int fo_rng_uniform(uint64_t seed, size_t n, double* out) {
  mt64 s;
  mt64_seed(&s, seed);
  for (size_t i = 0; i < n; ++i) out[i] = rng_uniform(&s);
  return FO_OK;
}

/* ------------------------------------------------------------------------ */
/* Synthetic model and inputs (src/model.cpp:87-141)                         */
/* ------------------------------------------------------------------------ */
size_t fo_param_count(const fo_config* c) {
  size_t e = (size_t)c->embed, f = (size_t)c->ffn, k = (size_t)c->classes;
  size_t per_layer = 4 * (e * e + e) + e * f + f + f * e + e;
  return (size_t)c->layers * per_layer + e * k + k;
}

/* gen_tensor (model.cpp:87-95) */
static double* gen_tensor(mt64* rng, double* out, size_t n, size_t fan_in) {
  double bound = 0.5 / sqrt((double)fan_in);
  for (size_t i = 0; i < n; ++i) out[i] = (double)(float)rng_uniform_range(rng, -bound, bound);
  return out + n;
}

/* gen_synthetic (model.cpp:99-131); validate()'s num_layers<=6 cap is not
 * applied (config 5 has 12 layers). */
int fo_gen_model(const fo_config* c, uint64_t seed, double* p) {
  if (c->layers < 1 || c->heads < 1 || c->embed % c->heads != 0) return FO_EINVAL;
  mt64 rng;
  mt64_seed(&rng, seed);
  size_t e = (size_t)c->embed, f = (size_t)c->ffn, k = (size_t)c->classes;
  for (int l = 0; l < c->layers; ++l) {
    p = gen_tensor(&rng, p, e * e, e); /* wq */
    p = gen_tensor(&rng, p, e, e);     /* bq */
    p = gen_tensor(&rng, p, e * e, e); /* wk */
    p = gen_tensor(&rng, p, e, e);
    p = gen_tensor(&rng, p, e * e, e); /* wv */
    p = gen_tensor(&rng, p, e, e);
    p = gen_tensor(&rng, p, e * e, e); /* wo */
    p = gen_tensor(&rng, p, e, e);
    p = gen_tensor(&rng, p, e * f, e); /* w1 */
    p = gen_tensor(&rng, p, f, e);
    p = gen_tensor(&rng, p, f * e, f); /* w2 */
    p = gen_tensor(&rng, p, e, f);
  }
  p = gen_tensor(&rng, p, e * k, e); /* wc */
  gen_tensor(&rng, p, k, e);         /* bc */
  return FO_OK;
}

/* gen_synthetic_input (model.cpp:133-141) */
int fo_gen_input(const fo_config* c, uint64_t seed, double* x) {
  mt64 rng;
  mt64_seed(&rng, seed ^ 0x9e3779b97f4a7c15ULL);
  size_t n = (size_t)c->length * (size_t)c->embed;
  for (size_t i = 0; i < n; ++i) x[i] = (double)(float)rng_uniform_range(&rng, -0.5, 0.5);
  return FO_OK;
}

/* Word positions (BASELINE.md §3 / SURVEY §8d): W distinct draws of
 * Rng(seed).uniform_index(L), sorted.  (Not in the reference: SURVEY G1.) */
int fo_gen_positions(uint64_t seed, int length, int words, int* pos) {
  if (words < 1 || words > length) return FO_EINVAL;
  mt64 rng;
  mt64_seed(&rng, seed);
  int n = 0;
  while (n < words) {
    int v = (int)rng_uniform_index(&rng, (uint64_t)length);
    int dup = 0;
    for (int i = 0; i < n; ++i) dup |= (pos[i] == v);
    if (!dup) pos[n++] = v;
  }
  for (int i = 1; i < n; ++i)
    for (int j = i; j > 0 && pos[j - 1] > pos[j]; --j) {
      int t = pos[j];
      pos[j] = pos[j - 1];
      pos[j - 1] = t;
    }
  return FO_OK;
}

/* Parameter views in gen_synthetic order. */
typedef struct {
  const double *wq, *bq, *wk, *bk, *wv, *bv, *wo, *bo, *w1, *b1, *w2, *b2;
} layer_w;

static const double* layer_view(const fo_config* c, const double* p, int l, layer_w* w) {
  size_t e = (size_t)c->embed, f = (size_t)c->ffn;
  size_t per_layer = 4 * (e * e + e) + e * f + f + f * e + e;
  p += (size_t)l * per_layer;
  w->wq = p; p += e * e; w->bq = p; p += e;
  w->wk = p; p += e * e; w->bk = p; p += e;
  w->wv = p; p += e * e; w->bv = p; p += e;
  w->wo = p; p += e * e; w->bo = p; p += e;
  w->w1 = p; p += e * f; w->b1 = p; p += f;
  w->w2 = p; p += f * e; w->b2 = p; p += e;
  return p;
}

/* ------------------------------------------------------------------------ */
/* Exact forward (ForwardEvaluator::operator(), model.cpp:491-564)           */
/* ------------------------------------------------------------------------ */
static double silu_scalar(double x) { return x * (1.0 / (1.0 + exp(-x))); } /* relax.cpp:128 */
static double silu_derivative(double x) {                                   /* relax.cpp:130 */
  double s = 1.0 / (1.0 + exp(-x));
  return s * (1.0 + x * (1.0 - s));
}

static double apply_activation(int a, double x) { /* model.cpp:456-467 */
  switch (a) {
    case FO_ACT_RELU: return x > 0.0 ? x : 0.0;
    case FO_ACT_TANH: return tanh(x);
    case FO_ACT_SILU: return silu_scalar(x);
  }
  return x;
}

/* dense (model.cpp:470-483) */
static void dense(const double* x, size_t rows, size_t c, size_t o, const double* w,
                  const double* b, double* out) {
  memset(out, 0, rows * o * sizeof(double));
  for (size_t r = 0; r < rows; ++r) {
    const double* xr = x + r * c;
    for (size_t i = 0; i < c; ++i) {
      double xv = xr[i];
      const double* wr = w + i * o;
      double* orow = out + r * o;
      for (size_t j = 0; j < o; ++j) orow[j] += xv * wr[j];
    }
    for (size_t j = 0; j < o; ++j) out[r * o + j] += b[j];
  }
}

int fo_forward(const fo_config* c, const double* params, const double* x, double* logits) {
  size_t len = (size_t)c->length, e = (size_t)c->embed, f = (size_t)c->ffn;
  size_t heads = (size_t)c->heads, hd = e / heads, rows = len;
  double inv_sqrt_hd = 1.0 / sqrt((double)hd);
  double* cur = malloc(rows * e * sizeof(double));
  double* q = malloc(rows * e * sizeof(double));
  double* k = malloc(rows * e * sizeof(double));
  double* v = malloc(rows * e * sizeof(double));
  double* sc = malloc(heads * len * len * sizeof(double));
  double* ctx = malloc(rows * e * sizeof(double));
  double* attn = malloc(rows * e * sizeof(double));
  double* ffn = malloc(rows * f * sizeof(double));
  memcpy(cur, x, rows * e * sizeof(double));
  const double* tail = params;
  for (int l = 0; l < c->layers; ++l) {
    layer_w w;
    tail = layer_view(c, params, l, &w);
    dense(cur, rows, e, e, w.wq, w.bq, q);
    dense(cur, rows, e, e, w.wk, w.bk, k);
    dense(cur, rows, e, e, w.wv, w.bv, v);
    for (size_t h = 0; h < heads; ++h) {
      for (size_t i = 0; i < len; ++i) {
        for (size_t j = 0; j < len; ++j) {
          double acc = 0.0;
          const double* qi = q + i * e + h * hd;
          const double* kj = k + j * e + h * hd;
          for (size_t d = 0; d < hd; ++d) acc += qi[d] * kj[d];
          sc[(h * len + i) * len + j] = acc * inv_sqrt_hd;
        }
        double* row = sc + (h * len + i) * len;
        double mx = row[0];
        for (size_t j = 1; j < len; ++j) mx = mx < row[j] ? row[j] : mx; /* std::max */
        double sum = 0.0;
        for (size_t j = 0; j < len; ++j) {
          row[j] = exp(row[j] - mx);
          sum += row[j];
        }
        for (size_t j = 0; j < len; ++j) row[j] /= sum;
      }
    }
    memset(ctx, 0, rows * e * sizeof(double));
    for (size_t h = 0; h < heads; ++h) {
      for (size_t i = 0; i < len; ++i) {
        const double* prow = sc + (h * len + i) * len;
        double* crow = ctx + i * e + h * hd;
        for (size_t j = 0; j < len; ++j) {
          const double* vj = v + j * e + h * hd;
          double pv = prow[j];
          for (size_t d = 0; d < hd; ++d) crow[d] += pv * vj[d];
        }
      }
    }
    dense(ctx, rows, e, e, w.wo, w.bo, attn);
    for (size_t i = 0; i < rows * e; ++i) cur[i] += attn[i];
    dense(cur, rows, e, f, w.w1, w.b1, ffn);
    for (size_t i = 0; i < rows * f; ++i) ffn[i] = apply_activation(c->activation, ffn[i]);
    dense(ffn, rows, f, e, w.w2, w.b2, attn);
    for (size_t i = 0; i < rows * e; ++i) cur[i] += attn[i];
  }
  const double* wc = tail;
  const double* bc = wc + e * (size_t)c->classes;
  double* pooled = calloc(e, sizeof(double));
  for (size_t i = 0; i < len; ++i)
    for (size_t d = 0; d < e; ++d) pooled[d] += cur[i * e + d];
  for (size_t d = 0; d < e; ++d) pooled[d] /= (double)len;
  dense(pooled, 1, e, (size_t)c->classes, wc, bc, logits);
  free(pooled); free(cur); free(q); free(k); free(v); free(sc); free(ctx); free(attn); free(ffn);
  for (int i = 0; i < c->classes; ++i)
    if (!isfinite(logits[i])) return FO_EINVAL; /* Tensor ctor finiteness (tensor.cpp:54) */
  return FO_OK;
}

/* ------------------------------------------------------------------------ */
/* Bounds (src/bounds.cpp)                                                   */
/* ------------------------------------------------------------------------ */
typedef struct {
  size_t n, d;
  double *lw, *lb, *uw, *ub;
} bnd;

static int bnd_alloc(bnd* b, size_t n, size_t d) {
  b->n = n;
  b->d = d;
  b->lw = calloc((n * d) > 0 ? n * d : 1, sizeof(double));
  b->uw = calloc((n * d) > 0 ? n * d : 1, sizeof(double));
  b->lb = calloc(n ? n : 1, sizeof(double));
  b->ub = calloc(n ? n : 1, sizeof(double));
  return (b->lw && b->uw && b->lb && b->ub) ? FO_OK : FO_EINVAL;
}
static void bnd_free(bnd* b) {
  free(b->lw); free(b->uw); free(b->lb); free(b->ub);
  memset(b, 0, sizeof(*b));
}
static bnd bnd_view(size_t n, size_t d, const double* lw, const double* lb, const double* uw,
                    const double* ub) {
  bnd b = {n, d, (double*)lw, (double*)lb, (double*)uw, (double*)ub};
  return b;
}
static void bnd_export(const bnd* b, double* lw, double* lb, double* uw, double* ub) {
  memcpy(lw, b->lw, b->n * b->d * sizeof(double));
  memcpy(uw, b->uw, b->n * b->d * sizeof(double));
  memcpy(lb, b->lb, b->n * sizeof(double));
  memcpy(ub, b->ub, b->n * sizeof(double));
}

static int dual_norm(int p) { /* bounds.cpp:9-19 */
  return p == FO_NORM_L1 ? FO_NORM_LINF : (p == FO_NORM_L2 ? FO_NORM_L2 : FO_NORM_L1);
}

/* row_norm (bounds.cpp:80-99) */
static double row_norm(const double* row, size_t d, int q) {
  if (q == FO_NORM_L1) {
    double s = 0.0;
    for (size_t k = 0; k < d; ++k) s += fabs(row[k]);
    return s;
  }
  if (q == FO_NORM_L2) {
    double s = 0.0;
    for (size_t k = 0; k < d; ++k) s += row[k] * row[k];
    return sqrt(s);
  }
  double m = 0.0;
  for (size_t k = 0; k < d; ++k) {
    double a = fabs(row[k]);
    m = (m < a) ? a : m; /* std::max(m, a) */
  }
  return m;
}

/* concretize (bounds.cpp:122-140) */
static void concretize(const bnd* b, int p, double eps, double* lo, double* hi) {
  int q = dual_norm(p);
  for (size_t i = 0; i < b->n; ++i) {
    double ln = row_norm(b->lw + i * b->d, b->d, q);
    double un = row_norm(b->uw + i * b->d, b->d, q);
    lo[i] = b->lb[i] - eps * ln;
    hi[i] = b->ub[i] + eps * un;
  }
}

int fo_concretize(size_t n, size_t d, const double* lw, const double* lb, const double* uw,
                  const double* ub, int norm, double eps, double* lo, double* hi) {
  if (!(eps >= 0.0) || !isfinite(eps)) return FO_EINVAL; /* PerturbationSpec (bounds.cpp:41) */
  bnd b = bnd_view(n, d, lw, lb, uw, ub);
  concretize(&b, norm, eps, lo, hi);
  return FO_OK;
}

/* check_robust (bounds.cpp:142-157) */
int fo_check_robust(size_t n, const double* lo, const double* hi, size_t t, double margin,
                    int* verified) {
  if (t >= n) return FO_ERANGE;
  if (margin < 0.0) return FO_EINVAL;
  double lo_t = lo[t];
  *verified = 1;
  for (size_t j = 0; j < n; ++j) {
    if (j == t) continue;
    if (!(lo_t > hi[j] + margin)) {
      *verified = 0;
      return FO_OK;
    }
  }
  return FO_OK;
}

/* ------------------------------------------------------------------------ */
/* propagate_affine (relax.cpp:237-307)                                      */
/* ------------------------------------------------------------------------ */
static void affine(const bnd* x, size_t rows, size_t c, size_t o, const double* w,
                   const double* bias, bnd* y) {
  size_t d = x->d;
  double* uw_neg = malloc((d ? d : 1) * sizeof(double));
  double* lw_neg = malloc((d ? d : 1) * sizeof(double));
  for (size_t r = 0; r < rows; ++r) {
    for (size_t j = 0; j < o; ++j) {
      double ub_pos = 0.0, ub_neg = 0.0, lb_pos = 0.0, lb_neg = 0.0;
      double* yuw = y->uw + (r * o + j) * d;
      double* ylw = y->lw + (r * o + j) * d;
      memset(uw_neg, 0, d * sizeof(double));
      memset(lw_neg, 0, d * sizeof(double));
      for (size_t i = 0; i < c; ++i) {
        double wv = w[i * o + j];
        double wp = (wv < 0.0) ? 0.0 : wv; /* std::max(wv, 0.0) */
        double wn = (0.0 < wv) ? 0.0 : wv; /* std::min(wv, 0.0) */
        ub_pos += wp * x->ub[r * c + i];
        ub_neg += wn * x->lb[r * c + i];
        lb_pos += wp * x->lb[r * c + i];
        lb_neg += wn * x->ub[r * c + i];
        const double* xur = x->uw + (r * c + i) * d;
        const double* xlr = x->lw + (r * c + i) * d;
        for (size_t k = 0; k < d; ++k) {
          yuw[k] += wp * xur[k];
          uw_neg[k] += wn * xlr[k];
          ylw[k] += wp * xlr[k];
          lw_neg[k] += wn * xur[k];
        }
      }
      double bv = bias ? bias[j] : 0.0;
      y->ub[r * o + j] = ub_pos + ub_neg + bv;
      y->lb[r * o + j] = lb_pos + lb_neg + bv;
      for (size_t k = 0; k < d; ++k) {
        yuw[k] += uw_neg[k];
        ylw[k] += lw_neg[k];
      }
    }
  }
  free(uw_neg);
  free(lw_neg);
}

int fo_affine(size_t rows, size_t c, size_t o, size_t d, const double* xlw, const double* xlb,
              const double* xuw, const double* xub, const double* w, const double* bias,
              double* ylw, double* ylb, double* yuw, double* yub) {
  bnd x = bnd_view(rows * c, d, xlw, xlb, xuw, xub), y;
  if (bnd_alloc(&y, rows * o, d) != FO_OK) return FO_EINVAL;
  affine(&x, rows, c, o, w, bias, &y);
  bnd_export(&y, ylw, ylb, yuw, yub);
  bnd_free(&y);
  return FO_OK;
}

/* ------------------------------------------------------------------------ */
/* Elementwise relaxations (relax.cpp:12-108, 313-468)                       */
/* ------------------------------------------------------------------------ */
typedef struct {
  double a, b;
} line;

static double sech2(double x) { double t = tanh(x); return 1.0 - t * t; } /* relax.cpp:12 */

static line chord(double lo, double hi, double flo, double fhi) { /* relax.cpp:24-27 */
  double s = (fhi - flo) / (hi - lo);
  line l = {s, flo - s * lo};
  return l;
}

static double bisect_tanh_tangent(double anchor, double blo, double bhi) { /* relax.cpp:33 */
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

static void tanh_lines_nonneg(double lo, double hi, line* lower, line* upper) { /* :56-62 */
  *lower = chord(lo, hi, tanh(lo), tanh(hi));
  double m = 0.5 * (lo + hi);
  double a = sech2(m);
  upper->a = a;
  upper->b = tanh(m) - a * m;
}

static void tanh_lines(double lo, double hi, line* lower, line* upper) { /* relax.cpp:64-108 */
  if (lo == hi) {
    double a = sech2(lo);
    double b = tanh(lo) - a * lo;
    lower->a = a; lower->b = b;
    upper->a = a; upper->b = b;
    return;
  }
  if (lo >= 0.0) {
    tanh_lines_nonneg(lo, hi, lower, upper);
    return;
  }
  if (hi <= 0.0) {
    line ml, mu;
    tanh_lines_nonneg(-hi, -lo, &ml, &mu);
    lower->a = mu.a; lower->b = -mu.b;
    upper->a = ml.a; upper->b = -ml.b;
    return;
  }
  double flo = tanh(lo);
  double gap_hi = tanh(hi) + sech2(hi) * (lo - hi) - flo;
  if (gap_hi < 0.0) {
    *upper = chord(lo, hi, flo, tanh(hi));
  } else {
    double dd = bisect_tanh_tangent(lo, 0.0, hi);
    double a = sech2(dd);
    upper->a = a;
    upper->b = tanh(dd) - a * dd;
  }
  line mu;
  double mflo = tanh(-hi);
  double mgap = tanh(-lo) + sech2(-lo) * (-hi + lo) - mflo;
  if (mgap < 0.0) {
    mu = chord(-hi, -lo, mflo, tanh(-lo));
  } else {
    double dd = bisect_tanh_tangent(-hi, 0.0, -lo);
    double a = sech2(dd);
    mu.a = a;
    mu.b = tanh(dd) - a * dd;
  }
  lower->a = mu.a;
  lower->b = -mu.b;
}

/* relax_{relu,tanh,silu,exp,recip}; returns FO_EINVAL when the concretized
 * interval is inverted (ConcreteBounds::validate, bounds.cpp:69-78) and
 * FO_EDOMAIN on the reference's domain errors (relax.cpp:389-391, 406-409). */
static int relax(int kind, size_t n, const double* lo_, const double* hi_, double* a_low,
                 double* b_low, double* a_up, double* b_up) {
  for (size_t i = 0; i < n; ++i)
    if (lo_[i] > hi_[i]) return FO_EINVAL;
  for (size_t i = 0; i < n; ++i) {
    double lo = lo_[i], hi = hi_[i];
    a_low[i] = b_low[i] = a_up[i] = b_up[i] = 0.0;
    switch (kind) {
      case FO_RELAX_RELU: /* relax.cpp:313-337 */
        if (lo >= 0.0) {
          a_low[i] = 1.0;
          a_up[i] = 1.0;
        } else if (hi <= 0.0) {
        } else {
          double s = hi / (hi - lo);
          a_up[i] = s;
          b_up[i] = -s * lo;
          a_low[i] = (fabs(lo) > fabs(hi)) ? 0.0 : 1.0;
        }
        break;
      case FO_RELAX_TANH: { /* relax.cpp:339-356 */
        line lower, upper;
        tanh_lines(lo, hi, &lower, &upper);
        a_low[i] = lower.a; b_low[i] = lower.b;
        a_up[i] = upper.a; b_up[i] = upper.b;
        break;
      }
      case FO_RELAX_EXP: { /* relax.cpp:363-394 */
        double m = 0.5 * (lo + hi), c2 = lo + 15.0 / 16.0;
        double d = (c2 < m) ? c2 : m; /* std::min(mid, lo + 15/16) */
        double ed = exp(d);
        a_low[i] = ed;
        b_low[i] = ed - ed * d;
        if (lo == hi) {
          a_up[i] = ed;
          b_up[i] = ed - ed * d;
        } else {
          line up = chord(lo, hi, exp(lo), exp(hi));
          a_up[i] = up.a;
          b_up[i] = up.b;
        }
        if (!isfinite(b_low[i]) || !isfinite(a_up[i]) || !isfinite(b_up[i])) return FO_EDOMAIN;
        break;
      }
      case FO_RELAX_RECIP: { /* relax.cpp:396-424 */
        if (lo <= 0.0) return FO_EDOMAIN;
        double m = 0.5 * (lo + hi);
        double am = -1.0 / (m * m);
        a_low[i] = am;
        b_low[i] = 2.0 / m;
        if (lo == hi) {
          a_up[i] = am;
          b_up[i] = 2.0 / m;
        } else {
          line up = chord(lo, hi, 1.0 / lo, 1.0 / hi);
          a_up[i] = up.a;
          b_up[i] = up.b;
        }
        break;
      }
      case FO_RELAX_SILU: { /* relax.cpp:426-468 */
        if (lo == hi) {
          double a = silu_derivative(lo);
          a_low[i] = a;
          a_up[i] = a;
          b_low[i] = silu_scalar(lo) - a * lo;
          b_up[i] = b_low[i];
          break;
        }
        double s = (silu_scalar(hi) - silu_scalar(lo)) / (hi - lo);
        double step = (hi - lo) / 256;
        double gmin = HUGE_VAL, gmax = -HUGE_VAL;
        for (int k = 0; k <= 256; ++k) {
          double x = (k == 256) ? hi : lo + step * k;
          double g = silu_scalar(x) - s * x;
          gmin = (g < gmin) ? g : gmin;
          gmax = (gmax < g) ? g : gmax;
        }
        double margin = 0.6 * step * step / 8.0 + 1e-12;
        a_low[i] = s;
        a_up[i] = s;
        b_low[i] = gmin - margin;
        b_up[i] = gmax + margin;
        break;
      }
      default:
        return FO_EINVAL;
    }
  }
  return FO_OK;
}

int fo_relax(int kind, size_t n, const double* lo, const double* hi, double* a_low,
             double* b_low, double* a_up, double* b_up) {
  return relax(kind, n, lo, hi, a_low, b_low, a_up, b_up);
}

/* compose_elementwise (relax.cpp:470-497) */
static void compose(const bnd* x, const double* a_low, const double* b_low, const double* a_up,
                    const double* b_up, bnd* y) {
  size_t d = x->d;
  for (size_t i = 0; i < x->n; ++i) {
    double au = a_up[i];
    const double* src_u = (au >= 0.0) ? x->uw + i * d : x->lw + i * d;
    y->ub[i] = au * ((au >= 0.0) ? x->ub[i] : x->lb[i]) + b_up[i];
    double* dst_u = y->uw + i * d;
    for (size_t k = 0; k < d; ++k) dst_u[k] = au * src_u[k];
    double al = a_low[i];
    const double* src_l = (al >= 0.0) ? x->lw + i * d : x->uw + i * d;
    y->lb[i] = al * ((al >= 0.0) ? x->lb[i] : x->ub[i]) + b_low[i];
    double* dst_l = y->lw + i * d;
    for (size_t k = 0; k < d; ++k) dst_l[k] = al * src_l[k];
  }
}

int fo_compose(size_t n, size_t d, const double* xlw, const double* xlb, const double* xuw,
               const double* xub, const double* a_low, const double* b_low,
               const double* a_up, const double* b_up, double* ylw, double* ylb, double* yuw,
               double* yub) {
  bnd x = bnd_view(n, d, xlw, xlb, xuw, xub), y;
  if (bnd_alloc(&y, n, d) != FO_OK) return FO_EINVAL;
  compose(&x, a_low, b_low, a_up, b_up, &y);
  bnd_export(&y, ylw, ylb, yuw, yub);
  bnd_free(&y);
  return FO_OK;
}

/* elementwise_verify (graph.cpp:484-501): concretize -> relax -> compose */
static int elementwise_verify(int kind, const bnd* x, int p, double eps, bnd* y) {
  size_t n = x->n;
  double* buf = malloc(6 * (n ? n : 1) * sizeof(double));
  double *lo = buf, *hi = buf + n, *al = buf + 2 * n, *bl = buf + 3 * n, *au = buf + 4 * n,
         *bu = buf + 5 * n;
  concretize(x, p, eps, lo, hi);
  int st = relax(kind, n, lo, hi, al, bl, au, bu);
  if (st == FO_OK) compose(x, al, bl, au, bu, y);
  free(buf);
  return st;
}

int fo_elementwise_verify(int kind, size_t n, size_t d, const double* xlw, const double* xlb,
                          const double* xuw, const double* xub, int norm, double eps,
                          double* ylw, double* ylb, double* yuw, double* yub) {
  bnd x = bnd_view(n, d, xlw, xlb, xuw, xub), y;
  if (bnd_alloc(&y, n, d) != FO_OK) return FO_EINVAL;
  int st = elementwise_verify(kind, &x, norm, eps, &y);
  if (st == FO_OK) bnd_export(&y, ylw, ylb, yuw, yub);
  bnd_free(&y);
  return st;
}

/* ------------------------------------------------------------------------ */
/* McCormick products (relax.cpp:533-654, 744-775)                           */
/* ------------------------------------------------------------------------ */
/* accumulate_product_term (relax.cpp:533-569) */
static void product_term(const bnd* a, const bnd* b, const double* alo, const double* blo,
                         const double* bhi, size_t xi, size_t yi, double* out_lb, double* out_ub,
                         double* out_lw, double* out_uw) {
  size_t d = a->d;
  double lx = alo[xi], ly = blo[yi], uy = bhi[yi];
  {
    double cx = ly, cy = lx;
    const double* xr = (cx >= 0.0) ? a->lw + xi * d : a->uw + xi * d;
    const double* yr = (cy >= 0.0) ? b->lw + yi * d : b->uw + yi * d;
    *out_lb += cx * ((cx >= 0.0) ? a->lb[xi] : a->ub[xi]) +
               cy * ((cy >= 0.0) ? b->lb[yi] : b->ub[yi]) - lx * ly;
    if (cx != 0.0)
      for (size_t k = 0; k < d; ++k) out_lw[k] += cx * xr[k];
    if (cy != 0.0)
      for (size_t k = 0; k < d; ++k) out_lw[k] += cy * yr[k];
  }
  {
    double cx = uy, cy = lx;
    const double* xr = (cx >= 0.0) ? a->uw + xi * d : a->lw + xi * d;
    const double* yr = (cy >= 0.0) ? b->uw + yi * d : b->lw + yi * d;
    *out_ub += cx * ((cx >= 0.0) ? a->ub[xi] : a->lb[xi]) +
               cy * ((cy >= 0.0) ? b->ub[yi] : b->lb[yi]) - lx * uy;
    if (cx != 0.0)
      for (size_t k = 0; k < d; ++k) out_uw[k] += cx * xr[k];
    if (cy != 0.0)
      for (size_t k = 0; k < d; ++k) out_uw[k] += cy * yr[k];
  }
}

/* propagate_dot_product (relax.cpp:573-654), batch 1 */
static int dot(int layout, size_t len, size_t e, size_t heads, const bnd* a, const bnd* b,
               int p, double eps, bnd* y) {
  size_t d = a->d;
  if (heads == 0 || e % heads != 0 || b->d != d) return FO_EINVAL;
  size_t hd = e / heads;
  double* ca = malloc(2 * a->n * sizeof(double));
  double* cb = malloc(2 * b->n * sizeof(double));
  concretize(a, p, eps, ca, ca + a->n);
  concretize(b, p, eps, cb, cb + b->n);
  if (layout == FO_DOT_SIMILARITY) {
    for (size_t h = 0; h < heads; ++h)
      for (size_t i = 0; i < len; ++i)
        for (size_t j = 0; j < len; ++j) {
          size_t oidx = (h * len + i) * len + j;
          for (size_t k = 0; k < hd; ++k) {
            size_t xi = i * e + h * hd + k, yi = j * e + h * hd + k;
            product_term(a, b, ca, cb, cb + b->n, xi, yi, &y->lb[oidx], &y->ub[oidx],
                         y->lw + oidx * d, y->uw + oidx * d);
          }
        }
  } else {
    for (size_t i = 0; i < len; ++i)
      for (size_t h = 0; h < heads; ++h)
        for (size_t k = 0; k < hd; ++k) {
          size_t oidx = i * e + h * hd + k;
          for (size_t j = 0; j < len; ++j) {
            size_t xi = (h * len + i) * len + j, yi = j * e + h * hd + k;
            product_term(a, b, ca, cb, cb + b->n, xi, yi, &y->lb[oidx], &y->ub[oidx],
                         y->lw + oidx * d, y->uw + oidx * d);
          }
        }
  }
  free(ca);
  free(cb);
  return FO_OK;
}

int fo_dot(int layout, size_t len, size_t embed, size_t heads, size_t d, const double* alw,
           const double* alb, const double* auw, const double* aub, const double* blw,
           const double* blb, const double* buw, const double* bub, int norm, double eps,
           double* ylw, double* ylb, double* yuw, double* yub) {
  if (heads == 0 || embed % heads != 0) return FO_EINVAL;
  size_t na = layout == FO_DOT_SIMILARITY ? len * embed : heads * len * len;
  size_t nb = len * embed;
  size_t ny = layout == FO_DOT_SIMILARITY ? heads * len * len : len * embed;
  bnd a = bnd_view(na, d, alw, alb, auw, aub), b = bnd_view(nb, d, blw, blb, buw, bub), y;
  if (bnd_alloc(&y, ny, d) != FO_OK) return FO_EINVAL;
  int st = dot(layout, len, embed, heads, &a, &b, norm, eps, &y);
  if (st == FO_OK) bnd_export(&y, ylw, ylb, yuw, yub);
  bnd_free(&y);
  return st;
}

/* propagate_scale (relax.cpp:676-703) */
static void scale(const bnd* x, double s, bnd* y) {
  size_t n = x->n, nd = x->n * x->d;
  if (s >= 0.0) {
    for (size_t i = 0; i < n; ++i) { y->lb[i] = s * x->lb[i]; y->ub[i] = s * x->ub[i]; }
    for (size_t i = 0; i < nd; ++i) { y->lw[i] = s * x->lw[i]; y->uw[i] = s * x->uw[i]; }
  } else {
    for (size_t i = 0; i < n; ++i) { y->lb[i] = s * x->ub[i]; y->ub[i] = s * x->lb[i]; }
    for (size_t i = 0; i < nd; ++i) { y->lw[i] = s * x->uw[i]; y->uw[i] = s * x->lw[i]; }
  }
}

/* propagate_add (relax.cpp:656-674) */
static void add(const bnd* a, const bnd* b, bnd* y) {
  for (size_t i = 0; i < a->n; ++i) { y->lb[i] = a->lb[i] + b->lb[i]; y->ub[i] = a->ub[i] + b->ub[i]; }
  for (size_t i = 0; i < a->n * a->d; ++i) {
    y->lw[i] = a->lw[i] + b->lw[i];
    y->uw[i] = a->uw[i] + b->uw[i];
  }
}

/* propagate_sum_axis (relax.cpp:705-742) on [outer, n, inner] */
static void sum_axis(const bnd* x, size_t outer, size_t n, size_t inner, bnd* y) {
  size_t d = x->d;
  for (size_t oi = 0; oi < outer; ++oi)
    for (size_t ii = 0; ii < inner; ++ii) {
      size_t oidx = oi * inner + ii;
      double* ylw = y->lw + oidx * d;
      double* yuw = y->uw + oidx * d;
      for (size_t j = 0; j < n; ++j) {
        size_t idx = (oi * n + j) * inner + ii;
        y->lb[oidx] += x->lb[idx];
        y->ub[oidx] += x->ub[idx];
        const double* xlr = x->lw + idx * d;
        const double* xur = x->uw + idx * d;
        for (size_t k = 0; k < d; ++k) {
          ylw[k] += xlr[k];
          yuw[k] += xur[k];
        }
      }
    }
}

/* propagate_mul_broadcast (relax.cpp:744-775) on [outer, n, inner] x r[outer, 1, inner] */
static void mul_broadcast(const bnd* x, const bnd* r, size_t outer, size_t n, size_t inner,
                          int p, double eps, bnd* y) {
  size_t d = x->d;
  double* cx = malloc(2 * x->n * sizeof(double));
  double* cr = malloc(2 * r->n * sizeof(double));
  concretize(x, p, eps, cx, cx + x->n);
  concretize(r, p, eps, cr, cr + r->n);
  for (size_t oi = 0; oi < outer; ++oi)
    for (size_t ii = 0; ii < inner; ++ii) {
      size_t ridx = oi * inner + ii;
      for (size_t j = 0; j < n; ++j) {
        size_t idx = (oi * n + j) * inner + ii;
        product_term(x, r, cx, cr, cr + r->n, idx, ridx, &y->lb[idx], &y->ub[idx],
                     y->lw + idx * d, y->uw + idx * d);
      }
    }
  free(cx);
  free(cr);
}

/* Softmax as the fused graph evaluates it (graph.cpp:237-240): ExpVerify ->
 * SumReduce -> RecipVerify -> MulBroadcast, each a separate node.  The
 * intermediate nodes are returned so the pass can dump them. */
static int softmax_chain(const bnd* x, size_t rows, size_t n, int p, double eps, bnd* e, bnd* s,
                         bnd* r, bnd* y) {
  size_t d = x->d;
  int st;
  if ((st = bnd_alloc(e, rows * n, d)) != FO_OK) return st;
  if ((st = elementwise_verify(FO_RELAX_EXP, x, p, eps, e)) != FO_OK) return st;
  if ((st = bnd_alloc(s, rows, d)) != FO_OK) return st;
  sum_axis(e, rows, n, 1, s);
  if ((st = bnd_alloc(r, rows, d)) != FO_OK) return st;
  if ((st = elementwise_verify(FO_RELAX_RECIP, s, p, eps, r)) != FO_OK) return st;
  if ((st = bnd_alloc(y, rows * n, d)) != FO_OK) return st;
  mul_broadcast(e, r, rows, n, 1, p, eps, y);
  return FO_OK;
}

int fo_softmax(size_t rows, size_t n, size_t d, const double* xlw, const double* xlb,
               const double* xuw, const double* xub, int norm, double eps, double* ylw,
               double* ylb, double* yuw, double* yub) {
  /* propagate_softmax (relax.cpp:777-790) computes the same chain. */
  bnd x = bnd_view(rows * n, d, xlw, xlb, xuw, xub);
  bnd e = {0}, s = {0}, r = {0}, y = {0};
  int st = softmax_chain(&x, rows, n, norm, eps, &e, &s, &r, &y);
  if (st == FO_OK) bnd_export(&y, ylw, ylb, yuw, yub);
  bnd_free(&e); bnd_free(&s); bnd_free(&r); bnd_free(&y);
  return st;
}

/* ------------------------------------------------------------------------ */
/* Pass: graph::evaluate over fuse_all(build_graph(spec)) (graph.cpp:505-673,
 * model.cpp:393-448), word-level input binding.                 */
/* ------------------------------------------------------------------------ */
size_t fo_node_dump_size(const fo_config* c) {
  size_t L = (size_t)c->length, E = (size_t)c->embed, H = (size_t)c->heads,
         F = (size_t)c->ffn;
  size_t per_layer = 8 * L * E + 4 * H * L * L + 2 * H * L + 2 * L * F;
  return (size_t)c->layers * per_layer + E + (size_t)c->classes;
}

typedef struct {
  double *lo, *hi;
  size_t off;
  int p;
  double eps;
  int count, max_nodes; /* max_nodes > 0: stop the pass after that many nodes */
} dumper;

/* returns 1 when the node budget of a prefix pass is exhausted */
static int dump(dumper* dp, const bnd* b) {
  if (dp->lo) concretize(b, dp->p, dp->eps, dp->lo + dp->off, dp->hi + dp->off);
  dp->off += b->n;
  return dp->max_nodes > 0 && ++dp->count >= dp->max_nodes;
}

static int all_finite(const bnd* b) {
  for (size_t i = 0; i < b->n; ++i)
    if (!isfinite(b->lb[i]) || !isfinite(b->ub[i])) return 0;
  for (size_t i = 0; i < b->n * b->d; ++i)
    if (!isfinite(b->lw[i]) || !isfinite(b->uw[i])) return 0;
  return 1;
}

#define TRY(x)                 \
  do {                         \
    if ((st = (x)) != FO_OK) { \
      goto done;               \
    }                          \
  } while (0)

static int bound_pass(const fo_config* c, const double* params, const double* x,
                      const int* positions, int words, int norm, double eps, double* logits_lo,
                      double* logits_hi, double* node_lo, double* node_hi, int max_nodes) {
  if (!(eps >= 0.0) || !isfinite(eps)) return FO_EINVAL;
  size_t L = (size_t)c->length, E = (size_t)c->embed, H = (size_t)c->heads,
         F = (size_t)c->ffn, C = (size_t)c->classes, D = (size_t)words * E;
  if (words < 1 || H == 0 || E % H != 0) return FO_EINVAL;
  dumper dp = {node_lo, node_hi, 0, norm, eps, 0, max_nodes};
  int st = FO_OK;
  bnd cur = {0}, q = {0}, k = {0}, v = {0}, sc = {0}, scl = {0}, e = {0}, s = {0}, r = {0},
      pr = {0}, ctx = {0}, attn = {0}, res1 = {0}, f1 = {0}, act = {0}, f2 = {0}, sum = {0},
      pooled = {0}, logits = {0};

  /* Input binding: lb = ub = x; rows of perturbed positions one-hot. */
  TRY(bnd_alloc(&cur, L * E, D));
  memcpy(cur.lb, x, L * E * sizeof(double));
  memcpy(cur.ub, x, L * E * sizeof(double));
  for (int w = 0; w < words; ++w)
    for (size_t ee = 0; ee < E; ++ee) {
      size_t row = (size_t)positions[w] * E + ee, col = (size_t)w * E + ee;
      cur.lw[row * D + col] = 1.0;
      cur.uw[row * D + col] = 1.0;
    }

  double inv_sqrt_hd = 1.0 / sqrt((double)(E / H)); /* model.cpp:417 */
  const double* tail = params;
  for (int l = 0; l < c->layers; ++l) {
    layer_w w;
    tail = layer_view(c, params, l, &w);
    TRY(bnd_alloc(&q, L * E, D)); affine(&cur, L, E, E, w.wq, w.bq, &q); if (dump(&dp, &q)) { st = FO_STOPPED; goto done; }
    TRY(bnd_alloc(&k, L * E, D)); affine(&cur, L, E, E, w.wk, w.bk, &k); if (dump(&dp, &k)) { st = FO_STOPPED; goto done; }
    TRY(bnd_alloc(&v, L * E, D)); affine(&cur, L, E, E, w.wv, w.bv, &v); if (dump(&dp, &v)) { st = FO_STOPPED; goto done; }
    TRY(bnd_alloc(&sc, H * L * L, D));
    TRY(dot(FO_DOT_SIMILARITY, L, E, H, &q, &k, norm, eps, &sc));
    if (dump(&dp, &sc)) { st = FO_STOPPED; goto done; }
    bnd_free(&q); bnd_free(&k);
    TRY(bnd_alloc(&scl, H * L * L, D)); scale(&sc, inv_sqrt_hd, &scl); if (dump(&dp, &scl)) { st = FO_STOPPED; goto done; }
    bnd_free(&sc);
    TRY(softmax_chain(&scl, H * L, L, norm, eps, &e, &s, &r, &pr));
    if (dump(&dp, &e)) { st = FO_STOPPED; goto done; } if (dump(&dp, &s)) { st = FO_STOPPED; goto done; } if (dump(&dp, &r)) { st = FO_STOPPED; goto done; } if (dump(&dp, &pr)) { st = FO_STOPPED; goto done; }
    bnd_free(&scl); bnd_free(&e); bnd_free(&s); bnd_free(&r);
    TRY(bnd_alloc(&ctx, L * E, D));
    TRY(dot(FO_DOT_WEIGHTED_VALUES, L, E, H, &pr, &v, norm, eps, &ctx));
    if (dump(&dp, &ctx)) { st = FO_STOPPED; goto done; }
    bnd_free(&pr); bnd_free(&v);
    TRY(bnd_alloc(&attn, L * E, D)); affine(&ctx, L, E, E, w.wo, w.bo, &attn); if (dump(&dp, &attn)) { st = FO_STOPPED; goto done; }
    bnd_free(&ctx);
    TRY(bnd_alloc(&res1, L * E, D)); add(&cur, &attn, &res1); if (dump(&dp, &res1)) { st = FO_STOPPED; goto done; }
    bnd_free(&cur); bnd_free(&attn);
    TRY(bnd_alloc(&f1, L * F, D)); affine(&res1, L, E, F, w.w1, w.b1, &f1); if (dump(&dp, &f1)) { st = FO_STOPPED; goto done; }
    int kind = c->activation == FO_ACT_TANH   ? FO_RELAX_TANH
               : c->activation == FO_ACT_SILU ? FO_RELAX_SILU
                                              : FO_RELAX_RELU;
    TRY(bnd_alloc(&act, L * F, D));
    TRY(elementwise_verify(kind, &f1, norm, eps, &act));
    if (dump(&dp, &act)) { st = FO_STOPPED; goto done; }
    bnd_free(&f1);
    TRY(bnd_alloc(&f2, L * E, D)); affine(&act, L, F, E, w.w2, w.b2, &f2); if (dump(&dp, &f2)) { st = FO_STOPPED; goto done; }
    bnd_free(&act);
    TRY(bnd_alloc(&cur, L * E, D)); add(&res1, &f2, &cur); if (dump(&dp, &cur)) { st = FO_STOPPED; goto done; }
    bnd_free(&res1); bnd_free(&f2);
  }
  /* MeanPool (graph.cpp:628-634) then the classifier head. */
  TRY(bnd_alloc(&sum, E, D));
  sum_axis(&cur, 1, L, E, &sum);
  TRY(bnd_alloc(&pooled, E, D));
  scale(&sum, 1.0 / (double)L, &pooled);
  if (dump(&dp, &pooled)) { st = FO_STOPPED; goto done; }
  {
    const double* wc = tail;
    const double* bc = wc + E * C;
    TRY(bnd_alloc(&logits, C, D));
    affine(&pooled, 1, E, C, wc, bc, &logits);
  }
  if (dump(&dp, &logits)) { st = FO_STOPPED; goto done; }
  if (!all_finite(&logits)) { /* graph.cpp:663-671 */
    st = FO_EDOMAIN;
    goto done;
  }
  concretize(&logits, norm, eps, logits_lo, logits_hi); /* cli.cpp:90 */
done:
  bnd_free(&cur); bnd_free(&q); bnd_free(&k); bnd_free(&v); bnd_free(&sc); bnd_free(&scl);
  bnd_free(&e); bnd_free(&s); bnd_free(&r); bnd_free(&pr); bnd_free(&ctx); bnd_free(&attn);
  bnd_free(&res1); bnd_free(&f1); bnd_free(&act); bnd_free(&f2); bnd_free(&sum);
  bnd_free(&pooled); bnd_free(&logits);
  return st;
}

int fo_bound_pass(const fo_config* c, const double* params, const double* x,
                  const int* positions, int words, int norm, double eps, double* logits_lo,
                  double* logits_hi, double* node_lo, double* node_hi) {
  return bound_pass(c, params, x, positions, words, norm, eps, logits_lo, logits_hi, node_lo,
                    node_hi, 0);
}

int fo_bound_pass_prefix(const fo_config* c, const double* params, const double* x,
                         const int* positions, int words, int norm, double eps, int max_nodes) {
  double lo[64], hi[64];
  if (c->classes > 64) return FO_EINVAL;
  return bound_pass(c, params, x, positions, words, norm, eps, lo, hi, NULL, NULL, max_nodes);
}

/* cmd_maxeps (cli.cpp:135-193) on the word-level pass. */
int fo_maxeps(const fo_config* c, const double* params, const double* x, const int* positions,
              int words, int norm, double eps_max, double tol, double* eps_out, int* calls_out,
              int* predicted_out) {
  size_t C = (size_t)c->classes;
  double* logits = malloc(C * sizeof(double));
  double* lo = malloc(C * sizeof(double));
  double* hi = malloc(C * sizeof(double));
  int st = fo_forward(c, params, x, logits);
  if (st != FO_OK) goto out;
  size_t predicted = 0; /* argmax (cli.cpp:54-60) */
  for (size_t i = 1; i < C; ++i)
    if (logits[i] > logits[predicted]) predicted = i;
  *predicted_out = (int)predicted;
  int calls = 0;
  /* verified_at(eps, tolerate) (cli.cpp:144-157) */
#define VERIFIED_AT(EPS, TOL, OUT)                                                    \
  do {                                                                                \
    ++calls;                                                                          \
    int s_ = fo_bound_pass(c, params, x, positions, words, norm, (EPS), lo, hi, NULL, \
                           NULL);                                                     \
    if (s_ == FO_OK) {                                                                \
      int v_ = 0;                                                                     \
      s_ = fo_check_robust(C, lo, hi, predicted, 0.0, &v_);                           \
      if (s_ != FO_OK) { st = s_; goto out; }                                         \
      (OUT) = v_;                                                                     \
    } else if ((s_ == FO_EDOMAIN || s_ == FO_EINVAL) && (TOL)) {                      \
      (OUT) = 0;                                                                      \
    } else {                                                                          \
      st = s_;                                                                        \
      goto out;                                                                       \
    }                                                                                 \
  } while (0)
  int ok = 0;
  VERIFIED_AT(0.0, 0, ok);
  if (!ok) { /* misclassified input (cli.cpp:159-161) */
    st = FO_ERUNTIME;
    goto out;
  }
  double result;
  VERIFIED_AT(eps_max, 1, ok);
  if (ok) {
    result = eps_max;
  } else {
    double l = 0.0, h = eps_max;
    while (h - l > tol) {
      double mid = 0.5 * (l + h);
      VERIFIED_AT(mid, 1, ok);
      if (ok) l = mid;
      else h = mid;
    }
    result = l;
  }
#undef VERIFIED_AT
  *eps_out = result;
  *calls_out = calls;
out:
  free(logits); free(lo); free(hi);
  return st;
}

const char* fo_impl_name(void) { return "port"; }
