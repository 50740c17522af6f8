// fg_host.cu -- C++ host side of libfaith_gpu.so: the C ABI of include/faith_gpu.h.
//
//   * operator level: host f64 buffers in the reference layout, uploaded into the
//     device's center/radius f32 Λ planes, run through the same kernels as the
//     fused pass, downloaded back (value semantics of proj/src/relax.cpp).
//   * model level: weights uploaded once; one bound pass = the node sequence of
//     graph::evaluate over fuse_all(build_graph(spec)) (graph.cpp:531-661,
//     model.cpp:406-445) as ~11 fused kernels per layer, batched over S
//     independent sentences, captured once into a CUDA graph and replayed;
//   * drivers: certify (cli::cmd_verify, cli.cpp:64-133) and the epsilon
//     bisection (cli::cmd_maxeps, cli.cpp:135-193) with continuous batching.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <future>
#include <limits>
#include <memory>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "../../include/faith_gpu.h"
#include "fg_host.h"
#include "fg_internal.cuh"

using namespace fg;
using fgh::DBuf;
using fgh::fail;

namespace {

const char* kVersion = "faith-b200 0.2 (sm_100a)";

// Optional per-launch-site profiler (fg_profile_pass): events around each LAUNCH.
struct Profiler {
  struct Site {
    std::string tag;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
    int kernels = 0;
  };
  std::vector<Site> sites;
  cudaStream_t st = nullptr;
  Site& site(const char* tag) {
    for (auto& x : sites)
      if (x.tag == tag) return x;
    sites.push_back(Site{tag, {}, 0});
    return sites.back();
  }
};
thread_local Profiler* g_prof = nullptr;
thread_local const char* g_tag = "other";

struct ProfScope {
  Profiler::Site* site = nullptr;
  cudaEvent_t b = nullptr, e = nullptr;
  ProfScope() {
    if (!g_prof) return;
    site = &g_prof->site(g_tag);
    cudaEventCreate(&b);
    cudaEventCreate(&e);
    cudaEventRecord(b, g_prof->st);
  }
  void done(int kernels) {
    if (!site) return;
    cudaEventRecord(e, g_prof->st);
    site->ev.emplace_back(b, e);
    site->kernels += kernels;
  }
};

#define LAUNCH(expr)                                                     \
  do {                                                                   \
    ProfScope ps_;                                                       \
    int n_ = (expr);                                                     \
    ps_.done(n_);                                                        \
    if (n_ < 0) return fail(ctx, FG_EINVAL, "unsupported shape: " #expr); \
    ctx->launches += (uint64_t)n_;                                       \
    cudaError_t e_ = cudaGetLastError();                                 \
    if (e_ != cudaSuccess)                                               \
      return fail(ctx, FG_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

inline int round4(size_t d) { return (int)((d + 3) / 4 * 4); }

fg_status decode_status(int v) {
  if (v == kStatusClear) return FG_OK;
  int code = v & 15;
  return code == kCodeInval ? FG_EINVAL : FG_EDOMAIN;
}

// Device-resident bound tensor for the operator-level API: n neurons, padded D.
struct OpBounds {
  DBuf lam, lb, ub;
  long long n = 0;
  int d = 0, Dp = 0;
  long long cr() const { return n * (long long)Dp; }
  float* c() const { return lam.as<float>(); }
};

fg_status op_alloc(fg_ctx* ctx, OpBounds& b, long long n, int d) {
  b.n = n;
  b.d = d;
  b.Dp = round4(d > 0 ? d : 1);
  CK(b.lam.alloc(sizeof(float) * 2 * (size_t)n * b.Dp));
  CK(b.lb.alloc(sizeof(double) * (size_t)n));
  CK(b.ub.alloc(sizeof(double) * (size_t)n));
  return FG_OK;
}

fg_status op_upload(fg_ctx* ctx, OpBounds& b, long long n, int d, const double* lw, const double* lb,
                    const double* uw, const double* ub) {
  fg_status s = op_alloc(ctx, b, n, d);
  if (s) return s;
  DBuf tl, tu;
  size_t nd = (size_t)n * d;
  CK(tl.alloc(sizeof(double) * nd));
  CK(tu.alloc(sizeof(double) * nd));
  if (nd) {
    CK(cudaMemcpyAsync(tl.p, lw, sizeof(double) * nd, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(tu.p, uw, sizeof(double) * nd, cudaMemcpyHostToDevice, ctx->stream));
  }
  CK(cudaMemcpyAsync(b.lb.p, lb, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(b.ub.p, ub, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  LAUNCH(launch_ul_to_cr(tl.as<double>(), tu.as<double>(), b.c(), b.cr(), n, d, b.Dp, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return FG_OK;
}

fg_status op_download(fg_ctx* ctx, const OpBounds& b, double* lw, double* lb, double* uw, double* ub) {
  DBuf tl, tu;
  size_t nd = (size_t)b.n * b.d;
  CK(tl.alloc(sizeof(double) * nd));
  CK(tu.alloc(sizeof(double) * nd));
  LAUNCH(launch_cr_to_ul(b.c(), b.cr(), tl.as<double>(), tu.as<double>(), b.n, b.d, b.Dp, ctx->stream));
  if (nd) {
    CK(cudaMemcpyAsync(lw, tl.p, sizeof(double) * nd, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(uw, tu.p, sizeof(double) * nd, cudaMemcpyDeviceToHost, ctx->stream));
  }
  CK(cudaMemcpyAsync(lb, b.lb.p, sizeof(double) * b.n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(ub, b.ub.p, sizeof(double) * b.n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return FG_OK;
}

struct DevScalar {  // eps + status for operator-level calls (one "sentence")
  DBuf eps, status;
};

fg_status op_scalar(fg_ctx* ctx, DevScalar& s, double eps) {
  CK(s.eps.alloc(sizeof(double)));
  CK(s.status.alloc(sizeof(int)));
  CK(cudaMemcpyAsync(s.eps.p, &eps, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  LAUNCH(launch_fill_int(s.status.as<int>(), kStatusClear, 1, ctx->stream));
  return FG_OK;
}

fg_status op_status(fg_ctx* ctx, DevScalar& s) {
  int v = 0;
  CK(cudaMemcpyAsync(&v, s.status.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  fg_status st = decode_status(v);
  if (st == FG_EINVAL) return fail(ctx, st, "invalid_argument: concretized lo > hi");
  if (st == FG_EDOMAIN) return fail(ctx, st, "domain_error: relaxation domain / overflow");
  return FG_OK;
}

bool eps_ok(double eps) { return eps >= 0.0 && std::isfinite(eps); }  // bounds.cpp:38-44

// Weights of one affine layer on the device: W and |W| as f32 [C][O] (M-major
// GEMM A operand: A[m=j, k=i] = W[i*O + j]), W as f64 for the bias path, bias f64.
struct alignas(64) TensorMap {
  unsigned char bytes[128];
};

// Round to the nearest TF32 value (ties away from zero), as cvt.rna.tf32.f32.
float tf32_rna(float x) {
  uint32_t b;
  std::memcpy(&b, &x, 4);
  if ((b & 0x7f800000u) != 0x7f800000u) {
    b += 0x1000u;
    b &= 0xffffe000u;
  }
  std::memcpy(&x, &b, 4);
  return x;
}

struct DevAffine {
  DBuf w32, w64, b64;
  DBuf a_hi, a_lo;        // [2][O][C] f32: (W^T, |W|^T) split for 3xTF32 (tcgen05 path)
  TensorMap tm_hi, tm_lo;
  TensorMap tm2_hi, tm2_lo;  // box height bn/2: one CTA's half of a W tile (CTA-pair kernel)
  TensorMap tmA_hi, tmA_lo;  // box height 128: the N tile of the TMEM-operand engine
  bool umma = false, umma2 = false, ummaA = false;
  int bn = 0;
  int C = 0, O = 0;
};

fg_status upload_affine(fg_ctx* ctx, DevAffine& a, int C, int O, const std::vector<double>& w,
                        const double* bias) {
  a.C = C;
  a.O = O;
  std::vector<float> w32(2 * (size_t)C * O);
  for (size_t i = 0; i < (size_t)C * O; ++i) {
    w32[i] = (float)w[i];
    w32[(size_t)C * O + i] = std::fabs((float)w[i]);
  }
  CK(a.w32.alloc(sizeof(float) * w32.size()));
  CK(a.w64.alloc(sizeof(double) * w.size()));
  CK(a.b64.alloc(sizeof(double) * O));
  CK(cudaMemcpy(a.w32.p, w32.data(), sizeof(float) * w32.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(a.w64.p, w.data(), sizeof(double) * w.size(), cudaMemcpyHostToDevice));
  if (bias) {
    CK(cudaMemcpy(a.b64.p, bias, sizeof(double) * O, cudaMemcpyHostToDevice));
  } else {
    CK(cudaMemset(a.b64.p, 0, sizeof(double) * O));
  }
  // tcgen05 operands: transposed (K-major) and split into TF32 hi/lo parts once.
  a.bn = umma_pick_bn(O);
  if (const char* e = std::getenv("FG_AFFINE_BN")) {  // tuning knob: N tile of the affine GEMM
    const int want = std::atoi(e);
    if (want >= 32 && want <= a.bn && O % want == 0) a.bn = want;
  }
  if (umma_available() && a.bn > 0 && C % 32 == 0) {
    std::vector<float> hi(2 * (size_t)C * O), lo(2 * (size_t)C * O);
    for (int plane = 0; plane < 2; ++plane)
      for (int j = 0; j < O; ++j)
        for (int i = 0; i < C; ++i) {
          float v = w32[(size_t)plane * C * O + (size_t)i * O + j];
          float h = tf32_rna(v);
          size_t o = (size_t)plane * O * C + (size_t)j * C + i;
          hi[o] = h;
          lo[o] = v - h;
        }
    CK(a.a_hi.alloc(sizeof(float) * hi.size()));
    CK(a.a_lo.alloc(sizeof(float) * lo.size()));
    CK(cudaMemcpy(a.a_hi.p, hi.data(), sizeof(float) * hi.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(a.a_lo.p, lo.data(), sizeof(float) * lo.size(), cudaMemcpyHostToDevice));
    a.umma = umma_tmap_wop(a.tm_hi.bytes, a.a_hi.as<float>(), C, O, 2, 1, a.bn) &&
             umma_tmap_wop(a.tm_lo.bytes, a.a_lo.as<float>(), C, O, 2, 1, a.bn);
    a.umma2 = a.umma && a.bn >= 64 && umma_tmap_wop(a.tm2_hi.bytes, a.a_hi.as<float>(), C, O, 2, 1, a.bn / 2) &&
              umma_tmap_wop(a.tm2_lo.bytes, a.a_lo.as<float>(), C, O, 2, 1, a.bn / 2);
    a.ummaA = a.umma && O % 128 == 0 && umma_tmap_wop(a.tmA_hi.bytes, a.a_hi.as<float>(), C, O, 2, 1, 128) &&
              umma_tmap_wop(a.tmA_lo.bytes, a.a_lo.as<float>(), C, O, 2, 1, 128);
  }
  return FG_OK;
}

GemmArgs affine_gemm(const DevAffine& a, const float* in, long long in_cr, float* out, long long out_cr,
                     const float* res, long long res_cr, long long nrows, int D);

bool umma_enabled() {
  const char* e = std::getenv("FG_NO_UMMA");
  return !(e && e[0] == '1');
}
bool umma_dots_enabled() {
  const char* e = std::getenv("FG_NO_UMMA_DOTS");
  return umma_enabled() && !(e && e[0] == '1');
}
bool umma_affine_enabled() {
  const char* e = std::getenv("FG_NO_UMMA_AFFINE");
  return umma_enabled() && !(e && e[0] == '1');
}
// affine GEMMs with the split Λ operand in tensor memory (LamGemm::tmem_a, N tile 128):
// FG_AFFINE_TMEM_A=1.  Off by default: measured 8 % slower than the shared-memory engine at N tile
// 256, whose two 256-column accumulators leave no tensor memory for operand stages.
bool affine_tmem_a_enabled() {
  const char* e = std::getenv("FG_AFFINE_TMEM_A");
  return e && e[0] == '1';
}
// McCormick GEMMs with the split Λ operand in tensor memory (FG_DOTS_TMEM_A=0: shared memory)
bool dots_tmem_a_enabled() {
  const char* e = std::getenv("FG_DOTS_TMEM_A");
  return !(e && e[0] == '0');
}

// Λ bound GEMM of one affine over `rows` token rows: tcgen05 3xTF32 when the shape and
// the input tensor map allow it, the FP32 SIMT kernel otherwise.
// tcgen05 descriptor of the affine: batch (token row, plane); Λ map (d, C, rows, 2).
// mean relative shortening of a tcgen05 f32 accumulation per accumulating MMA, units of 2^-24
constexpr double kTruncCentre = 0.30, kTruncRadius = 0.45;

LamGemm affine_lam(const DevAffine& a, float* out, long long out_cr, const float* res, long long res_cr,
                   long long rows, int D) {
  LamGemm g{};
  g.M = D; g.N = a.O; g.K = a.C; g.K0 = a.C;
  g.nb[0] = (int)rows; g.nb[1] = 2; g.nb[2] = 1; g.nb[3] = 1;
  if (D == 64) g.fold1 = 1;  // two token rows per 128-lane tile
  g.kdim = 1;
  g.lam_c[1][0] = 1;  // c2 = token row
  g.lam_c[2][1] = 1;  // c3 = plane
  g.w_c[0][1] = 1;    // weights plane: W^T (c) or |W|^T (r)
  g.out = out;
  g.out_c[0] = (long long)a.O * D; g.out_c[1] = out_cr; g.ldn_out = D;
  g.res = res;
  g.res_c[0] = (long long)a.O * D; g.res_c[1] = res_cr; g.ldn_res = D;
  // tcgen05's accumulation truncates toward zero at every MMA instruction, which shortens the
  // sums by a near-constant fraction per accumulating MMA (3 per 8-deep K step in 3xTF32):
  // measured with fg_selftest_affine (median signed relative error, K = 256..1024) 0.45 * 2^-24
  // per MMA on the radius plane (non-negative sums) and 0.30 * 2^-24 on the centre plane.  The
  // epilogue scales each plane back by its expected shortening.
  const double nmma = 3.0 * a.C / 8.0;
  g.alpha = (float)(1.0 + kTruncCentre * nmma * 0x1p-24);
  g.alpha_r_dim1 = 2;  // b[1] = plane (0 = centre, 1 = radius)
  g.alpha_r = (float)(1.0 + kTruncRadius * nmma * 0x1p-24);
  return g;
}

// whether launch_affine_lambda runs this affine on the tcgen05 engine (which honours
// LamGemm::kmask; the FP32 SIMT fallback does not)
bool affine_on_umma(const DevAffine& a, const TensorMap* tm_in, long long rows, int D) {
  return a.umma && tm_in && umma_affine_enabled() && (D % 128 == 0 || (D == 64 && rows % 2 == 0));
}

// `skip_status` (per sentence slot, rows_per_slot token rows each): tiles of slots whose pass has
// already failed are skipped (early exit, LamGemm::skip_status).  `kmask`: zero input rows
// (LamGemm::kmask; tcgen05 engine only, see affine_on_umma).
int launch_affine_lambda(const DevAffine& a, const TensorMap* tm_in, const float* in, long long in_cr,
                         float* out, long long out_cr, const float* res, long long res_cr, long long rows,
                         int D, cudaStream_t st, const int* skip_status = nullptr, int rows_per_slot = 1,
                         const unsigned char* kmask = nullptr) {
  if (affine_on_umma(a, tm_in, rows, D)) {
    LamGemm g = affine_lam(a, out, out_cr, res, res_cr, rows, D);
    g.kmask = kmask;
    g.skip_status = skip_status;
    g.skip_div = rows_per_slot;
    g.skip_slots = (int)(rows / rows_per_slot);
    if (a.ummaA && D % 128 == 0 && affine_tmem_a_enabled()) {
      g.tmem_a = 1;
      return launch_lam_gemm(tm_in->bytes, a.tmA_hi.bytes, a.tmA_lo.bytes, g, 128, st);
    }
    return launch_lam_gemm(tm_in->bytes, a.tm_hi.bytes, a.tm_lo.bytes, g, a.bn, st,
                           a.umma2 ? a.tm2_hi.bytes : nullptr, a.umma2 ? a.tm2_lo.bytes : nullptr);
  }
  return launch_gemm(affine_gemm(a, in, in_cr, out, out_cr, res, res_cr, rows, D), st);
}

bool lam_map(TensorMap& tm, const float* base, long long cr, int D, int C, long long rows, int kdim) {
  unsigned long long dims[4] = {(unsigned long long)D, (unsigned long long)C, (unsigned long long)rows, 2};
  unsigned long long strides[3] = {(unsigned long long)D * 4, (unsigned long long)C * D * 4,
                                   (unsigned long long)cr * 4};
  return umma_tmap_lam(tm.bytes, base, dims, strides, kdim);
}

// Λ GEMM of propagate_affine for `rows` token rows per sentence:
//   out_c = W^T in_c (+res_c),  out_r = |W|^T in_r (+res_r)   (see fg_internal.cuh)
GemmArgs affine_gemm(const DevAffine& a, const float* in, long long in_cr, float* out,
                     long long out_cr, const float* res, long long res_cr, long long nrows, int D) {
  GemmArgs g{};
  g.M = a.O; g.N = D; g.K = a.C; g.K0 = a.C;
  g.A = a.w32.as<float>(); g.lda = a.O;
  g.B = in; g.ldb = D; g.b_off1 = 0;
  g.C = out; g.ldc = D;
  g.R = res; g.ldr = D;
  g.alpha = 1.0f; g.accumulate = 0;
  g.nb[0] = (int)nrows; g.nb[1] = 2; g.nb[2] = 1; g.nb[3] = 1;
  g.sA[1] = (long long)a.C * a.O;
  g.sB[0] = (long long)a.C * D; g.sB[1] = in_cr;
  g.sC[0] = (long long)a.O * D; g.sC[1] = out_cr;
  g.sR[0] = (long long)a.O * D; g.sR[1] = res_cr;
  return g;
}

}  // namespace

// ============================================================================
// context
// ============================================================================
extern "C" {

const char* fg_version(void) { return kVersion; }

fg_status fg_ctx_create(int device, fg_ctx** out) {
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count <= device || device < 0)
    return FG_ECUDA;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major != 10) return FG_ECUDA;
  if (cudaSetDevice(device) != cudaSuccess) return FG_ECUDA;
  fg_ctx* ctx = new fg_ctx();
  ctx->device = device;
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return FG_ECUDA;
  }
  // The exact-mode paths allocate their f64 tensors stream-ordered from the default pool
  // (DBuf::alloc_async); the pool keeps what it has mapped across calls instead of returning
  // it to the driver at every synchronisation (re-mapping GBs per exact pass cost 100s of ms).
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  *out = ctx;
  return FG_OK;
}

void fg_ctx_destroy(fg_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

const char* fg_last_error(const fg_ctx* ctx) { return ctx ? ctx->err.c_str() : "no context"; }
uint64_t fg_kernel_launches(const fg_ctx* ctx) { return ctx ? ctx->launches : 0; }

// ============================================================================
// operator level
// ============================================================================
fg_status fg_check_robust(size_t n, const double* lo, const double* hi, size_t t, double margin,
                          int* verified) {
  if (t >= n) return FG_ERANGE;      // bounds.cpp:144-147
  if (margin < 0.0) return FG_EINVAL;  // bounds.cpp:148-150
  *verified = 1;
  for (size_t j = 0; j < n; ++j) {
    if (j == t) continue;
    if (!(lo[t] > hi[j] + margin)) {
      *verified = 0;
      break;
    }
  }
  return FG_OK;
}

fg_status fg_concretize(fg_ctx* ctx, size_t n, size_t d, const double* lw, const double* lb,
                        const double* uw, const double* ub, int norm, double eps, double* lo,
                        double* hi) {
  if (!eps_ok(eps)) return fail(ctx, FG_EINVAL, "PerturbationSpec: epsilon must be finite and >= 0");
  cudaSetDevice(ctx->device);
  if (ctx->precision == FG_PRECISION_F64) return fgh::x64_concretize(ctx, n, d, lw, lb, uw, ub, norm, eps, lo, hi);
  OpBounds x;
  fg_status s = op_upload(ctx, x, (long long)n, (int)d, lw, lb, uw, ub);
  if (s) return s;
  DevScalar sc;
  if ((s = op_scalar(ctx, sc, eps))) return s;
  DBuf dlo, dhi;
  CK(dlo.alloc(sizeof(double) * n));
  CK(dhi.alloc(sizeof(double) * n));
  LAUNCH(launch_concretize(x.c(), x.cr(), x.lb.as<double>(), x.ub.as<double>(), (long long)n,
                           (long long)n, x.Dp, norm, sc.eps.as<double>(), dlo.as<double>(),
                           dhi.as<double>(), ctx->stream));
  CK(cudaMemcpyAsync(lo, dlo.p, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(hi, dhi.p, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return FG_OK;
}

fg_status fg_affine(fg_ctx* ctx, size_t rows, size_t c, size_t o, size_t d, const double* xlw,
                    const double* xlb, const double* xuw, const double* xub, const double* w,
                    const double* bias, double* ylw, double* ylb, double* yuw, double* yub) {
  cudaSetDevice(ctx->device);
  if (rows == 0 || c == 0 || o == 0) return fail(ctx, FG_EINVAL, "propagate_affine: empty shape");
  if (ctx->precision == FG_PRECISION_F64)
    return fgh::x64_affine(ctx, rows, c, o, d, xlw, xlb, xuw, xub, w, bias, ylw, ylb, yuw, yub);
  OpBounds x, y;
  fg_status s = op_upload(ctx, x, (long long)(rows * c), (int)d, xlw, xlb, xuw, xub);
  if (s) return s;
  if ((s = op_alloc(ctx, y, (long long)(rows * o), (int)d))) return s;
  DevAffine a;
  std::vector<double> wv(w, w + c * o);
  if ((s = upload_affine(ctx, a, (int)c, (int)o, wv, bias))) return s;
  LAUNCH(launch_gemm(affine_gemm(a, x.c(), x.cr(), y.c(), y.cr(), nullptr, 0, (long long)rows, x.Dp),
                     ctx->stream));
  LAUNCH(launch_affine_bias(x.lb.as<double>(), x.ub.as<double>(), a.w64.as<double>(),
                            bias ? a.b64.as<double>() : nullptr, nullptr, nullptr, y.lb.as<double>(),
                            y.ub.as<double>(), 1, (int)rows, (int)c, (int)o, ctx->stream));
  return op_download(ctx, y, ylw, ylb, yuw, yub);
}

fg_status fg_relax(fg_ctx* ctx, int kind, size_t n, const double* lo, const double* hi,
                   double* a_low, double* b_low, double* a_up, double* b_up) {
  cudaSetDevice(ctx->device);
  if (kind < 0 || kind > FG_RELAX_SQUARE) return fail(ctx, FG_EINVAL, "relax: unknown kind");
  DBuf dlo, dhi, out;
  CK(dlo.alloc(sizeof(double) * n));
  CK(dhi.alloc(sizeof(double) * n));
  CK(out.alloc(sizeof(double) * 4 * n));
  CK(cudaMemcpyAsync(dlo.p, lo, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(dhi.p, hi, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  DevScalar sc;
  fg_status s = op_scalar(ctx, sc, 0.0);
  if (s) return s;
  double* o = out.as<double>();
  LAUNCH(launch_relax(kind, dlo.as<double>(), dhi.as<double>(), (long long)n, o, o + n, o + 2 * n,
                      o + 3 * n, sc.status.as<int>(), ctx->stream));
  if ((s = op_status(ctx, sc))) return s;
  std::vector<double> h(4 * n);
  CK(cudaMemcpy(h.data(), out.p, sizeof(double) * 4 * n, cudaMemcpyDeviceToHost));
  std::memcpy(a_low, h.data(), sizeof(double) * n);
  std::memcpy(b_low, h.data() + n, sizeof(double) * n);
  std::memcpy(a_up, h.data() + 2 * n, sizeof(double) * n);
  std::memcpy(b_up, h.data() + 3 * n, sizeof(double) * n);
  return FG_OK;
}

fg_status fg_compose(fg_ctx* ctx, size_t n, size_t d, const double* xlw, const double* xlb,
                     const double* xuw, const double* xub, const double* a_low,
                     const double* b_low, const double* a_up, const double* b_up, double* ylw,
                     double* ylb, double* yuw, double* yub) {
  cudaSetDevice(ctx->device);
  if (ctx->precision == FG_PRECISION_F64)
    return fgh::x64_compose(ctx, n, d, xlw, xlb, xuw, xub, a_low, b_low, a_up, b_up, ylw, ylb, yuw, yub);
  OpBounds x, y;
  fg_status s = op_upload(ctx, x, (long long)n, (int)d, xlw, xlb, xuw, xub);
  if (s) return s;
  if ((s = op_alloc(ctx, y, (long long)n, (int)d))) return s;
  DBuf rel;
  CK(rel.alloc(sizeof(double) * 4 * n));
  double* r = rel.as<double>();
  CK(cudaMemcpyAsync(r, a_low, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(r + n, b_low, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(r + 2 * n, a_up, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(r + 3 * n, b_up, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  LAUNCH(launch_compose(x.c(), x.cr(), x.lb.as<double>(), x.ub.as<double>(), r, r + n, r + 2 * n,
                        r + 3 * n, y.c(), y.cr(), y.lb.as<double>(), y.ub.as<double>(), (long long)n,
                        x.Dp, ctx->stream));
  return op_download(ctx, y, ylw, ylb, yuw, yub);
}

fg_status fg_elementwise_verify(fg_ctx* ctx, int kind, size_t n, size_t d, const double* xlw,
                                const double* xlb, const double* xuw, const double* xub,
                                int norm, double eps, double* ylw, double* ylb, double* yuw,
                                double* yub) {
  if (!eps_ok(eps)) return fail(ctx, FG_EINVAL, "PerturbationSpec: epsilon must be finite and >= 0");
  cudaSetDevice(ctx->device);
  if (kind < 0 || kind > FG_RELAX_SQUARE) return fail(ctx, FG_EINVAL, "elementwise_verify: unknown kind");
  if (ctx->precision == FG_PRECISION_F64)
    return fgh::x64_elementwise_verify(ctx, kind, n, d, xlw, xlb, xuw, xub, norm, eps, ylw, ylb, yuw, yub);
  OpBounds x;
  fg_status s = op_upload(ctx, x, (long long)n, (int)d, xlw, xlb, xuw, xub);
  if (s) return s;
  DevScalar sc;
  if ((s = op_scalar(ctx, sc, eps))) return s;
  LAUNCH(launch_elementwise_verify(kind, x.c(), x.cr(), x.lb.as<double>(), x.ub.as<double>(),
                                   (long long)n, (long long)n, x.Dp, norm, sc.eps.as<double>(),
                                   sc.status.as<int>(), 0, nullptr, nullptr, ctx->stream));
  if ((s = op_status(ctx, sc))) return s;
  return op_download(ctx, x, ylw, ylb, yuw, yub);
}

fg_status fg_dot(fg_ctx* ctx, int layout, size_t len, size_t embed, size_t heads, size_t d,
                 const double* alw, const double* alb, const double* auw, const double* aub,
                 const double* blw, const double* blb, const double* buw, const double* bub,
                 int norm, double eps, double* ylw, double* ylb, double* yuw, double* yub) {
  if (!eps_ok(eps)) return fail(ctx, FG_EINVAL, "PerturbationSpec: epsilon must be finite and >= 0");
  if (heads == 0 || embed % heads != 0)
    return fail(ctx, FG_EINVAL, "propagate_dot_product: feature dim not divisible by heads");
  cudaSetDevice(ctx->device);
  if (ctx->precision == FG_PRECISION_F64)
    return fgh::x64_dot(ctx, layout, 1, len, embed, heads, d, alw, alb, auw, aub, blw, blb, buw, bub, norm, eps,
                        ylw, ylb, yuw, yub);
  const int L = (int)len, E = (int)embed, H = (int)heads, hd = E / H;
  const bool sim = layout == FG_DOT_SIMILARITY;
  long long na = sim ? (long long)L * E : (long long)H * L * L;
  long long nb = (long long)L * E;
  long long ny = sim ? (long long)H * L * L : (long long)L * E;
  OpBounds a, b, y;
  fg_status s = op_upload(ctx, a, na, (int)d, alw, alb, auw, aub);
  if (s) return s;
  if ((s = op_upload(ctx, b, nb, (int)d, blw, blb, buw, bub))) return s;
  if ((s = op_alloc(ctx, y, ny, (int)d))) return s;
  DevScalar sc;
  if ((s = op_scalar(ctx, sc, eps))) return s;
  DBuf alo, ahi, blo, bhi, ws;
  CK(alo.alloc(sizeof(double) * na));
  CK(ahi.alloc(sizeof(double) * na));
  CK(blo.alloc(sizeof(double) * nb));
  CK(bhi.alloc(sizeof(double) * nb));
  size_t wsz = sim ? 6ull * hd * L * H : (4ull * L * hd + 2ull * L * L) * H;
  CK(ws.alloc(sizeof(float) * wsz));
  const int Dp = a.Dp;
  LAUNCH(launch_concretize(a.c(), a.cr(), a.lb.as<double>(), a.ub.as<double>(), na, na, Dp, norm,
                           sc.eps.as<double>(), alo.as<double>(), ahi.as<double>(), ctx->stream));
  LAUNCH(launch_concretize(b.c(), b.cr(), b.lb.as<double>(), b.ub.as<double>(), nb, nb, Dp, norm,
                           sc.eps.as<double>(), blo.as<double>(), bhi.as<double>(), ctx->stream));
  NView va{a.c(), a.cr(), a.lb.as<double>(), a.ub.as<double>(), alo.as<double>(), ahi.as<double>(),
           na, sim ? E : L, 0};
  NView vb{b.c(), b.cr(), b.lb.as<double>(), b.ub.as<double>(), blo.as<double>(), bhi.as<double>(),
           nb, E, 0};
  NView vy{y.c(), y.cr(), y.lb.as<double>(), y.ub.as<double>(), nullptr, nullptr, ny,
           sim ? L : E, 0};
  if (sim) {
    LAUNCH(launch_dot_similarity(va, vb, vy, 1, L, H, hd, Dp, ws.as<float>(), 1.0f, ctx->stream));
  } else {
    LAUNCH(launch_dot_weighted(va, vb, vy, 1, L, H, hd, Dp, ws.as<float>(), ctx->stream));
  }
  return op_download(ctx, y, ylw, ylb, yuw, yub);
}

fg_status fg_softmax(fg_ctx* ctx, size_t rows, size_t n, size_t d, const double* xlw,
                     const double* xlb, const double* xuw, const double* xub, int norm,
                     double eps, double* ylw, double* ylb, double* yuw, double* yub) {
  if (!eps_ok(eps)) return fail(ctx, FG_EINVAL, "PerturbationSpec: epsilon must be finite and >= 0");
  cudaSetDevice(ctx->device);
  if (ctx->precision == FG_PRECISION_F64)
    return fgh::x64_softmax(ctx, rows, n, 1, d, xlw, xlb, xuw, xub, norm, eps, ylw, ylb, yuw, yub);
  OpBounds x;
  long long N = (long long)(rows * n);
  fg_status s = op_upload(ctx, x, N, (int)d, xlw, xlb, xuw, xub);
  if (s) return s;
  DevScalar sc;
  if ((s = op_scalar(ctx, sc, eps))) return s;
  DBuf lo, hi;
  CK(lo.alloc(sizeof(double) * N));
  CK(hi.alloc(sizeof(double) * N));
  NView v{x.c(), x.cr(), x.lb.as<double>(), x.ub.as<double>(), lo.as<double>(), hi.as<double>(), N,
          (int)n, 0};
  LAUNCH(launch_softmax(v, 1, (int)rows, (int)n, x.Dp, norm, sc.eps.as<double>(),
                        sc.status.as<int>(), 0, 1, ctx->stream));
  if ((s = op_status(ctx, sc))) return s;
  return op_download(ctx, x, ylw, ylb, yuw, yub);
}

fg_status fg_add(fg_ctx* ctx, size_t n, size_t d, const double* alw, const double* alb,
                 const double* auw, const double* aub, const double* blw, const double* blb,
                 const double* buw, const double* bub, double* ylw, double* ylb, double* yuw,
                 double* yub) {
  cudaSetDevice(ctx->device);
  if (ctx->precision == FG_PRECISION_F64)
    return fgh::x64_add(ctx, n, d, alw, alb, auw, aub, blw, blb, buw, bub, ylw, ylb, yuw, yub);
  OpBounds a, b, y;
  fg_status s = op_upload(ctx, a, (long long)n, (int)d, alw, alb, auw, aub);
  if (s) return s;
  if ((s = op_upload(ctx, b, (long long)n, (int)d, blw, blb, buw, bub))) return s;
  if ((s = op_alloc(ctx, y, (long long)n, (int)d))) return s;
  LAUNCH(launch_add(a.c(), a.cr(), a.lb.as<double>(), a.ub.as<double>(), b.c(), b.cr(),
                    b.lb.as<double>(), b.ub.as<double>(), y.c(), y.cr(), y.lb.as<double>(),
                    y.ub.as<double>(), (long long)n, a.Dp, ctx->stream));
  return op_download(ctx, y, ylw, ylb, yuw, yub);
}

fg_status fg_scale(fg_ctx* ctx, size_t n, size_t d, const double* xlw, const double* xlb,
                   const double* xuw, const double* xub, double sv, double* ylw, double* ylb,
                   double* yuw, double* yub) {
  cudaSetDevice(ctx->device);
  if (ctx->precision == FG_PRECISION_F64) return fgh::x64_scale(ctx, n, d, xlw, xlb, xuw, xub, sv, ylw, ylb, yuw, yub);
  OpBounds x, y;
  fg_status s = op_upload(ctx, x, (long long)n, (int)d, xlw, xlb, xuw, xub);
  if (s) return s;
  if ((s = op_alloc(ctx, y, (long long)n, (int)d))) return s;
  LAUNCH(launch_scale(x.c(), x.cr(), x.lb.as<double>(), x.ub.as<double>(), sv, y.c(), y.cr(),
                      y.lb.as<double>(), y.ub.as<double>(), (long long)n, x.Dp, ctx->stream));
  return op_download(ctx, y, ylw, ylb, yuw, yub);
}

fg_status fg_dot_batched(fg_ctx* ctx, int layout, size_t batch, size_t len, size_t embed, size_t heads,
                         size_t d, const double* alw, const double* alb, const double* auw, const double* aub,
                         const double* blw, const double* blb, const double* buw, const double* bub, int norm,
                         double eps, double* ylw, double* ylb, double* yuw, double* yub) {
  if (!eps_ok(eps)) return fail(ctx, FG_EINVAL, "PerturbationSpec: epsilon must be finite and >= 0");
  if (heads == 0 || embed % heads != 0)
    return fail(ctx, FG_EINVAL, "propagate_dot_product: feature dim not divisible by heads");
  cudaSetDevice(ctx->device);
  if (ctx->precision == FG_PRECISION_F64)
    return fgh::x64_dot(ctx, layout, batch, len, embed, heads, d, alw, alb, auw, aub, blw, blb, buw, bub, norm,
                        eps, ylw, ylb, yuw, yub);
  const bool sim = layout == FG_DOT_SIMILARITY;
  const size_t na = sim ? len * embed : heads * len * len, nb = len * embed;
  const size_t ny = sim ? heads * len * len : len * embed;
  for (size_t bi = 0; bi < batch; ++bi) {  // batch slices are independent problems
    fg_status s = fg_dot(ctx, layout, len, embed, heads, d, alw + bi * na * d, alb + bi * na, auw + bi * na * d,
                         aub + bi * na, blw + bi * nb * d, blb + bi * nb, buw + bi * nb * d, bub + bi * nb, norm,
                         eps, ylw + bi * ny * d, ylb + bi * ny, yuw + bi * ny * d, yub + bi * ny);
    if (s) return s;
  }
  return FG_OK;
}

fg_status fg_softmax_axis(fg_ctx* ctx, size_t outer, size_t n, size_t inner, size_t d, const double* xlw,
                          const double* xlb, const double* xuw, const double* xub, int norm, double eps,
                          double* ylw, double* ylb, double* yuw, double* yub) {
  if (!eps_ok(eps)) return fail(ctx, FG_EINVAL, "PerturbationSpec: epsilon must be finite and >= 0");
  cudaSetDevice(ctx->device);
  if (inner == 1 && ctx->precision == FG_PRECISION_F32)
    return fg_softmax(ctx, outer, n, d, xlw, xlb, xuw, xub, norm, eps, ylw, ylb, yuw, yub);
  return fgh::x64_softmax(ctx, outer, n, inner, d, xlw, xlb, xuw, xub, norm, eps, ylw, ylb, yuw, yub);
}

}  // extern "C"

// ============================================================================
// model level
// ============================================================================
namespace {

struct DevLayer {
  DevAffine qkv, wo, w1, w2;
};

// Pass workspace for S resident sentences.
struct Workspace {
  int S = 0, D = 0, W = 0, Ntot = 0;  // slots, pert dim, words, sentences uploaded
  DBuf X, R1, QF, SC, CTX;            // Λ planes (f32)
  TensorMap tm_X, tm_R1, tm_CTX, tm_F;  // tcgen05 input maps of the four affine inputs
  bool tm_ok = false;
  // tcgen05 McCormick dot products: Λ maps of the operands, split coefficient buffers + maps
  TensorMap tm_QKVk, tm_QKVrow, tm_SC;
  DBuf cf_sim_x[2], cf_sim_y[2], cf_wv_x[2], cf_wv_y[2];  // [hi, lo]
  TensorMap tm_sim_x[2], tm_sim_y[2], tm_wv_x[2], tm_wv_y[2];
  TensorMap tm2_sim_x[2], tm2_sim_y[2], tm2_wv_x[2], tm2_wv_y[2];  // half-height boxes (CTA pairs)
  bool dots2_ok = false;
  int bn_sim = 0, bn_simx = 0, bn_wvx = 0;
  bool dots_ok = false;
  bool fold64 = false;  // D = 64: the McCormick GEMMs fold pairs of query tokens / keys / head features
  int kp = 0;            // head dimension rounded up to the GEMM engine's 32-deep K steps
  long long crX = 0, crQKV = 0, crF = 0, crSC = 0;
  DBuf X_b, R1_b, QKV_b, SC_b, CTX_b, F_b;  // f64 lb/ub(/lo/hi) blocks
  DBuf keepF;  // per FFN row (s, t, f): 0 = Λ row zero after the activation (LamGemm::kmask of W2)
  DBuf pooled, pooled_b, coef;
  DBuf eps, status, logits, slot_map, x_all, pos_all;
  DBuf active;  // per slot: 1 = holds a probe this pass, 0 = idle (status kStatusIdle, skipped)
  DBuf dump_lo, dump_hi;
  // column-sharded pass: concretization partials and the softmax chain's phase buffers
  int col0 = 0;
  DBuf part, sm_ex, sm_sig, sm_rows, head_part;
  double* h_eps = nullptr;  // pinned
  int* h_slot = nullptr;
  int* h_active = nullptr;  // all 1 outside fg_maxeps
  double* h_logits = nullptr;
  int* h_status = nullptr;
  // captured passes: [0] plain, [1] with early exit (the GEMMs skip slots that already failed)
  cudaGraphExec_t graph[2] = {nullptr, nullptr};
  int graph_norm[2] = {-1, -1};
  uint64_t graph_launches[2] = {0, 0};
  ~Workspace() { release_host(); }
  void release_host() {
    for (auto& g : graph) {
      if (g) cudaGraphExecDestroy(g);
      g = nullptr;
    }
    if (h_eps) cudaFreeHost(h_eps);
    if (h_slot) cudaFreeHost(h_slot);
    if (h_active) cudaFreeHost(h_active);
    if (h_logits) cudaFreeHost(h_logits);
    if (h_status) cudaFreeHost(h_status);
    h_eps = nullptr;
    h_slot = nullptr;
    h_active = nullptr;
    h_logits = nullptr;
    h_status = nullptr;
  }
};

size_t bytes_per_sentence(const fg_config& c, int D) {
  size_t L = c.length, E = c.embed, F = c.ffn, H = c.heads;
  size_t lam = 2 * sizeof(float) * D;
  size_t qf = std::max(3 * E, F);
  size_t n_tok = L * E;
  size_t total = lam * (n_tok * 3 + L * qf + H * L * L)  // X, R1, CTX, QKV/F, SC
                 + sizeof(double) * (2 * n_tok * 3 + 4 * L * 3 * E + 4 * H * L * L + 2 * L * F) +
                 2 * sizeof(double) * E * D + sizeof(float) * H * (6 * (E / H) * L + 2 * L * L);
  return total;
}

}  // namespace

struct fg_model {
  fg_ctx* ctx = nullptr;
  fg_config cfg{};
  std::vector<double> params;
  std::vector<DevLayer> layers;
  DBuf wc64, bc64;
  Workspace ws;
  std::unique_ptr<Workspace> ws0;  // ε = 0 probe workspace (narrow, all-zero Λ; fg_maxeps)
  fg_run_stats stats{};
  fgh::ShardState shard;  // column sharding of the perturbation dimension (fg_model_set_column_shard)
  DBuf params64;          // f64 weights on the device for the exact pass (uploaded on first use)
  double kappa = FG_DEFAULT_KAPPA;  // ambiguity band of the decision-exact verdicts (outer limit)
  // per-model calibrated band [band_lo, band_hi] (units of the widths W), from the measured
  // (m_f32 - m_exact) / W of this model's own re-decided probes (see ambiguous_verdict)
  double band_lo = -FG_DEFAULT_KAPPA, band_hi = FG_DEFAULT_KAPPA / 8;
  double err_min = 0.0, err_max = 0.0;
  int err_samples = 0;
  int speculate = FG_SPECULATE_PREDICTED;  // fg_maxeps while a re-decision runs (fg_model_set_speculation)
  int exact_probes = 0;   // per call: probes re-decided by the exact pass, and their time
  double exact_ms = 0.0;
  // asynchronous re-decisions (fg_maxeps): a low-priority side stream and reusable jobs
  static constexpr int kExactStreams = 4;  // concurrent re-decisions (one exact pass fills ~half the FP64 pipe)
  cudaStream_t exact_stream[kExactStreams] = {};
  int exact_rr = 0;
  std::vector<std::unique_ptr<fgh::ExactJob>> jobs;
  ~fg_model() {
    for (auto& j : jobs) {
      if (j->host) cudaFreeHost(j->host);
      if (j->hstat) cudaFreeHost(j->hstat);
      if (j->start) cudaEventDestroy(j->start);
      if (j->done) cudaEventDestroy(j->done);
    }
    for (cudaStream_t st : exact_stream)
      if (st) cudaStreamDestroy(st);
  }
  // offsets of the layers in params (gen_synthetic order)
  size_t layer_off(int l) const {
    size_t e = cfg.embed, f = cfg.ffn;
    return (size_t)l * (4 * (e * e + e) + e * f + f + f * e + e);
  }
};

namespace {

// `zero_d` > 0 plans the ε = 0 probe workspace instead (fg_maxeps): zero_d columns that lie
// past every perturbation column (col0 = W·E), so Λ0 — and with it every Λ of the pass — is
// zero and each concretization reduces to its bias, exactly what ε·‖Λ‖ = 0 gives at full width.
fg_status ensure_workspace(fg_model* m, int S, int W, int Ntot, Workspace* wsp = nullptr, int zero_d = 0) {
  fg_ctx* ctx = m->ctx;
  Workspace& w = wsp ? *wsp : m->ws;
  const fg_config& c = m->cfg;
  const int Dg = W * c.embed;  // global perturbation columns
  const int nr = m->shard.active() ? m->shard.nranks : 1;
  if (Dg % (4 * nr) != 0) return fail(ctx, FG_EINVAL, "column shard: words*embed must be a multiple of 4*nranks");
  const int D = zero_d > 0 ? zero_d : Dg / nr;  // columns of this rank
  if (w.S == S && w.D == D && w.W == W && w.Ntot >= Ntot) return FG_OK;
  w.col0 = zero_d > 0 ? Dg : (m->shard.active() ? m->shard.rank : 0) * D;
  w.release_host();
  const long long L = c.length, E = c.embed, F = c.ffn, H = c.heads, hd = E / H;
  const long long nX = S * L * E, nQKV = S * L * 3 * E, nF = S * L * F, nSC = S * H * L * L;
  w.crX = nX * D;
  w.crQKV = nQKV * D;
  w.crF = nF * D;
  w.crSC = nSC * D;
  CK(w.X.alloc(sizeof(float) * 2 * w.crX));
  CK(w.R1.alloc(sizeof(float) * 2 * w.crX));
  CK(w.CTX.alloc(sizeof(float) * 2 * w.crX));
  CK(w.QF.alloc(sizeof(float) * 2 * std::max(w.crQKV, w.crF)));
  CK(w.SC.alloc(sizeof(float) * 2 * w.crSC));
  CK(w.X_b.alloc(sizeof(double) * 2 * nX));
  CK(w.R1_b.alloc(sizeof(double) * 2 * nX));
  CK(w.CTX_b.alloc(sizeof(double) * 4 * nX));
  CK(w.QKV_b.alloc(sizeof(double) * 4 * nQKV));
  CK(w.F_b.alloc(sizeof(double) * 4 * nF));
  CK(w.keepF.alloc((size_t)nF));
  CK(w.SC_b.alloc(sizeof(double) * 4 * nSC));
  CK(w.pooled.alloc(sizeof(double) * 2 * S * E * D));
  CK(w.pooled_b.alloc(sizeof(double) * 4 * S * E));
  CK(w.coef.alloc(sizeof(float) * S * H * std::max(6 * hd * L, 4 * L * hd + 2 * L * L)));
  CK(w.eps.alloc(sizeof(double) * S));
  CK(w.status.alloc(sizeof(int) * S));
  CK(w.logits.alloc(sizeof(double) * 2 * S * c.classes));
  CK(w.slot_map.alloc(sizeof(int) * S));
  CK(w.active.alloc(sizeof(int) * S));
  CK(w.x_all.alloc(sizeof(double) * (size_t)std::max(Ntot, 1) * L * E));
  CK(w.pos_all.alloc(sizeof(int) * (size_t)std::max(Ntot, 1) * W));
  size_t dmax = std::max({(size_t)nQKV, (size_t)nF, (size_t)nSC});
  CK(w.dump_lo.alloc(sizeof(double) * dmax));
  CK(w.dump_hi.alloc(sizeof(double) * dmax));
  if (m->shard.active()) {
    const long long rows = (long long)S * H * L;
    CK(w.part.alloc(sizeof(double) * 2 * std::max({nQKV, nF, nSC})));
    CK(w.sm_ex.alloc(sizeof(double) * 5 * nSC));
    CK(w.sm_sig.alloc(sizeof(double) * 2 * rows * D));
    CK(w.sm_rows.alloc(sizeof(double) * 14 * rows));  // p_row, p_row2, sb (2 each), rb (6)
    CK(w.head_part.alloc(sizeof(double) * 4 * S * c.classes));
  }
  CK(cudaMallocHost(&w.h_eps, sizeof(double) * S));
  CK(cudaMallocHost(&w.h_slot, sizeof(int) * S));
  CK(cudaMallocHost(&w.h_active, sizeof(int) * S));
  std::fill(w.h_active, w.h_active + S, 1);
  CK(cudaMemcpy(w.active.p, w.h_active, sizeof(int) * S, cudaMemcpyHostToDevice));
  CK(cudaMallocHost(&w.h_logits, sizeof(double) * 2 * S * c.classes));
  CK(cudaMallocHost(&w.h_status, sizeof(int) * S));
  w.S = S;
  w.D = D;
  w.W = W;
  w.Ntot = Ntot;
  const long long rows = (long long)S * L;
  // tcgen05 needs 128 TMEM lanes of perturbation columns: D % 128 == 0, or D = 64 with token
  // rows folded in pairs (affine GEMMs only; the McCormick GEMMs' folded coordinates are
  // gathered in layer 1, so they keep the FP32 SIMT path at D = 64)
  const bool dok = umma_available() && (D % 128 == 0 || (D == 64 && rows % 2 == 0));
  w.tm_ok = dok && lam_map(w.tm_X, w.X.as<float>(), w.crX, D, (int)E, rows, 1) &&
            lam_map(w.tm_R1, w.R1.as<float>(), w.crX, D, (int)E, rows, 1) &&
            lam_map(w.tm_CTX, w.CTX.as<float>(), w.crX, D, (int)E, rows, 1) &&
            lam_map(w.tm_F, w.QF.as<float>(), w.crF, D, (int)F, rows, 1);
  // McCormick dot products on tcgen05 (shapes: K multiples of 32, N multiples of 32)
  w.bn_sim = umma_pick_bn((int)L);       // y-side GEMMs: N = L
  w.bn_simx = umma_pick_bn((int)(2 * L)); // Q.K^T x-side: both output planes in N = 2L
  w.bn_wvx = umma_pick_bn((int)(2 * hd)); // P.V x-side: N = 2hd
  w.dots_ok = false;
  w.fold64 = false;
  // head dimension padded to whole K steps (zero coefficients: c1's hd = 16 contracts over 32)
  w.kp = (int)((hd + 31) / 32 * 32);
  // D = 64 (c1) folds pairs of a batch coordinate into the 128 TMEM lanes, which a gathered
  // coordinate cannot provide (one perturbed word), so the layer-1 products run dense there
  const bool fold = D == 64;
  if (w.tm_ok && (D % 128 == 0 || fold) && w.bn_sim > 0 && w.bn_simx > 0 && w.bn_wvx > 0 && L % 32 == 0 &&
      (!fold || (L % 2 == 0 && hd % 2 == 0))) {
    const long long SH = (long long)S * H;
    bool ok = lam_map(w.tm_QKVk, w.QF.as<float>(), w.crQKV, D, (int)(3 * E), rows, 1) &&
              lam_map(w.tm_QKVrow, w.QF.as<float>(), w.crQKV, D, (int)(3 * E), rows, 2) &&
              lam_map(w.tm_SC, w.SC.as<float>(), w.crSC, D, (int)L, SH * L, 1);
    for (int part = 0; part < 2 && ok; ++part) {
      CK(w.cf_sim_x[part].alloc(sizeof(float) * SH * 2 * L * 2 * w.kp));
      CK(w.cf_sim_y[part].alloc(sizeof(float) * SH * 2 * L * w.kp));
      CK(w.cf_wv_x[part].alloc(sizeof(float) * SH * 2 * hd * 2 * L));
      CK(w.cf_wv_y[part].alloc(sizeof(float) * SH * 2 * L * L));
      // x-side coefficient arrays [SH][2 planes][rows][K] are read as [SH][2*rows][K]
      ok = ok && umma_tmap_wop(w.tm_sim_x[part].bytes, w.cf_sim_x[part].as<float>(), 2 * w.kp, (int)(2 * L), 1, (int)SH, w.bn_simx) &&
           umma_tmap_wop(w.tm_sim_y[part].bytes, w.cf_sim_y[part].as<float>(), w.kp, (int)L, 2, (int)SH, w.bn_sim) &&
           umma_tmap_wop(w.tm_wv_x[part].bytes, w.cf_wv_x[part].as<float>(), (int)(2 * L), (int)(2 * hd), 1, (int)SH, w.bn_wvx) &&
           umma_tmap_wop(w.tm_wv_y[part].bytes, w.cf_wv_y[part].as<float>(), (int)L, (int)L, 2, (int)SH, w.bn_sim);
    }
    w.dots_ok = ok;
    w.fold64 = ok && fold;
    bool ok2 = w.dots_ok && !fold && w.bn_sim >= 64 && w.bn_simx >= 64 && w.bn_wvx >= 64;
    for (int part = 0; part < 2 && ok2; ++part)
      ok2 = umma_tmap_wop(w.tm2_sim_x[part].bytes, w.cf_sim_x[part].as<float>(), 2 * w.kp, (int)(2 * L), 1, (int)SH, w.bn_simx / 2) &&
            umma_tmap_wop(w.tm2_sim_y[part].bytes, w.cf_sim_y[part].as<float>(), w.kp, (int)L, 2, (int)SH, w.bn_sim / 2) &&
            umma_tmap_wop(w.tm2_wv_x[part].bytes, w.cf_wv_x[part].as<float>(), (int)(2 * L), (int)(2 * hd), 1, (int)SH, w.bn_wvx / 2) &&
            umma_tmap_wop(w.tm2_wv_y[part].bytes, w.cf_wv_y[part].as<float>(), (int)L, (int)L, 2, (int)SH, w.bn_sim / 2);
    w.dots2_ok = ok2;
  }
  return FG_OK;
}

// Host-side dump helper (S = 1 debug pass): copies device lo/hi into node slots.
struct Dumper {
  double* lo = nullptr;
  double* hi = nullptr;
  fg_ctx* ctx = nullptr;
  fg_status copy(size_t off, const double* dlo, const double* dhi, size_t n, size_t src_stride = 1,
                 size_t src_cols = 0, size_t src_col0 = 0, size_t rows = 0) {
    if (!lo) return FG_OK;
    std::vector<double> a, b;
    size_t total = src_cols ? rows * src_stride : n;
    a.resize(total);
    b.resize(total);
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaMemcpy(a.data(), dlo, sizeof(double) * total, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(b.data(), dhi, sizeof(double) * total, cudaMemcpyDeviceToHost));
    if (!src_cols) {
      std::memcpy(lo + off, a.data(), sizeof(double) * n);
      std::memcpy(hi + off, b.data(), sizeof(double) * n);
    } else {  // strided slice: rows x src_cols starting at src_col0 of each src_stride row
      for (size_t r = 0; r < rows; ++r)
        for (size_t k = 0; k < src_cols; ++k) {
          lo[off + r * src_cols + k] = a[r * src_stride + src_col0 + k];
          hi[off + r * src_cols + k] = b[r * src_stride + src_col0 + k];
        }
    }
    return FG_OK;
  }
};

bool no_qk_skip() {  // comparison runs: write the layer-1 Q/K zero rows as well
  static const bool v = std::getenv("FG_ONEHOT_DENSE_QK") != nullptr;
  return v;
}

bool onehot_first_layer() {
  const char* e = std::getenv("FG_NO_ONEHOT");
  return !(e && e[0] == '1');
}

// All-reduce of concretization partials across the column shards (stream-ordered).
fg_status shard_allreduce(fg_model* m, double* buf, size_t count, int norm) {
  fg_ctx* ctx = m->ctx;
  if (m->shard.nranks <= 1 && !m->shard.fn) return FG_OK;
  const int op = reduce_op_for_norm(norm) ? FG_REDUCE_MAX : FG_REDUCE_SUM;
  if (m->shard.fn(m->shard.user, buf, count, op, (void*)ctx->stream) != 0)
    return fail(ctx, FG_ECUDA, "column shard: all-reduce failed");
  ++ctx->launches;
  return FG_OK;
}

// Concretization of `nrows` rows of a Λ: fused kernel when unsharded; partial norms ->
// all-reduce -> finish when the perturbation columns are sharded.
fg_status concretize_site(fg_model* m, const float* lam, long long cr, const double* lb, const double* ub,
                          long long rows_per_s, long long nrows, int D, int norm, const double* eps, double* lo,
                          double* hi, const int* skip = nullptr) {
  fg_ctx* ctx = m->ctx;
  cudaStream_t st = ctx->stream;
  if (!m->shard.active()) {
    LAUNCH(launch_concretize(lam, cr, lb, ub, rows_per_s, nrows, D, norm, eps, lo, hi, st, skip));
    return FG_OK;
  }
  double* part = m->ws.part.as<double>();
  LAUNCH(launch_partial_norms(lam, cr, nrows, D, norm, part, st));
  if (fg_status s = shard_allreduce(m, part, 2 * (size_t)nrows, norm)) return s;
  LAUNCH(launch_finish_concretize(part, lb, ub, rows_per_s, nrows, norm, eps, lo, hi, st));
  return FG_OK;
}

// One batched bound pass over the resident slots (graph.cpp:531-673 node order).
// Reads ws.eps / ws.slot_map; writes ws.logits / ws.status.
fg_status enqueue_pass(fg_model* m, int norm, Dumper* dump, Workspace* wsp = nullptr, bool early_exit = false) {
  fg_ctx* ctx = m->ctx;
  Workspace& w = wsp ? *wsp : m->ws;
  const fg_config& c = m->cfg;
  const int S = w.S, D = w.D, L = c.length, E = c.embed, F = c.ffn, H = c.heads, hd = E / H;
  const int C = c.classes;
  cudaStream_t st = ctx->stream;
  const long long nX = (long long)S * L * E, nQKV = (long long)S * L * 3 * E,
                  nF = (long long)S * L * F, nSC = (long long)S * H * L * L;
  float* X = w.X.as<float>();
  float* R1 = w.R1.as<float>();
  float* QKV = w.QF.as<float>();
  float* Fl = w.QF.as<float>();
  float* SC = w.SC.as<float>();
  float* CTX = w.CTX.as<float>();
  double *X_lb = w.X_b.as<double>(), *X_ub = X_lb + nX;
  double *R1_lb = w.R1_b.as<double>(), *R1_ub = R1_lb + nX;
  double *CTX_lb = w.CTX_b.as<double>(), *CTX_ub = CTX_lb + nX, *CTX_lo = CTX_ub + nX,
         *CTX_hi = CTX_lo + nX;
  double *Q_lb = w.QKV_b.as<double>(), *Q_ub = Q_lb + nQKV, *Q_lo = Q_ub + nQKV, *Q_hi = Q_lo + nQKV;
  double *F_lb = w.F_b.as<double>(), *F_ub = F_lb + nF, *F_lo = F_ub + nF, *F_hi = F_lo + nF;
  double *S_lb = w.SC_b.as<double>(), *S_ub = S_lb + nSC, *S_lo = S_ub + nSC, *S_hi = S_lo + nSC;
  double* eps = w.eps.as<double>();
  int* status = w.status.as<int>();
  // early exit: the GEMMs skip the tiles of slots whose pass already failed (a per-tile test
  // that costs ~5 % of the GEMMs, so it is only on when a pass is expected to carry failures)
  const int* skip = early_exit ? status : nullptr;
  double* dlo = w.dump_lo.as<double>();
  double* dhi = w.dump_hi.as<double>();
  const size_t per_layer = 8ull * L * E + 4ull * H * L * L + 2ull * H * L + 2ull * L * F;
  auto site = [](int l, int k) { return l * 8 + k; };

  g_tag = "init";
  LAUNCH(launch_init_status(status, w.active.as<int>(), S, st));
  // Λ0 is one-hot: the first layer consumes it analytically (no Λ0 in HBM) unless dumping
  const bool onehot = !dump && onehot_first_layer();
  LAUNCH(launch_init_input(onehot ? nullptr : X, w.crX, X_lb, X_ub, w.x_all.as<double>(), w.pos_all.as<int>(),
                           w.slot_map.as<int>(), S, L, E, w.W, st, D, w.col0));
  const bool sharded = m->shard.active();
  for (int l = 0; l < c.layers; ++l) {
    const DevLayer& lw = m->layers[l];
    const size_t base = (size_t)l * per_layer;
    // Q, K, V = propagate_affine(cur, Wq|Wk|Wv)   (one N=3E affine)
    g_tag = "affine_gemm";
    if (l == 0 && onehot) {
      // Q/K rows at unperturbed tokens are never read in layer 1 on the gathered tcgen05 path
      const bool gathered = !sharded && w.dots_ok && !w.fold64 && umma_dots_enabled() && !no_qk_skip();
      LAUNCH(launch_onehot_affine(QKV, w.crQKV, lw.qkv.w32.as<float>(), w.pos_all.as<int>(), w.slot_map.as<int>(), S,
                                  L, E, 3 * E, w.W, D, w.col0, st, gathered ? 2 * E : 0));
    } else {
      LAUNCH(launch_affine_lambda(lw.qkv, w.tm_ok ? &w.tm_X : nullptr, X, w.crX, QKV, w.crQKV, nullptr, 0,
                                  (long long)S * L, D, st, skip, L));
    }
    g_tag = "affine_bias";
    LAUNCH(launch_affine_bias(X_lb, X_ub, lw.qkv.w64.as<double>(), lw.qkv.b64.as<double>(), nullptr,
                              nullptr, Q_lb, Q_ub, S, L, E, 3 * E, st, skip));
    g_tag = "concretize";
    // first layer under the one-hot binding: Q/K/V Λ rows are zero outside the perturbed tokens
    const bool sparse0 = l == 0 && onehot && !sharded;
    if (sparse0) {
      LAUNCH(launch_concretize_tokens(QKV, w.crQKV, Q_lb, Q_ub, (long long)L * 3 * E, nQKV, D, norm, eps, Q_lo, Q_hi,
                                      w.pos_all.as<int>(), w.slot_map.as<int>(), w.W, 3 * E, st));
    } else if (fg_status s = concretize_site(m, QKV, w.crQKV, Q_lb, Q_ub, (long long)L * 3 * E, nQKV, D, norm,
                                             eps, Q_lo, Q_hi, skip)) {
      return s;
    }
    if (dump) {
      for (int t = 0; t < 3; ++t)
        if (fg_status s = dump->copy(base + (size_t)t * L * E, Q_lo, Q_hi, 0, 3 * E, E, (size_t)t * E, L)) return s;
    }
    NView q{QKV, w.crQKV, Q_lb, Q_ub, Q_lo, Q_hi, (long long)L * 3 * E, 3 * E, 0};
    NView k = q, v = q;
    k.col0 = E;
    v.col0 = 2 * E;
    NView sc{SC, w.crSC, S_lb, S_ub, S_lo, S_hi, (long long)H * L * L, L, 0};
    // scores = DotProduct(q, k); scaled = Scale(scores, 1/sqrt(hd))   (model.cpp:410-418)
    const double scale = 1.0 / std::sqrt((double)hd);
    g_tag = "dot_similarity";
    if (w.dots_ok && umma_dots_enabled()) {
      LAUNCH(launch_sim_coef_split(q, k, S, H, L, hd, w.kp, w.cf_sim_x[0].as<float>(), w.cf_sim_x[1].as<float>(),
                                   w.cf_sim_y[0].as<float>(), w.cf_sim_y[1].as<float>(), st));
      LAUNCH(launch_sim_bias(q, k, sc, S, H, L, hd, scale, st));
      // x-side: scores[s,h,i,j,:] = sum_k2 Cx[j,k2] (Qc|Qr)[i, h*hd + k2]   (K0 = hd: c|r concat)
      // (both output planes in one N = 2L range: n -> plane n / L, key j = n % L)
      LamGemm gx{};
      gx.M = D; gx.N = 2 * L; gx.K = 2 * w.kp; gx.K0 = w.kp;
      gx.nb[0] = S; gx.nb[1] = H; gx.nb[2] = L; gx.nb[3] = 1;
      gx.kdim = 1;
      gx.lam_c[0][1] = hd;                    // neuron h*hd (+k)
      gx.lam_c[1][0] = L; gx.lam_c[1][2] = 1;  // row s*L + i
      gx.w_c[1][0] = H; gx.w_c[1][1] = 1;      // (s, h)
      gx.out = SC;
      gx.out_c[0] = (long long)H * L * L * D; gx.out_c[1] = (long long)L * L * D; gx.out_c[2] = (long long)L * D;
      gx.ldn_out = D;
      gx.n_split = L; gx.split_stride = w.crSC;
      gx.alpha = (float)scale;
      gx.skip_status = sharded ? nullptr : skip;  // b[0] = sentence slot
      gx.skip_div = 1;
      gx.skip_slots = S;
      if (w.fold64) gx.fold1 = 3;  // pairs of query tokens i
      if (l == 0 && onehot && !w.fold64) {
        // Q/K Λ rows vanish off the perturbed tokens: scores Λ[i, j] != 0 only for i or j
        // perturbed -> zero the scores, x-side terms for perturbed queries i, y-side terms for
        // perturbed keys j (gathered batch coordinate)
        CK(cudaMemsetAsync(SC, 0, sizeof(float) * 2 * w.crSC, st));
        gx.nb[2] = w.W;
        gx.gather = w.pos_all.as<int>();
        gx.gather_slot = w.slot_map.as<int>();
        gx.gather_ld = w.W;
      }
      gx.tmem_a = dots_tmem_a_enabled();
      LAUNCH(launch_lam_gemm(w.tm_QKVk.bytes, w.tm_sim_x[0].bytes, w.tm_sim_x[1].bytes, gx, w.bn_simx, st,
                             w.dots2_ok ? w.tm2_sim_x[0].bytes : nullptr, w.dots2_ok ? w.tm2_sim_x[1].bytes : nullptr));
      // y-side: scores[s,h,i,j,:] += sum_k lx[i,k] K_p[j, E + h*hd + k]   (per plane p)
      LamGemm gy{};
      gy.M = D; gy.N = L; gy.K = w.kp; gy.K0 = w.kp;
      gy.nb[0] = S; gy.nb[1] = H; gy.nb[2] = L; gy.nb[3] = 2;
      gy.kdim = 1;
      gy.lam_c[0][1] = hd; gy.lam_c[0][4] = E;
      gy.lam_c[1][0] = L; gy.lam_c[1][2] = 1;
      gy.lam_c[2][3] = 1;
      gy.w_c[0][3] = 1;
      gy.w_c[1][0] = H; gy.w_c[1][1] = 1;
      gy.out = SC;
      gy.out_c[0] = (long long)H * L * L * D; gy.out_c[1] = (long long)L * L * D; gy.out_c[2] = D;
      gy.out_c[3] = w.crSC; gy.ldn_out = (long long)L * D;
      gy.alpha = (float)scale;
      gy.accumulate = 1;
      gy.skip_status = sharded ? nullptr : skip;
      gy.skip_div = 1;
      gy.skip_slots = S;
      if (w.fold64) gy.fold1 = 3;  // pairs of keys j
      if (l == 0 && onehot && !w.fold64) {
        gy.nb[2] = w.W;
        gy.gather = w.pos_all.as<int>();
        gy.gather_slot = w.slot_map.as<int>();
        gy.gather_ld = w.W;
      }
      gy.tmem_a = dots_tmem_a_enabled();
      LAUNCH(launch_lam_gemm(w.tm_QKVk.bytes, w.tm_sim_y[0].bytes, w.tm_sim_y[1].bytes, gy, w.bn_sim, st,
                             w.dots2_ok ? w.tm2_sim_y[0].bytes : nullptr, w.dots2_ok ? w.tm2_sim_y[1].bytes : nullptr));
    } else {
      LAUNCH(launch_dot_similarity(q, k, sc, S, L, H, hd, D, w.coef.as<float>(), (float)scale, st));
    }
    if (dump) {
      LAUNCH(launch_concretize(SC, w.crSC, S_lb, S_ub, (long long)H * L * L, nSC, D, norm, eps, dlo, dhi, st));
      if (fg_status s = dump->copy(base + 3ull * L * E + (size_t)H * L * L, dlo, dhi, (size_t)H * L * L)) return s;
    }
    // softmax: exp -> sum -> recip -> mul (graph.cpp:237-240), in place
    g_tag = "softmax";
    if (!sharded) {
      LAUNCH(launch_softmax(sc, S, H * L, L, D, norm, eps, status, site(l, 0), site(l, 1), st));
    } else {  // exp -> sum -> recip -> multiply around four all-reduces of the partial norms
      const long long rows = (long long)S * H * L;
      double* pr = w.sm_rows.as<double>();
      SmShardBufs b{w.part.as<double>(), pr, pr + 2 * rows, w.sm_ex.as<double>(), w.sm_sig.as<double>(),
                    pr + 4 * rows, pr + 6 * rows};
      const size_t counts[4] = {2 * (size_t)nSC, 2 * (size_t)rows, 2 * (size_t)rows, 2 * (size_t)nSC};
      double* bufs[4] = {b.p_key, b.p_row, b.p_row2, b.p_key};
      for (int ph = 0; ph < 5; ++ph) {
        LAUNCH(launch_sm_shard(ph, sc, S, H * L, L, D, norm, eps, status, site(l, 0), site(l, 1), b, st));
        if (ph < 4)
          if (fg_status s = shard_allreduce(m, bufs[ph], counts[ph], norm)) return s;
      }
    }
    if (dump) {
      if (fg_status s = dump->copy(base + 3ull * L * E + 3ull * H * L * L + 2ull * H * L, S_lo, S_hi,
                                   (size_t)H * L * L)) return s;
    }
    // ctx = DotProduct(probs, v)
    NView cx{CTX, w.crX, CTX_lb, CTX_ub, nullptr, nullptr, (long long)L * E, E, 0};
    g_tag = "dot_weighted";
    if (w.dots_ok && umma_dots_enabled()) {
      LAUNCH(launch_wv_coef_split(sc, v, S, H, L, hd, w.cf_wv_x[0].as<float>(), w.cf_wv_x[1].as<float>(),
                                  w.cf_wv_y[0].as<float>(), w.cf_wv_y[1].as<float>(), st));
      LAUNCH(launch_wv_bias(sc, v, cx, S, H, L, hd, st));
      // x-side: ctx[s,i,h*hd+k,:] = sum_j2 Cx[k,j2] (Pc|Pr)[s,h,i,j2]   (K0 = L: c|r concat)
      // (both output planes in one N = 2hd range: n -> plane n / hd, k = n % hd)
      LamGemm gx{};
      gx.M = D; gx.N = 2 * hd; gx.K = 2 * L; gx.K0 = L;
      gx.nb[0] = S; gx.nb[1] = H; gx.nb[2] = L; gx.nb[3] = 1;
      gx.kdim = 1;
      gx.lam_c[1][0] = H * L; gx.lam_c[1][1] = L; gx.lam_c[1][2] = 1;  // score row (s, h, i)
      gx.w_c[1][0] = H; gx.w_c[1][1] = 1;
      gx.out = CTX;
      gx.out_c[0] = (long long)L * E * D; gx.out_c[1] = (long long)hd * D; gx.out_c[2] = (long long)E * D;
      gx.ldn_out = D;
      gx.n_split = hd; gx.split_stride = w.crX;
      gx.alpha = 1.0f;
      gx.skip_status = sharded ? nullptr : skip;
      gx.skip_div = 1;
      gx.skip_slots = S;
      if (w.fold64) gx.fold1 = 3;  // pairs of query tokens i
      gx.tmem_a = dots_tmem_a_enabled();
      LAUNCH(launch_lam_gemm(w.tm_SC.bytes, w.tm_wv_x[0].bytes, w.tm_wv_x[1].bytes, gx, w.bn_wvx, st,
                             w.dots2_ok ? w.tm2_wv_x[0].bytes : nullptr, w.dots2_ok ? w.tm2_wv_x[1].bytes : nullptr));
      // y-side: ctx[s,i,h*hd+k,:] += sum_j lx[i,j] V_p[j, 2E + h*hd + k]   (K along token rows)
      LamGemm gy{};
      gy.M = D; gy.N = L; gy.K = L; gy.K0 = L;
      gy.nb[0] = S; gy.nb[1] = H; gy.nb[2] = hd; gy.nb[3] = 2;
      gy.kdim = 2;
      gy.lam_c[0][1] = hd; gy.lam_c[0][2] = 1; gy.lam_c[0][4] = 2 * E;  // neuron 2E + h*hd + k
      gy.lam_c[1][0] = L;                                               // row s*L (+ j)
      gy.lam_c[2][3] = 1;
      gy.w_c[0][3] = 1;
      gy.w_c[1][0] = H; gy.w_c[1][1] = 1;
      gy.out = CTX;
      gy.out_c[0] = (long long)L * E * D; gy.out_c[1] = (long long)hd * D; gy.out_c[2] = D;
      gy.out_c[3] = w.crX; gy.ldn_out = (long long)E * D;
      gy.alpha = 1.0f;
      gy.accumulate = 1;
      gy.skip_status = sharded ? nullptr : skip;
      gy.skip_div = 1;
      gy.skip_slots = S;
      if (w.fold64) gy.fold1 = 3;  // pairs of head features k
      gy.tmem_a = dots_tmem_a_enabled();
      LAUNCH(launch_lam_gemm(w.tm_QKVrow.bytes, w.tm_wv_y[0].bytes, w.tm_wv_y[1].bytes, gy, w.bn_sim, st,
                             w.dots2_ok ? w.tm2_wv_y[0].bytes : nullptr, w.dots2_ok ? w.tm2_wv_y[1].bytes : nullptr));
    } else {
      LAUNCH(launch_dot_weighted(sc, v, cx, S, L, H, hd, D, w.coef.as<float>(), st));
    }
    const size_t off_ctx = 3ull * L * E + 4ull * H * L * L + 2ull * H * L;
    if (dump) {
      LAUNCH(launch_concretize(CTX, w.crX, CTX_lb, CTX_ub, (long long)L * E, nX, D, norm, eps, CTX_lo, CTX_hi, st));
      if (fg_status s = dump->copy(base + off_ctx, CTX_lo, CTX_hi, (size_t)L * E)) return s;
    }
    // res1 = cur + affine(ctx, Wo)
    g_tag = "affine_gemm";
    const bool res0 = l == 0 && onehot;  // the Λ0 residual is a +1 scatter instead of a read
    LAUNCH(launch_affine_lambda(lw.wo, w.tm_ok ? &w.tm_CTX : nullptr, CTX, w.crX, R1, w.crX, res0 ? nullptr : X,
                                res0 ? 0 : w.crX, (long long)S * L, D, st, skip, L));
    if (res0) LAUNCH(launch_add_onehot(R1, w.pos_all.as<int>(), w.slot_map.as<int>(), S, L, E, w.W, D, w.col0, st));
    g_tag = "affine_bias";
    LAUNCH(launch_affine_bias(CTX_lb, CTX_ub, lw.wo.w64.as<double>(), lw.wo.b64.as<double>(), X_lb, X_ub,
                              R1_lb, R1_ub, S, L, E, E, st, skip));
    if (dump) {
      LAUNCH(launch_concretize(R1, w.crX, R1_lb, R1_ub, (long long)L * E, nX, D, norm, eps, dlo, dhi, st));
      if (fg_status s = dump->copy(base + off_ctx + 2ull * L * E, dlo, dhi, (size_t)L * E)) return s;
    }
    // f1 = affine(res1, W1); act = ReluVerify/TanhVerify/SiluVerify(f1)
    g_tag = "affine_gemm";
    LAUNCH(launch_affine_lambda(lw.w1, w.tm_ok ? &w.tm_R1 : nullptr, R1, w.crX, Fl, w.crF, nullptr, 0,
                                (long long)S * L, D, st, skip, L));
    g_tag = "affine_bias";
    LAUNCH(launch_affine_bias(R1_lb, R1_ub, lw.w1.w64.as<double>(), lw.w1.b64.as<double>(), nullptr,
                              nullptr, F_lb, F_ub, S, L, E, F, st, skip));
    g_tag = "act_verify";
    // W2 on the tcgen05 engine takes the activation's zero rows as a mask, so the verify kernel
    // leaves rows that the relaxation keeps or zeroes as they are (the dump re-reads Λ_F: no mask)
    unsigned char* keepF =
        (!sharded && !dump && affine_on_umma(lw.w2, w.tm_ok ? &w.tm_F : nullptr, (long long)S * L, D))
            ? w.keepF.as<unsigned char>() : nullptr;
    if (!sharded) {
      LAUNCH(launch_elementwise_verify(c.activation, Fl, w.crF, F_lb, F_ub, (long long)L * F, nF, D, norm,
                                       eps, status, site(l, 2), dump ? F_lo : nullptr,
                                       dump ? F_hi : nullptr, st, nullptr, nullptr, skip, keepF));
    } else {
      if (fg_status s = concretize_site(m, Fl, w.crF, F_lb, F_ub, (long long)L * F, nF, D, norm, eps, F_lo, F_hi))
        return s;
      LAUNCH(launch_elementwise_verify(c.activation, Fl, w.crF, F_lb, F_ub, (long long)L * F, nF, D, norm, eps,
                                       status, site(l, 2), nullptr, nullptr, st, F_lo, F_hi));
    }
    const size_t off_f1 = off_ctx + 3ull * L * E;
    if (dump) {
      if (fg_status s = dump->copy(base + off_f1, F_lo, F_hi, (size_t)L * F)) return s;
      LAUNCH(launch_concretize(Fl, w.crF, F_lb, F_ub, (long long)L * F, nF, D, norm, eps, F_lo, F_hi, st));
      if (fg_status s = dump->copy(base + off_f1 + (size_t)L * F, F_lo, F_hi, (size_t)L * F)) return s;
    }
    // cur = res1 + affine(act, W2)
    g_tag = "affine_gemm";
    LAUNCH(launch_affine_lambda(lw.w2, w.tm_ok ? &w.tm_F : nullptr, Fl, w.crF, X, w.crX, R1, w.crX,
                                (long long)S * L, D, st, skip, L, keepF));
    g_tag = "affine_bias";
    LAUNCH(launch_affine_bias(F_lb, F_ub, lw.w2.w64.as<double>(), lw.w2.b64.as<double>(), R1_lb, R1_ub,
                              X_lb, X_ub, S, L, F, E, st, skip));
    if (dump) {
      LAUNCH(launch_concretize(X, w.crX, X_lb, X_ub, (long long)L * E, nX, D, norm, eps, dlo, dhi, st));
      if (fg_status s = dump->copy(base + off_f1 + 2ull * L * F + (size_t)L * E, dlo, dhi, (size_t)L * E)) return s;
    }
  }
  // MeanPool + classifier head + final concretization (graph.cpp:628-634, 663-671; cli.cpp:90)
  double* pc = w.pooled.as<double>();
  double* pr = pc + (long long)S * E * D;
  double* plb = w.pooled_b.as<double>();
  double* pub = plb + (long long)S * E;
  double* plo = pub + (long long)S * E;
  double* phi = plo + (long long)S * E;
  g_tag = "head";
  LAUNCH(launch_meanpool(X, w.crX, X_lb, X_ub, pc, pr, plb, pub, S, L, E, D, st));
  double* lg = w.logits.as<double>();
  if (!sharded) {
    LAUNCH(launch_head(pc, pr, plb, pub, m->wc64.as<double>(), m->bc64.as<double>(), S, E, C, D, norm,
                       eps, lg, lg + (long long)S * C, status, c.layers * 8, dump ? plo : nullptr,
                       dump ? phi : nullptr, st));
  } else {
    double* hp = w.head_part.as<double>();
    LAUNCH(launch_head_partial(pc, pr, plb, pub, m->wc64.as<double>(), m->bc64.as<double>(), S, E, C, D, norm, hp,
                               hp + 2 * S * C, st));
    if (fg_status s = shard_allreduce(m, hp, 2 * (size_t)S * C, norm)) return s;
    LAUNCH(launch_head_finish(hp, hp + 2 * S * C, S, C, norm, eps, lg, lg + (long long)S * C, status,
                              c.layers * 8, st));
  }
  if (dump) {
    size_t off = (size_t)c.layers * per_layer;
    if (fg_status s = dump->copy(off, plo, phi, (size_t)E)) return s;
    if (fg_status s = dump->copy(off + E, lg, lg + C, (size_t)C)) return s;
  }
  return FG_OK;
}

bool use_graphs() {
  const char* e = std::getenv("FG_NO_GRAPH");
  return !(e && e[0] == '1');
}

// Runs one pass over all slots; eps/slot_map must be staged in the pinned host
// buffers.  Results land in w.h_logits / w.h_status after the call returns.
fg_status run_pass(fg_model* m, int norm, cudaEvent_t ev0, cudaEvent_t ev1, float* ms, Workspace* wsp = nullptr,
                   bool early_exit = false) {
  fg_ctx* ctx = m->ctx;
  Workspace& w = wsp ? *wsp : m->ws;
  cudaStream_t st = ctx->stream;
  const int S = w.S, C = m->cfg.classes;
  CK(cudaMemcpyAsync(w.eps.p, w.h_eps, sizeof(double) * S, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(w.slot_map.p, w.h_slot, sizeof(int) * S, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(w.active.p, w.h_active, sizeof(int) * S, cudaMemcpyHostToDevice, st));
  if (ev0) CK(cudaEventRecord(ev0, st));
  if (use_graphs() && m->shard.capturable) {
    const int gi = early_exit ? 1 : 0;
    if (!w.graph[gi] || w.graph_norm[gi] != norm) {
      if (w.graph[gi]) cudaGraphExecDestroy(w.graph[gi]);
      w.graph[gi] = nullptr;
      cudaGraph_t g;
      uint64_t before = ctx->launches;
      CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      fg_status s = enqueue_pass(m, norm, nullptr, &w, early_exit);
      cudaError_t ce = cudaStreamEndCapture(st, &g);
      if (s) return s;
      if (ce != cudaSuccess) return fail(ctx, FG_ECUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
      CK(cudaGraphInstantiate(&w.graph[gi], g, 0));
      cudaGraphDestroy(g);
      w.graph_norm[gi] = norm;
      w.graph_launches[gi] = ctx->launches - before;
      ctx->launches = before;
    }
    CK(cudaGraphLaunch(w.graph[gi], st));
    ctx->launches += w.graph_launches[gi];
  } else {
    fg_status s = enqueue_pass(m, norm, nullptr, &w, early_exit);
    if (s) return s;
  }
  if (ev1) CK(cudaEventRecord(ev1, st));
  CK(cudaMemcpyAsync(w.h_logits, w.logits.p, sizeof(double) * 2 * S * C, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(w.h_status, w.status.p, sizeof(int) * S, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (ev0 && ev1 && ms) CK(cudaEventElapsedTime(ms, ev0, ev1));
  return FG_OK;
}

fg_status stage_inputs(fg_model* m, int S, const double* x, const int* positions, int words) {
  fg_ctx* ctx = m->ctx;
  const fg_config& c = m->cfg;
  for (int s = 0; s < S; ++s)
    for (int wd = 0; wd < words; ++wd) {
      int p = positions[(size_t)s * words + wd];
      if (p < 0 || p >= c.length) return fail(ctx, FG_EINVAL, "word position out of range");
      for (int u = 0; u < wd; ++u)
        if (positions[(size_t)s * words + u] == p) return fail(ctx, FG_EINVAL, "duplicate word position");
    }
  Workspace& w = m->ws;
  CK(cudaMemcpyAsync(w.x_all.p, x, sizeof(double) * (size_t)S * c.length * c.embed,
                     cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(w.pos_all.p, positions, sizeof(int) * (size_t)S * words, cudaMemcpyHostToDevice,
                     ctx->stream));
  return FG_OK;
}

// Exact f64 forward pass (model.cpp:470-564): dense layers, softmax attention,
// residuals, mean pool, linear head.  Same loop order as the reference.
void forward_host(const fg_config& c, const double* p, const double* x, double* logits) {
  const size_t L = c.length, E = c.embed, F = c.ffn, H = c.heads, hd = E / H, C = c.classes;
  auto dense = [](const std::vector<double>& in, size_t rows, size_t ci, size_t o, const double* w,
                  const double* b, std::vector<double>& out) {
    out.assign(rows * o, 0.0);
    for (size_t r = 0; r < rows; ++r) {
      for (size_t i = 0; i < ci; ++i) {
        double xv = in[r * ci + i];
        const double* wr = w + i * o;
        double* orow = out.data() + r * o;
        for (size_t j = 0; j < o; ++j) orow[j] += xv * wr[j];
      }
      for (size_t j = 0; j < o; ++j) out[r * o + j] += b[j];
    }
  };
  std::vector<double> cur(x, x + L * E), q, k, v, sc(H * L * L), ctx, attn, ffn;
  const double inv = 1.0 / std::sqrt((double)hd);
  const double* pp = p;
  for (int l = 0; l < c.layers; ++l) {
    const double *wq = pp, *bq = wq + E * E, *wk = bq + E, *bk = wk + E * E, *wv = bk + E,
                 *bv = wv + E * E, *wo = bv + E, *bo = wo + E * E, *w1 = bo + E, *b1 = w1 + E * F,
                 *w2 = b1 + F, *b2 = w2 + F * E;
    pp = b2 + E;
    dense(cur, L, E, E, wq, bq, q);
    dense(cur, L, E, E, wk, bk, k);
    dense(cur, L, E, E, wv, bv, v);
    for (size_t h = 0; h < H; ++h)
      for (size_t i = 0; i < L; ++i) {
        for (size_t j = 0; j < L; ++j) {
          double acc = 0.0;
          for (size_t d = 0; d < hd; ++d) acc += q[i * E + h * hd + d] * k[j * E + h * hd + d];
          sc[(h * L + i) * L + j] = acc * inv;
        }
        double* row = sc.data() + (h * L + i) * L;
        double mx = row[0];
        for (size_t j = 1; j < L; ++j) mx = std::max(mx, row[j]);
        double sum = 0.0;
        for (size_t j = 0; j < L; ++j) {
          row[j] = std::exp(row[j] - mx);
          sum += row[j];
        }
        for (size_t j = 0; j < L; ++j) row[j] /= sum;
      }
    ctx.assign(L * E, 0.0);
    for (size_t h = 0; h < H; ++h)
      for (size_t i = 0; i < L; ++i)
        for (size_t j = 0; j < L; ++j) {
          double pv = sc[(h * L + i) * L + j];
          for (size_t d = 0; d < hd; ++d) ctx[i * E + h * hd + d] += pv * v[j * E + h * hd + d];
        }
    dense(ctx, L, E, E, wo, bo, attn);
    for (size_t i = 0; i < L * E; ++i) cur[i] += attn[i];
    dense(cur, L, E, F, w1, b1, ffn);
    for (double& t : ffn) {
      if (c.activation == FG_RELAX_TANH) t = std::tanh(t);
      else if (c.activation == FG_RELAX_SILU) t = t * (1.0 / (1.0 + std::exp(-t)));
      else t = t > 0.0 ? t : 0.0;
    }
    dense(ffn, L, F, E, w2, b2, attn);
    for (size_t i = 0; i < L * E; ++i) cur[i] += attn[i];
  }
  std::vector<double> pooled(E, 0.0), out;
  for (size_t i = 0; i < L; ++i)
    for (size_t d = 0; d < E; ++d) pooled[d] += cur[i * E + d];
  for (size_t d = 0; d < E; ++d) pooled[d] /= (double)L;
  dense(pooled, 1, E, C, pp, pp + E * C, out);
  std::memcpy(logits, out.data(), sizeof(double) * C);
}

std::vector<int> predict_all(const fg_model* m, int S, const double* x) {
  const fg_config& c = m->cfg;
  std::vector<int> pred(S, 0);
  unsigned nt = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), (unsigned)S));
  std::atomic<int> next{0};
  auto worker = [&] {
    std::vector<double> logits(c.classes);
    for (int s; (s = next.fetch_add(1)) < S;) {
      forward_host(c, m->params.data(), x + (size_t)s * c.length * c.embed, logits.data());
      int best = 0;  // argmax (cli.cpp:54-60)
      for (int i = 1; i < c.classes; ++i)
        if (logits[i] > logits[best]) best = i;
      pred[s] = best;
    }
  };
  std::vector<std::thread> th;
  for (unsigned t = 0; t < nt; ++t) th.emplace_back(worker);
  for (auto& t : th) t.join();
  return pred;
}

int default_slots(const fg_model* m, int S, int D) {
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  size_t per = bytes_per_sentence(m->cfg, m->shard.active() ? D / m->shard.nranks : D);
  size_t cap = (size_t)(0.8 * (double)free_b) / std::max<size_t>(per, 1);
  if (m->shard.active())  // every rank must batch identically: plan from total HBM, not free HBM
    cap = (size_t)(0.6 * (double)total_b / m->shard.ranks_per_device) / std::max<size_t>(per, 1);
  if (const char* e = std::getenv("FG_SLOTS")) cap = std::min<size_t>(cap, (size_t)std::atoi(e));
  int slots = (int)std::min<size_t>({cap, (size_t)S, (size_t)64});
  int maxb = 65535 / (2 * m->cfg.length);  // GEMM batch-grid limit
  return std::max(1, std::min(slots, maxb));
}

// ---- decision-exact verdicts (fg_model_set_exact_resolve) -----------------------------
// check_robust's strict test lo_t > hi_j + margin (bounds.cpp:142-157) is AMBIGUOUS on the f32-Λ
// pass when the margin lies within the error band of that pass, which scales with the
// Λ-derived widths W = (hi_t - lo_t) + (hi_j - lo_j) (the f32 Λ / 3xTF32 error enters every
// bound through ε·‖Λ‖ and the envelope lines built from it) plus an f64 rounding floor.  The
// band is asymmetric because the error is: measured (m_f32 - m_exact) / W over 576 probes per
// config straddling each sentence's ε* (tools/exact_margin_study.py) lies in
// [-3.0e-6, -7.5e-7] at c3, [-1.3e-6, -8.9e-7] at c2 (the truncation compensation of the
// affine GEMMs and the 2^-20 norm pad make the fused pass conservative) and +-7.7e-9 at c1
// (FP32 SIMT), so a probe is ambiguous when  -kappa * W - f <= m <= kappa / 8 * W + f
// (kappa = 6e-6: 2x the extreme).  Such a probe is re-decided by the exact pass, whose
// arithmetic is the reference's.
// The class j != t with the smallest margin and that margin / widths.
int closest_class(const double* lo, const double* hi, int C, int t, double margin, double* m_out, double* w_out) {
  int jb = -1;
  for (int j = 0; j < C; ++j) {
    if (j == t) continue;
    const double m = lo[t] - hi[j] - margin;
    if (jb < 0 || m < *m_out) {
      jb = j;
      *m_out = m;
      *w_out = (hi[t] - lo[t]) + (hi[j] - lo[j]);
    }
  }
  return jb;
}

// The exact verdict an ambiguous probe most likely gets (fg_maxeps speculates on it): every
// f32 margin corrected by the model's mean measured error (m_f32 - m_exact) / W, or before any
// calibration sample by -1e-6 (the fused pass's margins run below the exact ones).
int guess_verdict(const fg_model* m, const double* lo, const double* hi, int C, int t) {
  const double mid = m->err_samples ? 0.5 * (m->err_min + m->err_max) : -1e-6;
  for (int j = 0; j < C; ++j) {
    if (j == t) continue;
    const double w = (hi[t] - lo[t]) + (hi[j] - lo[j]);
    if (!(lo[t] - hi[j] - mid * w > 0.0)) return 0;
  }
  return 1;
}

bool ambiguous_verdict(const fg_model* m, const double* lo, const double* hi, int C, int t, double margin) {
  if (!(m->kappa > 0.0)) return false;
  for (int j = 0; j < C; ++j) {
    if (j == t) continue;
    const double mg = lo[t] - hi[j] - margin;
    const double w = (hi[t] - lo[t]) + (hi[j] - lo[j]);
    const double floor64 = 1e-11 * std::max({1.0, std::fabs(lo[t]), std::fabs(hi[j])});
    if (!(mg > m->band_hi * w + floor64) && !(mg < m->band_lo * w - floor64))
      return true;  // NaN-safe: a non-finite margin is ambiguous
  }
  return false;
}

// One re-decided probe's error sample (m_f32 - m_exact) / W.  After kCalibSamples samples the
// model's band becomes twice the observed extremes (plus 1e-7), where a verdict can flip --
// m_f32 in [min(err, 0), max(err, 0)] * W -- never wider than the default [-kappa, kappa / 8];
// later samples keep widening it if they fall outside.
constexpr int kCalibSamples = 16;
void calibrate_band(fg_model* m, const double* lo32, const double* hi32, const double* lo64, const double* hi64,
                    int C, int t) {
  double m32 = 0.0, w = 0.0;
  const int j = closest_class(lo32, hi32, C, t, 0.0, &m32, &w);
  if (j < 0 || !(w > 0.0) || !std::isfinite(m32)) return;
  const double m64 = lo64[t] - hi64[j];
  if (!std::isfinite(m64)) return;
  const double err = (m32 - m64) / w;
  m->err_min = m->err_samples ? std::min(m->err_min, err) : err;
  m->err_max = m->err_samples ? std::max(m->err_max, err) : err;
  ++m->err_samples;
  if (m->err_samples >= kCalibSamples) {
    m->band_lo = std::max(-m->kappa, 2.0 * std::min(m->err_min, 0.0) - 1e-7);
    m->band_hi = std::min(m->kappa / 8, 2.0 * std::max(m->err_max, 0.0) + 1e-7);
  }
}

fg_status upload_params64(fg_model* m) {
  fg_ctx* ctx = m->ctx;
  if (m->params64.p) return FG_OK;
  CK(m->params64.alloc(sizeof(double) * m->params.size()));
  CK(cudaMemcpy(m->params64.p, m->params.data(), sizeof(double) * m->params.size(), cudaMemcpyHostToDevice));
  const fg_config& c = m->cfg;
  const size_t ffn = (size_t)c.length * c.ffn * (size_t)c.embed * 2 * sizeof(double) * 2;  // 2 words, lw + uw
  DBuf warm;
  CK(warm.alloc_async(std::min<size_t>(8 * ffn, 4ull << 30), ctx->stream));
  warm.reset();
  CK(cudaStreamSynchronize(ctx->stream));
  return FG_OK;
}

// Verdict of one probe (sentence s of the call's inputs at radius eps) from the fused pass's
// logits bounds and status; ambiguous ones go through the exact pass.  `ps` is updated to the
// status the decision rests on.  Returns the call status (a failure of the exact pass itself).
fg_status decide_probe(fg_model* m, const double* x_s, const int* pos_s, int words, int norm, double eps,
                       const double* lo, const double* hi, int pred, double margin, fg_status& ps, int& ok) {
  const int C = m->cfg.classes;
  ok = 0;
  if (ps != FG_OK) return FG_OK;
  fg_check_robust((size_t)C, lo, hi, (size_t)pred, margin, &ok);
  if (!ambiguous_verdict(m, lo, hi, C, pred, margin)) return FG_OK;
  fg_ctx* ctx = m->ctx;
  if (fg_status st = upload_params64(m)) return st;
  std::vector<double> elo(C), ehi(C);
  int est = FG_OK;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, ctx->stream);
  fg_status st = fgh::exact_pass(ctx, m->cfg, m->params64.as<double>(), x_s, pos_s, words, norm, eps, elo.data(),
                                 ehi.data(), nullptr, nullptr, &est);
  cudaEventRecord(b, ctx->stream);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (st) return st;
  ++m->exact_probes;
  m->exact_ms += ms;
  ps = (fg_status)est;
  ok = 0;
  if (ps == FG_OK) {
    fg_check_robust((size_t)C, elo.data(), ehi.data(), (size_t)pred, margin, &ok);
    if (margin == 0.0) calibrate_band(m, lo, hi, elo.data(), ehi.data(), C, pred);
  }
  return FG_OK;
}

// Asynchronous re-decision (fg_maxeps): the exact pass of an ambiguous probe is enqueued on the
// model's side stream and the sentence waits out of its slot while the fused passes of the other
// sentences continue; `poll` applies the verdict once the job's event has fired.
fgh::ExactJob* start_exact_job(fg_model* m, const double* x_s, const int* pos_s, int words, int norm, double eps,
                               int sentence, fg_status& st) {
  fg_ctx* ctx = m->ctx;
  st = upload_params64(m);
  if (st) return nullptr;
  if (!m->exact_stream[0]) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    for (cudaStream_t& es : m->exact_stream)
      if (cudaStreamCreateWithPriority(&es, cudaStreamNonBlocking, lo) != cudaSuccess) {
        st = fail(ctx, FG_ECUDA, "exact side stream");
        return nullptr;
      }
  }
  fgh::ExactJob* job = nullptr;
  for (auto& j : m->jobs)
    if (!j->busy) job = j.get();
  if (!job) {
    auto j = std::make_unique<fgh::ExactJob>();
    const int C = m->cfg.classes, nsites = 3 * m->cfg.layers;
    j->lo32.resize(C);
    j->hi32.resize(C);
    if (cudaMallocHost(&j->host, sizeof(double) * 2 * C) != cudaSuccess ||
        cudaMallocHost(&j->hstat, sizeof(int) * (nsites + 1)) != cudaSuccess ||
        cudaEventCreate(&j->start) != cudaSuccess || cudaEventCreate(&j->done) != cudaSuccess) {
      st = fail(ctx, FG_ENOMEM, "exact job buffers");
      return nullptr;
    }
    job = j.get();
    m->jobs.push_back(std::move(j));
  }
  fg_ctx side = *ctx;  // the same device, launches counted on the side stream
  side.stream = m->exact_stream[m->exact_rr++ % fg_model::kExactStreams];
  side.launches = 0;
  cudaEventRecord(job->start, side.stream);
  st = fgh::exact_pass(&side, m->cfg, m->params64.as<double>(), x_s, pos_s, words, norm, eps, nullptr, nullptr,
                       nullptr, nullptr, nullptr, job);
  ctx->launches += side.launches;
  if (st) {
    ctx->err = side.err;
    return nullptr;
  }
  job->busy = true;
  job->sentence = sentence;
  job->eps = eps;
  ++m->exact_probes;
  return job;
}

// Verdict of a finished job (the reference's exception order: first failing relaxation site,
// then the sink finiteness check, graph.cpp:663-671).
int finish_exact_job(fg_model* m, fgh::ExactJob* job, int pred, fg_status& ps) {
  float ms = 0.f;
  cudaEventElapsedTime(&ms, job->start, job->done);
  m->exact_ms += ms;
  job->busy = false;
  ps = FG_OK;
  for (int i = 0; i < job->nsites && ps == FG_OK; ++i)
    if (job->hstat[i] != kStatusClear) ps = (job->hstat[i] & 15) == kCodeInval ? FG_EINVAL : FG_EDOMAIN;
  if (ps == FG_OK && job->hstat[job->nsites]) ps = FG_EDOMAIN;
  int ok = 0;
  if (ps == FG_OK) {
    fg_check_robust((size_t)job->classes, job->host, job->host + job->classes, (size_t)pred, 0.0, &ok);
    calibrate_band(m, job->lo32.data(), job->hi32.data(), job->host, job->host + job->classes, job->classes, pred);
  }
  return ok;
}

// Narrow workspace for the ε = 0 probes of fg_maxeps (see ensure_workspace's zero_d), with
// the staged inputs of m->ws copied in; nullptr where it would not pay (D <= 128), when the
// pass is column-sharded, under FG_NO_ZERO_PROBE=1, or when it does not fit in free HBM.
Workspace* zero_workspace(fg_model* m, int S, int words) {
  const char* e = std::getenv("FG_NO_ZERO_PROBE");
  if ((e && e[0] == '1') || m->shard.active()) return nullptr;
  const int D = words * m->cfg.embed;
  const int zd = D > 128 ? 128 : 0;  // D = 128 -> 64 (SIMT GEMMs) measured slower at c2
  if (!zd) return nullptr;
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  const size_t per = bytes_per_sentence(m->cfg, zd);
  const int maxb = 65535 / (2 * m->cfg.length);
  int slots = (int)std::min<size_t>({(size_t)(0.5 * (double)free_b) / std::max<size_t>(per, 1), (size_t)S,
                                     (size_t)256, (size_t)maxb});
  const Workspace& w = m->ws;
  if (!m->ws0) m->ws0.reset(new Workspace());
  Workspace* z = m->ws0.get();
  if (slots < 1 || ensure_workspace(m, slots, words, S, z, zd) != FG_OK) {
    cudaGetLastError();
    m->ctx->err.clear();
    m->ws0.reset();
    return nullptr;
  }
  cudaStream_t st = m->ctx->stream;
  if (cudaMemcpyAsync(z->x_all.p, w.x_all.p, sizeof(double) * (size_t)S * m->cfg.length * m->cfg.embed,
                      cudaMemcpyDeviceToDevice, st) != cudaSuccess ||
      cudaMemcpyAsync(z->pos_all.p, w.pos_all.p, sizeof(int) * (size_t)S * words, cudaMemcpyDeviceToDevice,
                      st) != cudaSuccess)
    return nullptr;
  return z;
}

}  // namespace

extern "C" {

fg_status fg_model_create(fg_ctx* ctx, const fg_config* cfg, const double* params, fg_model** out) {
  *out = nullptr;
  if (!cfg || cfg->layers < 1 || cfg->heads < 1 || cfg->embed % cfg->heads != 0 || cfg->classes < 1 ||
      cfg->length < 1 || cfg->ffn < 1 || cfg->embed % 4 != 0)
    return fail(ctx, FG_EINVAL, "fg_model_create: invalid config");
  if (cfg->activation != FG_RELAX_RELU && cfg->activation != FG_RELAX_TANH &&
      cfg->activation != FG_RELAX_SILU)
    return fail(ctx, FG_EINVAL, "fg_model_create: activation must be relu/tanh/silu");
  cudaSetDevice(ctx->device);
  auto m = std::make_unique<fg_model>();
  m->ctx = ctx;
  m->cfg = *cfg;
  const size_t E = cfg->embed, F = cfg->ffn, C = cfg->classes;
  const size_t per_layer = 4 * (E * E + E) + E * F + F + F * E + E;
  m->params.assign(params, params + cfg->layers * per_layer + E * C + C);
  m->layers.resize(cfg->layers);
  for (int l = 0; l < cfg->layers; ++l) {
    const double* p = m->params.data() + m->layer_off(l);
    const double *wq = p, *bq = wq + E * E, *wk = bq + E, *bk = wk + E * E, *wv = bk + E, *bv = wv + E * E,
                 *wo = bv + E, *bo = wo + E * E, *w1 = bo + E, *b1 = w1 + E * F, *w2 = b1 + F, *b2 = w2 + F * E;
    std::vector<double> qkv(E * 3 * E), bqkv(3 * E);
    for (size_t i = 0; i < E; ++i)
      for (size_t j = 0; j < E; ++j) {
        qkv[i * 3 * E + j] = wq[i * E + j];
        qkv[i * 3 * E + E + j] = wk[i * E + j];
        qkv[i * 3 * E + 2 * E + j] = wv[i * E + j];
      }
    for (size_t j = 0; j < E; ++j) {
      bqkv[j] = bq[j];
      bqkv[E + j] = bk[j];
      bqkv[2 * E + j] = bv[j];
    }
    fg_status s;
    if ((s = upload_affine(ctx, m->layers[l].qkv, (int)E, (int)(3 * E), qkv, bqkv.data()))) return s;
    if ((s = upload_affine(ctx, m->layers[l].wo, (int)E, (int)E, std::vector<double>(wo, wo + E * E), bo))) return s;
    if ((s = upload_affine(ctx, m->layers[l].w1, (int)E, (int)F, std::vector<double>(w1, w1 + E * F), b1))) return s;
    if ((s = upload_affine(ctx, m->layers[l].w2, (int)F, (int)E, std::vector<double>(w2, w2 + F * E), b2))) return s;
  }
  const double* wc = m->params.data() + m->layer_off(cfg->layers);
  CK(m->wc64.alloc(sizeof(double) * E * C));
  CK(m->bc64.alloc(sizeof(double) * C));
  CK(cudaMemcpy(m->wc64.p, wc, sizeof(double) * E * C, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(m->bc64.p, wc + E * C, sizeof(double) * C, cudaMemcpyHostToDevice));
  // the uploads above ran on the legacy stream, which does not order the context's non-blocking
  // stream: wait for them before any pass can read the weights
  CK(cudaStreamSynchronize(0));
  *out = m.release();
  return FG_OK;
}

void fg_model_destroy(fg_model* m) {
  if (!m) return;
  cudaSetDevice(m->ctx->device);
  delete m;
}

fg_status fg_forward(fg_model* m, const double* x, double* logits) {
  forward_host(m->cfg, m->params.data(), x, logits);
  for (int i = 0; i < m->cfg.classes; ++i)
    if (!std::isfinite(logits[i])) return fail(m->ctx, FG_EINVAL, "forward: non-finite logits");
  return FG_OK;
}

fg_status fg_forward_batch(fg_model* m, int N, const double* x, double* logits) {
  fg_ctx* ctx = m->ctx;
  cudaSetDevice(ctx->device);
  if (N < 1) return fail(ctx, FG_EINVAL, "fg_forward_batch: N must be >= 1");
  const fg_config& c = m->cfg;
  const long long L = c.length, E = c.embed, F = c.ffn, C = c.classes, rows = (long long)N * L;
  cudaStream_t st = ctx->stream;
  DBuf X, QKV, CT, FF, LG;
  CK(X.alloc(sizeof(double) * rows * E));
  CK(QKV.alloc(sizeof(double) * rows * 3 * E));
  CK(CT.alloc(sizeof(double) * rows * E));
  CK(FF.alloc(sizeof(double) * rows * F));
  CK(LG.alloc(sizeof(double) * N * C));
  CK(cudaMemcpyAsync(X.p, x, sizeof(double) * rows * E, cudaMemcpyHostToDevice, st));
  double *xd = X.as<double>(), *qkv = QKV.as<double>(), *ct = CT.as<double>(), *ff = FF.as<double>();
  for (int l = 0; l < c.layers; ++l) {
    const DevLayer& L_ = m->layers[l];
    LAUNCH(launch_dense_f64(xd, L_.qkv.w64.as<double>(), L_.qkv.b64.as<double>(), nullptr, qkv, rows, (int)E,
                            (int)(3 * E), -1, st));
    LAUNCH(launch_attention_f64(qkv, ct, N, (int)L, (int)E, c.heads, st));
    LAUNCH(launch_dense_f64(ct, L_.wo.w64.as<double>(), L_.wo.b64.as<double>(), xd, xd, rows, (int)E, (int)E, -1,
                            st));
    LAUNCH(launch_dense_f64(xd, L_.w1.w64.as<double>(), L_.w1.b64.as<double>(), nullptr, ff, rows, (int)E, (int)F,
                            c.activation, st));
    LAUNCH(launch_dense_f64(ff, L_.w2.w64.as<double>(), L_.w2.b64.as<double>(), xd, xd, rows, (int)F, (int)E, -1,
                            st));
  }
  LAUNCH(launch_pool_head_f64(xd, m->wc64.as<double>(), m->bc64.as<double>(), LG.as<double>(), N, (int)L, (int)E,
                              (int)C, st));
  CK(cudaMemcpyAsync(logits, LG.p, sizeof(double) * N * C, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return FG_OK;
}

size_t fg_node_dump_size(const fg_config* c) {
  size_t L = c->length, E = c->embed, H = c->heads, F = c->ffn;
  return c->layers * (8 * L * E + 4 * H * L * L + 2 * H * L + 2 * L * F) + E + c->classes;
}

fg_status fg_bound_pass(fg_model* m, int S, const double* x, const int* positions, int words, int norm,
                        const double* eps, double* logits_lo, double* logits_hi, int* status) {
  fg_ctx* ctx = m->ctx;
  cudaSetDevice(ctx->device);
  if (S < 1 || words < 1 || words > m->cfg.length) return fail(ctx, FG_EINVAL, "fg_bound_pass: bad sizes");
  for (int s = 0; s < S; ++s)
    if (!eps_ok(eps[s])) return fail(ctx, FG_EINVAL, "PerturbationSpec: epsilon must be finite and >= 0");
  const int C = m->cfg.classes;
  int slots = default_slots(m, S, words * m->cfg.embed);
  fg_status st = ensure_workspace(m, slots, words, S);
  if (st) return st;
  if ((st = stage_inputs(m, S, x, positions, words))) return st;
  Workspace& w = m->ws;
  cudaEvent_t e0, e1, t0, t1;
  cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&t0); cudaEventCreate(&t1);
  uint64_t launches0 = ctx->launches;
  double total_ms = 0.0;
  int passes = 0;
  for (int s0 = 0; s0 < S; s0 += slots) {
    for (int i = 0; i < slots; ++i) {
      int s = std::min(s0 + i, S - 1);
      w.h_slot[i] = s;
      w.h_eps[i] = eps[s];
    }
    float ms = 0.f;
    if ((st = run_pass(m, norm, e0, e1, &ms))) break;
    total_ms += ms;
    ++passes;
    for (int i = 0; i < slots && s0 + i < S; ++i) {
      int s = s0 + i;
      for (int k = 0; k < C; ++k) {
        logits_lo[(size_t)s * C + k] = w.h_logits[(size_t)i * C + k];
        logits_hi[(size_t)s * C + k] = w.h_logits[(size_t)slots * C + (size_t)i * C + k];
      }
      status[s] = decode_status(w.h_status[i]);
    }
  }
  cudaEventDestroy(e0); cudaEventDestroy(e1); cudaEventDestroy(t0); cudaEventDestroy(t1);
  m->stats = fg_run_stats{total_ms, passes ? total_ms / passes : 0.0, passes, slots,
                          ctx->launches - launches0, (double)S, 0, 0.0, m->band_lo, m->band_hi, m->err_samples};
  return st;
}

fg_status fg_bound_pass_dump(fg_model* m, const double* x, const int* positions, int words, int norm,
                             double eps, double* logits_lo, double* logits_hi, double* node_lo,
                             double* node_hi, int* status) {
  fg_ctx* ctx = m->ctx;
  cudaSetDevice(ctx->device);
  if (!eps_ok(eps)) return fail(ctx, FG_EINVAL, "PerturbationSpec: epsilon must be finite and >= 0");
  if (m->shard.active()) return fail(ctx, FG_EINVAL, "fg_bound_pass_dump: not available on a column-sharded model");
  fg_status st = ensure_workspace(m, 1, words, 1);
  if (st) return st;
  if ((st = stage_inputs(m, 1, x, positions, words))) return st;
  Workspace& w = m->ws;
  size_t nd = fg_node_dump_size(&m->cfg);
  for (size_t i = 0; i < nd; ++i) node_lo[i] = node_hi[i] = std::numeric_limits<double>::quiet_NaN();
  w.h_eps[0] = eps;
  w.h_slot[0] = 0;
  CK(cudaMemcpyAsync(w.eps.p, w.h_eps, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(w.slot_map.p, w.h_slot, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
  w.h_active[0] = 1;
  CK(cudaMemcpyAsync(w.active.p, w.h_active, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
  Dumper d{node_lo, node_hi, ctx};
  if ((st = enqueue_pass(m, norm, &d))) return st;
  const int C = m->cfg.classes;
  std::vector<double> lg(2 * C);
  int sv = 0;
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaMemcpy(lg.data(), w.logits.p, sizeof(double) * 2 * C, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&sv, w.status.p, sizeof(int), cudaMemcpyDeviceToHost));
  for (int k = 0; k < C; ++k) {
    logits_lo[k] = lg[k];
    logits_hi[k] = lg[C + k];
  }
  *status = decode_status(sv);
  return FG_OK;
}

fg_status fg_certify(fg_model* m, int S, const double* x, const int* positions, int words, int norm,
                     const double* eps, double margin, int* verified, int* bounded, int* predicted,
                     double* logits_lo, double* logits_hi, int* status) {
  if (margin < 0.0) return fail(m->ctx, FG_EINVAL, "check_robust: margin must be >= 0");
  std::vector<int> pred = predict_all(m, S, x);
  fg_status st = fg_bound_pass(m, S, x, positions, words, norm, eps, logits_lo, logits_hi, status);
  if (st) return st;
  const int C = m->cfg.classes;
  const size_t LE = (size_t)m->cfg.length * m->cfg.embed;
  fg_run_stats stats = m->stats;
  m->exact_probes = 0;
  m->exact_ms = 0.0;
  for (int s = 0; s < S; ++s) {
    predicted[s] = pred[s];
    fg_status ps = (fg_status)status[s];
    if ((st = decide_probe(m, x + s * LE, positions + (size_t)s * words, words, norm, eps[s],
                           logits_lo + (size_t)s * C, logits_hi + (size_t)s * C, pred[s], margin, ps, verified[s])))
      return st;
    status[s] = ps;
    bounded[s] = status[s] != FG_EDOMAIN;  // cli.cpp:92-94
  }
  stats.exact_probes = m->exact_probes;
  stats.exact_ms = m->exact_ms;
  stats.band_lo = m->band_lo;
  stats.band_hi = m->band_hi;
  stats.band_samples = m->err_samples;
  stats.device_ms += m->exact_ms;
  m->stats = stats;
  return FG_OK;
}

fg_status fg_maxeps(fg_model* m, int S, const double* x, const int* positions, int words, int norm,
                    double eps_max, double tol, int slots, double* eps_out, int* calls_out,
                    int* predicted_out, int* status_out) {
  fg_ctx* ctx = m->ctx;
  cudaSetDevice(ctx->device);
  if (S < 1 || words < 1 || words > m->cfg.length) return fail(ctx, FG_EINVAL, "fg_maxeps: bad sizes");
  if (!eps_ok(eps_max)) return fail(ctx, FG_EINVAL, "fg_maxeps: eps_max must be finite and >= 0");
  const int C = m->cfg.classes;
  if (slots <= 0) slots = default_slots(m, S, words * m->cfg.embed);
  slots = std::min(slots, S);
  fg_status st = ensure_workspace(m, slots, words, S);
  if (st) return st;
  if ((st = stage_inputs(m, S, x, positions, words))) return st;
  Workspace& w = m->ws;
  cudaEvent_t c0, c1, e0, e1;
  cudaEventCreate(&c0); cudaEventCreate(&c1); cudaEventCreate(&e0); cudaEventCreate(&e1);
  CK(cudaEventRecord(c0, ctx->stream));
  uint64_t launches0 = ctx->launches;
  m->exact_probes = 0;
  m->exact_ms = 0.0;
  // predicted classes on host threads, overlapped with the first passes
  std::future<std::vector<int>> fut = std::async(std::launch::async, predict_all, m, S, x);
  std::vector<int> pred;
  bool have_pred = false;

  // bisection state per sentence (cli.cpp:144-177)
  enum Phase { P_ZERO = 0, P_MAX = 1, P_BISECT = 2, P_DONE = 3 };
  struct Sent { int phase = P_ZERO; double lo = 0.0, hi = 0.0, eps = 0.0; int calls = 0; };
  std::vector<Sent> sent(S);
  std::vector<int> slot(slots, -1);
  int next = 0, done = 0, passes = 0;
  double pass_ms_sum = 0.0, sentence_passes = 0.0;
  for (int s = 0; s < S; ++s) status_out[s] = FG_OK;
  // The first probe of every sentence, verified_at(0) (cli.cpp:159), runs up front on the
  // narrow all-zero-Λ workspace: at ε = 0 every concretization is bias ± 0·‖Λ‖, so the
  // verdicts, status codes and logits are those of the full-width pass at a fraction of its
  // GEMM work.  Each sentence keeps its probe sequence; only the ε = 0 probes move earlier.
  auto zero_phase = [&](int s, fg_status ps, int ok) {
    Sent& t = sent[s];
    ++t.calls;
    if (ps != FG_OK || !ok) {
      status_out[s] = ps != FG_OK ? ps : FG_ERUNTIME;  // misclassified input (cli.cpp:159-161)
      t.phase = P_DONE;
      eps_out[s] = std::numeric_limits<double>::quiet_NaN();
      calls_out[s] = t.calls;
      ++done;
    } else {
      t.phase = P_MAX;
      t.eps = eps_max;
    }
  };
  // The verdicts are decoded after the first full-width pass has run, so the host forward
  // behind the predicted classes (predict_all) stays overlapped with GPU work; sentences enter
  // that pass at ε_max tentatively, and one that fails at ε = 0 has its ε_max result dropped.
  std::vector<int> zst;
  std::vector<double> zlog;
  if (Workspace* z = zero_workspace(m, S, words)) {
    zst.resize(S);
    zlog.resize((size_t)S * 2 * C);
    for (int s0 = 0; s0 < S && !st; s0 += z->S) {
      for (int i = 0; i < z->S; ++i) {
        z->h_slot[i] = s0 + i < S ? s0 + i : 0;
        z->h_eps[i] = 0.0;
      }
      if ((st = run_pass(m, norm, nullptr, nullptr, nullptr, z))) break;
      for (int i = 0; i < z->S && s0 + i < S; ++i) {
        zst[s0 + i] = z->h_status[i];
        for (int k = 0; k < C; ++k) {
          zlog[(size_t)(s0 + i) * 2 * C + k] = z->h_logits[(size_t)i * C + k];
          zlog[(size_t)(s0 + i) * 2 * C + C + k] = z->h_logits[(size_t)z->S * C + (size_t)i * C + k];
        }
      }
    }
    for (int s = 0; s < S; ++s) {
      sent[s].phase = P_MAX;
      sent[s].eps = eps_max;
    }
  }
  const size_t LE = (size_t)m->cfg.length * m->cfg.embed;
  auto decode_zero = [&]() -> fg_status {
    for (int s = 0; s < S; ++s) {
      fg_status ps = decode_status(zst[s]);
      int ok = 0;
      if (fg_status e = decide_probe(m, x + s * LE, positions + (size_t)s * words, words, norm, 0.0,
                                     &zlog[(size_t)s * 2 * C], &zlog[(size_t)s * 2 * C + C], pred[s], 0.0, ps, ok))
        return e;
      zero_phase(s, ps, ok);
    }
    return FG_OK;
  };
  // A probe after ε = 0 (P_MAX / P_BISECT) whose f32 verdict is ambiguous is re-decided
  // asynchronously (start_exact_job) while its sentence keeps its slot and bisects on
  // speculatively with the verdict the f32 margin predicts (guess_verdict).  When the exact
  // verdict lands it either confirms the guess, or the sentence rolls back to its state at that
  // probe, is advanced with the exact verdict -- the reference's bisection step -- and every
  // re-decision started on the abandoned path is cancelled (per-sentence sequence numbers).
  // The call returns only when every re-decision has landed, so each verdict on the final path
  // is the exact one.  Column-sharded models decide synchronously (every rank must run the same
  // sentences in the same slots).
  const bool async_exact = !m->shard.active();
  struct Pend {
    fgh::ExactJob* job;
    int s;
    Sent snap;  // the sentence before this probe's (guessed) bisection step
    int guess, seq;
    bool cancelled;
  };
  std::vector<Pend> pending;
  std::vector<int> next_seq(S, 0);
  std::vector<char> queued(S, 0);
  std::vector<int> ready;  // rolled-back sentences waiting for a slot, FIFO
  size_t ready_head = 0;
  int rollbacks = 0;
  // one bisection step of sentence s with verdict ok (cli.cpp:163-177); true when finished
  auto advance = [&](int s, int ok) -> bool {
    Sent& t = sent[s];
    ++t.calls;
    bool finished = false;
    if (t.phase == P_MAX) {
      if (ok) {
        t.lo = eps_max;
        finished = true;
      } else {
        t.lo = 0.0;
        t.hi = eps_max;
        t.phase = P_BISECT;
      }
    } else {
      if (ok) t.lo = t.eps;
      else t.hi = t.eps;
    }
    if (!finished && t.phase == P_BISECT) {
      if (t.hi - t.lo > tol) t.eps = 0.5 * (t.lo + t.hi);
      else finished = true;
    }
    if (finished) {
      t.phase = P_DONE;
      eps_out[s] = status_out[s] == FG_OK ? t.lo : std::numeric_limits<double>::quiet_NaN();
      calls_out[s] = t.calls;
      ++done;
    }
    return finished;
  };
  // applies finished jobs (block: wait for the oldest one)
  auto poll = [&](bool block) {
    for (size_t k = 0; k < pending.size();) {
      Pend& pj = pending[k];
      cudaError_t q = block && k == 0 ? cudaEventSynchronize(pj.job->done) : cudaEventQuery(pj.job->done);
      if (q == cudaErrorNotReady) {
        ++k;
        continue;
      }
      if (q != cudaSuccess) {
        st = fail(ctx, FG_ECUDA, std::string("exact re-decision: ") + cudaGetErrorString(q));
        return;
      }
      const int s = pj.s;
      fg_status ps = FG_OK;
      const int verdict = finish_exact_job(m, pj.job, pred[s], ps) && ps == FG_OK;
      if (pj.cancelled) {
      } else if (pj.guess < 0) {  // no speculation: the sentence waited out of its slot
        if (!advance(s, verdict)) {
          queued[s] = 1;
          ready.push_back(s);
        }
      } else if (verdict != pj.guess) {  // wrong guess: back to the probe
        ++rollbacks;
        for (Pend& o : pending)
          if (o.s == s && o.seq > pj.seq) o.cancelled = true;
        if (sent[s].phase == P_DONE) --done;
        sent[s] = pj.snap;
        int in_slot = -1;
        for (int i = 0; i < slots; ++i)
          if (slot[i] == s) in_slot = i;
        if (advance(s, verdict)) {
          if (in_slot >= 0) slot[in_slot] = -1;
        } else if (in_slot < 0 && !queued[s]) {
          queued[s] = 1;
          ready.push_back(s);
        }
      }
      pending.erase(pending.begin() + (long)k);
      block = false;
    }
  };
  // early exit is switched on for a pass when at least a quarter of the previous pass's probes
  // failed (domain / validation errors): deep random-init models (c4, c5) fail almost every probe
  // above eps ~ 1e-7 part-way through the pass, c1-c3 almost none
  bool early_exit = false;
  while ((done < S || !pending.empty()) && !st) {
    bool any = false;
    int idle = 0;
    for (int i = 0; i < slots; ++i) {
      while (slot[i] < 0 && ready_head < ready.size()) {
        const int r = ready[ready_head++];
        queued[r] = 0;
        if (sent[r].phase != P_DONE) slot[i] = r;
      }
      while (slot[i] < 0 && next < S && sent[next].phase == P_DONE) ++next;
      if (slot[i] < 0 && next < S) slot[i] = next++;
      int s = slot[i];
      any = any || s >= 0;
      idle += s < 0;
      w.h_slot[i] = s >= 0 ? s : 0;
      w.h_eps[i] = s >= 0 ? sent[s].eps : 0.0;
      w.h_active[i] = s >= 0;
    }
    if (!any) {  // every sentence is done, some speculatively: wait for their exact verdicts
      poll(true);
      continue;
    }
    float ms = 0.f;
    // idle slots (finished sentences, or ones waiting for an exact verdict) are skipped like
    // failed ones: the tail of a batch, when few sentences remain, costs only their tiles
    if ((st = run_pass(m, norm, e0, e1, &ms, nullptr, early_exit || 4 * idle >= slots))) break;
    pass_ms_sum += ms;
    ++passes;
    {
      int active = 0, failed = 0;
      for (int i = 0; i < slots; ++i)
        if (slot[i] >= 0) {
          ++active;
          failed += decode_status(w.h_status[i]) != FG_OK;
        }
      early_exit = active > 0 && 4 * failed >= active;
    }
    if (!have_pred) {
      pred = fut.get();
      have_pred = true;
      if (!zst.empty() && (st = decode_zero())) break;
    }
    for (int i = 0; i < slots; ++i) {
      int s = slot[i];
      if (s < 0) continue;
      Sent& t = sent[s];
      if (t.phase == P_DONE) {  // failed at ε = 0 (decode_zero): this ε_max probe never happened
        slot[i] = -1;
        continue;
      }
      sentence_passes += 1.0;
      fg_status ps = decode_status(w.h_status[i]);
      const double* plo = w.h_logits + (size_t)i * C;
      const double* phi = w.h_logits + (size_t)slots * C + (size_t)i * C;
      int ok = 0;
      if (async_exact && t.phase != P_ZERO && ps == FG_OK && ambiguous_verdict(m, plo, phi, C, pred[s], 0.0)) {
        fgh::ExactJob* job = start_exact_job(m, x + s * LE, positions + (size_t)s * words, words, norm, t.eps, s, st);
        if (st) break;
        std::copy(plo, plo + C, job->lo32.begin());
        std::copy(phi, phi + C, job->hi32.begin());
        const int guess = m->speculate == FG_SPECULATE_OFF       ? -1
                          : m->speculate == FG_SPECULATE_VERIFIED  ? 1
                          : m->speculate == FG_SPECULATE_FAILED    ? 0
                                                                   : guess_verdict(m, plo, phi, C, pred[s]);
        pending.push_back(Pend{job, s, t, guess, next_seq[s]++, false});
        if (guess < 0 || advance(s, guess)) slot[i] = -1;
        continue;
      }
      if ((st = decide_probe(m, x + s * LE, positions + (size_t)s * words, words, norm, t.eps, plo, phi, pred[s],
                             0.0, ps, ok)))
        break;
      if (t.phase == P_ZERO) {  // verified_at(0, tolerate=false)
        zero_phase(s, ps, ok);
        if (t.phase == P_DONE) slot[i] = -1;
        continue;
      }
      if (advance(s, ps == FG_OK && ok)) slot[i] = -1;
    }
    if (!st) poll(false);
  }
  while (!pending.empty() && !st) poll(true);  // (an error left jobs in flight)
  std::fill(w.h_active, w.h_active + slots, 1);  // every other entry point runs all slots
  cudaMemcpyAsync(w.active.p, w.h_active, sizeof(int) * slots, cudaMemcpyHostToDevice, ctx->stream);
  for (cudaStream_t es : m->exact_stream)
    if (es) cudaStreamSynchronize(es);
  if (!have_pred) pred = fut.get();
  for (int s = 0; s < S; ++s) predicted_out[s] = pred[s];
  CK(cudaEventRecord(c1, ctx->stream));
  CK(cudaEventSynchronize(c1));
  float total = 0.f;
  cudaEventElapsedTime(&total, c0, c1);
  cudaEventDestroy(c0); cudaEventDestroy(c1); cudaEventDestroy(e0); cudaEventDestroy(e1);
  m->stats = fg_run_stats{(double)total, passes ? pass_ms_sum / passes : 0.0, passes, slots,
                          ctx->launches - launches0, sentence_passes, m->exact_probes, m->exact_ms,
                          m->band_lo, m->band_hi, m->err_samples, rollbacks};
  return st;
}


// Speculative bisection (see faith_gpu.h).  Probe list per round and sentence:
//   first round: eps = 0, eps = eps_max, then the subtree under [0, eps_max];
//   later rounds: the subtree under the current [lo, hi].
// Subtree nodes are enumerated level by level; a node (lo, hi) is a probe iff hi - lo > tol
// (the sequential loop's condition), its midpoint is 0.5 * (lo + hi) exactly as in cli.cpp:168.
namespace {
struct SpecProbe {
  int sent;
  double eps;
};
struct SpecNode {
  double lo, hi;
};
}  // namespace

fg_status fg_maxeps_spec(fg_model* m, int S, const double* x, const int* positions, int words, int norm,
                         double eps_max, double tol, int depth, int rank, int nranks, fg_exchange_fn exchange,
                         void* user, double* eps_out, int* calls_out, int* rounds_out, int* predicted_out,
                         int* status_out) {
  fg_ctx* ctx = m->ctx;
  cudaSetDevice(ctx->device);
  if (S < 1 || words < 1 || words > m->cfg.length || depth < 1 || depth > 10 || nranks < 1 || rank < 0 ||
      rank >= nranks || (nranks > 1 && !exchange))
    return fail(ctx, FG_EINVAL, "fg_maxeps_spec: bad arguments");
  if (!eps_ok(eps_max)) return fail(ctx, FG_EINVAL, "fg_maxeps_spec: eps_max must be finite and >= 0");
  const int C = m->cfg.classes;
  const int per_sent = 2 + (1 << depth) - 1;
  const int total_max = S * per_sent;
  const int mine_max = (total_max + nranks - 1) / nranks;
  int slots = std::min(mine_max, default_slots(m, mine_max, words * m->cfg.embed));
  slots = std::max(1, slots);
  fg_status st = ensure_workspace(m, slots, words, S);
  if (st) return st;
  if ((st = stage_inputs(m, S, x, positions, words))) return st;
  Workspace& w = m->ws;
  std::vector<int> pred = predict_all(m, S, x);
  enum { P_FIRST = 0, P_BISECT = 1, P_DONE = 2 };
  std::vector<int> phase(S, P_FIRST);
  std::vector<double> lo(S, 0.0), hi(S, eps_max);
  std::vector<int> calls(S, 0);
  for (int s = 0; s < S; ++s) status_out[s] = FG_OK;
  int rounds = 0, done = 0;
  uint64_t launches0 = ctx->launches;
  double pass_ms_sum = 0.0, sentence_passes = 0.0;
  int passes = 0;
  m->exact_probes = 0;
  m->exact_ms = 0.0;
  const size_t LE = (size_t)m->cfg.length * m->cfg.embed;
  cudaEvent_t e0, e1, c0, c1;  // e0/e1 per batched pass; c0/c1 span the whole call
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventCreate(&c0);
  cudaEventCreate(&c1);
  cudaEventRecord(c0, ctx->stream);
  while (done < S) {
    // ---- probes of this round
    std::vector<SpecProbe> probes;
    std::vector<std::vector<SpecNode>> trees(S);
    std::vector<int> first_probe(S, -1), tree_base(S, -1);
    for (int s = 0; s < S; ++s) {
      if (phase[s] == P_DONE) continue;
      first_probe[s] = (int)probes.size();
      if (phase[s] == P_FIRST) {
        probes.push_back({s, 0.0});
        probes.push_back({s, eps_max});
      }
      tree_base[s] = (int)probes.size();
      std::vector<SpecNode> level{{lo[s], hi[s]}};  // BFS: nodes of the next `depth` levels
      for (int d = 0; d < depth && !level.empty(); ++d) {
        std::vector<SpecNode> next;
        for (const SpecNode& nd : level) {
          if (!(nd.hi - nd.lo > tol)) continue;
          const double mid = 0.5 * (nd.lo + nd.hi);
          trees[s].push_back(nd);
          probes.push_back({s, mid});
          next.push_back({nd.lo, mid});
          next.push_back({mid, nd.hi});
        }
        level.swap(next);
      }
    }
    // ---- evaluate this rank's share in batched passes of `slots` probes.  The last word of
    // the verdict vector carries this rank's call status, so a failure on one rank ends the
    // call on every rank after the exchange instead of leaving the others waiting in it.
    std::vector<int> verdict(probes.size() + 1, 0);
    std::vector<int> mine;
    for (int i = rank; i < (int)probes.size(); i += nranks) mine.push_back(i);
    for (size_t b0 = 0; b0 < mine.size(); b0 += slots) {
      const size_t nb = std::min(mine.size() - b0, (size_t)slots);
      for (int i = 0; i < slots; ++i) {
        const SpecProbe& pr = probes[mine[b0 + std::min((size_t)i, nb - 1)]];
        w.h_slot[i] = pr.sent;
        w.h_eps[i] = pr.eps;
        w.h_active[i] = (size_t)i < nb;  // padding slots of a short batch: skipped
      }
      float ms = 0.f;
      if ((st = run_pass(m, norm, e0, e1, &ms, nullptr, 4 * (slots - (int)nb) >= slots))) break;
      pass_ms_sum += ms;
      ++passes;
      sentence_passes += (double)nb;
      for (size_t i = 0; i < nb && !st; ++i) {
        const int pi = mine[b0 + i];
        const int s = probes[pi].sent;
        fg_status ps = decode_status(w.h_status[i]);
        int ok = 0;
        st = decide_probe(m, x + s * LE, positions + (size_t)s * words, words, norm, probes[pi].eps,
                          w.h_logits + i * C, w.h_logits + (size_t)slots * C + i * C, pred[s], 0.0, ps, ok);
        verdict[pi] = ps != FG_OK ? 10 + ps : (ok ? 2 : 1);
      }
      if (st) break;
    }
    verdict.back() = st;
    if (nranks > 1 && exchange(user, verdict.data(), verdict.size()) != 0) {
      st = fail(ctx, FG_ERUNTIME, "fg_maxeps_spec: verdict exchange failed");
      break;
    }
    if (verdict.back() != FG_OK) {  // this rank or another one failed (MAX over the ranks' codes)
      if (!st) st = fail(ctx, (fg_status)verdict.back(), "fg_maxeps_spec: a pass failed on another rank");
      break;
    }
    ++rounds;
    // ---- walk each sentence's probes along the sequential decision path
    for (int s = 0; s < S; ++s) {
      if (phase[s] == P_DONE) continue;
      const int pi = first_probe[s];
      bool finished = false;
      if (phase[s] == P_FIRST) {
        const int v0 = verdict[pi], vmax = verdict[pi + 1];
        calls[s] = 1;
        if (v0 >= 10) {  // verified_at(0, tolerate = false) rethrows (cli.cpp:146-156)
          status_out[s] = v0 - 10;
          finished = true;
        } else if (v0 != 2) {
          status_out[s] = FG_ERUNTIME;  // misclassified input (cli.cpp:159-161)
          finished = true;
        } else {
          calls[s] = 2;
          if (vmax == 2) {
            lo[s] = eps_max;
            finished = true;
          } else {
            lo[s] = 0.0;
            hi[s] = eps_max;
            phase[s] = P_BISECT;
          }
        }
      }
      if (!finished) {
        // follow the decision path through this round's subtree (nodes matched by interval)
        const std::vector<SpecNode>& tr = trees[s];
        double l = lo[s], h = hi[s];
        for (int d = 0; d < depth; ++d) {
          if (!(h - l > tol)) break;
          int k = -1;
          for (size_t i = 0; i < tr.size(); ++i)
            if (tr[i].lo == l && tr[i].hi == h) {
              k = (int)i;
              break;
            }
          if (k < 0) break;
          const double mid = 0.5 * (l + h);
          ++calls[s];
          if (verdict[tree_base[s] + k] == 2) l = mid;
          else h = mid;
        }
        lo[s] = l;
        hi[s] = h;
        if (!(h - l > tol)) finished = true;
      }
      if (finished) {
        phase[s] = P_DONE;
        eps_out[s] = status_out[s] == FG_OK ? lo[s] : std::numeric_limits<double>::quiet_NaN();
        calls_out[s] = calls[s];
        ++done;
      }
    }
  }
  std::fill(w.h_active, w.h_active + slots, 1);
  cudaMemcpyAsync(w.active.p, w.h_active, sizeof(int) * slots, cudaMemcpyHostToDevice, ctx->stream);
  cudaEventRecord(c1, ctx->stream);
  cudaEventSynchronize(c1);
  float total = 0.f;  // the whole call, host-side forward / exchanges / exact passes included
  cudaEventElapsedTime(&total, c0, c1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(c0);
  cudaEventDestroy(c1);
  for (int s = 0; s < S; ++s) predicted_out[s] = pred[s];
  *rounds_out = rounds;
  m->stats = fg_run_stats{(double)total, passes ? pass_ms_sum / passes : 0.0, passes, slots,
                          ctx->launches - launches0, sentence_passes, m->exact_probes, m->exact_ms,
                          m->band_lo, m->band_hi, m->err_samples};
  return st;
}

}  // extern "C"

// ---- synthetic model / inputs: the reference's seeded generators (model.cpp:87-141,
// rng.hpp:11-32) so that a user of the library gets bit-identical weights/inputs.
namespace {
struct Rng64 {  // faith::Rng over std::mt19937_64 (rng.hpp:11-54)
  std::mt19937_64 eng;
  explicit Rng64(uint64_t s) : eng(s) {}
  double uniform() { return (double)(eng() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  uint64_t uniform_index(uint64_t n) {
    uint64_t limit = UINT64_MAX - UINT64_MAX % n, v;
    do {
      v = eng();
    } while (v >= limit);
    return v % n;
  }
};
}  // namespace

extern "C" {

fg_status fg_gen_synthetic(const fg_config* c, uint64_t seed, double* p) {
  if (!c || c->layers < 1 || c->heads < 1 || c->embed % c->heads) return FG_EINVAL;
  Rng64 rng(seed);
  const size_t e = c->embed, f = c->ffn, k = c->classes;
  auto gen = [&](size_t n, size_t fan_in) {  // gen_tensor (model.cpp:87-95)
    double bound = 0.5 / std::sqrt((double)fan_in);
    for (size_t i = 0; i < n; ++i) *p++ = (double)(float)rng.uniform(-bound, bound);
  };
  for (int l = 0; l < c->layers; ++l) {
    gen(e * e, e); gen(e, e); gen(e * e, e); gen(e, e); gen(e * e, e); gen(e, e);
    gen(e * e, e); gen(e, e); gen(e * f, e); gen(f, e); gen(f * e, f); gen(e, f);
  }
  gen(e * k, e);
  gen(k, e);
  return FG_OK;
}

size_t fg_param_count(const fg_config* c) {
  size_t e = c->embed, f = c->ffn, k = c->classes;
  return c->layers * (4 * (e * e + e) + e * f + f + f * e + e) + e * k + k;
}

fg_status fg_gen_input(const fg_config* c, uint64_t seed, double* x) {  // model.cpp:133-141
  Rng64 rng(seed ^ 0x9e3779b97f4a7c15ull);
  for (size_t i = 0; i < (size_t)c->length * c->embed; ++i) x[i] = (double)(float)rng.uniform(-0.5, 0.5);
  return FG_OK;
}

fg_status fg_gen_positions(uint64_t seed, int length, int words, int* pos) {
  if (words < 1 || words > length) return FG_EINVAL;
  Rng64 rng(seed);
  int n = 0;
  while (n < words) {
    int v = (int)rng.uniform_index((uint64_t)length);
    bool dup = false;
    for (int i = 0; i < n; ++i) dup |= pos[i] == v;
    if (!dup) pos[n++] = v;
  }
  std::sort(pos, pos + n);
  return FG_OK;
}

// One eager (non-graph) pass over the resident slots with CUDA events around every
// launch site; per-site device time (ms) and kernel counts.
fg_status fg_profile_pass(fg_model* m, int norm, double eps, int max_sites, char* names, double* ms,
                          int* kernels, int* nsites) {
  fg_ctx* ctx = m->ctx;
  cudaSetDevice(ctx->device);
  Workspace& w = m->ws;
  if (w.S <= 0) return fail(ctx, FG_EINVAL, "fg_profile_pass: run fg_maxeps/fg_bound_pass first");
  for (int i = 0; i < w.S; ++i) {
    w.h_eps[i] = eps;
    w.h_slot[i] = i % std::max(1, w.Ntot);
  }
  CK(cudaMemcpyAsync(w.eps.p, w.h_eps, sizeof(double) * w.S, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(w.slot_map.p, w.h_slot, sizeof(int) * w.S, cudaMemcpyHostToDevice, ctx->stream));
  Profiler prof;
  prof.st = ctx->stream;
  g_prof = &prof;
  fg_status st = enqueue_pass(m, norm, nullptr);
  g_prof = nullptr;
  g_tag = "other";
  if (st) return st;
  CK(cudaStreamSynchronize(ctx->stream));
  int n = 0;
  for (auto& site : prof.sites) {
    double t = 0.0;
    for (auto& be : site.ev) {
      float x = 0.f;
      cudaEventElapsedTime(&x, be.first, be.second);
      t += x;
      cudaEventDestroy(be.first);
      cudaEventDestroy(be.second);
    }
    if (n < max_sites) {
      std::snprintf(names + 32 * n, 32, "%s", site.tag.c_str());
      ms[n] = t;
      kernels[n] = site.kernels;
      ++n;
    }
  }
  *nsites = n;
  return FG_OK;
}

// Self-test of the affine bound GEMM paths on random data: both planes of
// Y = A X over `rows` token rows (A = W^T / |W|^T) by the tcgen05 3xTF32 kernel and
// by the FP32 SIMT kernel, each compared with an f64 device reference.
// err_* = max |Y - Y_ref| / max |Y_ref|; err_umma = -1 when the shape is not
// eligible for tcgen05.
fg_status fg_selftest_affine(fg_ctx* ctx, int rows, int C, int O, int D, uint64_t seed, double* err_umma,
                             double* err_simt, double* ms_umma, double* ms_simt, double* bias_umma) {
  cudaSetDevice(ctx->device);
  std::mt19937_64 rng(seed);
  auto uni = [&](double lo, double hi) { return lo + (hi - lo) * ((rng() >> 11) * 0x1.0p-53); };
  std::vector<double> w((size_t)C * O);
  for (double& v : w) v = (double)(float)uni(-0.5 / std::sqrt((double)C), 0.5 / std::sqrt((double)C));
  DevAffine a;
  fg_status s = upload_affine(ctx, a, C, O, w, nullptr);
  if (s) return s;
  const long long nin = (long long)rows * C * D, nout = (long long)rows * O * D;
  std::vector<float> x(2 * nin);  // centre plane in [-1, 1], radius plane in [0, 1]
  for (long long i = 0; i < 2 * nin; ++i) x[i] = (float)(i < nin ? uni(-1.0, 1.0) : uni(0.0, 1.0));
  DBuf X, Y1, Y2, Yref;
  CK(X.alloc(sizeof(float) * 2 * nin));
  CK(Y1.alloc(sizeof(float) * 2 * nout));
  CK(Y2.alloc(sizeof(float) * 2 * nout));
  CK(Yref.alloc(sizeof(double) * 2 * nout));
  CK(cudaMemcpy(X.p, x.data(), sizeof(float) * x.size(), cudaMemcpyHostToDevice));
  // on the context's (non-blocking) stream: a legacy-stream memset is not ordered before its kernels
  CK(cudaMemsetAsync(Y1.p, 0, sizeof(float) * 2 * nout, ctx->stream));
  CK(cudaMemsetAsync(Y2.p, 0, sizeof(float) * 2 * nout, ctx->stream));
  CK(cudaStreamSynchronize(0));  // the legacy-stream uploads (weights, X) have landed
  TensorMap tm;
  bool have_tm = (D % 128 == 0 || (D == 64 && rows % 2 == 0)) && lam_map(tm, X.as<float>(), nin, D, C, rows, 1);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float t = 0.f;
  CK(cudaEventRecord(e0, ctx->stream));
  LAUNCH(launch_gemm(affine_gemm(a, X.as<float>(), nin, Y1.as<float>(), nout, nullptr, 0, rows, D), ctx->stream));
  CK(cudaEventRecord(e1, ctx->stream));
  CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&t, e0, e1);
  *ms_simt = t;
  *ms_umma = -1.0;
  bool umma = a.umma && have_tm;
  if (umma) {
    CK(cudaEventRecord(e0, ctx->stream));
    if (a.ummaA && D % 128 == 0 && affine_tmem_a_enabled()) {
      LamGemm g = affine_lam(a, Y2.as<float>(), nout, nullptr, 0, rows, D);
      g.tmem_a = 1;
      LAUNCH(launch_lam_gemm(tm.bytes, a.tmA_hi.bytes, a.tmA_lo.bytes, g, 128, ctx->stream));
    } else {
      LAUNCH(launch_lam_gemm(tm.bytes, a.tm_hi.bytes, a.tm_lo.bytes, affine_lam(a, Y2.as<float>(), nout, nullptr, 0, rows, D),
                             a.bn, ctx->stream, a.umma2 ? a.tm2_hi.bytes : nullptr,
                             a.umma2 ? a.tm2_lo.bytes : nullptr));
    }
    CK(cudaEventRecord(e1, ctx->stream));
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&t, e0, e1);
    *ms_umma = t;
  }
  LAUNCH(launch_ref_affine_f64(a.w32.as<float>(), X.as<float>(), nin, Yref.as<double>(), C, O, D, rows,
                               ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  std::vector<float> y1(2 * nout), y2(2 * nout);
  std::vector<double> yr(2 * nout);
  CK(cudaMemcpy(y1.data(), Y1.p, sizeof(float) * y1.size(), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(y2.data(), Y2.p, sizeof(float) * y2.size(), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(yr.data(), Yref.p, sizeof(double) * yr.size(), cudaMemcpyDeviceToHost));
  // reference kernel output order is (row, plane, j, d); kernels write plane-major (plane, row, j, d)
  double mx = 0.0, e1s = 0.0, e2s = 0.0;
  for (long long r = 0; r < rows; ++r)
    for (int plane = 0; plane < 2; ++plane)
      for (long long jd = 0; jd < (long long)O * D; ++jd) {
        double ref = yr[(r * 2 + plane) * (long long)O * D + jd];
        long long k = plane * nout + r * (long long)O * D + jd;
        mx = std::max(mx, std::fabs(ref));
        e1s = std::max(e1s, std::fabs((double)y1[k] - ref));
        e2s = std::max(e2s, std::fabs((double)y2[k] - ref));
      }
  *err_simt = e1s / std::max(mx, 1e-300);
  *err_umma = umma ? e2s / std::max(mx, 1e-300) : -1.0;
  if (bias_umma) {  // median signed relative error of the tcgen05 result per plane (|ref| > mx / 4)
    for (int plane = 0; plane < 2; ++plane) {
      std::vector<double> rel;
      for (long long r = 0; r < rows; ++r)
        for (long long jd = 0; jd < (long long)O * D; ++jd) {
          double ref = yr[(r * 2 + plane) * (long long)O * D + jd];
          if (std::fabs(ref) < 0.25 * mx) continue;
          rel.push_back(((double)y2[plane * nout + r * (long long)O * D + jd] - ref) / ref);
        }
      if (!umma || rel.empty()) {
        bias_umma[plane] = 0.0;
        continue;
      }
      std::nth_element(rel.begin(), rel.begin() + rel.size() / 2, rel.end());
      bias_umma[plane] = rel[rel.size() / 2];
    }
  }
  return FG_OK;
}

static fg_status set_shard(fg_model* m, fgh::ShardState sh) {
  if (sh.nranks < 1 || sh.rank < 0 || sh.rank >= sh.nranks)
    return fail(m->ctx, FG_EINVAL, "column shard: bad rank / nranks");
  m->shard = std::move(sh);
  m->ws.release_host();  // drop the captured graph; buffers are re-planned for the local columns
  m->ws.S = 0;
  return FG_OK;
}

fg_status fg_model_set_column_shard(fg_model* m, int rank, int nranks, fg_allreduce_fn fn, void* user,
                                    int graph_capturable) {
  fgh::ShardState sh;
  sh.rank = rank;
  sh.nranks = nranks;
  sh.fn = fn;
  sh.user = user;
  sh.capturable = graph_capturable != 0;
  if (!fn && nranks != 1) return fail(m->ctx, FG_EINVAL, "column shard: an all-reduce is required for nranks > 1");
  return set_shard(m, std::move(sh));
}

fg_status fg_model_shard_nccl(fg_model* m, int rank, int nranks, const unsigned char id[128]) {
  cudaSetDevice(m->ctx->device);
  fgh::ShardState sh;
  std::string err;
  if (fg_status s = fgh::nccl_exchange(rank, nranks, id, sh, err)) return fail(m->ctx, s, err);
  return set_shard(m, std::move(sh));
}

fg_status fg_model_shard_loopback(fg_model* m, fg_loopback* g, int rank) {
  fgh::ShardState sh;
  if (fg_status s = fgh::loopback_exchange(g, rank, sh)) return fail(m->ctx, s, "column shard: bad loopback rank");
  return set_shard(m, std::move(sh));
}

fg_status fg_selftest_mma_peak(fg_ctx* ctx, int kind, int iters, double* ms, double* tflops) {
  cudaSetDevice(ctx->device);
  if ((kind != 0 && kind != 1) || iters < 1) return fail(ctx, FG_EINVAL, "fg_selftest_mma_peak: kind / iters");
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch_mma_peak(kind, 16, ctx->stream);  // warm-up (module load, clocks)
  CK(cudaEventRecord(a, ctx->stream));
  const int ctas = launch_mma_peak(kind, iters, ctx->stream);
  CK(cudaEventRecord(b, ctx->stream));
  CK(cudaEventSynchronize(b));
  CK(cudaGetLastError());
  float t = 0.f;
  cudaEventElapsedTime(&t, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  ctx->launches += 2;
  const double k = kind == 0 ? 8.0 : 16.0;
  *ms = t;
  *tflops = (double)ctas * iters * 4.0 * (2.0 * 128 * 256 * k) / (t * 1e-3) / 1e12;
  return FG_OK;
}

fg_status fg_bound_pass_exact(fg_model* m, const double* x, const int* positions, int words, int norm, double eps,
                              double* logits_lo, double* logits_hi, double* node_lo, double* node_hi,
                              int* status) {
  fg_ctx* ctx = m->ctx;
  cudaSetDevice(ctx->device);
  if (!eps_ok(eps)) return fail(ctx, FG_EINVAL, "PerturbationSpec: epsilon must be finite and >= 0");
  if (words < 1 || words > m->cfg.length) return fail(ctx, FG_EINVAL, "fg_bound_pass_exact: bad sizes");
  for (int w = 0; w < words; ++w)
    if (positions[w] < 0 || positions[w] >= m->cfg.length)
      return fail(ctx, FG_EINVAL, "fg_bound_pass_exact: position out of range");
  if (fg_status st = upload_params64(m)) return st;
  return fgh::exact_pass(ctx, m->cfg, m->params64.as<double>(), x, positions, words, norm, eps, logits_lo,
                         logits_hi, node_lo, node_hi, status);
}

fg_status fg_model_set_speculation(fg_model* m, int mode) {
  if (!m) return FG_EINVAL;
  if (mode < FG_SPECULATE_OFF || mode > FG_SPECULATE_FAILED)
    return fail(m->ctx, FG_EINVAL, "fg_model_set_speculation: unknown mode");
  m->speculate = mode;
  return FG_OK;
}

fg_status fg_model_set_exact_resolve(fg_model* m, double kappa) {
  if (!(kappa >= 0.0) || !std::isfinite(kappa)) return fail(m->ctx, FG_EINVAL, "fg_model_set_exact_resolve: kappa");
  m->kappa = kappa;
  m->band_lo = -kappa;  // recalibrated from this model's next re-decisions
  m->band_hi = kappa / 8;
  m->err_samples = 0;
  return FG_OK;
}

fg_status fg_last_run_stats(const fg_model* m, fg_run_stats* out) {
  *out = m->stats;
  return FG_OK;
}

}  // extern "C"
