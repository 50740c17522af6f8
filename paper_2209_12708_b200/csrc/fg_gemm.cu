// fg_gemm.cu -- batched f32 GEMM for the Λ contractions of the bound pass.
//
// This is the FP32 SIMT kernel: exact f32 FMA arithmetic, 128x128 (or 64x128)
// CTA tiles, 8x8 (4x8) register blocking, double-buffered shared memory.  It is
// the correctness baseline for every Λ contraction and the path
// for the small attention contractions; the affine bound GEMM additionally has
// a tcgen05 path (fg_umma.cu).
#include <algorithm>

#include "fg_internal.cuh"

namespace fg {

namespace {

constexpr int BN = 128;
constexpr int BK = 8;
constexpr int kThreads = 256;

template <int BM, bool ALIGNED>
__global__ void __launch_bounds__(kThreads) gemm_simt_kernel(GemmArgs g) {
  constexpr int TM = BM / 16;  // rows per thread (8 or 4)
  __shared__ __align__(16) float As[2][BK][BM];
  __shared__ __align__(16) float Bs[2][BK][BN];

  long long z = blockIdx.z;
  const int b3 = (int)(z % g.nb[3]);
  z /= g.nb[3];
  const int b2 = (int)(z % g.nb[2]);
  z /= g.nb[2];
  const int b1 = (int)(z % g.nb[1]);
  const int b0 = (int)(z / g.nb[1]);
  const float* A = g.A + b0 * g.sA[0] + b1 * g.sA[1] + b2 * g.sA[2] + b3 * g.sA[3];
  const float* B = g.B + b0 * g.sB[0] + b1 * g.sB[1] + b2 * g.sB[2] + b3 * g.sB[3];
  float* Cp = g.C + b0 * g.sC[0] + b1 * g.sC[1] + b2 * g.sC[2] + b3 * g.sC[3];
  const float* Rp = g.R ? g.R + b0 * g.sR[0] + b1 * g.sR[1] + b2 * g.sR[2] + b3 * g.sR[3] : nullptr;

  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;

  // loader mapping: one float4 of A (threads < BM*BK/4) and one float4 of B per thread
  const int a_k = tid / (BM / 4), a_m = (tid % (BM / 4)) * 4;
  const bool a_active = tid < BM * BK / 4;
  const int b_k = tid / (BN / 4), b_n = (tid % (BN / 4)) * 4;

  auto load_a = [&](int k0) -> float4 {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    const int m = m0 + a_m, k = k0 + a_k;
    if (a_active && k < g.K && m < g.M) {
      const float* p = A + (long long)k * g.lda + m;
      if (ALIGNED) {
        v = __ldg(reinterpret_cast<const float4*>(p));
      } else {
        v.x = p[0];
        if (m + 1 < g.M) v.y = p[1];
        if (m + 2 < g.M) v.z = p[2];
        if (m + 3 < g.M) v.w = p[3];
      }
    }
    return v;
  };
  auto load_b = [&](int k0) -> float4 {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    const int k = k0 + b_k, n = n0 + b_n;
    if (k < g.K && n < g.N) {
      const float* row = (k < g.K0) ? B + (long long)k * g.ldb : B + g.b_off1 + (long long)(k - g.K0) * g.ldb;
      if (ALIGNED) {
        v = *reinterpret_cast<const float4*>(row + n);
      } else {
        v.x = row[n];
        if (n + 1 < g.N) v.y = row[n + 1];
        if (n + 2 < g.N) v.z = row[n + 2];
        if (n + 3 < g.N) v.w = row[n + 3];
      }
    }
    return v;
  };

  float acc[TM][8];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

  float4 ra = load_a(0), rb = load_b(0);
  const int ktiles = (g.K + BK - 1) / BK;
  for (int kt = 0; kt < ktiles; ++kt) {
    const int buf = kt & 1;
    if (a_active) *reinterpret_cast<float4*>(&As[buf][a_k][a_m]) = ra;
    *reinterpret_cast<float4*>(&Bs[buf][b_k][b_n]) = rb;
    __syncthreads();
    if (kt + 1 < ktiles) {
      ra = load_a((kt + 1) * BK);
      rb = load_b((kt + 1) * BK);
    }
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      float a[TM], b[8];
      float4 a0 = *reinterpret_cast<const float4*>(&As[buf][k][ty * 4]);
      a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
      if (TM == 8) {
        float4 a1 = *reinterpret_cast<const float4*>(&As[buf][k][BM / 2 + ty * 4]);
        a[TM - 4] = a1.x; a[TM - 3] = a1.y; a[TM - 2] = a1.z; a[TM - 1] = a1.w;
      }
      float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][k][tx * 4]);
      float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][k][64 + tx * 4]);
      b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w;
      b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    // the next iteration writes the other buffer; one barrier per k-tile suffices
  }

#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int m = m0 + ((TM == 8 && i >= 4) ? BM / 2 + ty * 4 + (i - 4) : ty * 4 + i);
    if (m >= g.M) continue;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int n = n0 + half * 64 + tx * 4;
      if (n >= g.N) continue;
      float v[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) v[t] = g.alpha * acc[i][half * 4 + t];
      float* dst = Cp + (long long)m * g.ldc + n;
      const float* res = Rp ? Rp + (long long)m * g.ldr + n : nullptr;
      if (ALIGNED) {
        if (g.accumulate) {
          float4 o = *reinterpret_cast<const float4*>(dst);
          v[0] += o.x; v[1] += o.y; v[2] += o.z; v[3] += o.w;
        }
        if (res) {
          float4 r = *reinterpret_cast<const float4*>(res);
          v[0] += r.x; v[1] += r.y; v[2] += r.z; v[3] += r.w;
        }
        *reinterpret_cast<float4*>(dst) = make_float4(v[0], v[1], v[2], v[3]);
      } else {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          if (n + t >= g.N) break;
          float o = v[t];
          if (g.accumulate) o += dst[t];
          if (res) o += res[t];
          dst[t] = o;
        }
      }
    }
  }
}

}  // namespace

static bool al4(long long v) { return (v & 3) == 0; }
static bool al16(const void* p) { return ((uintptr_t)p & 15) == 0; }

int launch_gemm(const GemmArgs& g0, cudaStream_t st) {
  if (g0.M <= 0 || g0.N <= 0) return 0;
  const long long inner = (long long)g0.nb[1] * g0.nb[2] * g0.nb[3];
  if (g0.nb[0] <= 0 || inner <= 0 || inner > 65535 || g0.K <= 0) return -1;
  if ((long long)g0.nb[0] * inner > 65535) {  // gridDim.z limit: launch slices of the outermost batch dim
    const int per = (int)(65535 / inner);
    int n = 0;
    for (int b0 = 0; b0 < g0.nb[0]; b0 += per) {
      GemmArgs g = g0;
      g.nb[0] = std::min(per, g0.nb[0] - b0);
      g.A += b0 * g0.sA[0];
      g.B += b0 * g0.sB[0];
      g.C += b0 * g0.sC[0];
      if (g.R) g.R += b0 * g0.sR[0];
      const int r = launch_gemm(g, st);
      if (r < 0) return r;
      n += r;
    }
    return n;
  }
  const GemmArgs& g = g0;
  long long batches = (long long)g.nb[0] * g.nb[1] * g.nb[2] * g.nb[3];
  bool aligned = al4(g.M) && al4(g.N) && al4(g.lda) && al4(g.ldb) && al4(g.ldc) && al4(g.b_off1) &&
                 al16(g.A) && al16(g.B) && al16(g.C) && (!g.R || (al16(g.R) && al4(g.ldr)));
  for (int i = 0; i < 4; ++i)
    aligned = aligned && al4(g.sA[i]) && al4(g.sB[i]) && al4(g.sC[i]) && (!g.R || al4(g.sR[i]));
  dim3 block(kThreads);
  if (g.M <= 64) {
    dim3 grid((g.N + BN - 1) / BN, (g.M + 63) / 64, (unsigned)batches);
    if (aligned) gemm_simt_kernel<64, true><<<grid, block, 0, st>>>(g);
    else gemm_simt_kernel<64, false><<<grid, block, 0, st>>>(g);
  } else {
    dim3 grid((g.N + BN - 1) / BN, (g.M + 127) / 128, (unsigned)batches);
    if (aligned) gemm_simt_kernel<128, true><<<grid, block, 0, st>>>(g);
    else gemm_simt_kernel<128, false><<<grid, block, 0, st>>>(g);
  }
  return 1;
}

}  // namespace fg
