// fg_umma.cu -- tcgen05 (UMMA) bound GEMM of propagate_affine for sm_100a.
//
// Per (sentence s, token row r, plane p) the affine bound in center/radius form is
//   Y_p[j, d] = sum_i A_p[j, i] X_p[i, d],   A_c = W^T, A_r = |W|^T      (relax.cpp:237-307)
// i.e. a batched GEMM with M = O (output neurons), N = D (perturbation columns), K = C.
//
// FP32-class accuracy on the TF32 tensor pipe by error-compensated 3xTF32:
//   A = A_hi + A_lo (split once at model upload), X = X_hi + X_lo (split per tile in SMEM),
//   Y = A_hi X_hi + A_hi X_lo + A_lo X_hi   (the dropped A_lo X_lo term is < 2^-22 |A||X|).
//
// Kernel structure (persistent, one CTA per SM, 384 threads):
//   warp 0      TMA producer: A_hi, A_lo (K-major, SWIZZLE_128B) and the X tile
//               (MN-major, SWIZZLE_128B: BN/32 boxes of 32 columns x 32 rows) per stage
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (kind::tf32, M=128)
//   warps 4-7   split warps: X tile -> X_hi (in place) + X_lo, fence.proxy.async
//   warps 8-11  epilogue: tcgen05.ld TMEM -> registers, (+ residual), st.global
// Pipelines: smem stages full/split/empty, TMEM accumulators double-buffered
// (tmem_full/tmem_empty) so a tile's epilogue overlaps the next tile's mainloop.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "fg_internal.cuh"

namespace fg {

namespace {

constexpr int kBM = 128;
constexpr int kBK = 32;  // 32 fp32 = 128 B rows: one SWIZZLE_128B atom width
constexpr int kThreads = 384;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"(tm), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0, int c1,
                                            int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"(tm), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// SMEM matrix descriptor, SWIZZLE_128B (layout type 2), Blackwell version bit 46.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__device__ __forceinline__ void umma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

struct UmmaParams {
  float* C;
  long long ldc, c_sr, c_plane;
  const float* R;
  long long ldr, r_sr, r_plane;
  int M, N, K;
  int tiles_m, tiles_n, num_tiles;
  float alpha;
};

// Stage = { A_hi, A_lo (K-major SW128, TMA) | X raw [BK][BN] (TMA, no swizzle) |
//           X_hi, X_lo (K-major SW128: row n = 32 k values, written by the split warps) }.
// The tensor core reads both operands K-major: with kind::tf32 an MN-major B operand
// returned zeros on B200 (probe in DESIGN.md), so the split transposes the Λ tile.
template <int BN, int STAGES>
struct SmemLayout {
  static constexpr int kA = kBM * kBK * 4;  // 16 KB per A tile (hi or lo)
  static constexpr int kB = kBK * BN * 4;   // X tile (raw, hi or lo)
  static constexpr int kRaw = 2 * kA;       // offset of the raw X tile in a stage
  static constexpr int kHi = 2 * kA + kB;   // X_hi
  static constexpr int kLo = 2 * kA + 2 * kB;
  static constexpr int kStage = 2 * kA + 3 * kB;
  static constexpr int kBarOff = STAGES * kStage;
  static constexpr int kBytes = kBarOff + 256 + 1024;  // + barriers/tmem slot + alignment slack
};

template <int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    affine_umma_kernel(const __grid_constant__ CUtensorMap tm_ahi, const __grid_constant__ CUtensorMap tm_alo,
                       const __grid_constant__ CUtensorMap tm_b, const UmmaParams p) {
  using SL = SmemLayout<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SL::kBarOff);
  uint64_t* split = full + STAGES;
  uint64_t* empty = split + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkb = p.K / kBK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&split[s], 128);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_ahi) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_alo) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_b) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(2 * BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto tile_coords = [&](int t, int& sr, int& plane, int& m0, int& n0) {
    int mt = t % p.tiles_m;
    int rest = t / p.tiles_m;
    int nt = rest % p.tiles_n;
    int batch = rest / p.tiles_n;
    sr = batch >> 1;
    plane = batch & 1;
    m0 = mt * kBM;
    n0 = nt * BN;
  };

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int g = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        int sr, plane, m0, n0;
        tile_coords(t, sr, plane, m0, n0);
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          const int s = g % STAGES;
          const uint32_t ph = (g / STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* st = smem + s * SL::kStage;
          mbar_expect_tx(&full[s], 2 * SL::kA + SL::kB);
          tma_load_3d(st, &tm_ahi, &full[s], kb * kBK, m0, plane);
          tma_load_3d(st + SL::kA, &tm_alo, &full[s], kb * kBK, m0, plane);
          tma_load_4d(st + SL::kRaw, &tm_b, &full[s], n0, kb * kBK, sr, plane);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    // instruction descriptor: D f32, A/B tf32, both K-major, N=BN, M=128
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (0u << 16) |
                           ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(kBM >> 4) << 24);
    int g = 0, it = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++it) {
      const int acc = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      mbar_wait(&tempty[acc], aph ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = 0; kb < nkb; ++kb, ++g) {
        const int s = g % STAGES;
        const uint32_t ph = (g / STAGES) & 1;
        mbar_wait(&split[s], ph);
        tc_fence_after();
        if (lane == 0) {
          uint8_t* st = smem + s * SL::kStage;
          const uint32_t a_hi = smem_u32(st), a_lo = smem_u32(st + SL::kA);
          const uint32_t b_hi = smem_u32(st + SL::kHi), b_lo = smem_u32(st + SL::kLo);
#pragma unroll
          for (int ks = 0; ks < kBK / 8; ++ks) {
            // K-major SW128 operands (rows of 128 B, 8-row groups 1024 B apart): +32 B per 8 tf32 of K
            const uint64_t ahi = sw128_desc(a_hi + ks * 32, 16, 1024);
            const uint64_t alo = sw128_desc(a_lo + ks * 32, 16, 1024);
            const uint64_t bhi = sw128_desc(b_hi + ks * 32, 16, 1024);
            const uint64_t blo = sw128_desc(b_lo + ks * 32, 16, 1024);
            const uint32_t first = (kb | ks) != 0;
            umma_tf32(d_tmem, ahi, bhi, idesc, first);
            umma_tf32(d_tmem, ahi, blo, idesc, 1);
            umma_tf32(d_tmem, alo, bhi, idesc, 1);
          }
          umma_commit(&empty[s]);
          if (kb == nkb - 1) umma_commit(&tfull[acc]);
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ---------------- split + transpose: raw X [k][n] -> X_hi, X_lo (K-major SW128) ----------------
    // thread t owns row n = t of the K-major tiles: 32 conflict-free column reads of the raw
    // tile, 8 float4 stores per output tile (the 128B swizzle spreads a warp's rows over all banks).
    static_assert(BN == 128, "split maps one thread per output row");
    const int n = threadIdx.x - 128;
    int g = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
      for (int kb = 0; kb < nkb; ++kb, ++g) {
        const int s = g % STAGES;
        const uint32_t ph = (g / STAGES) & 1;
        mbar_wait(&full[s], ph);
        uint8_t* st = smem + s * SL::kStage;
        const float* raw = reinterpret_cast<const float*>(st + SL::kRaw);
#pragma unroll
        for (int j = 0; j < kBK / 4; ++j) {
          float h[4], l[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float v = raw[(4 * j + q) * BN + n];
            uint32_t hb;
            asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(v));
            h[q] = __uint_as_float(hb);
            l[q] = v - h[q];
          }
          const int off = n * 128 + ((j ^ (n & 7)) << 4);
          *reinterpret_cast<float4*>(st + SL::kHi + off) = make_float4(h[0], h[1], h[2], h[3]);
          *reinterpret_cast<float4*>(st + SL::kLo + off) = make_float4(l[0], l[1], l[2], l[3]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&split[s]);
      }
    }
  } else if (warp >= 8) {
    // ---------------- epilogue: TMEM -> registers -> global ----------------
    const int q = warp & 3;  // TMEM lane quarter accessible by this warp
    int it = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++it) {
      int sr, plane, m0, n0;
      tile_coords(t, sr, plane, m0, n0);
      const int acc = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const int m = m0 + q * 32 + lane;
      float* crow = p.C + sr * p.c_sr + plane * p.c_plane + (long long)m * p.ldc + n0;
      const float* rrow = p.R ? p.R + sr * p.r_sr + plane * p.r_plane + (long long)m * p.ldr + n0 : nullptr;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c * 32, v);
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          float4 o = make_float4(p.alpha * __uint_as_float(v[j]), p.alpha * __uint_as_float(v[j + 1]),
                                 p.alpha * __uint_as_float(v[j + 2]), p.alpha * __uint_as_float(v[j + 3]));
          if (rrow) {
            float4 r = *reinterpret_cast<const float4*>(rrow + c * 32 + j);
            o.x += r.x; o.y += r.y; o.z += r.z; o.w += r.w;
          }
          *reinterpret_cast<float4*>(crow + c * 32 + j) = o;
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(2 * BN));
  }
}

// ---- host helpers --------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

int g_num_sms = 0;

}  // namespace

bool umma_tmap_weights(void* tm, const float* a, int C, int O) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)C, (cuuint64_t)O, 2};
  cuuint64_t strides[2] = {(cuuint64_t)C * 4, (cuuint64_t)C * O * 4};
  cuuint32_t box[3] = {kBK, kBM, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(static_cast<CUtensorMap*>(tm), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(a), dims,
             strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool umma_tmap_lambda(void* tm, const float* lam, long long cr, int D, int C, long long rows) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[4] = {(cuuint64_t)D, (cuuint64_t)C, (cuuint64_t)rows, 2};
  cuuint64_t strides[3] = {(cuuint64_t)D * 4, (cuuint64_t)C * D * 4, (cuuint64_t)cr * 4};
  cuuint32_t box[4] = {128, kBK, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(static_cast<CUtensorMap*>(tm), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(lam), dims,
             strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool umma_supported(int M, int N, int K) {
  return encode_fn() != nullptr && M % kBM == 0 && K % kBK == 0 && N % 128 == 0 && M > 0 && N > 0;
}

int launch_affine_umma(const void* tm_ahi, const void* tm_alo, const void* tm_b, float* C, long long c_sr,
                       long long c_plane, const float* R, long long r_sr, long long r_plane, int M, int N, int K,
                       long long rows, float alpha, cudaStream_t st) {
  if (!umma_supported(M, N, K)) return -1;
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  UmmaParams p{};
  p.C = C; p.ldc = N; p.c_sr = c_sr; p.c_plane = c_plane;
  p.R = R; p.ldr = N; p.r_sr = r_sr; p.r_plane = r_plane;
  p.M = M; p.N = N; p.K = K;
  p.alpha = alpha;
  p.tiles_m = M / kBM;
  p.tiles_n = N / 128;
  long long tiles = (long long)p.tiles_m * p.tiles_n * rows * 2;
  if (tiles > 0x7fffffff) return -1;
  p.num_tiles = (int)tiles;
  int grid = (int)std::min<long long>(tiles, g_num_sms);
  const CUtensorMap& a = *static_cast<const CUtensorMap*>(tm_ahi);
  const CUtensorMap& b = *static_cast<const CUtensorMap*>(tm_alo);
  const CUtensorMap& x = *static_cast<const CUtensorMap*>(tm_b);
  using SL = SmemLayout<128, 2>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(affine_umma_kernel<128, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, SL::kBytes);
    attr = true;
  }
  affine_umma_kernel<128, 2><<<grid, kThreads, SL::kBytes, st>>>(a, b, x, p);
  return 1;
}

// f64 reference of the plane GEMM for fg_selftest_affine (test facility, not on the pass).
__global__ void ref_affine_f64_kernel(const float* A, const float* X, long long x_cr, double* Y, int C, int O,
                                      int D, long long rows) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long total = rows * 2 * O * (long long)D;
  if (t >= total) return;
  int d = (int)(t % D);
  int j = (int)((t / D) % O);
  int plane = (int)((t / ((long long)D * O)) % 2);
  long long r = t / ((long long)D * O * 2);
  const float* x = X + plane * x_cr + r * (long long)C * D + d;
  double acc = 0.0;
  for (int i = 0; i < C; ++i) {
    double w = A[(long long)i * O + j];
    if (plane) w = fabs(w);
    acc += w * (double)x[(long long)i * D];
  }
  Y[t] = acc;
}

int launch_ref_affine_f64(const float* W, const float* X, long long x_cr, double* Y, int C, int O, int D,
                          long long rows, cudaStream_t st) {
  long long total = rows * 2 * O * (long long)D;
  ref_affine_f64_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(W, X, x_cr, Y, C, O, D, rows);
  return 1;
}

}  // namespace fg
