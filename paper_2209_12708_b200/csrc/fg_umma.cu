// fg_umma.cu -- tcgen05 (UMMA) engine for the Λ contractions of the bound pass (sm_100a).
//
// Every Λ contraction of the pass has the form (per batch b, both Λ planes c / r)
//     Out_b[n, d] (+)= alpha * sum_k  Wop_b[n, k] * Λ_b[k, d]                (+ R_b[n, d])
// with Λ stored [neuron][d] (d contiguous):
//   * propagate_affine (relax.cpp:237-307):   Wop = W^T or |W|^T,  k = input neuron
//   * McCormick x-side / y-side terms of propagate_dot_product (relax.cpp:533-654):
//     Wop = per-(sentence, head) coefficient matrices built from the concretized operands.
// The engine computes the transposed tile C^T[d, n] = sum_k Λ^T[d, k] Wop^T[k, n]:
//   M = 128 perturbation columns d (TMEM lanes), N = BN output neurons, K loop of 32.
// So the epilogue writes are coalesced along d and N can be as wide as 256.
//
// FP32-class accuracy on the TF32 pipe by error-compensated 3xTF32:
//   Wop = W_hi + W_lo (split when built), Λ = L_hi + L_lo (split per tile in SMEM),
//   C = L_hi W_hi + L_lo W_hi + L_hi W_lo   (dropped L_lo W_lo < 2^-22 |L||W|).
//
// Persistent, warp-specialized kernel (one CTA per SM, 384 threads):
//   warp 0     TMA producer: W_hi, W_lo tiles [BN][32] (K-major SWIZZLE_128B) and the raw
//              Λ tile [32][128] (no swizzle) per stage
//   warp 1     TMEM allocator + single-thread tcgen05.mma issuer (kind::tf32, M=128, N=BN)
//   warps 4-7  split warps: raw Λ [k][d] -> L_hi, L_lo [d][k] K-major SWIZZLE_128B
//              (transposed: kind::tf32 with an MN-major operand returned zeros on B200,
//              profiles/r1_umma_major_probe.txt)
//   warps 8-15 epilogue, two groups (one per TMEM accumulator): tcgen05.ld TMEM -> registers
//              -> coalesced st.global (+acc/+residual, prefetched)
// Pipelines: SMEM stages full/split/empty mbarriers; TMEM accumulators double-buffered.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "fg_internal.cuh"

namespace fg {

namespace {

constexpr int kBM = 128;  // d rows per tile (TMEM lanes)
constexpr int kBK = 32;   // 32 fp32 = 128 B rows: one SWIZZLE_128B atom width
constexpr int kThreads = 512;  // 4 role warps, 4 split warps, 2 x 4 epilogue warps

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

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0, int c1,
                                            int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"(tm), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// SMEM matrix descriptor, K-major SWIZZLE_128B: LBO 16 B (unused), SBO 1024 B (8-row groups),
// Blackwell version bit 46, layout type 2.
__device__ __forceinline__ uint64_t kmajor_sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
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
// One K chunk (32 deep = 4 K-steps of 8) of the 3xTF32 product, issued by one elected lane of a
// converged warp: D (+)= A_hi B_hi + A_lo B_hi + A_hi B_lo per K-step.  The descriptors of the
// four operand tiles are passed once; the K-step advances by +32 B (+2 in the descriptor's
// address field).  A single asm block keeps the twelve tcgen05.mma on uniform operands
// (no per-instruction elect / R2UR sequences around each MMA).
template <bool PAIR>
__device__ __forceinline__ void umma3_kchunk(uint32_t d_tmem, uint64_t ahi, uint64_t alo, uint64_t bhi, uint64_t blo,
                                             uint32_t idesc, uint32_t acc_first) {
#define FG_MMA(CG)                                                                          \
  asm volatile(                                                                             \
      "{\n\t.reg .pred e, p, t;\n\t.reg .b64 a0, a1, b0, b1;\n\t"                           \
      "elect.sync _|e, 0xffffffff;\n\t"                                                     \
      "setp.ne.b32 p, %5, 0;\n\t"                                                           \
      "setp.eq.b32 t, 0, 0;\n\t"                                                            \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], %1, %3, %6, p;\n\t"               \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], %2, %3, %6, t;\n\t"               \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], %1, %4, %6, t;\n\t"               \
      "add.s64 a0, %1, 2;\n\tadd.s64 a1, %2, 2;\n\tadd.s64 b0, %3, 2;\n\tadd.s64 b1, %4, 2;\n\t" \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], a0, b0, %6, t;\n\t"               \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], a1, b0, %6, t;\n\t"               \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], a0, b1, %6, t;\n\t"               \
      "add.s64 a0, %1, 4;\n\tadd.s64 a1, %2, 4;\n\tadd.s64 b0, %3, 4;\n\tadd.s64 b1, %4, 4;\n\t" \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], a0, b0, %6, t;\n\t"               \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], a1, b0, %6, t;\n\t"               \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], a0, b1, %6, t;\n\t"               \
      "add.s64 a0, %1, 6;\n\tadd.s64 a1, %2, 6;\n\tadd.s64 b0, %3, 6;\n\tadd.s64 b1, %4, 6;\n\t" \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], a0, b0, %6, t;\n\t"               \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], a1, b0, %6, t;\n\t"               \
      "@e tcgen05.mma.cta_group::" CG ".kind::tf32 [%0], a0, b1, %6, t;\n}"                 \
      ::"r"(d_tmem), "l"(ahi), "l"(alo), "l"(bhi), "l"(blo), "r"(acc_first), "r"(idesc))
  if (PAIR) FG_MMA("2");
  else FG_MMA("1");
#undef FG_MMA
}

// The same K chunk with the Λ operand (A) read from tensor memory: a_hi / a_lo are the TMEM
// addresses of the chunk's 32 hi / 32 lo columns (one tf32 per 32-bit column, row d = lane d),
// advanced by 8 columns per K-step.  Only the W operand (B) is read from shared memory.
__device__ __forceinline__ void umma3_kchunk_ts(uint32_t d_tmem, uint32_t ahi, uint32_t alo, uint64_t bhi,
                                                uint64_t blo, uint32_t idesc, uint32_t acc_first) {
  asm volatile(
      "{\n\t.reg .pred e, p, t;\n\t.reg .b32 a0, a1;\n\t.reg .b64 b0, b1;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "setp.eq.b32 t, 0, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %3, %6, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %3, %6, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %4, %6, t;\n\t"
      "add.u32 a0, %1, 8;\n\tadd.u32 a1, %2, 8;\n\tadd.s64 b0, %3, 2;\n\tadd.s64 b1, %4, 2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a0], b0, %6, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a1], b0, %6, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a0], b1, %6, t;\n\t"
      "add.u32 a0, %1, 16;\n\tadd.u32 a1, %2, 16;\n\tadd.s64 b0, %3, 4;\n\tadd.s64 b1, %4, 4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a0], b0, %6, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a1], b0, %6, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a0], b1, %6, t;\n\t"
      "add.u32 a0, %1, 24;\n\tadd.u32 a1, %2, 24;\n\tadd.s64 b0, %3, 6;\n\tadd.s64 b1, %4, 6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a0], b0, %6, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a1], b0, %6, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a0], b1, %6, t;\n}"
      ::"r"(d_tmem), "r"(ahi), "r"(alo), "l"(bhi), "l"(blo), "r"(acc_first), "r"(idesc));
}

// 32 consecutive 32-bit TMEM columns of this thread's lane (warp w accesses lanes 32(w%4)..+31)
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, "
      "%17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
// commit of the pair's MMAs, arriving on `bar` in both CTAs of the cluster
__device__ __forceinline__ void umma2_commit_both(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
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

// b[i] of a 4-entry batch coordinate held in registers (runtime i without a local-memory array)
__device__ __forceinline__ int get_at(const int (&b)[4], int i) {
  return i == 0 ? b[0] : (i == 1 ? b[1] : (i == 2 ? b[2] : b[3]));
}
__device__ __forceinline__ void add_at(int (&b)[4], int i, int v) {
  b[0] += i == 0 ? v : 0;
  b[1] += i == 1 ? v : 0;
  b[2] += i == 2 ? v : 0;
  b[3] += i == 3 ? v : 0;
}

__device__ __forceinline__ int lin5(const int* co, const int* b) {
  return co[0] * b[0] + co[1] * b[1] + co[2] * b[2] + co[3] * b[3] + co[4];
}
__device__ __forceinline__ long long lin5l(const long long* co, const int* b) {
  return co[0] * b[0] + co[1] * b[1] + co[2] * b[2] + co[3] * b[3] + co[4];
}

// Arrive on the pair leader's (CTA rank 0) copy of a barrier.  The release is restricted to
// shared memory (fence.release.sync_restrict::shared::cta.cluster + a relaxed cluster arrive:
// MEMBAR.CTA + FENCE.VIEW.ASYNC instead of the MEMBAR.GPU a .release.cluster arrive costs); the
// writes it publishes are this CTA's shared-memory operand tiles (already fenced to the async
// proxy) or, for the accumulator drain, ordered by tcgen05.fence::before_thread_sync.
__device__ __forceinline__ void mbar_arrive_cta0(uint64_t* local_bar) {
  uint32_t a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(a) : "r"(smem_u32(local_bar)));
  asm volatile("fence.release.sync_restrict::shared::cta.cluster;" ::: "memory");
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
}
// Wait on a local barrier that remote CTAs of the cluster arrive on (cluster-scope acquire).
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITC_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// SMEM plan: an operand ring of S stages {W_hi, W_lo, L_hi, L_lo} feeding the MMA and a raw
// ring of R Λ tiles feeding the split warps, so Λ loads run ahead of the operand stages.
// TA: the split Λ operand lives in tensor memory (S stages of 64 columns after the two
// accumulators), so a shared-memory operand stage holds only {W_hi, W_lo}.
template <int BN, int S, int R, bool PAIR, bool TA = false>
struct Ring {
  static constexpr int kWT = (PAIR ? BN / 2 : BN) * kBK * 4;  // this CTA's W tile, hi or lo
  static constexpr int kL = kBK * kBM * 4;                    // Λ tile: 16 KB
  static constexpr int kWlo = kWT;
  static constexpr int kLhi = 2 * kWT;
  static constexpr int kLlo = 2 * kWT + kL;
  static constexpr int kOp = TA ? 2 * kWT : 2 * kWT + 2 * kL;
  static constexpr int kTmemCols = TA ? 512 : (2 * BN < 32 ? 32 : 2 * BN);  // allocation: a power of 2
  static_assert(!TA || (2 * BN + S * 2 * kBK <= 512 && !PAIR), "TMEM plan of the TA engine: 2 accumulators + S A stages");
  static constexpr int kRawOff = S * kOp;
  static constexpr int kBarOff = kRawOff + R * kL;
  static constexpr int kMaskOff = kBarOff + 256;        // early-exit slot bitmask (32 words)
  static constexpr int kBytes = kMaskOff + 128 + 1024;  // + barriers / TMEM slot, mask, alignment slack
  static_assert(kBytes <= 227 * 1024, "rings exceed shared memory");
  static_assert(3 * S + 2 * R + 4 <= 31, "barrier area");
};

// Persistent warp-specialized tcgen05 3xTF32 engine (see the file header).  PAIR = CTA-pair
// variant (2-CTA cluster, cta_group::2, M = 256): CTA r holds d-rows m0 + 128r.. of Λ and W
// rows n0 + r*BN/2.. of the weight operand; the leader issues the MMA over both CTAs' SMEM and
// commits multicast; operand readiness of both CTAs is collected on the leader's `split`
// barrier (split warps wait for their CTA's W tile before arriving), accumulator drain on the
// leader's `tempty`.
//   warp 0: W producer    warp 1: TMEM alloc + MMA issuer    warp 2: Λ producer
//   warps 4-7: split/transpose Λ -> L_hi/L_lo    warps 8-15: epilogue (2 groups)
template <int BN, int S, int R, bool PAIR, bool TA = false>
__global__ void __launch_bounds__(kThreads, 1)
    lam_gemm_kernel(const __grid_constant__ CUtensorMap tm_lam, const __grid_constant__ CUtensorMap tm_whi,
                    const __grid_constant__ CUtensorMap tm_wlo, const LamGemm p) {
  using RL = Ring<BN, S, R, PAIR, TA>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* wfull = reinterpret_cast<uint64_t*>(smem + RL::kBarOff);
  uint64_t* split = wfull + S;
  uint64_t* opempty = split + S;
  uint64_t* rawfull = opempty + S;
  uint64_t* rawfree = rawfull + R;
  uint64_t* tfull = rawfree + R;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkb = p.K / kBK;
  // slots whose pass already failed (early exit), one bit each; everything the per-tile test
  // needs is re-read from the kernel parameters / shared memory (no registers held across the
  // role loops: this kernel runs at its 128-register limit)
  if (p.skip_tiles_per_b0)
    for (int base = warp * 32; base < p.skip_slots; base += kThreads) {
      const int slot = base + lane;
      const uint32_t bits = __ballot_sync(0xffffffffu, slot < p.skip_slots && p.skip_status[slot] != kStatusClear);
      if (lane == 0) reinterpret_cast<uint32_t*>(smem + RL::kMaskOff)[base >> 5] = bits;
    }
  uint32_t rank = 0;
  if (PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int unit = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int nunits = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  // pair_b0: the pair's two 128-row halves are batch rows 2b and 2b + 1 (M = D = 128), not d-tiles
  const int tiles_m = (PAIR && !p.pair_b0) ? p.tiles_m / 2 : p.tiles_m;
  const int num_tiles = PAIR ? p.num_tiles / 2 : p.num_tiles;
  // arrivals on the leader's split / tempty barriers: every split / epilogue thread of a single
  // CTA; one elected thread per CTA of a pair (after a named barrier of its 128 threads: remote
  // mbarrier arrivals cross the cluster's DSMEM path, 128 of them per stage serialise)
  constexpr int kGather = PAIR ? 2 : 128;

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&wfull[i], 1);
      mbar_init(&split[i], kGather);
      mbar_init(&opempty[i], 1);
    }
    for (int i = 0; i < R; ++i) {
      mbar_init(&rawfull[i], 1);
      mbar_init(&rawfree[i], 128);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kGather);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_lam) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_whi) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_wlo) : "memory");
  }
  if (warp == 1) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(2 * BN < 32 ? 32 : 2 * BN));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(RL::kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  if (PAIR) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // tile t -> (batch b0..b3, m-tile over d, n-tile over output neurons); n fastest so that
  // units running concurrently share the (HBM-resident) Λ tiles through L2.
  auto decode = [&](int t, int (&b)[4], int& m0, int& n0) {
    const int rest = (int)fdiv((uint32_t)t, p.f_tn);
    const int nt = t - rest * p.tiles_n;
    int batch = (int)fdiv((uint32_t)rest, p.f_tm);
    const int mt = rest - batch * tiles_m;
    int q = (int)fdiv((uint32_t)batch, p.f_nb3);
    b[3] = batch - q * p.nb[3];
    batch = q;
    q = (int)fdiv((uint32_t)batch, p.f_nb2);
    b[2] = batch - q * p.nb[2];
    batch = q;
    q = (int)fdiv((uint32_t)batch, p.f_nb1);
    b[1] = batch - q * p.nb[1];
    b[0] = q;
    if (p.gather) b[2] = p.gather[p.gather_slot[b[0]] * p.gather_ld + b[2]];
    if (p.fold1) add_at(b, p.fold1 - 1, get_at(b, p.fold1 - 1));  // the pair (2b, 2b + 1) of the folded coordinate
    if (PAIR && p.pair_b0) {  // this CTA's batch row of the pair
      b[0] = 2 * b[0] + (int)rank;
      m0 = mt * kBM;
    } else {
      m0 = mt * (PAIR ? 2 : 1) * kBM + (int)rank * kBM;  // this CTA's first d-row
    }
    n0 = nt * BN;
  };
  // every role skips the same tiles (the status words are not written during this kernel), so
  // the stage / accumulator counters stay in step
  // b[0] is the slowest tile coordinate: one division per tile, no full decode
  auto skipped = [&](int t) -> bool {
    if (!p.skip_tiles_per_b0) return false;
    const int slot = (int)fdiv(fdiv((uint32_t)t, p.f_skip_t) * p.skip_b0_scale, p.f_skip_div);
    return (reinterpret_cast<const uint32_t*>(smem + RL::kMaskOff)[slot >> 5] >> (slot & 31)) & 1u;
  };

  if (warp == 0) {
    // ---------------- W producer ----------------
    if (lane == 0) {
      int g = 0;
#pragma unroll 1
    for (int t = unit; t < num_tiles; t += nunits) {
        if (skipped(t)) continue;
        int b[4], m0, n0;
        decode(t, b, m0, n0);
        const int wc2 = lin5(p.w_c[0], b), wc3 = lin5(p.w_c[1], b);
        const int nw0 = n0 + (PAIR ? (int)rank * (BN / 2) : 0);
#pragma unroll 1
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          const int s = g % S;
          mbar_wait(&opempty[s], ((g / S) & 1) ^ 1);
          uint8_t* st = smem + s * RL::kOp;
          mbar_expect_tx(&wfull[s], 2 * RL::kWT);
          tma_load_4d(st, &tm_whi, &wfull[s], kb * kBK, nw0, wc2, wc3);
          tma_load_4d(st + RL::kWlo, &tm_wlo, &wfull[s], kb * kBK, nw0, wc2, wc3);
        }
      }
    }
  } else if (warp == 2) {
    // ---------------- Λ producer (raw ring) ----------------
    if (lane == 0) {
      int g = 0;
#pragma unroll 1
    for (int t = unit; t < num_tiles; t += nunits) {
        if (skipped(t)) continue;
        int b[4], m0, n0;
        decode(t, b, m0, n0);
        const int lc1 = lin5(p.lam_c[0], b), lc2 = lin5(p.lam_c[1], b), lc3 = lin5(p.lam_c[2], b);
#pragma unroll 1
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          const int r = g % R;
          mbar_wait(&rawfree[r], ((g / R) & 1) ^ 1);
          mbar_expect_tx(&rawfull[r], RL::kL);
          int kl = kb * kBK, plane = 0;
          if (kl >= p.K0) {  // c/r concatenation along K: second half reads the r plane
            kl -= p.K0;
            plane = 1;
          }
          if (p.fold1) {  // two 64-row halves: batch coordinate b and b + 1
            const int f = p.fold1 - 1;
            for (int half = 0; half < 2; ++half) {
              const int h1 = lc1 + half * p.lam_c[0][f], h2 = lc2 + half * p.lam_c[1][f],
                        h3 = lc3 + half * p.lam_c[2][f];
              tma_load_4d(smem + RL::kRawOff + r * RL::kL + half * (RL::kL / 2), &tm_lam, &rawfull[r], 0,
                          h1 + (p.kdim == 1 ? kl : 0), h2 + (p.kdim == 2 ? kl : 0), h3 + plane);
            }
          } else {
            tma_load_4d(smem + RL::kRawOff + r * RL::kL, &tm_lam, &rawfull[r], m0, lc1 + (p.kdim == 1 ? kl : 0),
                        lc2 + (p.kdim == 2 ? kl : 0), lc3 + plane);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (the leader CTA of a pair) ----------------
    if (!PAIR || rank == 0) {
      // D f32, A/B tf32, both K-major, N = BN, M = 128 (256 for a pair)
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)((PAIR ? 2 : 1) * kBM >> 4) << 24);
      int g = 0, it = -1;
#pragma unroll 1
    for (int t = unit; t < num_tiles; t += nunits) {
        if (skipped(t)) continue;
        ++it;
        const int acc = it & 1;
        if (PAIR) mbar_wait_cluster(&tempty[acc], ((it >> 1) & 1) ^ 1);
        else mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
#pragma unroll 1
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          const int s = g % S;
          if (PAIR) mbar_wait_cluster(&split[s], (g / S) & 1);
          else mbar_wait(&split[s], (g / S) & 1);
          tc_fence_after();
          {
            // +32 B per 8 tf32 of K inside the 128 B rows (umma3_kchunk)
            const uint32_t st = smem_u32(smem) + s * RL::kOp;
            if (TA) {
              const uint32_t a = tmem_base + 2 * BN + s * 2 * kBK;
              umma3_kchunk_ts(d_tmem, a, a + kBK, kmajor_sw128_desc(st), kmajor_sw128_desc(st + RL::kWlo), idesc,
                              kb != 0);
            } else {
              umma3_kchunk<PAIR>(d_tmem, kmajor_sw128_desc(st + RL::kLhi), kmajor_sw128_desc(st + RL::kLlo),
                                 kmajor_sw128_desc(st), kmajor_sw128_desc(st + RL::kWlo), idesc, kb != 0);
            }
          }
          if (lane == 0) {
            if (PAIR) {
              umma2_commit_both(&opempty[s]);
              if (kb == nkb - 1) umma2_commit_both(&tfull[acc]);
            } else {
              umma_commit(&opempty[s]);
              if (kb == nkb - 1) umma_commit(&tfull[acc]);
            }
          }
          __syncwarp();
        }
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ---------------- split + transpose: raw Λ [k][d] -> L_hi, L_lo [d][k] ----------------
    // thread = output row d: 32 conflict-free column reads, 8 float4 stores per tile
    // (the 128 B swizzle spreads a warp's rows over all banks).
    const int d = threadIdx.x - 128;
    int g = 0;
#pragma unroll 1
    for (int t = unit; t < num_tiles; t += nunits) {
      if (skipped(t)) continue;
      const unsigned char* mrow = nullptr;  // K-row mask of this thread's batch row (LamGemm::kmask)
      if (p.kmask) {
        int b[4], m0, n0;
        decode(t, b, m0, n0);
        mrow = p.kmask + (long long)(b[0] + (p.fold1 == 1 ? (d >> 6) : 0)) * p.K;
      }
#pragma unroll 1
      for (int kb = 0; kb < nkb; ++kb, ++g) {
        const int s = g % S, r = g % R;
        uint4 mk0 = make_uint4(0, 0, 0, 0), mk1 = mk0;
        if (mrow) {  // issued before the waits: its latency overlaps them
          mk0 = __ldg(reinterpret_cast<const uint4*>(mrow + kb * kBK));
          mk1 = __ldg(reinterpret_cast<const uint4*>(mrow + kb * kBK) + 1);
        }
        mbar_wait(&rawfull[r], (g / R) & 1);
        mbar_wait(&opempty[s], ((g / S) & 1) ^ 1);  // the MMAs of this stage's previous use are done
        uint8_t* st = smem + s * RL::kOp;
        const float* raw = reinterpret_cast<const float*>(smem + RL::kRawOff + r * RL::kL);
        float v[kBK];
        if (p.fold1) {  // raw = two [k][64] halves
          const float* rh = raw + (d >> 6) * (kBK * 64) + (d & 63);
#pragma unroll
          for (int k = 0; k < kBK; ++k) v[k] = rh[k * 64];
        } else {
#pragma unroll
          for (int k = 0; k < kBK; ++k) v[k] = raw[k * kBM + d];
        }
        // raw tile consumed: order these generic-proxy reads before the Λ producer's next TMA
        // (async-proxy) write into the same buffer, then release it
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&rawfree[r]);
        if (mrow) {
          const uint32_t mw[8] = {mk0.x, mk0.y, mk0.z, mk0.w, mk1.x, mk1.y, mk1.z, mk1.w};
#pragma unroll
          for (int k = 0; k < kBK; ++k)
            if (((mw[k >> 2] >> (8 * (k & 3))) & 0xffu) == 0) v[k] = 0.f;
        }
        if (TA) {
          // hi / lo parts into this stage's tensor-memory columns (lane d = this thread's row)
          tc_fence_after();  // after the opempty wait: the stage's previous MMAs are done
          uint32_t hl[kBK], lo[kBK];
#pragma unroll
          for (int k = 0; k < kBK; ++k) {
            asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hl[k]) : "f"(v[k]));
            lo[k] = __float_as_uint(v[k] - __uint_as_float(hl[k]));
          }
          const uint32_t ta = tmem_base + ((uint32_t)((warp & 3) * 32) << 16) + 2 * BN + s * 2 * kBK;
          tmem_st32(ta, hl);
          tmem_st32(ta + kBK, lo);
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          tc_fence_before();
          mbar_wait(&wfull[s], (g / S) & 1);  // this CTA's W tile landed too
          mbar_arrive(&split[s]);
          continue;
        }
#pragma unroll
        for (int j = 0; j < kBK / 4; ++j) {
          float h[4], l[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint32_t hb;
            asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(v[4 * j + q]));
            h[q] = __uint_as_float(hb);
            l[q] = v[4 * j + q] - h[q];
          }
          const int off = d * 128 + ((j ^ (d & 7)) << 4);
          *reinterpret_cast<float4*>(st + RL::kLhi + off) = make_float4(h[0], h[1], h[2], h[3]);
          *reinterpret_cast<float4*>(st + RL::kLlo + off) = make_float4(l[0], l[1], l[2], l[3]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (PAIR) {
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (d == 0) {
            mbar_wait(&wfull[s], (g / S) & 1);  // this CTA's W tile landed too
            mbar_arrive_cta0(&split[s]);
          }
        } else {
          mbar_wait(&wfull[s], (g / S) & 1);  // this CTA's W tile landed too
          mbar_arrive(&split[s]);
        }
      }
    }
  } else if (warp >= 8) {
    // ---------------- epilogue: TMEM -> registers -> global (coalesced along d) ----------------
    // The operand added to the accumulator (the previous value when accumulating, else the
    // residual) is software-prefetched: chunk 0 before waiting for the accumulator (its load
    // latency overlaps the tile's MMAs), chunk c+1 while chunk c is finished.
    // Two epilogue groups (warps 8-11, 12-15), one per TMEM accumulator: group g drains the
    // tiles with it % 2 == g, so two tiles' read-modify-write epilogues are in flight.
    const int q = warp & 3;  // TMEM lane quarter accessible by this warp
    const int grp = (warp - 8) >> 2;
    const bool has_x = p.accumulate || p.res;
    const long long xld = p.accumulate ? p.ldn_out : p.ldn_res;
    int it = -1;
#pragma unroll 1
    for (int t = unit; t < num_tiles; t += nunits) {
      if (skipped(t)) continue;
      ++it;
      if (p.epi_groups == 2 ? ((it & 1) != grp) : (grp != 0)) continue;
      int b[4], m0, n0;
      decode(t, b, m0, n0);
      const int acc = it & 1;
      int dd = m0 + q * 32 + lane;
      if (p.fold1) {  // lanes 64..127 hold the second of the folded pair (warp-uniform: q >> 1)
        add_at(b, p.fold1 - 1, q >> 1);
        dd &= 63;
      }
      float* out_b = p.out + lin5l(p.out_c, b) + dd;
      const float* res = p.res ? p.res + lin5l(p.res_c, b) + (long long)n0 * p.ldn_res + dd : nullptr;
      auto chunk_out = [&](int c) -> float* {
        const int n = n0 + c * 32;
        const int pl = p.n_split ? (int)fdiv((uint32_t)n, p.f_nsplit) : 0;
        float* out = p.n_split ? out_b + (long long)pl * p.split_stride +
                                     (long long)(n - pl * p.n_split) * p.ldn_out - (long long)c * 32 * p.ldn_out
                               : out_b + (long long)n0 * p.ldn_out;
        return out + (long long)c * 32 * p.ldn_out;
      };
      auto chunk_x = [&](int c) -> const float* {
        return p.accumulate ? chunk_out(c) : res + (long long)c * 32 * p.ldn_res;
      };
      // two chunks of the added operand in flight before the accumulator is ready, then a
      // rolling refill two chunks ahead (register double buffer pa / pb)
      constexpr int NCH = BN / 32;
      float pa[32], pb[32];
      // a plane boundary inside a 32-column chunk (n_split < 32, e.g. hd = 16): per-element
      // addresses, stepped incrementally (two divisions per chunk)
      auto split_off = [&](int c, int j, int& pl, int& nn) -> long long {
        if (j == 0) {
          const int nb0 = n0 + c * 32;
          pl = (int)fdiv((uint32_t)nb0, p.f_nsplit);
          nn = nb0 - pl * p.n_split;
        } else if (++nn == p.n_split) {
          nn = 0;
          ++pl;
        }
        return (long long)pl * p.split_stride + (long long)nn * p.ldn_out;
      };
      auto load_x = [&](int c, float (&dst)[32]) {
        if (p.accumulate && (p.n_split & 31)) {
          int pl = 0, nn = 0;
#pragma unroll
          for (int j = 0; j < 32; ++j) dst[j] = out_b[split_off(c, j, pl, nn)];
          return;
        }
        const float* xs = chunk_x(c);
#pragma unroll
        for (int j = 0; j < 32; ++j) dst[j] = xs[j * xld];
      };
      auto finish = [&](int c, const float (&xv)[32]) {
        uint32_t v[32];
        tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c * 32, v);
        float* oc = chunk_out(c);
        float o[32];
        const float al = (p.alpha_r_dim1 > 0 && get_at(b, p.alpha_r_dim1 - 1) == 1) ? p.alpha_r : p.alpha;
#pragma unroll
        for (int j = 0; j < 32; ++j) o[j] = al * __uint_as_float(v[j]);
        if (has_x) {
#pragma unroll
          for (int j = 0; j < 32; ++j) o[j] += xv[j];
        }
        if (p.n_split & 31) {  // a plane boundary inside the chunk (split_off)
          int pl = 0, nn = 0;
#pragma unroll
          for (int j = 0; j < 32; ++j) __stcs(out_b + split_off(c, j, pl, nn), o[j]);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) __stcs(oc + j * p.ldn_out, o[j]);
        }
      };
      if (has_x) {
        load_x(0, pa);
        if (NCH > 1) load_x(1, pb);
      }
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < NCH; c += 2) {
        finish(c, pa);
        if (has_x && c + 2 < NCH) load_x(c + 2, pa);
        if (c + 1 < NCH) {
          finish(c + 1, pb);
          if (has_x && c + 3 < NCH) load_x(c + 3, pb);
        }
      }
      tc_fence_before();
      if (PAIR) {
        asm volatile("bar.sync %0, 128;" ::"r"(2 + grp) : "memory");
        if ((threadIdx.x & 127) == 0) mbar_arrive_cta0(&tempty[acc]);
      } else {
        mbar_arrive(&tempty[acc]);
      }
    }
  }

  tc_fence_before();
  if (PAIR) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(2 * BN < 32 ? 32 : 2 * BN));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(RL::kTmemCols));
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

template <int BN, int S, int R, bool PAIR, bool TA = false>
int launch_ring(const void* tm_lam, const void* tm_whi, const void* tm_wlo, const LamGemm& p, int grid,
                cudaStream_t st) {
  using RL = Ring<BN, S, R, PAIR, TA>;
  auto kern = lam_gemm_kernel<BN, S, R, PAIR, TA>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, RL::kBytes);
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = RL::kBytes;
  cfg.stream = st;
  cudaLaunchAttribute attr2[1];
  attr2[0].id = cudaLaunchAttributeClusterDimension;
  attr2[0].val.clusterDim.x = PAIR ? 2 : 1;
  attr2[0].val.clusterDim.y = 1;
  attr2[0].val.clusterDim.z = 1;
  cfg.attrs = attr2;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, *static_cast<const CUtensorMap*>(tm_lam), *static_cast<const CUtensorMap*>(tm_whi),
                     *static_cast<const CUtensorMap*>(tm_wlo), p);
  return 1;
}

}  // namespace

int umma_pick_bn(int N) {
  return N % 256 == 0 ? 256 : (N % 128 == 0 ? 128 : (N % 64 == 0 ? 64 : (N % 32 == 0 ? 32 : 0)));
}

bool umma_available() { return encode_fn() != nullptr; }

bool umma_tmap_lam(void* tm, const float* base, const unsigned long long dims[4],
                   const unsigned long long strides_bytes[3], int kdim) {
  EncodeTiledFn enc = encode_fn();
  if (!enc || (kdim != 1 && kdim != 2)) return false;
  cuuint64_t dm[4] = {dims[0], dims[1], dims[2], dims[3]};
  cuuint64_t sd[3] = {strides_bytes[0], strides_bytes[1], strides_bytes[2]};
  // D = 64 (M folding, LamGemm::fold1): a 64-wide box, two loads fill one 128-row tile
  const cuuint32_t bm = dims[0] == 64 ? 64u : (cuuint32_t)kBM;
  cuuint32_t box[4] = {bm, kdim == 1 ? (cuuint32_t)kBK : 1u, kdim == 2 ? (cuuint32_t)kBK : 1u, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(static_cast<CUtensorMap*>(tm), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(base), dm, sd,
             box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool umma_tmap_wop(void* tm, const float* base, int K, int N, int P2, int P3, int bn) {
  EncodeTiledFn enc = encode_fn();
  if (!enc || bn <= 0 || N % bn != 0 || K % kBK != 0) return false;
  cuuint64_t dm[4] = {(cuuint64_t)K, (cuuint64_t)N, (cuuint64_t)P2, (cuuint64_t)P3};
  cuuint64_t sd[3] = {(cuuint64_t)K * 4, (cuuint64_t)K * N * 4, (cuuint64_t)K * N * P2 * 4};
  cuuint32_t box[4] = {kBK, (cuuint32_t)bn, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(static_cast<CUtensorMap*>(tm), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(base), dm, sd,
             box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool umma_pair_enabled() {
  static int v = -1;
  if (v < 0) {
    // CTA-pair kernel (cta_group::2, M = 256) wherever the shape allows it: half the W tile per
    // CTA and per-pair operand handoffs with a shared-memory-restricted cluster release
    // (mbar_arrive_cta0); measured 53-55 -> 47-48 ms per c3 pass on the affine GEMMs.  FG_2CTA=0: one CTA
    const char* e = std::getenv("FG_2CTA");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

int launch_lam_gemm(const void* tm_lam, const void* tm_whi, const void* tm_wlo, LamGemm p, int bn,
                    cudaStream_t st, const void* tm2_whi, const void* tm2_wlo) {
  {
    static int groups = 0;
    if (!groups) {
      const char* e = std::getenv("FG_EPI_GROUPS");
      groups = (e && e[0] == '1') ? 1 : 2;
    }
    p.epi_groups = groups;
  }
  if (p.fold1) {  // D = 64: pairs of coordinate fold1 - 1 fill one 128-row tile
    if (p.M != 64 || p.nb[p.fold1 - 1] % 2 || p.gather || p.K % kBK || p.K0 % kBK || bn <= 0 || p.N % bn)
      return -1;
    p.nb[p.fold1 - 1] /= 2;
    p.M = kBM;
    tm2_whi = tm2_wlo = nullptr;
  }
  if (p.M % kBM || p.K % kBK || p.K0 % kBK || bn <= 0 || p.N % bn) return -1;
  if (p.accumulate && p.res) return -1;  // one added operand: the previous output or a residual
  auto set_divisors = [&](int tiles_m_walk) {
    p.f_tn = make_fastdiv((uint32_t)p.tiles_n);
    p.f_tm = make_fastdiv((uint32_t)tiles_m_walk);
    p.f_nb1 = make_fastdiv((uint32_t)p.nb[1]);
    p.f_nb2 = make_fastdiv((uint32_t)p.nb[2]);
    p.f_nb3 = make_fastdiv((uint32_t)p.nb[3]);
    p.f_skip_t = make_fastdiv((uint32_t)std::max(p.skip_tiles_per_b0, 1));
    p.f_skip_div = make_fastdiv((uint32_t)std::max(p.skip_div, 1));
    p.f_nsplit = make_fastdiv((uint32_t)std::max(p.n_split, 1));
  };
  // pairs over batch rows (M = 128): both rows must share the W tile (W independent of b0) and an
  // early-exit slot
  const bool skip_on = p.skip_status && p.skip_slots > 0 && p.skip_slots <= 1024 && p.skip_div > 0;
  const bool pair_rows = p.M == kBM && !p.fold1 && !p.gather && p.nb[0] % 2 == 0 && p.w_c[0][0] == 0 &&
                         p.w_c[1][0] == 0 && (!skip_on || p.skip_div % 2 == 0);
  if (!p.tmem_a && tm2_whi && tm2_wlo && (p.M % (2 * kBM) == 0 || pair_rows) && bn >= 64 && umma_pair_enabled()) {
    if (!g_num_sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    p.pair_b0 = p.M % (2 * kBM) != 0;
    p.tiles_m = p.M / kBM;
    p.tiles_n = p.N / bn;
    long long tiles = (long long)p.tiles_m * p.tiles_n * p.nb[0] * p.nb[1] * p.nb[2] * p.nb[3];
    if (tiles <= 0 || tiles > 0x7fffffff) return -1;
    p.num_tiles = (int)tiles;  // single-CTA tiles; the pair kernel walks tiles / 2 pair tiles
    p.skip_tiles_per_b0 = 0;
    if (skip_on) {  // per pair unit of b0 (a b0 pair when pair_b0)
      p.skip_tiles_per_b0 = (p.pair_b0 ? p.tiles_m : p.tiles_m / 2) * p.tiles_n * p.nb[1] * p.nb[2] * p.nb[3];
      p.skip_b0_scale = p.pair_b0 ? 2 : 1;
    }
    if (p.pair_b0) p.nb[0] /= 2;  // the kernel walks b0 pairs, b0 = 2 b' + rank
    set_divisors(p.pair_b0 ? p.tiles_m : p.tiles_m / 2);
    const int grid = 2 * (int)std::min<long long>(tiles / 2, g_num_sms / 2);
    switch (bn) {
      case 256: return launch_ring<256, 3, 2, true>(tm_lam, tm2_whi, tm2_wlo, p, grid, st);
      case 128: return launch_ring<128, 4, 2, true>(tm_lam, tm2_whi, tm2_wlo, p, grid, st);
      case 64: return launch_ring<64, 4, 3, true>(tm_lam, tm2_whi, tm2_wlo, p, grid, st);
    }
  }
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  p.tiles_m = p.M / kBM;
  p.tiles_n = p.N / bn;
  long long tiles = (long long)p.tiles_m * p.tiles_n * p.nb[0] * p.nb[1] * p.nb[2] * p.nb[3];
  if (tiles <= 0 || tiles > 0x7fffffff) return -1;
  p.num_tiles = (int)tiles;
  p.skip_tiles_per_b0 = 0;  // early exit (see LamGemm::skip_status)
  if (p.skip_status && p.skip_slots > 0 && p.skip_slots <= 1024 && p.skip_div > 0) {
    p.skip_tiles_per_b0 = p.tiles_m * p.tiles_n * p.nb[1] * p.nb[2] * p.nb[3];
    p.skip_b0_scale = p.fold1 == 1 ? 2 : 1;
  }
  set_divisors(p.tiles_m);
  const int grid = (int)std::min<long long>(tiles, g_num_sms);
  if (p.tmem_a) {  // Λ operand from tensor memory: two accumulators + 4 operand stages of 64 columns
    if (bn == 128) return launch_ring<128, 4, 6, false, true>(tm_lam, tm_whi, tm_wlo, p, grid, st);
    if (bn == 64) return launch_ring<64, 4, 6, false, true>(tm_lam, tm_whi, tm_wlo, p, grid, st);
  }
  switch (bn) {
    case 256: return launch_ring<256, 2, 2, false>(tm_lam, tm_whi, tm_wlo, p, grid, st);
    case 128: return launch_ring<128, 3, 2, false>(tm_lam, tm_whi, tm_wlo, p, grid, st);
    // skinny K / small N (McCormick y-side terms): HBM-bound, so a deep Λ ring
    case 64: return launch_ring<64, 2, 6, false>(tm_lam, tm_whi, tm_wlo, p, grid, st);
    case 32: return launch_ring<32, 4, 3, false>(tm_lam, tm_whi, tm_wlo, p, grid, st);
  }
  return -1;
}

// Dense tensor-pipe peak microbenchmark (fg_selftest_mma_peak; the roofline denominator of the
// 3xTF32 GEMMs): one CTA per SM, one thread issuing back-to-back tcgen05.mma M=128 N=256 on
// SMEM-resident operands (no loads), 4 K-steps per 128 B operand row, committed every 64 MMAs.
// kind::tf32 (K = 8 per MMA) or kind::f16 with bf16 operands (K = 16 per MMA).
template <int KIND>
__global__ void __launch_bounds__(128, 1) mma_peak_kernel(int iters) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* a = smem;                 // 128 rows x 128 B
  uint8_t* b = smem + 128 * 128;     // 256 rows x 128 B
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 384 * 128);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  for (int i = threadIdx.x; i < 384 * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (threadIdx.x == 0) {
    // D f32; A/B tf32 (kind::tf32: format 2) or bf16 (kind::f16: format 1); K-major; N = 256, M = 128
    const uint32_t fmt = KIND == 0 ? 2u : 1u;
    const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(256 >> 3) << 17) |
                           ((uint32_t)(128 >> 4) << 24);
    uint32_t phase = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const uint64_t ad = kmajor_sw128_desc(smem_u32(a) + ks * 32), bd = kmajor_sw128_desc(smem_u32(b) + ks * 32);
        if (KIND == 0)
          umma_tf32(tmem, ad, bd, idesc, (it | ks) != 0);
        else
          asm volatile(
              "{\n\t.reg .pred p;\n\t"
              "setp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
              "l"(ad), "l"(bd), "r"(idesc), "r"((uint32_t)((it | ks) != 0)));
      }
      if ((it & 15) == 15 || it == iters - 1) {
        umma_commit(bar);
        mbar_wait(bar, phase);
        phase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
  }
}

int launch_mma_peak(int kind, int iters, cudaStream_t st) {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int bytes = 384 * 128 + 64 + 1024;
  auto k0 = mma_peak_kernel<0>;
  auto k1 = mma_peak_kernel<1>;
  cudaFuncSetAttribute(k0, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (kind == 0) k0<<<g_num_sms, 128, bytes, st>>>(iters);
  else k1<<<g_num_sms, 128, bytes, st>>>(iters);
  return g_num_sms;
}

// f64 reference of the affine plane GEMM for fg_selftest_affine (test facility, not on the pass).
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
