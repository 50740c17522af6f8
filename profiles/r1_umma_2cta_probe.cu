// Probe (round 1): tcgen05.mma.cta_group::2.kind::tf32, M=256, N=NN, K=8, on a CTA pair.
// Checks the operand split the bound-GEMM engine relies on: each CTA holds its 128 rows of A
// and N/2 rows of B (both K-major SWIZZLE_128B), the leader issues, the commit multicasts to
// both CTAs, each CTA reads its 128 TMEM lanes x N columns.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o probe r1_umma_2cta_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

constexpr int NN = 256;

__device__ float a_val(int m, int k) { return (k < 8) ? ((k == (m % 8)) ? 1.0f : 0.0f) + 0.001f * (m % 97) : 0.0f; }
__device__ float b_val(int n, int k) { return (k < 8) ? (float)((n % 61) + 100 * k) : 0.0f; }

__global__ void __cluster_dims__(2, 1, 1) probe(float* out) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  float* A = (float*)sm;            // 128 rows x 32 k
  float* B = (float*)(sm + 16384);  // NN/2 rows x 32 k
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int tid = threadIdx.x;
  for (int i = tid; i < 128 * 32; i += blockDim.x) {
    int r = i / 32, k = i % 32, m = rank * 128 + r;
    A[r * 32 + (((k / 4) ^ (r % 8)) * 4) + k % 4] = a_val(m, k);
  }
  for (int i = tid; i < (NN / 2) * 32; i += blockDim.x) {
    int r = i / 32, k = i % 32, n = rank * (NN / 2) + r;
    B[r * 32 + (((k / 4) ^ (r % 8)) * 4) + k % 4] = b_val(n, k);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(NN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = tslot;
  if (rank == 0 && tid == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
    const uint64_t ad = sw128_desc(smem_u32(A)), bd = sw128_desc(smem_u32(B));
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tbase),
                 "l"(ad), "l"(bd), "r"(idesc), "r"(0));
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                     smem_u32(&bar)), "h"((uint16_t)3)
                 : "memory");
  }
  asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(
                   smem_u32(&bar))
               : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int warp = tid / 32, lane = tid % 32;
  for (int c = 0; c < NN; c += 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tbase + ((uint32_t)(warp * 32) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) out[(rank * 128 + warp * 32 + lane) * NN + c + j] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(NN));
}

int main() {
  float* d;
  cudaMalloc(&d, 256 * NN * 4);
  cudaMemset(d, 0, 256 * NN * 4);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  probe<<<2, 128, 64 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  static float h[256 * NN];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double maxerr = 0;
  for (int m = 0; m < 256; ++m)
    for (int n = 0; n < NN; ++n) {
      double ref = 0;
      for (int k = 0; k < 8; ++k) {
        double a = ((k == (m % 8)) ? 1.0 : 0.0) + 0.001 * (m % 97), b = (n % 61) + 100.0 * k;
        ref += a * b;
      }
      maxerr = fmax(maxerr, fabs(h[m * NN + n] - ref) / fmax(1.0, fabs(ref)));
    }
  printf("cta_group::2 M=256 N=%d: err=%s maxrel=%g  D[0][0..2]=%g %g %g  D[200][130]=%g\n", NN, cudaGetErrorString(e),
         maxerr, h[0], h[1], h[2], h[200 * NN + 130]);
  return 0;
}
