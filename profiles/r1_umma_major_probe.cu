// Minimal tcgen05 probe: D[128 x N] = A[128 x 8] * B[8 x N] (tf32), A K-major SW128, B MN-major SW128.
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, int layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

constexpr int N = 128;

__global__ void probe(float* out, int bmajor, int mode) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  float* A = (float*)sm;             // 128 rows x 32 k (128 B rows), 16 KB
  float* B = (float*)(sm + 16384);   // MN-major: [chunk 4][k 32][32] ; K-major: [n 128][k 32]
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  int tid = threadIdx.x;
  // A[m][k] = (k == m % 8) ? 1 : 0  (+ small k term), swizzled 128B rows
  for (int i = tid; i < 128 * 32; i += blockDim.x) {
    int m = i / 32, k = i % 32;
    float v = (k < 8) ? ((k == (m % 8)) ? 1.0f : 0.0f) + 0.001f * m : 0.0f;
    int chunk = k / 4, w = k % 4;
    int phys = ((chunk ^ (m % 8)) * 4) + w;
    A[m * 32 + phys] = v;
  }
  for (int i = tid; i < 32 * N; i += blockDim.x) {
    int k = i / N, n = i % N;
    float v = (k < 8) ? (float)(n + 1000 * k) : 0.0f;
    if (bmajor == 1) {  // MN-major: chunk c = n/32 at c*4096, row k at k*128, 16B chunk j swizzled by k%8
      int c = n / 32, nn = n % 32, j = nn / 4, w = nn % 4;
      B[c * 1024 + k * 32 + ((j ^ (k % 8)) * 4) + w] = v;
    } else {  // K-major: row n at n*128 bytes (32 floats), k contiguous, swizzled by n%8
      int j = k / 4, w = k % 4;
      B[n * 32 + ((j ^ (n % 8)) * 4) + w] = v;
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t tbase = tslot;
  if (tid == 0) {
    uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | ((uint32_t)bmajor << 16) |
                     ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    uint64_t ad = sw128_desc(smem_u32(A), 16, 1024, 2);
    uint64_t bd = bmajor ? sw128_desc(smem_u32(B), 4096, 1024, 2) : sw128_desc(smem_u32(B), 16, 1024, 2);
    if (mode == 1) {  // the CUTLASS form with disable-output-lane mask
      uint32_t z = 0;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5, %5, %5, %5}, p;\n}" ::"r"(tbase),
                   "l"(ad), "l"(bd), "r"(idesc), "r"(0), "r"(z));
    } else {
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tbase),
                   "l"(ad), "l"(bd), "r"(idesc), "r"(0));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
  }
  __syncwarp();
  asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(smem_u32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  int warp = tid / 32, lane = tid % 32;
  for (int c = 0; c < N; c += 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tbase + ((uint32_t)(warp * 32) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) out[(warp * 32 + lane) * N + c + j] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(128));
}

int main(int argc, char** argv) {
  float* d;
  cudaMalloc(&d, 128 * N * 4);
  for (int bmajor = 0; bmajor < 2; ++bmajor)
    for (int mode = 0; mode < 2; ++mode) {
      cudaMemset(d, 0, 128 * N * 4);
      cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
      probe<<<1, 128, 64 * 1024>>>(d, bmajor, mode);
      cudaError_t e = cudaDeviceSynchronize();
      float h[128 * N];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double maxerr = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < N; ++n) {
          double ref = 0;
          for (int k = 0; k < 8; ++k) ref += (((k == m % 8) ? 1.0 : 0.0) + 0.001 * m) * (n + 1000.0 * k);
          maxerr = fmax(maxerr, fabs(h[m * N + n] - ref) / fmax(1.0, fabs(ref)));
        }
      printf("bmajor=%d mode=%d err=%s maxrel=%g  D[0][0..3]=%g %g %g %g  D[5][1]=%g\n", bmajor, mode,
             cudaGetErrorString(e), maxerr, h[0], h[1], h[2], h[3], h[5 * N + 1]);
    }
  return 0;
}
