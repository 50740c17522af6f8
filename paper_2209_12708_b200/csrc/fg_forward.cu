// fg_forward.cu -- exact f64 forward pass on the GPU for batches of (perturbed) inputs:
// the soundness oracle of the bound pass at full model sizes.
//
// model::forward / ForwardEvaluator (proj/src/model.cpp:487-571): per layer
//   q,k,v = x Wq,k,v + b;  s_ij = q_i.k_j / sqrt(hd);  p = softmax_j(s);  ctx_i = sum_j p_ij v_j;
//   x += ctx Wo + bo;  x += act(x W1 + b1) W2 + b2;  logits = mean_i(x_i) Wc + bc.
// f64 throughout (FMA allowed: this is an oracle of the exact function, compared with slack,
// not a bit-level restatement; the bit-level forward is the host one, fg_forward).
#include <math.h>

#include "fg_internal.cuh"

namespace fg {

namespace {

constexpr int kT = 32;  // DGEMM tile

// Y[r, j] = sum_i X[r, i] W[i, j] + b[j] (+ R[r, j]) (act applied before the residual if act >= 0)
__global__ void __launch_bounds__(kT * 8) dense_f64_kernel(const double* __restrict__ X, const double* __restrict__ W,
                                                           const double* __restrict__ b, const double* R, double* Y,
                                                           long long rows, int C, int O, int act) {
  __shared__ double xs[kT][kT + 1];
  __shared__ double ws[kT][kT + 1];
  const int tx = threadIdx.x % kT, ty = threadIdx.x / kT;  // 32 x 8 threads, 4 rows each
  const long long r0 = (long long)blockIdx.y * kT;
  const int j = blockIdx.x * kT + tx;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int i0 = 0; i0 < C; i0 += kT) {
    for (int q = 0; q < 4; ++q) {
      const int rr = ty + 8 * q;
      const long long r = r0 + rr;
      xs[rr][tx] = (r < rows && i0 + tx < C) ? X[r * C + i0 + tx] : 0.0;
      ws[rr][tx] = (i0 + rr < C && j < O) ? W[(long long)(i0 + rr) * O + j] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int i = 0; i < kT; ++i) {
      const double wv = ws[i][tx];
      for (int q = 0; q < 4; ++q) acc[q] = fma(xs[ty + 8 * q][i], wv, acc[q]);
    }
    __syncthreads();
  }
  if (j >= O) return;
  for (int q = 0; q < 4; ++q) {
    const long long r = r0 + ty + 8 * q;
    if (r >= rows) continue;
    double v = acc[q] + b[j];
    if (act == RELAX_RELU) v = v > 0.0 ? v : 0.0;
    else if (act == RELAX_TANH) v = tanh(v);
    else if (act == RELAX_SILU) v = v * (1.0 / (1.0 + exp(-v)));
    if (R) v += R[r * O + j];
    Y[r * O + j] = v;
  }
}

// softmax attention for one (sample, head, query i): qkv [N, L, 3E] -> ctx [N, L, E]
__global__ void attention_f64_kernel(const double* __restrict__ qkv, double* __restrict__ ctx, int L, int E, int H) {
  extern __shared__ double sa[];  // [L] probabilities + 32 scratch
  double* p = sa;
  double* red = sa + L;
  const int hd = E / H;
  const long long n = blockIdx.x / ((long long)H * L);
  const int h = (int)((blockIdx.x / L) % H), i = (int)(blockIdx.x % L);
  const double* base = qkv + n * (long long)L * 3 * E;
  const double* q = base + (long long)i * 3 * E + h * hd;
  const double inv = 1.0 / sqrt((double)hd);
  double mx = -HUGE_VAL;
  for (int j = threadIdx.x; j < L; j += blockDim.x) {
    const double* k = base + (long long)j * 3 * E + E + h * hd;
    double s = 0.0;
    for (int d = 0; d < hd; ++d) s = fma(q[d], k[d], s);
    s *= inv;
    p[j] = s;
    mx = fmax(mx, s);
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = red[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, red[w]);
  __syncthreads();
  double sum = 0.0;
  for (int j = threadIdx.x; j < L; j += blockDim.x) {
    const double e = exp(p[j] - mx);
    p[j] = e;
    sum += e;
  }
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
  __syncthreads();
  sum = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) sum += red[w];
  for (int d = threadIdx.x; d < hd; d += blockDim.x) {
    double acc = 0.0;
    for (int j = 0; j < L; ++j) acc = fma(p[j], base[(long long)j * 3 * E + 2 * E + h * hd + d], acc);
    ctx[(n * L + i) * E + h * hd + d] = acc / sum;
  }
}

// logits[n, c] = (mean_i x[n, i, :]) . Wc[:, c] + bc[c]
__global__ void pool_head_f64_kernel(const double* __restrict__ x, const double* __restrict__ wc,
                                     const double* __restrict__ bc, double* __restrict__ logits, int L, int E, int C) {
  __shared__ double red[32];
  const int n = blockIdx.x / C, c = blockIdx.x % C;
  double acc = 0.0;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    double s = 0.0;
    for (int i = 0; i < L; ++i) s += x[((long long)n * L + i) * E + e];
    acc = fma(s / (double)L, wc[(long long)e * C + c], acc);
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    logits[(long long)n * C + c] = t + bc[c];
  }
}

}  // namespace

int launch_dense_f64(const double* X, const double* W, const double* b, const double* R, double* Y, long long rows,
                     int C, int O, int act, cudaStream_t st) {
  if (rows <= 0) return 0;
  dim3 grid((O + kT - 1) / kT, (unsigned)((rows + kT - 1) / kT));
  dense_f64_kernel<<<grid, kT * 8, 0, st>>>(X, W, b, R, Y, rows, C, O, act);
  return 1;
}

int launch_attention_f64(const double* qkv, double* ctx, long long N, int L, int E, int H, cudaStream_t st) {
  if (N <= 0) return 0;
  attention_f64_kernel<<<(unsigned)(N * H * L), 128, (L + 32) * sizeof(double), st>>>(qkv, ctx, L, E, H);
  return 1;
}

int launch_pool_head_f64(const double* x, const double* wc, const double* bc, double* logits, long long N, int L,
                         int E, int C, cudaStream_t st) {
  if (N <= 0) return 0;
  pool_head_f64_kernel<<<(unsigned)(N * C), 128, 0, st>>>(x, wc, bc, logits, L, E, C);
  return 1;
}

}  // namespace fg
