// fg_internal.cuh -- shared declarations of the B200 bound-propagation kernels.
//
// Data model on the device:
//   A bound tensor over N neurons with D perturbation columns is stored as
//   * Λ in CENTER/RADIUS form, f32, two planes of [N, D] (D contiguous):
//       c = (Λᵁ + Λᴸ) / 2,   r = (Λᵁ − Λᴸ) / 2       (plane r at +cr elements)
//     so the sign-split affine bound  Λᵁ' = W⁺Λᵁ + W⁻Λᴸ,  Λᴸ' = W⁺Λᴸ + W⁻Λᵁ
//     (relax.cpp:237-307) becomes two dense GEMMs  c' = Wc,  r' = |W| r;
//   * lb, ub (and concretized lo, hi) in f64, [N].
//   Sentences of a batch are the outermost axis of every tensor.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fg {

// Per-sentence status word: atomicMin of (site << 4 | code).  The smallest site
// wins (the reference throws at the first failing node); within a site
// EINVAL (1) beats EDOMAIN (2) because ConcreteBounds::validate runs over all
// neurons before any domain check (relax.cpp:314-335, 364-392, 397-410).
constexpr int kStatusClear = 0x7fffffff;
// status of a slot that holds no probe in this pass (fg_maxeps: its sentence finished or waits
// for an exact re-decision): not clear, so every early-exit kernel skips it
constexpr int kStatusIdle = 0x7ffffffe;
constexpr int kCodeInval = 1;
constexpr int kCodeDomain = 2;

enum Norm { NORM_L1 = 0, NORM_L2 = 1, NORM_LINF = 2 };
enum Relax {
  RELAX_RELU = 0, RELAX_TANH = 1, RELAX_SILU = 2, RELAX_EXP = 3, RELAX_RECIP = 4,
  // extension (no reference counterpart): the LayerNorm bound chain's envelopes
  RELAX_SQRT = 5, RELAX_SQUARE = 6
};

// A neuron-indexed view into a batched bound tensor.
//   neuron(s, row, f) = s*s_stride + row*row_stride + col0 + f
struct NView {
  float* lam;           // plane c; plane r at lam + cr
  long long cr;
  double* lb;
  double* ub;
  double* lo;           // concretized bounds (may be null when not needed)
  double* hi;
  long long s_stride;   // neurons per sentence
  int row_stride;       // neurons per token row
  int col0;             // first neuron of the slice
};

// Generic batched f32 GEMM on N-contiguous operands:
//   C[b][m, n] = alpha * sum_k A[b][m, k] * B[b][k, n]  (+ C[b] if accumulate) (+ R[b])
//   A is M-major: A[m, k] at A + k*lda + m.
//   B rows k <  K0 at B + k*ldb,  rows k >= K0 at B + b_off1 + (k-K0)*ldb.
//   Batch index b = ((b0*nb1 + b1)*nb2 + b2)*nb3 + b3 with per-level strides.
struct GemmArgs {
  int M, N, K, K0;
  const float* A;
  long long lda;
  const float* B;
  long long ldb, b_off1;
  float* C;
  long long ldc;
  const float* R;
  long long ldr;
  float alpha;
  int accumulate;
  int nb[4];
  long long sA[4], sB[4], sC[4], sR[4];
};

// ---- launchers (fg_kernels.cu / fg_gemm.cu); all return the number of kernels launched
int launch_gemm(const GemmArgs& g, cudaStream_t st);

int launch_concretize(const float* lam, long long cr, const double* lb, const double* ub,
                      long long rows_per_s, long long nrows, int D, int norm, const double* eps,
                      double* lo, double* hi, cudaStream_t st, const int* skip = nullptr);

// concretize of token rows whose Λ is zero outside the perturbed tokens (first-layer Q/K/V)
int launch_concretize_tokens(const float* lam, long long cr, const double* lb, const double* ub,
                             long long rows_per_s, long long nrows, int D, int norm, const double* eps,
                             double* lo, double* hi, const int* positions, const int* slot_map, int W, int width,
                             cudaStream_t st);

int launch_elementwise_verify(int kind, float* lam, long long cr, double* lb, double* ub,
                              long long rows_per_s, long long nrows, int D, int norm,
                              const double* eps, int* status, int site, double* lo_out,
                              double* hi_out, cudaStream_t st, const double* lo_in = nullptr,
                              const double* hi_in = nullptr, const int* skip = nullptr,
                              unsigned char* keep = nullptr);

// Standalone envelope / compose (operator-level API).
int launch_relax(int kind, const double* lo, const double* hi, long long n, double* a_low,
                 double* b_low, double* a_up, double* b_up, int* status, cudaStream_t st);
int launch_compose(float* lam_in, long long cr_in, const double* lb_in, const double* ub_in,
                   const double* a_low, const double* b_low, const double* a_up,
                   const double* b_up, float* lam_out, long long cr_out, double* lb_out,
                   double* ub_out, long long n, int D, cudaStream_t st);

// Affine bias path in f64 with the reference's accumulation order (relax.cpp:273-299),
// optional residual add (propagate_add(res, y), relax.cpp:656-674).
int launch_affine_bias(const double* lb_in, const double* ub_in, const double* w64,
                       const double* bias, const double* res_lb, const double* res_ub,
                       double* lb_out, double* ub_out, int S, int rows, int C, int O,
                       cudaStream_t st, const int* skip = nullptr);

// Pairwise-similarity McCormick dot product Q.K^T (relax.cpp:573-617) scaled by `scale`
// (the following Scale node, model.cpp:416-418).  out: [S, H, L, L] neurons.
int launch_dot_similarity(const NView& q, const NView& k, const NView& out, int S, int L, int H,
                          int hd, int D, float* coef_ws, float scale, cudaStream_t st);
// Weighted-values McCormick dot product P.V (relax.cpp:618-652).  p: [S, H, L, L] neurons;
// v: token rows; out: token rows [S, L, E].
int launch_dot_weighted(const NView& p, const NView& v, const NView& out, int S, int L, int H,
                        int hd, int D, float* coef_ws, cudaStream_t st);

// Softmax chain along the key axis of scores [S, H*L rows, L keys] (graph.cpp:237-240):
// exp -> sum -> recip -> McCormick multiply, in place; also writes probs lo/hi.
int launch_softmax(const NView& sc, int S, int rows_per_s, int n, int D, int norm,
                   const double* eps, int* status, int site_exp, int site_recip,
                   cudaStream_t st);

// Word-level input binding: lb = ub = x, Λ rows of perturbed positions one-hot.
int launch_init_input(float* lam, long long cr, double* lb, double* ub, const double* x,
                      const int* positions, const int* slot_map, int S, int L, int E, int W,
                      cudaStream_t st, int D = 0, int col0 = 0);
// First layer from the one-hot Λ0 analytically: Q/K/V Λ = W scattered into the perturbed rows
// (exact, no GEMM), and the Λ0 residual of the first attention block as a +1 scatter.
// launch_init_input with lam == nullptr binds lb/ub only.
int launch_onehot_affine(float* lam, long long cr, const float* w, const int* positions, const int* slot_map, int S,
                         int L, int E, int O, int W, int D, int col0, cudaStream_t st, int skip_o = 0);
int launch_add_onehot(float* lam, const int* positions, const int* slot_map, int S, int L, int E, int W, int D,
                      int col0, cudaStream_t st);
// MeanPool (graph.cpp:628-634) -> pooled f64 planes [S, E, D] (+ lb/ub [S, E]).
int launch_meanpool(const float* lam, long long cr, const double* lb, const double* ub,
                    double* pooled_c, double* pooled_r, double* plb, double* pub, int S, int L,
                    int E, int D, cudaStream_t st);
// Classifier affine + final concretization + finiteness check (graph.cpp:663-671).
int launch_head(const double* pooled_c, const double* pooled_r, const double* plb,
                const double* pub, const double* wc, const double* bc, int S, int E, int C,
                int D, int norm, const double* eps, double* logits_lo, double* logits_hi,
                int* status, int site, double* pooled_lo, double* pooled_hi,
                cudaStream_t st);

// Layout conversion for the operator-level API: reference (lw, uw) f64 <-> (c, r) f32.
int launch_ul_to_cr(const double* lw, const double* uw, float* lam, long long cr, long long n,
                    int d, int Dp, cudaStream_t st);
int launch_cr_to_ul(const float* lam, long long cr, double* lw, double* uw, long long n, int d,
                    int Dp, cudaStream_t st);
int launch_add(const float* a, long long acr, const double* alb, const double* aub,
               const float* b, long long bcr, const double* blb, const double* bub, float* y,
               long long ycr, double* ylb, double* yub, long long n, int D, cudaStream_t st);
int launch_scale(const float* x, long long xcr, const double* xlb, const double* xub, double s,
                 float* y, long long ycr, double* ylb, double* yub, long long n, int D,
                 cudaStream_t st);
int launch_fill_int(int* p, int v, long long n, cudaStream_t st);
// status[i] = active[i] ? kStatusClear : kStatusIdle (start of a pass)
int launch_init_status(int* status, const int* active, int n, cudaStream_t st);

// ---- tcgen05 3xTF32 engine for Λ contractions (fg_umma.cu) ---------------------------
// Out_b[n, d] (+)= alpha * sum_k Wop_b[n, k] * Λ_b[k, d] (+ R_b[n, d]), computed as
// C^T[d, n] tiles with M = 128 d-rows, N = BN output neurons, K in steps of 32.
//   Λ: 4-D tensor map (d, c1, c2, c3) over a Λ buffer (c3 = plane); the K index runs along
//      coordinate `kdim` (1 or 2); for k >= K0 it continues in plane c3 + 1 at k - K0 (the
//      c/r concatenation of the McCormick x-side terms).
//   Wop: two 4-D tensor maps (k, n, c2, c3) over the TF32 hi / lo parts, K-major.
//   Batch b = ((b0*nb1 + b1)*nb2 + b2)*nb3 + b3; every coordinate / offset is
//   co[0]*b0 + co[1]*b1 + co[2]*b2 + co[3]*b3 + co[4].
// Tensor maps are opaque 128-byte CUtensorMap objects (64-byte aligned storage).
// Division by a runtime divisor d >= 1 as a multiply-high (x < 2^31): q = (umulhi(x, m) + x) >> s
// with s = ceil(log2 d), m = floor(2^32 (2^s - d) / d) + 1 (set on the host by make_fastdiv).
struct FastDiv {
  uint32_t m = 0, s = 0;
};
inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f;
  while ((1ull << f.s) < d) ++f.s;
  f.m = (uint32_t)((((1ull << 32) * ((1ull << f.s) - d)) / d) + 1);
  return f;
}
#ifdef __CUDACC__
__device__ __forceinline__ uint32_t fdiv(uint32_t x, FastDiv f) { return (__umulhi(x, f.m) + x) >> f.s; }
#endif

struct LamGemm {
  int M, N, K, K0;
  int nb[4];
  int kdim;
  int lam_c[3][5];
  int w_c[2][5];
  long long out_c[5], res_c[5];
  long long ldn_out, ldn_res;
  // output column n goes to (n / n_split) * split_stride + (n % n_split) * ldn_out
  // (both Λ planes of a McCormick x-side term in one N range); n_split = 0: no split
  int n_split;
  long long split_stride;
  float* out;
  const float* res;
  float alpha;
  // tiles whose batch coordinate b[alpha_r_dim1 - 1] == 1 (the radius plane of an affine) are
  // scaled by alpha_r instead of alpha; alpha_r_dim1 = 0 (zero-initialised LamGemm): alpha everywhere
  int alpha_r_dim1;
  float alpha_r;
  int accumulate;
  int tiles_m, tiles_n, num_tiles;  // set by launch_lam_gemm
  int epi_groups;                   // epilogue warp groups draining tiles (1 or 2; launch_lam_gemm)
  // optional K-row mask (keep[b0 * K + k] == 0: Λ row k of batch row b0 is zero, whatever the
  // buffer holds; written by elementwise_verify's `keep`): the split warps zero those rows
  const unsigned char* kmask;
  // 1: the split Λ operand is staged in tensor memory instead of shared memory (tcgen05.mma
  // with A from TMEM; N tile 128, single CTA): shared memory then carries only the W operand
  // stages, the raw Λ ring and the tensor core's W reads
  int tmem_a;
  int pair_b0;  // CTA pair over batch rows 2b, 2b + 1 instead of d-tiles (M = 128; launch_lam_gemm)
  // optional gather of batch coordinate b2 (sparse first-layer McCormick terms): when set,
  // b2 <- gather[slot_map[b0] * gather_ld + b2] (the perturbed token of word b2 of sentence b0)
  const int* gather;
  const int* gather_slot;
  int gather_ld;
  // M folding for D = 64 (M = 64 < the 128 TMEM lanes): when fold1 > 0, consecutive pairs of
  // batch coordinate b[fold1 - 1] (e.g. two token rows) fill the upper / lower 64 lanes of one
  // 128-row tile; the Λ tensor map then has a 64-wide box (umma_tmap_lam with dims[0] = 64)
  int fold1;
  // early exit: tiles of a sentence slot whose status word is already set (a relaxation raised
  // a domain / validation error earlier in the pass) are skipped; slot = b[0] / skip_div, for
  // skip_slots <= 1024 slots (the kernel keeps a bitmask of them in shared memory)
  const int* skip_status;
  int skip_div, skip_slots;
  int skip_tiles_per_b0, skip_b0_scale;  // set by launch_lam_gemm
  // divisors of the tile decode, set by launch_lam_gemm
  FastDiv f_tn, f_tm, f_nb1, f_nb2, f_nb3, f_skip_t, f_skip_div, f_nsplit;
};
bool umma_available();
int umma_pick_bn(int N);  // 256 / 128 / 64, or 0 when N is not a multiple of 64
bool umma_tmap_lam(void* tm, const float* base, const unsigned long long dims[4],
                   const unsigned long long strides_bytes[3], int kdim);
bool umma_tmap_wop(void* tm, const float* base, int K, int N, int P2, int P3, int bn);
// tm2_whi / tm2_wlo: the same operands mapped with box height bn/2 (one CTA's half of a W tile);
// when given and M % 256 == 0 the CTA-pair (cta_group::2, M = 256) kernel runs.
int launch_lam_gemm(const void* tm_lam, const void* tm_whi, const void* tm_wlo, LamGemm p, int bn,
                    cudaStream_t st, const void* tm2_whi = nullptr, const void* tm2_wlo = nullptr);
// dense tcgen05 peak microbenchmark: kind 0 = kind::tf32, 1 = kind::f16 (bf16); returns CTAs launched
int launch_mma_peak(int kind, int iters, cudaStream_t st);
int launch_ref_affine_f64(const float* W, const float* X, long long x_cr, double* Y, int C, int O, int D,
                          long long rows, cudaStream_t st);

// McCormick coefficient matrices split into TF32 hi/lo, K-major, per (sentence, head):
//   sim_x [S*H][2][L][2hd]   x-side of Q.K^T (rows j, K = (c | r) of the Q slice)
//   sim_y [S*H][2][L][hd]    y-side (lx, |lx| of Q rows i)
//   wv_x  [S*H][2][hd][2L]   x-side of P.V (rows k, K = (c | r) of the P rows)
//   wv_y  [S*H][2][L][L]     y-side (lx, |lx| of P, rows i, K = j)
int launch_sim_coef_split(const NView& q, const NView& k, int S, int H, int L, int hd, int kp, float* x_hi,
                          float* x_lo, float* y_hi, float* y_lo, cudaStream_t st);
int launch_wv_coef_split(const NView& p, const NView& v, int S, int H, int L, int hd, float* x_hi,
                         float* x_lo, float* y_hi, float* y_lo, cudaStream_t st);
int launch_sim_bias(const NView& q, const NView& k, const NView& out, int S, int H, int L, int hd,
                    double scale, cudaStream_t st);
int launch_wv_bias(const NView& p, const NView& v, const NView& out, int S, int H, int L, int hd,
                   cudaStream_t st);

// ---- exact f64 operator kernels (fg_exact.cu; FG_PRECISION_F64 mode of the operator ABI) ----
// Reference layout: lw/uw [n, d] row-major f64, lb/ub [n] f64; reference operation order.
struct XDotArgs {
  const double *alw, *alb, *auw, *aub, *alo;        // operand a (+ concretized lo)
  const double *blw, *blb, *buw, *bub, *blo, *bhi;  // operand b (+ concretized lo, hi)
  double *ylw, *ylb, *yuw, *yub;
  int layout;  // 0 = pairwise similarity, 1 = weighted values
  long long batch;
  int len, e, heads, d;
};
int launch_x_affine(const double* xlw, const double* xlb, const double* xuw, const double* xub, const double* w,
                    const double* bias, double* ylw, double* ylb, double* yuw, double* yub, long long rows, int c,
                    int o, int d, cudaStream_t st);
int launch_x_concretize(const double* lw, const double* lb, const double* uw, const double* ub, long long n,
                        int d, int norm, double eps, double* lo, double* hi, cudaStream_t st);
int launch_x_compose(const double* xlw, const double* xlb, const double* xuw, const double* xub,
                     const double* a_low, const double* b_low, const double* a_up, const double* b_up, double* ylw,
                     double* ylb, double* yuw, double* yub, long long n, int d, cudaStream_t st);
int launch_x_dot(const XDotArgs& a, cudaStream_t st);
// x = operand a [outer, n, inner], r = operand b [outer, 1, inner]
int launch_x_mul_broadcast(const XDotArgs& a, long long outer, int n, long long inner, cudaStream_t st);
int launch_x_sum_axis(const double* xlw, const double* xlb, const double* xuw, const double* xub, double* ylw,
                      double* ylb, double* yuw, double* yub, long long outer, int n, long long inner, int d,
                      cudaStream_t st);
int launch_x_add(const double* a, const double* b, double* y, long long n, cudaStream_t st);
int launch_x_scale(const double* xl, const double* xu, double s, double* yl, double* yu, long long n,
                   cudaStream_t st);
// out6 = lo_x, lo_y, lo_c, up_x, up_y, up_c (each n); status <- kCodeInval if lo > hi
int launch_x_bilinear(const double* xlo, const double* xhi, const double* ylo, const double* yhi, double* out6,
                      long long n, int* status, cudaStream_t st);

// ---- column-sharded pass (fg_kernels.cu): partial norms / finish, softmax in 5 phases ----
int launch_partial_norms(const float* lam, long long cr, long long nrows, int D, int norm, double* part,
                         cudaStream_t st);
int launch_finish_concretize(const double* part, const double* lb, const double* ub, long long rows_per_s,
                             long long nrows, int norm, const double* eps, double* lo, double* hi, cudaStream_t st);
int reduce_op_for_norm(int norm);  // all-reduce op of the partials: 0 SUM, 1 MAX
struct SmShardBufs {
  double* p_key;   // [2][nSC] per-key partial norms (exp input, later outputs)
  double* p_row;   // [2][rows] Σ partial norms
  double* p_row2;  // [2][rows] r partial norms
  double* ex;      // [5][nSC] a_lo, a_up, e_lb, e_ub, e_lo
  double* sig;     // [rows][2][D] Σ rows, then r rows
  double* sb;      // [2][rows] Σ_j e_lb, Σ_j e_ub
  double* rb;      // [6][rows] r_al, r_au, r_lb, r_ub, r_lo, r_hi
};
// phase 0: key partials -> (all-reduce p_key) -> 1 -> (p_row) -> 2 -> (p_row2) -> 3 -> (p_key) -> 4
int launch_sm_shard(int phase, const NView& sc, int S, int rows_per_s, int n, int D, int norm, const double* eps,
                    int* status, int site_exp, int site_recip, SmShardBufs b, cudaStream_t st);
int launch_head_partial(const double* pc, const double* pr, const double* plb, const double* pub, const double* wc,
                        const double* bc, int S, int E, int C, int D, int norm, double* part, double* bias,
                        cudaStream_t st);
int launch_head_finish(const double* part, const double* bias, int S, int C, int norm, const double* eps,
                       double* out_lo, double* out_hi, int* status, int site, cudaStream_t st);

// ---- exact f64 forward on the GPU (fg_forward.cu): the soundness oracle at full sizes ----
int launch_dense_f64(const double* X, const double* W, const double* b, const double* R, double* Y, long long rows,
                     int C, int O, int act, cudaStream_t st);  // act: RELAX_RELU/TANH/SILU or -1
int launch_attention_f64(const double* qkv, double* ctx, long long N, int L, int E, int H, cudaStream_t st);
int launch_pool_head_f64(const double* x, const double* wc, const double* bc, double* logits, long long N, int L,
                         int E, int C, cudaStream_t st);

}  // namespace fg
