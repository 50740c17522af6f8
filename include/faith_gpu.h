/*
 * faith_gpu.h -- C ABI of the B200-native bound-propagation library
 * (paper_2209_12708_b200/_lib/libfaith_gpu.so).
 *
 * Drop-in boundary for the hot path of the Faith verifier reproduction
 * (/root/reference/proj): the free functions of faith::relax / faith::
 * bounds ops that graph::evaluate calls node by node, the fused bound pass
 * that replaces graph::evaluate, and the certify / max-epsilon drivers that
 * replace cli::cmd_verify / cli::cmd_maxeps.  Plain pointers and sizes only.
 *
 * Two levels:
 *   (1) operator level -- host f64 buffers in the reference layout
 *       (faith::LinearBounds: lw/uw [n, d] row-major, lb/ub [n];
 *       proj/include/faith/bounds.hpp:34-45).  Each call uploads, runs the same
 *       CUDA kernels the fused pass uses, and downloads (value semantics, like
 *       the reference's const&-in / fresh-value-out functions).
 *   (2) model level -- weights uploaded once (fg_model_create); fg_bound_pass /
 *       fg_certify / fg_maxeps run whole verification passes for a batch of
 *       independent sentences with Λ resident in HBM.
 *
 * Errors: every entry returns an fg_status.  Numeric failures inside a pass are
 * reported per sentence with the same taxonomy as the reference's exceptions:
 *   FG_EINVAL  <- std::invalid_argument (shape mismatch; concretized lo > hi,
 *                 bounds.cpp:69-78)
 *   FG_EDOMAIN <- std::domain_error (relax_exp overflow relax.cpp:389-391,
 *                 relax_recip lo<=0 relax.cpp:406-409, non-finite result
 *                 graph.cpp:663-671)
 *   FG_ERANGE  <- std::out_of_range (check_robust true_class, bounds.cpp:144)
 * fg_last_error() returns a message for the last failing call on a context.
 * There is no CPU fallback: without a usable sm_100 device fg_ctx_create
 * fails with FG_ECUDA.
 */
#ifndef FAITH_GPU_H
#define FAITH_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int fg_status;
#define FG_OK 0
#define FG_EINVAL 1
#define FG_EDOMAIN 2
#define FG_ERANGE 3
#define FG_ERUNTIME 4 /* std::runtime_error, e.g. "misclassified input" in maxeps */
#define FG_ECUDA 5
#define FG_ENOMEM 6

/* faith::Norm (bounds.hpp:12): perturbation norm p; concretization uses dual(p) */
#define FG_NORM_L1 0
#define FG_NORM_L2 1
#define FG_NORM_LINF 2

/* elementwise relaxations (relax.hpp:62-66) */
#define FG_RELAX_RELU 0
#define FG_RELAX_TANH 1
#define FG_RELAX_SILU 2
#define FG_RELAX_EXP 3
#define FG_RELAX_RECIP 4
/* Extension (no reference counterpart): the envelopes of the LayerNorm bound chain.
 * sqrt on [lo, hi], lo >= 0 (else domain error): lower = chord, upper = tangent at the midpoint;
 * square: lower = tangent at the midpoint, upper = chord.  Usable wherever a relaxation kind is
 * (fg_relax, fg_elementwise_verify); Context.propagate_layernorm chains them. */
#define FG_RELAX_SQRT 5
#define FG_RELAX_SQUARE 6

/* faith::relax::DotLayout (relax.hpp:79) */
#define FG_DOT_SIMILARITY 0
#define FG_DOT_WEIGHTED_VALUES 1

/* Operator-level arithmetic of a context (fg_ctx_set_precision):
 *   FG_PRECISION_F32  Λ in f32 centre/radius planes, O(N) state (biases, concretized
 *                     bounds, envelope lines) in f64 -- the arithmetic of the fused pass;
 *                     results agree with the reference within 1e-4*max(1,|ref|).
 *   FG_PRECISION_F64  every operator in f64 in the reference's operation order (one thread
 *                     per output element, no FMA contraction): the arithmetic operators are
 *                     bit-identical to proj/src/relax.cpp / bounds.cpp, the exp/tanh/SiLU
 *                     envelopes agree to the device libm's last ulp.  The C++ drop-in layer
 *                     (compat/) uses this mode by default. */
#define FG_PRECISION_F32 0
#define FG_PRECISION_F64 1

typedef struct fg_ctx fg_ctx;
typedef struct fg_model fg_model;

/* ---- context ----------------------------------------------------------- */
/* One context per (host thread, device).  Fails with FG_ECUDA when the device
 * is absent or is not compute capability 10.x. */
fg_status fg_ctx_create(int device, fg_ctx** out);
void fg_ctx_destroy(fg_ctx* ctx);
const char* fg_last_error(const fg_ctx* ctx);
/* Operator-level precision of the context (FG_PRECISION_*; default F32).  Model-level
 * passes (fg_bound_pass / fg_certify / fg_maxeps) always run the F32 fused kernels. */
fg_status fg_ctx_set_precision(fg_ctx* ctx, int precision);
int fg_ctx_precision(const fg_ctx* ctx);
/* Number of kernels this context has launched so far (evidence counter). */
uint64_t fg_kernel_launches(const fg_ctx* ctx);
const char* fg_version(void);

/* ---- operator level (host buffers, reference layout) -------------------- */
/* concretize (bounds.cpp:122-140): lo = lb - eps*||lw||_q, hi = ub + eps*||uw||_q */
fg_status fg_concretize(fg_ctx* ctx, size_t n, size_t d, const double* lw, const double* lb,
                        const double* uw, const double* ub, int norm, double eps, double* lo,
                        double* hi);
/* check_robust (bounds.cpp:142-157); host-side, no device work */
fg_status fg_check_robust(size_t n, const double* lo, const double* hi, size_t true_class,
                          double margin, int* verified);
/* propagate_affine (relax.cpp:237-307): x is rows x c neurons, w [c, o] row-major,
 * bias [o] or NULL -> y rows x o neurons */
fg_status fg_affine(fg_ctx* ctx, size_t rows, size_t c, size_t o, size_t d, const double* xlw,
                    const double* xlb, const double* xuw, const double* xub, const double* w,
                    const double* bias, double* ylw, double* ylb, double* yuw, double* yub);
/* relax_{relu,tanh,silu,exp,recip} (relax.cpp:313-468) */
fg_status fg_relax(fg_ctx* ctx, int kind, size_t n, const double* lo, const double* hi,
                   double* a_low, double* b_low, double* a_up, double* b_up);
/* compose_elementwise (relax.cpp:470-497) */
fg_status fg_compose(fg_ctx* ctx, size_t n, size_t d, const double* xlw, const double* xlb,
                     const double* xuw, const double* xub, const double* a_low,
                     const double* b_low, const double* a_up, const double* b_up, double* ylw,
                     double* ylb, double* yuw, double* yub);
/* concretize -> relax_<kind> -> compose as one fused kernel (graph.cpp:484-501) */
fg_status fg_elementwise_verify(fg_ctx* ctx, int kind, size_t n, size_t d, const double* xlw,
                                const double* xlb, const double* xuw, const double* xub,
                                int norm, double eps, double* ylw, double* ylb, double* yuw,
                                double* yub);
/* propagate_dot_product (relax.cpp:573-654), batch 1:
 *   SIMILARITY:      a, b [len, embed]          -> y [heads, len, len]
 *   WEIGHTED_VALUES: a [heads, len, len], b [len, embed] -> y [len, embed] */
fg_status fg_dot(fg_ctx* ctx, int layout, size_t len, size_t embed, size_t heads, size_t d,
                 const double* alw, const double* alb, const double* auw, const double* aub,
                 const double* blw, const double* blb, const double* buw, const double* bub,
                 int norm, double eps, double* ylw, double* ylb, double* yuw, double* yub);
/* propagate_softmax along the last axis of [rows, n] (relax.cpp:777-790), evaluated as
 * the fused graph does (exp -> sum -> recip -> McCormick multiply, graph.cpp:237-240) */
fg_status fg_softmax(fg_ctx* ctx, size_t rows, size_t n, size_t d, const double* xlw,
                     const double* xlb, const double* xuw, const double* xub, int norm,
                     double eps, double* ylw, double* ylb, double* yuw, double* yub);
/* propagate_dot_product with a leading batch axis (relax.cpp:573-654): the same as fg_dot
 * for each of `batch` independent [len, ...] slices, which share the perturbation columns. */
fg_status fg_dot_batched(fg_ctx* ctx, int layout, size_t batch, size_t len, size_t embed, size_t heads,
                         size_t d, const double* alw, const double* alb, const double* auw,
                         const double* aub, const double* blw, const double* blb, const double* buw,
                         const double* bub, int norm, double eps, double* ylw, double* ylb, double* yuw,
                         double* yub);
/* propagate_softmax along the middle axis of [outer, n, inner] (relax.cpp:777-790).  F32
 * precision runs the fused single-read kernel when inner == 1; every other case runs the f64
 * operator chain exp -> sum -> recip -> McCormick multiply. */
fg_status fg_softmax_axis(fg_ctx* ctx, size_t outer, size_t n, size_t inner, size_t d,
                          const double* xlw, const double* xlb, const double* xuw, const double* xub,
                          int norm, double eps, double* ylw, double* ylb, double* yuw, double* yub);
/* propagate_sum_axis (relax.cpp:705-742): [outer, n, inner] -> [outer, 1, inner].  f64. */
fg_status fg_sum_axis(fg_ctx* ctx, size_t outer, size_t n, size_t inner, size_t d, const double* xlw,
                      const double* xlb, const double* xuw, const double* xub, double* ylw, double* ylb,
                      double* yuw, double* yub);
/* propagate_mul_broadcast (relax.cpp:744-775): x [outer, n, inner] times r [outer, 1, inner]
 * under McCormick planes of the concretized operands.  f64. */
fg_status fg_mul_broadcast(fg_ctx* ctx, size_t outer, size_t n, size_t inner, size_t d,
                           const double* xlw, const double* xlb, const double* xuw, const double* xub,
                           const double* rlw, const double* rlb, const double* ruw, const double* rub,
                           int norm, double eps, double* ylw, double* ylb, double* yuw, double* yub);
/* relax_bilinear (relax.cpp:499-523): McCormick planes of z = x*y on [xlo,xhi] x [ylo,yhi];
 * FG_EINVAL when lo > hi for either operand (ConcreteBounds::validate).  f64. */
fg_status fg_bilinear(fg_ctx* ctx, size_t n, const double* xlo, const double* xhi, const double* ylo,
                      const double* yhi, double* lo_x, double* lo_y, double* lo_c, double* up_x,
                      double* up_y, double* up_c);
/* propagate_add (relax.cpp:656-674) and propagate_scale (relax.cpp:676-703) */
fg_status fg_add(fg_ctx* ctx, size_t n, size_t d, const double* alw, const double* alb,
                 const double* auw, const double* aub, const double* blw, const double* blb,
                 const double* buw, const double* bub, double* ylw, double* ylb, double* yuw,
                 double* yub);
fg_status fg_scale(fg_ctx* ctx, size_t n, size_t d, const double* xlw, const double* xlb,
                   const double* xuw, const double* xub, double s, double* ylw, double* ylb,
                   double* yuw, double* yub);

/* ---- model level --------------------------------------------------------- */
typedef struct {
  int layers, heads, embed, ffn, length, classes, activation; /* activation: FG_RELAX_* of
                                                                  relu/tanh/silu */
} fg_config;

/* params: gen_synthetic order (model.cpp:99-131) -- per layer wq[E,E] bq wk bk wv bv wo bo
 * w1[E,F] b1 w2[F,E] b2, then wc[E,C] bc; row-major [in, out], f64 values (the reference
 * stores f32-rounded weights as f64, model.cpp:92). */
fg_status fg_model_create(fg_ctx* ctx, const fg_config* cfg, const double* params,
                          fg_model** out);
void fg_model_destroy(fg_model* model);
/* Exact f64 forward pass (model::forward, model.cpp:566-571) -> logits[classes]; host. */
fg_status fg_forward(fg_model* model, const double* x, double* logits);
/* The same function for N inputs on the GPU (f64 kernels, FMA-contracted: agrees with the
 * host forward to ~1e-13 relative): the soundness oracle for sampled perturbations at full
 * model sizes.  x [N, L, E] host, logits [N, classes] host. */
fg_status fg_forward_batch(fg_model* model, int N, const double* x, double* logits);

/* One word-level verification pass (graph::evaluate over fuse_all(build_graph), graph.cpp:
 * 505-673) for S independent sentences.  x [S, L, E] host f64; positions [S, words];
 * D = words*E perturbation columns.  eps[S] per sentence.  Outputs per
 * sentence: logits_lo/hi [S, classes] and status[S] (FG_OK / FG_EINVAL / FG_EDOMAIN). */
fg_status fg_bound_pass(fg_model* model, int S, const double* x, const int* positions, int words,
                        int norm, const double* eps, double* logits_lo, double* logits_hi,
                        int* status);
/* Debug/parity variant for ONE sentence: also writes the concretized lo/hi of the nodes
 * the fused pass materialises, in fo_bound_pass node order (oracle/faith_oracle.h);
 * entries for nodes that stay on chip are NaN.  node_lo/hi sized fg_node_dump_size(). */
size_t fg_node_dump_size(const fg_config* cfg);
fg_status fg_bound_pass_dump(fg_model* model, const double* x, const int* positions, int words,
                             int norm, double eps, double* logits_lo, double* logits_hi,
                             double* node_lo, double* node_hi, int* status);

/* The same pass in the exact precision mode (FG_PRECISION_F64 arithmetic: f64 Λ in the
 * reference layout, every operator in the reference's operation order, no FMA contraction) for
 * ONE sentence, entirely on the device.  Bit-identical to graph::evaluate + concretize for the
 * arithmetic operators; the exp/tanh/SiLU envelopes agree to an ulp or two of the device libm.
 * node_lo/node_hi (fg_node_dump_size() each) may be NULL; when given, every node's concretized
 * bounds are written in fo_bound_pass order (no NaN entries).  status as fg_bound_pass. */
fg_status fg_bound_pass_exact(fg_model* model, const double* x, const int* positions, int words,
                              int norm, double eps, double* logits_lo, double* logits_hi,
                              double* node_lo, double* node_hi, int* status);

/* Decision-exact verdicts.  fg_certify, fg_maxeps and fg_maxeps_spec decide every probe with
 * check_robust on the fused f32-Λ pass; a probe is AMBIGUOUS when for some class j != t its
 * margin m = lo_t - hi_j - margin lies in the model's error band of that pass,
 *   band_lo * W - f <= m <= band_hi * W + f,   W = (hi_t - lo_t) + (hi_j - lo_j),
 *   f = 1e-11 * max(1, |lo_t|, |hi_j|).
 * The band starts at [-kappa, kappa / 8] and is calibrated per model: every re-decided probe
 * gives a sample of (m_f32 - m_exact) / W, and after 16 samples the band is twice the observed
 * extremes (where a verdict can flip: [min(err, 0), max(err, 0)] * W) plus 1e-7, never wider
 * than the default, widened again by any later sample outside it.
 * Ambiguous probes are re-decided by fg_bound_pass_exact, so every verdict is the reference's.
 * kappa = 0 turns the re-decision off (raw f32 verdicts); setting kappa restarts calibration. */
#define FG_DEFAULT_KAPPA 6e-6
fg_status fg_model_set_exact_resolve(fg_model* model, double kappa);

/* What fg_maxeps does with a sentence while its ambiguous probe is re-decided (asynchronously,
 * on side streams).  PREDICTED (default): the sentence keeps its slot and bisects on with the
 * verdict its f32 margins predict after correcting them by the model's mean measured error;
 * when the exact verdict differs, the sentence is rolled back to that probe and advanced with
 * the exact verdict, and re-decisions started on the abandoned path are dropped.  VERIFIED /
 * FAILED: always guess that verdict (tests of the roll-back path).  OFF: the sentence leaves its
 * slot until the exact verdict is in.  Every mode returns the same eps / calls: only verdicts
 * confirmed by the exact pass stay on a sentence's bisection path. */
#define FG_SPECULATE_OFF 0
#define FG_SPECULATE_PREDICTED 1
#define FG_SPECULATE_VERIFIED 2
#define FG_SPECULATE_FAILED 3
fg_status fg_model_set_speculation(fg_model* model, int mode);

/* certify(sentence, p, eps) -- cmd_verify (cli.cpp:64-133) for S sentences:
 * predicted = argmax(forward); verified = check_robust(concretize(pass), predicted, margin).
 * bounded[s] = 0 when the pass raised a domain error (cli.cpp:92-94). */
fg_status fg_certify(fg_model* model, int S, const double* x, const int* positions, int words,
                     int norm, const double* eps, double margin, int* verified, int* bounded,
                     int* predicted, double* logits_lo, double* logits_hi, int* status);

/* cmd_maxeps (cli.cpp:135-193) for S sentences: per sentence the same bisection path
 * (verified_at(0) must hold, then eps_max, then midpoints while hi-lo > tol), all sentences
 * advancing together on the GPU (continuous batching over `slots` resident sentences;
 * slots <= 0 picks a default from free HBM).  status[s] = FG_ERUNTIME for a
 * misclassified input (cli.cpp:159-161).  When words*E > 128 and the model is not column
 * sharded, the eps = 0 probes of all S sentences run first on a second, 128-column workspace
 * whose Λ is identically zero (the verdict at eps = 0 does not depend on Λ); it stays
 * allocated with the model.  FG_NO_ZERO_PROBE=1 keeps them on the full-width workspace. */
fg_status fg_maxeps(fg_model* model, int S, const double* x, const int* positions, int words,
                    int norm, double eps_max, double tol, int slots, double* eps_out,
                    int* calls_out, int* predicted_out, int* status);

/* ---- column sharding -------------------------------------------------
 * The perturbation columns D = words*E of every Λ are split across `nranks` ranks (one GPU
 * each): rank r owns columns [r*D/nranks, (r+1)*D/nranks).  Every operator of the pass is
 * column-separable except concretization, whose partial q-norms (raw sums / sums of squares /
 * maxima) are all-reduced across the ranks at every concretization site: Q/K/V, the four
 * concretizations of the softmax chain, the FFN activation, the logits.  All O(N) state is
 * replicated, so every rank takes identical envelope decisions and returns identical results.
 * All ranks must call fg_bound_pass / fg_certify / fg_maxeps with the same arguments.
 * D must be a multiple of 4*nranks.  fg_bound_pass_dump is not available on a sharded model. */
#define FG_REDUCE_SUM 0
#define FG_REDUCE_MAX 1
/* In-place all-reduce of `count` doubles on device memory, stream-ordered on `cuda_stream`
 * (a cudaStream_t); returns 0 on success. */
typedef int (*fg_allreduce_fn)(void* user, double* buf, size_t count, int op, void* cuda_stream);
fg_status fg_model_set_column_shard(fg_model* model, int rank, int nranks, fg_allreduce_fn fn, void* user,
                                    int graph_capturable);
/* Built-in exchange over NCCL (ncclAllReduce, loaded at run time from libnccl.so.2): rank 0
 * creates the id, every rank passes the same 128 bytes (e.g. through torch.distributed). */
fg_status fg_nccl_unique_id(unsigned char id[128]);
fg_status fg_model_shard_nccl(fg_model* model, int rank, int nranks, const unsigned char id[128]);
/* Built-in in-process exchange: `nranks` models on ONE device, driven by one host thread each
 * (a deterministic rank-ordered reduction kernel between CUDA events); used to exercise the
 * sharded pass on a single GPU. */
typedef struct fg_loopback fg_loopback;
fg_status fg_loopback_create(int nranks, fg_loopback** out);
void fg_loopback_destroy(fg_loopback* group);
fg_status fg_model_shard_loopback(fg_model* model, fg_loopback* group, int rank);

/* Speculative ε bisection: the same decision path as fg_maxeps /
 * cmd_maxeps (cli.cpp:144-177), but each round evaluates a whole subtree of the next `depth`
 * bisection levels (2^depth - 1 midpoints, computed with the sequential algorithm's own
 * expressions) in one batched pass, then walks it -- the first round also carries the ε = 0
 * and ε = eps_max probes.  Latency per sentence drops from 2 + n passes to about 1 + n/depth
 * rounds for about 2^depth / depth times the work.  Multi-GPU: rank `rank` of `nranks`
 * evaluates the probes whose index % nranks == rank and `exchange` combines the per-probe
 * verdict words across ranks (element-wise MAX over ranks, in place; NULL when nranks == 1).
 * calls_out = verification calls on the decision path (what cmd_maxeps reports),
 * rounds_out = batched rounds used.  All ranks return identical results. */
typedef int (*fg_exchange_fn)(void* user, int* verdicts, size_t count);
fg_status fg_maxeps_spec(fg_model* model, int S, const double* x, const int* positions, int words, int norm,
                         double eps_max, double tol, int depth, int rank, int nranks, fg_exchange_fn exchange,
                         void* user, double* eps_out, int* calls_out, int* rounds_out, int* predicted_out,
                         int* status_out);

/* Synthetic model / inputs with the reference's seeded recipe (model.cpp:87-141):
 * gen_synthetic weights U(+-0.5/sqrt(fan_in)) rounded to f32, gen_synthetic_input
 * U(-0.5, 0.5); word positions = `words` distinct Rng(seed).uniform_index(length) draws,
 * sorted.  fg_param_count() doubles are written to params. */
size_t fg_param_count(const fg_config* cfg);
fg_status fg_gen_synthetic(const fg_config* cfg, uint64_t seed, double* params);
fg_status fg_gen_input(const fg_config* cfg, uint64_t seed, double* x);
fg_status fg_gen_positions(uint64_t seed, int length, int words, int* positions);

/* Profiling: one eager pass over the sentences resident from the last fg_maxeps /
 * fg_bound_pass call, with CUDA events around every launch site.  Writes up to
 * max_sites site names (32 chars each), device ms and kernel counts. */
fg_status fg_profile_pass(fg_model* model, int norm, double eps, int max_sites, char* names,
                          double* ms, int* kernels, int* nsites);

/* Self-test of the affine bound GEMM (propagate_affine's Λ contraction) on random data:
 * tcgen05 3xTF32 kernel and FP32 SIMT kernel vs an f64 device reference.  err_* =
 * max|Y - Y_ref| / max|Y_ref| (err_umma = -1 if the shape is not tcgen05-eligible:
 * O % 32, C % 32, D % 128 or D = 64 with an even row count -- token rows folded in pairs); ms_* = CUDA-event time of one launch; bias_umma[2] (may be NULL) =
 * median signed relative error of the tcgen05 centre / radius planes (radius inputs >= 0). */
fg_status fg_selftest_affine(fg_ctx* ctx, int rows, int C, int O, int D, uint64_t seed, double* err_umma,
                             double* err_simt, double* ms_umma, double* ms_simt, double* bias_umma);

/* Dense tensor-pipe peak on this device (the roofline denominator of the 3xTF32 GEMMs): one CTA
 * per SM issuing tcgen05.mma M=128 N=256 back to back on SMEM-resident operands, `iters` x 4
 * MMAs each.  kind 0 = kind::tf32, 1 = kind::f16 with bf16 operands.  ms = CUDA-event time,
 * tflops = 2*M*N*K*MMAs / time. */
fg_status fg_selftest_mma_peak(fg_ctx* ctx, int kind, int iters, double* ms, double* tflops);

/* Timing of the last fg_maxeps / fg_bound_pass call, measured with CUDA events on the
 * library's stream (device time), and pass counts. */
typedef struct {
  double device_ms;      /* total device time of the last call */
  double pass_ms;        /* mean device time of one batched bound pass */
  int passes;            /* batched passes run */
  int slots;             /* sentences resident per pass */
  uint64_t launches;     /* kernels launched by the last call */
  double sentence_passes;/* sentence-passes executed (sum over passes of active slots) */
  int exact_probes;      /* probes re-decided by the exact pass (fg_model_set_exact_resolve) */
  double exact_ms;       /* time spent in those exact passes (included in device_ms) */
  double band_lo, band_hi; /* the model's ambiguity band after the call (units of W) */
  int band_samples;      /* re-decided probes it was calibrated on so far */
  int spec_rollbacks;    /* fg_maxeps: speculative bisection steps whose guessed verdict the
                            exact re-decision overturned (the sentence was rolled back) */
} fg_run_stats;
fg_status fg_last_run_stats(const fg_model* model, fg_run_stats* out);

/* ---- verification-graph executor (faith-graph/v1) ------------------------
 * graph::evaluate (proj/src/graph.cpp:505-673) over an arbitrary verification graph:
 * every node -- the split (SplitSigns / MatmulPair / CombineHalves), per-side (AffineBound /
 * MergeSides) and fused (AffineVerify) affine forms, dot products, scales, adds, mean-pool,
 * the activation / exp / recip envelopes, Softmax, SumReduce and MulBroadcast -- runs on the
 * device in the exact f64 arithmetic of FG_PRECISION_F64 (reference operation order), with
 * every intermediate value resident in HBM and released after its last consumer, as the
 * reference does (graph.cpp:655-660).  The JSON schema (graph.cpp:781-850) is parsed on the
 * host (paper_2209_12708_b200/graph.py); this level takes the decoded node table. */
#define FG_NODE_INPUT 0
#define FG_NODE_WEIGHT 1
#define FG_NODE_SPLIT_SIGNS 2
#define FG_NODE_MATMUL_PAIR 3
#define FG_NODE_COMBINE_HALVES 4
#define FG_NODE_AFFINE_BOUND 5
#define FG_NODE_MERGE_SIDES 6
#define FG_NODE_AFFINE_VERIFY 7
#define FG_NODE_DOT_PRODUCT 8
#define FG_NODE_SCALE 9
#define FG_NODE_ADD 10
#define FG_NODE_MEAN_POOL 11
#define FG_NODE_RELU_VERIFY 12
#define FG_NODE_TANH_VERIFY 13
#define FG_NODE_SILU_VERIFY 14
#define FG_NODE_SOFTMAX 15
#define FG_NODE_EXP_VERIFY 16
#define FG_NODE_SUM_REDUCE 17
#define FG_NODE_RECIP_VERIFY 18
#define FG_NODE_MUL_BROADCAST 19
#define FG_GRAPH_MAX_RANK 8

typedef struct fg_graph fg_graph;
/* One node of graph::VerGraph (graph.hpp:59-75).  inputs[] in the reference's edge-role order
 * (graph.cpp:684-706): MatmulPair {x, halves}; CombineHalves {pos, neg[, bias]}; affine
 * {x, w[, bias]}; MergeSides / DotProduct / Add {a, b}; MulBroadcast {x, r}; others {x}. */
typedef struct {
  int kind;       /* FG_NODE_* */
  int n_inputs;   /* 0..3 */
  int inputs[3];  /* producer node ids, each < this node's index */
  int sign;       /* MatmulPair: 0 positive half, 1 negative half */
  int side;       /* AffineBound: 0 lower, 1 upper */
  int layout;     /* DotProduct: FG_DOT_* */
  int heads;      /* DotProduct */
  int axis;       /* Softmax / SumReduce / MulBroadcast / MeanPool */
  double scale;   /* Scale */
  int constant;   /* Weight: index into the constant table */
  int input;      /* Input: binding slot of fg_graph_evaluate */
} fg_node;
/* Constants (the Weight table) are uploaded once.  const_shape is [n_constants][FG_GRAPH_MAX_RANK].
 * Structural errors of VerGraph::validate (graph.cpp:133-160) -> FG_EINVAL. */
fg_status fg_graph_create(fg_ctx* ctx, size_t n_nodes, const fg_node* nodes, size_t n_constants,
                          const size_t* const_rank, const size_t* const_shape, const double* const* const_data,
                          fg_graph** out);
void fg_graph_destroy(fg_graph* graph);
/* Binds input slot i to the tensor (in_rank[i], in_shape[i][..], in_data[i]) -- input_bounds
 * (bounds.cpp:101-120): numel must equal dim -- and evaluates to the unique operator sink.
 * The result stays on the device until the next evaluate or destroy. */
fg_status fg_graph_evaluate(fg_graph* graph, size_t n_inputs, const size_t* in_rank, const size_t* in_shape,
                            const double* const* in_data, int norm, double eps, size_t dim);
fg_status fg_graph_result_shape(const fg_graph* graph, size_t* rank, size_t* shape, size_t* d);
fg_status fg_graph_result(fg_graph* graph, double* lw, double* lb, double* uw, double* ub);

#ifdef __cplusplus
}
#endif

#endif
