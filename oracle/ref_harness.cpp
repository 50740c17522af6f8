// ref_harness.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Exposes the C interface of oracle/faith_oracle.h on top of the UNMODIFIED
// reference library (/root/reference/proj/src/*.cpp compiled by
// oracle/Makefile into oracle/_ref/).  Nothing here re-implements bound
// arithmetic: every operator call goes to faith::relax::* / faith::concretize
// / faith::model::*.  The only additions are the ones SURVEY.md 0.1 requires:
//   G1  word-level input binding (Λ0 rows of the W perturbed positions one-hot
//       into D = W*E columns) -- done here because graph::evaluate hard-codes
//       input_bounds (graph.cpp:523-529);
//   G2  >6-layer weight generation with the gen_synthetic draw order
//       (model.cpp:99-131) because TransformerSpec::validate caps layers at 6.
// The node walk mirrors graph::evaluate over fuse_all(build_graph(spec))
// (graph.cpp:531-661); fo_ref_selfcheck() proves it equals graph::evaluate
// bit-for-bit in the reference's own whole-embedding mode.
#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <thread>
#include <vector>

#include "faith/bounds.hpp"
#include "faith/cli.hpp"
#include "faith/graph.hpp"
#include "faith/model.hpp"
#include "faith/relax.hpp"
#include "faith/rng.hpp"
#include "faith/tensor.hpp"
#include "faith_oracle.h"

using namespace faith;
namespace rx = faith::relax;
namespace md = faith::model;

namespace {

Norm to_norm(int p) {
  return p == FO_NORM_L1 ? Norm::L1 : (p == FO_NORM_L2 ? Norm::L2 : Norm::LInf);
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return FO_OK;
  } catch (const std::domain_error&) {
    return FO_EDOMAIN;
  } catch (const std::invalid_argument&) {
    return FO_EINVAL;
  } catch (const std::out_of_range&) {
    return FO_ERANGE;
  } catch (const std::exception&) {
    return FO_ERUNTIME;
  }
}

Tensor tensor_from(std::vector<std::size_t> shape, const double* p) {
  std::size_t n = shape_numel(shape);
  return Tensor(std::move(shape), std::vector<double>(p, p + n));
}

LinearBounds bounds_from(std::vector<std::size_t> nshape, std::size_t d, const double* lw,
                         const double* lb, const double* uw, const double* ub) {
  std::vector<std::size_t> wshape = nshape;
  wshape.push_back(d);
  LinearBounds b;
  b.lw = tensor_from(wshape, lw);
  b.uw = tensor_from(wshape, uw);
  b.lb = tensor_from(nshape, lb);
  b.ub = tensor_from(nshape, ub);
  return b;
}

void export_bounds(const LinearBounds& b, double* lw, double* lb, double* uw, double* ub) {
  std::memcpy(lw, b.lw.data(), b.lw.numel() * sizeof(double));
  std::memcpy(uw, b.uw.data(), b.uw.numel() * sizeof(double));
  std::memcpy(lb, b.lb.data(), b.lb.numel() * sizeof(double));
  std::memcpy(ub, b.ub.data(), b.ub.numel() * sizeof(double));
}

md::TransformerSpec spec_from(const fo_config* c, const double* p) {
  md::TransformerSpec s;
  s.num_layers = c->layers;
  s.num_heads = c->heads;
  s.embed_dim = c->embed;
  s.ffn_dim = c->ffn;
  s.length = c->length;
  s.num_classes = c->classes;
  s.activation = c->activation == FO_ACT_TANH   ? md::Activation::Tanh
                 : c->activation == FO_ACT_SILU ? md::Activation::SiLU
                                                : md::Activation::ReLU;
  std::size_t e = c->embed, f = c->ffn, k = c->classes;
  auto take = [&](std::vector<std::size_t> shape) {
    Tensor t = tensor_from(shape, p);
    p += t.numel();
    return t;
  };
  for (int l = 0; l < c->layers; ++l) {
    md::LayerWeights w;
    w.wq = take({e, e}); w.bq = take({e});
    w.wk = take({e, e}); w.bk = take({e});
    w.wv = take({e, e}); w.bv = take({e});
    w.wo = take({e, e}); w.bo = take({e});
    w.w1 = take({e, f}); w.b1 = take({f});
    w.w2 = take({f, e}); w.b2 = take({e});
    s.layers.push_back(std::move(w));
  }
  s.wc = take({e, k});
  s.bc = take({k});
  return s;
}

// Node walk of graph::evaluate over fuse_all(build_graph(spec)), reference
// operators only.  `x0` is the already-bound input (word-level or identity).
struct StopWalk {};  // prefix budget reached (fo_bound_pass_prefix)

struct Walk {
  const md::TransformerSpec& s;
  PerturbationSpec ps;
  double* node_lo;
  double* node_hi;
  int max_nodes = 0;
  int count = 0;
  std::size_t off = 0;
  std::function<void()> gate;  // paced walks (fo_paced_*): called before every node

  void dump(const LinearBounds& b) {
    if (max_nodes > 0 && ++count >= max_nodes) throw StopWalk{};
    if (gate) gate();
    if (!node_lo) return;
    ConcreteBounds c = concretize(b, ps);
    std::memcpy(node_lo + off, c.lo.data(), c.lo.numel() * sizeof(double));
    std::memcpy(node_hi + off, c.hi.data(), c.hi.numel() * sizeof(double));
    off += c.lo.numel();
  }

  LinearBounds elementwise(const LinearBounds& x, md::Activation a) {
    ConcreteBounds c = concretize(x, ps);  // graph.cpp:484-501
    switch (a) {
      case md::Activation::Tanh: return rx::compose_elementwise(x, rx::relax_tanh(c));
      case md::Activation::SiLU: return rx::compose_elementwise(x, rx::relax_silu(c));
      default: return rx::compose_elementwise(x, rx::relax_relu(c));
    }
  }

  LinearBounds run(LinearBounds cur) {
    if (gate) gate();
    std::size_t L = s.length;
    // Every value is released after its last consumer, as graph::evaluate does
    // (graph.cpp:655-660), so the deep / wide shapes (c5) fit in host memory.
    auto drop = [](LinearBounds& b) { b = LinearBounds(); };
    for (const md::LayerWeights& w : s.layers) {
      LinearBounds v, probs;
      {
        LinearBounds q = rx::propagate_affine(cur, w.wq, &w.bq); dump(q);
        LinearBounds k = rx::propagate_affine(cur, w.wk, &w.bk); dump(k);
        v = rx::propagate_affine(cur, w.wv, &w.bv); dump(v);
        LinearBounds scores = rx::propagate_dot_product(q, k, ps, rx::DotLayout::PairwiseSimilarity,
                                                        s.num_heads);
        dump(scores);
        drop(q);
        drop(k);
        LinearBounds scaled =
            rx::propagate_scale(scores, 1.0 / std::sqrt(static_cast<double>(s.head_dim())));
        dump(scaled);
        drop(scores);
        // expand_softmax (graph.cpp:209-244), evaluated node by node.
        ConcreteBounds cs = concretize(scaled, ps);
        LinearBounds e = rx::compose_elementwise(scaled, rx::relax_exp(cs)); dump(e);
        drop(scaled);
        LinearBounds sm = rx::propagate_sum_axis(e, 3); dump(sm);
        ConcreteBounds css = concretize(sm, ps);
        LinearBounds r = rx::compose_elementwise(sm, rx::relax_recip(css)); dump(r);
        probs = rx::propagate_mul_broadcast(e, r, 3, ps); dump(probs);
      }
      LinearBounds ctx = rx::propagate_dot_product(probs, v, ps, rx::DotLayout::WeightedValues,
                                                   s.num_heads);
      dump(ctx);
      drop(probs);
      drop(v);
      LinearBounds attn = rx::propagate_affine(ctx, w.wo, &w.bo); dump(attn);
      drop(ctx);
      LinearBounds res1 = rx::propagate_add(cur, attn); dump(res1);
      drop(cur);
      drop(attn);
      LinearBounds act;
      {
        LinearBounds f1 = rx::propagate_affine(res1, w.w1, &w.b1); dump(f1);
        act = elementwise(f1, s.activation); dump(act);
      }
      LinearBounds f2 = rx::propagate_affine(act, w.w2, &w.b2); dump(f2);
      drop(act);
      cur = rx::propagate_add(res1, f2); dump(cur);
    }
    LinearBounds pooled = rx::propagate_scale(rx::propagate_sum_axis(cur, 1),
                                              1.0 / static_cast<double>(L));  // graph.cpp:628-634
    dump(pooled);
    LinearBounds logits = rx::propagate_affine(pooled, s.wc, &s.bc);
    dump(logits);
    logits.validate("evaluate result");
    for (const Tensor* t : {&logits.lb, &logits.ub, &logits.lw, &logits.uw})
      for (std::size_t i = 0; i < t->numel(); ++i)
        if (!std::isfinite((*t)[i])) throw std::domain_error("evaluate: bounds overflowed");
    return logits;
  }
};

LinearBounds word_input(const md::TransformerSpec& s, const double* x, const int* pos, int words) {
  std::size_t L = s.length, E = s.embed_dim, D = static_cast<std::size_t>(words) * E;
  LinearBounds b;
  b.lb = tensor_from({1, L, E}, x);
  b.ub = b.lb;
  b.lw = Tensor::zeros({1, L, E, D});
  b.uw = Tensor::zeros({1, L, E, D});
  for (int w = 0; w < words; ++w)
    for (std::size_t e = 0; e < E; ++e) {
      std::size_t row = static_cast<std::size_t>(pos[w]) * E + e, col = w * E + e;
      b.lw[row * D + col] = 1.0;
      b.uw[row * D + col] = 1.0;
    }
  return b;
}

std::size_t argmax(const double* v, std::size_t n) {
  std::size_t best = 0;
  for (std::size_t i = 1; i < n; ++i)
    if (v[i] > v[best]) best = i;
  return best;
}

}  // namespace

extern "C" {

const char* fo_impl_name(void) { return "reference"; }

size_t fo_param_count(const fo_config* c) {
  std::size_t e = c->embed, f = c->ffn, k = c->classes;
  return c->layers * (4 * (e * e + e) + e * f + f + f * e + e) + e * k + k;
}

int fo_gen_model(const fo_config* c, uint64_t seed, double* out) {
  return guarded([&] {
    if (c->layers <= 6) {
      md::SyntheticConfig sc;
      sc.num_layers = c->layers;
      sc.num_heads = c->heads;
      sc.embed_dim = c->embed;
      sc.ffn_dim = c->ffn;
      sc.length = c->length;
      sc.num_classes = c->classes;
      md::TransformerSpec s = md::gen_synthetic(seed, sc);
      auto put = [&](const Tensor& t) {
        std::memcpy(out, t.data(), t.numel() * sizeof(double));
        out += t.numel();
      };
      for (const auto& w : s.layers) {
        put(w.wq); put(w.bq); put(w.wk); put(w.bk); put(w.wv); put(w.bv);
        put(w.wo); put(w.bo); put(w.w1); put(w.b1); put(w.w2); put(w.b2);
      }
      put(s.wc);
      put(s.bc);
      return;
    }
    // G2: same Rng and draw order as gen_tensor (model.cpp:87-95) without validate().
    Rng rng(seed);
    std::size_t e = c->embed, f = c->ffn, k = c->classes;
    auto gen = [&](std::size_t n, std::size_t fan_in) {
      double bound = 0.5 / std::sqrt(static_cast<double>(fan_in));
      for (std::size_t i = 0; i < n; ++i)
        *out++ = static_cast<double>(static_cast<float>(rng.uniform(-bound, bound)));
    };
    for (int l = 0; l < c->layers; ++l) {
      gen(e * e, e); gen(e, e); gen(e * e, e); gen(e, e); gen(e * e, e); gen(e, e);
      gen(e * e, e); gen(e, e); gen(e * f, e); gen(f, e); gen(f * e, f); gen(e, f);
    }
    gen(e * k, e);
    gen(k, e);
  });
}

int fo_gen_input(const fo_config* c, uint64_t seed, double* x) {
  return guarded([&] {
    md::TransformerSpec s;
    s.length = c->length;
    s.embed_dim = c->embed;
    Tensor t = md::gen_synthetic_input(seed, s);
    std::memcpy(x, t.data(), t.numel() * sizeof(double));
  });
}

int fo_gen_positions(uint64_t seed, int length, int words, int* pos) {
  if (words < 1 || words > length) return FO_EINVAL;
  Rng rng(seed);
  int n = 0;
  while (n < words) {
    int v = static_cast<int>(rng.uniform_index(static_cast<std::uint64_t>(length)));
    bool dup = false;
    for (int i = 0; i < n; ++i) dup |= pos[i] == v;
    if (!dup) pos[n++] = v;
  }
  std::sort(pos, pos + n);
  return FO_OK;
}

int fo_rng_uniform(uint64_t seed, size_t n, double* out) {
  Rng rng(seed);
  for (size_t i = 0; i < n; ++i) out[i] = rng.uniform();
  return FO_OK;
}

int fo_forward(const fo_config* c, const double* params, const double* x, double* logits) {
  return guarded([&] {
    md::TransformerSpec s = spec_from(c, params);  // validate(): <= 6 layers (G2)
    Tensor t = md::forward(s, tensor_from({1, (std::size_t)c->length, (std::size_t)c->embed}, x));
    std::memcpy(logits, t.data(), t.numel() * sizeof(double));
  });
}

int fo_concretize(size_t n, size_t d, const double* lw, const double* lb, const double* uw,
                  const double* ub, int norm, double eps, double* lo, double* hi) {
  return guarded([&] {
    ConcreteBounds c = concretize(bounds_from({n}, d, lw, lb, uw, ub),
                                  PerturbationSpec(to_norm(norm), eps, d ? d : 1));
    std::memcpy(lo, c.lo.data(), n * sizeof(double));
    std::memcpy(hi, c.hi.data(), n * sizeof(double));
  });
}

int fo_check_robust(size_t n, const double* lo, const double* hi, size_t t, double margin,
                    int* verified) {
  return guarded([&] {
    ConcreteBounds c;
    c.lo = tensor_from({n}, lo);
    c.hi = tensor_from({n}, hi);
    *verified = check_robust(c, t, margin) ? 1 : 0;
  });
}

int fo_affine(size_t rows, size_t c, size_t o, size_t d, const double* xlw, const double* xlb,
              const double* xuw, const double* xub, const double* w, const double* bias,
              double* ylw, double* ylb, double* yuw, double* yub) {
  return guarded([&] {
    Tensor wt = tensor_from({c, o}, w);
    Tensor bt;
    if (bias) bt = tensor_from({o}, bias);
    LinearBounds y = rx::propagate_affine(bounds_from({rows, c}, d, xlw, xlb, xuw, xub), wt,
                                          bias ? &bt : nullptr);
    export_bounds(y, ylw, ylb, yuw, yub);
  });
}

static rx::ElementwiseLinearRelaxation relax_kind(int kind, const ConcreteBounds& c) {
  switch (kind) {
    case FO_RELAX_RELU: return rx::relax_relu(c);
    case FO_RELAX_TANH: return rx::relax_tanh(c);
    case FO_RELAX_SILU: return rx::relax_silu(c);
    case FO_RELAX_EXP: return rx::relax_exp(c);
    case FO_RELAX_RECIP: return rx::relax_recip(c);
  }
  throw std::invalid_argument("relax: unknown kind");
}

int fo_relax(int kind, size_t n, const double* lo, const double* hi, double* a_low,
             double* b_low, double* a_up, double* b_up) {
  return guarded([&] {
    ConcreteBounds c;
    c.lo = tensor_from({n}, lo);
    c.hi = tensor_from({n}, hi);
    rx::ElementwiseLinearRelaxation r = relax_kind(kind, c);
    std::memcpy(a_low, r.a_low.data(), n * sizeof(double));
    std::memcpy(b_low, r.b_low.data(), n * sizeof(double));
    std::memcpy(a_up, r.a_up.data(), n * sizeof(double));
    std::memcpy(b_up, r.b_up.data(), n * sizeof(double));
  });
}

int fo_compose(size_t n, size_t d, const double* xlw, const double* xlb, const double* xuw,
               const double* xub, const double* a_low, const double* b_low,
               const double* a_up, const double* b_up, double* ylw, double* ylb, double* yuw,
               double* yub) {
  return guarded([&] {
    rx::ElementwiseLinearRelaxation r;
    r.a_low = tensor_from({n}, a_low);
    r.b_low = tensor_from({n}, b_low);
    r.a_up = tensor_from({n}, a_up);
    r.b_up = tensor_from({n}, b_up);
    export_bounds(rx::compose_elementwise(bounds_from({n}, d, xlw, xlb, xuw, xub), r), ylw, ylb,
                  yuw, yub);
  });
}

int fo_elementwise_verify(int kind, size_t n, size_t d, const double* xlw, const double* xlb,
                          const double* xuw, const double* xub, int norm, double eps,
                          double* ylw, double* ylb, double* yuw, double* yub) {
  return guarded([&] {
    LinearBounds x = bounds_from({n}, d, xlw, xlb, xuw, xub);
    ConcreteBounds c = concretize(x, PerturbationSpec(to_norm(norm), eps, d ? d : 1));
    export_bounds(rx::compose_elementwise(x, relax_kind(kind, c)), ylw, ylb, yuw, yub);
  });
}

int fo_dot(int layout, size_t len, size_t embed, size_t heads, size_t d, const double* alw,
           const double* alb, const double* auw, const double* aub, const double* blw,
           const double* blb, const double* buw, const double* bub, int norm, double eps,
           double* ylw, double* ylb, double* yuw, double* yub) {
  return guarded([&] {
    PerturbationSpec ps(to_norm(norm), eps, d ? d : 1);
    LinearBounds a = layout == FO_DOT_SIMILARITY
                         ? bounds_from({1, len, embed}, d, alw, alb, auw, aub)
                         : bounds_from({1, heads, len, len}, d, alw, alb, auw, aub);
    LinearBounds b = bounds_from({1, len, embed}, d, blw, blb, buw, bub);
    LinearBounds y = rx::propagate_dot_product(
        a, b, ps,
        layout == FO_DOT_SIMILARITY ? rx::DotLayout::PairwiseSimilarity
                                    : rx::DotLayout::WeightedValues,
        heads);
    export_bounds(y, ylw, ylb, yuw, yub);
  });
}

int fo_softmax(size_t rows, size_t n, size_t d, const double* xlw, const double* xlb,
               const double* xuw, const double* xub, int norm, double eps, double* ylw,
               double* ylb, double* yuw, double* yub) {
  return guarded([&] {
    PerturbationSpec ps(to_norm(norm), eps, d ? d : 1);
    LinearBounds y =
        rx::propagate_softmax(bounds_from({rows, n}, d, xlw, xlb, xuw, xub), 1, ps);
    export_bounds(y, ylw, ylb, yuw, yub);
  });
}

size_t fo_node_dump_size(const fo_config* c) {
  std::size_t L = c->length, E = c->embed, H = c->heads, F = c->ffn;
  return c->layers * (8 * L * E + 4 * H * L * L + 2 * H * L + 2 * L * F) + E + c->classes;
}

int fo_bound_pass(const fo_config* c, const double* params, const double* x,
                  const int* positions, int words, int norm, double eps, double* logits_lo,
                  double* logits_hi, double* node_lo, double* node_hi) {
  return guarded([&] {
    md::TransformerSpec s = spec_from(c, params);
    std::size_t D = static_cast<std::size_t>(words) * c->embed;
    Walk walk{s, PerturbationSpec(to_norm(norm), eps, D), node_lo, node_hi};
    LinearBounds out = walk.run(word_input(s, x, positions, words));
    ConcreteBounds cb = concretize(out, walk.ps);
    std::memcpy(logits_lo, cb.lo.data(), cb.lo.numel() * sizeof(double));
    std::memcpy(logits_hi, cb.hi.data(), cb.hi.numel() * sizeof(double));
  });
}

int fo_bound_pass_prefix(const fo_config* c, const double* params, const double* x,
                         const int* positions, int words, int norm, double eps, int max_nodes) {
  bool stopped = false;
  int st = guarded([&] {
    md::TransformerSpec s = spec_from(c, params);
    std::size_t D = static_cast<std::size_t>(words) * c->embed;
    Walk walk{s, PerturbationSpec(to_norm(norm), eps, D), nullptr, nullptr, max_nodes};
    try {
      walk.run(word_input(s, x, positions, words));
    } catch (const StopWalk&) {
      stopped = true;
    }
  });
  return stopped ? FO_STOPPED : st;
}

int fo_maxeps(const fo_config* c, const double* params, const double* x, const int* positions,
              int words, int norm, double eps_max, double tol, double* eps_out, int* calls_out,
              int* predicted_out) {
  // cmd_maxeps (cli.cpp:135-193) with the word-level pass in place of
  // graph::evaluate(g, {{"x", x}}, pspec).
  return guarded([&] {
    std::size_t C = c->classes;
    std::vector<double> logits(C), lo(C), hi(C);
    md::TransformerSpec s = spec_from(c, params);
    Tensor t = md::forward(s, tensor_from({1, (std::size_t)c->length, (std::size_t)c->embed}, x));
    std::size_t predicted = argmax(t.data(), C);
    *predicted_out = static_cast<int>(predicted);
    int calls = 0;
    auto verified_at = [&](double eps, bool tolerate) {
      ++calls;
      try {
        std::size_t D = static_cast<std::size_t>(words) * c->embed;
        Walk walk{s, PerturbationSpec(to_norm(norm), eps, D), nullptr, nullptr};
        LinearBounds out = walk.run(word_input(s, x, positions, words));
        return check_robust(concretize(out, walk.ps), predicted, 0.0);
      } catch (const std::domain_error&) {
        if (!tolerate) throw;
        return false;
      } catch (const std::invalid_argument&) {
        if (!tolerate) throw;
        return false;
      }
    };
    if (!verified_at(0.0, false)) throw std::runtime_error("misclassified input");
    double result;
    if (verified_at(eps_max, true)) {
      result = eps_max;
    } else {
      double l = 0.0, h = eps_max;
      while (h - l > tol) {
        double mid = 0.5 * (l + h);
        if (verified_at(mid, true)) l = mid;
        else h = mid;
      }
      result = l;
    }
    *eps_out = result;
    *calls_out = calls;
  });
}

// Self-check: in the reference's whole-embedding mode (D = L*E, Λ0 = I) the
// harness walk must equal graph::evaluate(fuse_all(build_graph(spec)))
// bit-for-bit.  Returns 1 when equal, 0 when not, negative on error.
int fo_ref_selfcheck(const fo_config* c, const double* params, const double* x, int norm,
                     double eps) {
  int result = -1;
  int st = guarded([&] {
    md::TransformerSpec s = spec_from(c, params);
    Tensor xt = tensor_from({1, (std::size_t)c->length, (std::size_t)c->embed}, x);
    PerturbationSpec ps(to_norm(norm), eps, xt.numel());
    LinearBounds want = graph::evaluate(graph::fuse_all(md::build_graph(s)), {{"x", xt}}, ps);
    Walk walk{s, ps, nullptr, nullptr};
    LinearBounds got = walk.run(input_bounds(xt, ps));
    auto same = [](const Tensor& a, const Tensor& b) {
      return a.numel() == b.numel() &&
             std::memcmp(a.data(), b.data(), a.numel() * sizeof(double)) == 0;
    };
    result = same(want.lb, got.lb) && same(want.ub, got.ub) && same(want.lw, got.lw) &&
             same(want.uw, got.uw);
  });
  return st == FO_OK ? result : -st;
}


// ---- paced walks (bench.py --impl reference) ------------------------------------------------
// A full word-level pass of the unmodified reference, run on its own thread and advanced a
// given number of nodes per call, so that one complete pass per host core can be spread over
// the timed steps of a benchmark run instead of being extrapolated from a prefix.
struct fo_paced {
  std::mutex mu;
  std::condition_variable cv;
  int allowed = 0, done = 0;  // gates the walk may pass / has passed (one before every node)
  bool at_gate = false, finished = false, cancel = false;
  int status = FO_OK;
  std::vector<double> lo, hi;
  std::thread th;
};

fo_paced* fo_paced_begin(const fo_config* c, const double* params, const double* x, const int* positions,
                         int words, int norm, double eps) {
  auto* p = new fo_paced();
  md::TransformerSpec s = spec_from(c, params);
  std::vector<double> xv(x, x + static_cast<std::size_t>(c->length) * c->embed);
  std::vector<int> pv(positions, positions + words);
  p->lo.resize(c->classes);
  p->hi.resize(c->classes);
  p->th = std::thread([p, s = std::move(s), xv = std::move(xv), pv = std::move(pv), words, norm, eps]() {
    int st = guarded([&] {
      std::size_t D = static_cast<std::size_t>(words) * s.embed_dim;
      Walk walk{s, PerturbationSpec(to_norm(norm), eps, D), nullptr, nullptr};
      walk.gate = [p] {  // the previous node is complete; wait for an allowance for the next one
        std::unique_lock<std::mutex> lk(p->mu);
        p->at_gate = true;
        p->cv.notify_all();
        p->cv.wait(lk, [p] { return p->cancel || p->done < p->allowed; });
        p->at_gate = false;
        if (p->cancel) throw StopWalk{};
        ++p->done;
      };
      try {
        LinearBounds out = walk.run(word_input(s, xv.data(), pv.data(), words));
        ConcreteBounds cb = concretize(out, walk.ps);
        std::copy(cb.lo.data(), cb.lo.data() + cb.lo.numel(), p->lo.begin());
        std::copy(cb.hi.data(), cb.hi.data() + cb.hi.numel(), p->hi.begin());
      } catch (const StopWalk&) {
        throw std::runtime_error("paced walk cancelled");
      }
    });
    std::lock_guard<std::mutex> lk(p->mu);
    p->status = st;
    p->finished = true;
    p->cv.notify_all();
  });
  return p;
}

// Lets each of the n walks run `nodes` more nodes and waits until all of them have finished
// those nodes (or the whole pass).  Returns the number of walks that finished.
int fo_paced_step(fo_paced** walks, int n, int nodes) {
  for (int i = 0; i < n; ++i) {
    std::lock_guard<std::mutex> lk(walks[i]->mu);
    walks[i]->allowed += nodes;
    walks[i]->cv.notify_all();
  }
  int fin = 0;
  for (int i = 0; i < n; ++i) {
    fo_paced* p = walks[i];
    std::unique_lock<std::mutex> lk(p->mu);
    // the allowed nodes are complete when the walk waits at the gate after them (or finished)
    p->cv.wait(lk, [p] { return p->finished || (p->at_gate && p->done >= p->allowed); });
    fin += p->finished ? 1 : 0;
  }
  return fin;
}

// Lets the walk run to completion (finish != 0) or stops it at its next node (finish == 0:
// status FO_ERUNTIME); joins the thread and returns the walk's status.
int fo_paced_end(fo_paced* p, int finish, double* logits_lo, double* logits_hi) {
  {
    std::lock_guard<std::mutex> lk(p->mu);
    p->allowed = 1 << 30;
    p->cancel = finish == 0;
    p->cv.notify_all();
  }
  p->th.join();
  int st = p->status;
  if (logits_lo) std::copy(p->lo.begin(), p->lo.end(), logits_lo);
  if (logits_hi) std::copy(p->hi.begin(), p->hi.end(), logits_hi);
  delete p;
  return st;
}

}  // extern "C"
