// faith_fused.cpp -- faith::gpu::FusedVerifier over the model-level C ABI (see the header).
#include "faith_fused.hpp"

#include <stdexcept>
#include <string>

#include "faith_gpu.h"

namespace faith::gpu {

namespace {
int norm_code(Norm p) { return p == Norm::L1 ? FG_NORM_L1 : p == Norm::L2 ? FG_NORM_L2 : FG_NORM_LINF; }

void raise(fg_status s, fg_ctx* ctx, const std::string& what) {
  const std::string msg = what + ": " + (ctx ? fg_last_error(ctx) : "");
  if (s == FG_EINVAL) throw std::invalid_argument(msg);
  if (s == FG_EDOMAIN) throw std::domain_error(msg);
  if (s == FG_ERANGE) throw std::out_of_range(msg);
  throw std::runtime_error(msg);
}
}  // namespace

struct FusedVerifier::Impl {
  fg_ctx* ctx = nullptr;
  fg_model* model = nullptr;
  std::size_t length = 0, embed = 0, classes = 0;
  std::vector<int> positions;  // whole embedding: every token is a perturbed "word"
  ~Impl() {
    if (model) fg_model_destroy(model);
    if (ctx) fg_ctx_destroy(ctx);
  }
  void check_input(const Tensor& x) const {
    if (x.numel() != length * embed)
      throw std::runtime_error("input embedding " + x.shape_str() + " does not match the model");
  }
};

FusedVerifier::FusedVerifier(const model::TransformerSpec& spec, int device) : impl_(new Impl) {
  spec.validate();
  if (fg_ctx_create(device, &impl_->ctx) != FG_OK)
    throw std::runtime_error("faith-gpu: no usable sm_100 device (there is no CPU fallback)");
  const int act = spec.activation == model::Activation::ReLU   ? FG_RELAX_RELU
                  : spec.activation == model::Activation::Tanh ? FG_RELAX_TANH
                                                               : FG_RELAX_SILU;
  fg_config cfg{(int)spec.num_layers, (int)spec.num_heads, (int)spec.embed_dim, (int)spec.ffn_dim,
                (int)spec.length,     (int)spec.num_classes, act};
  std::vector<double> params;  // gen_synthetic order (model.cpp:99-131)
  auto put = [&](const Tensor& t) { params.insert(params.end(), t.data(), t.data() + t.numel()); };
  for (const model::LayerWeights& l : spec.layers) {
    for (const Tensor* t : {&l.wq, &l.bq, &l.wk, &l.bk, &l.wv, &l.bv, &l.wo, &l.bo, &l.w1, &l.b1, &l.w2, &l.b2})
      put(*t);
  }
  put(spec.wc);
  put(spec.bc);
  if (params.size() != fg_param_count(&cfg)) throw std::invalid_argument("FusedVerifier: parameter count mismatch");
  if (fg_status s = fg_model_create(impl_->ctx, &cfg, params.data(), &impl_->model))
    raise(s, impl_->ctx, "fg_model_create");
  impl_->length = spec.length;
  impl_->embed = spec.embed_dim;
  impl_->classes = spec.num_classes;
  for (std::size_t t = 0; t < spec.length; ++t) impl_->positions.push_back((int)t);
}

FusedVerifier::~FusedVerifier() = default;

bool FusedVerifier::certify(const Tensor& x, Norm p, double eps, double margin, std::size_t* predicted,
                            ConcreteBounds* logits, bool* bounded) {
  impl_->check_input(x);
  const std::size_t C = impl_->classes;
  std::vector<double> lo(C), hi(C);
  int verified = 0, bnd = 0, pred = 0, st = 0;
  if (fg_status s = fg_certify(impl_->model, 1, x.data(), impl_->positions.data(), (int)impl_->length, norm_code(p),
                               &eps, margin, &verified, &bnd, &pred, lo.data(), hi.data(), &st))
    raise(s, impl_->ctx, "fg_certify");
  if (st == FG_EINVAL) raise(st, impl_->ctx, "certify");
  if (bounded) *bounded = bnd != 0;
  if (predicted) *predicted = (std::size_t)pred;
  if (logits) {
    logits->lo = Tensor({1, 1, C}, lo);
    logits->hi = Tensor({1, 1, C}, hi);
  }
  return verified != 0;
}

std::vector<MaxEpsResult> FusedVerifier::max_epsilon(const std::vector<Tensor>& xs, Norm p, double eps_max,
                                                     double tol) {
  const int S = (int)xs.size();
  std::vector<double> x, eps(S);
  std::vector<int> pos, calls(S), pred(S), st(S);
  for (const Tensor& t : xs) {
    impl_->check_input(t);
    x.insert(x.end(), t.data(), t.data() + t.numel());
    pos.insert(pos.end(), impl_->positions.begin(), impl_->positions.end());
  }
  if (fg_status s = fg_maxeps(impl_->model, S, x.data(), pos.data(), (int)impl_->length, norm_code(p), eps_max, tol,
                              0, eps.data(), calls.data(), pred.data(), st.data()))
    raise(s, impl_->ctx, "fg_maxeps");
  std::vector<MaxEpsResult> out(S);
  for (int s = 0; s < S; ++s) {
    if (st[s] == FG_ERUNTIME) throw std::runtime_error("misclassified input: not verifiable at epsilon = 0");
    if (st[s] != FG_OK) raise(st[s], impl_->ctx, "max_epsilon");
    out[s] = {eps[s], (std::size_t)calls[s], (std::size_t)pred[s]};
  }
  return out;
}

}  // namespace faith::gpu
