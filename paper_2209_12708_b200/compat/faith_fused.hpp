// faith_fused.hpp -- pass-level fast path for the reference's own types.
//
// The operator-level drop-in (faith_compat.cpp) keeps graph::evaluate walking node by node on
// the host; this class hands whole bound passes of a faith::model::TransformerSpec (as loaded by
// model::load_model, model.cpp:285-335) to the fused B200 pass: weights uploaded once, Λ resident
// in HBM, sentences batched, CUDA-graph replay.  The perturbation is the reference's own
// whole-embedding ε-ball (input_bounds, bounds.cpp:101-120): D = L*E columns.
#pragma once

#include <cstddef>
#include <memory>
#include <vector>

#include "faith/bounds.hpp"
#include "faith/model.hpp"

namespace faith::gpu {

struct MaxEpsResult {
  double epsilon = 0.0;        // cmd_maxeps "max verified epsilon"
  std::size_t calls = 0;       // verification calls on the bisection path
  std::size_t predicted = 0;   // argmax of the exact forward
};

class FusedVerifier {
 public:
  explicit FusedVerifier(const model::TransformerSpec& spec, int device = 0);
  ~FusedVerifier();
  FusedVerifier(const FusedVerifier&) = delete;
  FusedVerifier& operator=(const FusedVerifier&) = delete;

  // cmd_verify (cli.cpp:64-133) for x [1, L, E]: concretized logit bounds at (p, eps); returns
  // check_robust(., argmax forward, margin).  bounded = false when the pass hit a domain error.
  bool certify(const Tensor& x, Norm p, double eps, double margin = 0.0, std::size_t* predicted = nullptr,
               ConcreteBounds* logits = nullptr, bool* bounded = nullptr);
  // cmd_maxeps (cli.cpp:135-193) for a batch of inputs, all advancing together on the GPU.
  std::vector<MaxEpsResult> max_epsilon(const std::vector<Tensor>& xs, Norm p, double eps_max, double tol);

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};

}  // namespace faith::gpu
