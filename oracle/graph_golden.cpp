// TEST INFRASTRUCTURE ONLY (oracle/Makefile target `graphs`): golden faith-graph/v1 cases from the
// UNMODIFIED reference.  For each case it writes the graph exactly as graph::to_json emits it
// (proj/src/graph.cpp:781-814) and, per perturbation spec, the result of graph::evaluate
// (graph.cpp:505-673) -- lb/ub/lw/uw of the sink, or the exception it raised.
//   * random verification workloads: proj/tests/workloads.hpp random_workload, seeded and drawn
//     exactly as acceptance.cpp:215-225 does (Rng(2026), len 3, e 4, input random_tensor 0.5),
//     both as built (split / per-side affine forms) and after graph::fuse_all;
//   * the transformer graph of model::build_graph (model.cpp:393-448) for a gen_synthetic model,
//     unfused and fused.
// Usage: make -C oracle graphs && oracle/_ref/graph_golden tests/golden/graphs
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include <json.hpp>

#include "faith/graph.hpp"
#include "faith/model.hpp"
#include "workloads.hpp"

using namespace faith;
using nlohmann::json;

namespace {

json tensor_json(const Tensor& t) {
  return json{{"shape", t.shape()}, {"data", std::vector<double>(t.data(), t.data() + t.numel())}};
}

const char* golden_norm_name(Norm n) { return n == Norm::L1 ? "l1" : (n == Norm::L2 ? "l2" : "linf"); }

json run(const graph::VerGraph& g, const Tensor& x, Norm norm, double eps) {
  json r{{"norm", golden_norm_name(norm)}, {"eps", eps}, {"dim", x.numel()}};
  try {
    PerturbationSpec spec(norm, eps, x.numel());
    LinearBounds b = graph::evaluate(g, {{"x", x}}, spec);
    r["lb"] = tensor_json(b.lb);
    r["ub"] = tensor_json(b.ub);
    r["lw"] = tensor_json(b.lw);
    r["uw"] = tensor_json(b.uw);
  } catch (const std::invalid_argument& e) {
    r["error"] = "invalid_argument";
    r["what"] = e.what();
  } catch (const std::domain_error& e) {
    r["error"] = "domain_error";
    r["what"] = e.what();
  }
  return r;
}

void emit(const std::string& dir, const std::string& name, const graph::VerGraph& g, const Tensor& x,
          const std::vector<std::pair<Norm, double>>& specs) {
  {
    std::ofstream f(dir + "/" + name + ".graph.json");
    f << graph::to_json(g) << "\n";
  }
  json c{{"graph", name + ".graph.json"}, {"input", tensor_json(x)}, {"runs", json::array()}};
  for (const auto& [n, e] : specs) c["runs"].push_back(run(g, x, n, e));
  std::ofstream f(dir + "/" + name + ".expect.json");
  f << c.dump() << "\n";
}

}  // namespace

int main(int argc, char** argv) {
  if (argc != 2) {
    std::fprintf(stderr, "usage: %s <out_dir>\n", argv[0]);
    return 2;
  }
  const std::string dir = argv[1];
  const std::vector<std::pair<Norm, double>> specs = {
      {Norm::LInf, 0.02}, {Norm::L2, 0.05}, {Norm::L1, 0.1}, {Norm::LInf, 0.0}, {Norm::LInf, 3.0}, {Norm::LInf, 60.0}};
  Rng rng(2026);
  for (int rep = 0; rep < 12; ++rep) {
    graph::VerGraph g = testing::random_workload(rng, 3, 4);
    graph::VerGraph fused = graph::fuse_all(g);
    Tensor x = testing::random_tensor(rng, {1, 3, 4}, 0.5);
    emit(dir, "random" + std::to_string(rep), g, x, specs);
    emit(dir, "random" + std::to_string(rep) + "_fused", fused, x, specs);
  }
  for (const char* act : {"relu", "tanh", "silu"}) {
    model::SyntheticConfig c;
    c.num_layers = 1;
    c.num_heads = 2;
    c.embed_dim = 8;
    c.ffn_dim = 16;
    c.length = 4;
    c.num_classes = 2;
    c.activation = model::activation_from_name(act);
    model::TransformerSpec spec = model::gen_synthetic(77, c);
    Tensor x = model::gen_synthetic_input(78, spec);
    graph::VerGraph g = model::build_graph(spec);
    const std::vector<std::pair<Norm, double>> ts = {{Norm::LInf, 0.01}, {Norm::L2, 0.02}, {Norm::L1, 0.05}};
    emit(dir, std::string("transformer_") + act, g, x, ts);
    emit(dir, std::string("transformer_") + act + "_fused", graph::fuse_all(g), x, ts);
  }
  return 0;
}
