// TEST INFRASTRUCTURE.  A minimal argument front-end for the reference's own command bodies
// (proj/src/cli.cpp: cmd_verify, cmd_maxeps) and its model generator/serialisers
// (proj/src/model.cpp), standing in for tools/faith_main.cpp, whose CLI11 dependency is
// absent here.  Linked against the UNMODIFIED reference objects; whether the bound operators
// come from the reference (libfaith_ref) or from the GPU drop-in (libfaith_compat) is decided
// at link time (oracle/Makefile targets faith_cli_ref / faith_cli_gpu).
//
//   gen       --layers N --heads H --embed E --ffn F --length L --classes C --act relu|tanh|silu
//             --seed S --model OUT.json [--input-seed S2 --input OUT2.json]
//   verify    --model M --input X --eps E --norm l1|l2|linf [--margin m] [--naive] [--out R.json]
//   maxeps    --model M --input X --norm N [--tol t] [--eps-max e] [--out R.json]
// and, in the GPU build (-DFAITH_FUSED), the pass-level fast path on the same files:
//   verify-fused / maxeps-fused   same options, faith::gpu::FusedVerifier (whole bound passes on
//                                 the B200, f32 Λ + f64 O(N) state), same output lines
#include <cstdio>
#include <cstdlib>
#include <map>
#include <stdexcept>
#include <string>

#include "faith/cli.hpp"
#include "faith/model.hpp"
#ifdef FAITH_FUSED
#include "faith_fused.hpp"
#endif

using namespace faith;

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s gen|verify|maxeps --key value ...\n", argv[0]);
    return 2;
  }
  const std::string cmd = argv[1];
  std::map<std::string, std::string> a;
  for (int i = 2; i < argc; ++i) {
    std::string k = argv[i];
    if (k.rfind("--", 0) != 0) continue;
    k = k.substr(2);
    if (i + 1 < argc && std::string(argv[i + 1]).rfind("--", 0) != 0) a[k] = argv[++i];
    else a[k] = "1";
  }
  auto get = [&](const char* k, const char* def) { return a.count(k) ? a[k] : std::string(def); };
  try {
    if (cmd == "gen") {
      model::SyntheticConfig c;
      c.num_layers = std::stoul(get("layers", "1"));
      c.num_heads = std::stoul(get("heads", "4"));
      c.embed_dim = std::stoul(get("embed", "64"));
      c.ffn_dim = std::stoul(get("ffn", "0"));
      c.length = std::stoul(get("length", "16"));
      c.num_classes = std::stoul(get("classes", "2"));
      c.activation = model::activation_from_name(get("act", "relu"));
      model::TransformerSpec spec = model::gen_synthetic(std::stoull(get("seed", "1")), c);
      model::save_model(spec, get("model", "model.json"));
      if (a.count("input"))
        model::save_embedding(model::gen_synthetic_input(std::stoull(get("input-seed", "2")), spec), a["input"]);
      return 0;
    }
    if (cmd == "verify") {
      cli::VerifyOptions o;
      o.model_path = get("model", "");
      o.input_path = get("input", "");
      o.out_path = get("out", "");
      o.epsilon = std::stod(get("eps", "0"));
      o.norm = norm_from_name(get("norm", "linf"));
      o.margin = std::stod(get("margin", "0"));
      o.fused = !a.count("naive");
      return cli::cmd_verify(o);
    }
    if (cmd == "maxeps") {
      cli::MaxEpsOptions o;
      o.model_path = get("model", "");
      o.input_path = get("input", "");
      o.out_path = get("out", "");
      o.norm = norm_from_name(get("norm", "linf"));
      o.tol = std::stod(get("tol", "1e-3"));
      o.eps_max = std::stod(get("eps-max", "1.0"));
      return cli::cmd_maxeps(o);
    }
#ifdef FAITH_FUSED
    if (cmd == "verify-fused" || cmd == "maxeps-fused") {
      model::TransformerSpec spec = model::load_model(get("model", ""));
      Tensor x = model::load_embedding(get("input", ""));
      gpu::FusedVerifier fv(spec);
      const Norm p = norm_from_name(get("norm", "linf"));
      if (cmd == "verify-fused") {
        const double eps = std::stod(get("eps", "0"));
        bool bounded = true;
        std::size_t cls = 0;
        const bool ok = fv.certify(x, p, eps, std::stod(get("margin", "0")), &cls, nullptr, &bounded);
        std::printf("%s eps=%g norm=%s class=%zu\n", ok ? "verified" : "not verified", eps, norm_name(p).c_str(), cls);
        return ok ? 0 : 1;
      }
      auto r = fv.max_epsilon({x}, p, std::stod(get("eps-max", "1.0")), std::stod(get("tol", "1e-3")));
      std::printf("max verified epsilon = %g (%zu calls)\n", r[0].epsilon, r[0].calls);
      return 0;
    }
#endif
  } catch (const std::exception& e) {
    std::fprintf(stderr, "%s: %s\n", cmd.c_str(), e.what());
    return 2;
  }
  std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
  return 2;
}
