"""TEST INFRASTRUCTURE ONLY: generates tests/golden/ from the reference build.

Runs the UNMODIFIED reference (oracle/_ref/libfaith_ref.so, built from /root/reference by
oracle/Makefile) on the BASELINE workloads and writes small fixtures:

  <cfg>_pass_s<s>.npz   one word-level bound pass at the config's fixed ε (or --eps):
                        logits lo/hi, status, and the concretized lo/hi of every node
                        (float64, bit-exact; a strided subsample of the values for the
                        larger configs) in fo_bound_pass order
  <cfg>_maxeps_s<s>.json cmd_maxeps result (ε, verification calls, predicted class)

Usage: python oracle/make_golden.py c1|c2|c3|c4m|c4|c5s [--what pass|maxeps] [--sentence S] [--eps E]

c4 and c5s are walked at a radius below the BASELINE one (--eps): on random-init weights the
bound width grows ~1e3x per layer at E >= 512 (profiles/r1_width_growth_by_depth.txt), so at
the BASELINE radius the reference's own walk ends in an exp-envelope domain error;
tools/golden_eps_scan.py picks the radius at which the walk is bounded with O(1e-2..1)
logit widths.
"""
import argparse, json, os, sys, time
import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.oracle import Oracle, ModelConfig  # noqa: E402
from paper_2209_12708_b200.configs import ALL as CONFIGS  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
# every value for c1-c3; a prime stride over the flattened node dump for the big ones
STRIDE = {"c1": 1, "c2": 1, "c3": 1, "c4m": 7, "c4": 61, "c5s": 29}


def model_config(w):
    return ModelConfig(w.layers, w.heads, w.embed, w.ffn, w.length, w.classes, w.activation)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg")
    ap.add_argument("--what", default="pass")
    ap.add_argument("--sentence", type=int, default=0)
    ap.add_argument("--impl", default="reference")
    ap.add_argument("--eps", type=float, default=None, help="pass radius (default: the config's)")
    a = ap.parse_args()
    w = CONFIGS[a.cfg]
    o = Oracle(a.impl)
    cfg = model_config(w)
    params = o.gen_model(cfg, w.model_seed)
    s = a.sentence
    x = o.gen_input(cfg, w.input_seed(s))
    pos = o.gen_positions(w.position_seed(s), w.length, w.words)
    os.makedirs(OUT, exist_ok=True)
    t0 = time.time()
    if a.what == "pass":
        eps = w.eps if a.eps is None else a.eps
        st, lo, hi, nlo, nhi = o.bound_pass(cfg, params, x, pos, w.norm, eps, dump=True)
        idx = np.arange(0, len(nlo), STRIDE[a.cfg])
        np.savez_compressed(os.path.join(OUT, f"{a.cfg}_pass_s{s}.npz"), status=st, eps=eps, norm=w.norm,
                            logits_lo=lo, logits_hi=hi, node_index=idx.astype(np.int64),
                            node_lo=nlo[idx], node_hi=nhi[idx],
                            positions=pos, impl=o.impl)
        print(f"{a.cfg} pass s{s} eps {eps:g}: status {st} logits lo {lo} hi {hi} ({time.time()-t0:.1f}s)")
    else:
        st, eps, calls, pred = o.maxeps(cfg, params, x, pos, w.norm, w.eps_max, w.tol)
        rec = {"config": a.cfg, "sentence": s, "status": st, "max_epsilon": eps, "calls": calls,
               "predicted": pred, "eps_max": w.eps_max, "tol": w.tol, "norm": w.norm,
               "positions": pos.tolist(), "impl": o.impl, "seconds": time.time() - t0}
        with open(os.path.join(OUT, f"{a.cfg}_maxeps_s{s}.json"), "w") as f:
            json.dump(rec, f, indent=1)
        print(json.dumps(rec))


if __name__ == "__main__":
    main()
