"""Subprocess helper for test_gpu_variants.py: one fg_maxeps run under the environment it is
started with (the FG_* comparison knobs are read once per process), printed as one JSON line."""
import json
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tests/", 1)[0])
from paper_2209_12708_b200 import faith_gpu as F  # noqa: E402
from paper_2209_12708_b200.configs import CONFIGS  # noqa: E402


def main():
    name, n, slots = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    w = CONFIGS[name]
    cfg = F.ModelConfig(w.layers, w.heads, w.embed, w.ffn, w.length, w.classes, w.activation)
    m = F.Model(F.Context(0), cfg, F.gen_synthetic(cfg, w.model_seed))
    xs = np.stack([F.gen_input(cfg, w.input_seed(s)) for s in range(n)])
    ps = np.stack([F.gen_positions(w.position_seed(s), w.length, w.words) for s in range(n)])
    r = m.maxeps(xs, ps, w.norm, w.eps_max, 1e-4, slots=slots)
    out = {k: np.asarray(r[k]).tolist() for k in ("eps", "calls", "status", "predicted")}
    out["eps"] = [None if v != v else v for v in out["eps"]]  # NaN (no certificate) -> null
    print(json.dumps(out))


if __name__ == "__main__":
    main()
