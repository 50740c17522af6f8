#!/usr/bin/env python
"""Diagnostic: status of the bound pass along the bisection's upper probes (eps = 2^-k), per
config -- how many of a search's probes end in a domain error, and at which site."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_12708_b200 import faith_gpu as F  # noqa: E402
from paper_2209_12708_b200.configs import CONFIGS  # noqa: E402

ctx = F.Context(0)
for name in sys.argv[1:] or ["c2", "c3"]:
    w = CONFIGS[name]
    cfg = F.ModelConfig(w.layers, w.heads, w.embed, w.ffn, w.length, w.classes, w.activation)
    m = F.Model(ctx, cfg, F.gen_synthetic(cfg, w.model_seed))
    n = 32
    xs = np.stack([F.gen_input(cfg, w.input_seed(s)) for s in range(n)])
    ps = np.stack([F.gen_positions(w.position_seed(s), w.length, w.words) for s in range(n)])
    r = m.maxeps(xs, ps, w.norm, w.eps_max, w.tol)
    print(name, "eps* median", float(np.median(r["eps"])), flush=True)
    for k in range(0, 12):
        eps = 2.0 ** -k
        lo, hi, st = m.bound_pass(xs, ps, w.norm, np.full(n, eps))
        print(f"  eps 2^-{k}: domain/invalid {int(np.sum(st != 0))}/{n}", flush=True)
