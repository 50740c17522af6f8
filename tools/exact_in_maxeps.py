#!/usr/bin/env python
"""Diagnostic: exact-pass wall time alone, interleaved with fused passes, and inside fg_maxeps."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_12708_b200 import faith_gpu as F  # noqa: E402
from paper_2209_12708_b200.configs import CONFIGS  # noqa: E402

w = CONFIGS["c3"]
cfg = F.ModelConfig(w.layers, w.heads, w.embed, w.ffn, w.length, w.classes, w.activation)
m = F.Model(F.Context(0), cfg, F.gen_synthetic(cfg, w.model_seed))
xs = np.stack([F.gen_input(cfg, w.input_seed(s)) for s in range(64)])
ps = np.stack([F.gen_positions(w.position_seed(s), w.length, w.words) for s in range(64)])


def exact_ms():
    t0 = time.perf_counter()
    m.bound_pass_exact(xs[0], ps[0], w.norm, 0.0123)
    return round(1e3 * (time.perf_counter() - t0), 1)


print("alone", [exact_ms() for _ in range(3)], flush=True)
out = []
for _ in range(4):
    m.bound_pass(xs, ps, w.norm, np.full(64, 0.0123))
    out.append(exact_ms())
print("interleaved with 64-sentence fused passes", out, flush=True)
for rep in range(3):
    m.maxeps(xs, ps, w.norm, w.eps_max, w.tol)
    st = m.last_stats()
    print("maxeps", round(st["device_ms"]), "ms, exact probes", st["exact_probes"], "exact ms",
          round(st["exact_ms"]), flush=True)
print("alone after", [exact_ms() for _ in range(3)], flush=True)
