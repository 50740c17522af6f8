#!/usr/bin/env python
"""Diagnostic: wall time of fg_bound_pass_exact for one sentence of a config (after a warm-up
call), for ncu launch lists of the exact pass (`--repeat 1`).

  python tools/exact_pass_time.py [--config c3] [--repeat 3]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2209_12708_b200 import faith_gpu as F  # noqa: E402
from paper_2209_12708_b200.configs import ALL  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--repeat", type=int, default=3)
a = ap.parse_args()
w = ALL[a.config]
cfg = F.ModelConfig(w.layers, w.heads, w.embed, w.ffn, w.length, w.classes, w.activation)
m = F.Model(F.Context(0), cfg, F.gen_synthetic(cfg, w.model_seed))
x, pos = F.gen_input(cfg, w.input_seed(0)), F.gen_positions(w.position_seed(0), w.length, w.words)
m.bound_pass_exact(x, pos, w.norm, w.eps)
for _ in range(a.repeat):
    t0 = time.perf_counter()
    m.bound_pass_exact(x, pos, w.norm, w.eps)
    print(f"{a.config} exact pass {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
