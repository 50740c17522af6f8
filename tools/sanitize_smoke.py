#!/usr/bin/env python
"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
every kernel family of the library on shapes small enough for the sanitizer's slowdown.

  compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
  compute-sanitizer --tool racecheck python tools/sanitize_smoke.py --part fused

Parts: fused (word-level bound pass, batched, CUDA graph; tcgen05 GEMMs, streaming softmax),
exact (reference-order f64 pass), search (fg_maxeps with exact re-decisions and the eps = 0
workspace), ops (operator level, both precisions).
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2209_12708_b200 import faith_gpu as F  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--part", default="fused,exact,search,ops")
a = ap.parse_args()
parts = a.part.split(",")
ctx = F.Context(0)
# c4-shaped mini (8 heads, 128 tokens) at E 128 / F 256 / D 128: tcgen05 engine + streaming softmax;
# c1 shape (D 64): FP32 SIMT GEMMs and the narrow-row softmax
shapes = [(F.ModelConfig(1, 8, 128, 256, 128, 2, "relu"), 1, "linf", 1e-4),
          (F.ModelConfig(1, 4, 64, 128, 32, 2, "relu"), 1, "l2", 0.01)]
for cfg, words, norm, eps in shapes:
    m = F.Model(ctx, cfg, F.gen_synthetic(cfg, 7))
    xs = np.stack([F.gen_input(cfg, 100 + s) for s in range(2)])
    ps = np.stack([F.gen_positions(200 + s, cfg.length, words) for s in range(2)])
    if "fused" in parts:
        m.bound_pass(xs, ps, norm, [eps, 2 * eps])
        m.bound_pass_dump(xs[0], ps[0], norm, eps)
    if "exact" in parts:
        m.bound_pass_exact(xs[0], ps[0], norm, eps, dump=True)
    if "search" in parts:
        m.maxeps(xs, ps, norm, 1.0, 1e-2)
        m.certify(xs, ps, norm, [eps, eps])
    print(f"ok {cfg.embed}x{cfg.length}", flush=True)
if "ops" in parts:
    rng = np.random.default_rng(3)
    for precision in ("f32", "f64"):
        ctx.set_precision(precision)
        lw = rng.uniform(-1, 1, (5, 3))
        lb = rng.normal(size=5)
        x = (lw, lb, lw.copy(), lb + 2.0)  # consistent bounds (lb <= ub)
        ctx.concretize(x, "l2", 0.1)
        ctx.propagate_affine(x, rng.normal(size=(5, 4)), rng.normal(size=4))
        ctx.elementwise_verify("relu", x, "linf", 0.05)
        lam, x0 = rng.uniform(-0.2, 0.2, (2, 8, 3)), rng.normal(size=(2, 8))
        ctx.propagate_layernorm((lam, x0, lam.copy(), x0.copy()), np.ones(8), np.zeros(8), "l2", 0.01)
    print("ok ops", flush=True)
print("sanitize smoke done", flush=True)
