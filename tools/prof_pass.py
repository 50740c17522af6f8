#!/usr/bin/env python
"""Profiling driver (not a benchmark): stages S synthetic sentences of a workload and runs
a few batched bound passes through the C ABI, so `ncu -k regex:<kernel>` can capture one
launch of a pass kernel.

  python tools/prof_pass.py [--config c3] [--sentences 32] [--passes 3]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2209_12708_b200 import faith_gpu as F  # noqa: E402
from paper_2209_12708_b200.configs import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--sentences", type=int, default=32)
    ap.add_argument("--passes", type=int, default=3)
    a = ap.parse_args()
    w = CONFIGS[a.config]
    cfg = F.ModelConfig(w.layers, w.heads, w.embed, w.ffn, w.length, w.classes, w.activation)
    params = F.gen_synthetic(cfg, w.model_seed)
    x = np.stack([F.gen_input(cfg, w.input_seed(s)) for s in range(a.sentences)])
    pos = np.stack([F.gen_positions(w.position_seed(s), w.length, w.words) for s in range(a.sentences)])
    ctx = F.Context(0)
    model = F.Model(ctx, cfg, params)
    for _ in range(a.passes):
        model.bound_pass(x, pos, w.norm, [w.eps] * a.sentences)
    print("stats", model.last_stats())
    prof = model.profile_pass(w.norm, w.eps)
    print("sites", {k: round(v[0], 3) for k, v in prof.items()})


if __name__ == "__main__":
    main()
