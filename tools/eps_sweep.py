#!/usr/bin/env python
"""Diagnostic (not a benchmark): batched bound-pass device time and per-site profile as a
function of epsilon (the bisection visits eps = 0, eps_max and midpoints).

  python tools/eps_sweep.py [--config c3] [--sentences 32]
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
    a = ap.parse_args()
    w = CONFIGS[a.config]
    cfg = F.ModelConfig(w.layers, w.heads, w.embed, w.ffn, w.length, w.classes, w.activation)
    params = F.gen_synthetic(cfg, w.model_seed)
    x = np.stack([F.gen_input(cfg, w.input_seed(s)) for s in range(a.sentences)])
    pos = np.stack([F.gen_positions(w.position_seed(s), w.length, w.words) for s in range(a.sentences)])
    model = F.Model(F.Context(0), cfg, params)
    for eps in (0.0, w.eps, 1e-4, 1e-2, 0.5, 1.0):
        ms = []
        for _ in range(4):
            _, _, st = model.bound_pass(x, pos, w.norm, [eps] * a.sentences)
            ms.append(model.last_stats()["pass_ms"])
        prof = model.profile_pass(w.norm, eps)
        print(f"eps {eps:g}: pass_ms {[round(v, 2) for v in ms]} status {np.bincount(st.astype(np.int64) + 8).nonzero()[0] - 8}"
              f" sites {sum(v[0] for v in prof.values()):.2f} " + str({k: round(v[0], 2) for k, v in prof.items()}),
              flush=True)


if __name__ == "__main__":
    main()
