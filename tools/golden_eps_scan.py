#!/usr/bin/env python
"""Diagnostic (not a benchmark): where is a deep workload's bound pass still bounded?

Runs the GPU pass of sentence 0 over a grid of radii and prints the status and the bound
width (hi - lo) of the logits and of the widest node, so a golden radius can be picked at
which the reference's own walk stays finite and the widths are large enough to be a
non-trivial parity check (widths near 1e-9 would let a wrong Λ hide behind the biases).

  python tools/golden_eps_scan.py c4 c5s
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.oracle import ModelConfig as OCfg, node_layout  # noqa: E402
from paper_2209_12708_b200 import faith_gpu as F  # noqa: E402
from paper_2209_12708_b200.configs import ALL  # noqa: E402


def main():
    ctx = F.Context(0)
    for name in sys.argv[1:] or ["c4", "c5s"]:
        w = ALL[name]
        cfg = F.ModelConfig(w.layers, w.heads, w.embed, w.ffn, w.length, w.classes, w.activation)
        ocfg = OCfg(w.layers, w.heads, w.embed, w.ffn, w.length, w.classes, w.activation)
        m = F.Model(ctx, cfg, F.gen_synthetic(cfg, w.model_seed))
        x = F.gen_input(cfg, w.input_seed(0))
        pos = F.gen_positions(w.position_seed(0), w.length, w.words)
        for eps in (1e-3, 1e-4, 1e-5, 1e-6, 1e-7, 1e-8, 1e-9, 1e-10, 1e-11):
            st, lo, hi, nlo, nhi = m.bound_pass_dump(x, pos, w.norm, eps)
            widths = []
            for nm, off, n in node_layout(ocfg):
                d = nhi[off:off + n] - nlo[off:off + n]
                d = d[~np.isnan(d)]
                if d.size:
                    widths.append((nm, float(np.max(d))))
            top = max(widths, key=lambda t: t[1]) if widths else None
            print(f"{name} eps {eps:g}: status {st} logit width {np.max(hi - lo):.3e} widest node {top} "
                  f"last-layer res2 width {[v for k, v in widths if k.endswith('res2')][-1:]}", flush=True)


if __name__ == "__main__":
    main()
