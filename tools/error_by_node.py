#!/usr/bin/env python
"""Diagnostic: where does the fused f32-Λ pass depart from the exact pass?  Per node, the
relative error of the bound widths (hi - lo) and of lo/hi relative to the node's widths, for
one sentence at one radius.

  python tools/error_by_node.py [--config c3] [--sentence 3] [--eps 0.0133342]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.oracle import ModelConfig as OCfg, node_layout  # noqa: E402
from paper_2209_12708_b200 import faith_gpu as F  # noqa: E402
from paper_2209_12708_b200.configs import ALL  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--sentence", type=int, default=3)
ap.add_argument("--eps", type=float, default=0.0133342742919921875)
a = ap.parse_args()
w = ALL[a.config]
cfg = F.ModelConfig(w.layers, w.heads, w.embed, w.ffn, w.length, w.classes, w.activation)
ocfg = OCfg(w.layers, w.heads, w.embed, w.ffn, w.length, w.classes, w.activation)
m = F.Model(F.Context(0), cfg, F.gen_synthetic(cfg, w.model_seed))
x, pos = F.gen_input(cfg, w.input_seed(a.sentence)), F.gen_positions(w.position_seed(a.sentence), w.length, w.words)
st, lo, hi, nlo, nhi = m.bound_pass_dump(x, pos, w.norm, a.eps)
est, elo, ehi, xlo, xhi = m.bound_pass_exact(x, pos, w.norm, a.eps, dump=True)
print(f"status {st}/{est}; logits f32 {lo} {hi}; exact {elo} {ehi}")
for nm, off, n in node_layout(ocfg):
    a32, b32 = nlo[off:off + n], nhi[off:off + n]
    if np.all(np.isnan(a32)):
        print(f"{nm:10s} (on chip)")
        continue
    a64, b64 = xlo[off:off + n], xhi[off:off + n]
    w64 = b64 - a64
    w32 = b32 - a32
    big = w64 > 1e-3 * np.max(w64)
    rw = np.abs(w32 - w64)[big] / w64[big]
    rl = np.abs(a32 - a64)[big] / w64[big]
    rh = np.abs(b32 - b64)[big] / w64[big]
    sgn = np.median(((w32 - w64)[big] / w64[big]))
    print(f"{nm:10s} width rel err median {np.median(rw):.2e} max {np.max(rw):.2e} signed median {sgn:+.2e} | "
          f"lo/width max {np.max(rl):.2e} hi/width max {np.max(rh):.2e}")
