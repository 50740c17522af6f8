#!/usr/bin/env python
"""Diagnostic: per-layer max scaled error of the fused pass and of the exact pass against a
golden pass of the reference (tests/golden/<cfg>_pass_s0.npz).

  python tools/golden_layer_errors.py c4
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.oracle import ModelConfig as OCfg, node_layout  # noqa: E402
from paper_2209_12708_b200 import faith_gpu as F  # noqa: E402
from paper_2209_12708_b200.configs import ALL  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
g = np.load(os.path.join(ROOT, "tests", "golden", f"{name}_pass_s0.npz"))
w = ALL[name]
cfg = F.ModelConfig(w.layers, w.heads, w.embed, w.ffn, w.length, w.classes, w.activation)
ocfg = OCfg(w.layers, w.heads, w.embed, w.ffn, w.length, w.classes, w.activation)
m = F.Model(F.Context(0), cfg, F.gen_synthetic(cfg, w.model_seed))
x, pos = F.gen_input(cfg, w.input_seed(0)), F.gen_positions(w.position_seed(0), w.length, w.words)
eps = float(g["eps"])
st, lo, hi, nlo, nhi = m.bound_pass_dump(x, pos, w.norm, eps)
est, elo, ehi, xlo, xhi = m.bound_pass_exact(x, pos, w.norm, eps, dump=True)
idx = g["node_index"]
print(f"{name} eps {eps:g}: status ref {int(g['status'])} f32 {st} exact {est}")
print("logits ref", g["logits_lo"], g["logits_hi"], "f32", lo, hi, "exact", elo, ehi)
for nm, off, n in node_layout(ocfg):
    keep = (idx >= off) & (idx < off + n)
    if not keep.any():
        continue
    gi = idx[keep]
    wl, wh = g["node_lo"][keep], g["node_hi"][keep]
    sc = np.maximum(1.0, np.maximum(np.abs(wl), np.abs(wh)))
    e32 = np.nanmax(np.maximum(np.abs(nlo[gi] - wl), np.abs(nhi[gi] - wh)) / sc) if not np.all(np.isnan(nlo[gi])) else np.nan
    e64 = np.max(np.maximum(np.abs(xlo[gi] - wl), np.abs(xhi[gi] - wh)) / sc)
    print(f"{nm:12s} f32 {e32:.2e}  exact {e64:.2e}  max|v| {np.max(sc):.2e}")
