import glob, os, sys, numpy as np
sys.path.insert(0, os.getcwd())
from paper_2209_12708_b200 import faith_gpu as F
from paper_2209_12708_b200.configs import ALL
ctx = F.Context(0)
for p in sorted(glob.glob("tests/golden/*_pass_s*.npz")):
    g = np.load(p); name = os.path.basename(p).split("_")[0]; w = ALL[name]
    cfg = F.ModelConfig(w.layers, w.heads, w.embed, w.ffn, w.length, w.classes, w.activation)
    m = F.Model(ctx, cfg, F.gen_synthetic(cfg, w.model_seed))
    x = F.gen_input(cfg, w.input_seed(0)); pos = F.gen_positions(w.position_seed(0), w.length, w.words)
    st, lo, hi, nlo, nhi = m.bound_pass_exact(x, pos, w.norm, float(g["eps"]), dump=True)
    idx = g["node_index"]
    a = np.concatenate([nlo[idx], nhi[idx], lo, hi]); b = np.concatenate([g["node_lo"], g["node_hi"], g["logits_lo"], g["logits_hi"]])
    same = np.sum(a == b); err = np.max(np.abs(a - b) / np.maximum(1, np.abs(b)))
    print(f"EXACT vs golden {name}: status {st}/{int(g['status'])} bit-identical {same}/{a.size} max scaled err {err:.3e} logits {lo} {hi} vs {g['logits_lo']} {g['logits_hi']}", flush=True)
