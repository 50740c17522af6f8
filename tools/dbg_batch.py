import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2209_12708_b200 import faith_gpu as F
from paper_2209_12708_b200.configs import CONFIGS
for name in ("c2", "c3"):
    w = CONFIGS[name]
    cfg = F.ModelConfig(w.layers, w.heads, w.embed, w.ffn, w.length, w.classes, w.activation)
    params = F.gen_synthetic(cfg, w.model_seed)
    m = F.Model(F.Context(0), cfg, params)
    xs = np.stack([F.gen_input(cfg, w.input_seed(s)) for s in range(6)])
    ps = np.stack([F.gen_positions(w.position_seed(s), w.length, w.words) for s in range(6)])
    eps = np.array([0.0, 0.01, 0.02, 0.05, 0.1, 0.01])
    a = m.bound_pass(xs, ps, w.norm, eps)
    b = m.bound_pass(xs, ps, w.norm, eps)
    print(name, "repeat diff", np.abs(a[0] - b[0]).max(), np.abs(a[1] - b[1]).max())
    for s in range(6):
        l1, h1, s1 = m.bound_pass(xs[s], ps[s], w.norm, eps[s])
        print(name, s, "single-vs-batched", np.abs(l1[0] - a[0][s]).max(), np.abs(h1[0] - a[1][s]).max())
