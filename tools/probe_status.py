import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2209_12708_b200 import faith_gpu as F
from paper_2209_12708_b200.configs import CONFIGS
w = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
cfg = F.ModelConfig(w.layers, w.heads, w.embed, w.ffn, w.length, w.classes, w.activation)
m = F.Model(F.Context(0), cfg, F.gen_synthetic(cfg, w.model_seed))
n = 8
x = np.stack([F.gen_input(cfg, w.input_seed(s)) for s in range(n)])
pos = np.stack([F.gen_positions(w.position_seed(s), w.length, w.words) for s in range(n)])
r = m.maxeps(x, pos, w.norm, w.eps_max, w.tol)
print("eps*", r["eps"])
eps_grid = [1.0 / 2 ** k for k in range(0, 12)]
for e in eps_grid:
    lo, hi, st = m.bound_pass(x, pos, w.norm, [e] * n)
    print(f"eps {e:.6f} status {st.tolist()}")
