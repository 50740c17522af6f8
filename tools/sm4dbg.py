import sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2209_12708_b200 import faith_gpu as F
from paper_2209_12708_b200.configs import CONFIGS
w = CONFIGS[sys.argv[1]]
cfg = F.ModelConfig(w.layers, w.heads, w.embed, w.ffn, w.length, w.classes, w.activation)
params = F.gen_synthetic(cfg, w.model_seed)
for S in [int(a) for a in sys.argv[2:]]:
    m = F.Model(F.Context(0), cfg, params)
    x = np.stack([F.gen_input(cfg, w.input_seed(s)) for s in range(S)])
    pos = np.stack([F.gen_positions(w.position_seed(s), w.length, w.words) for s in range(S)])
    try:
        lo, hi, st = m.bound_pass(x, pos, w.norm, [w.eps] * S)
        print("S", S, "ok", st[:4], flush=True)
    except Exception as e:
        print("S", S, "FAIL", e, flush=True)
        break
