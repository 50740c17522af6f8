"""Single-thread CPU-baseline calibration: full word-level bound pass time / time of its first
SAMPLE_NODES nodes, medians over 15 sentences, oracle/_ref (unmodified reference sources).
Usage: python tools/cpu_calibrate.py CONFIG [REPS] -> a row for profiles/cpu_calibration.json"""
import sys, time, ctypes as C, numpy as np
sys.path.insert(0, '/root/repo')
import bench
from oracle.oracle import NORM, ModelConfig, Oracle, _d, _i
w = bench.CONFIGS[sys.argv[1]]
o = Oracle("reference")
o.lib.fo_bound_pass_prefix.restype = C.c_int
cfg = ModelConfig(w.layers, w.heads, w.embed, w.ffn, w.length, w.classes, w.activation)
params = o.gen_model(cfg, w.model_seed); fc = cfg.fo()
def t(nodes, reps):
    ts = []
    for s in range(reps):
        x = o.gen_input(cfg, w.input_seed(s)); pos = np.ascontiguousarray(o.gen_positions(w.position_seed(s), w.length, w.words), dtype=np.int32)
        t0 = time.perf_counter()
        o.lib.fo_bound_pass_prefix(C.byref(fc), _d(params), _d(x), _i(pos), w.words, NORM[w.norm], C.c_double(w.eps), nodes)
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts))
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 15
ps = t(bench.SAMPLE_NODES, reps); pf = t(10**9, reps)
print(w.name, "pass_s", pf, "sample_s", ps, "ratio", pf / ps)
