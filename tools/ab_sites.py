#!/usr/bin/env python
"""A/B of pass site times between library builds on one box (diagnostic, not a benchmark):
each round copies every given libfaith_gpu.so over the in-tree one and runs tools/prof_pass.py,
so the builds alternate under the same clocks.  The in-tree library is restored at the end.

  python tools/ab_sites.py ab/base.so ab/new.so [--rounds 3] [--config c3] [--sentences 64]
"""
import argparse
import ast
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2209_12708_b200", "_lib", "libfaith_gpu.so")

ap = argparse.ArgumentParser()
ap.add_argument("libs", nargs="+")
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--config", default="c3")
ap.add_argument("--sentences", type=int, default=64)
a = ap.parse_args()
keep = LIB + ".ab_keep"
shutil.copy(LIB, keep)
res = {lib: [] for lib in a.libs}
try:
    for _ in range(a.rounds):
        for lib in a.libs:
            shutil.copy(lib, LIB)
            out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "prof_pass.py"), "--config", a.config,
                                  "--sentences", str(a.sentences), "--passes", "2"],
                                 capture_output=True, text=True, check=True).stdout
            line = [ln for ln in out.splitlines() if ln.startswith("sites")][-1]
            res[lib].append(ast.literal_eval(line[len("sites "):]))
finally:
    shutil.copy(keep, LIB)
    os.remove(keep)
for lib, runs in res.items():
    keys = runs[0].keys()
    best = {k: round(min(r[k] for r in runs), 3) for k in keys}
    print(os.path.basename(lib), "total", round(sum(best.values()), 2), best, flush=True)
