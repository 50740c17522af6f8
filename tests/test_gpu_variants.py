"""The comparison knobs of DESIGN.md §7 (read once per process, so each run is a subprocess):
every variant certifies the same sentences.  Exact variants (graph replay, row batching, the
layer-1 Q/K skip, the ε = 0 probe workspace) must reproduce the default run bit for bit;
variants that change the arithmetic or its order (FP32 SIMT instead of tcgen05 3xTF32, one CTA instead of
CTA pairs, one epilogue group, dense layer 1, another softmax kernel, shared-memory instead of
tensor-memory GEMM operands) must give the same status / predicted class, certified ε
within 1e-3 relative (+ tol) and calls within one bisection step."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
TOL = 1e-4


def run(name, n, slots, **env):
    e = dict(os.environ)
    for k in list(e):
        if k.startswith("FG_"):
            del e[k]
    e.update(env)
    p = subprocess.run([sys.executable, os.path.join(HERE, "variant_run.py"), name, str(n), str(slots)],
                       capture_output=True, text=True, env=e, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


EXACT = [{"FG_NO_GRAPH": "1"}, {"FG_NO_ROWS2": "1"}, {"FG_ONEHOT_DENSE_QK": "1"}, {"FG_NO_ZERO_PROBE": "1"},
         {"FG_MEANPOOL_SCALAR": "1"}, {"FG_TOKENS_ONEPASS": "1"}]
CLOSE = [{"FG_NO_UMMA": "1"}, {"FG_NO_UMMA_DOTS": "1"}, {"FG_NO_UMMA_AFFINE": "1"}, {"FG_2CTA": "0"},
         {"FG_EPI_GROUPS": "1"}, {"FG_NO_ONEHOT": "1"}, {"FG_DOTS_TMEM_A": "0"}, {"FG_AFFINE_TMEM_A": "1"}]


@pytest.fixture(scope="module")
def base():
    return {name: run(name, 6, 4) for name in ("c2", "c3")}


@pytest.mark.parametrize("name", ["c2", "c3"])
@pytest.mark.parametrize("env", EXACT, ids=lambda d: ",".join(d))
def test_exact_variants(base, name, env):
    got = run(name, 6, 4, **env)
    assert got == base[name]


@pytest.mark.parametrize("name", ["c2", "c3"])
@pytest.mark.parametrize("env", CLOSE, ids=lambda d: ",".join(d))
def test_close_variants(base, name, env):
    got, want = run(name, 6, 4, **env), base[name]
    assert got["status"] == want["status"] and got["predicted"] == want["predicted"]
    for s, st in enumerate(want["status"]):
        if st == 0:
            a, b = got["eps"][s], want["eps"][s]
            assert abs(a - b) <= 1e-3 * abs(b) + TOL, (s, a, b)
            assert abs(got["calls"][s] - want["calls"][s]) <= 1
