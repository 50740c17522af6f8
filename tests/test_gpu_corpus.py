"""The corpus runner on the GPU: an interrupted run (first half) resumed (second half) gives
the same per-sentence results as one uninterrupted fg_maxeps call over all sentences."""
import json

import numpy as np
import pytest

from paper_2209_12708_b200 import faith_gpu as F
from paper_2209_12708_b200.configs import CONFIGS
from paper_2209_12708_b200.corpus import run_corpus

pytestmark = pytest.mark.gpu


def test_resumed_corpus_equals_one_search(tmp_path):
    w = CONFIGS["c2"]
    cfg = F.ModelConfig(w.layers, w.heads, w.embed, w.ffn, w.length, w.classes, w.activation)
    m = F.Model(F.Context(0), cfg, F.gen_synthetic(cfg, w.model_seed))
    out = str(tmp_path / "c2.jsonl")
    run_corpus(m, w, range(6), out, batch=4)
    res = run_corpus(m, w, range(12), out, batch=4)
    assert res == {"new": 6, "skipped": 6}
    rows = {r["sentence"]: r for r in (json.loads(ln) for ln in open(out))}
    xs = np.stack([F.gen_input(cfg, w.input_seed(s)) for s in range(12)])
    ps = np.stack([F.gen_positions(w.position_seed(s), w.length, w.words) for s in range(12)])
    ref = m.maxeps(xs, ps, w.norm, w.eps_max, w.tol)
    for s in range(12):
        assert rows[s]["eps"] == ref["eps"][s] and rows[s]["calls"] == ref["calls"][s]
        assert rows[s]["predicted"] == ref["predicted"][s] and rows[s]["status"] == ref["status"][s]
