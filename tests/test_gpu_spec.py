"""Speculative ε bisection: several bisection levels per batched round,
spread over ranks.  It must reproduce cmd_maxeps's decision path exactly -- the same certified
ε and the same number of verification calls on the path as the sequential search (fg_maxeps),
for any depth and rank count -- in fewer rounds."""
import math
import threading

import numpy as np
import pytest

from paper_2209_12708_b200 import faith_gpu as F
from paper_2209_12708_b200.configs import CONFIGS

pytestmark = pytest.mark.gpu


def _setup(name, n):
    w = CONFIGS[name]
    cfg = F.ModelConfig(w.layers, w.heads, w.embed, w.ffn, w.length, w.classes, w.activation)
    params = F.gen_synthetic(cfg, w.model_seed)
    x = np.stack([F.gen_input(cfg, w.input_seed(s)) for s in range(n)])
    pos = np.stack([F.gen_positions(w.position_seed(s), w.length, w.words) for s in range(n)])
    return w, cfg, params, x, pos


@pytest.mark.parametrize("depth", [1, 2, 3, 5])
def test_speculative_equals_sequential_c1(depth):
    w, cfg, params, x, pos = _setup("c1", 1)
    m = F.Model(F.Context(0), cfg, params)
    seq = m.maxeps(x, pos, w.norm, w.eps_max, w.tol)
    spec = m.maxeps_speculative(x, pos, w.norm, w.eps_max, w.tol, depth=depth)
    assert spec["eps"].tolist() == seq["eps"].tolist()
    assert spec["calls"].tolist() == seq["calls"].tolist()
    assert spec["status"].tolist() == seq["status"].tolist()
    n = int(seq["calls"][0]) - 2  # bisection steps on the path
    assert spec["rounds"] <= 1 + math.ceil(n / depth)


def test_speculative_batch_c2():
    w, cfg, params, x, pos = _setup("c2", 4)
    m = F.Model(F.Context(0), cfg, params)
    seq = m.maxeps(x, pos, w.norm, w.eps_max, 1e-5)
    spec = m.maxeps_speculative(x, pos, w.norm, w.eps_max, 1e-5, depth=3)
    assert spec["eps"].tolist() == seq["eps"].tolist()
    assert spec["calls"].tolist() == seq["calls"].tolist()


class _ThreadGroup:
    """torch.distributed stand-in for ranks running as threads in one process: all_reduce(MAX)."""

    def __init__(self, world):
        self.world, self.bar, self.bufs, self.lock = world, threading.Barrier(world), {}, threading.Lock()

    def view(self, rank):
        g = self

        class V:
            def get_world_size(self):
                return g.world

            def get_rank(self):
                return rank

            def get_backend(self):
                return "gloo"

            class ReduceOp:
                MAX = "max"

            def all_reduce(self, t, op=None):
                with g.lock:
                    g.bufs[rank] = t.clone()
                g.bar.wait()
                import torch
                out = g.bufs[0].clone()
                for r in range(1, g.world):
                    out = torch.maximum(out, g.bufs[r])
                g.bar.wait()
                t.copy_(out)

        return V()


@pytest.mark.parametrize("world", [2, 3])
def test_speculative_across_ranks(world):
    import torch  # noqa: F401  (the exchange callback moves verdicts through torch tensors)
    w, cfg, params, x, pos = _setup("c1", 1)
    seq = F.Model(F.Context(0), cfg, params).maxeps(x, pos, w.norm, w.eps_max, w.tol)
    group = _ThreadGroup(world)
    out, errs = [None] * world, []
    models = [F.Model(F.Context(0), cfg, params) for _ in range(world)]

    def run(r):
        try:
            out[r] = models[r].maxeps_speculative(x, pos, w.norm, w.eps_max, w.tol, depth=3, dist=group.view(r))
        except Exception as e:  # pragma: no cover
            errs.append(e)

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for r in range(world):
        assert out[r]["eps"].tolist() == seq["eps"].tolist()
        assert out[r]["calls"].tolist() == seq["calls"].tolist()
