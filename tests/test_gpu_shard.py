"""Column-sharded pass on one B200: the perturbation columns of every Λ
are split over virtual ranks (fg_loopback: one model + host thread per rank on the same GPU,
rank-ordered reduction kernel between CUDA events) or over a world-size-1 NCCL communicator.
Every rank must return identical results, and they must match the unsharded pass (only the
summation order of the norms and the f64 element math of the 5-kernel softmax chain differ)
and the reference oracle."""
import threading

import numpy as np
import pytest

from helpers import close
from paper_2209_12708_b200 import faith_gpu as F
from paper_2209_12708_b200.configs import CONFIGS

pytestmark = pytest.mark.gpu


def _inputs(w, n):
    cfg = F.ModelConfig(w.layers, w.heads, w.embed, w.ffn, w.length, w.classes, w.activation)
    params = F.gen_synthetic(cfg, w.model_seed)
    x = np.stack([F.gen_input(cfg, w.input_seed(s)) for s in range(n)])
    pos = np.stack([F.gen_positions(w.position_seed(s), w.length, w.words) for s in range(n)])
    return cfg, params, x, pos


def _run_ranks(nranks, cfg, params, job):
    group = F.LoopbackGroup(nranks)
    out, errs = [None] * nranks, []
    models = []
    for r in range(nranks):
        ctx = F.Context(0)
        m = F.Model(ctx, cfg, params)
        m.shard_columns_loopback(group, r)
        models.append(m)

    def worker(r):
        try:
            out[r] = job(models[r])
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    ts = [threading.Thread(target=worker, args=(r,)) for r in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    return out


@pytest.mark.parametrize("nranks", [2, 4])
def test_column_shard_matches_unsharded_c3(nranks):
    w = CONFIGS["c3"]
    cfg, params, x, pos = _inputs(w, 3)
    eps = [w.eps, 0.004, 0.0]
    base = F.Model(F.Context(0), cfg, params).bound_pass(x, pos, w.norm, eps)
    res = _run_ranks(nranks, cfg, params, lambda m: m.bound_pass(x, pos, w.norm, eps))
    for r in range(1, nranks):  # identical on every rank
        for a, b in zip(res[0], res[r]):
            assert np.array_equal(a, b)
    lo, hi, st = res[0]
    assert np.array_equal(st, base[2])
    assert close(lo, base[0], 1e-6)[0] and close(hi, base[1], 1e-6)[0], (close(lo, base[0], 1e-6), close(hi, base[1], 1e-6))


def test_column_shard_matches_oracle_c1(port):
    from oracle.oracle import ModelConfig
    w = CONFIGS["c1"]
    cfg, params, x, pos = _inputs(w, 1)
    res = _run_ranks(2, cfg, params, lambda m: m.bound_pass(x, pos, w.norm, [w.eps]))
    ocfg = ModelConfig(w.layers, w.heads, w.embed, w.ffn, w.length, w.classes, w.activation)
    pst, plo, phi, _, _ = port.bound_pass(ocfg, params, x[0], pos[0], w.norm, w.eps)
    lo, hi, st = res[0]
    assert st[0] == pst == 0
    assert close(lo[0], plo)[0] and close(hi[0], phi)[0]


def test_column_shard_maxeps_matches_unsharded():
    w = CONFIGS["c2"]
    cfg, params, x, pos = _inputs(w, 3)
    base = F.Model(F.Context(0), cfg, params).maxeps(x, pos, w.norm, w.eps_max, 1e-5)
    res = _run_ranks(2, cfg, params, lambda m: m.maxeps(x, pos, w.norm, w.eps_max, 1e-5))
    assert res[0]["eps"].tolist() == res[1]["eps"].tolist()
    eps0, eps1 = np.asarray(base["eps"]), np.asarray(res[0]["eps"])
    assert np.all(np.abs(eps0 - eps1) <= 1e-3 * eps0 + 1e-5), (eps0, eps1)


def test_column_shard_nccl_world1():
    """The NCCL exchange (ncclAllReduce on the pass stream, graph-captured) with one rank."""
    w = CONFIGS["c3"]
    cfg, params, x, pos = _inputs(w, 2)
    base = F.Model(F.Context(0), cfg, params).bound_pass(x, pos, w.norm, [w.eps] * 2)
    m = F.Model(F.Context(0), cfg, params)
    m.shard_columns_nccl(0, 1, F.nccl_unique_id())
    lo, hi, st = m.bound_pass(x, pos, w.norm, [w.eps] * 2)
    assert np.array_equal(st, base[2])
    assert close(lo, base[0], 1e-6)[0] and close(hi, base[1], 1e-6)[0]


def test_column_shard_c5_bert_base_shape():
    """c5 (12 layers, d=768, 12 heads, ffn=3072, seq 128, two words l2: D=1536) split over 4
    column shards of 384 columns, against the unsharded pass on the same GPU."""
    w = CONFIGS["c5"]
    cfg, params, x, pos = _inputs(w, 1)
    base = F.Model(F.Context(0), cfg, params).bound_pass(x, pos, w.norm, [w.eps])
    res = _run_ranks(4, cfg, params, lambda m: m.bound_pass(x, pos, w.norm, [w.eps]))
    lo, hi, st = res[0]
    assert np.array_equal(st, base[2])
    assert close(lo, base[0], 1e-5)[0] and close(hi, base[1], 1e-5)[0], (lo, base[0], hi, base[1])
