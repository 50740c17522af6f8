"""Corpus runs with per-sentence JSONL checkpointing (paper_2209_12708_b200/corpus.py): resume
skips finished ids, a torn last line is redone, per-rank files merge in id order.  The model is a
stand-in with Model.maxeps's interface (host logic only; the GPU path is tests/test_gpu_corpus)."""
import json

import numpy as np

from paper_2209_12708_b200.configs import CONFIGS
from paper_2209_12708_b200.corpus import merge_results, run_corpus


class FakeModel:
    def __init__(self):
        self.seen = []

    def maxeps(self, xs, ps, norm, eps_max, tol, slots=0):
        ids = [int(x[0, 0]) for x in xs]
        self.seen.extend(ids)
        n = len(ids)
        return {"eps": np.array([1e-3 * i for i in ids]), "calls": np.full(n, 22), "predicted": np.zeros(n, int),
                "status": np.zeros(n, int)}


def _gen(w):
    return (lambda s: np.full((w.length, w.embed), float(s))), (lambda s: np.zeros(w.words, dtype=np.int32))


def test_resume_skips_finished_sentences(tmp_path):
    w = CONFIGS["c4"]
    gi, gp = _gen(w)
    out = str(tmp_path / "r.jsonl")
    m = FakeModel()
    assert run_corpus(m, w, range(10), out, batch=4, gen_input=gi, gen_positions=gp) == {"new": 10, "skipped": 0}
    m2 = FakeModel()
    assert run_corpus(m2, w, range(14), out, batch=4, gen_input=gi, gen_positions=gp) == {"new": 4, "skipped": 10}
    assert m2.seen == [10, 11, 12, 13]
    rows = [json.loads(ln) for ln in open(out)]
    assert [r["sentence"] for r in rows] == list(range(14))
    assert rows[5]["eps"] == 5e-3 and rows[5]["calls"] == 22


def test_torn_line_is_redone(tmp_path):
    w = CONFIGS["c4"]
    gi, gp = _gen(w)
    out = tmp_path / "r.jsonl"
    out.write_text(json.dumps({"sentence": 0, "eps": 0.0, "calls": 22, "predicted": 0, "status": 0}) + "\n"
                   + '{"sentence": 1, "eps"')  # interrupted write
    m = FakeModel()
    run_corpus(m, w, range(3), str(out), batch=8, gen_input=gi, gen_positions=gp)
    assert m.seen == [1, 2]


def test_merge_rank_files(tmp_path):
    a, b = tmp_path / "o.rank0", tmp_path / "o.rank1"
    a.write_text("".join(json.dumps({"sentence": s, "eps": 0.1}) + "\n" for s in (2, 0)))
    b.write_text("".join(json.dumps({"sentence": s, "eps": 0.2}) + "\n" for s in (3, 1)))
    n = merge_results([str(a), str(b)], str(tmp_path / "o"))
    assert n == 4
    assert [json.loads(ln)["sentence"] for ln in open(tmp_path / "o")] == [0, 1, 2, 3]
