"""Corpus runs with per-sentence checkpointing (the 4096-sentence c4 workload).

`run_corpus` certifies the maximum ε of many synthetic sentences (cmd_maxeps semantics,
proj/src/cli.cpp:135-193, through `Model.maxeps`) in batches and appends one JSON line per
finished sentence to a results file; a rerun skips every sentence id already present, so an
interrupted multi-hour run resumes where it stopped.  Under torch.distributed each rank takes a
contiguous shard of the ids (`dist.shard`) and writes its own `<out>.rank<r>` file;
`merge_results` joins them in id order.

  python -m paper_2209_12708_b200.corpus --config c4 --sentences 4096 --out c4.jsonl
"""
from __future__ import annotations

import argparse
import json
import os
from typing import Iterable, Optional

import numpy as np


def _done_ids(path: str) -> set:
    done = set()
    if not os.path.exists(path):
        return done
    with open(path) as f:
        for ln in f:
            ln = ln.strip()
            if not ln:
                continue
            try:
                done.add(int(json.loads(ln)["sentence"]))
            except (ValueError, KeyError):
                break  # a torn last line from an interrupted write: everything after it is redone
    return done


def run_corpus(model, workload, ids: Iterable[int], out_path: str, batch: int = 64, gen_input=None,
               gen_positions=None) -> dict:
    """ε search for every id not yet in `out_path`; returns {"new": n, "skipped": k}."""
    ids = list(ids)
    done = _done_ids(out_path)
    todo = [i for i in ids if i not in done]
    w = workload
    if gen_input is None or gen_positions is None:
        from . import faith_gpu as F
        cfg = F.ModelConfig(w.layers, w.heads, w.embed, w.ffn, w.length, w.classes, w.activation)
        gen_input = gen_input or (lambda s: F.gen_input(cfg, w.input_seed(s)))
        gen_positions = gen_positions or (lambda s: F.gen_positions(w.position_seed(s), w.length, w.words))
    new = 0
    with open(out_path, "a") as f:
        for b0 in range(0, len(todo), batch):
            chunk = todo[b0:b0 + batch]
            xs = np.stack([gen_input(s) for s in chunk])
            ps = np.stack([gen_positions(s) for s in chunk])
            r = model.maxeps(xs, ps, w.norm, w.eps_max, w.tol, slots=min(batch, len(chunk)))
            for k, s in enumerate(chunk):
                eps = float(r["eps"][k])
                f.write(json.dumps({"sentence": int(s), "eps": None if np.isnan(eps) else eps,
                                    "calls": int(r["calls"][k]), "predicted": int(r["predicted"][k]),
                                    "status": int(r["status"][k])}) + "\n")
            f.flush()
            os.fsync(f.fileno())
            new += len(chunk)
    return {"new": new, "skipped": len(ids) - len(todo)}


def merge_results(paths: Iterable[str], out_path: str) -> int:
    """Joins per-rank result files into one, ordered by sentence id (duplicates collapse)."""
    rows = {}
    for p in paths:
        with open(p) as f:
            for ln in f:
                if ln.strip():
                    rec = json.loads(ln)
                    rows[int(rec["sentence"])] = rec
    with open(out_path, "w") as f:
        for s in sorted(rows):
            f.write(json.dumps(rows[s]) + "\n")
    return len(rows)


def main(argv: Optional[list] = None) -> int:
    from . import dist as D
    from . import faith_gpu as F
    from .configs import CONFIGS
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--sentences", type=int, default=4096)
    ap.add_argument("--out", required=True)
    ap.add_argument("--batch", type=int, default=16)
    a = ap.parse_args(argv)
    w = CONFIGS[a.config]
    info = D.rank_info()
    dist = D.init(backend="nccl", device_index=info.local_rank)
    cfg = F.ModelConfig(w.layers, w.heads, w.embed, w.ffn, w.length, w.classes, w.activation)
    model = F.Model(F.Context(info.local_rank), cfg, F.gen_synthetic(cfg, w.model_seed))
    out = a.out if info.world == 1 else f"{a.out}.rank{info.rank}"
    res = run_corpus(model, w, D.shard(a.sentences, info.rank, info.world), out, a.batch)
    print(json.dumps({"rank": info.rank, **res, "out": out}), flush=True)
    if dist:
        dist.barrier()
        if info.rank == 0:
            merge_results([f"{a.out}.rank{r}" for r in range(info.world)], a.out)
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
