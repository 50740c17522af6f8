#!/usr/bin/env python
"""Diagnostic (not a benchmark): how far is the fused f32-Λ pass from the exact pass?

1. margin error: for c3 sentences, probes at radii around each sentence's certified ε; the
   error |m_f32 - m_exact| of every check_robust margin m_j = lo_t - hi_j, relative to the
   Λ-derived widths (hi_t - lo_t) + (hi_j - lo_j) of the f32 pass.  This ratio is what the
   ambiguity band kappa of fg_model_set_exact_resolve must dominate.
2. node error: f32 pass vs exact pass per node (scaled |d| / max(1, |v|) and width error) at
   the deep configs' candidate golden radii.
3. cost: exact-pass time per sentence; maxeps with and without the exact re-decision.

  python tools/exact_margin_study.py [--sentences 24] [--parts margin,nodes,maxeps] [--configs c1,c2,c3]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.oracle import ModelConfig as OCfg, node_layout  # noqa: E402
from paper_2209_12708_b200 import faith_gpu as F  # noqa: E402
from paper_2209_12708_b200.configs import ALL  # noqa: E402


def load(ctx, name):
    w = ALL[name]
    cfg = F.ModelConfig(w.layers, w.heads, w.embed, w.ffn, w.length, w.classes, w.activation)
    m = F.Model(ctx, cfg, F.gen_synthetic(cfg, w.model_seed))
    return w, cfg, m


def sent(w, cfg, s):
    return F.gen_input(cfg, w.input_seed(s)), F.gen_positions(w.position_seed(s), w.length, w.words)


def margin_part(ctx, n, name="c3"):
    w, cfg, m = load(ctx, name)
    xs, ps = zip(*[sent(w, cfg, s) for s in range(n)])
    m.set_exact_resolve(0.0)
    r = m.maxeps(np.stack(xs), np.stack(ps), w.norm, w.eps_max, w.tol)
    preds = r["predicted"]
    ratios, signed, exact_ms, worst = [], [], [], None
    for s in range(n):
        e0 = float(r["eps"][s])
        if not np.isfinite(e0) or e0 <= 0:
            continue
        for f in (0.5, 0.9, 0.99, 0.999, 1.0, 1.001, 1.01, 1.1, 2.0):
            eps = e0 * f
            lo, hi, st = m.bound_pass(xs[s], ps[s], w.norm, eps)
            t0 = time.perf_counter()
            est, elo, ehi, _, _ = m.bound_pass_exact(xs[s], ps[s], w.norm, eps)
            exact_ms.append(1e3 * (time.perf_counter() - t0))
            if st[0] != 0 or est != 0:
                if st[0] != est:
                    print(f"STATUS MISMATCH s{s} eps {eps:.9g}: f32 {st[0]} exact {est}", flush=True)
                continue
            t = preds[s]
            for j in range(cfg.classes):
                if j == t:
                    continue
                m32 = lo[0][t] - hi[0][j]
                m64 = elo[t] - ehi[j]
                wd = (hi[0][t] - lo[0][t]) + (hi[0][j] - lo[0][j])
                q = abs(m32 - m64) / wd if wd > 0 else 0.0
                ratios.append(q)
                signed.append((m32 - m64) / wd if wd > 0 else 0.0)
                if worst is None or q > worst[0]:
                    worst = (q, s, eps, m32, m64, wd)
                if (m32 > 0) != (m64 > 0):
                    print(f"VERDICT FLIP s{s} eps {eps:.12g}: m32 {m32:.3e} m64 {m64:.3e} widths {wd:.3e} "
                          f"ratio {q:.3e}", flush=True)
    ratios = np.array(ratios)
    out = {"probes": int(ratios.size), "ratio_max": float(ratios.max()), "ratio_p99": float(np.quantile(ratios, 0.99)),
           "ratio_median": float(np.median(ratios)), "signed_min": float(np.min(signed)),
           "signed_max": float(np.max(signed)), "worst": worst, "exact_ms_median": float(np.median(exact_ms)),
           "exact_ms_max": float(np.max(exact_ms))}
    print("MARGIN", name, json.dumps(out), flush=True)


def nodes_part(ctx):
    for name, grid in (("c3", (0.01,)), ("c4m", (1e-4,)), ("c4", (1e-8, 3e-9, 1e-9)), ("c5s", (1e-3, 3e-3, 1e-2))):
        w, cfg, m = load(ctx, name)
        ocfg = OCfg(w.layers, w.heads, w.embed, w.ffn, w.length, w.classes, w.activation)
        x, pos = sent(w, cfg, 0)
        for eps in grid:
            st, lo, hi, nlo, nhi = m.bound_pass_dump(x, pos, w.norm, eps)
            t0 = time.perf_counter()
            est, elo, ehi, xlo, xhi = m.bound_pass_exact(x, pos, w.norm, eps, dump=True)
            ms = 1e3 * (time.perf_counter() - t0)
            worst, wworst = (0.0, ""), (0.0, "")
            for nm, off, nn in node_layout(ocfg):
                a, b = nlo[off:off + nn], nhi[off:off + nn]
                keep = ~np.isnan(a)
                if not keep.any():
                    continue
                sc = np.maximum(1.0, np.abs(xlo[off:off + nn][keep]))
                e = max(np.max(np.abs(a[keep] - xlo[off:off + nn][keep]) / sc),
                        np.max(np.abs(b[keep] - xhi[off:off + nn][keep]) / np.maximum(1.0, np.abs(xhi[off:off + nn][keep]))))
                if e > worst[0]:
                    worst = (float(e), nm)
                wg = (b - a)[keep]
                wx = (xhi - xlo)[off:off + nn][keep]
                we = float(np.max(np.abs(wg - wx) / np.maximum(np.abs(wx), 1e-300)))
                if we > wworst[0]:
                    wworst = (we, nm)
            print(f"NODES {name} eps {eps:g}: status f32 {st} exact {est}; logits f32 {lo} {hi} exact {elo} {ehi}; "
                  f"max scaled node err {worst}; max relative width err {wworst}; exact pass {ms:.0f} ms", flush=True)


def maxeps_part(ctx, n):
    w, cfg, m = load(ctx, "c3")
    xs, ps = zip(*[sent(w, cfg, s) for s in range(n)])
    xs, ps = np.stack(xs), np.stack(ps)
    res = {}
    for kappa in (0.0, F.DEFAULT_KAPPA if hasattr(F, "DEFAULT_KAPPA") else 1e-5):
        m.set_exact_resolve(kappa)
        r = m.maxeps(xs, ps, w.norm, w.eps_max, w.tol)
        st = m.last_stats()
        res[kappa] = r
        print(f"MAXEPS kappa {kappa:g}: {n / (st['device_ms'] / 1e3):.2f} sentences/s, exact probes "
              f"{st['exact_probes']} ({st['exact_ms']:.0f} ms of {st['device_ms']:.0f} ms)", flush=True)
    a, b = list(res.values())
    diff = [(s, a["eps"][s], b["eps"][s], a["calls"][s], b["calls"][s]) for s in range(n)
            if not (a["eps"][s] == b["eps"][s] or (np.isnan(a["eps"][s]) and np.isnan(b["eps"][s])))]
    print("MAXEPS decisions changed by the exact re-decision:", diff, flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sentences", type=int, default=24)
    ap.add_argument("--parts", default="nodes,margin,maxeps")
    ap.add_argument("--configs", default="c3")
    a = ap.parse_args()
    ctx = F.Context(0)
    parts = a.parts.split(",")
    if "nodes" in parts:
        nodes_part(ctx)
    if "margin" in parts:
        for name in a.configs.split(","):
            margin_part(ctx, a.sentences, name)
    if "maxeps" in parts:
        maxeps_part(ctx, 64)


if __name__ == "__main__":
    main()
