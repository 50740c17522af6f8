"""Decision-exact verdicts and the exact-mode device pass.

fg_bound_pass_exact walks the reference's node sequence in f64 with the reference's operation
order on the device; it must reproduce the reference's golden vectors (tests/golden/, written by
the unmodified reference build) to the last bits.  fg_maxeps / fg_certify decide every probe on
the fused f32-Λ pass and re-decide the ambiguous ones (margin within kappa x widths of zero) on
the exact pass, so their verdicts -- and therefore the whole ε bisection path -- are the
reference's (proj/src/cli.cpp:144-177, proj/src/bounds.cpp:142-157)."""
import glob
import json
import os

import numpy as np
import pytest

from helpers import model_config
from oracle.oracle import ModelConfig as OCfg, node_layout
from paper_2209_12708_b200 import faith_gpu as F
from paper_2209_12708_b200.configs import ALL as CONFIGS

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def gpu_model(ctx, cfg, params):
    return F.Model(ctx, F.ModelConfig(cfg.layers, cfg.heads, cfg.embed, cfg.ffn, cfg.length, cfg.classes,
                                      cfg.activation), params)


@pytest.fixture(scope="module")
def models(ctx, port):
    cache = {}

    def get(name):
        if name not in cache:
            w = CONFIGS[name]
            cfg = model_config(w)
            params = port.gen_model(cfg, w.model_seed)
            cache[name] = (w, cfg, params, gpu_model(ctx, cfg, params))
        return cache[name]
    return get


def sentence(port, w, cfg, s):
    return port.gen_input(cfg, w.input_seed(s)), port.gen_positions(w.position_seed(s), w.length, w.words)


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "*_pass_s*.npz"))), ids=os.path.basename)
def test_exact_pass_matches_golden(models, port, path):
    """Every stored node bound of the reference walk, f64: at most a few ulps apart (the device
    libm's exp differs from glibc's in the last bit on some arguments; everything else is the
    reference's operation order), most of them bit-identical."""
    g = np.load(path)
    name = os.path.basename(path).split("_")[0]
    s = int(os.path.basename(path).split("_s")[1].split(".")[0])
    w, cfg, params, m = models(name)
    x, pos = sentence(port, w, cfg, s)
    st, lo, hi, nlo, nhi = m.bound_pass_exact(x, pos, w.norm, float(g["eps"]), dump=True)
    assert st == int(g["status"])
    idx = g["node_index"]
    if name == "c4":  # chaotic from layer 3 on (test_gpu_pass.CHAOTIC_FROM): the well-conditioned layers
        end = [off for nm, off, n in node_layout(cfg) if nm == "l3.q"][0]
        keep = idx < end
        got, want = np.concatenate([nlo[idx[keep]], nhi[idx[keep]]]), np.concatenate([g["node_lo"][keep],
                                                                                       g["node_hi"][keep]])
        assert np.max(np.abs(got - want) / np.maximum(1.0, np.abs(want))) <= 1e-9  # growing x30 per layer
        return
    got = np.concatenate([nlo[idx], nhi[idx], lo, hi])
    want = np.concatenate([g["node_lo"], g["node_hi"], g["logits_lo"], g["logits_hi"]])
    err = np.abs(got - want) / np.maximum(1.0, np.abs(want))
    same = float(np.mean(got == want))
    print(f"{name}: {same:.1%} of {got.size} values bit-identical, max scaled error {err.max():.2e}")
    assert err.max() <= 1e-12
    assert same >= 0.5


@pytest.mark.parametrize("cfg,words,norm,eps", [
    (OCfg(1, 2, 16, 32, 8, 2, "relu"), 1, "linf", 0.05),
    (OCfg(2, 2, 16, 32, 8, 2, "tanh"), 2, "l2", 0.1),
    (OCfg(1, 1, 8, 16, 4, 3, "silu"), 1, "l1", 0.2),
    (OCfg(2, 4, 32, 64, 16, 2, "relu"), 2, "l1", 0.02),
    (OCfg(1, 4, 20, 36, 6, 3, "relu"), 3, "l2", 0.03),  # o % 8 != 0: one-output affine kernel
])
def test_exact_pass_matches_port(ctx, port, cfg, words, norm, eps):
    params = port.gen_model(cfg, 321)
    x = port.gen_input(cfg, 322)
    pos = port.gen_positions(323, cfg.length, words)
    m = gpu_model(ctx, cfg, params)
    st, lo, hi, nlo, nhi = m.bound_pass_exact(x, pos, norm, eps, dump=True)
    pst, plo, phi, pnlo, pnhi = port.bound_pass(cfg, params, x, pos, norm, eps, dump=True)
    assert st == pst
    got, want = np.concatenate([nlo, nhi, lo, hi]), np.concatenate([pnlo, pnhi, plo, phi])
    assert np.max(np.abs(got - want) / np.maximum(1.0, np.abs(want))) <= 1e-12


def test_exact_pass_domain_error(models, port):
    w, cfg, params, m = models("c1")
    x, pos = sentence(port, w, cfg, 0)
    st = m.bound_pass_exact(x, pos, "linf", 50.0)[0]
    assert st == port.bound_pass(cfg, params, x, pos, "linf", 50.0)[0] == F.FG_EDOMAIN


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "*_maxeps_s*.json"))), ids=os.path.basename)
def test_maxeps_golden_decisions_and_f32_flips(models, port, path):
    """The reference's ε and calls exactly with the default re-decision; with it off (kappa 0,
    raw f32 verdicts) the bisection may leave the reference's path near ε* -- reported, and
    still within the north-star tolerance of 1e-3 relative."""
    rec = json.load(open(path))
    w, cfg, params, m = models(rec["config"])
    x, pos = sentence(port, w, cfg, rec["sentence"])
    r = m.maxeps(x, pos, rec["norm"], rec["eps_max"], rec["tol"])
    assert (int(r["status"][0]), int(r["calls"][0]), int(r["predicted"][0])) == \
        (rec["status"], rec["calls"], rec["predicted"])
    assert r["eps"][0] == rec["max_epsilon"]
    try:
        m.set_exact_resolve(0.0)
        raw = m.maxeps(x, pos, rec["norm"], rec["eps_max"], rec["tol"])
    finally:
        m.set_exact_resolve(F.DEFAULT_KAPPA)
    if raw["eps"][0] != rec["max_epsilon"]:
        print(f"{os.path.basename(path)}: raw f32 verdicts leave the reference path: eps {raw['eps'][0]!r} vs "
              f"{rec['max_epsilon']!r}")
    if rec["status"] == 0:
        assert abs(raw["eps"][0] - rec["max_epsilon"]) <= 1e-3 * rec["max_epsilon"] + rec["tol"]


def test_certify_near_threshold_matches_exact(models, port):
    """Probes straddling a sentence's ε* (where f32 and f64 margins can disagree in sign): the
    certify verdict equals check_robust on the exact pass every time."""
    w, cfg, params, m = models("c3")
    n = 4
    xs, ps = zip(*[sentence(port, w, cfg, s) for s in range(n)])
    r = m.maxeps(np.stack(xs), np.stack(ps), w.norm, w.eps_max, w.tol)
    checked = 0
    for s in range(n):
        e0 = float(r["eps"][s])
        if not np.isfinite(e0) or e0 <= 0:
            continue
        for eps in (e0, e0 + 0.25 * w.tol, e0 + 0.5 * w.tol, e0 + w.tol, e0 * (1 + 1e-7)):
            c = m.certify(xs[s], ps[s], w.norm, eps)
            st, lo, hi, _, _ = m.bound_pass_exact(xs[s], ps[s], w.norm, eps)
            want = st == 0 and F.Context.check_robust(lo, hi, int(c["predicted"][0]))
            assert bool(c["verified"][0]) == bool(want), (s, eps)
            checked += 1
    assert checked >= 8


def test_maxeps_exact_probe_accounting(models, port):
    """last_stats() counts the probes that went to the exact pass; with kappa 0 there are none."""
    w, cfg, params, m = models("c2")
    xs, ps = zip(*[sentence(port, w, cfg, s) for s in range(8)])
    m.maxeps(np.stack(xs), np.stack(ps), w.norm, w.eps_max, w.tol)
    st = m.last_stats()
    assert st["exact_probes"] >= 0 and st["exact_ms"] >= 0.0
    try:
        m.set_exact_resolve(0.0)
        m.maxeps(np.stack(xs), np.stack(ps), w.norm, w.eps_max, w.tol)
        assert m.last_stats()["exact_probes"] == 0
    finally:
        m.set_exact_resolve(F.DEFAULT_KAPPA)
    with pytest.raises(F.InvalidArgument):
        m.set_exact_resolve(-1.0)


@pytest.mark.parametrize("mode", ["off", "predicted", "verified", "failed"])
def test_maxeps_speculation_modes_match_golden(models, port, mode):
    """While a re-decision runs, fg_maxeps bisects on with a guessed verdict and rolls the
    sentence back when the exact verdict differs.  Whatever the guesses -- predicted, always
    verified, always failed (forcing roll-backs), or no speculation -- the ε and calls are the
    reference's.  A wide band (kappa 1e-4 until 16 calibration samples) sends many probes to the
    exact pass, so the roll-back path runs."""
    recs = [json.load(open(p)) for p in sorted(glob.glob(os.path.join(GOLDEN, "c3_maxeps_s*.json")))]
    w, cfg, params, m = models("c3")
    xs, ps = zip(*[sentence(port, w, cfg, rec["sentence"]) for rec in recs])
    try:
        m.set_exact_resolve(1e-4)
        m.set_speculation(mode)
        r = m.maxeps(np.stack(xs), np.stack(ps), recs[0]["norm"], recs[0]["eps_max"], recs[0]["tol"])
        st = m.last_stats()
    finally:
        m.set_speculation("predicted")
        m.set_exact_resolve(F.DEFAULT_KAPPA)
    for k, rec in enumerate(recs):
        assert (int(r["status"][k]), int(r["calls"][k])) == (rec["status"], rec["calls"]), rec["sentence"]
        assert r["eps"][k] == rec["max_epsilon"], rec["sentence"]
    print(f"{mode}: {st['exact_probes']} exact probes, {st['spec_rollbacks']} roll-backs")
    assert st["exact_probes"] >= 8
    if mode == "off":
        assert st["spec_rollbacks"] == 0
    if mode in ("verified", "failed"):
        assert st["spec_rollbacks"] >= 1


def test_speculation_mode_validation(models):
    w, cfg, params, m = models("c1")
    with pytest.raises(F.InvalidArgument):
        m.ctx._check(m.lib.fg_model_set_speculation(m.handle, 7), "fg_model_set_speculation")
    with pytest.raises(KeyError):
        m.set_speculation("sometimes")
