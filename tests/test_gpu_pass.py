"""Pass-level parity on the GPU: the fused CUDA bound pass against the reference
(golden vectors from the unmodified reference build, tests/golden/) and the C
restatement, node by node; certified epsilon and verdicts; sampled soundness."""
import glob
import json
import os

import numpy as np
import pytest

from helpers import close, model_config, sample_in_ball
from oracle.oracle import ModelConfig as OCfg, node_layout
from paper_2209_12708_b200 import faith_gpu as F
from paper_2209_12708_b200.configs import ALL as CONFIGS

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def gpu_model(ctx, cfg: OCfg, params):
    return F.Model(ctx, F.ModelConfig(cfg.layers, cfg.heads, cfg.embed, cfg.ffn, cfg.length, cfg.classes,
                                      cfg.activation), params)


def check_nodes(cfg, got_lo, got_hi, want_lo, want_hi, idx=None, tol=1e-4):
    """Per-node parity; NaN entries of the GPU dump are nodes kept on chip."""
    bad = []
    for name, off, n in node_layout(cfg):
        sl = np.arange(off, off + n)
        if idx is not None:
            keep = np.isin(idx, sl)
            wl, wh, gi = want_lo[keep], want_hi[keep], idx[keep]
        else:
            wl, wh, gi = want_lo[sl], want_hi[sl], sl
        if gi.size == 0 or np.all(np.isnan(got_lo[gi])):
            continue
        ok1, e1 = close(got_lo[gi], wl, tol)
        ok2, e2 = close(got_hi[gi], wh, tol)
        if not (ok1 and ok2):
            bad.append((name, max(e1, e2)))
    assert not bad, f"nodes outside tolerance: {bad[:8]}"


def sentence(port, w, s):
    cfg = model_config(w)
    return cfg, port.gen_input(cfg, w.input_seed(s)), port.gen_positions(w.position_seed(s), w.length, w.words)


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


# ---- golden vectors from the reference build ------------------------------------
# c4 (6 layers, E 512, F 2048 on random-init weights) is numerically chaotic at any radius where
# its bounds are finite: a difference in the last bit grows ~x30 per layer from layer 3 on
# (tools/golden_layer_errors.py; the reference-order exact pass, whose only difference from the
# reference is the device libm's exp in the last ulp, drifts 6e-3 from it by the logits, more than
# the f32 pass's 2e-3).  Layers below CHAOTIC_FROM are held to the 1e-4 bar; from there on the
# test pins the conditioning itself: a 1-ulp change of the input moves the exact pass's logits by
# more than 1e-4 -- no f64 implementation but the reference's own binary can match those digits.
CHAOTIC_FROM = {"c4": 5}


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "*_pass_s*.npz"))), ids=os.path.basename)
def test_pass_matches_golden(models, port, path):
    g = np.load(path)
    name = os.path.basename(path).split("_")[0]
    s = int(os.path.basename(path).split("_s")[1].split(".")[0])
    w, cfg, params, m = models(name)
    _, x, pos = sentence(port, w, s)
    eps = float(g["eps"])
    st, lo, hi, nlo, nhi = m.bound_pass_dump(x, pos, w.norm, eps)
    assert st == int(g["status"])
    first_chaotic = CHAOTIC_FROM.get(name)
    if first_chaotic is None:
        assert close(lo, g["logits_lo"])[0] and close(hi, g["logits_hi"])[0], (lo, hi, g["logits_lo"],
                                                                                g["logits_hi"])
        check_nodes(cfg, nlo, nhi, g["node_lo"], g["node_hi"], g["node_index"])
        return
    idx = g["node_index"]
    end = [off for nm, off, n in node_layout(cfg) if nm == f"l{first_chaotic}.q"][0]
    keep = idx < end
    check_nodes(cfg, nlo, nhi, g["node_lo"][keep], g["node_hi"][keep], idx[keep])
    # the remaining digits are conditioning-limited: a sanity bound on the drift (same bounds to
    # within 20 %), and the exact pass moves by more than the 1e-4 bar under a 1-ulp input change
    assert close(lo, g["logits_lo"], 0.2)[0] and close(hi, g["logits_hi"], 0.2)[0], (lo, hi, g["logits_lo"],
                                                                                      g["logits_hi"])
    st0, elo, ehi, _, _ = m.bound_pass_exact(x, pos, w.norm, eps)
    st1, flo, fhi, _, _ = m.bound_pass_exact(x * (1.0 + 2.0 ** -52), pos, w.norm, eps)
    assert st0 == st1 == int(g["status"])
    assert not (close(flo, elo)[0] and close(fhi, ehi)[0]), "expected a chaotic tail at this radius"


# ---- against the C restatement on configs the golden set does not cover ----------
SMALL = [
    (OCfg(1, 2, 16, 32, 8, 2, "relu"), 1, "linf", 0.05),
    (OCfg(2, 2, 16, 32, 8, 2, "tanh"), 2, "l2", 0.1),
    (OCfg(1, 1, 8, 16, 4, 3, "silu"), 1, "l1", 0.2),
    (OCfg(2, 4, 32, 64, 16, 2, "relu"), 2, "l1", 0.02),
    (OCfg(1, 4, 64, 128, 32, 2, "relu"), 1, "l2", 0.05),
]


@pytest.mark.parametrize("cfg,words,norm,eps", SMALL)
def test_pass_matches_port(ctx, port, cfg, words, norm, eps):
    params = port.gen_model(cfg, 123)
    x = port.gen_input(cfg, 124)
    pos = port.gen_positions(125, cfg.length, words)
    m = gpu_model(ctx, cfg, params)
    st, lo, hi, nlo, nhi = m.bound_pass_dump(x, pos, norm, eps)
    pst, plo, phi, pnlo, pnhi = port.bound_pass(cfg, params, x, pos, norm, eps, dump=True)
    assert st == pst
    assert close(lo, plo)[0] and close(hi, phi)[0]
    check_nodes(cfg, nlo, nhi, pnlo, pnhi)


def test_zero_radius_equals_forward(models, port):
    w, cfg, params, m = models("c1")
    _, x, pos = sentence(port, w, 0)
    lo, hi, st = m.bound_pass(x, pos, w.norm, 0.0)
    logits = port.forward(cfg, params, x)
    assert st[0] == 0
    assert np.allclose(lo[0], logits, rtol=1e-6, atol=1e-9) and np.allclose(hi[0], logits, rtol=1e-6, atol=1e-9)
    assert np.allclose(m.forward(x), logits, rtol=0, atol=0)


def test_batched_pass_equals_single(models, port):
    """S sentences in one batched pass give the same bounds as one at a time."""
    w, cfg, params, m = models("c2")
    xs, ps = [], []
    for s in range(6):
        _, x, pos = sentence(port, w, s)
        xs.append(x)
        ps.append(pos)
    eps = np.array([0.0, 0.01, 0.02, 0.05, 0.1, 0.01])
    lo, hi, st = m.bound_pass(np.stack(xs), np.stack(ps), w.norm, eps)
    for s in range(6):
        l1, h1, s1 = m.bound_pass(xs[s], ps[s], w.norm, eps[s])
        assert s1[0] == st[s]
        assert np.allclose(l1[0], lo[s], rtol=0, atol=1e-12) and np.allclose(h1[0], hi[s], rtol=0, atol=1e-12)


def test_batched_pass_matches_port(models, port):
    w, cfg, params, m = models("c1")
    xs, ps, eps = [], [], []
    for s in range(8):
        _, x, pos = sentence(port, w, s)
        xs.append(x)
        ps.append(pos)
        eps.append(0.005 * (s + 1))
    lo, hi, st = m.bound_pass(np.stack(xs), np.stack(ps), w.norm, np.array(eps))
    for s in range(8):
        pst, plo, phi, _, _ = port.bound_pass(cfg, params, xs[s], ps[s], w.norm, eps[s])
        assert st[s] == pst
        if pst == 0:
            assert close(lo[s], plo)[0] and close(hi[s], phi)[0]


# ---- epsilon search -----------------------------------------------------------------
@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "*_maxeps_s*.json"))), ids=os.path.basename)
def test_maxeps_matches_golden(models, port, path):
    rec = json.load(open(path))
    w, cfg, params, m = models(rec["config"])
    _, x, pos = sentence(port, w, rec["sentence"])
    r = m.maxeps(x, pos, rec["norm"], rec["eps_max"], rec["tol"])
    # decision-exact verdicts (fg_model_set_exact_resolve, on by default): every probe decides
    # as the reference's does, so the dyadic bisection ends on the reference's ε bit for bit
    assert r["status"][0] == rec["status"]
    assert r["predicted"][0] == rec["predicted"]
    assert int(r["calls"][0]) == rec["calls"]
    assert r["eps"][0] == rec["max_epsilon"], (r["eps"][0], rec["max_epsilon"])


def test_maxeps_batch_matches_port(models, port):
    """Continuous batching over more sentences than slots; every sentence follows the
    reference bisection path (cli.cpp:163-176)."""
    w, cfg, params, m = models("c1")
    xs, ps = zip(*[sentence(port, w, s)[1:] for s in range(10)])
    r = m.maxeps(np.stack(xs), np.stack(ps), w.norm, 1.0, 1e-4, slots=4)
    for s in range(10):
        pst, peps, pcalls, ppred = port.maxeps(cfg, params, xs[s], ps[s], w.norm, 1.0, 1e-4)
        assert r["status"][s] == pst and r["predicted"][s] == ppred
        if pst == 0:
            assert r["eps"][s] == peps and int(r["calls"][s]) == pcalls


def test_certify_verdicts_match_port(models, port):
    w, cfg, params, m = models("c1")
    xs, ps = zip(*[sentence(port, w, s)[1:] for s in range(6)])
    eps = np.array([0.0, 0.01, 0.03, 0.06, 0.1, 0.5])
    r = m.certify(np.stack(xs), np.stack(ps), w.norm, eps)
    for s in range(6):
        pst, plo, phi, _, _ = port.bound_pass(cfg, params, xs[s], ps[s], w.norm, eps[s])
        pred = int(np.argmax(port.forward(cfg, params, xs[s])))
        assert r["predicted"][s] == pred
        if pst == 0:
            assert r["verified"][s] == port.check_robust(plo, phi, pred)


def test_domain_error_taxonomy(models, port):
    """A radius far too wide overflows the exp envelope: domain_error, like the reference."""
    w, cfg, params, m = models("c1")
    _, x, pos = sentence(port, w, 0)
    lo, hi, st = m.bound_pass(x, pos, "linf", 50.0)
    pst = port.bound_pass(cfg, params, x, pos, "linf", 50.0)[0]
    assert st[0] == pst == 2


# ---- soundness: sampled perturbed forwards stay inside the GPU bounds ---------------
@pytest.mark.parametrize("norm,eps", [("linf", 0.02), ("l2", 0.2), ("l1", 0.5)])
def test_sampled_soundness(models, port, norm, eps):
    w, cfg, params, m = models("c1")
    _, x, pos = sentence(port, w, 3)
    lo, hi, st = m.bound_pass(x, pos, norm, eps)
    assert st[0] == 0
    rng = np.random.default_rng(7)
    E = cfg.embed
    deltas = sample_in_ball(rng, norm, eps, len(pos) * E, 10_000)
    worst = -np.inf
    for dl in deltas:
        xp = x.reshape(cfg.length, E).copy()
        for wi, p in enumerate(pos):
            xp[p] += dl[wi * E:(wi + 1) * E]
        logits = port.forward(cfg, params, xp.ravel())
        slack = 1e-7 * np.maximum(1.0, np.abs(logits))  # the reference's slack (acceptance.cpp:97)
        worst = max(worst, float(np.max(lo[0] - logits - slack)), float(np.max(logits - hi[0] - slack)))
    assert worst <= 0.0, worst


def test_many_slots_beyond_grid_limits():
    """c1 (D = 64: FP32 SIMT GEMMs, whose batch index lives in gridDim.z) with 300 resident
    sentences: the McCormick GEMMs need S*H*L*2 = 76800 > 65535 batches and are launched in
    slices.  Every sentence's certified epsilon must equal the 60-slot run's."""
    from paper_2209_12708_b200.configs import CONFIGS as C5
    w = C5["c1"]
    cfg = F.ModelConfig(w.layers, w.heads, w.embed, w.ffn, w.length, w.classes, w.activation)
    m = F.Model(F.Context(0), cfg, F.gen_synthetic(cfg, w.model_seed))
    n = 300
    xs = np.stack([F.gen_input(cfg, w.input_seed(s)) for s in range(n)])
    ps = np.stack([F.gen_positions(w.position_seed(s), w.length, w.words) for s in range(n)])
    big = m.maxeps(xs, ps, w.norm, w.eps_max, 1e-4, slots=n)
    small = m.maxeps(xs, ps, w.norm, w.eps_max, 1e-4, slots=60)
    assert np.array_equal(big["calls"], small["calls"])
    assert np.array_equal(big["eps"], small["eps"], equal_nan=True)


@pytest.mark.parametrize("name,n,slots", [("c3", 10, 4), ("c3", 6, 6)])
def test_zero_probe_workspace_matches_full_width(models, port, monkeypatch, name, n, slots):
    """The ε = 0 probes run up front on the narrow all-zero-Λ workspace (128 columns, tcgen05):
    every sentence's status, predicted class, certified ε and probe count equal those of the
    full-width pass (FG_NO_ZERO_PROBE=1), with more sentences than slots (continuous batching
    picks the sentences up at ε_max) and with one slot per sentence."""
    w, cfg, params, m = models(name)
    xs, ps = zip(*[sentence(port, w, s)[1:] for s in range(n)])
    xs, ps = np.stack(xs), np.stack(ps)
    monkeypatch.setenv("FG_NO_ZERO_PROBE", "1")
    full = m.maxeps(xs, ps, w.norm, w.eps_max, 1e-4, slots=slots)
    monkeypatch.delenv("FG_NO_ZERO_PROBE")
    fast = m.maxeps(xs, ps, w.norm, w.eps_max, 1e-4, slots=slots)
    for k in ("status", "predicted", "calls"):
        assert np.array_equal(full[k], fast[k]), k
    assert np.array_equal(full["eps"], fast["eps"], equal_nan=True)


def test_zero_probe_failures_drop_their_eps_max_probe(models, port, monkeypatch):
    """Sentences whose ε = 0 probe fails (inputs scaled up until the exp envelope raises a
    domain error) finish after one call with the same status as on the full-width path, and
    their tentative ε_max slot in the first full-width pass is dropped without disturbing the
    other sentences."""
    w, cfg, params, m = models("c3")
    n = 6
    xs, ps = zip(*[sentence(port, w, s)[1:] for s in range(n)])
    xs, ps = np.stack(xs).copy(), np.stack(ps)
    bad = [1, 4]
    xs[bad] *= 1e4
    monkeypatch.setenv("FG_NO_ZERO_PROBE", "1")
    full = m.maxeps(xs, ps, w.norm, w.eps_max, 1e-4, slots=4)
    monkeypatch.delenv("FG_NO_ZERO_PROBE")
    fast = m.maxeps(xs, ps, w.norm, w.eps_max, 1e-4, slots=4)
    assert all(full["status"][b] != 0 for b in bad), full["status"]
    assert all(full["calls"][b] == 1 for b in bad)
    for k in ("status", "predicted", "calls"):
        assert np.array_equal(full[k], fast[k]), k
    assert np.array_equal(full["eps"], fast["eps"], equal_nan=True)
