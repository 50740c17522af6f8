"""CPU tests of the oracle (no GPU): the C restatement is pinned bit-for-bit to the
unmodified reference build and to the committed golden vectors, and passes the
reference test-suite's known-answer tests (proj/tests/test_core.cpp, test_relax.cpp)."""
import glob
import json
import math
import os

import numpy as np
import pytest

from helpers import model_config, random_bounds, random_consistent_bounds
from oracle.oracle import ModelConfig, node_layout
from paper_2209_12708_b200.configs import ALL as CONFIGS

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------------------
# known-answer tests from the reference suite, run on the port
# ---------------------------------------------------------------------------
def test_concretize_linf_corner_kat(port):  # test_core.cpp:76-94
    lo, hi = port.concretize(np.array([[1.0, -2.0]]), np.array([0.5]), np.array([[1.0, -2.0]]), np.array([0.5]),
                             "linf", 0.1)
    assert lo[0] == pytest.approx(0.2, abs=1e-12)
    corners = [0.5 + 1.0 * a - 2.0 * b for a in (-0.1, 0.1) for b in (-0.1, 0.1)]
    assert lo[0] == pytest.approx(min(corners), abs=1e-12)


def test_concretize_l2_345_kat(port):  # test_core.cpp:96-108
    w = np.array([[3.0, 4.0]])
    lo, _ = port.concretize(w, np.array([1.0]), w, np.array([1.0]), "l2", 1.0)
    assert lo[0] == pytest.approx(-4.0, abs=1e-12)


def test_concretize_zero_radius_returns_biases(port):  # test_core.cpp:62-74
    rng = np.random.default_rng(3)
    lw, lb, uw, ub = random_consistent_bounds(rng, (4,), 5)
    lo, hi = port.concretize(lw, lb, uw, ub, "l2", 0.0)
    assert np.array_equal(lo, lb) and np.array_equal(hi, ub)


def test_check_robust_strict(port):  # test_core.cpp:110-129
    assert port.check_robust(np.array([0.4, 0.1]), np.array([0.6, 0.39]), 0)
    assert not port.check_robust(np.array([0.4, 0.1]), np.array([0.6, 0.4]), 0)
    assert port.check_robust(np.array([1.0, 0.0]), np.array([1.5, 0.5]), 0, 0.4)
    assert not port.check_robust(np.array([1.0, 0.0]), np.array([1.5, 0.5]), 0, 0.6)


def test_affine_corner_kat(port):  # test_relax.cpp:49-66
    x = (np.zeros((1, 2, 1)), np.zeros((1, 2)), np.zeros((1, 2, 1)), np.ones((1, 2)))
    y = port.affine(x, np.array([[2.0], [-3.0]]))
    assert y[3][0, 0] == 2.0 and y[1][0, 0] == -3.0


def test_relu_region_kats(port):  # test_relax.cpp:103-123
    al, bl, au, bu = port.relax("relu", np.array([2.0, -3.0, -1.0, -2.0]), np.array([3.0, -1.0, 1.0, 1.0]))
    assert (al[0], au[0], bl[0], bu[0]) == (1.0, 1.0, 0.0, 0.0)
    assert (al[1], au[1], bu[1]) == (0.0, 0.0, 0.0)
    assert au[2] == pytest.approx(0.5) and bu[2] == pytest.approx(0.5) and al[2] == 1.0  # tie -> identity
    assert al[3] == 0.0


def test_exp_recip_kats(port):  # test_relax.cpp:155-171
    al, bl, au, bu = port.relax("exp", np.array([0.0, 0.0]), np.array([0.0, 1.0]))
    assert al[0] == pytest.approx(1.0) and bl[0] == pytest.approx(1.0)
    assert au[1] == pytest.approx(math.e - 1.0)
    al, bl, au, bu = port.relax("recip", np.array([1.0]), np.array([2.0]))
    assert au[0] == pytest.approx(-0.5) and bu[0] == pytest.approx(1.5)
    from oracle.oracle import OracleError
    with pytest.raises(OracleError) as e:
        port.relax("recip", np.array([0.0]), np.array([1.0]))
    assert e.value.kind == "domain_error"


def test_tanh_kats(port):  # test_relax.cpp:125-153
    al, bl, au, bu = port.relax("tanh", np.array([0.0]), np.array([0.0]))
    assert (al[0], bl[0], au[0], bu[0]) == pytest.approx((1.0, 0.0, 1.0, 0.0))


def test_softmax_uniform_at_zero_radius(port):  # test_relax.cpp:356-366
    n = 4
    lw = np.eye(n).reshape(1, n, n)
    lb = np.full((1, n), 0.3)
    y = port.softmax((lw, lb, lw.copy(), lb.copy()), "linf", 0.0)
    assert np.allclose(y[1], 0.25, atol=1e-6) and np.allclose(y[3], 0.25, atol=1e-6)


# ---------------------------------------------------------------------------
# port == unmodified reference, bit for bit
# ---------------------------------------------------------------------------
SMALL = [
    (ModelConfig(1, 2, 16, 32, 8, 2, "relu"), 1, "linf", 0.05),
    (ModelConfig(2, 2, 16, 32, 8, 2, "tanh"), 2, "l2", 0.1),
    (ModelConfig(1, 1, 8, 16, 4, 3, "silu"), 1, "l1", 0.2),
    (ModelConfig(2, 4, 16, 24, 8, 2, "relu"), 2, "l1", 0.02),
]


@pytest.mark.parametrize("cfg,words,norm,eps", SMALL)
def test_port_equals_reference_pass(port, ref, cfg, words, norm, eps):
    params = ref.gen_model(cfg, 77)
    assert np.array_equal(params, port.gen_model(cfg, 77))
    x = ref.gen_input(cfg, 78)
    assert np.array_equal(x, port.gen_input(cfg, 78))
    pos = ref.gen_positions(79, cfg.length, words)
    assert np.array_equal(pos, port.gen_positions(79, cfg.length, words))
    a = port.bound_pass(cfg, params, x, pos, norm, eps, dump=True)
    b = ref.bound_pass(cfg, params, x, pos, norm, eps, dump=True)
    assert a[0] == b[0]
    for u, v in zip(a[1:], b[1:]):
        assert np.array_equal(u, v)


@pytest.mark.parametrize("kind", ["relu", "tanh", "silu", "exp", "recip"])
def test_port_equals_reference_relax(port, ref, kind):
    rng = np.random.default_rng(5)
    a = rng.uniform(-4, 4, 400)
    w = np.where(rng.uniform(size=400) < 0.1, 0.0, rng.uniform(0, 5, 400))
    lo, hi = a, a + w
    if kind == "recip":
        lo, hi = np.abs(lo) + 0.01, np.abs(lo) + 0.01 + w
    assert all(np.array_equal(u, v) for u, v in zip(port.relax(kind, lo, hi), ref.relax(kind, lo, hi)))


def test_port_equals_reference_ops(port, ref):
    rng = np.random.default_rng(9)
    for rep in range(5):
        c, o, d, rows = (int(v) for v in rng.integers(1, 9, 4))
        x = random_bounds(rng, (rows, c), d)
        w = rng.uniform(-1.5, 1.5, (c, o))
        b = rng.uniform(-0.5, 0.5, o)
        assert all(np.array_equal(u, v) for u, v in zip(port.affine(x, w, b), ref.affine(x, w, b)))
    L, E, H, d = 3, 4, 2, 5
    qa = random_consistent_bounds(rng, (L, E), d)
    kb = random_consistent_bounds(rng, (L, E), d)
    for norm in ("l1", "l2", "linf"):
        assert all(np.array_equal(u, v) for u, v in zip(port.dot("similarity", qa, kb, H, norm, 0.1),
                                                        ref.dot("similarity", qa, kb, H, norm, 0.1)))
    pa = random_consistent_bounds(rng, (H * L * L,), d)
    assert all(np.array_equal(u, v) for u, v in zip(port.dot("weighted_values", pa, kb, H, "l2", 0.05),
                                                    ref.dot("weighted_values", pa, kb, H, "l2", 0.05)))
    sx = random_consistent_bounds(rng, (3, 5), d, 0.5)
    assert all(np.array_equal(u, v) for u, v in zip(port.softmax(sx, "linf", 0.05), ref.softmax(sx, "linf", 0.05)))


def test_reference_harness_walk_equals_graph_evaluate(ref):
    """The harness walk (word-level binding aside) is graph::evaluate bit-for-bit."""
    for cfg, norm, eps in [(ModelConfig(1, 2, 16, 32, 8), "linf", 0.05), (ModelConfig(2, 2, 8, 16, 4, 2, "tanh"), "l2", 0.1)]:
        params, x = ref.gen_model(cfg, 5), ref.gen_input(cfg, 6)
        assert ref.selfcheck(cfg, params, x, norm, eps) == 1


# ---------------------------------------------------------------------------
# port == golden vectors generated by the reference build (tests/golden/)
# ---------------------------------------------------------------------------
def _golden_passes():
    return sorted(glob.glob(os.path.join(GOLDEN, "*_pass_s*.npz")))


@pytest.mark.parametrize("path", _golden_passes(), ids=os.path.basename)
def test_port_matches_golden_pass(port, path):
    g = np.load(path)
    name = os.path.basename(path).split("_")[0]
    s = int(os.path.basename(path).split("_s")[1].split(".")[0])
    w = CONFIGS[name]
    if name in ("c3", "c4m") and not os.environ.get("FAITH_SLOW_TESTS"):
        pytest.skip(f"{name} reference pass takes minutes on one core (set FAITH_SLOW_TESTS=1)")
    if name in ("c4", "c5s") and not os.environ.get("FAITH_VERY_SLOW_TESTS"):
        pytest.skip(f"{name} reference pass takes hours on one core (set FAITH_VERY_SLOW_TESTS=1)")
    cfg = model_config(w)
    params = port.gen_model(cfg, w.model_seed)
    x = port.gen_input(cfg, w.input_seed(s))
    pos = port.gen_positions(w.position_seed(s), w.length, w.words)
    assert np.array_equal(pos, g["positions"])
    st, lo, hi, nlo, nhi = port.bound_pass(cfg, params, x, pos, w.norm, float(g["eps"]), dump=True)
    assert st == int(g["status"])
    assert np.array_equal(lo, g["logits_lo"]) and np.array_equal(hi, g["logits_hi"])
    idx = g["node_index"]
    assert g["node_lo"].dtype == np.float64  # golden node bounds are stored bit-exact
    assert np.array_equal(nlo[idx], g["node_lo"])
    assert np.array_equal(nhi[idx], g["node_hi"])


def _golden_maxeps():
    return sorted(glob.glob(os.path.join(GOLDEN, "*_maxeps_s*.json")))


@pytest.mark.parametrize("path", [p for p in _golden_maxeps() if "c1_" in p], ids=os.path.basename)
def test_port_matches_golden_maxeps(port, path):
    rec = json.load(open(path))
    w = CONFIGS[rec["config"]]
    cfg = model_config(w)
    params = port.gen_model(cfg, w.model_seed)
    s = rec["sentence"]
    x = port.gen_input(cfg, w.input_seed(s))
    pos = port.gen_positions(w.position_seed(s), w.length, w.words)
    st, eps, calls, pred = port.maxeps(cfg, params, x, pos, rec["norm"], rec["eps_max"], rec["tol"])
    assert (st, eps, calls, pred) == (rec["status"], rec["max_epsilon"], rec["calls"], rec["predicted"])


def test_node_layout_matches_dump_size(port):
    for w in CONFIGS.values():
        cfg = model_config(w)
        lay = node_layout(cfg)
        assert lay[-1][1] + lay[-1][2] == port.node_dump_size(cfg)
