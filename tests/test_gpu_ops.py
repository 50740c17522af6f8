"""Operator-level parity on the GPU: every bound operator of the C ABI against the
C restatement of the reference (oracle/faith_oracle.c), on seeded random inputs incl.
ragged shapes, plus the reference suite's known-answer tests.  Tolerance: the
north_star's 1e-4 with the acceptance.cpp:122 scale rule (Λ is f32 on the device)."""
import math

import numpy as np
import pytest

from helpers import close, random_bounds, random_consistent_bounds
from paper_2209_12708_b200 import faith_gpu as F

pytestmark = pytest.mark.gpu

NORMS = ["l1", "l2", "linf"]


def _ul(t):
    lw, lb, uw, ub = t
    return lw, lb, uw, ub


def assert_bounds_close(got, want, tol=1e-4, what=""):
    for name, g, w in zip(("lw", "lb", "uw", "ub"), got, want):
        ok, err = close(np.asarray(g).ravel(), np.asarray(w).ravel(), tol)
        assert ok, f"{what} {name}: max scaled error {err:.3e}"


# ---- known-answer tests (proj/tests/test_core.cpp, test_relax.cpp) ----------------
def test_concretize_kats(ctx):
    lo, hi = ctx.concretize((np.array([[1.0, -2.0]]), np.array([0.5]), np.array([[1.0, -2.0]]), np.array([0.5])),
                            "linf", 0.1)
    # the f32 kernels pad every concretized norm outward by 2^-20 (fg_kernels.cu kNormPad):
    # lo moves down by at most eps * ||lw|| * 2^-20, never up
    assert 0.2 - 0.3 * 2.0 ** -19 <= lo[0] <= 0.2 + 1e-12
    w = np.array([[3.0, 4.0]])
    lo, _ = ctx.concretize((w, np.array([1.0]), w, np.array([1.0])), "l2", 1.0)
    assert -4.0 - 5.0 * 2.0 ** -19 <= lo[0] <= -4.0 + 1e-12


def test_affine_corner_kat(ctx):
    x = (np.zeros((2, 1)), np.zeros(2), np.zeros((2, 1)), np.ones(2))
    y = ctx.propagate_affine(x, np.array([[2.0], [-3.0]]))
    assert y.ub[0] == 2.0 and y.lb[0] == -3.0


def test_relax_kats(ctx):
    r = ctx.relax("relu", [2.0, -3.0, -1.0, -2.0], [3.0, -1.0, 1.0, 1.0])
    assert (r.a_low[0], r.a_up[0]) == (1.0, 1.0)
    assert r.a_up[2] == pytest.approx(0.5) and r.a_low[2] == 1.0 and r.a_low[3] == 0.0
    r = ctx.relax("exp", [0.0, 0.0], [0.0, 1.0])
    assert r.a_low[0] == pytest.approx(1.0) and r.b_low[0] == pytest.approx(1.0)
    assert r.a_up[1] == pytest.approx(math.e - 1)
    r = ctx.relax("recip", [1.0], [2.0])
    assert r.a_up[0] == pytest.approx(-0.5) and r.b_up[0] == pytest.approx(1.5)
    with pytest.raises(F.DomainError):
        ctx.relax("recip", [0.0], [1.0])
    with pytest.raises(F.InvalidArgument):
        ctx.relax("relu", [1.0], [0.0])  # lo > hi (bounds.cpp:69-78)


def test_softmax_uniform_kat(ctx):
    n = 4
    lw = np.eye(n).reshape(1, n, n)
    y = ctx.propagate_softmax((lw, np.full((1, n), 0.3), lw.copy(), np.full((1, n), 0.3)), "linf", 0.0)
    assert np.allclose(y.lb, 0.25, atol=1e-6) and np.allclose(y.ub, 0.25, atol=1e-6)


# ---- parity against the oracle -------------------------------------------------------
@pytest.mark.parametrize("norm", NORMS)
@pytest.mark.parametrize("n,d", [(1, 1), (7, 3), (64, 128), (33, 515)])
def test_concretize_parity(ctx, port, norm, n, d):
    rng = np.random.default_rng(n * 1000 + d)
    b = random_bounds(rng, (n,), d)
    lo, hi = ctx.concretize(b, norm, 0.37)
    plo, phi = port.concretize(*b, norm, 0.37)
    assert close(lo, plo)[0] and close(hi, phi)[0]


@pytest.mark.parametrize("rows,c,o,d", [(1, 1, 1, 1), (3, 5, 7, 3), (4, 12, 9, 8), (8, 64, 96, 64), (2, 256, 130, 132)])
def test_affine_parity(ctx, port, rows, c, o, d):
    rng = np.random.default_rng(rows * 7 + c * 13 + o * 17 + d)
    x = random_bounds(rng, (rows, c), d)
    w = rng.uniform(-1.5, 1.5, (c, o)).astype(np.float32).astype(np.float64)  # reference weights are f32-rounded
    b = rng.uniform(-0.5, 0.5, o)
    got = ctx.propagate_affine(x, w, b)
    want = port.affine(x, w, b)
    assert_bounds_close(got, want, what="affine")
    # bias path is f64 (FMA-contracted sum of the sign-selected products): f64 rounding only
    assert np.allclose(got.lb, want[1], rtol=1e-13, atol=1e-14) and np.allclose(got.ub, want[3], rtol=1e-13,
                                                                                atol=1e-14)


@pytest.mark.parametrize("kind", ["relu", "tanh", "silu", "exp", "recip"])
def test_relax_parity(ctx, port, kind):
    rng = np.random.default_rng(11)
    a = rng.uniform(-4, 4, 1000)
    w = np.where(rng.uniform(size=1000) < 0.1, 0.0, rng.uniform(0, 5, 1000))
    lo, hi = (np.abs(a) + 0.01, np.abs(a) + 0.01 + w) if kind == "recip" else (a, a + w)
    got = ctx.relax(kind, lo, hi)
    want = port.relax(kind, lo, hi)
    for g, p in zip(got, want):
        assert close(g, p, 1e-12)[0]


@pytest.mark.parametrize("kind", ["relu", "tanh", "silu", "exp"])
@pytest.mark.parametrize("norm", NORMS)
def test_elementwise_verify_parity(ctx, port, kind, norm):
    rng = np.random.default_rng(21)
    b = random_consistent_bounds(rng, (96,), 40, 0.5)
    got = ctx.elementwise_verify(kind, b, norm, 0.05)
    want = port.elementwise_verify(kind, b, norm, 0.05)
    assert_bounds_close(got, want, what=kind)


def test_compose_parity_with_sign_swap(ctx, port):
    rng = np.random.default_rng(23)
    b = random_bounds(rng, (50,), 7)
    rel = tuple(rng.uniform(-2, 2, 50) for _ in range(4))
    assert_bounds_close(ctx.compose_elementwise(b, rel), port.compose(b, rel), what="compose")


@pytest.mark.parametrize("L,E,H,d", [(3, 4, 2, 5), (8, 16, 2, 12), (16, 32, 4, 64)])
@pytest.mark.parametrize("norm", NORMS)
def test_dot_similarity_parity(ctx, port, L, E, H, d, norm):
    rng = np.random.default_rng(L * 100 + d)
    a = random_consistent_bounds(rng, (1, L, E), d, 0.5)
    b = random_consistent_bounds(rng, (1, L, E), d, 0.5)
    got = ctx.propagate_dot_product(a, b, norm, 0.1, "similarity", H)
    want = port.dot("similarity", [t.reshape(L * E, -1) if t.ndim == 4 else t.reshape(L, E) for t in a],
                    [t.reshape(L * E, -1) if t.ndim == 4 else t.reshape(L, E) for t in b], H, norm, 0.1)
    assert_bounds_close([g.reshape(-1) for g in got], [w.reshape(-1) for w in want], what="QK^T")


@pytest.mark.parametrize("L,E,H,d", [(3, 4, 2, 5), (8, 16, 2, 12), (16, 32, 4, 64)])
def test_dot_weighted_parity(ctx, port, L, E, H, d):
    rng = np.random.default_rng(L * 10 + d)
    a = random_consistent_bounds(rng, (1, H, L, L), d, 0.5)
    b = random_consistent_bounds(rng, (1, L, E), d, 0.5)
    got = ctx.propagate_dot_product(a, b, "l2", 0.05, "weighted_values", H)
    want = port.dot("weighted_values", [t.reshape(H * L * L, -1) if t.ndim == 5 else t.reshape(-1) for t in a],
                    [t.reshape(L * E, -1) if t.ndim == 4 else t.reshape(L, E) for t in b], H, "l2", 0.05)
    assert_bounds_close([g.reshape(-1) for g in got], [w.reshape(-1) for w in want], what="PV")


@pytest.mark.parametrize("rows,n,d", [(1, 4, 4), (3, 5, 7), (16, 64, 128), (4, 128, 1536)])
@pytest.mark.parametrize("norm", NORMS)
def test_softmax_parity(ctx, port, rows, n, d, norm):
    rng = np.random.default_rng(rows + n + d)
    b = random_consistent_bounds(rng, (rows, n), d, 0.3 / math.sqrt(d))
    got = ctx.propagate_softmax(b, norm, 0.1)
    want = port.softmax(b, norm, 0.1)
    assert_bounds_close(got, want, what="softmax")


def test_softmax_domain_error_on_wide_interval(ctx, port):  # test_relax.cpp:506-520
    b = (np.ones((1, 3, 2)) * 50.0, np.zeros((1, 3)), np.ones((1, 3, 2)) * 50.0, np.zeros((1, 3)))
    from oracle.oracle import OracleError
    with pytest.raises(OracleError) as e:
        port.softmax(b, "linf", 20.0)
    with pytest.raises(F.DomainError):
        ctx.propagate_softmax(b, "linf", 20.0)
    assert e.value.kind == "domain_error"


def test_add_scale(ctx, port):
    rng = np.random.default_rng(31)
    a = random_bounds(rng, (20,), 6)
    b = random_bounds(rng, (20,), 6)
    y = ctx.propagate_add(a, b)
    assert np.allclose(y.lw, a[0] + b[0], atol=1e-6) and np.array_equal(y.lb, a[1] + b[1])
    s = ctx.propagate_scale(a, -0.5)  # sign swap (relax.cpp:692-701)
    assert np.allclose(s.lw, -0.5 * a[2], atol=1e-6) and np.array_equal(s.ub, -0.5 * a[1])
