"""EXTENSION: the sqrt / square envelopes and the LayerNorm bound chain.

The reference has neither (proj/include/faith/model.hpp:22-24: no layer normalization;
proj/include/faith/relax.hpp:62-66: no sqrt), so there is no oracle: these tests are
soundness-only, as G3 prescribes -- envelope containment on dense grids, and 10^4 sampled
perturbations of a LayerNorm input whose every output lies inside the propagated linear
bounds -- plus F32-mode vs F64-mode agreement of the chain."""
import numpy as np
import pytest

from helpers import sample_in_ball
from paper_2209_12708_b200 import faith_gpu as F

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,fn,intervals", [
    ("sqrt", np.sqrt, [(0.0, 1.0), (0.25, 4.0), (1e-6, 1e-3), (2.0, 2.0), (0.0, 0.0), (3.0, 3.5)]),
    ("square", np.square, [(-1.0, 2.0), (-3.0, -1.0), (0.5, 0.75), (2.0, 2.0), (-1e-3, 1e-3)]),
])
def test_envelope_contains_function(ctx, kind, fn, intervals):
    lo = np.array([a for a, _ in intervals])
    hi = np.array([b for _, b in intervals])
    r = ctx.relax(kind, lo, hi)
    for i, (a, b) in enumerate(intervals):
        xs = np.linspace(a, b, 1001)
        f = fn(xs)
        low = r.a_low[i] * xs + r.b_low[i]
        up = r.a_up[i] * xs + r.b_up[i]
        tol = 1e-12 * np.maximum(1.0, np.abs(f))
        assert np.all(low <= f + tol) and np.all(f <= up + tol), (kind, a, b)
        if a == b:  # a point interval collapses onto the function value
            assert low[0] == pytest.approx(f[0], abs=1e-15) and up[0] == pytest.approx(f[0], abs=1e-15)


def test_sqrt_domain_error(ctx):
    with pytest.raises(F.DomainError):
        ctx.relax("sqrt", [-0.1], [1.0])


def _ln(x, gamma, beta, delta):
    mu = x.mean(axis=-1, keepdims=True)
    c = x - mu
    return c / np.sqrt((c * c).mean(axis=-1, keepdims=True) + delta) * gamma + beta


@pytest.mark.parametrize("precision", ["f32", "f64"])
@pytest.mark.parametrize("norm,eps", [("linf", 0.02), ("l2", 0.05), ("l1", 0.1)])
def test_layernorm_bounds_are_sound(precision, norm, eps):
    ctx = F.Context(0)
    ctx.set_precision(precision)
    rng = np.random.default_rng(5)
    n, E, d = 6, 16, 8
    x0 = rng.normal(size=(n, E))
    lam = rng.uniform(-0.5, 0.5, size=(n, E, d))  # x(δ) = x0 + lam δ exactly: lw = uw = lam
    gamma, beta, delta = rng.uniform(0.5, 1.5, E), rng.normal(size=E), 1e-5
    y = ctx.propagate_layernorm((lam, x0, lam.copy(), x0.copy()), gamma, beta, norm, eps, delta)
    deltas = sample_in_ball(rng, norm, eps, d, 10_000)
    xs = x0[None] + np.einsum("ned,sd->sne", lam, deltas)
    out = _ln(xs, gamma, beta, delta)
    low = y.lb[None] + np.einsum("ned,sd->sne", y.lw, deltas)
    up = y.ub[None] + np.einsum("ned,sd->sne", y.uw, deltas)
    slack = (1e-6 if precision == "f32" else 1e-9) * np.maximum(1.0, np.abs(out))
    assert np.max(low - out - slack) <= 0.0 and np.max(out - up - slack) <= 0.0
    # the concretized bounds contain every sample too, and are not vacuous
    lo, hi = ctx.concretize(y, norm, eps)
    assert np.all(lo[None] <= out + slack) and np.all(out <= hi[None] + slack)
    assert np.all(hi - lo < 10.0)


def test_layernorm_f32_matches_f64():
    rng = np.random.default_rng(9)
    n, E, d = 4, 32, 16
    x0 = rng.normal(size=(n, E))
    lam = rng.uniform(-0.2, 0.2, size=(n, E, d))
    gamma, beta = rng.uniform(0.5, 1.5, E), rng.normal(size=E)
    res = {}
    for precision in ("f32", "f64"):
        ctx = F.Context(0)
        ctx.set_precision(precision)
        y = ctx.propagate_layernorm((lam, x0, lam.copy(), x0.copy()), gamma, beta, "l2", 0.01)
        res[precision] = ctx.concretize(y, "l2", 0.01)
    for a, b in zip(res["f32"], res["f64"]):
        assert np.allclose(a, b, rtol=1e-4, atol=1e-4)


def test_layernorm_zero_radius_is_exact():
    ctx = F.Context(0)
    ctx.set_precision("f64")
    rng = np.random.default_rng(2)
    x0 = rng.normal(size=(3, 8))
    lam = rng.uniform(-1, 1, size=(3, 8, 4))
    gamma, beta = np.ones(8), np.zeros(8)
    y = ctx.propagate_layernorm((lam, x0, lam.copy(), x0.copy()), gamma, beta, "linf", 0.0)
    lo, hi = ctx.concretize(y, "linf", 0.0)
    want = _ln(x0, gamma, beta, 1e-5)
    assert np.allclose(lo, want, atol=1e-9) and np.allclose(hi, want, atol=1e-9)
