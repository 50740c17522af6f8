"""Exact precision mode (FG_PRECISION_F64) of the operator-level C ABI: f64 kernels in the
reference's operation order.  The arithmetic operators must be BIT-IDENTICAL to the
reference (checked against the plain-C restatement oracle/faith_oracle.c, itself pinned
bit-for-bit to the unmodified reference build by tests/test_oracle.py); operators that go
through exp/tanh agree to the device libm's last ulps (rel 1e-12).  The extra operators that
the restatement does not export (sum_axis, mul_broadcast, bilinear) are checked against
numpy restatements that keep relax.cpp's accumulation order."""
import numpy as np
import pytest

from helpers import random_bounds, random_consistent_bounds
from paper_2209_12708_b200 import faith_gpu as F

pytestmark = pytest.mark.gpu

NORMS = ["l1", "l2", "linf"]


@pytest.fixture(scope="module")
def ctx64():
    c = F.Context(0)
    c.set_precision("f64")
    assert c.precision == "f64"
    return c


def same(got, want):
    for g, w in zip(got, want):
        g, w = np.asarray(g).ravel(), np.asarray(w).ravel()
        assert g.shape == w.shape
        assert np.array_equal(g.view(np.int64), w.view(np.int64)), f"max diff {np.max(np.abs(g - w)):.3e}"


def near(got, want, rel=1e-12):
    for g, w in zip(got, want):
        g, w = np.asarray(g).ravel(), np.asarray(w).ravel()
        assert np.all(np.abs(g - w) <= rel * np.maximum(1.0, np.abs(w))), f"max diff {np.max(np.abs(g - w)):.3e}"


def test_affine_bitwise_acceptance_criterion3(ctx64, port):
    """acceptance.cpp:133-156: 100 random shapes, bitwise equal to the four-multiplication order."""
    rng = np.random.default_rng(2024)
    for _ in range(100):
        c, o, rows, d = (int(rng.integers(1, 33)), int(rng.integers(1, 33)), int(rng.integers(1, 33)),
                         int(rng.integers(1, 9)))
        lw, lb, _, ub = random_consistent_bounds(rng, (rows, c), d)
        uw = rng.uniform(-1, 1, (rows, c, d))
        w = rng.uniform(-1.5, 1.5, (c, o))
        bias = rng.uniform(-0.5, 0.5, o)
        got = ctx64.propagate_affine((lw, lb, uw, ub), w, bias)
        want = port.affine((lw, lb, uw, ub), w, bias)
        same(got, want)


@pytest.mark.parametrize("rows,c,o,d", [(4, 256, 130, 132), (64, 64, 192, 64)])
def test_affine_bitwise_large(ctx64, port, rows, c, o, d):
    rng = np.random.default_rng(rows + c + o + d)
    x = random_bounds(rng, (rows, c), d)
    w = rng.uniform(-0.1, 0.1, (c, o))
    same(ctx64.propagate_affine(x, w), port.affine(x, w))


@pytest.mark.parametrize("norm", NORMS)
def test_concretize_bitwise(ctx64, port, norm):
    rng = np.random.default_rng(7)
    for n, d in [(1, 1), (9, 5), (300, 513)]:
        b = random_bounds(rng, (n,), d)
        same(ctx64.concretize(b, norm, 0.37), port.concretize(*b, norm, 0.37))


@pytest.mark.parametrize("kind", ["relu", "recip", "exp", "tanh", "silu"])
def test_relax_compose_verify(ctx64, port, kind):
    rng = np.random.default_rng(11)
    n, d = 257, 17
    x = random_consistent_bounds(rng, (n,), d, 0.4)
    if kind == "recip":
        x = (x[0], x[1] + 3.0, x[2], x[3] + 3.0)
    lo, hi = port.concretize(*x, "l2", 0.05)
    check = same if kind in ("relu", "recip") else near
    rel = ctx64.relax(kind, lo, hi)
    prel = port.relax(kind, lo, hi)
    check(rel, prel)
    same(ctx64.compose_elementwise(x, prel), port.compose(x, prel))
    check(ctx64.elementwise_verify(kind, x, "l2", 0.05), port.elementwise_verify(kind, x, "l2", 0.05))


@pytest.mark.parametrize("norm", NORMS)
def test_dot_products_bitwise(ctx64, port, norm):
    rng = np.random.default_rng(13)
    L, E, H, d = 6, 8, 2, 5
    q = random_consistent_bounds(rng, (1, L, E), d, 0.5)
    k = random_consistent_bounds(rng, (1, L, E), d, 0.5)
    got = ctx64.propagate_dot_product(q, k, norm, 0.03, "similarity", H)
    want = port.dot("similarity", tuple(t[0] for t in q), tuple(t[0] for t in k), H, norm, 0.03)
    same(got, want)
    p = random_consistent_bounds(rng, (1, H, L, L), d, 0.5)
    got = ctx64.propagate_dot_product(p, k, norm, 0.03, "weighted_values", H)
    want = port.dot("weighted_values", tuple(t[0] for t in p), tuple(t[0] for t in k), H, norm, 0.03)
    same(got, want)


def test_dot_batched_equals_slices(ctx64):
    rng = np.random.default_rng(17)
    B, L, E, H, d = 3, 5, 6, 3, 4
    q = random_consistent_bounds(rng, (B, L, E), d, 0.5)
    k = random_consistent_bounds(rng, (B, L, E), d, 0.5)
    got = ctx64.propagate_dot_product_batched(q, k, "l2", 0.02, "similarity", H)
    for b in range(B):
        one = ctx64.propagate_dot_product(tuple(t[b:b + 1] for t in q), tuple(t[b:b + 1] for t in k), "l2", 0.02,
                                          "similarity", H)
        same(tuple(t[b:b + 1] for t in got), one)


def test_add_scale_bitwise(ctx64):
    rng = np.random.default_rng(19)
    a = random_bounds(rng, (40,), 7)
    b = random_bounds(rng, (40,), 7)
    y = ctx64.propagate_add(a, b)
    same(y, tuple(np.asarray(s) + np.asarray(t) for s, t in zip(a, b)))
    for s in (0.125, -0.7):
        y = ctx64.propagate_scale(a, s)
        lw, lb, uw, ub = a
        want = (s * lw, s * lb, s * uw, s * ub) if s >= 0 else (s * uw, s * ub, s * lw, s * lb)
        same(y, want)


def _sum_axis_np(x, axis):
    lw, lb, uw, ub = (np.asarray(t) for t in x)
    n = lb.shape[axis]
    acc = [np.zeros_like(np.take(t, [0], axis=axis)) for t in (lw, lb, uw, ub)]
    for j in range(n):  # relax.cpp:728-737: sequential over the reduced axis
        for a, t in zip(acc, (lw, lb, uw, ub)):
            a += np.take(t, [j], axis=axis)
    return tuple(acc)


def test_sum_axis_bitwise(ctx64):
    rng = np.random.default_rng(23)
    x = random_bounds(rng, (3, 7, 4), 6)
    for axis in (0, 1, 2):
        same(ctx64.propagate_sum_axis(x, axis), _sum_axis_np(x, axis))


def _mul_broadcast_np(x, r, axis, port, norm, eps):
    """relax.cpp:744-775 with accumulate_product_term's order, elementwise in numpy."""
    xlw, xlb, xuw, xub = (np.asarray(t) for t in x)
    rlw, rlb, ruw, rub = (np.asarray(t) for t in r)
    d = xlw.shape[-1]
    xlo, _ = port.concretize(xlw.reshape(-1, d), xlb.ravel(), xuw.reshape(-1, d), xub.ravel(), norm, eps)
    rlo, rhi = port.concretize(rlw.reshape(-1, d), rlb.ravel(), ruw.reshape(-1, d), rub.ravel(), norm, eps)
    rlo = np.broadcast_to(rlo.reshape(rlb.shape), xlb.shape)
    rhi = np.broadcast_to(rhi.reshape(rlb.shape), xlb.shape)
    lx, ly, uy = xlo.reshape(xlb.shape), rlo, rhi
    bl = lambda a, b: np.broadcast_to(a, b.shape)  # noqa: E731
    rlb_, rub_ = bl(rlb, xlb), bl(rub, xlb)
    rlw_, ruw_ = np.broadcast_to(rlw, xlw.shape), np.broadcast_to(ruw, xlw.shape)
    out_lb = np.zeros_like(xlb) + (ly * np.where(ly >= 0, xlb, xub) + lx * np.where(lx >= 0, rlb_, rub_) - lx * ly)
    out_ub = np.zeros_like(xub) + (uy * np.where(uy >= 0, xub, xlb) + lx * np.where(lx >= 0, rub_, rlb_) - lx * uy)
    e = lambda v: v[..., None]  # noqa: E731
    out_lw = np.zeros_like(xlw)
    out_lw = out_lw + np.where(e(ly) != 0, e(ly) * np.where(e(ly) >= 0, xlw, xuw), 0.0)
    out_lw = out_lw + np.where(e(lx) != 0, e(lx) * np.where(e(lx) >= 0, rlw_, ruw_), 0.0)
    out_uw = np.zeros_like(xuw)
    out_uw = out_uw + np.where(e(uy) != 0, e(uy) * np.where(e(uy) >= 0, xuw, xlw), 0.0)
    out_uw = out_uw + np.where(e(lx) != 0, e(lx) * np.where(e(lx) >= 0, ruw_, rlw_), 0.0)
    return out_lw, out_lb, out_uw, out_ub


@pytest.mark.parametrize("norm", NORMS)
def test_mul_broadcast_bitwise(ctx64, port, norm):
    rng = np.random.default_rng(29)
    x = random_consistent_bounds(rng, (2, 5, 3), 4, 0.5)
    r = random_consistent_bounds(rng, (2, 1, 3), 4, 0.5)
    got = ctx64.propagate_mul_broadcast(x, r, 1, norm, 0.05)
    same(got, _mul_broadcast_np(x, r, 1, port, norm, 0.05))


def test_bilinear_bitwise_and_validation(ctx64):
    rng = np.random.default_rng(31)
    xlo = rng.uniform(-2, 2, 50)
    xhi = xlo + rng.uniform(0, 2, 50)
    ylo = rng.uniform(-2, 2, 50)
    yhi = ylo + rng.uniform(0, 2, 50)
    got = ctx64.relax_bilinear(xlo, xhi, ylo, yhi)
    same(got, (ylo, xlo, -xlo * ylo, yhi, xlo, -xlo * yhi))
    with pytest.raises(F.InvalidArgument):
        ctx64.relax_bilinear([1.0], [0.0], [0.0], [1.0])


def test_softmax_f64_matches_port(ctx64, port):
    rng = np.random.default_rng(37)
    x = random_consistent_bounds(rng, (6, 9), 5, 0.3)
    near(ctx64.propagate_softmax(x, "l2", 0.05), port.softmax(x, "l2", 0.05))
    # general axis: softmax over axis 0 == softmax over the last axis of the transpose
    xt = tuple(np.ascontiguousarray(np.swapaxes(t, 0, 1)) for t in (x[0], x[1], x[2], x[3]))
    got = ctx64.propagate_softmax_axis(xt, 0, "l2", 0.05)
    want = port.softmax(x, "l2", 0.05)
    near(tuple(np.swapaxes(g, 0, 1) for g in got), want)


def test_error_taxonomy_f64(ctx64):
    with pytest.raises(F.DomainError):
        ctx64.relax("recip", [0.0], [1.0])
    with pytest.raises(F.InvalidArgument):
        ctx64.relax("exp", [1.0], [0.0])
    x = (np.ones((1, 2)), np.zeros(1), np.ones((1, 2)), np.zeros(1))
    with pytest.raises(F.InvalidArgument):
        ctx64.concretize(x, "l2", -1.0)
