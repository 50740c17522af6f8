"""Shared test helpers (mirrors proj/tests/helpers.hpp where noted)."""
from __future__ import annotations

import numpy as np

TOL = 1e-4  # BASELINE.json north_star: per-neuron bounds within 1e-4, scale rule of acceptance.cpp:122


def close(got, want, tol=TOL):
    """abs(got - want) <= tol * max(1, abs(want)) elementwise (NaN in `got` = not materialised, skipped)."""
    got, want = np.asarray(got, dtype=np.float64), np.asarray(want, dtype=np.float64)
    mask = ~np.isnan(got)
    err = np.abs(got[mask] - want[mask]) / np.maximum(1.0, np.abs(want[mask]))
    return err.size == 0 or bool(np.all(err <= tol)), (float(err.max()) if err.size else 0.0)


def random_consistent_bounds(rng: np.random.Generator, shape, pert, scale=1.0):
    """helpers.hpp:172-189: shared weight rows, lb <= ub."""
    shape = tuple(shape)
    lw = rng.uniform(-scale, scale, shape + (pert,))
    c = rng.uniform(-scale, scale, shape)
    lb = c - rng.uniform(0, scale, shape)
    ub = c + rng.uniform(0, scale, shape)
    return lw, lb, lw.copy(), ub


def random_bounds(rng, shape, pert, scale=1.0):
    """Independent lower/upper rows (decoupled, as test_relax.cpp:86 does for the affine KAT)."""
    lw, lb, _, ub = random_consistent_bounds(rng, shape, pert, scale)
    uw = rng.uniform(-scale, scale, tuple(shape) + (pert,))
    return lw, lb, uw, ub


def sample_in_ball(rng: np.random.Generator, p: str, eps: float, dim: int, n: int) -> np.ndarray:
    """helpers.hpp:16-54 (same distributions; numpy RNG): n samples with ||delta||_p <= eps,
    a quarter of them pushed onto the sphere."""
    if p == "linf":
        d = rng.uniform(-eps, eps, (n, dim))
        edge = rng.uniform(size=n) < 0.25
        d[edge] = np.where(d[edge] >= 0, eps, -eps)
        return d
    if p == "l2":
        g = rng.normal(size=(n, dim))
        norm = np.linalg.norm(g, axis=1, keepdims=True)
        norm[norm == 0] = 1.0
        radius = eps * rng.uniform(size=(n, 1)) ** (1.0 / dim)
        radius[rng.uniform(size=n) < 0.25] = eps
        return g / norm * radius
    v = -np.log(1.0 - rng.uniform(size=(n, dim)))
    radius = eps * rng.uniform(size=(n, 1))
    radius[rng.uniform(size=n) < 0.25] = eps
    v = v / v.sum(axis=1, keepdims=True) * radius
    return np.where(rng.uniform(size=(n, dim)) < 0.5, -v, v)


def model_config(w):
    from oracle.oracle import ModelConfig
    return ModelConfig(w.layers, w.heads, w.embed, w.ffn, w.length, w.classes, w.activation)
