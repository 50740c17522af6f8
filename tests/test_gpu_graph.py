"""Device graph executor (fg_graph_*) against the UNMODIFIED reference's
graph::evaluate on the golden faith-graph/v1 cases (tests/golden/graphs, oracle/graph_golden.cpp):
random verification workloads in their split / per-side / fused affine forms with activations,
scales, residual adds and attention blocks (workloads.hpp random_workload, acceptance.cpp:215-225),
and model::build_graph transformers (relu / tanh / silu), unfused and after fuse_all; five
perturbation specs each, including eps = 0 and radii where the reference raises.

Bar: graphs whose nodes are arithmetic only (affine forms, scale, add, relu, dot products) are
BIT-IDENTICAL to the reference (exact f64 mode, reference operation order); graphs with exp / tanh /
SiLU / recip envelopes agree to 1e-12 * max(1, |ref|) (device libm vs host libm last-ulp); every
reference exception is reproduced with the same taxonomy (domain_error / invalid_argument)."""
import glob
import json
import os

import numpy as np
import pytest

from paper_2209_12708_b200 import faith_gpu as F
from paper_2209_12708_b200 import graph as G

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "graphs")
CASES = sorted(glob.glob(os.path.join(GOLD, "*.expect.json")))
TRANSCENDENTAL = {"tanh_verify", "silu_verify", "exp_verify", "recip_verify", "softmax"}


@pytest.fixture(scope="module")
def ctx():
    return F.Context(0)


def _t(d):
    return np.asarray(d["data"], dtype=np.float64).reshape(d["shape"])


@pytest.mark.parametrize("case", CASES, ids=[os.path.basename(p)[:-12] for p in CASES])
def test_graph_matches_reference_evaluate(ctx, case):
    with open(case) as f:
        c = json.load(f)
    vg = G.load_graph(os.path.join(GOLD, c["graph"]))
    exact = not ({n.kind for n in vg.nodes} & TRANSCENDENTAL)
    g = G.Graph(ctx, vg)
    x = _t(c["input"])
    for run in c["runs"]:
        if "error" in run:
            exc = F.DomainError if run["error"] == "domain_error" else F.InvalidArgument
            with pytest.raises(exc):
                g.evaluate({"x": x}, run["norm"], run["eps"], run["dim"])
            continue
        y = g.evaluate({"x": x}, run["norm"], run["eps"], run["dim"])
        for name, got in zip(("lw", "lb", "uw", "ub"), y):
            ref = _t(run[name])
            assert got.shape == ref.shape, (name, got.shape, ref.shape)
            if exact:
                assert np.array_equal(got, ref), (name, run["norm"], run["eps"], np.max(np.abs(got - ref)))
            else:
                err = np.max(np.abs(got - ref) / np.maximum(1.0, np.abs(ref)))
                assert err <= 1e-12, (name, run["norm"], run["eps"], err)


def test_graph_errors_and_bindings(ctx):
    vg = G.load_graph(os.path.join(GOLD, "random0.graph.json"))
    g = G.Graph(ctx, vg)
    x = np.zeros((1, 3, 4))
    with pytest.raises(F.InvalidArgument, match="missing input binding 'x'"):
        g.evaluate({"y": x}, "linf", 0.1)
    with pytest.raises(F.InvalidArgument, match="spec.dim"):
        g.evaluate({"x": x}, "linf", 0.1, dim=5)
    with pytest.raises(F.InvalidArgument, match="epsilon"):
        g.evaluate({"x": x}, "linf", -1.0)
    y = g.evaluate({"x": x}, "linf", 0.0)  # re-evaluation on the same resident graph
    assert y.lw.shape == (1, 3, 4, 12)
