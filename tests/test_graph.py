"""faith-graph/v1 host side: the graphs the UNMODIFIED reference exported
with graph::to_json (tests/golden/graphs, oracle/graph_golden.cpp) parse and validate like
graph::graph_from_json / VerGraph::validate (proj/src/graph.cpp:133-160, 816-850), and malformed
graphs are rejected with the reference's messages.  The device evaluation is tests/test_gpu_graph.py."""
import glob
import json
import os

import pytest

from paper_2209_12708_b200 import graph as G
from paper_2209_12708_b200.faith_gpu import InvalidArgument

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "graphs")
GRAPHS = sorted(glob.glob(os.path.join(GOLD, "*.graph.json")))


def test_golden_set_present():
    assert len(GRAPHS) == 30


@pytest.mark.parametrize("path", GRAPHS, ids=[os.path.basename(p)[:-11] for p in GRAPHS])
def test_reference_graphs_parse(path):
    g = G.load_graph(path)
    with open(path) as f:
        j = json.load(f)
    assert [n.kind for n in g.nodes] == [n["kind"] for n in j["nodes"]]
    assert g.input_names() == ["x"]
    kinds = {n.kind for n in g.nodes}
    if "_fused" in path:  # fuse_all leaves only fused affine / expanded softmax forms
        assert not kinds & {"split_signs", "matmul_pair", "combine_halves", "affine_bound", "merge_sides",
                            "softmax"}
    for n in g.nodes:
        for role, src in zip(G.input_roles(n.kind, len(n.inputs)), n.inputs):
            assert j["nodes"][n.id]["edges"][role] == src


def _mutate(fn):
    with open(os.path.join(GOLD, "random0.graph.json")) as f:
        j = json.load(f)
    fn(j)
    return json.dumps(j)


def test_malformed_graphs_rejected():
    with pytest.raises(InvalidArgument, match="unsupported format"):
        G.graph_from_json(_mutate(lambda j: j.update(format="faith-graph/v0")))
    with pytest.raises(InvalidArgument, match="unknown kind 'conv'"):
        G.graph_from_json(_mutate(lambda j: j["nodes"][3].update(kind="conv")))
    with pytest.raises(InvalidArgument, match="ids must be dense and ordered"):
        G.graph_from_json(_mutate(lambda j: j["nodes"][2].update(id=7)))

    def forward(j):
        n = next(n for n in j["nodes"] if "edges" in n)
        n["edges"][next(iter(n["edges"]))] = len(j["nodes"]) - 1
    with pytest.raises(InvalidArgument, match="cycle or forward edge"):
        G.graph_from_json(_mutate(forward))
    with pytest.raises(InvalidArgument, match="weight node without constant"):
        G.graph_from_json(_mutate(lambda j: next(n for n in j["nodes"] if n["kind"] == "weight").update(constant=999)))
    with pytest.raises(InvalidArgument, match="missing from fusion groups"):
        G.graph_from_json(_mutate(lambda j: j["fusion_groups"].pop()))
    with pytest.raises(InvalidArgument, match="node in two fusion groups"):
        G.graph_from_json(_mutate(lambda j: j["fusion_groups"].append(j["fusion_groups"][0])))
    with pytest.raises(InvalidArgument, match="non-operator node"):
        G.graph_from_json(_mutate(lambda j: j["fusion_groups"].append([0])))


def test_missing_fusion_groups_default_to_singletons():
    g = G.graph_from_json(_mutate(lambda j: j.pop("fusion_groups")))
    ops = [n.id for n in g.nodes if n.kind not in ("input", "weight")]
    assert g.fusion_groups == [[i] for i in ops]


@pytest.mark.parametrize("path", GRAPHS, ids=[os.path.basename(p)[:-11] for p in GRAPHS])
def test_export_is_byte_identical_to_reference(path):
    """graph::to_json (graph.cpp:781-814): parse -> export reproduces the reference's own bytes."""
    with open(path) as f:
        text = f.read().strip()
    assert G.to_json(G.graph_from_json(text)) == text
