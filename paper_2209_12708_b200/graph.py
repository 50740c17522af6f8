"""faith-graph/v1 verification graphs on the device.

``load_graph`` / ``graph_from_json`` / ``to_json`` read and write the reference's graph schema (``graph::to_json`` /
``graph_from_json``, proj/src/graph.cpp:781-850, README "File formats") and check it the way
``VerGraph::validate`` does (graph.cpp:133-160: dense ordered ids, no forward edges, weights bound
to constants, every operator in exactly one fusion group).  :class:`Graph` uploads the constant
table once and runs ``graph::evaluate`` (graph.cpp:505-673) through the C-ABI graph executor
(fg_graph_* in include/faith_gpu.h): every node on the GPU in the exact f64 arithmetic, values
resident in HBM, the sink's LinearBounds returned.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field
from typing import List, Mapping, Optional

import numpy as np

from .faith_gpu import NORM, Context, InvalidArgument, LinearBounds, _dp

KINDS = ["input", "weight", "split_signs", "matmul_pair", "combine_halves", "affine_bound", "merge_sides",
         "affine_verify", "dot_product", "scale", "add", "mean_pool", "relu_verify", "tanh_verify", "silu_verify",
         "softmax", "exp_verify", "sum_reduce", "recip_verify", "mul_broadcast"]  # graph.cpp:14-35, FG_NODE_*
KIND = {k: i for i, k in enumerate(KINDS)}
MAX_RANK = 8


def input_roles(kind: str, count: int) -> List[str]:
    """Edge role names per operator kind, in input order (graph.cpp:684-706)."""
    if kind == "split_signs":
        return ["w"]
    if kind == "matmul_pair":
        return ["x", "halves"]
    if kind == "combine_halves":
        return ["pos", "neg", "bias"] if count == 3 else ["pos", "neg"]
    if kind in ("affine_bound", "affine_verify"):
        return ["x", "w", "bias"] if count == 3 else ["x", "w"]
    if kind in ("merge_sides", "dot_product", "add"):
        return ["a", "b"]
    if kind == "mul_broadcast":
        return ["x", "r"]
    return ["x"]


class FgNode(C.Structure):
    _fields_ = [("kind", C.c_int), ("n_inputs", C.c_int), ("inputs", C.c_int * 3), ("sign", C.c_int),
                ("side", C.c_int), ("layout", C.c_int), ("heads", C.c_int), ("axis", C.c_int),
                ("scale", C.c_double), ("constant", C.c_int), ("input", C.c_int)]


@dataclass
class Node:
    """graph::Node (graph.hpp:59-67)."""
    id: int
    kind: str
    inputs: List[int] = field(default_factory=list)
    attrs: dict = field(default_factory=dict)
    shape: List[int] = field(default_factory=list)
    constant: int = -1


@dataclass
class VerGraph:
    nodes: List[Node]
    constants: List[np.ndarray]
    fusion_groups: List[List[int]]

    def input_names(self) -> List[str]:
        return [n.attrs["name"] for n in self.nodes if n.kind == "input"]

    def validate(self) -> None:
        """VerGraph::validate (graph.cpp:133-160)."""
        for i, n in enumerate(self.nodes):
            if n.id != i:
                raise InvalidArgument("VerGraph: node id out of order")
            if any(x >= i or x < 0 for x in n.inputs):
                raise InvalidArgument("VerGraph: cycle or forward edge")
            if n.kind == "weight" and not 0 <= n.constant < len(self.constants):
                raise InvalidArgument("VerGraph: weight node without constant")
        seen = [0] * len(self.nodes)
        for group in self.fusion_groups:
            for i in group:
                if not 0 <= i < len(self.nodes) or self.nodes[i].kind in ("input", "weight"):
                    raise InvalidArgument("VerGraph: fusion group contains non-operator node")
                seen[i] += 1
                if seen[i] > 1:
                    raise InvalidArgument("VerGraph: node in two fusion groups")
        for n in self.nodes:
            if n.kind not in ("input", "weight") and not seen[n.id]:
                raise InvalidArgument("VerGraph: operator node missing from fusion groups")


def graph_from_json(text: str) -> VerGraph:
    """graph::graph_from_json (graph.cpp:816-850)."""
    j = json.loads(text)
    if j.get("format") != "faith-graph/v1":
        raise InvalidArgument("graph_from_json: unsupported format")
    constants = []
    for c in j["constants"]:
        shape = [int(s) for s in c["shape"]]
        data = np.asarray(c["data"], dtype=np.float64).reshape(-1)
        if data.size != int(np.prod(shape, dtype=np.int64)):
            raise InvalidArgument("Tensor: data size does not match shape")
        constants.append(data.reshape(shape))
    nodes = []
    for i, jn in enumerate(j["nodes"]):
        kind = jn["kind"]
        if kind not in KIND:
            raise InvalidArgument(f"node_kind_from_name: unknown kind '{kind}'")
        a = jn.get("attrs", {})
        attrs = {}
        if kind == "matmul_pair":
            attrs["sign"] = a["sign"]
        elif kind == "affine_bound":
            attrs["side"] = a["side"]
        elif kind == "dot_product":
            attrs["layout"], attrs["heads"] = a["layout"], int(a["heads"])
        elif kind == "scale":
            attrs["scale"] = float(a["scale"])
        elif kind in ("softmax", "sum_reduce", "recip_verify", "exp_verify", "mul_broadcast", "mean_pool"):
            attrs["axis"] = int(a["axis"])
        elif kind == "input":
            attrs["name"] = a["name"]
        inputs = []
        if kind not in ("input", "weight") and "edges" in jn:
            edges = jn["edges"]
            inputs = [int(edges[r]) for r in input_roles(kind, len(edges))]
        node = Node(i, kind, inputs, attrs, [int(s) for s in jn["shape"]],
                    int(jn["constant"]) if kind == "weight" else -1)
        if int(jn["id"]) != i:
            raise InvalidArgument("graph_from_json: node ids must be dense and ordered")
        nodes.append(node)
    if "fusion_groups" in j:
        groups = [[int(x) for x in g] for g in j["fusion_groups"]]
    else:  # reset_fusion_groups: one singleton group per operator node
        groups = [[n.id] for n in nodes if n.kind not in ("input", "weight")]
    g = VerGraph(nodes, constants, groups)
    g.validate()
    return g


def to_json(g: VerGraph) -> str:
    """graph::to_json (graph.cpp:781-814): nodes with kind, attrs, role-named edges, shape and
    the constant index of weights; the constant table; the fusion groups.  Keys sorted and
    compact separators, as nlohmann::json::dump() writes them."""
    nodes = []
    for n in g.nodes:
        jn = {"id": n.id, "kind": n.kind, "attrs": dict(n.attrs), "shape": list(n.shape)}
        if n.inputs:
            jn["edges"] = {r: x for r, x in zip(input_roles(n.kind, len(n.inputs)), n.inputs)}
        if n.kind == "weight":
            jn["constant"] = n.constant
        nodes.append(jn)
    consts = [{"shape": list(c.shape), "data": [float(v) for v in np.asarray(c, dtype=np.float64).reshape(-1)]}
              for c in g.constants]
    j = {"format": "faith-graph/v1", "nodes": nodes, "constants": consts, "fusion_groups": g.fusion_groups}
    return json.dumps(j, sort_keys=True, separators=(",", ":"))


def load_graph(path: str) -> VerGraph:
    with open(path) as f:
        return graph_from_json(f.read())


class Graph:
    """A VerGraph resident on one device: constants uploaded once, evaluate() per input binding."""

    def __init__(self, ctx: Context, g: VerGraph):
        g.validate()
        self.ctx, self.lib, self.graph = ctx, ctx.lib, g
        L = self.lib
        if not getattr(L, "_graph_types", False):
            vp, sz = C.c_void_p, C.c_size_t
            L.fg_graph_create.argtypes = [vp, sz, C.POINTER(FgNode), sz, C.POINTER(sz), C.POINTER(sz),
                                          C.POINTER(_dp), C.POINTER(vp)]
            L.fg_graph_destroy.argtypes = [vp]
            L.fg_graph_evaluate.argtypes = [vp, sz, C.POINTER(sz), C.POINTER(sz), C.POINTER(_dp), C.c_int,
                                            C.c_double, sz]
            L.fg_graph_result_shape.argtypes = [vp, C.POINTER(sz), C.POINTER(sz), C.POINTER(sz)]
            L.fg_graph_result.argtypes = [vp, _dp, _dp, _dp, _dp]
            L._graph_types = True
        self.names = g.input_names()
        slot = {name: i for i, name in enumerate(dict.fromkeys(self.names))}
        self.slots = list(slot)
        arr = (FgNode * len(g.nodes))()
        for n, fn in zip(g.nodes, arr):
            fn.kind = KIND[n.kind]
            fn.n_inputs = len(n.inputs)
            for k, x in enumerate(n.inputs[:3]):
                fn.inputs[k] = x
            fn.sign = 0 if n.attrs.get("sign", "pos") == "pos" else 1
            fn.side = 0 if n.attrs.get("side", "lower") == "lower" else 1
            fn.layout = 0 if n.attrs.get("layout", "similarity") == "similarity" else 1
            fn.heads = int(n.attrs.get("heads", 1))
            fn.axis = int(n.attrs.get("axis", 0))
            fn.scale = float(n.attrs.get("scale", 1.0))
            fn.constant = n.constant
            fn.input = slot[n.attrs["name"]] if n.kind == "input" else -1
        nc = len(g.constants)
        self._consts = [np.ascontiguousarray(c, dtype=np.float64) for c in g.constants]
        for c in self._consts:
            if c.ndim > MAX_RANK:
                raise InvalidArgument("graph constant rank too large")
        ranks = (C.c_size_t * max(1, nc))(*[c.ndim for c in self._consts])
        shapes = (C.c_size_t * (max(1, nc) * MAX_RANK))()
        for i, c in enumerate(self._consts):
            for k, e in enumerate(c.shape):
                shapes[i * MAX_RANK + k] = e
        ptrs = (_dp * max(1, nc))(*[c.ctypes.data_as(_dp) for c in self._consts])
        h = C.c_void_p()
        ctx._check(L.fg_graph_create(ctx.handle, len(g.nodes), arr, nc, ranks, shapes, ptrs, C.byref(h)),
                   "fg_graph_create")
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            self.lib.fg_graph_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def evaluate(self, inputs: Mapping[str, np.ndarray], norm: str, eps: float,
                 dim: Optional[int] = None) -> LinearBounds:
        """graph::evaluate(g, inputs, PerturbationSpec{norm, eps, dim}) -> LinearBounds of the sink
        (lw/uw shaped [*sink_shape, dim]).  dim defaults to the inputs' element count."""
        arrays = []
        for name in self.slots:
            if name not in inputs:
                raise InvalidArgument(f"evaluate: missing input binding '{name}'")
            arrays.append(np.ascontiguousarray(inputs[name], dtype=np.float64))
        if dim is None:
            dim = arrays[0].size if arrays else 1
        n = max(1, len(arrays))
        ranks = (C.c_size_t * n)(*[a.ndim for a in arrays])
        shapes = (C.c_size_t * (n * MAX_RANK))()
        for i, a in enumerate(arrays):
            if a.ndim > MAX_RANK:
                raise InvalidArgument("input_bounds: input rank too large")
            for k, e in enumerate(a.shape):
                shapes[i * MAX_RANK + k] = e
        ptrs = (_dp * n)(*[a.ctypes.data_as(_dp) for a in arrays])
        self.ctx._check(self.lib.fg_graph_evaluate(self.handle, len(arrays), ranks, shapes, ptrs, NORM[norm],
                                                   float(eps), int(dim)), "evaluate")
        rank, d = C.c_size_t(), C.c_size_t()
        shape = (C.c_size_t * MAX_RANK)()
        self.ctx._check(self.lib.fg_graph_result_shape(self.handle, C.byref(rank), shape, C.byref(d)), "evaluate")
        s = tuple(shape[i] for i in range(rank.value))
        lb, ub = np.zeros(s), np.zeros(s)
        lw, uw = np.zeros(s + (d.value,)), np.zeros(s + (d.value,))
        self.ctx._check(self.lib.fg_graph_result(self.handle, lw.ctypes.data_as(_dp), lb.ctypes.data_as(_dp),
                                                 uw.ctypes.data_as(_dp), ub.ctypes.data_as(_dp)), "evaluate")
        return LinearBounds(lw, lb, uw, ub)
