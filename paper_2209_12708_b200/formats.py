"""The reference's persistent formats, read and written on the host so a model file produced by
the reference (``faith gen`` / ``model::save_model``) goes straight into a device-resident
:class:`faith_gpu.Model` (weights uploaded and pre-split into f32 hi/lo planes once at model
creation) -- SURVEY 8(f) rank 2.

* ``faith-model/v1`` manifest: ``model::save_model`` / ``model::load_model``
  (proj/src/model.cpp:235-335; README.md "File formats").  Tensor references are inline
  ``{"shape", "values"}`` or ``{"shape", "blob", "offset"}`` into a little-endian f32 blob next to
  the manifest, offset in elements (model.cpp:147-223).
* ``faith-embedding/v1``: ``model::save_embedding`` / ``load_embedding`` (model.cpp:337-369).

Errors mirror the reference's ``std::runtime_error`` texts (prefix ``load_model: <path>: ``) and
raise :class:`FormatError` (a ``RuntimeError``).  Weights are f32 on disk, so a save/load round
trip is exact; values are handed to the model as f64 like ``Tensor`` holds them (model.cpp:92).
"""
from __future__ import annotations

import json
import os
from typing import Dict, List, Sequence, Tuple

import numpy as np

from .faith_gpu import ModelConfig

ACTIVATIONS = ("relu", "tanh", "silu")
LAYER_KEYS = ("wq", "bq", "wk", "bk", "wv", "bv", "wo", "bo", "w1", "b1", "w2", "b2")


class FormatError(RuntimeError):
    pass


def _layer_shapes(cfg: ModelConfig) -> List[Tuple[str, Tuple[int, ...]]]:
    E, F = cfg.embed, cfg.ffn
    return [("wq", (E, E)), ("bq", (E,)), ("wk", (E, E)), ("bk", (E,)), ("wv", (E, E)), ("bv", (E,)),
            ("wo", (E, E)), ("bo", (E,)), ("w1", (E, F)), ("b1", (F,)), ("w2", (F, E)), ("b2", (E,))]


def param_count(cfg: ModelConfig) -> int:
    """TransformerSpec::parameter_count (model.cpp:75-79)."""
    E, F, C = cfg.embed, cfg.ffn, cfg.classes
    return cfg.layers * (4 * (E * E + E) + E * F + F + F * E + E) + E * C + C


def _shape_str(shape: Sequence[int]) -> str:
    return "[" + ", ".join(str(int(s)) for s in shape) + "]"


class _Blobs:
    """BlobCache (model.cpp:171-193): each blob file read once, as little-endian f32."""

    def __init__(self, base: str):
        self.base, self.cache = base, {}

    def get(self, name: str, context: str) -> np.ndarray:
        if name not in self.cache:
            path = os.path.join(self.base, name)
            try:
                with open(path, "rb") as f:
                    raw = f.read()
            except OSError:
                raise FormatError(f"cannot open blob '{name}' (referenced by {context})") from None
            self.cache[name] = np.frombuffer(raw[: len(raw) // 4 * 4], dtype="<f4")
        return self.cache[name]


def _read_tensor(ref: dict, blobs: _Blobs, context: str) -> Tuple[Tuple[int, ...], np.ndarray]:
    """read_tensor (model.cpp:195-223) -> (shape, f64 values)."""
    if "shape" not in ref:
        raise FormatError(f"{context}: tensor reference needs 'shape'")
    shape = tuple(int(s) for s in ref["shape"])
    n = int(np.prod(shape, dtype=np.int64)) if shape else 1
    if "values" in ref:
        vals = np.asarray(ref["values"], dtype=np.float64).reshape(-1)
        if vals.size != n:
            raise FormatError(f"{context}: shape {_shape_str(shape)} expects {n} values, got {vals.size}")
    elif "blob" in ref:
        name = str(ref["blob"])
        blob = blobs.get(name, context)
        off = int(ref.get("offset", 0))
        if off + n > blob.size:
            raise FormatError(f"blob '{name}' truncated reading {context} ({off + n} elements needed, "
                              f"{blob.size} present)")
        vals = blob[off:off + n].astype(np.float64)
    else:
        raise FormatError(f"{context}: tensor reference needs 'values' or 'blob'")
    if not np.all(np.isfinite(vals)):  # Tensor's constructor (tensor.cpp:26-60)
        raise FormatError(f"{context}: Tensor: non-finite value")
    return shape, vals


def _validate(cfg: ModelConfig, shapes: Dict[str, Tuple[int, ...]], nlayers: int, strict: bool):
    """TransformerSpec::validate (model.cpp:39-73).  strict=False lifts only the [1, 6] layer
    cap (the BERT-base-shaped c5 workload is 12 layers)."""
    if cfg.layers < 1 or (strict and cfg.layers > 6):
        raise FormatError("TransformerSpec: num_layers must be in [1, 6]")
    if cfg.heads == 0 or cfg.embed % cfg.heads:
        raise FormatError("TransformerSpec: embed_dim must be divisible by num_heads")
    if nlayers != cfg.layers:
        raise FormatError("TransformerSpec: layer weight count mismatch")
    for l in range(cfg.layers):
        for key, want in _layer_shapes(cfg):
            got = shapes[f"layers[{l}].{key}"]
            if got != want:
                raise FormatError(f"TransformerSpec: layers[{l}].{key} has shape {_shape_str(got)}, expected "
                                  f"{_shape_str(want)}")
    for key, want in (("classifier.w", (cfg.embed, cfg.classes)), ("classifier.b", (cfg.classes,))):
        if shapes[key] != want:
            raise FormatError(f"TransformerSpec: {key} has shape {_shape_str(shapes[key])}, expected "
                              f"{_shape_str(want)}")


def load_model(path: str, strict: bool = True) -> Tuple[ModelConfig, np.ndarray]:
    """model::load_model (model.cpp:287-335) -> (config, params in fg_model_create order)."""
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise FormatError(f"load_model: cannot open '{path}'") from None
    try:
        j = json.loads(text)
    except ValueError as e:
        raise FormatError(f"load_model: {path}: {e}") from None
    try:
        if j.get("format") != "faith-model/v1":
            raise FormatError("unsupported format")
        act = j["activation"]
        if act not in ACTIVATIONS:
            raise FormatError(f"unknown activation '{act}'")
        cfg = ModelConfig(int(j["num_layers"]), int(j["num_heads"]), int(j["embed_dim"]), int(j["ffn_dim"]),
                          int(j["length"]), int(j["num_classes"]), act)
        blobs = _Blobs(os.path.dirname(os.path.abspath(path)))
        shapes, parts = {}, []
        for l, jl in enumerate(j["layers"]):
            for key in LAYER_KEYS:
                ctx = f"layers[{l}].{key}"
                shapes[ctx], v = _read_tensor(jl[key], blobs, ctx)
                parts.append(v)
        for key in ("w", "b"):
            ctx = f"classifier.{key}"
            shapes[ctx], v = _read_tensor(j["classifier"][key], blobs, ctx)
            parts.append(v)
        _validate(cfg, shapes, len(j["layers"]), strict)
    except KeyError as e:
        raise FormatError(f"load_model: {path}: missing key {e}") from None
    except FormatError as e:
        raise FormatError(f"load_model: {path}: {e}") from None
    return cfg, np.concatenate(parts)


def load_embedding(path: str, cfg: ModelConfig = None) -> np.ndarray:
    """model::load_embedding (model.cpp:353-369) -> [L*E] f64.  With cfg, the shape must be
    [1, length, embed_dim] (the batch-1 input the model consumes)."""
    try:
        with open(path) as f:
            j = json.load(f)
    except OSError:
        raise FormatError(f"load_embedding: cannot open '{path}'") from None
    except ValueError as e:
        raise FormatError(f"load_embedding: {path}: {e}") from None
    try:
        if j.get("format") != "faith-embedding/v1":
            raise FormatError("unsupported format")
        shape, v = _read_tensor(j["tensor"], _Blobs(os.path.dirname(os.path.abspath(path))), "embedding")
    except KeyError as e:
        raise FormatError(f"load_embedding: {path}: missing key {e}") from None
    except FormatError as e:
        raise FormatError(f"load_embedding: {path}: {e}") from None
    if cfg is not None and shape != (1, cfg.length, cfg.embed):
        raise FormatError(f"load_embedding: {path}: shape {_shape_str(shape)}, expected "
                          f"{_shape_str((1, cfg.length, cfg.embed))}")
    return v


class _BlobWriter:
    """BlobWriter (model.cpp:147-165): tensors appended as f32, offsets in elements."""

    def __init__(self, path: str):
        self.f = open(path, "wb")
        self.name = os.path.basename(path)
        self.offset = 0

    def ref(self, shape, v) -> dict:
        a = np.asarray(v, dtype="<f4").reshape(-1)
        self.f.write(a.tobytes())
        r = {"shape": list(shape), "blob": self.name, "offset": self.offset}
        self.offset += a.size
        return r


def _inline(shape, v) -> dict:
    return {"shape": list(shape), "values": np.asarray(v, dtype=np.float32).astype(np.float64).reshape(-1).tolist()}


def save_model(cfg: ModelConfig, params: np.ndarray, path: str, inline: bool = False) -> None:
    """model::save_model (model.cpp:235-285): manifest + <stem>.bin blob (or inline values)."""
    params = np.asarray(params, dtype=np.float64).reshape(-1)
    if params.size != param_count(cfg):
        raise FormatError(f"save_model: {params.size} parameters, expected {param_count(cfg)}")
    blob = None if inline else _BlobWriter(os.path.splitext(path)[0] + ".bin")
    ref = _inline if inline else blob.ref
    pos = 0

    def take(shape):
        nonlocal pos
        n = int(np.prod(shape))
        v = params[pos:pos + n]
        pos += n
        return ref(shape, v)

    layers = []
    for _ in range(cfg.layers):
        layers.append({key: take(shape) for key, shape in _layer_shapes(cfg)})
    j = {"format": "faith-model/v1", "num_layers": cfg.layers, "num_heads": cfg.heads, "embed_dim": cfg.embed,
         "ffn_dim": cfg.ffn, "length": cfg.length, "batch_size": 1, "num_classes": cfg.classes,
         "activation": cfg.activation, "layers": layers,
         "classifier": {"w": take((cfg.embed, cfg.classes)), "b": take((cfg.classes,))}}
    if blob:
        blob.f.close()
    with open(path, "w") as f:
        json.dump(j, f, indent=1)
        f.write("\n")


def save_embedding(x: np.ndarray, cfg: ModelConfig, path: str, inline: bool = False) -> None:
    """model::save_embedding (model.cpp:337-351), shape [1, length, embed_dim]."""
    shape = (1, cfg.length, cfg.embed)
    x = np.asarray(x, dtype=np.float64).reshape(-1)
    if x.size != cfg.length * cfg.embed:
        raise FormatError(f"save_embedding: {x.size} values, expected {cfg.length * cfg.embed}")
    if inline:
        t = _inline(shape, x)
    else:
        w = _BlobWriter(os.path.splitext(path)[0] + ".bin")
        t = w.ref(shape, x)
        w.f.close()
    with open(path, "w") as f:
        json.dump({"format": "faith-embedding/v1", "tensor": t}, f, indent=1)
        f.write("\n")
