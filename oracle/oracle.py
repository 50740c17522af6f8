"""TEST INFRASTRUCTURE ONLY -- ctypes front-end of the CPU oracles.

Loads either implementation of ``oracle/faith_oracle.h``:

* ``port``      -- ``oracle/_build/libfaith_oracle.so``, the plain-C restatement
                   (always available; travels to the GPU box as a built .so);
* ``reference`` -- ``oracle/_ref/libfaith_ref.so``, the unmodified reference
                   sources + harness (built only where /root/reference exists).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (CPU baseline /
reference arm) may import this module: it is the checker, never the product.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "port": os.path.join(HERE, "_build", "libfaith_oracle.so"),
    "reference": os.path.join(HERE, "_ref", "libfaith_ref.so"),
}

NORM = {"l1": 0, "l2": 1, "linf": 2}
ACT = {"relu": 0, "tanh": 1, "silu": 2}
RELAX = {"relu": 0, "tanh": 1, "silu": 2, "exp": 3, "recip": 4}
STATUS = {0: "ok", 1: "invalid_argument", 2: "domain_error", 3: "out_of_range", 4: "runtime_error"}


class FoConfig(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("layers", "heads", "embed", "ffn", "length", "classes", "activation")]


@dataclass(frozen=True)
class ModelConfig:
    layers: int
    heads: int
    embed: int
    ffn: int
    length: int
    classes: int = 2
    activation: str = "relu"

    def fo(self) -> FoConfig:
        return FoConfig(self.layers, self.heads, self.embed, self.ffn, self.length, self.classes, ACT[self.activation])


_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


def _d(a):
    return None if a is None else a.ctypes.data_as(_dp)


def _i(a):
    return a.ctypes.data_as(_ip)


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: {STATUS.get(code, code)}")
        self.code = code
        self.kind = STATUS.get(code, str(code))


class Oracle:
    def __init__(self, impl: str = "port"):
        path = LIBS[impl]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library {path} not built (run `make -C oracle`)")
        self.impl = impl
        self.lib = L = C.CDLL(path)
        L.fo_param_count.restype = C.c_size_t
        L.fo_node_dump_size.restype = C.c_size_t
        L.fo_impl_name.restype = C.c_char_p
        for name in ("fo_gen_model", "fo_gen_input", "fo_gen_positions", "fo_forward", "fo_concretize",
                     "fo_check_robust", "fo_affine", "fo_relax", "fo_compose", "fo_elementwise_verify",
                     "fo_dot", "fo_softmax", "fo_bound_pass", "fo_maxeps", "fo_rng_uniform"):
            getattr(L, name).restype = C.c_int
        L.fo_gen_model.argtypes = [C.POINTER(FoConfig), C.c_uint64, _dp]
        L.fo_gen_input.argtypes = [C.POINTER(FoConfig), C.c_uint64, _dp]
        L.fo_rng_uniform.argtypes = [C.c_uint64, C.c_size_t, _dp]
        L.fo_concretize.argtypes = [C.c_size_t, C.c_size_t, _dp, _dp, _dp, _dp, C.c_int, C.c_double, _dp, _dp]
        L.fo_check_robust.argtypes = [C.c_size_t, _dp, _dp, C.c_size_t, C.c_double, _ip]
        L.fo_affine.argtypes = [C.c_size_t] * 4 + [_dp] * 10
        L.fo_relax.argtypes = [C.c_int, C.c_size_t] + [_dp] * 6
        L.fo_compose.argtypes = [C.c_size_t, C.c_size_t] + [_dp] * 12
        L.fo_elementwise_verify.argtypes = [C.c_int, C.c_size_t, C.c_size_t] + [_dp] * 4 + [C.c_int, C.c_double] + [_dp] * 4
        L.fo_dot.argtypes = [C.c_int] + [C.c_size_t] * 4 + [_dp] * 8 + [C.c_int, C.c_double] + [_dp] * 4
        L.fo_softmax.argtypes = [C.c_size_t] * 3 + [_dp] * 4 + [C.c_int, C.c_double] + [_dp] * 4
        L.fo_bound_pass.argtypes = [C.POINTER(FoConfig), _dp, _dp, _ip, C.c_int, C.c_int, C.c_double, _dp, _dp, _dp, _dp]
        L.fo_maxeps.argtypes = [C.POINTER(FoConfig), _dp, _dp, _ip, C.c_int, C.c_int, C.c_double, C.c_double, _dp, _ip, _ip]
        if impl == "reference":
            L.fo_ref_selfcheck.restype = C.c_int
            L.fo_ref_selfcheck.argtypes = [C.POINTER(FoConfig), _dp, _dp, C.c_int, C.c_double]

    @staticmethod
    def _check(code: int, what: str):
        if code != 0:
            raise OracleError(code, what)

    # ---- model / inputs ---------------------------------------------------
    def param_count(self, cfg: ModelConfig) -> int:
        return int(self.lib.fo_param_count(C.byref(cfg.fo())))

    def gen_model(self, cfg: ModelConfig, seed: int) -> np.ndarray:
        p = np.zeros(self.param_count(cfg))
        self._check(self.lib.fo_gen_model(C.byref(cfg.fo()), seed, _d(p)), "gen_model")
        return p

    def gen_input(self, cfg: ModelConfig, seed: int) -> np.ndarray:
        x = np.zeros(cfg.length * cfg.embed)
        self._check(self.lib.fo_gen_input(C.byref(cfg.fo()), seed, _d(x)), "gen_input")
        return x

    def gen_positions(self, seed: int, length: int, words: int) -> np.ndarray:
        p = np.zeros(words, dtype=np.int32)
        self._check(self.lib.fo_gen_positions(C.c_uint64(seed), length, words, _i(p)), "gen_positions")
        return p

    def rng_uniform(self, seed: int, n: int) -> np.ndarray:
        out = np.zeros(n)
        self.lib.fo_rng_uniform(seed, n, _d(out))
        return out

    def forward(self, cfg: ModelConfig, params, x) -> np.ndarray:
        out = np.zeros(cfg.classes)
        self._check(self.lib.fo_forward(C.byref(cfg.fo()), _d(params), _d(x), _d(out)), "forward")
        return out

    # ---- operators (reference u/l layout) ----------------------------------
    def concretize(self, lw, lb, uw, ub, norm: str, eps: float):
        n, d = lw.shape
        lo, hi = np.zeros(n), np.zeros(n)
        self._check(self.lib.fo_concretize(n, d, _d(lw), _d(lb), _d(uw), _d(ub), NORM[norm], eps, _d(lo), _d(hi)),
                    "concretize")
        return lo, hi

    def check_robust(self, lo, hi, true_class: int, margin: float = 0.0) -> bool:
        v = np.zeros(1, dtype=np.int32)
        self._check(self.lib.fo_check_robust(len(lo), _d(lo), _d(hi), true_class, margin, _i(v)), "check_robust")
        return bool(v[0])

    def affine(self, x, w, bias=None):
        lw, lb, uw, ub = x
        rows, c = lb.shape
        o = w.shape[1]
        d = lw.shape[-1]
        y = [np.zeros((rows, o, d)), np.zeros((rows, o)), np.zeros((rows, o, d)), np.zeros((rows, o))]
        self._check(self.lib.fo_affine(rows, c, o, d, *map(_d, (lw, lb, uw, ub)), _d(w), _d(bias), *map(_d, y)),
                    "affine")
        return tuple(y)

    def relax(self, kind: str, lo, hi):
        n = len(lo)
        out = [np.zeros(n) for _ in range(4)]
        self._check(self.lib.fo_relax(RELAX[kind], n, _d(lo), _d(hi), *map(_d, out)), f"relax_{kind}")
        return tuple(out)

    def compose(self, x, rel):
        lw, lb, uw, ub = x
        n, d = lw.shape
        y = [np.zeros((n, d)), np.zeros(n), np.zeros((n, d)), np.zeros(n)]
        self._check(self.lib.fo_compose(n, d, *map(_d, (lw, lb, uw, ub)), *map(_d, rel), *map(_d, y)), "compose")
        return tuple(y)

    def elementwise_verify(self, kind: str, x, norm: str, eps: float):
        lw, lb, uw, ub = x
        n, d = lw.shape
        y = [np.zeros((n, d)), np.zeros(n), np.zeros((n, d)), np.zeros(n)]
        self._check(self.lib.fo_elementwise_verify(RELAX[kind], n, d, *map(_d, (lw, lb, uw, ub)), NORM[norm], eps,
                                                   *map(_d, y)), f"elementwise_verify({kind})")
        return tuple(y)

    def dot(self, layout: str, a, b, heads: int, norm: str, eps: float):
        alw, alb, auw, aub = a
        blw, blb, buw, bub = b
        length, embed = blb.shape
        d = blw.shape[-1]
        lay = 0 if layout == "similarity" else 1
        ny = heads * length * length if lay == 0 else length * embed
        y = [np.zeros((ny, d)), np.zeros(ny), np.zeros((ny, d)), np.zeros(ny)]
        self._check(self.lib.fo_dot(lay, length, embed, heads, d, *map(_d, (alw, alb, auw, aub)),
                                    *map(_d, (blw, blb, buw, bub)), NORM[norm], eps, *map(_d, y)), "dot")
        return tuple(y)

    def softmax(self, x, norm: str, eps: float):
        lw, lb, uw, ub = x
        rows, n = lb.shape
        d = lw.shape[-1]
        y = [np.zeros((rows, n, d)), np.zeros((rows, n)), np.zeros((rows, n, d)), np.zeros((rows, n))]
        self._check(self.lib.fo_softmax(rows, n, d, *map(_d, (lw, lb, uw, ub)), NORM[norm], eps, *map(_d, y)),
                    "softmax")
        return tuple(y)

    # ---- pass level ---------------------------------------------------------
    def node_dump_size(self, cfg: ModelConfig) -> int:
        return int(self.lib.fo_node_dump_size(C.byref(cfg.fo())))

    def bound_pass(self, cfg: ModelConfig, params, x, positions, norm: str, eps: float, dump: bool = False):
        """Returns (status, logits_lo, logits_hi, node_lo, node_hi)."""
        lo, hi = np.zeros(cfg.classes), np.zeros(cfg.classes)
        nlo = nhi = None
        if dump:
            n = self.node_dump_size(cfg)
            nlo, nhi = np.zeros(n), np.zeros(n)
        pos = np.ascontiguousarray(positions, dtype=np.int32)
        st = self.lib.fo_bound_pass(C.byref(cfg.fo()), _d(params), _d(x), _i(pos), len(pos), NORM[norm], eps,
                                    _d(lo), _d(hi), _d(nlo), _d(nhi))
        return st, lo, hi, nlo, nhi

    def maxeps(self, cfg: ModelConfig, params, x, positions, norm: str, eps_max: float, tol: float):
        """Returns (status, eps, calls, predicted)."""
        e = np.zeros(1)
        calls = np.zeros(1, dtype=np.int32)
        pred = np.zeros(1, dtype=np.int32)
        pos = np.ascontiguousarray(positions, dtype=np.int32)
        st = self.lib.fo_maxeps(C.byref(cfg.fo()), _d(params), _d(x), _i(pos), len(pos), NORM[norm], eps_max, tol,
                                _d(e), _i(calls), _i(pred))
        return st, float(e[0]), int(calls[0]), int(pred[0])

    def selfcheck(self, cfg: ModelConfig, params, x, norm: str, eps: float) -> int:
        return int(self.lib.fo_ref_selfcheck(C.byref(cfg.fo()), _d(params), _d(x), NORM[norm], eps))


def node_layout(cfg: ModelConfig):
    """Names and sizes of the nodes fo_bound_pass dumps, in order."""
    L, E, H, F = cfg.length, cfg.embed, cfg.heads, cfg.ffn
    per = [("q", L * E), ("k", L * E), ("v", L * E), ("scores", H * L * L), ("scaled", H * L * L),
           ("exp", H * L * L), ("sum", H * L), ("recip", H * L), ("probs", H * L * L), ("ctx", L * E),
           ("attn", L * E), ("res1", L * E), ("f1", L * F), ("act", L * F), ("f2", L * E), ("res2", L * E)]
    out, off = [], 0
    for layer in range(cfg.layers):
        for name, n in per:
            out.append((f"l{layer}.{name}", off, n))
            off += n
    out.append(("pooled", off, E))
    off += E
    out.append(("logits", off, cfg.classes))
    return out
