"""Python front-end of libfaith_gpu.so (include/faith_gpu.h) via ctypes.

Mirrors the reference verifier's operator interface (proj/include/faith/relax.hpp,
bounds.hpp) and its certify / max-epsilon commands (proj/include/faith/cli.hpp) with
the same names, argument meaning and error behaviour: reference exceptions map to
``InvalidArgument`` (std::invalid_argument), ``DomainError`` (std::domain_error) and
``OutOfRange`` (std::out_of_range).

There is no CPU fallback: importing works without a GPU, but creating a ``Context``
requires the in-tree CUDA library and an sm_100 device and raises otherwise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import NamedTuple, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libfaith_gpu.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "faith_gpu.h")

FG_OK, FG_EINVAL, FG_EDOMAIN, FG_ERANGE, FG_ERUNTIME, FG_ECUDA, FG_ENOMEM = range(7)
NORM = {"l1": 0, "l2": 1, "linf": 2}
RELAX = {"relu": 0, "tanh": 1, "silu": 2, "exp": 3, "recip": 4,
         "sqrt": 5, "square": 6}  # extension: LayerNorm bound chain (no reference counterpart)
DOT = {"similarity": 0, "weighted_values": 1}
# ambiguity band of the decision-exact verdicts (FG_DEFAULT_KAPPA, include/faith_gpu.h)
SPECULATE = {"off": 0, "predicted": 1, "verified": 2, "failed": 3}  # FG_SPECULATE_*
DEFAULT_KAPPA = 6e-6
STATUS_NAME = {0: "ok", 1: "invalid_argument", 2: "domain_error", 3: "out_of_range", 4: "runtime_error",
               5: "cuda_error", 6: "out_of_memory"}


class FaithGPUError(RuntimeError):
    code = FG_ERUNTIME


class InvalidArgument(FaithGPUError, ValueError):
    code = FG_EINVAL


class DomainError(FaithGPUError, ArithmeticError):
    code = FG_EDOMAIN


class OutOfRange(FaithGPUError, IndexError):
    code = FG_ERANGE


class CudaError(FaithGPUError):
    code = FG_ECUDA


_EXC = {FG_EINVAL: InvalidArgument, FG_EDOMAIN: DomainError, FG_ERANGE: OutOfRange, FG_ECUDA: CudaError}


class LinearBounds(NamedTuple):
    """faith::LinearBounds (bounds.hpp:34-45): lw/uw [*neurons, d], lb/ub [*neurons]."""
    lw: np.ndarray
    lb: np.ndarray
    uw: np.ndarray
    ub: np.ndarray


class Relaxation(NamedTuple):
    """faith::relax::ElementwiseLinearRelaxation (relax.hpp:15-20)."""
    a_low: np.ndarray
    b_low: np.ndarray
    a_up: np.ndarray
    b_up: np.ndarray


class RunStats(C.Structure):
    _fields_ = [("device_ms", C.c_double), ("pass_ms", C.c_double), ("passes", C.c_int), ("slots", C.c_int),
                ("launches", C.c_uint64), ("sentence_passes", C.c_double), ("exact_probes", C.c_int),
                ("exact_ms", C.c_double), ("band_lo", C.c_double), ("band_hi", C.c_double),
                ("band_samples", C.c_int), ("spec_rollbacks", C.c_int)]


class FgConfig(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("layers", "heads", "embed", "ffn", "length", "classes", "activation")]


_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_lib = None


def exported_symbols() -> list[str]:
    """Function names declared in include/faith_gpu.h."""
    import re
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(fg_[a-z0-9_]+)\s*\(", text)))


def load_library():
    """Loads the in-tree CUDA library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise FileNotFoundError(f"{LIB_PATH} missing: run `python -m paper_2209_12708_b200.build` "
                                "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    sz = C.c_size_t
    L.fg_version.restype = C.c_char_p
    L.fg_last_error.restype = C.c_char_p
    L.fg_last_error.argtypes = [vp]
    L.fg_kernel_launches.restype = C.c_uint64
    L.fg_kernel_launches.argtypes = [vp]
    L.fg_ctx_create.argtypes = [C.c_int, C.POINTER(vp)]
    L.fg_ctx_destroy.argtypes = [vp]
    L.fg_concretize.argtypes = [vp, sz, sz, _dp, _dp, _dp, _dp, C.c_int, C.c_double, _dp, _dp]
    L.fg_check_robust.argtypes = [sz, _dp, _dp, sz, C.c_double, _ip]
    L.fg_affine.argtypes = [vp, sz, sz, sz, sz] + [_dp] * 10
    L.fg_relax.argtypes = [vp, C.c_int, sz] + [_dp] * 6
    L.fg_compose.argtypes = [vp, sz, sz] + [_dp] * 12
    L.fg_elementwise_verify.argtypes = [vp, C.c_int, sz, sz] + [_dp] * 4 + [C.c_int, C.c_double] + [_dp] * 4
    L.fg_dot.argtypes = [vp, C.c_int, sz, sz, sz, sz] + [_dp] * 8 + [C.c_int, C.c_double] + [_dp] * 4
    L.fg_softmax.argtypes = [vp, sz, sz, sz] + [_dp] * 4 + [C.c_int, C.c_double] + [_dp] * 4
    L.fg_add.argtypes = [vp, sz, sz] + [_dp] * 12
    L.fg_scale.argtypes = [vp, sz, sz] + [_dp] * 4 + [C.c_double] + [_dp] * 4
    L.fg_model_create.argtypes = [vp, C.POINTER(FgConfig), _dp, C.POINTER(vp)]
    L.fg_model_destroy.argtypes = [vp]
    L.fg_forward.argtypes = [vp, _dp, _dp]
    L.fg_forward_batch.argtypes = [vp, C.c_int, _dp, _dp]
    L.fg_node_dump_size.restype = sz
    L.fg_node_dump_size.argtypes = [C.POINTER(FgConfig)]
    L.fg_bound_pass.argtypes = [vp, C.c_int, _dp, _ip, C.c_int, C.c_int, _dp, _dp, _dp, _ip]
    L.fg_bound_pass_dump.argtypes = [vp, _dp, _ip, C.c_int, C.c_int, C.c_double, _dp, _dp, _dp, _dp, _ip]
    L.fg_bound_pass_exact.argtypes = [vp, _dp, _ip, C.c_int, C.c_int, C.c_double, _dp, _dp, _dp, _dp, _ip]
    L.fg_model_set_exact_resolve.argtypes = [vp, C.c_double]
    L.fg_model_set_speculation.argtypes = [vp, C.c_int]
    L.fg_certify.argtypes = [vp, C.c_int, _dp, _ip, C.c_int, C.c_int, _dp, C.c_double, _ip, _ip, _ip, _dp, _dp, _ip]
    L.fg_maxeps.argtypes = [vp, C.c_int, _dp, _ip, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, _dp, _ip,
                            _ip, _ip]
    L.fg_last_run_stats.argtypes = [vp, C.POINTER(RunStats)]
    L.fg_param_count.restype = sz
    L.fg_param_count.argtypes = [C.POINTER(FgConfig)]
    L.fg_gen_synthetic.argtypes = [C.POINTER(FgConfig), C.c_uint64, _dp]
    L.fg_gen_input.argtypes = [C.POINTER(FgConfig), C.c_uint64, _dp]
    L.fg_gen_positions.argtypes = [C.c_uint64, C.c_int, C.c_int, _ip]
    L.fg_profile_pass.argtypes = [vp, C.c_int, C.c_double, C.c_int, C.c_char_p, _dp, _ip, _ip]
    L.fg_selftest_affine.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, _dp, _dp, _dp, _dp, _dp]
    L.fg_ctx_set_precision.argtypes = [vp, C.c_int]
    L.fg_selftest_mma_peak.argtypes = [vp, C.c_int, C.c_int, _dp, _dp]
    L.fg_ctx_precision.argtypes = [vp]
    L.fg_dot_batched.argtypes = [vp, C.c_int, sz, sz, sz, sz, sz] + [_dp] * 8 + [C.c_int, C.c_double] + [_dp] * 4
    L.fg_softmax_axis.argtypes = [vp, sz, sz, sz, sz] + [_dp] * 4 + [C.c_int, C.c_double] + [_dp] * 4
    L.fg_sum_axis.argtypes = [vp, sz, sz, sz, sz] + [_dp] * 8
    L.fg_mul_broadcast.argtypes = [vp, sz, sz, sz, sz] + [_dp] * 8 + [C.c_int, C.c_double] + [_dp] * 4
    L.fg_bilinear.argtypes = [vp, sz] + [_dp] * 10
    L.fg_nccl_unique_id.argtypes = [C.c_char_p]
    L.fg_model_shard_nccl.argtypes = [vp, C.c_int, C.c_int, C.c_char_p]
    L.fg_loopback_create.argtypes = [C.c_int, C.POINTER(vp)]
    L.fg_loopback_destroy.argtypes = [vp]
    L.fg_model_shard_loopback.argtypes = [vp, vp, C.c_int]
    L.fg_model_set_column_shard.argtypes = [vp, C.c_int, C.c_int, vp, vp, C.c_int]
    L.fg_maxeps_spec.argtypes = [vp, C.c_int, _dp, _ip, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int,
                                 C.c_int, C.c_int, EXCHANGE_FN, vp, _dp, _ip, _ip, _ip, _ip]
    _lib = L
    return L


def _d(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(_dp)


def _i(a: np.ndarray):
    return a.ctypes.data_as(_ip)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _bounds(b) -> LinearBounds:
    return LinearBounds(*(_f64(t) for t in b))


PRECISION = {"f32": 0, "f64": 1}
# int (*fg_exchange_fn)(void* user, int* verdicts, size_t count): element-wise MAX over ranks, in place
EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_int), C.c_size_t)


class Context:
    """fg_ctx: one CUDA stream on one device (faith_gpu.h).  Raises CudaError without an sm_100 GPU."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        h = C.c_void_p()
        st = self.lib.fg_ctx_create(device, C.byref(h))
        if st != FG_OK:
            raise CudaError(f"fg_ctx_create(device={device}) failed: no usable sm_100 device")
        self.handle = h
        self.device = device

    def close(self):
        if getattr(self, "handle", None):
            self.lib.fg_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def precision(self) -> str:
        return {0: "f32", 1: "f64"}[int(self.lib.fg_ctx_precision(self.handle))]

    def set_precision(self, precision: str):
        """Operator-level arithmetic: "f32" (f32 Λ planes + f64 O(N) state, the fused pass's
        arithmetic) or "f64" (reference operation order, bit-identical arithmetic operators)."""
        self._check(self.lib.fg_ctx_set_precision(self.handle, PRECISION[precision]), "set_precision")

    @property
    def kernel_launches(self) -> int:
        return int(self.lib.fg_kernel_launches(self.handle))

    def _check(self, st: int, what: str):
        if st != FG_OK:
            msg = self.lib.fg_last_error(self.handle).decode()
            raise _EXC.get(st, FaithGPUError)(f"{what}: {msg}")

    def selftest_affine(self, rows: int, c: int, o: int, d: int, seed: int = 1) -> dict:
        """tcgen05 3xTF32 and FP32 SIMT affine GEMMs vs an f64 reference (fg_selftest_affine)."""
        out = [np.zeros(1) for _ in range(4)] + [np.zeros(2)]
        self._check(self.lib.fg_selftest_affine(self.handle, rows, c, o, d, seed, *map(_d, out)),
                    "fg_selftest_affine")
        return {"err_umma": float(out[0][0]), "err_simt": float(out[1][0]), "ms_umma": float(out[2][0]),
                "ms_simt": float(out[3][0]), "bias_umma_centre": float(out[4][0]),
                "bias_umma_radius": float(out[4][1])}

    # ---- bounds.hpp ------------------------------------------------------------------
    def mma_peak(self, kind: str = "tf32", iters: int = 20000) -> dict:
        """fg_selftest_mma_peak: measured dense tcgen05 throughput (kind "tf32" or "bf16")."""
        ms, tf = np.zeros(1), np.zeros(1)
        self._check(self.lib.fg_selftest_mma_peak(self.handle, {"tf32": 0, "bf16": 1}[kind], iters, _d(ms), _d(tf)),
                    "fg_selftest_mma_peak")
        return {"ms": float(ms[0]), "tflops": float(tf[0])}

    def concretize(self, b, norm: str, eps: float):
        """faith::concretize (bounds.cpp:122-140) -> (lo, hi)."""
        b = _bounds(b)
        shape = b.lb.shape
        n = b.lb.size
        d = b.lw.shape[-1] if b.lw.ndim else 0
        lo, hi = np.zeros(n), np.zeros(n)
        self._check(self.lib.fg_concretize(self.handle, n, d, *map(_d, b), NORM[norm], eps, _d(lo), _d(hi)),
                    "concretize")
        return lo.reshape(shape), hi.reshape(shape)

    @staticmethod
    def check_robust(lo, hi, true_class: int, margin: float = 0.0) -> bool:
        """faith::check_robust (bounds.cpp:142-157)."""
        lib = load_library()
        lo, hi = _f64(lo).ravel(), _f64(hi).ravel()
        v = np.zeros(1, dtype=np.int32)
        st = lib.fg_check_robust(lo.size, _d(lo), _d(hi), true_class, margin, _i(v))
        if st != FG_OK:
            raise _EXC.get(st, FaithGPUError)("check_robust")
        return bool(v[0])

    # ---- relax.hpp -------------------------------------------------------------------
    def propagate_affine(self, x, w, bias=None) -> LinearBounds:
        """faith::relax::propagate_affine (relax.cpp:237-307); x neuron shape [..., c]."""
        x = _bounds(x)
        w = _f64(w)
        if w.ndim != 2:
            raise InvalidArgument("propagate_affine: weight must be rank 2")
        c, o = w.shape
        if x.lb.ndim == 0 or x.lb.shape[-1] != c:
            raise InvalidArgument("propagate_affine: inner dimensions do not conform")
        if bias is not None:
            bias = _f64(bias)
            if bias.size != o:
                raise InvalidArgument("propagate_affine: bias length mismatch")
        rows = x.lb.size // c
        d = x.lw.shape[-1]
        oshape = x.lb.shape[:-1] + (o,)
        y = [np.zeros(oshape + (d,)), np.zeros(oshape), np.zeros(oshape + (d,)), np.zeros(oshape)]
        self._check(self.lib.fg_affine(self.handle, rows, c, o, d, *map(_d, x), _d(w), _d(bias), *map(_d, y)),
                    "propagate_affine")
        return LinearBounds(*y)

    def relax(self, kind: str, lo, hi) -> Relaxation:
        """relax_relu / relax_tanh / relax_silu / relax_exp / relax_recip (relax.cpp:313-468)."""
        lo, hi = _f64(lo), _f64(hi)
        shape = lo.shape
        n = lo.size
        out = [np.zeros(n) for _ in range(4)]
        self._check(self.lib.fg_relax(self.handle, RELAX[kind], n, _d(lo.ravel()), _d(hi.ravel()), *map(_d, out)),
                    f"relax_{kind}")
        return Relaxation(*(o.reshape(shape) for o in out))

    def compose_elementwise(self, x, r) -> LinearBounds:
        """faith::relax::compose_elementwise (relax.cpp:470-497)."""
        x = _bounds(x)
        r = [_f64(t) for t in r]
        if r[0].shape != x.lb.shape:
            raise InvalidArgument("compose_elementwise: relaxation shape does not match bounds")
        n, d = x.lb.size, x.lw.shape[-1]
        y = [np.zeros(x.lw.shape), np.zeros(x.lb.shape), np.zeros(x.lw.shape), np.zeros(x.lb.shape)]
        self._check(self.lib.fg_compose(self.handle, n, d, *map(_d, x), *map(_d, r), *map(_d, y)),
                    "compose_elementwise")
        return LinearBounds(*y)

    def elementwise_verify(self, kind: str, x, norm: str, eps: float) -> LinearBounds:
        """concretize -> relax_<kind> -> compose (graph.cpp:484-501), fused."""
        x = _bounds(x)
        n, d = x.lb.size, x.lw.shape[-1]
        y = [np.zeros(x.lw.shape), np.zeros(x.lb.shape), np.zeros(x.lw.shape), np.zeros(x.lb.shape)]
        self._check(self.lib.fg_elementwise_verify(self.handle, RELAX[kind], n, d, *map(_d, x), NORM[norm], eps,
                                                   *map(_d, y)), f"elementwise_verify({kind})")
        return LinearBounds(*y)

    def propagate_dot_product(self, a, b, norm: str, eps: float, layout: str, num_heads: int = 1) -> LinearBounds:
        """faith::relax::propagate_dot_product (relax.cpp:573-654), batch 1.
        similarity: a, b [1, L, E] -> [1, H, L, L]; weighted_values: a [1, H, L, L], b [1, L, E] -> [1, L, E]."""
        a, b = _bounds(a), _bounds(b)
        d = a.lw.shape[-1]
        if b.lw.shape[-1] != d:
            raise InvalidArgument("propagate_dot_product: perturbation dims differ")
        _, length, embed = b.lb.shape
        if layout == "similarity":
            yshape = (1, num_heads, length, length)
        else:
            yshape = (1, length, embed)
        y = [np.zeros(yshape + (d,)), np.zeros(yshape), np.zeros(yshape + (d,)), np.zeros(yshape)]
        self._check(self.lib.fg_dot(self.handle, DOT[layout], length, embed, num_heads, d, *map(_d, a), *map(_d, b),
                                    NORM[norm], eps, *map(_d, y)), "propagate_dot_product")
        return LinearBounds(*y)

    def propagate_softmax(self, x, norm: str, eps: float) -> LinearBounds:
        """faith::relax::propagate_softmax along the last neuron axis (relax.cpp:777-790)."""
        x = _bounds(x)
        n = x.lb.shape[-1]
        rows = x.lb.size // n
        d = x.lw.shape[-1]
        y = [np.zeros(x.lw.shape), np.zeros(x.lb.shape), np.zeros(x.lw.shape), np.zeros(x.lb.shape)]
        self._check(self.lib.fg_softmax(self.handle, rows, n, d, *map(_d, x), NORM[norm], eps, *map(_d, y)),
                    "propagate_softmax")
        return LinearBounds(*y)

    def propagate_dot_product_batched(self, a, b, norm: str, eps: float, layout: str,
                                      num_heads: int = 1) -> LinearBounds:
        """propagate_dot_product with a leading batch axis B (relax.cpp:573-654)."""
        a, b = _bounds(a), _bounds(b)
        d = a.lw.shape[-1]
        if b.lw.shape[-1] != d:
            raise InvalidArgument("propagate_dot_product: perturbation dims differ")
        batch, length, embed = b.lb.shape
        yshape = (batch, num_heads, length, length) if layout == "similarity" else (batch, length, embed)
        y = [np.zeros(yshape + (d,)), np.zeros(yshape), np.zeros(yshape + (d,)), np.zeros(yshape)]
        self._check(self.lib.fg_dot_batched(self.handle, DOT[layout], batch, length, embed, num_heads, d,
                                            *map(_d, a), *map(_d, b), NORM[norm], eps, *map(_d, y)),
                    "propagate_dot_product")
        return LinearBounds(*y)

    @staticmethod
    def _axis_split(shape, axis):
        n = shape[axis]
        inner = int(np.prod(shape[axis + 1:], dtype=np.int64))
        outer = int(np.prod(shape[:axis], dtype=np.int64))
        return outer, n, inner

    def propagate_softmax_axis(self, x, axis: int, norm: str, eps: float) -> LinearBounds:
        """faith::relax::propagate_softmax along `axis` of the neuron shape (relax.cpp:777-790)."""
        x = _bounds(x)
        outer, n, inner = self._axis_split(x.lb.shape, axis)
        d = x.lw.shape[-1]
        y = [np.zeros(x.lw.shape), np.zeros(x.lb.shape), np.zeros(x.lw.shape), np.zeros(x.lb.shape)]
        self._check(self.lib.fg_softmax_axis(self.handle, outer, n, inner, d, *map(_d, x), NORM[norm], eps,
                                             *map(_d, y)), "propagate_softmax")
        return LinearBounds(*y)

    def propagate_sum_axis(self, x, axis: int) -> LinearBounds:
        """faith::relax::propagate_sum_axis (relax.cpp:705-742); the reduced axis keeps extent 1."""
        x = _bounds(x)
        outer, n, inner = self._axis_split(x.lb.shape, axis)
        d = x.lw.shape[-1]
        oshape = x.lb.shape[:axis] + (1,) + x.lb.shape[axis + 1:]
        y = [np.zeros(oshape + (d,)), np.zeros(oshape), np.zeros(oshape + (d,)), np.zeros(oshape)]
        self._check(self.lib.fg_sum_axis(self.handle, outer, n, inner, d, *map(_d, x), *map(_d, y)),
                    "propagate_sum_axis")
        return LinearBounds(*y)

    def propagate_mul_broadcast(self, x, r, axis: int, norm: str, eps: float) -> LinearBounds:
        """faith::relax::propagate_mul_broadcast (relax.cpp:744-775)."""
        x, r = _bounds(x), _bounds(r)
        outer, n, inner = self._axis_split(x.lb.shape, axis)
        if r.lb.ndim != x.lb.ndim or r.lb.shape[axis] != 1:
            raise InvalidArgument("propagate_mul_broadcast: operand shapes incompatible")
        d = x.lw.shape[-1]
        y = [np.zeros(x.lw.shape), np.zeros(x.lb.shape), np.zeros(x.lw.shape), np.zeros(x.lb.shape)]
        self._check(self.lib.fg_mul_broadcast(self.handle, outer, n, inner, d, *map(_d, x), *map(_d, r),
                                              NORM[norm], eps, *map(_d, y)), "propagate_mul_broadcast")
        return LinearBounds(*y)

    def propagate_layernorm(self, x, gamma, beta, norm: str, eps: float, delta: float = 1e-5) -> LinearBounds:
        """EXTENSION (no reference counterpart: the reference model has no LayerNorm,
        proj/include/faith/model.hpp:22-24).  Linear bounds of
        y = (x - mean(x)) / sqrt(var(x) + delta) * gamma + beta over the last axis of x [n, E],
        as a chain of the reference's own bound operators plus the sqrt / square envelopes:
          c = propagate_affine(x, I - 1/E)               (centring: exact, linear)
          s = ElementwiseVerify(square, c)               (convex: tangent below, chord above)
          v = propagate_affine(s, 1/E column, + delta)   (variance + delta)
          r = ElementwiseVerify(sqrt, v)                 (concave: chord below, tangent above)
          q = ElementwiseVerify(recip, r)                (relax.cpp:396-424)
          z = propagate_mul_broadcast(c, q, axis 1)      (McCormick, relax.cpp:744-775)
          y = propagate_affine(z, diag(gamma), beta)
        Sound by construction (every step is); checked by sampling in tests/test_gpu_layernorm.py."""
        x = _bounds(x)
        if x.lb.ndim != 2:
            raise InvalidArgument("propagate_layernorm: x must have neuron shape [n, E]")
        E = x.lb.shape[1]
        gamma, beta = _f64(gamma).ravel(), _f64(beta).ravel()
        if gamma.size != E or beta.size != E or not (delta > 0.0):
            raise InvalidArgument("propagate_layernorm: gamma / beta length or delta")
        c = self.propagate_affine(x, np.eye(E) - 1.0 / E)
        sq = self.elementwise_verify("square", c, norm, eps)
        v = self.propagate_affine(sq, np.full((E, 1), 1.0 / E), np.array([delta]))
        r = self.elementwise_verify("sqrt", v, norm, eps)
        q = self.elementwise_verify("recip", r, norm, eps)
        z = self.propagate_mul_broadcast(c, q, 1, norm, eps)
        return self.propagate_affine(z, np.diag(gamma), beta)

    def relax_bilinear(self, xlo, xhi, ylo, yhi) -> tuple:
        """faith::relax::relax_bilinear (relax.cpp:499-523) -> (lo_x, lo_y, lo_c, up_x, up_y, up_c)."""
        xlo, xhi, ylo, yhi = (_f64(t) for t in (xlo, xhi, ylo, yhi))
        shape, n = xlo.shape, xlo.size
        out = [np.zeros(n) for _ in range(6)]
        self._check(self.lib.fg_bilinear(self.handle, n, _d(xlo.ravel()), _d(xhi.ravel()), _d(ylo.ravel()),
                                         _d(yhi.ravel()), *map(_d, out)), "relax_bilinear")
        return tuple(o.reshape(shape) for o in out)

    def propagate_add(self, a, b) -> LinearBounds:
        a, b = _bounds(a), _bounds(b)
        if a.lb.shape != b.lb.shape or a.lw.shape != b.lw.shape:
            raise InvalidArgument("propagate_add: operand shape mismatch")
        y = [np.zeros(a.lw.shape), np.zeros(a.lb.shape), np.zeros(a.lw.shape), np.zeros(a.lb.shape)]
        self._check(self.lib.fg_add(self.handle, a.lb.size, a.lw.shape[-1], *map(_d, a), *map(_d, b), *map(_d, y)),
                    "propagate_add")
        return LinearBounds(*y)

    def propagate_scale(self, x, s: float) -> LinearBounds:
        x = _bounds(x)
        y = [np.zeros(x.lw.shape), np.zeros(x.lb.shape), np.zeros(x.lw.shape), np.zeros(x.lb.shape)]
        self._check(self.lib.fg_scale(self.handle, x.lb.size, x.lw.shape[-1], *map(_d, x), s, *map(_d, y)),
                    "propagate_scale")
        return LinearBounds(*y)


@dataclass(frozen=True)
class ModelConfig:
    layers: int
    heads: int
    embed: int
    ffn: int
    length: int
    classes: int = 2
    activation: str = "relu"

    def fg(self) -> FgConfig:
        return FgConfig(self.layers, self.heads, self.embed, self.ffn, self.length, self.classes,
                        RELAX[self.activation])


def gen_synthetic(cfg: "ModelConfig", seed: int) -> np.ndarray:
    """model::gen_synthetic weights (model.cpp:99-131) in gen_synthetic order."""
    lib = load_library()
    fc = cfg.fg()
    p = np.zeros(int(lib.fg_param_count(C.byref(fc))))
    if lib.fg_gen_synthetic(C.byref(fc), seed, _d(p)) != FG_OK:
        raise InvalidArgument("gen_synthetic: invalid config")
    return p


def gen_input(cfg: "ModelConfig", seed: int) -> np.ndarray:
    """model::gen_synthetic_input (model.cpp:133-141) -> [L*E]."""
    lib = load_library()
    x = np.zeros(cfg.length * cfg.embed)
    lib.fg_gen_input(C.byref(cfg.fg()), seed, _d(x))
    return x


def gen_positions(seed: int, length: int, words: int) -> np.ndarray:
    lib = load_library()
    p = np.zeros(words, dtype=np.int32)
    if lib.fg_gen_positions(seed, length, words, _i(p)) != FG_OK:
        raise InvalidArgument("gen_positions: words must be in [1, length]")
    return p


def _preload_nccl() -> None:
    """Make the NCCL the library dlopen()s (by soname) the one torch ships (nvidia-nccl wheel):
    loading the system libnccl first would leave a different NCCL version resident, and a later
    `import torch` fails to bind libtorch_cuda against it."""
    global _nccl_preloaded
    if _nccl_preloaded:
        return
    _nccl_preloaded = True
    try:
        import nvidia.nccl as nn
        base = nn.__file__ and os.path.dirname(nn.__file__) or list(nn.__path__)[0]
        path = os.path.join(base, "lib", "libnccl.so.2")
        if os.path.exists(path):
            C.CDLL(path, mode=os.RTLD_NOW | os.RTLD_GLOBAL)
    except (ImportError, OSError):
        pass


_nccl_preloaded = False


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id for fg_model_shard_nccl (create on rank 0, share with all ranks)."""
    _preload_nccl()
    lib = load_library()
    buf = C.create_string_buffer(128)
    if lib.fg_nccl_unique_id(buf) != FG_OK:
        raise CudaError("fg_nccl_unique_id: libnccl.so.2 unavailable")
    return buf.raw


class LoopbackGroup:
    """fg_loopback: `nranks` column-sharded models on ONE device, one host thread per rank."""

    def __init__(self, nranks: int):
        self.lib = load_library()
        h = C.c_void_p()
        if self.lib.fg_loopback_create(nranks, C.byref(h)) != FG_OK:
            raise CudaError("fg_loopback_create failed")
        self.handle, self.nranks = h, nranks

    def close(self):
        if getattr(self, "handle", None):
            self.lib.fg_loopback_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Model:
    """fg_model: weights resident in HBM; batched bound passes, certify and max-epsilon."""

    def shard_columns_nccl(self, rank: int, nranks: int, uid: bytes):
        """Column-shard the perturbation dimension over `nranks` GPUs; partial norms all-reduced
        with NCCL.  Every rank must then call the same passes."""
        _preload_nccl()
        self.ctx._check(self.lib.fg_model_shard_nccl(self.handle, rank, nranks, uid), "fg_model_shard_nccl")

    def shard_columns_loopback(self, group: LoopbackGroup, rank: int):
        """Column-shard over a LoopbackGroup (virtual ranks on one device, one thread each)."""
        self._loop = group  # keep the group alive as long as the model
        self.ctx._check(self.lib.fg_model_shard_loopback(self.handle, group.handle, rank), "fg_model_shard_loopback")

    def __init__(self, ctx: Context, cfg: ModelConfig, params: np.ndarray):
        self.ctx, self.cfg, self.lib = ctx, cfg, ctx.lib
        self.params = _f64(params)
        h = C.c_void_p()
        ctx._check(self.lib.fg_model_create(ctx.handle, C.byref(cfg.fg()), _d(self.params), C.byref(h)),
                   "fg_model_create")
        self.handle = h

    @classmethod
    def from_file(cls, ctx: Context, manifest: str, strict: bool = True) -> "Model":
        """A faith-model/v1 manifest (model::load_model, model.cpp:287-335) straight to the device."""
        from .formats import load_model
        cfg, params = load_model(manifest, strict=strict)
        return cls(ctx, cfg, params)

    def close(self):
        if getattr(self, "handle", None):
            self.lib.fg_model_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def forward(self, x) -> np.ndarray:
        out = np.zeros(self.cfg.classes)
        x = _f64(x)
        self.ctx._check(self.lib.fg_forward(self.handle, _d(x), _d(out)), "forward")
        return out

    def _inputs(self, x, positions):
        x = _f64(x).reshape(-1, self.cfg.length * self.cfg.embed)
        pos = np.ascontiguousarray(positions, dtype=np.int32)
        if pos.ndim == 1:
            pos = pos[None, :]
        if pos.shape[0] != x.shape[0]:
            raise InvalidArgument("positions / inputs batch mismatch")
        return x, pos

    def forward_batch(self, xs) -> np.ndarray:
        """fg_forward_batch: exact f64 forward of N inputs [N, L*E] on the GPU -> logits [N, C]."""
        xs = _f64(xs).reshape(-1, self.cfg.length * self.cfg.embed)
        out = np.zeros((xs.shape[0], self.cfg.classes))
        self.ctx._check(self.lib.fg_forward_batch(self.handle, xs.shape[0], _d(xs), _d(out)), "fg_forward_batch")
        return out

    def bound_pass(self, x, positions, norm: str, eps):
        """fg_bound_pass -> (logits_lo [S,C], logits_hi [S,C], status [S])."""
        x, pos = self._inputs(x, positions)
        S = x.shape[0]
        eps = np.broadcast_to(_f64(eps), (S,)).copy()
        lo, hi = np.zeros((S, self.cfg.classes)), np.zeros((S, self.cfg.classes))
        st = np.zeros(S, dtype=np.int32)
        self.ctx._check(self.lib.fg_bound_pass(self.handle, S, _d(x), _i(pos), pos.shape[1], NORM[norm], _d(eps),
                                               _d(lo), _d(hi), _i(st)), "fg_bound_pass")
        return lo, hi, st

    def bound_pass_dump(self, x, positions, norm: str, eps: float):
        """Single sentence; returns (status, logits_lo, logits_hi, node_lo, node_hi) in oracle node order."""
        x, pos = self._inputs(x, positions)
        n = int(self.lib.fg_node_dump_size(C.byref(self.cfg.fg())))
        nlo, nhi = np.zeros(n), np.zeros(n)
        lo, hi = np.zeros(self.cfg.classes), np.zeros(self.cfg.classes)
        st = np.zeros(1, dtype=np.int32)
        self.ctx._check(self.lib.fg_bound_pass_dump(self.handle, _d(x[0]), _i(pos[0]), pos.shape[1], NORM[norm],
                                                    eps, _d(lo), _d(hi), _d(nlo), _d(nhi), _i(st)),
                        "fg_bound_pass_dump")
        return int(st[0]), lo, hi, nlo, nhi

    def bound_pass_exact(self, x, positions, norm: str, eps: float, dump: bool = False):
        """fg_bound_pass_exact: one sentence in the exact (reference-order f64) mode on the device
        -> (status, logits_lo, logits_hi, node_lo, node_hi); node arrays None unless dump."""
        x, pos = self._inputs(x, positions)
        nlo = nhi = None
        if dump:
            n = int(self.lib.fg_node_dump_size(C.byref(self.cfg.fg())))
            nlo, nhi = np.zeros(n), np.zeros(n)
        lo, hi = np.zeros(self.cfg.classes), np.zeros(self.cfg.classes)
        st = np.zeros(1, dtype=np.int32)
        self.ctx._check(self.lib.fg_bound_pass_exact(self.handle, _d(x[0]), _i(pos[0]), pos.shape[1], NORM[norm],
                                                     eps, _d(lo), _d(hi), _d(nlo), _d(nhi), _i(st)),
                        "fg_bound_pass_exact")
        return int(st[0]), lo, hi, nlo, nhi

    def set_exact_resolve(self, kappa: float):
        """Ambiguity band of the decision-exact verdicts (include/faith_gpu.h); 0 = raw f32 verdicts."""
        self.ctx._check(self.lib.fg_model_set_exact_resolve(self.handle, float(kappa)), "fg_model_set_exact_resolve")

    def set_speculation(self, mode: str):
        """fg_maxeps while a re-decision runs: "predicted" (default), "verified", "failed", "off"
        (include/faith_gpu.h fg_model_set_speculation)."""
        code = SPECULATE[mode]
        self.ctx._check(self.lib.fg_model_set_speculation(self.handle, code), "fg_model_set_speculation")

    def certify(self, x, positions, norm: str, eps, margin: float = 0.0):
        """cmd_verify semantics per sentence -> dict of arrays."""
        x, pos = self._inputs(x, positions)
        S = x.shape[0]
        eps = np.broadcast_to(_f64(eps), (S,)).copy()
        ver, bnd, pred, st = (np.zeros(S, dtype=np.int32) for _ in range(4))
        lo, hi = np.zeros((S, self.cfg.classes)), np.zeros((S, self.cfg.classes))
        self.ctx._check(self.lib.fg_certify(self.handle, S, _d(x), _i(pos), pos.shape[1], NORM[norm], _d(eps), margin,
                                            _i(ver), _i(bnd), _i(pred), _d(lo), _d(hi), _i(st)), "fg_certify")
        return {"verified": ver.astype(bool), "bounded": bnd.astype(bool), "predicted": pred, "lo": lo, "hi": hi,
                "status": st}

    def maxeps(self, x, positions, norm: str, eps_max: float = 1.0, tol: float = 1e-3, slots: int = 0):
        """cmd_maxeps semantics per sentence -> dict(eps, calls, predicted, status)."""
        x, pos = self._inputs(x, positions)
        S = x.shape[0]
        eps = np.zeros(S)
        calls, pred, st = (np.zeros(S, dtype=np.int32) for _ in range(3))
        self.ctx._check(self.lib.fg_maxeps(self.handle, S, _d(x), _i(pos), pos.shape[1], NORM[norm], eps_max, tol,
                                           slots, _d(eps), _i(calls), _i(pred), _i(st)), "fg_maxeps")
        return {"eps": eps, "calls": calls, "predicted": pred, "status": st}

    def maxeps_speculative(self, x, positions, norm: str, eps_max: float = 1.0, tol: float = 1e-3, depth: int = 3,
                           dist=None):
        """fg_maxeps_spec: cmd_maxeps's decision path, `depth` bisection levels per batched round.
        With a torch.distributed group `dist`, the probes of each round are split across ranks and
        the verdicts combined with an all-reduce(MAX) -> dict(eps, calls, rounds, predicted, status)."""
        x, pos = self._inputs(x, positions)
        S = x.shape[0]
        eps = np.zeros(S)
        calls, pred, st = (np.zeros(S, dtype=np.int32) for _ in range(3))
        rounds = np.zeros(1, dtype=np.int32)
        rank, world, cb = 0, 1, EXCHANGE_FN()
        if dist is not None and dist.get_world_size() > 1:
            import torch
            rank, world = dist.get_rank(), dist.get_world_size()

            def _exchange(user, buf, count):
                t = torch.from_numpy(np.ctypeslib.as_array(buf, shape=(count,)).copy())
                if dist.get_backend() == "nccl":
                    t = t.cuda()
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                np.ctypeslib.as_array(buf, shape=(count,))[:] = t.cpu().numpy()
                return 0

            cb = EXCHANGE_FN(_exchange)
        self._spec_cb = cb  # keep the callback alive during the call
        self.ctx._check(self.lib.fg_maxeps_spec(self.handle, S, _d(x), _i(pos), pos.shape[1], NORM[norm], eps_max,
                                                tol, depth, rank, world, cb, None, _d(eps), _i(calls), _i(rounds),
                                                _i(pred), _i(st)), "fg_maxeps_spec")
        return {"eps": eps, "calls": calls, "rounds": int(rounds[0]), "predicted": pred, "status": st}

    def profile_pass(self, norm: str, eps: float) -> dict:
        """One eager pass with CUDA events around every launch site -> {site: (ms, kernels)}."""
        names = C.create_string_buffer(32 * 64)
        ms = np.zeros(64)
        kern = np.zeros(64, dtype=np.int32)
        n = np.zeros(1, dtype=np.int32)
        self.ctx._check(self.lib.fg_profile_pass(self.handle, NORM[norm], eps, 64, names, _d(ms), _i(kern), _i(n)),
                        "fg_profile_pass")
        raw = names.raw
        out = {}
        for i in range(int(n[0])):
            tag = raw[32 * i:32 * (i + 1)].split(b"\0", 1)[0].decode()
            out[tag] = (float(ms[i]), int(kern[i]))
        return out

    def last_stats(self) -> dict:
        s = RunStats()
        self.lib.fg_last_run_stats(self.handle, C.byref(s))
        return {f: getattr(s, f) for f, _ in RunStats._fields_}
