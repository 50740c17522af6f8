"""The five BASELINE.json workloads.

Synthetic model: ``gen_synthetic(seed=1000+k)`` for config ck (proj/src/model.cpp:99-131,
weights U(±0.5/sqrt(fan_in)) rounded to f32).  Sentence s: ``gen_synthetic_input(2000+s)``
(model.cpp:133-141) with W perturbed words at distinct positions drawn from
``Rng(3000+s).uniform_index(L)`` (sorted); Λ0 columns are ordered (word, embedding index),
so D = W*E.  ε search follows ``cmd_maxeps`` (proj/src/cli.cpp:135-193) with
eps_max=1.0 and tol=1e-6 (22 bound passes per sentence unless eps_max verifies).
"""
from __future__ import annotations

from dataclasses import dataclass, field


@dataclass(frozen=True)
class Workload:
    name: str
    layers: int
    heads: int
    embed: int
    ffn: int
    length: int
    words: int
    norm: str  # "l1" | "l2" | "linf"
    eps: float  # fixed-ε pass timing
    sentences: int
    classes: int = 2
    activation: str = "relu"
    eps_max: float = 1.0
    tol: float = 1e-6
    description: str = field(default="", compare=False)

    @property
    def model_seed(self) -> int:
        return 1000 + int("".join(ch for ch in self.name[1:] if ch.isdigit()))

    @property
    def pert_dim(self) -> int:
        return self.words * self.embed

    @staticmethod
    def input_seed(s: int) -> int:
        return 2000 + s

    @staticmethod
    def position_seed(s: int) -> int:
        return 3000 + s

    def as_dict(self) -> dict:
        return {
            "workload": self.name, "layers": self.layers, "heads": self.heads, "embed": self.embed,
            "ffn": self.ffn, "seq_len": self.length, "words": self.words, "norm": self.norm,
            "pert_dim": self.pert_dim, "classes": self.classes, "activation": self.activation,
            "eps_max": self.eps_max, "tol": self.tol,
        }


CONFIGS = {
    "c1": Workload("c1", 1, 4, 64, 128, 32, 1, "linf", 0.01, 1,
                   description="1-layer d=64 4 heads ffn=128, seq 32, one word linf, single sentence"),
    "c2": Workload("c2", 2, 4, 128, 256, 64, 1, "l2", 0.01, 256,
                   description="2-layer d=128 ffn=256, seq 64, one word l2, batch of 256 sentences"),
    "c3": Workload("c3", 3, 4, 256, 512, 64, 2, "l1", 0.01, 64,
                   description="3-layer d=256 ffn=512, seq 64, two words l1, eps binary search"),
    "c4": Workload("c4", 6, 8, 512, 2048, 128, 1, "linf", 0.001, 4096,
                   description="6-layer d=512 8 heads ffn=2048, seq 128, one word linf, 4096 sentences"),
    "c5": Workload("c5", 12, 12, 768, 3072, 128, 2, "l2", 0.001, 8,
                   description="12-layer BERT-base-shaped d=768 12 heads ffn=3072, seq 128, two words l2"),
}


# Shape-coverage workloads for the parity tests (not benchmarks): the c4/c5 structure (8 heads,
# 128 tokens) at sizes the reference itself evaluates in minutes on one core, so their golden
# vectors come from the unmodified reference build (oracle/make_golden.py).
SHAPE_CHECKS = {
    "c4m": Workload("c4m", 2, 8, 256, 512, 128, 1, "linf", 1e-4, 1,
                    description="c4-shaped mini: 2 layers d=256 8 heads ffn=512, seq 128, one word linf"),
    # c5-shaped slice: the BERT-base layer (E 768, 12 heads, F 3072, 128 tokens, two words l2,
    # D = 1536) at 2 layers, which the reference walks in about two hours on one core.
    "c5s": Workload("c5s", 2, 12, 768, 3072, 128, 2, "l2", 1e-5, 1,
                    description="c5-shaped slice: 2 layers d=768 12 heads ffn=3072, seq 128, two words l2"),
}
ALL = {**CONFIGS, **SHAPE_CHECKS}
