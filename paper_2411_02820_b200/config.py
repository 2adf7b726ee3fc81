"""Configuration types of the reuse API, same names/semantics as crosskv.model.

ModelConfig       model.py:70-124
PerturbationSpec  model.py:127-152
RecomputeConfig   model.py:155-211 (normal form: sorted, touching/overlapping
                  ranges merged, inclusive; empty = full reuse)
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, Sequence


@dataclass(frozen=True)
class ModelConfig:
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    d_ff: int
    vocab_size: int
    max_seq: int
    base_seed: int
    # "ungated" = the reference block (model.py:532-533); "swiglu" = the Llama-3
    # MLP (a B200-path extension: the second row of config 2)
    mlp_kind: str = "ungated"

    def __post_init__(self) -> None:
        if self.mlp_kind not in ("ungated", "swiglu"):
            raise ValueError(f"unknown mlp_kind {self.mlp_kind!r}")
        for name in ("n_layers", "d_model", "n_heads", "n_kv_heads", "head_dim", "d_ff", "vocab_size"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be positive, got {getattr(self, name)}")
        if self.d_model != self.n_heads * self.head_dim:
            raise ValueError(f"d_model ({self.d_model}) must equal n_heads*head_dim "
                             f"({self.n_heads}*{self.head_dim})")
        if self.n_heads % self.n_kv_heads:
            raise ValueError(f"n_kv_heads ({self.n_kv_heads}) must divide n_heads ({self.n_heads})")
        if self.max_seq < 2:
            raise ValueError("max_seq must be at least 2")
        if self.base_seed < 0:
            raise ValueError("base_seed must be a non-negative 64-bit integer")

    # Reference byte laws (float32 storage, model.py:116-124).
    @property
    def kv_bytes_per_position(self) -> int:
        return 2 * self.n_kv_heads * self.head_dim * 4

    @property
    def e_bytes_per_position(self) -> int:
        return self.d_model * 4

    # What this build stores: K/V in bf16 (half the reference's bytes), E in
    # f32 like the reference (the recompute resumes the residual stream exactly).
    @property
    def kv_bytes_per_position_bf16(self) -> int:
        return 2 * self.n_kv_heads * self.head_dim * 2

    @property
    def e_bytes_per_position_stored(self) -> int:
        return self.d_model * 4


@dataclass(frozen=True)
class PerturbationSpec:
    eps: tuple[float, ...]
    noise_seed: int

    def __init__(self, eps: Sequence[float], noise_seed: int):
        object.__setattr__(self, "eps", tuple(float(e) for e in eps))
        object.__setattr__(self, "noise_seed", int(noise_seed))
        if any(e < 0 for e in self.eps):
            raise ValueError("perturbation magnitudes must be non-negative")
        if self.noise_seed < 0:
            raise ValueError("noise_seed must be a non-negative 64-bit integer")

    @classmethod
    def block(cls, n_layers: int, layers: Iterable[int], eps: float, noise_seed: int) -> "PerturbationSpec":
        chosen = set(layers)
        return cls([eps if l in chosen else 0.0 for l in range(n_layers)], noise_seed)


@dataclass(frozen=True)
class RecomputeConfig:
    """Disjoint, sorted, inclusive layer ranges to recompute; () = full reuse."""

    groups: tuple[tuple[int, int], ...]

    def __init__(self, groups: Iterable[Sequence[int]] = ()):
        spans = sorted((int(a), int(b)) for a, b in groups)
        merged: list[tuple[int, int]] = []
        for a, b in spans:
            if a > b:
                raise ValueError(f"range [{a},{b}] is reversed")
            if a < 0:
                raise ValueError(f"range [{a},{b}] has a negative start")
            if merged and a <= merged[-1][1] + 1:   # touching or overlapping: merge
                merged[-1] = (merged[-1][0], max(merged[-1][1], b))
            else:
                merged.append((a, b))
        object.__setattr__(self, "groups", tuple(merged))

    @classmethod
    def full(cls, n_layers: int) -> "RecomputeConfig":
        return cls([(0, n_layers - 1)])

    @classmethod
    def none(cls) -> "RecomputeConfig":
        return cls()

    @property
    def recomputed_layer_count(self) -> int:
        return sum(b - a + 1 for a, b in self.groups)

    @property
    def transition_layers(self) -> tuple[int, ...]:
        """Group starts above layer 0: the layers whose E cache is needed."""
        return tuple(a for a, _ in self.groups if a > 0)

    def layer_set(self) -> frozenset[int]:
        return frozenset(l for a, b in self.groups for l in range(a, b + 1))

    def reused_layers(self, n_layers: int) -> tuple[int, ...]:
        cov = self.layer_set()
        return tuple(l for l in range(n_layers) if l not in cov)

    def validate_for(self, n_layers: int) -> None:
        if self.groups and self.groups[-1][1] > n_layers - 1:
            raise ValueError(f"config {self.groups} exceeds layer range [0,{n_layers - 1}]")

    def is_full(self, n_layers: int) -> bool:
        return self.groups == ((0, n_layers - 1),)
