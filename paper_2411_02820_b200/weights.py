"""Model weights in HBM, in the layout the sm_100a kernels consume.

Reference weights (model.py:287-334) are float32 [in, out] matrices applied
as ``x @ W``.  On device each projection is stored once, transposed to
K-major [out, in] bf16 (the B operand of the tcgen05 GEMM and the row-major
operand of the anchor GEMV); Q/K/V are concatenated into one [(H+2KVH)*D, d]
matrix so a single GEMM produces q, k and v.  Gains stay f32.  RoPE cos/sin
tables are precomputed exactly as the reference does (angles in float64,
cast to float32, model.py:475-479).
"""

from __future__ import annotations

import ctypes as C
import hashlib
import json
import math
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np
import torch

from . import _lib as L
from .config import ModelConfig, PerturbationSpec

_SLOTS = ("wq", "wk", "wv", "wo", "w1", "w2", "g_attn", "g_mlp")  # RNG stream order, model.py:248


def model_ident(config: ModelConfig, pert: PerturbationSpec | None) -> str:
    """Stable model id used as the store key (model.py:273-284)."""
    payload = {
        "config": [config.n_layers, config.d_model, config.n_heads, config.n_kv_heads, config.head_dim,
                   config.d_ff, config.vocab_size, config.base_seed],
        "eps": list(pert.eps) if pert else None,
        "noise_seed": pert.noise_seed if pert else None,
    }
    digest = hashlib.blake2b(json.dumps(payload, sort_keys=True).encode(), digest_size=6).hexdigest()
    kind = "base" if pert is None or not any(pert.eps) else "var"
    return f"m{config.base_seed:x}-{kind}-{digest}"


def _stream_normal(seed: int, tags: Sequence[int], shape, std: float) -> np.ndarray:
    return (np.random.default_rng([seed, *tags]).standard_normal(shape, dtype=np.float64) * std).astype(np.float32)


def reference_weights(config: ModelConfig, perturbation: PerturbationSpec | None = None) -> dict:
    """The reference's seeded float32 weights (host numpy), bit-identical streams.

    embed tags (0,0) std 1; unembed (0,1) std 1/sqrt(d); layer tensors
    (1,l,slot) std 1/sqrt(d) (w2: 1/sqrt(d_ff)); gains ones; a variant adds
    eps[l]*rms(w)*N(0,1) from tags (noise_seed,2,l,slot) (model.py:300-320).
    """
    if perturbation is not None and len(perturbation.eps) != config.n_layers:
        raise ValueError(f"perturbation has {len(perturbation.eps)} entries for {config.n_layers} layers")
    d, f = config.d_model, config.d_ff
    qd, kvd = config.n_heads * config.head_dim, config.n_kv_heads * config.head_dim
    shapes = {"wq": (d, qd), "wk": (d, kvd), "wv": (d, kvd), "wo": (qd, d), "w1": (d, f), "w2": (f, d)}
    out = {
        "embed": _stream_normal(config.base_seed, (0, 0), (config.vocab_size, d), 1.0),
        "unembed": _stream_normal(config.base_seed, (0, 1), (d, config.vocab_size), 1.0 / math.sqrt(d)),
        "g_final": np.ones(d, np.float32),
        "layers": [],
    }
    for l in range(config.n_layers):
        eps = perturbation.eps[l] if perturbation is not None else 0.0
        lw = {}
        for slot, name in enumerate(_SLOTS):
            if name.startswith("g_"):
                w = np.ones(d, np.float32)
            else:
                std = 1.0 / math.sqrt(f) if name == "w2" else 1.0 / math.sqrt(d)
                w = _stream_normal(config.base_seed, (1, l, slot), shapes[name], std)
            if eps > 0.0:
                rms = float(np.sqrt(np.mean(np.square(w, dtype=np.float64))))
                noise = np.random.default_rng([perturbation.noise_seed, 2, l, slot]).standard_normal(
                    w.shape, dtype=np.float64) * (eps * rms)
                w = (w + noise.astype(np.float32)).astype(np.float32)
            lw[name] = w
        out["layers"].append(lw)
    return out


def rope_tables(head_dim: int, max_seq: int) -> tuple[np.ndarray, np.ndarray]:
    half = head_dim // 2
    inv = 10000.0 ** (-np.arange(half, dtype=np.float64) * 2.0 / head_dim)
    ang = np.arange(max_seq, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)


@dataclass(eq=False)
class ModelWeights:
    """Device-resident weights + the ds_model descriptor the C ABI takes."""

    config: ModelConfig
    ident: str
    embed: torch.Tensor        # bf16 [V, d]
    unembed_t: torch.Tensor    # bf16 [V, d]
    g_final: torch.Tensor      # f32 [d]
    rope_cos: torch.Tensor     # f32 [max_seq, D/2]
    rope_sin: torch.Tensor
    layers: list = field(default_factory=list)  # dicts: wqkv, wo, w1, w2 (bf16 K-major), g_attn, g_mlp (f32)
    _desc: object = None
    _layer_arr: object = None

    @property
    def device(self) -> torch.device:
        return self.embed.device

    def desc(self) -> L.Model:
        if self._desc is None:
            cfg = self.config
            arr = (L.LayerWeights * cfg.n_layers)()
            for i, lw in enumerate(self.layers):
                arr[i] = L.LayerWeights(lw["wqkv"].data_ptr(), lw["wo"].data_ptr(), lw["w1"].data_ptr(),
                                        lw["w2"].data_ptr(), lw["g_attn"].data_ptr(), lw["g_mlp"].data_ptr())
            dims = L.Dims(cfg.n_layers, cfg.d_model, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.d_ff,
                          cfg.vocab_size, cfg.max_seq, L.MLP_KINDS[cfg.mlp_kind])
            self._layer_arr = arr
            self._desc = L.Model(dims, self.embed.data_ptr(), self.unembed_t.data_ptr(), self.g_final.data_ptr(),
                                 self.rope_cos.data_ptr(), self.rope_sin.data_ptr(),
                                 C.cast(arr, C.POINTER(L.LayerWeights)))
        return self._desc


def _bf16(x: np.ndarray, device) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(x)).to(device=device).to(torch.bfloat16)


def from_host(config: ModelConfig, host: dict, ident: str, device="cuda") -> ModelWeights:
    """Upload reference-layout float32 weights as the device layout (the
    reference block is ungated; a SwiGLU host dict carries "wg"/"wu" per layer
    and is interleaved here in blocks of 16 rows)."""
    cos, sin = rope_tables(config.head_dim, config.max_seq)
    layers = []
    for lw in host["layers"]:
        wqkv = np.concatenate([lw["wq"], lw["wk"], lw["wv"]], axis=1).T
        if config.mlp_kind == "swiglu":
            w1 = interleave_gate_up(lw["wg"].T, lw["wu"].T)
        else:
            w1 = lw["w1"].T
        layers.append({
            "wqkv": _bf16(wqkv, device), "wo": _bf16(lw["wo"].T, device),
            "w1": _bf16(w1, device), "w2": _bf16(lw["w2"].T, device),
            "g_attn": torch.from_numpy(lw["g_attn"]).to(device), "g_mlp": torch.from_numpy(lw["g_mlp"]).to(device),
        })
    return ModelWeights(
        config=config, ident=ident, embed=_bf16(host["embed"], device), unembed_t=_bf16(host["unembed"].T, device),
        g_final=torch.from_numpy(host["g_final"]).to(device), rope_cos=torch.from_numpy(cos).to(device),
        rope_sin=torch.from_numpy(sin).to(device), layers=layers)


def interleave_gate_up(wg_t: np.ndarray, wu_t: np.ndarray) -> np.ndarray:
    """[d_ff][d] gate and up (K-major) -> [2*d_ff][d] with rows 32b..32b+15 =
    gate rows 16b..16b+15 and rows 32b+16..32b+31 = the matching up rows."""
    f, d = wg_t.shape
    if f % 16:
        raise ValueError("d_ff must be a multiple of 16 for SwiGLU")
    return np.stack([wg_t.reshape(f // 16, 16, d), wu_t.reshape(f // 16, 16, d)], axis=1).reshape(2 * f, d)


def build_model(config: ModelConfig, perturbation: PerturbationSpec | None = None, device="cuda") -> ModelWeights:
    """build_model (model.py:287-334): the reference's seeded weights, on device."""
    return from_host(config, reference_weights(config, perturbation), model_ident(config, perturbation), device)


def random_model(config: ModelConfig, seed: int, device="cuda", base: ModelWeights | None = None,
                 perturb_layers: Sequence[int] = (), eps: float = 0.5) -> ModelWeights:
    """Same-architecture random weights generated on the GPU (benchmarks).

    With ``base``, returns the variant B = A + eps*rms*N(0,1) on
    ``perturb_layers`` (PerturbationSpec.block semantics); unperturbed layers
    and the embeddings are shared with ``base`` (bitwise equal, no copy).
    """
    g = torch.Generator(device=device).manual_seed(seed)
    d, f = config.d_model, config.d_ff
    f1 = 2 * f if config.mlp_kind == "swiglu" else f  # SwiGLU: interleaved gate/up rows (ds_dims)
    qkv = (config.n_heads + 2 * config.n_kv_heads) * config.head_dim

    def randn(*shape, std):
        return (torch.randn(*shape, device=device, generator=g) * std).to(torch.bfloat16)

    if base is None:
        cos, sin = rope_tables(config.head_dim, config.max_seq)
        embed = randn(config.vocab_size, d, std=1.0)
        unembed_t = randn(config.vocab_size, d, std=1.0 / math.sqrt(d))
        layers = []
        for _ in range(config.n_layers):
            layers.append({
                "wqkv": randn(qkv, d, std=1 / math.sqrt(d)), "wo": randn(d, config.n_heads * config.head_dim,
                                                                          std=1 / math.sqrt(d)),
                "w1": randn(f1, d, std=1 / math.sqrt(d)), "w2": randn(d, f, std=1 / math.sqrt(f)),
                "g_attn": torch.ones(d, device=device), "g_mlp": torch.ones(d, device=device),
            })
        return ModelWeights(config, f"rand{seed}", embed, unembed_t, torch.ones(d, device=device),
                            torch.from_numpy(cos).to(device), torch.from_numpy(sin).to(device), layers)
    layers = []
    chosen = set(perturb_layers)
    for l, lw in enumerate(base.layers):
        if l not in chosen:
            layers.append(lw)
            continue
        nl = {}
        for k, w in lw.items():
            wf = w.float()
            rms = wf.pow(2).mean().sqrt()
            nl[k] = (wf + torch.randn(wf.shape, device=device, generator=g) * (eps * rms)).to(w.dtype)
        layers.append(nl)
    return ModelWeights(config, f"{base.ident}-var{seed}", base.embed, base.unembed_t, base.g_final, base.rope_cos,
                        base.rope_sin, layers)
