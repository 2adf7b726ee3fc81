"""DroidSpeak cross-model prefill, B200-native (sm_100a kernels behind a C ABI).

Drop-in for the reuse path of the reference package ``crosskv``: the same
public names for the producer KV / hidden-state (E) export, the per-pair
recompute-layer set, and the consumer partial prefill.
"""

from .config import ModelConfig, PerturbationSpec, RecomputeConfig
from .engine import (
    ECache,
    LayerKV,
    MixedPrefill,
    PagedKV,
    PrefillResult,
    check_tokens,
    full_prefill,
    make_synthetic_dataset,
    partial_prefill,
    workspace_bytes,
)
from .errors import CacheMissError, CapacityError, DegenerateInputError, SchemaError
from .weights import ModelWeights, build_model, model_ident, random_model, reference_weights

__version__ = "0.1.0"

__all__ = [
    "CacheMissError", "CapacityError", "DegenerateInputError", "ECache", "LayerKV", "MixedPrefill",
    "ModelConfig", "ModelWeights", "PagedKV", "PerturbationSpec", "PrefillResult", "RecomputeConfig",
    "SchemaError", "build_model", "check_tokens", "full_prefill", "make_synthetic_dataset", "model_ident",
    "partial_prefill", "random_model", "reference_weights", "workspace_bytes",
]
