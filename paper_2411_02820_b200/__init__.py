"""DroidSpeak cross-model prefill, B200-native (sm_100a kernels behind a C ABI).

Drop-in for the reuse path of the reference package ``crosskv``: the same
public names for the producer KV / hidden-state (E) export, the per-pair
recompute-layer set, and the consumer partial prefill.
"""

from .config import ModelConfig, PerturbationSpec, RecomputeConfig
from .engine import (
    CapturedPartialPrefill,
    CapturedPartialPrefillBatch,
    ECache,
    LayerKV,
    MixedPrefill,
    PagedKV,
    PrefillResult,
    check_tokens,
    full_prefill,
    make_synthetic_dataset,
    partial_prefill,
    partial_prefill_batch,
    token_selective_prefill,
    workspace_bytes,
)
from .planner import AdaptDecision, CostModel, ScheduledRequest, SloPolicy, adapt_config, estimate_ttft, plan
from .selection import (build_frontier, enumerate_groups, load_profile, save_profile, select_by_layer_budget,
                        select_by_quality_floor)
from .store import CacheKey, CacheStore, FetchedKV, KVSlice, context_hash, fetch_context_caches, store_prefill
from .errors import CacheMissError, CapacityError, DegenerateInputError, SchemaError
from .weights import ModelWeights, build_model, model_ident, random_model, reference_weights

__version__ = "0.1.0"

__all__ = [
    "CapturedPartialPrefill", "CapturedPartialPrefillBatch", "CacheMissError", "CapacityError", "DegenerateInputError", "ECache", "LayerKV", "MixedPrefill",
    "ModelConfig", "ModelWeights", "PagedKV", "PerturbationSpec", "PrefillResult", "RecomputeConfig",
    "SchemaError", "build_model", "check_tokens", "full_prefill", "make_synthetic_dataset", "model_ident",
    "partial_prefill", "partial_prefill_batch", "random_model", "token_selective_prefill", "reference_weights", "workspace_bytes",
    "AdaptDecision", "CostModel", "ScheduledRequest", "SloPolicy", "adapt_config", "estimate_ttft", "plan", "build_frontier", "enumerate_groups", "load_profile",
    "save_profile", "select_by_layer_budget", "select_by_quality_floor", "CacheKey", "CacheStore", "FetchedKV",
    "KVSlice", "context_hash", "fetch_context_caches", "store_prefill",
]
