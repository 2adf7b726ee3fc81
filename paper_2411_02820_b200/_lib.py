"""ctypes binding of the C ABI (include/droidspeak.h).

The library is the product path: if it is missing or fails to load, every
entry point raises — there is no CPU or eager-PyTorch fallback.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import CacheMissError, DegenerateInputError

# DS_LIB: another build of the same library (same-box A/B measurements of kernel variants)
LIB_PATH = Path(os.environ.get("DS_LIB") or Path(__file__).resolve().parent / "libdroidspeak.so")

DS_OK, DS_ERR_INVALID, DS_ERR_CACHE_MISS, DS_ERR_DEGENERATE, DS_ERR_CUDA = range(5)
MISS_KIND = {1: "kv", 2: "e"}

# epilogue modes of ds_gemm
EPI_STORE_BF16, EPI_RESID_F32, EPI_SILU_BF16, EPI_QKV_ROPE, EPI_STORE_F32, EPI_SWIGLU_BF16 = range(6)
MLP_KINDS = {"ungated": 0, "swiglu": 1}
ABI_VERSION = 2  # include/droidspeak.h DS_ABI_VERSION
ANCHOR_SHAPES = {"auto": 0, "persistent": 1, "launch": 2}


class Dims(C.Structure):
    _fields_ = [(n, C.c_int32) for n in
                ("n_layers", "d_model", "n_heads", "n_kv_heads", "head_dim", "d_ff", "vocab_size", "max_seq",
                 "mlp_kind")]


class LayerWeights(C.Structure):
    _fields_ = [("wqkv", C.c_void_p), ("wo", C.c_void_p), ("w1", C.c_void_p), ("w2", C.c_void_p),
                ("g_attn", C.c_void_p), ("g_mlp", C.c_void_p)]


class Model(C.Structure):
    _fields_ = [("dims", Dims), ("embed", C.c_void_p), ("unembed", C.c_void_p), ("g_final", C.c_void_p),
                ("rope_cos", C.c_void_p), ("rope_sin", C.c_void_p), ("layers", C.POINTER(LayerWeights))]


class KvCache(C.Structure):
    _fields_ = [("k", C.c_void_p), ("v", C.c_void_p), ("layer_stride", C.c_int64), ("head_stride", C.c_int64),
                ("page_stride", C.c_int64), ("block_table", C.c_void_p), ("n_layers", C.c_int32),
                ("positions", C.c_int32), ("layer_k", C.POINTER(C.c_void_p)), ("layer_v", C.POINTER(C.c_void_p))]


class ECacheDesc(C.Structure):
    _fields_ = [("layer", C.c_int32), ("positions", C.c_int32), ("width", C.c_int32), ("hidden", C.c_void_p)]


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH.name} is not built; run `python -m paper_2411_02820_b200._build` "
                "(the CUDA path has no CPU fallback)")
        h = C.CDLL(str(LIB_PATH))
        P, I32, I64, SZ = C.c_void_p, C.c_int32, C.c_int64, C.c_size_t
        sig = {
            "ds_abi_version": (I32, []),
            "ds_last_error": (C.c_char_p, []),
            "ds_launch_count": (C.c_uint64, []),
            "ds_trace_begin": (I32, []),
            "ds_trace_end": (I32, [P, P, I32]),
            "ds_anchor_placement": (I32, [C.POINTER(Dims), I32, P, P, I32]),
            "ds_anchor_timeline": (I32, [C.POINTER(Dims), I32, P, P, I32]),
            "ds_workspace_size": (SZ, [C.POINTER(Dims), I32]),
            "ds_set_anchor_shape": (I32, [I32]),
            "ds_fused_fallbacks": (C.c_uint64, []),
            "ds_kv_ingest": (I32, [C.POINTER(KvCache), C.POINTER(KvCache), P, I32, I32, I32, I32, P,
                                   C.POINTER(I32)]),
            "ds_partial_prefill": (I32, [C.POINTER(Model), P, P, I32, P, I32, C.POINTER(KvCache),
                                         C.POINTER(ECacheDesc), I32, C.POINTER(KvCache), P, P, P, SZ, P, P,
                                         C.POINTER(I32), C.POINTER(I32)]),
            "ds_full_prefill": (I32, [C.POINTER(Model), P, P, I32, C.POINTER(KvCache), P, I32, P, P, P, P, SZ, P, P]),
            "ds_recompute_group": (I32, [C.POINTER(Model), P, I32, I32, I32, P, I32, C.POINTER(KvCache), P, SZ, P]),
            "ds_anchor": (I32, [C.POINTER(Model), P, I32, C.POINTER(KvCache), P, P, P, SZ, P]),
            "ds_token_selective_prefill": (I32, [C.POINTER(Model), P, P, I32, C.POINTER(KvCache), C.c_double,
                                                 C.POINTER(KvCache), P, P, C.POINTER(I32), P, SZ, P, C.POINTER(I32)]),
            "ds_decode_greedy": (I32, [C.POINTER(Model), C.POINTER(KvCache), I32, P, I32, P, P, SZ, P]),
            "ds_workspace_size_batch": (SZ, [C.POINTER(Dims), I32, I32]),
            "ds_partial_prefill_batch": (I32, [C.POINTER(Model), I32, P, P, P, P, I32, P, P, P, P, P, P, P, SZ, P,
                                               P, C.POINTER(I32), C.POINTER(I32), C.POINTER(I32)]),
            "ds_anchor_batch": (I32, [C.POINTER(Model), I32, P, P, P, P, P, P, SZ, P]),
            "ds_decode_greedy_batch": (I32, [C.POINTER(Model), I32, P, P, P, I32, P, P, SZ, P]),
            "ds_ipc_export": (I32, [P, P, C.POINTER(C.c_uint64)]),
            "ds_ipc_open": (I32, [P, C.c_uint64, C.POINTER(P), C.POINTER(P)]),
            "ds_ipc_close": (I32, [P]),
            "ds_gemm": (I32, [P, I64, P, I64, P, I64, P, I64, I32, I32, I32, I32, P]),
            "ds_rmsnorm": (I32, [P, I32, P, I32, I32, P, P, P, P, P]),
            "ds_attention_prefill": (I32, [P, I64, C.POINTER(KvCache), I32, I32, I32, I32, I32, I32, P, I64, P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        if h.ds_abi_version() != ABI_VERSION:
            raise RuntimeError("droidspeak ABI version mismatch")
        _lib = h
    return _lib


def check(rc: int, miss_layer: int | None = None, miss_kind: int | None = None) -> None:
    """Map a ds_status onto the reference's exception types (errors.py:6-27)."""
    if rc == DS_OK:
        return
    msg = lib().ds_last_error().decode(errors="replace")
    if rc == DS_ERR_CACHE_MISS:
        raise CacheMissError(int(miss_layer), MISS_KIND.get(miss_kind, "kv"), msg)
    if rc == DS_ERR_DEGENERATE:
        raise DegenerateInputError(msg)
    if rc == DS_ERR_INVALID:
        raise ValueError(msg)
    raise RuntimeError(f"droidspeak CUDA error: {msg}")


EXPORTED_SYMBOLS = ("ds_abi_version", "ds_last_error", "ds_launch_count", "ds_workspace_size", "ds_kv_ingest", "ds_partial_prefill",
                    "ds_full_prefill", "ds_gemm", "ds_rmsnorm", "ds_attention_prefill", "ds_recompute_group",
                    "ds_anchor", "ds_token_selective_prefill", "ds_decode_greedy", "ds_ipc_export", "ds_ipc_open", "ds_ipc_close",
                    "ds_trace_begin", "ds_trace_end", "ds_anchor_placement", "ds_anchor_timeline",
                    "ds_set_anchor_shape", "ds_fused_fallbacks", "ds_workspace_size_batch",
                    "ds_partial_prefill_batch", "ds_anchor_batch", "ds_decode_greedy_batch")


class anchor_shape:
    """Context manager forcing the anchor shape (ds_set_anchor_shape): "auto",
    "persistent" or "launch".  Process-wide; for measurements and tests."""

    def __init__(self, shape: str):
        self.shape = ANCHOR_SHAPES[shape]

    def __enter__(self):
        self.prev = lib().ds_set_anchor_shape(self.shape)
        return self

    def __exit__(self, *exc):
        lib().ds_set_anchor_shape(self.prev)
