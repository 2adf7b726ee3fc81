"""Producer export and consumer partial prefill on the B200 (the hot path).

Python mirror of the reference entry points — same names, argument meaning
and error behaviour as crosskv.model:

    full_prefill(model, tokens)                                   model.py:641-649
    partial_prefill(receiver, tokens, config, sender_kv, sender_e) model.py:660-679

Each call validates on the host in the reference's order (check_tokens,
validate_for, KV misses ascending, then E per group) and then makes ONE
C-ABI call (ds_full_prefill / ds_partial_prefill) that launches the sm_100a
kernel sequence on the caller's stream(s).  Torch only provides device
memory and streams.  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass
from typing import Iterable, Mapping, Sequence

import numpy as np
import torch

from . import _lib as L
from .config import ModelConfig, RecomputeConfig
from .errors import CacheMissError, DegenerateInputError
from .weights import ModelWeights

PAGE = 64


def check_tokens(tokens, config: ModelConfig) -> np.ndarray:
    """model.py:425-437: canonical int64 ids or raise."""
    ids = np.asarray(tokens.cpu() if isinstance(tokens, torch.Tensor) else tokens, dtype=np.int64)
    if ids.ndim != 1:
        raise ValueError("token sequence must be one-dimensional")
    n = ids.shape[0]
    if n < 2:
        raise DegenerateInputError(f"need at least 2 tokens, got {n}")
    if n > config.max_seq:
        raise ValueError(f"sequence length {n} exceeds max_seq {config.max_seq}")
    if ids.min() < 0 or ids.max() >= config.vocab_size:
        raise ValueError("token id out of vocabulary range")
    return np.ascontiguousarray(ids)


def make_synthetic_dataset(seed: int, size: int, length: int, vocab_size: int) -> list[np.ndarray]:
    """model.py:455-458."""
    rng = np.random.default_rng(seed)
    return [rng.integers(0, vocab_size, size=length, dtype=np.int64) for _ in range(size)]


# ---------------------------------------------------------------------------
# Caches
# ---------------------------------------------------------------------------


@dataclass(eq=False)
class LayerKV:
    """Dense per-layer K/V, [L, n_kv_heads, positions, head_dim] bf16 on device
    (the reference LayerKV layout, model.py:342-370; the producer export)."""

    k: torch.Tensor
    v: torch.Tensor
    context: str | None = None  # context_hash digest of the tokens it was prefilled from (store.py:55-63)

    def __post_init__(self) -> None:
        if self.k.shape != self.v.shape or self.k.dim() != 4:
            raise ValueError(f"inconsistent KV shapes {tuple(self.k.shape)} / {tuple(self.v.shape)}")

    @property
    def n_layers(self) -> int:
        return self.k.shape[0]

    @property
    def positions(self) -> int:
        return self.k.shape[2]

    def layer_bytes(self, layer: int) -> int:
        return int(self.k[layer].nbytes + self.v[layer].nbytes)

    def desc(self) -> L.KvCache:
        Ln, G, n, D = self.k.shape
        if not (self.k.is_contiguous() and self.v.is_contiguous()):
            raise ValueError("LayerKV tensors must be contiguous")
        return L.KvCache(self.k.data_ptr(), self.v.data_ptr(), G * n * D, n * D, PAGE * D, None, Ln, n)

    @classmethod
    def empty(cls, config: ModelConfig, positions: int, device="cuda") -> "LayerKV":
        # zero-filled: attention tiles may read (masked) positions beyond the
        # written ones, and p = 0 must not meet a NaN bit pattern
        shape = (config.n_layers, config.n_kv_heads, positions, config.head_dim)
        return cls(torch.zeros(shape, dtype=torch.bfloat16, device=device),
                   torch.zeros(shape, dtype=torch.bfloat16, device=device))


@dataclass(eq=False)
class PagedKV:
    """Consumer paged cache: [L, pages, n_kv_heads, 64, head_dim] bf16 + int32
    block table (position p lives in page table[p // 64], slot p % 64).  Each
    (layer, page, head) is one contiguous 64 x D block, the ingest/attention unit."""

    k: torch.Tensor
    v: torch.Tensor
    table: torch.Tensor
    positions: int

    @property
    def n_layers(self) -> int:
        return self.k.shape[0]

    def desc(self) -> L.KvCache:
        Ln, pages, G, ps, D = self.k.shape
        return L.KvCache(self.k.data_ptr(), self.v.data_ptr(), pages * G * PAGE * D, PAGE * D, G * PAGE * D,
                         self.table.data_ptr(), Ln, self.positions)

    @classmethod
    def allocate(cls, config: ModelConfig, positions: int, device="cuda", spare_pages: int = 0,
                 shuffle_seed: int | None = None, zero: bool = True) -> "PagedKV":
        """``zero=False`` skips the fill (1.07 GB at the 8B shape, 8K positions)
        for a cache a prefill writes completely: every position < ``positions``
        is written before anything reads it, and the kernels never let a value
        past the written positions reach a result (the FA prefill masks those
        keys' scores and zeroes their V rows in shared memory; the anchor and
        decode attention read keys < n only)."""
        need = (positions + PAGE - 1) // PAGE
        pages = need + spare_pages
        shape = (config.n_layers, pages, config.n_kv_heads, PAGE, config.head_dim)
        if shuffle_seed is None:
            table = torch.arange(need, dtype=torch.int32, device=device)
        else:
            g = torch.Generator().manual_seed(shuffle_seed)
            table = torch.randperm(pages, generator=g)[:need].to(torch.int32).to(device)
        make = torch.zeros if zero else torch.empty
        return cls(make(shape, dtype=torch.bfloat16, device=device), make(shape, dtype=torch.bfloat16, device=device),
                   table, positions)

    def dense(self) -> LayerKV:
        """Gather into the reference [L, KVH, n, D] layout (tests / export)."""
        idx = self.table.long()
        Ln, _, G, _, D = self.k.shape
        k = self.k[:, idx].permute(0, 2, 1, 3, 4).reshape(Ln, G, -1, D)[:, :, :self.positions]
        v = self.v[:, idx].permute(0, 2, 1, 3, 4).reshape(Ln, G, -1, D)[:, :, :self.positions]
        return LayerKV(k.contiguous(), v.contiguous())


@dataclass(eq=False)
class ECache:
    """Residual-stream input of one layer over the window, f32 [positions, d_model]
    (model.py:373-391)."""

    layer: int
    hidden: torch.Tensor

    def __post_init__(self) -> None:
        if self.hidden.dim() != 2:
            raise ValueError(f"E cache must be 2-D, got shape {tuple(self.hidden.shape)}")

    @property
    def positions(self) -> int:
        return self.hidden.shape[0]

    @property
    def nbytes(self) -> int:
        return int(self.hidden.nbytes)


@dataclass(eq=False)
class PrefillResult:
    kv: LayerKV
    e_caches: tuple
    logits: torch.Tensor       # f32 [V] on device
    token_dev: torch.Tensor    # int32 [1] greedy first token on device

    def e_map(self) -> dict:
        return {e.layer: e for e in self.e_caches}

    @property
    def token(self) -> int:
        return int(self.token_dev.item())


@dataclass(eq=False)
class MixedPrefill:
    kv: PagedKV
    logits: torch.Tensor
    token_dev: torch.Tensor

    @property
    def token(self) -> int:
        return int(self.token_dev.item())


# ---------------------------------------------------------------------------
# Workspace
# ---------------------------------------------------------------------------

# model -> {(device, stream): workspace}; weak keys, so a dead model's scratch
# goes with it and a recycled id() can never alias another model's entry
_WS: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def workspace_bytes(config: ModelConfig, n_tokens: int) -> int:
    dims = L.Dims(config.n_layers, config.d_model, config.n_heads, config.n_kv_heads, config.head_dim,
                  config.d_ff, config.vocab_size, config.max_seq, L.MLP_KINDS[config.mlp_kind])
    return int(L.lib().ds_workspace_size(C.byref(dims), n_tokens))


def _workspace(model: ModelWeights, n: int, stream=None) -> torch.Tensor:
    """Scratch for one eager call, cached per (model, device, stream): calls on
    the same stream are ordered, so they may share it; calls on different
    streams (a producer and a consumer prefilling concurrently) get their own.
    A larger n replaces the entry; the old buffer returns to the caching
    allocator of the stream it belongs to, so only later work on that same
    stream can reuse it.  CUDA graphs never use these: a capture gets a private
    workspace that lives as long as the graph (:class:`CapturedPartialPrefill`)."""
    need = workspace_bytes(model.config, n)
    s = stream if stream is not None else torch.cuda.current_stream(model.device)
    per_model = _WS.setdefault(model, {})
    key = (str(model.device), s.cuda_stream)
    ws = per_model.get(key)
    if ws is None or ws.numel() < need:
        with torch.cuda.stream(s):  # owned by the stream that uses it (allocator reuse across streams)
            ws = torch.empty(need, dtype=torch.uint8, device=model.device)
        per_model[key] = ws
    return ws


def _context_digest(tokens) -> str:
    from .store import context_hash  # store imports this module
    return context_hash(tokens).digest


def _normalize_e(sender_e) -> dict:
    if sender_e is None:
        return {}
    if isinstance(sender_e, Mapping):
        return dict(sender_e)
    return {e.layer: e for e in sender_e}


# ---------------------------------------------------------------------------
# Entry points
# ---------------------------------------------------------------------------


def full_prefill(model: ModelWeights, tokens, e_layers: Iterable[int] | None = None, *, out: LayerKV | None = None,
                 stream=None, copy_stream=None, tokens_dev: torch.Tensor | None = None,
                 workspace: torch.Tensor | None = None) -> PrefillResult:
    """Producer export: K/V at every layer over all n positions, E over the
    window (n-1 rows) at ``e_layers`` (default: every layer, profiling mode;
    pass the transition layers for the serving-mode filter, store.py:202-203),
    and first-token logits.  Same kernels and structure as a partial prefill
    with every layer recomputed (model.py:641-649), so the two agree bit for
    bit; ``copy_stream`` runs the anchor row beside the window."""
    cfg = model.config
    ids = check_tokens(tokens, cfg)
    n = ids.shape[0]
    layers = list(range(cfg.n_layers)) if e_layers is None else sorted(set(int(l) for l in e_layers))
    s = stream if stream is not None else torch.cuda.current_stream(model.device)
    with torch.cuda.stream(s):  # outputs belong to the stream that writes them (allocator reuse)
        kv = out if out is not None else LayerKV.empty(cfg, n, model.device)
        e_bufs = [torch.empty(n - 1, cfg.d_model, dtype=torch.float32, device=model.device) for _ in layers]
        logits = torch.empty(cfg.vocab_size, dtype=torch.float32, device=model.device)
        tok = torch.empty(1, dtype=torch.int32, device=model.device)
    ws = workspace if workspace is not None else _workspace(model, n, s)
    la = (C.c_int32 * max(1, len(layers)))(*layers)
    ptrs = (C.c_void_p * max(1, len(layers)))(*[b.data_ptr() for b in e_bufs])
    desc = kv.desc()
    with torch.cuda.device(model.device):  # the library launches on the current device
        rc = L.lib().ds_full_prefill(C.byref(model.desc()), ids.ctypes.data,
                                     tokens_dev.data_ptr() if tokens_dev is not None else None, n, C.byref(desc), la,
                                     len(layers), ptrs, logits.data_ptr(), tok.data_ptr(), ws.data_ptr(), ws.numel(),
                                     s.cuda_stream, copy_stream.cuda_stream if copy_stream is not None else None)
    L.check(rc)
    kv.context = _context_digest(ids)
    return PrefillResult(kv=kv, e_caches=tuple(ECache(l, b) for l, b in zip(layers, e_bufs)), logits=logits,
                         token_dev=tok)


def partial_prefill(receiver: ModelWeights, tokens, config: RecomputeConfig, sender_kv: LayerKV | None,
                    sender_e: Mapping[int, ECache] | Iterable[ECache] | None = None, *, out: PagedKV | None = None,
                    stream=None, copy_stream=None, tokens_dev: torch.Tensor | None = None,
                    workspace: torch.Tensor | None = None) -> MixedPrefill:
    """Consumer partial prefill (model.py:660-679): ingest the sender's K/V at
    reused layers, recompute each group over the window from embeddings (a=0)
    or the sender's E at its transition layer, run the anchor position through
    every layer, and produce first-token logits.  ``copy_stream`` runs the
    ingest concurrently with the recompute (pipelined plan, sched.py:212-263)."""
    cfg = receiver.config
    ids = check_tokens(tokens, cfg)
    config.validate_for(cfg.n_layers)
    n = ids.shape[0]
    e_map = _normalize_e(sender_e)
    s = stream if stream is not None else torch.cuda.current_stream(receiver.device)
    with torch.cuda.stream(s):  # outputs belong to the stream that writes them (allocator reuse)
        # every position of a fresh cache is written by this call: no zero fill
        cache = out if out is not None else PagedKV.allocate(cfg, n, receiver.device, zero=False)
        logits = torch.empty(cfg.vocab_size, dtype=torch.float32, device=receiver.device)
        tok = torch.empty(1, dtype=torch.int32, device=receiver.device)
    ws = workspace if workspace is not None else _workspace(receiver, n, s)
    groups = [x for g in config.groups for x in g]
    ga = (C.c_int32 * max(1, len(groups)))(*groups)
    for l, e in e_map.items():
        if e.hidden.dtype != torch.float32 or not e.hidden.is_cuda or not e.hidden.is_contiguous():
            raise ValueError(f"E cache of layer {l} must be a contiguous f32 device tensor")
    e_list = [L.ECacheDesc(l, e.positions, e.hidden.shape[1], e.hidden.data_ptr()) for l, e in sorted(e_map.items())]
    ea = (L.ECacheDesc * max(1, len(e_list)))(*e_list)
    skv = sender_kv.desc() if sender_kv is not None else None
    odesc = cache.desc()
    ml, mk = C.c_int32(-1), C.c_int32(0)
    with torch.cuda.device(receiver.device):
        rc = L.lib().ds_partial_prefill(
            C.byref(receiver.desc()), ids.ctypes.data, tokens_dev.data_ptr() if tokens_dev is not None else None, n,
            ga, len(config.groups), C.byref(skv) if skv is not None else None, ea, len(e_list), C.byref(odesc),
            logits.data_ptr(), tok.data_ptr(), ws.data_ptr(), ws.numel(), s.cuda_stream,
            copy_stream.cuda_stream if copy_stream is not None else None, C.byref(ml), C.byref(mk))
    L.check(rc, ml.value, mk.value)
    return MixedPrefill(kv=cache, logits=logits, token_dev=tok)


MAX_BATCH = 8  # include/droidspeak.h DS_MAX_BATCH


def batch_workspace_bytes(config: ModelConfig, max_tokens: int, batch: int) -> int:
    dims = L.Dims(config.n_layers, config.d_model, config.n_heads, config.n_kv_heads, config.head_dim,
                  config.d_ff, config.vocab_size, config.max_seq, L.MLP_KINDS[config.mlp_kind])
    return int(L.lib().ds_workspace_size_batch(C.byref(dims), max_tokens, batch))


def partial_prefill_batch(receiver: ModelWeights, tokens: Sequence, config: RecomputeConfig,
                          sender_kv: Sequence[LayerKV | None], sender_e: Sequence | None = None, *,
                          out: Sequence[PagedKV] | None = None, stream=None, copy_stream=None,
                          tokens_dev: Sequence[torch.Tensor] | None = None,
                          workspace: torch.Tensor | None = None) -> list[MixedPrefill]:
    """A consumer's batch of requests (BASELINE config 4): ``len(tokens)`` <= 8
    partial prefills with one recompute config, each request its own prefix
    (lengths may differ), producer export and output cache.  Each request is
    validated in the reference's order (check_tokens, validate_for, KV misses
    ascending, E per group; model.py:660-679), requests in order.  The
    recompute runs request after request on ``stream`` while ``copy_stream``
    ingests every request's reused layers; then ONE batched anchor pass streams
    each layer's weights once for all rows.  Results equal the requests'
    one-by-one :func:`partial_prefill` results bit for bit.  ``tokens_dev``:
    optional device copies of the requests' ids (int64, as in
    :func:`partial_prefill`; required under CUDA-graph capture)."""
    cfg = receiver.config
    nb = len(tokens)
    if not 1 <= nb <= MAX_BATCH:
        raise ValueError(f"batch of {nb} requests outside [1, {MAX_BATCH}]")
    if len(sender_kv) != nb or any(x is not None and len(x) != nb for x in (sender_e, out, tokens_dev)):
        raise ValueError("tokens, sender_kv, sender_e, out and tokens_dev must have one entry per request")
    ids = []
    for t in tokens:
        ids.append(check_tokens(t, cfg))
        config.validate_for(cfg.n_layers)
    ns = [x.shape[0] for x in ids]
    e_maps = [_normalize_e(e) for e in (sender_e if sender_e is not None else [None] * nb)]
    for em in e_maps:
        for l, e in em.items():
            if e.hidden.dtype != torch.float32 or not e.hidden.is_cuda or not e.hidden.is_contiguous():
                raise ValueError(f"E cache of layer {l} must be a contiguous f32 device tensor")
    s = stream if stream is not None else torch.cuda.current_stream(receiver.device)
    with torch.cuda.stream(s):
        caches = list(out) if out is not None else [PagedKV.allocate(cfg, n, receiver.device, zero=False) for n in ns]
        logits = torch.empty(nb, cfg.vocab_size, dtype=torch.float32, device=receiver.device)
        tok = torch.empty(nb, dtype=torch.int32, device=receiver.device)
    if workspace is None:
        need = batch_workspace_bytes(cfg, max(ns), nb)
        with torch.cuda.stream(s):
            workspace = torch.empty(need, dtype=torch.uint8, device=receiver.device)
    groups = [x for g in config.groups for x in g]
    ga = (C.c_int32 * max(1, len(groups)))(*groups)
    th = (C.c_void_p * nb)(*[x.ctypes.data for x in ids])
    td = (C.c_void_p * nb)(*[t.data_ptr() for t in tokens_dev]) if tokens_dev is not None else None
    nt = (C.c_int32 * nb)(*ns)
    empty = L.KvCache()
    skv = (L.KvCache * nb)(*[kv.desc() if kv is not None else empty for kv in sender_kv])
    e_arrays = [(L.ECacheDesc * max(1, len(em)))(*[L.ECacheDesc(l, e.positions, e.hidden.shape[1], e.hidden.data_ptr())
                                                   for l, e in sorted(em.items())]) for em in e_maps]
    ep = (C.c_void_p * nb)(*[C.cast(a, C.c_void_p) for a in e_arrays])
    ne = (C.c_int32 * nb)(*[len(em) for em in e_maps])
    odesc = (L.KvCache * nb)(*[c.desc() for c in caches])
    bad, ml, mk = C.c_int32(-1), C.c_int32(-1), C.c_int32(0)
    with torch.cuda.device(receiver.device):
        rc = L.lib().ds_partial_prefill_batch(
            C.byref(receiver.desc()), nb, th, td, nt, ga, len(config.groups), skv, ep, ne, odesc,
            logits.data_ptr(), tok.data_ptr(), workspace.data_ptr(), workspace.numel(), s.cuda_stream,
            copy_stream.cuda_stream if copy_stream is not None else None, C.byref(bad), C.byref(ml), C.byref(mk))
    L.check(rc, ml.value, mk.value)
    return [MixedPrefill(kv=caches[b], logits=logits[b], token_dev=tok[b:b + 1]) for b in range(nb)]


class CapturedPartialPrefill:
    """A consumer partial prefill captured once as a CUDA graph and replayed per
    request -- the serving form of :func:`partial_prefill` for a fixed receiver,
    recompute config, sender export, output cache and prefix length (CUDA graphs
    instead of a tracing compiler).

    The graph reads ONE export: the sender's K/V and E of one context.  Its
    context is ``context_hash(context)`` when ``context`` (the tokens the export
    was prefilled from) is given, else the export's own tag (``LayerKV.context``
    set by :func:`full_prefill`, ``FetchedKV.context`` by the store,
    ``RemoteKV.context`` by the IPC transport).  :meth:`run` hashes each
    request's tokens and raises ``CacheMissError`` -- what the reference's
    ``fetch_context_caches`` raises for a context it does not hold
    (store.py:351-395) -- when they are not that context, so a request can never
    be served another context's KV.  A config that reads no export (every layer
    recomputed from the embeddings) accepts any tokens.

    Construction runs the call once eagerly (all validation and cache-miss
    errors surface there, exactly as :func:`partial_prefill` raises them), then
    captures it into a graph with a PRIVATE workspace that lives as long as this
    object (eager calls on the same streams can never resize or free it).
    :meth:`run` validates the tokens on the host (check_tokens,
    model.py:425-437), copies them into a fixed device buffer (asynchronously
    from pinned memory) and replays the whole two-stream step: one graph launch
    instead of ~30 kernel launches.  The returned :class:`MixedPrefill` holds
    the same device tensors on every call (the graph writes into them); copy
    what must outlive the next request."""

    def __init__(self, receiver: ModelWeights, n_tokens: int, config: RecomputeConfig, sender_kv: LayerKV | None,
                 sender_e: Mapping[int, ECache] | Iterable[ECache] | None = None, *, out: PagedKV | None = None,
                 stream=None, copy_stream=None, context=None):
        cfg = receiver.config
        self.receiver, self.n = receiver, int(n_tokens)
        reads_export = sender_kv is not None or any(a > 0 for a, _ in config.groups)
        if context is not None:
            tag = _context_digest(check_tokens(context, cfg))
            own = getattr(sender_kv, "context", None)
            if own is not None and own != tag:
                raise ValueError("context= does not match the context the sender export was prefilled from")
        else:
            tag = getattr(sender_kv, "context", None)
        if reads_export and tag is None:
            raise ValueError("the sender export carries no context tag: pass context=<the tokens it was prefilled from>")
        self.context = tag if reads_export else None
        reused = config.reused_layers(cfg.n_layers)
        self._miss = (reused[0], "kv") if reused else (config.transition_layers[0] if config.transition_layers else 0,
                                                      "e")
        self.stream = stream if stream is not None else torch.cuda.Stream(device=receiver.device)
        self.copy_stream = copy_stream if copy_stream is not None else torch.cuda.Stream(device=receiver.device)
        with torch.cuda.stream(self.stream):
            self.tokens_dev = torch.zeros(self.n, dtype=torch.int64, device=receiver.device)
            self.workspace = torch.empty(workspace_bytes(cfg, self.n), dtype=torch.uint8, device=receiver.device)
        probe = np.zeros(self.n, dtype=np.int64)  # valid ids for the host-side checks during capture
        self.out = out if out is not None else PagedKV.allocate(cfg, self.n, receiver.device)

        def call():
            return partial_prefill(receiver, probe, config, sender_kv, sender_e, out=self.out, stream=self.stream,
                                   copy_stream=self.copy_stream, tokens_dev=self.tokens_dev, workspace=self.workspace)

        with torch.cuda.stream(self.stream):
            call()  # eager: raises like partial_prefill
        torch.cuda.synchronize(receiver.device)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            self.result = call()

    def run(self, tokens) -> MixedPrefill:
        if isinstance(tokens, torch.Tensor):
            src = tokens
            ids = check_tokens(tokens.numpy(), self.receiver.config)
        else:
            ids = check_tokens(tokens, self.receiver.config)
            src = torch.from_numpy(ids)
        if src.shape[0] != self.n:
            raise ValueError(f"captured for {self.n} tokens, got {src.shape[0]}")
        if self.context is not None and _context_digest(ids) != self.context:
            layer, kind = self._miss
            raise CacheMissError(layer, kind, "request tokens are not the context of the captured export")
        caller = torch.cuda.current_stream(self.receiver.device)
        self.stream.wait_stream(caller)  # the previous request's readers are done with the outputs
        with torch.cuda.stream(self.stream):
            self.tokens_dev.copy_(src, non_blocking=True)
            self.graph.replay()
        caller.wait_stream(self.stream)  # the caller's stream sees this request's outputs
        return self.result


class CapturedPartialPrefillBatch:
    """:func:`partial_prefill_batch` captured once as a CUDA graph and replayed
    per batch -- the serving form of config 4 for a fixed receiver, recompute
    config, request lengths and one export per batch slot.  As
    :class:`CapturedPartialPrefill`, slot b serves only the context of the export
    it was captured with: :meth:`run` hashes each request's tokens and raises
    ``CacheMissError`` for another context (store.py:351-395) instead of reusing
    the wrong KV.  Construction runs the batch once eagerly (every validation and
    cache-miss error surfaces there), then captures it with a private workspace
    and fixed device token buffers; :meth:`run` copies the batch's tokens in and
    replays the two-stream step.  The returned results are the same tensors on
    every call."""

    def __init__(self, receiver: ModelWeights, n_tokens: Sequence[int], config: RecomputeConfig,
                 sender_kv: Sequence[LayerKV | None], sender_e: Sequence | None = None, *,
                 out: Sequence[PagedKV] | None = None, stream=None, copy_stream=None, contexts=None):
        cfg = receiver.config
        self.receiver, self.ns = receiver, [int(n) for n in n_tokens]
        nb = len(self.ns)
        reads_export = bool(config.reused_layers(cfg.n_layers)) or any(a > 0 for a, _ in config.groups)
        self.contexts = []
        for b in range(nb):
            if contexts is not None and contexts[b] is not None:
                tag = _context_digest(check_tokens(contexts[b], cfg))
            else:
                tag = getattr(sender_kv[b], "context", None) if sender_kv[b] is not None else None
            if reads_export and tag is None:
                raise ValueError(f"slot {b}: the export carries no context tag: pass contexts=[...]")
            self.contexts.append(tag if reads_export else None)
        self.stream = stream if stream is not None else torch.cuda.Stream(device=receiver.device)
        self.copy_stream = copy_stream if copy_stream is not None else torch.cuda.Stream(device=receiver.device)
        with torch.cuda.stream(self.stream):
            self.tokens_dev = [torch.zeros(n, dtype=torch.int64, device=receiver.device) for n in self.ns]
            self.workspace = torch.empty(batch_workspace_bytes(cfg, max(self.ns), nb), dtype=torch.uint8,
                                         device=receiver.device)
        self.out = list(out) if out is not None else [PagedKV.allocate(cfg, n, receiver.device, zero=False)
                                                     for n in self.ns]
        probes = [np.zeros(n, dtype=np.int64) for n in self.ns]

        def call():
            return partial_prefill_batch(receiver, probes, config, sender_kv, sender_e, out=self.out,
                                         stream=self.stream, copy_stream=self.copy_stream,
                                         tokens_dev=self.tokens_dev, workspace=self.workspace)

        with torch.cuda.stream(self.stream):
            call()  # eager: raises like partial_prefill_batch
        torch.cuda.synchronize(receiver.device)
        reused = config.reused_layers(cfg.n_layers)
        self._miss = (reused[0], "kv") if reused else (config.transition_layers[0] if config.transition_layers else 0,
                                                      "e")
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            self.result = call()

    def run(self, tokens: Sequence) -> list:
        if len(tokens) != len(self.ns):
            raise ValueError(f"captured for a batch of {len(self.ns)}, got {len(tokens)}")
        srcs = []
        for b, t in enumerate(tokens):
            ids = check_tokens(t.numpy() if isinstance(t, torch.Tensor) else t, self.receiver.config)
            if ids.shape[0] != self.ns[b]:
                raise ValueError(f"slot {b}: captured for {self.ns[b]} tokens, got {ids.shape[0]}")
            if self.contexts[b] is not None and _context_digest(ids) != self.contexts[b]:
                layer, kind = self._miss
                raise CacheMissError(layer, kind, f"request {b} tokens are not the context of its captured export")
            srcs.append(t if isinstance(t, torch.Tensor) else torch.from_numpy(ids))
        caller = torch.cuda.current_stream(self.receiver.device)
        self.stream.wait_stream(caller)
        with torch.cuda.stream(self.stream):
            for dst, src in zip(self.tokens_dev, srcs):
                dst.copy_(src, non_blocking=True)
            self.graph.replay()
        caller.wait_stream(self.stream)
        return self.result


def token_selective_prefill(receiver: ModelWeights, tokens, sender_kv: LayerKV, ratio: float, *,
                            out: PagedKV | None = None, stream=None,
                            tokens_dev: torch.Tensor | None = None) -> MixedPrefill:
    """Token-selective baseline (model.py:682-743, the CacheBlend comparison
    point): every layer starts from the sender's K/V; the ceil(ratio * window)
    positions whose receiver layer-0 K/V deviate most from the sender's (ties to
    the lowest position) are recomputed through the whole stack, then the
    anchor runs through every layer.  ``n_selected`` on the result is the count."""
    cfg = receiver.config
    if not 0.0 < ratio <= 1.0:
        raise ValueError(f"ratio must lie in (0, 1], got {ratio}")
    ids = check_tokens(tokens, cfg)
    n = ids.shape[0]
    if sender_kv is None:
        raise CacheMissError(0, "kv", "sender cache missing layers")
    s = stream if stream is not None else torch.cuda.current_stream(receiver.device)
    with torch.cuda.stream(s):  # outputs belong to the stream that writes them (allocator reuse)
        cache = out if out is not None else PagedKV.allocate(cfg, n, receiver.device)
        logits = torch.empty(cfg.vocab_size, dtype=torch.float32, device=receiver.device)
        tok = torch.empty(1, dtype=torch.int32, device=receiver.device)
    ws = _workspace(receiver, n, s)
    skv, odesc = sender_kv.desc(), cache.desc()
    ml, nsel = C.c_int32(-1), C.c_int32(0)
    with torch.cuda.device(receiver.device):
        rc = L.lib().ds_token_selective_prefill(
            C.byref(receiver.desc()), ids.ctypes.data, tokens_dev.data_ptr() if tokens_dev is not None else None, n,
            C.byref(skv), float(ratio), C.byref(odesc), logits.data_ptr(), tok.data_ptr(), C.byref(nsel),
            ws.data_ptr(), ws.numel(), s.cuda_stream, C.byref(ml))
    L.check(rc, ml.value, 0)
    res = MixedPrefill(kv=cache, logits=logits, token_dev=tok)
    res.n_selected = int(nsel.value)
    return res
