"""Greedy decode, first-token / horizon agreement and the profiler sweep on the B200.

Mirrors of the reference's quality proxy:

    decode_greedy(model, cache, last, steps)     model.py:751-788  (ds_decode_greedy)
    greedy_agreement(reference, candidate)       model.py:791-807
    agreement_score(sender, receiver, tokens,
                    config, horizon)             model.py:810-831
    run_profile(sender, receiver, train_set,
                granularity, horizon)            profiler.py:124-184 (+ enumerate_groups)

Every forward pass runs on the sm_100a kernels through the C ABI; only the
token streams (ints) come back to the host.  Decoding appends K/V at positions
n, n+1, ... of the cache, so caches that will be decoded from are allocated
with capacity (``reserve`` below); positions 0..n-1 are never touched.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _lib as L
from .config import RecomputeConfig
from .engine import LayerKV, PagedKV, _workspace, check_tokens, full_prefill, partial_prefill
from .selection import ProfilePoint, enumerate_groups


@dataclass(frozen=True)
class Agreement:
    score: float
    first_divergence: int | None
    reference: tuple
    candidate: tuple


def decode_greedy(model, cache, last, steps: int, positions: int | None = None) -> np.ndarray:
    """``steps`` greedy tokens after a prefill (ties -> lowest id).

    ``cache``: the prefill's PagedKV or dense LayerKV, with capacity for
    ``positions + steps - 1`` positions.  ``last``: the prefill result (its
    device argmax token is step 0) or a device int32 token tensor.
    ``positions``: tokens already in the cache (default: the prefill's n).
    """
    cfg = model.config
    if steps < 1:
        raise ValueError("steps must be at least 1")
    first = getattr(last, "token_dev", last)
    if positions is None:
        positions = getattr(last, "n_tokens", None)
    if positions is None:
        raise ValueError("positions is required when `last` is not a prefill result")
    if positions < 1:
        raise ValueError("cache must hold at least one position")
    if positions + steps > cfg.max_seq:
        raise ValueError(f"decoding {steps} steps from {positions} positions exceeds max_seq {cfg.max_seq}")
    cap = cache.positions
    if positions + steps - 1 > cap:
        raise ValueError(f"cache capacity {cap} < {positions + steps - 1} positions needed; allocate with reserve")
    out = torch.empty(steps, dtype=torch.int32, device=model.device)
    ws = _workspace(model, positions + steps)
    desc = cache.desc()
    with torch.cuda.device(model.device):
        rc = L.lib().ds_decode_greedy(C.byref(model.desc()), C.byref(desc), positions, first.data_ptr(), steps,
                                      out.data_ptr(), ws.data_ptr(), ws.numel(),
                                      torch.cuda.current_stream(model.device).cuda_stream)
    L.check(rc)
    return out.cpu().numpy().astype(np.int64)


def decode_greedy_batch(model, caches, lasts, steps: int, positions) -> np.ndarray:
    """Greedy decode of up to 8 sequences at once (each its own cache and
    length): one batched anchor pass per step streams the weights once for
    every sequence.  Row b equals ``decode_greedy(model, caches[b], lasts[b],
    steps, positions[b])`` token for token.  Returns int64 [batch, steps]."""
    cfg = model.config
    nb = len(caches)
    if not 1 <= nb <= 8 or len(lasts) != nb or len(positions) != nb:
        raise ValueError("caches, lasts and positions must have 1..8 matching entries")
    if steps < 1:
        raise ValueError("steps must be at least 1")
    for c, p in zip(caches, positions):
        if p < 1:
            raise ValueError("cache must hold at least one position")
        if p + steps > cfg.max_seq:
            raise ValueError(f"decoding {steps} steps from {p} positions exceeds max_seq {cfg.max_seq}")
        if p + steps - 1 > c.positions:
            raise ValueError(f"cache capacity {c.positions} < {p + steps - 1} positions needed; allocate with reserve")
    dev = model.device
    first = torch.cat([getattr(x, "token_dev", x).reshape(1).to(torch.int32) for x in lasts])
    out = torch.empty(nb, steps, dtype=torch.int32, device=dev)
    need = int(L.lib().ds_workspace_size_batch(C.byref(model.desc().dims), max(p + steps for p in positions), nb))
    ws = torch.empty(need, dtype=torch.uint8, device=dev)
    descs = (L.KvCache * nb)(*[c.desc() for c in caches])
    pos = (C.c_int32 * nb)(*[int(p) for p in positions])
    with torch.cuda.device(dev):
        rc = L.lib().ds_decode_greedy_batch(C.byref(model.desc()), nb, descs, pos, first.data_ptr(), steps,
                                            out.data_ptr(), ws.data_ptr(), ws.numel(),
                                            torch.cuda.current_stream(dev).cuda_stream)
    L.check(rc)
    return out.cpu().numpy().astype(np.int64)


def greedy_agreement(reference, candidate) -> Agreement:
    ref, cand = np.asarray(reference), np.asarray(candidate)
    if ref.shape != cand.shape:
        raise ValueError("token streams must have equal length")
    same = ref == cand
    bad = np.flatnonzero(~same)
    return Agreement(float(np.mean(same)), int(bad[0]) if bad.size else None, tuple(int(t) for t in ref),
                     tuple(int(t) for t in cand))


def _receiver_reference(receiver, ids, horizon: int) -> np.ndarray:
    """The receiver's own greedy stream: a recompute-all partial prefill (the
    receiver's full prefill computed by the same kernels the candidates use, so
    recompute-all agrees with it bit for bit, as model.py guarantees for the
    reference: test_model.py:156-161) followed by ``horizon`` decode steps."""
    cfg = receiver.config
    cache = PagedKV.allocate(cfg, len(ids) + horizon, receiver.device)
    own = partial_prefill(receiver, ids, RecomputeConfig.full(cfg.n_layers), None, out=cache)
    return decode_greedy(receiver, cache, own.token_dev, horizon, positions=len(ids))


def _prefill_with_capacity(model, ids, reserve: int, e_layers=None):
    kv = LayerKV.empty(model.config, len(ids) + reserve, model.device)
    res = full_prefill(model, ids, e_layers=e_layers, out=kv)
    res.n_tokens = len(ids)
    return res


def agreement_score(sender, receiver, tokens, config: RecomputeConfig, horizon: int = 32) -> Agreement:
    """Receiver's own decode vs the decode after a partial prefill over the
    sender's caches (model.py:810-831)."""
    if horizon < 1:
        raise ValueError("horizon must be at least 1")
    ids = check_tokens(tokens, receiver.config)
    ref_tokens = _receiver_reference(receiver, ids, horizon)
    sent = full_prefill(sender, ids, e_layers=config.transition_layers)
    cand_tokens = _mixed_decode(receiver, ids, config, sent, horizon)
    return greedy_agreement(ref_tokens, cand_tokens)


def _mixed_decode(receiver, ids, config, sent, horizon):
    cache = PagedKV.allocate(receiver.config, len(ids) + horizon, receiver.device)
    mixed = partial_prefill(receiver, ids, config, sent.kv, sent.e_map(), out=cache)
    return decode_greedy(receiver, cache, mixed.token_dev, horizon, positions=len(ids))


class PairEvaluator:
    """Per training sequence: the receiver's reference decode and the sender's
    export, computed once; ``quality(config)`` = mean agreement over the set
    (profiler.py:124-155)."""

    def __init__(self, sender, receiver, train_set: Sequence, horizon: int):
        if not len(train_set):
            raise ValueError("training set is empty")
        if horizon < 1:
            raise ValueError("horizon must be at least 1")
        self.sender, self.receiver, self.horizon = sender, receiver, horizon
        self.items = []
        for seq in train_set:
            ids = check_tokens(seq, receiver.config)
            ref_tokens = _receiver_reference(receiver, ids, horizon)
            sent = full_prefill(sender, ids)  # profiling mode: E at every layer
            self.items.append((ids, sent, ref_tokens))

    def quality(self, config: RecomputeConfig) -> float:
        scores = [greedy_agreement(ref, _mixed_decode(self.receiver, ids, config, sent, self.horizon)).score
                  for ids, sent, ref in self.items]
        return float(np.mean(scores))


def run_profile(sender, receiver, train_set, granularity: int = 2, horizon: int = 32) -> list:
    """Score every contiguous block-run config (profiler.py:170-184) on the GPU."""
    ev = PairEvaluator(sender, receiver, train_set, horizon)
    pts = [ProfilePoint(cfg, cfg.recomputed_layer_count, ev.quality(cfg))
           for cfg in enumerate_groups(receiver.config.n_layers, granularity)]
    pts.sort(key=lambda p: (p.k, p.config.groups[0][0]))
    return pts
