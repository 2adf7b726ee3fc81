"""Layer-pipelined consumer scheduler on CUDA streams and events.

Realises the pipelined plan of the reference planner (sched.py:212-263,
restated in :mod:`.planner`) on one consumer GPU:

* a LINK stream executes the per-layer transfer jobs in the plan's FIFO order
  (``planner.link_order``: E of each transition layer first, then the reused
  layers' KV ascending).  With the producer on the same GPU or pulled over
  NVLink (P2P), a KV job is one ``ds_kv_ingest`` launch that reads the
  producer's export in place and scatters it into the consumer's paged cache;
  with the NCCL transport it is a ``recv`` into a staging slice followed by
  the same ingest.  Every job records an event;
* a COMPUTE stream runs each recompute group (``ds_recompute_group``) as soon
  as its seeding E has landed (groups starting at layer 0 start at once);
* the anchor pass (``ds_anchor``) waits for the last link event and the last
  recompute, exactly the plan's ``anchor_start = max(compute, transfers)``.

Numerically this is the same kernel sequence as ``ds_partial_prefill`` (the
fused single-call form), so the two agree bit for bit; the tests check it.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from .config import RecomputeConfig
from .engine import MixedPrefill, PagedKV, _normalize_e, _workspace, check_tokens
from .errors import CacheMissError
from .planner import ScheduledRequest, link_order


@dataclass
class StageTimes:
    """CUDA-event timestamps (ms from the request start) of one pipelined run."""

    link: list = field(default_factory=list)      # (label, start_ms, end_ms)
    compute: list = field(default_factory=list)
    ttft_ms: float = 0.0


class LocalTransport:
    """Sender caches already addressable from this GPU (same device, or a peer
    GPU's memory mapped through CUDA IPC / peer access): KV jobs ingest in
    place, E jobs are no-ops because the recompute's first kernel reads E where
    it lies."""

    def e_job(self, layer: int, e, link: torch.cuda.Stream):
        return e.hidden

    def kv_job(self, layer: int, src_desc, dst_desc, window, cfg, link):
        arr = (C.c_int32 * 1)(layer)
        miss = C.c_int32(-1)
        rc = L.lib().ds_kv_ingest(C.byref(src_desc), C.byref(dst_desc), arr, 1, window, cfg.n_kv_heads,
                                  cfg.head_dim, link.cuda_stream, C.byref(miss))
        L.check(rc, miss.value, 1)


class ConsumerPipeline:
    """One consumer model's partial prefill, layer-pipelined (see module doc)."""

    def __init__(self, receiver, device=None, transport=None, batch_kv_jobs: int = 1):
        self.receiver = receiver
        self.device = torch.device(device) if device is not None else receiver.device
        self.compute = torch.cuda.Stream(self.device)
        self.link = torch.cuda.Stream(self.device)
        self.transport = transport or LocalTransport()
        self.batch = max(1, int(batch_kv_jobs))
        self._events: list = []

    def _event(self, timing: bool):
        return torch.cuda.Event(enable_timing=timing)

    def run(self, tokens, config: RecomputeConfig, sender_kv, sender_e=None, *, out: PagedKV | None = None,
            tokens_dev: torch.Tensor | None = None, timing: bool = False, arrival_event=None):
        with torch.cuda.device(self.device):  # the library launches on the current device
            return self._run(tokens, config, sender_kv, sender_e, out=out, tokens_dev=tokens_dev, timing=timing,
                             arrival_event=arrival_event)

    def _run(self, tokens, config, sender_kv, sender_e, *, out, tokens_dev, timing, arrival_event):
        cfg = self.receiver.config
        ids = check_tokens(tokens, cfg)
        config.validate_for(cfg.n_layers)
        n = ids.shape[0]
        P = n - 1
        e_map = _normalize_e(sender_e)
        skv = sender_kv.desc() if sender_kv is not None else None
        if not getattr(self.transport, "provides_all", False):
            # reference error order: KV misses ascending, then E per group (model.py:590-617)
            for l in config.reused_layers(cfg.n_layers):
                if skv is None or l >= skv.n_layers or skv.positions < P or not _present(skv, l):
                    raise CacheMissError(l, "kv")
            for a, _ in config.groups:
                if a > 0:
                    e = e_map.get(a)
                    if e is None or e.positions < P or e.hidden.shape[1] != cfg.d_model:
                        raise CacheMissError(a, "e")
        with torch.cuda.stream(self.compute):  # outputs belong to the stream that writes them
            cache = out if out is not None else PagedKV.allocate(cfg, n, self.device)
            logits = torch.empty(cfg.vocab_size, dtype=torch.float32, device=self.device)
            tok = torch.empty(1, dtype=torch.int32, device=self.device)
        dst = cache.desc()
        ws = _workspace(self.receiver, n, self.compute)
        cur = torch.cuda.current_stream(self.device)
        start = arrival_event or self._event(timing)
        if arrival_event is None:
            start.record(cur)
        self.link.wait_event(start)
        self.compute.wait_event(start)
        if out is not None:
            self.compute.wait_stream(cur)  # the caller's pending work on its cache
        if tokens_dev is None:
            # on the compute stream, which every reader of the ids (the group seed,
            # the anchor) runs on: ordered before them whatever event gates the start
            with torch.cuda.stream(self.compute):
                tokens_dev = torch.from_numpy(ids).to(self.device, non_blocking=True)
        times = StageTimes()
        req = ScheduledRequest("r", 0.0, self.receiver.ident, config, cfg.n_layers)

        # ---- link: E first, then reused KV ascending (planner.link_order)
        e_ready, e_ptr = {}, {}
        jobs = link_order([req])
        i = 0
        marks = []
        with torch.cuda.stream(self.link):
            while i < len(jobs):
                job = jobs[i]
                if job.kind == "e":
                    e_ptr[job.layer] = self.transport.e_job(job.layer, e_map.get(job.layer), self.link)
                    ev = self._event(timing)
                    ev.record(self.link)
                    e_ready[job.layer] = ev
                    marks.append((f"E-transfer({job.layer})", ev))
                    i += 1
                    continue
                span = [job.layer]
                while (len(span) < self.batch and i + len(span) < len(jobs) and jobs[i + len(span)].kind == "kv"):
                    span.append(jobs[i + len(span)].layer)
                for l in span:
                    self.transport.kv_job(l, skv, dst, P, cfg, self.link)
                ev = self._event(timing)
                ev.record(self.link)
                marks.append((f"KV-transfer({span[0]}..{span[-1]})", ev))
                i += len(span)
            link_done = self._event(timing)
            link_done.record(self.link)

        # ---- compute: each group gated on its seeding E
        cmarks = []
        lib = L.lib()
        mdesc = self.receiver.desc()
        for a, b in config.groups:
            if a > 0:
                self.compute.wait_event(e_ready[a])
            seed = e_ptr.get(a)
            rc = lib.ds_recompute_group(C.byref(mdesc), tokens_dev.data_ptr(), n, a, b,
                                        seed.data_ptr() if seed is not None else None,
                                        seed.shape[0] if seed is not None else 0, C.byref(dst), ws.data_ptr(),
                                        ws.numel(), self.compute.cuda_stream)
            L.check(rc, a, 2)
            ev = self._event(timing)
            ev.record(self.compute)
            cmarks.append((f"recompute({a}..{b})", ev))
        # ---- anchor after every transfer and recompute (sched.py:256)
        self.compute.wait_event(link_done)
        rc = lib.ds_anchor(C.byref(mdesc), tokens_dev.data_ptr(), n, C.byref(dst), logits.data_ptr(), tok.data_ptr(),
                           ws.data_ptr(), ws.numel(), self.compute.cuda_stream)
        L.check(rc)
        done = self._event(timing)
        done.record(self.compute)
        cmarks.append(("anchor", done))
        cur.wait_stream(self.compute)
        self._last = (start, marks, cmarks, done) if timing else None
        return MixedPrefill(kv=cache, logits=logits, token_dev=tok)

    def stage_times(self) -> StageTimes:
        """Event times of the last ``run(timing=True)`` (synchronises)."""
        start, marks, cmarks, done = self._last
        done.synchronize()
        t = StageTimes()
        prev = 0.0
        for lab, ev in marks:
            e = start.elapsed_time(ev)
            t.link.append((lab, prev, e))
            prev = e
        prev = 0.0
        for lab, ev in cmarks:
            e = start.elapsed_time(ev)
            t.compute.append((lab, prev, e))
            prev = e
        t.ttft_ms = start.elapsed_time(done)
        return t


def _present(desc, layer: int) -> bool:
    if desc.layer_k:
        return bool(desc.layer_k[layer]) and bool(desc.layer_v[layer])
    return bool(desc.k) and bool(desc.v)
