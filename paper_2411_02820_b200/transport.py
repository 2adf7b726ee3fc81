"""Producer -> consumer transfer of the cross-model caches.

The path shards by consumer: each consumer GPU needs only the producer's KV
for its reused layers and the producer's E at its transition layers; nothing
flows between consumers.  Two transports realise the per-layer "link" of the
pipelined plan (sched.py:212-263):

* **P2P pull (primary).**  The producer exports its resident export buffers
  once (``export_prefill`` -> CUDA IPC handles, ``ds_ipc_export``).  A consumer
  maps them (``RemoteExport``, ``ds_ipc_open``) and its OWN kernels read the
  producer's HBM over NVLink in place: the KV-ingest kernel scatters peer pages
  straight into the local paged cache (transfer and scatter in one kernel) and
  the recompute group's first kernel reads the peer E.  The producer does no
  per-request work.
* **NCCL send/recv (baseline).**  ``NcclSender.serve`` sends E(a) then KV(l) in
  the planner's link order; the consumer's ``NcclTransport`` receives each job
  into a staging slot on the link stream and ingests it from there.
* **Broadcast fan-out.**  ``broadcast_export`` sends one context's export to
  every consumer with collectives (E first, then K/V per layer ascending): on
  NVSwitch systems NCCL runs them as in-switch multicast (NVLS), so the
  producer's egress is one copy of the export whatever the consumer count
  (unicast pulls cost it one copy per consumer).

Handles and metadata travel as small picklable objects (``torch.distributed``
object collectives), so the same code runs one process per GPU under torchrun.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import torch

from . import _lib as L
from .engine import PAGE, ECache, PrefillResult
from .planner import LinkJob, ScheduledRequest, link_order
from .store import context_hash


# ---------------------------------------------------------------------------
# P2P pull through CUDA IPC
# ---------------------------------------------------------------------------


def ipc_export(t: torch.Tensor) -> tuple:
    """(64-byte handle, byte offset) for a device tensor's storage."""
    h = (C.c_ubyte * 64)()
    off = C.c_uint64(0)
    L.check(L.lib().ds_ipc_export(t.data_ptr(), h, C.byref(off)))
    return bytes(h), int(off.value)


@dataclass
class ExportHandles:
    """What a producer publishes for one prefilled context (picklable)."""

    model_id: str
    context: str
    n_layers: int
    n_kv_heads: int
    positions: int
    head_dim: int
    d_model: int
    device: int
    k: tuple = ()
    v: tuple = ()
    e: dict = field(default_factory=dict)  # layer -> (handle, offset, rows)


def export_prefill(prefill: PrefillResult, model_id: str, tokens) -> ExportHandles:
    kv = prefill.kv
    if not (kv.k.is_contiguous() and kv.v.is_contiguous()):
        raise ValueError("export buffers must be contiguous")
    Ln, G, n, D = kv.k.shape
    d = prefill.e_caches[0].hidden.shape[1] if prefill.e_caches else 0
    out = ExportHandles(model_id, context_hash(tokens).digest, Ln, G, n, D, d, kv.k.device.index or 0,
                        ipc_export(kv.k), ipc_export(kv.v))
    for e in prefill.e_caches:
        h, off = ipc_export(e.hidden)
        out.e[e.layer] = (h, off, e.hidden.shape[0])
    return out


class PeerBuffer:
    """An f32 [rows, cols] region (an E export) of a peer GPU's HBM mapped into this process.
    Duck-types the few tensor properties the engine reads (data_ptr, shape,
    dtype, is_cuda, is_contiguous, dim, nbytes)."""

    dtype = torch.float32
    is_cuda = True

    def __init__(self, ptr: int, rows: int, cols: int):
        self.ptr, self.shape = int(ptr), (int(rows), int(cols))

    def data_ptr(self) -> int:
        return self.ptr

    def dim(self) -> int:
        return 2

    def is_contiguous(self) -> bool:
        return True

    @property
    def nbytes(self) -> int:
        return self.shape[0] * self.shape[1] * 4


class _DeviceArray:
    """__cuda_array_interface__ over a raw device pointer (a mapped peer buffer)."""

    def __init__(self, ptr: int, shape: tuple, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(int(x) for x in shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def peer_view(ptr: int, shape: tuple, dtype: torch.dtype) -> torch.Tensor:
    """A torch view (no copy) of a mapped peer buffer; bf16 travels as f16 bits."""
    typestr = {torch.float32: "<f4", torch.bfloat16: "<f2"}[dtype]
    t = torch.as_tensor(_DeviceArray(ptr, shape, typestr), device=torch.device("cuda", torch.cuda.current_device()))
    return t.view(dtype) if dtype == torch.bfloat16 else t


class RemoteKV:
    """The producer's dense [L, KVH, n, D] export, mapped; ``desc()`` for the ingest."""

    def __init__(self, k_ptr: int, v_ptr: int, n_layers: int, n_kv_heads: int, positions: int, head_dim: int,
                 context: str | None = None):
        self.k_ptr, self.v_ptr = k_ptr, v_ptr
        self.context = context
        self.n_layers, self.n_kv_heads, self.positions, self.head_dim = n_layers, n_kv_heads, positions, head_dim

    def desc(self) -> L.KvCache:
        G, n, D = self.n_kv_heads, self.positions, self.head_dim
        return L.KvCache(self.k_ptr, self.v_ptr, G * n * D, n * D, PAGE * D, None, self.n_layers, n)


class RemoteExport:
    """Consumer-side mapping of a producer's ExportHandles."""

    def __init__(self, handles: ExportHandles):
        self.handles = handles
        self._bases = []
        k = self._open(*handles.k)
        v = self._open(*handles.v)
        self.kv = RemoteKV(k, v, handles.n_layers, handles.n_kv_heads, handles.positions, handles.head_dim,
                           handles.context)
        self.e_map = {l: ECache(l, PeerBuffer(self._open(h, off), rows, handles.d_model))
                      for l, (h, off, rows) in handles.e.items()}

    def _open(self, handle: bytes, offset: int) -> int:
        base, ptr = C.c_void_p(), C.c_void_p()
        buf = (C.c_ubyte * 64).from_buffer_copy(handle)
        L.check(L.lib().ds_ipc_open(buf, offset, C.byref(base), C.byref(ptr)))
        self._bases.append(base.value)
        return ptr.value

    def local_copy(self, stream=None):
        """Pull the whole export over the link into this GPU's HBM (one copy per
        tensor): ``(LayerKV, {layer: ECache})`` with the export's context tag.
        The fan-out bench times the consumer step on it (local data) beside the
        step on the mapped export (NVLink) -- the §8d hidden fraction."""
        from .engine import LayerKV
        h = self.handles
        shape = (h.n_layers, h.n_kv_heads, h.positions, h.head_dim)
        s = stream if stream is not None else torch.cuda.current_stream()
        with torch.cuda.stream(s):
            k = peer_view(self.kv.k_ptr, shape, torch.bfloat16).clone()
            v = peer_view(self.kv.v_ptr, shape, torch.bfloat16).clone()
            e = {l: ECache(l, peer_view(ec.hidden.data_ptr(), ec.hidden.shape, torch.float32).clone())
                 for l, ec in self.e_map.items()}
        return LayerKV(k, v, context=h.context), e

    def close(self) -> None:
        for b in self._bases:
            L.lib().ds_ipc_close(b)
        self._bases.clear()


# ---------------------------------------------------------------------------
# NCCL send/recv (baseline transport)
# ---------------------------------------------------------------------------


def job_tensors(prefill: PrefillResult, job: LinkJob, window: int) -> list:
    """The producer-side tensors one link job moves: E(a) [window, d], or K and
    V of layer l over the window (contiguous [KVH, window, D] each)."""
    if job.kind == "e":
        return [job_tensor(prefill, job, window, 0)]
    return [job_tensor(prefill, job, window, 0), job_tensor(prefill, job, window, 1)]


def job_tensor(prefill: PrefillResult, job: LinkJob, window: int, part: int) -> torch.Tensor:
    """Message ``part`` of a link job: E(a) (part 0), or K (0) / V (1) of the layer."""
    if job.kind == "e":
        return prefill.e_map()[job.layer].hidden[:window]
    src = prefill.kv.k if part == 0 else prefill.kv.v
    return src[job.layer, :, :window].contiguous()


class NcclSender:
    """Producer side: serves link jobs to consumer ranks, each consumer's jobs
    in the planner's FIFO order (sched.py:217-223).  The consumers are served
    concurrently: message i of every consumer goes out in one grouped
    point-to-point call (``batch_isend_irecv``: one NCCL group, so the sends to
    different consumers overlap instead of queueing behind each other), and a
    round's payloads are staged only for that round."""

    def __init__(self, group=None):
        self.group = group

    def serve(self, prefill: PrefillResult, requests: list, n_layers: int) -> None:
        """requests: [(dst_rank, RecomputeConfig, n_tokens)] in arrival order."""
        import torch.distributed as dist
        sched = [ScheduledRequest(str(i), float(i), "m", cfg, n_layers) for i, (_, cfg, _) in enumerate(requests)]
        per_dst: dict = {}
        for job in link_order(sched):
            dst, _, n = requests[job.request]
            kinds = 1 if job.kind == "e" else 2  # E, or K then V
            per_dst.setdefault(dst, []).extend((job, n, part) for part in range(kinds))
        queues = list(per_dst.items())
        for i in range(max((len(q) for _, q in queues), default=0)):
            ops = []
            for dst, q in queues:
                if i < len(q):
                    job, n, part = q[i]
                    ops.append(dist.P2POp(dist.isend, job_tensor(prefill, job, n - 1, part), dst, group=self.group))
            for w in dist.batch_isend_irecv(ops):
                w.wait()


class NcclTransport:
    """Consumer side, used by :class:`~.pipeline.ConsumerPipeline`: each job is a
    recv into a staging slot on the link stream, then (KV) an ingest from it.
    The producer holds every job's payload (it serves the same link order), so
    the consumer has no local sender caches to validate."""

    provides_all = True

    def __init__(self, src_rank: int, config, n_tokens: int, device, group=None, slots: int = 2,
                 ingest=None):
        self.src, self.group = src_rank, group
        P = n_tokens - 1
        G, D = config.n_kv_heads, config.head_dim
        self.window = P
        self.slots = [(torch.empty(G, P, D, dtype=torch.bfloat16, device=device),
                       torch.empty(G, P, D, dtype=torch.bfloat16, device=device)) for _ in range(slots)]
        self.e_stage = {}
        self.d_model = config.d_model
        self.device = device
        self._next = 0
        self._ingest = ingest or _ingest_slot

    def _recv(self, t: torch.Tensor) -> None:
        import torch.distributed as dist
        dist.recv(t, self.src, group=self.group)

    def e_job(self, layer: int, e, link):
        buf = self.e_stage.get(layer)
        if buf is None:
            buf = torch.empty(self.window, self.d_model, dtype=torch.float32, device=self.device)
            self.e_stage[layer] = buf
        with torch.cuda.stream(link) if link is not None else _null():
            self._recv(buf)
        return buf

    def kv_job(self, layer: int, src_desc, dst_desc, window, cfg, link):
        k, v = self.slots[self._next]
        self._next = (self._next + 1) % len(self.slots)
        with torch.cuda.stream(link) if link is not None else _null():
            self._recv(k)
            self._recv(v)
            self._ingest(layer, k, v, dst_desc, window, cfg, link)


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def _ingest_slot(layer, k, v, dst_desc, window, cfg, link):
    """Ingest one staged layer: a per-layer pointer table with only ``layer`` set."""
    n_l = max(layer + 1, dst_desc.n_layers)
    ka = (C.c_void_p * n_l)()
    va = (C.c_void_p * n_l)()
    ka[layer], va[layer] = k.data_ptr(), v.data_ptr()
    G, P, D = k.shape
    src = L.KvCache(k.data_ptr(), v.data_ptr(), 0, P * D, PAGE * D, None, n_l, P)
    src.layer_k, src.layer_v = ka, va
    arr = (C.c_int32 * 1)(layer)
    miss = C.c_int32(-1)
    rc = L.lib().ds_kv_ingest(C.byref(src), C.byref(dst_desc), arr, 1, window, cfg.n_kv_heads, cfg.head_dim,
                              link.cuda_stream, C.byref(miss))
    L.check(rc, miss.value, 1)


# ---------------------------------------------------------------------------
# Broadcast fan-out (collectives; NVLS multicast on NVSwitch)
# ---------------------------------------------------------------------------


def broadcast_export(prefill: PrefillResult | None, src: int, config, n_tokens: int, e_layers, device,
                     layers=None, group=None):
    """One context's export from rank ``src`` to every rank of ``group``:
    E at ``e_layers`` first (it gates the recompute), then K and V of
    ``layers`` (default: all) ascending -- the planner's link order
    (sched.py:217-223) as collectives.  ``prefill`` is the producer's result on
    ``src`` (None elsewhere).  Returns ``(LayerKV, {layer: ECache})`` on every
    rank (the producer's own tensors on ``src``, fresh buffers elsewhere, with
    the producer's context tag); layers not broadcast stay zero on receivers."""
    import torch.distributed as dist
    from .engine import LayerKV
    rank = dist.get_rank(group) if group is not None else dist.get_rank()
    e_layers = sorted(set(int(l) for l in e_layers))
    layers = list(range(config.n_layers)) if layers is None else sorted(set(int(l) for l in layers))
    tag = [prefill.kv.context if rank == src else None]
    dist.broadcast_object_list(tag, src=src, group=group)
    if rank == src:
        kv = prefill.kv
        e = {l: prefill.e_map()[l].hidden for l in e_layers}
    else:
        kv = LayerKV.empty(config, n_tokens, device)
        e = {l: torch.empty(n_tokens - 1, config.d_model, dtype=torch.float32, device=device) for l in e_layers}
    for l in e_layers:
        dist.broadcast(e[l], src=src, group=group)
    for l in layers:
        dist.broadcast(kv.k[l], src=src, group=group)  # [KVH, n, D]: contiguous
        dist.broadcast(kv.v[l], src=src, group=group)
    kv.context = tag[0]
    return kv, {l: ECache(l, t) for l, t in e.items()}
