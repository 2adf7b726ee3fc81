"""Transfer/recompute planning semantics (the spec the CUDA scheduler realises).

Mirror of ``crosskv.sched`` (sched.py:34-47): a link carries per-layer
transfer jobs, each model owns one compute resource that rebuilds one layer
at a time, the anchor closes a request.

    CostModel / CostModel.from_model     sched.py:54-112
    bytes_of                             sched.py:115-123
    plan("naive"|"reuse_only"|"pipelined") sched.py:185-276
    estimate_ttft                        sched.py:279-281
    SloPolicy, AdaptDecision, adapt_config   sim.py:84-104, 171-202
    demo_scenario                        sched.py:358-369 (Fig. 9: totals 47 / 30 / 17)

The pipelined plan fixes the ORDER the GPU scheduler
(:mod:`paper_2411_02820_b200.pipeline`) issues work in: link jobs FIFO by
(arrival, request, E before KV, layer); a group's first recompute waits for
its seeding E (layer-0 groups start at arrival); the anchor waits for every
transfer and recompute of its request.  ``CostModel.from_measured`` turns
measured per-layer B200 times into a cost model so ``estimate_ttft`` predicts
the device pipeline (tested against measured TTFT in the bench).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

from .config import ModelConfig, RecomputeConfig

STRATEGIES = ("naive", "reuse_only", "pipelined")
LINK = "link"


@dataclass(frozen=True)
class CostModel:
    link_bandwidth: float = 1.0
    kv_layer_bytes: float = 1.0
    e_layer_bytes: float = 1.0
    layer_compute_time: float = 1.0
    anchor_time: float = 0.0
    unit_mode: bool = False

    def __post_init__(self) -> None:
        for f in ("link_bandwidth", "kv_layer_bytes", "e_layer_bytes", "layer_compute_time"):
            if getattr(self, f) <= 0:
                raise ValueError(f"{f} must be positive")
        if self.anchor_time < 0:
            raise ValueError("anchor_time must be non-negative")
        if self.unit_mode and (self.link_bandwidth, self.kv_layer_bytes, self.e_layer_bytes,
                               self.layer_compute_time, self.anchor_time) != (1.0, 1.0, 1.0, 1.0, 0.0):
            raise ValueError("unit mode fixes all per-layer costs at 1 and anchor at 0")

    @classmethod
    def unit(cls) -> "CostModel":
        return cls(unit_mode=True)

    @classmethod
    def from_model(cls, config: ModelConfig, positions: int, link_bandwidth: float,
                   compute_time_per_layer_position: float) -> "CostModel":
        """Byte sizes from the reference's float32 byte laws (sched.py:86-104)."""
        return cls(link_bandwidth=link_bandwidth,
                   kv_layer_bytes=float(bytes_of("kv", positions, config)),
                   e_layer_bytes=float(bytes_of("e", positions, config)),
                   layer_compute_time=compute_time_per_layer_position * positions,
                   anchor_time=compute_time_per_layer_position * config.n_layers)

    @classmethod
    def from_measured(cls, config: ModelConfig, positions: int, link_gbs: float, layer_ms: float,
                      anchor_ms: float, dtype_bytes: int = 2) -> "CostModel":
        """Cost model in milliseconds of the B200 path: bf16 KV and f32 E byte
        sizes, a link of ``link_gbs`` GB/s (NVLink P2P, or HBM for a same-GPU
        ingest), and the measured recompute time per layer and anchor pass time."""
        kv = 2 * config.n_kv_heads * config.head_dim * dtype_bytes * positions
        e = config.d_model * 4 * positions
        return cls(link_bandwidth=link_gbs * 1e6, kv_layer_bytes=float(kv), e_layer_bytes=float(e),
                   layer_compute_time=layer_ms, anchor_time=anchor_ms)

    @property
    def kv_transfer_time(self) -> float:
        return self.kv_layer_bytes / self.link_bandwidth

    @property
    def e_transfer_time(self) -> float:
        return self.e_layer_bytes / self.link_bandwidth


def bytes_of(kind: str, positions: int, config: ModelConfig) -> int:
    if positions < 1:
        raise ValueError("positions must be at least 1")
    per = {"kv": config.kv_bytes_per_position, "e": config.e_bytes_per_position}.get(kind)
    if per is None:
        raise ValueError(f"unknown cache kind {kind!r}")
    return per * positions


@dataclass(frozen=True)
class ScheduledRequest:
    id: str
    arrival: float
    model: str
    config: RecomputeConfig
    n_layers: int

    def __post_init__(self) -> None:
        if self.arrival < 0:
            raise ValueError("arrival must be non-negative")
        self.config.validate_for(self.n_layers)

    @property
    def reused_layers(self) -> tuple:
        return self.config.reused_layers(self.n_layers)


@dataclass(frozen=True)
class Event:
    request: str
    resource: str
    label: str
    start: float
    end: float


@dataclass(frozen=True)
class Timeline:
    events: tuple
    ready: dict
    ttft: dict

    @property
    def total_ttft(self) -> float:
        return sum(self.ttft.values())


@dataclass(frozen=True)
class LinkJob:
    """One per-layer transfer in link order: kind "e" (seeding hidden state of a
    transition layer) or "kv" (a reused layer's K/V)."""

    request: int
    kind: str
    layer: int


def link_order(requests: Sequence[ScheduledRequest]) -> list:
    """FIFO order of the link (sched.py:217-223): by arrival, then request
    order, E before KV, ascending layer."""
    keyed = []
    for i, r in enumerate(requests):
        keyed += [((r.arrival, i, 0, a), LinkJob(i, "e", a)) for a in r.config.transition_layers]
        keyed += [((r.arrival, i, 1, l), LinkJob(i, "kv", l)) for l in r.reused_layers]
    keyed.sort(key=lambda x: x[0])
    return [j for _, j in keyed]


def _label(job: LinkJob) -> str:
    return f"{'E' if job.kind == 'e' else 'KV'}-transfer({job.layer})"


def _serial(requests, cost: CostModel, every_layer_kv: bool) -> Timeline:
    ev, ready, ttft = [], {}, {}
    t_free = 0.0
    for r in requests:
        t = max(r.arrival, t_free)
        comp = f"compute:{r.model}"
        steps = [(LINK, f"E-transfer({a})", cost.e_transfer_time) for a in r.config.transition_layers]
        kv_layers = range(r.n_layers) if every_layer_kv else r.reused_layers
        steps += [(LINK, f"KV-transfer({l})", cost.kv_transfer_time) for l in kv_layers]
        steps += [(comp, f"recompute({l})", cost.layer_compute_time)
                  for a, b in r.config.groups for l in range(a, b + 1)]
        steps.append((comp, "anchor", cost.anchor_time))
        for res, lab, dur in steps:
            ev.append(Event(r.id, res, lab, t, t + dur))
            t += dur
        ready[r.id], ttft[r.id] = t, t - r.arrival
        t_free = t
    return Timeline(tuple(ev), ready, ttft)


def _pipelined(requests, cost: CostModel) -> Timeline:
    ev = []
    e_landed: dict = {}
    last_xfer = {i: r.arrival for i, r in enumerate(requests)}
    link_t = 0.0
    for job in link_order(requests):
        r = requests[job.request]
        start = max(link_t, r.arrival)
        link_t = start + (cost.e_transfer_time if job.kind == "e" else cost.kv_transfer_time)
        ev.append(Event(r.id, LINK, _label(job), start, link_t))
        last_xfer[job.request] = max(last_xfer[job.request], link_t)
        if job.kind == "e":
            e_landed[(job.request, job.layer)] = link_t
    free: dict = {}
    ready, ttft = {}, {}
    for i, r in enumerate(requests):
        comp = f"compute:{r.model}"
        t = free.get(comp, 0.0)
        done = r.arrival
        for a, b in r.config.groups:
            gate = r.arrival if a == 0 else e_landed[(i, a)]
            for l in range(a, b + 1):
                s = max(t, gate, r.arrival)
                t = s + cost.layer_compute_time
                ev.append(Event(r.id, comp, f"recompute({l})", s, t))
                done = t
        s = max(t, last_xfer[i], done)
        t = s + cost.anchor_time
        ev.append(Event(r.id, comp, "anchor", s, t))
        free[comp] = t
        ready[r.id], ttft[r.id] = t, t - r.arrival
    return Timeline(tuple(ev), ready, ttft)


def plan(strategy: str, requests: Sequence[ScheduledRequest], cost: CostModel) -> Timeline:
    if strategy not in STRATEGIES:
        raise ValueError(f"unknown strategy {strategy!r}; expected one of {STRATEGIES}")
    requests = list(requests)
    if any(requests[i + 1].arrival < requests[i].arrival for i in range(len(requests) - 1)):
        raise ValueError("requests must be sorted by arrival time")
    ids = [r.id for r in requests]
    if len(set(ids)) != len(ids):
        dup = next(x for x in ids if ids.count(x) > 1)
        raise ValueError(f"duplicate request id {dup!r}")
    if strategy == "pipelined":
        return _pipelined(requests, cost)
    return _serial(requests, cost, every_layer_kv=strategy == "naive")


def estimate_ttft(request: ScheduledRequest, cost: CostModel) -> float:
    """Solitary pipelined TTFT (sched.py:279-281)."""
    return plan("pipelined", [request], cost).ttft[request.id]


def demo_scenario():
    """Fig. 9 two-request handoff (unit costs, 10 layers, arrivals 0 and 2)."""
    return CostModel.unit(), [
        ScheduledRequest("A", 0.0, "A", RecomputeConfig([(3, 9)]), 10),
        ScheduledRequest("B", 2.0, "B", RecomputeConfig([(0, 2)]), 10),
    ]


# ---------------------------------------------------------------------------
# SLO-adaptive recompute-set choice (sim.py:84-104, 171-202)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class SloPolicy:
    slo: float
    q_min: float
    adaptation_enabled: bool = True

    def __post_init__(self) -> None:
        if self.slo <= 0:
            raise ValueError("slo must be positive")
        if not 0.0 <= self.q_min <= 1.0:
            raise ValueError("q_min must lie in [0, 1]")


@dataclass(frozen=True)
class AdaptDecision:
    config: RecomputeConfig
    k: int
    quality: float
    slo_feasible: bool


def adapt_config(queue_depth: int, request: ScheduledRequest, frontier, policy: SloPolicy,
                 cost: CostModel) -> AdaptDecision:
    """Pick a Pareto-frontier entry for one request given the replica's backlog
    (sim.py:171-202).  Candidates: entries meeting q_min (else the terminal
    recompute-all entry).  Loaded (queue_depth > 0) or adaptation off: the
    cheapest candidate.  Idle: the largest candidate whose solitary pipelined
    TTFT (estimate_ttft) fits the SLO, else the cheapest, flagged infeasible.
    With ``CostModel.from_measured`` the TTFTs are the B200's measured times."""
    qualifying = [e for e in frontier.entries if e.quality >= policy.q_min]
    if not qualifying:
        qualifying = [frontier.entries[-1]]
    if not policy.adaptation_enabled or queue_depth > 0:
        chosen = qualifying[0]
        return AdaptDecision(chosen.config, chosen.k, chosen.quality, True)
    best = None
    for entry in qualifying:
        trial = ScheduledRequest(request.id, 0.0, request.model, entry.config, request.n_layers)
        if estimate_ttft(trial, cost) <= policy.slo:
            best = entry  # entries ascend in k: the last fit is the largest
    if best is not None:
        return AdaptDecision(best.config, best.k, best.quality, True)
    chosen = qualifying[0]
    return AdaptDecision(chosen.config, chosen.k, chosen.quality, False)
