"""Generate golden fixtures by importing the REAL reference (crosskv 0.1.0).

Run in the build container only (``/root/reference`` is absent on GPU boxes):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes small ``.npz`` / ``.json`` files next to this script.  The oracle
(``oracle/crosskv_oracle.py``) and the host-side mirrors in the package are
pinned against these (``tests/test_oracle.py``, ``tests/test_host_*.py``).
"""

from __future__ import annotations

import json
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

REF = os.environ.get("CROSSKV_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from crosskv import model as M  # noqa: E402
from crosskv import profiler as PR  # noqa: E402
from crosskv import sched as S  # noqa: E402
from crosskv import sim as SIM  # noqa: E402
from crosskv import store as ST  # noqa: E402

OUT = Path(__file__).resolve().parent

# Fixture model shapes.  TOY = the reference test fixture (conftest.py:5-15),
# TINY = BASELINE config 1, MID = a head_dim-128 shape for the D=128 kernels.
SHAPES = {
    "toy": M.ModelConfig(8, 64, 4, 2, 16, 128, 256, 128, 7),
    "tiny": M.ModelConfig(4, 256, 4, 1, 64, 1024, 4096, 1024, 7),
    "mid": M.ModelConfig(2, 1024, 8, 2, 128, 2816, 8192, 1024, 11),
}


def _kv_digest(kv):
    """Size-independent summaries of a [L,G,n,D] cache (sum, abs-sum per layer)."""
    k = kv.k.astype(np.float64)
    v = kv.v.astype(np.float64)
    return np.stack([k.sum(axis=(1, 2, 3)), np.abs(k).sum(axis=(1, 2, 3)),
                     v.sum(axis=(1, 2, 3)), np.abs(v).sum(axis=(1, 2, 3))], axis=1)


def engine_fixtures():
    toy = SHAPES["toy"]
    base = M.build_model(toy)
    recv = M.build_model(toy, M.PerturbationSpec.block(8, [4, 5], 1.0, noise_seed=1000))
    toks = M.make_synthetic_dataset(42, 1, 40, toy.vocab_size)[0]
    full = M.full_prefill(base, toks)
    dec = M.decode_greedy(base, full.kv, full.logits, 32)
    part = M.partial_prefill(recv, toks, M.RecomputeConfig([(4, 5)]), full.kv, full.e_map())
    np.savez_compressed(
        OUT / "toy_engine.npz",
        tokens=toks, full_logits=full.logits, full_k=full.kv.k, full_v=full.kv.v,
        e2=full.e_map()[2].hidden, decode32=dec,
        part45_logits=part.logits, part45_k=part.kv.k, part45_v=part.kv.v,
        embed_row3=base.embed[3], wq0=base.layers[0].wq, w2_5_recv=recv.layers[5].w2,
    )

    tiny = SHAPES["tiny"]
    A = M.build_model(tiny)
    B = M.build_model(tiny, M.PerturbationSpec.block(4, [2], 0.5, 1000))
    rows = {"first_recv_full": [], "first_partial": [], "first_reuse_all": []}
    logits_partial, logits_full = [], []
    for i in range(16):
        t = M.make_synthetic_dataset(100 + i, 1, 512, tiny.vocab_size)[0]
        prod = M.full_prefill(A, t)
        cons = M.partial_prefill(B, t, M.RecomputeConfig([(2, 3)]), prod.kv, prod.e_map())
        own = M.full_prefill(B, t)
        reuse = M.partial_prefill(B, t, M.RecomputeConfig.none(), prod.kv, prod.e_map())
        rows["first_recv_full"].append(int(np.argmax(own.logits)))
        rows["first_partial"].append(int(np.argmax(cons.logits)))
        rows["first_reuse_all"].append(int(np.argmax(reuse.logits)))
        logits_partial.append(cons.logits)
        logits_full.append(own.logits)
        if i == 0:
            np.savez_compressed(
                OUT / "tiny_prefix0.npz", tokens=t, prod_logits=prod.logits,
                prod_kv_digest=_kv_digest(prod.kv), prod_e2=prod.e_map()[2].hidden[:8],
                cons_logits=cons.logits, cons_kv_digest=_kv_digest(cons.kv),
                cons_k_l3_head=cons.kv.k[3, :, :4], cons_k_anchor=cons.kv.k[:, :, -1],
            )
    np.savez_compressed(OUT / "tiny_16prefixes.npz",
                        logits_partial=np.stack(logits_partial), logits_full=np.stack(logits_full),
                        **{k: np.array(v) for k, v in rows.items()})

    mid = SHAPES["mid"]
    A = M.build_model(mid)
    B = M.build_model(mid, M.PerturbationSpec.block(2, [1], 0.5, 77))
    t = M.make_synthetic_dataset(9, 1, 384, mid.vocab_size)[0]
    prod = M.full_prefill(A, t)
    cons = M.partial_prefill(B, t, M.RecomputeConfig([(1, 1)]), prod.kv, prod.e_map())
    np.savez_compressed(OUT / "mid_engine.npz", tokens=t, prod_logits=prod.logits,
                        prod_kv_digest=_kv_digest(prod.kv), cons_logits=cons.logits,
                        cons_kv_digest=_kv_digest(cons.kv))


def profile_fixtures():
    """The reference profiler's recompute set for BASELINE config 1."""
    tiny = SHAPES["tiny"]
    A = M.build_model(tiny)
    B = M.build_model(tiny, M.PerturbationSpec.block(4, [2], 0.5, 1000))
    train = M.make_synthetic_dataset(5000, 4, 512, tiny.vocab_size)
    points = PR.run_profile(A, B, train, granularity=1, horizon=32)
    frontier = PR.build_frontier(points)
    art = PR.ProfileArtifact(pair=PR.PairMeta.from_weights(A, B), granularity=1, horizon=32,
                             points=tuple(points), frontier=frontier)
    PR.save_profile(art, OUT / "tiny_profile.json")
    chosen = PR.select_by_quality_floor(frontier)
    sel = {
        "floor_default": [list(g) for g in chosen.groups],
        "floor": {str(d): [list(g) for g in PR.select_by_quality_floor(frontier, d).groups]
                  for d in (0.0, 0.01, 0.05, 0.1, 0.2, 0.5, 1.0)},
        "budget": {str(b): [list(g) for g in PR.select_by_layer_budget(frontier, b).groups]
                   for b in range(0, 6)},
        "frontier": [[e.k, e.quality, [list(g) for g in e.config.groups]] for e in frontier.entries],
        "baseline_quality": frontier.baseline_quality,
    }
    # Random frontier cases (rng-generated points) for build_frontier parity.
    rng = np.random.default_rng(31)
    cases = []
    for _ in range(40):
        L = int(rng.integers(2, 12))
        g = int(rng.integers(1, L + 1))
        pts = []
        for cfg in PR.enumerate_groups(L, g):
            if cfg.is_full(L):
                q = 1.0
            else:
                q = float(np.round(rng.uniform(0, 1), 3)) if rng.random() < 0.9 else 1.0
            pts.append([cfg.groups[0][0], cfg.groups[0][1], q])
        ppts = [PR.ProfilePoint(M.RecomputeConfig([(a, b)]), b - a + 1, q) for a, b, q in pts]
        try:
            fr = PR.build_frontier(ppts)
            res = {"entries": [[e.k, e.quality, list(e.config.groups[0])] for e in fr.entries],
                   "floor": {str(d): list(PR.select_by_quality_floor(fr, d).groups)
                             for d in (0.0, 0.05, 0.3)},
                   "budget": {str(b): [list(x) for x in PR.select_by_layer_budget(fr, b).groups]
                              for b in range(0, L + 1)}}
        except ValueError as exc:
            res = {"error": str(exc)}
        cases.append({"n_layers": L, "granularity": g, "points": pts, "result": res,
                      "n_configs": len(PR.enumerate_groups(L, g))})
    sel["random_cases"] = cases
    (OUT / "selection.json").write_text(json.dumps(sel, indent=1, sort_keys=True) + "\n")


def config_and_hash_fixtures():
    rng = np.random.default_rng(5)
    norm = []
    for _ in range(200):
        n = int(rng.integers(0, 6))
        groups = []
        for _ in range(n):
            a, b = sorted(int(x) for x in rng.integers(0, 40, size=2))
            groups.append([a, b])
        cfg = M.RecomputeConfig(groups)
        L = int(rng.integers(1, 48))
        try:
            cfg.validate_for(L)
            valid = True
        except ValueError:
            valid = False
        norm.append({"in": groups, "groups": [list(g) for g in cfg.groups], "L": L,
                     "valid": valid, "transition": list(cfg.transition_layers),
                     "reused": list(cfg.reused_layers(L)), "k": cfg.recomputed_layer_count})
    hashes = []
    for n in (0, 1, 2, 40, 512, 8192):
        t = np.random.default_rng(n + 1).integers(0, 128256, size=n)
        hashes.append({"tokens_seed": n + 1, "n": n, "digest": ST.context_hash(t).digest})
    doc = {"normal_forms": norm, "hashes": hashes, "golden_decode": [
        68, 145, 7, 145, 7, 145, 7, 145, 7, 185, 138, 96, 253, 145, 7, 21,
        96, 253, 253, 145, 7, 146, 110, 138, 96, 253, 145, 7, 21, 96, 253, 145]}
    (OUT / "config_hash.json").write_text(json.dumps(doc, indent=1, sort_keys=True) + "\n")


def sched_fixtures():
    def dump(tl):
        return {"events": [[e.request, e.resource, e.label, e.start, e.end] for e in tl.events],
                "ttft": tl.ttft, "ready": tl.ready}

    cost, reqs = S.demo_scenario()
    out = {"demo": {s: dump(S.plan(s, reqs, cost)) for s in S.STRATEGIES}}
    rng = np.random.default_rng(2024)
    rand = []
    for _ in range(60):
        n_models = int(rng.integers(1, 4))
        n_req = int(rng.integers(1, 7))
        arrivals = np.sort(rng.uniform(0, 20, size=n_req))
        rq = []
        for i in range(n_req):
            L = int(rng.integers(4, 17))
            groups, cur = [], 0
            while cur < L and rng.random() < 0.7:
                a = int(rng.integers(cur, L))
                b = int(rng.integers(a, L))
                groups.append((a, b))
                cur = b + 2
            rq.append(S.ScheduledRequest(f"r{i}", float(arrivals[i]), f"m{int(rng.integers(0, n_models))}",
                                         M.RecomputeConfig(groups), L))
        if rng.random() < 0.5:
            c = S.CostModel.unit()
        else:
            c = S.CostModel(link_bandwidth=float(rng.uniform(0.5, 8.0)),
                            kv_layer_bytes=float(rng.uniform(0.5, 4.0)),
                            e_layer_bytes=float(rng.uniform(0.5, 8.0)),
                            layer_compute_time=float(rng.uniform(0.2, 3.0)),
                            anchor_time=float(rng.uniform(0.0, 1.0)))
        rand.append({
            "cost": [c.link_bandwidth, c.kv_layer_bytes, c.e_layer_bytes, c.layer_compute_time,
                     c.anchor_time, c.unit_mode],
            "requests": [[r.id, r.arrival, r.model, [list(g) for g in r.config.groups], r.n_layers]
                         for r in rq],
            "plans": {s: dump(S.plan(s, rq, c)) for s in S.STRATEGIES},
        })
    out["random"] = rand
    cfg = M.ModelConfig(32, 4096, 32, 8, 128, 14336, 128256, 32768, 0)
    out["cost_from_model_8b"] = list(vars(S.CostModel.from_model(cfg, 8191, 770e9, 1e-9)).values())
    (OUT / "sched.json").write_text(json.dumps(out, indent=0, sort_keys=True) + "\n")


def adapt_fixtures():
    """sim.adapt_config (sim.py:171-202) on random frontiers, policies, backlogs
    and cost models: the SLO-adaptive recompute-set choice."""
    rng = np.random.default_rng(77)
    cases = []
    for _ in range(80):
        L = int(rng.integers(4, 13))
        g = int(rng.integers(1, 3))
        pts = []
        for cfg in PR.enumerate_groups(L, g):
            pts.append({"groups": [list(x) for x in cfg.groups], "k": cfg.recomputed_layer_count,
                        "quality": 1.0 if cfg.is_full(L) else round(float(rng.uniform(0, 1)), 4)})
        points = [PR.ProfilePoint(M.RecomputeConfig(p["groups"]), p["k"], p["quality"]) for p in pts]
        frontier = PR.build_frontier(points)
        if rng.random() < 0.5:
            cost = S.CostModel.unit()
        else:
            cost = S.CostModel(link_bandwidth=float(rng.uniform(0.5, 8.0)), kv_layer_bytes=float(rng.uniform(0.5, 4.0)),
                               e_layer_bytes=float(rng.uniform(0.5, 8.0)),
                               layer_compute_time=float(rng.uniform(0.2, 3.0)),
                               anchor_time=float(rng.uniform(0.0, 1.0)))
        policy = SIM.SloPolicy(slo=float(rng.uniform(0.5, 40.0)), q_min=float(rng.uniform(0, 1)),
                               adaptation_enabled=bool(rng.random() < 0.8))
        qd = int(rng.integers(0, 3)) if rng.random() < 0.4 else 0
        req = S.ScheduledRequest("r0", 0.0, "m0", M.RecomputeConfig.full(L), L)
        dec = SIM.adapt_config(qd, req, frontier, policy, cost)
        cases.append({"L": L, "points": pts,
                      "cost": [cost.link_bandwidth, cost.kv_layer_bytes, cost.e_layer_bytes,
                               cost.layer_compute_time, cost.anchor_time, cost.unit_mode],
                      "policy": [policy.slo, policy.q_min, policy.adaptation_enabled], "queue_depth": qd,
                      "decision": {"groups": [list(x) for x in dec.config.groups], "k": dec.k,
                                   "quality": dec.quality, "slo_feasible": dec.slo_feasible}})
    (OUT / "adapt.json").write_text(json.dumps({"cases": cases}, indent=0, sort_keys=True) + "\n")


def store_fixtures():
    """Serving-mode filter and fetch assembly on TOY (store.py:199-221, 351-395)."""
    toy = SHAPES["toy"]
    base = M.build_model(toy)
    toks = M.make_synthetic_dataset(42, 1, 40, toy.vocab_size)[0]
    res = M.full_prefill(base, toks)
    out = {}
    for groups in ([(0, 1), (4, 5)], [(4, 5)], [], [(0, 7)], [(3, 3), (6, 7)]):
        cfg = M.RecomputeConfig(groups)
        st = ST.CacheStore(mode="serving", transition_layers=cfg.transition_layers)
        total = ST.store_prefill(st, base.ident, toks, res)
        kv, e_map = ST.fetch_context_caches(st, base.ident, toks, cfg, 8)
        out[str(groups)] = {
            "total": total,
            "kv_layers": sorted(k.layer for k in st.keys() if k.kind == "kv"),
            "e_layers": sorted(k.layer for k in st.keys() if k.kind == "e"),
            "fetched_e": sorted(e_map),
            "kv_positions": None if kv is None else kv.positions,
        }
    out["ident_base"] = base.ident
    out["ident_var"] = M.build_model(toy, M.PerturbationSpec.block(8, [4, 5], 1.0, 1000)).ident
    with tempfile.TemporaryDirectory() as d:
        st = ST.CacheStore(mode="serving", transition_layers=(4,), config=toy)
        ST.store_prefill(st, base.ident, toks, res)
        st.save_snapshot(d)
        out["snapshot_index"] = json.loads((Path(d) / "index.json").read_text())
    (OUT / "store.json").write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")


def selective_fixtures():
    """token_selective_prefill (model.py:682-743) on the toy fixture and on
    TINY (receiver perturbed at layers 0 and 2): logits, the selection (the
    layer-0 positions whose K differs from the sender's) and cache digests."""
    out = {}
    toy = SHAPES["toy"]
    base = M.build_model(toy)
    recv = M.build_model(toy, M.PerturbationSpec.block(8, [4, 5], 1.0, noise_seed=1000))
    toks = M.make_synthetic_dataset(42, 1, 40, toy.vocab_size)[0]
    full = M.full_prefill(base, toks)
    for r in (0.25, 1.0):
        sel = M.token_selective_prefill(recv, toks, full.kv, r)
        out[f"toy_r{int(r * 100)}_logits"] = sel.logits
        out[f"toy_r{int(r * 100)}_k"] = sel.kv.k
        out[f"toy_r{int(r * 100)}_v"] = sel.kv.v
    tiny = SHAPES["tiny"]
    A = M.build_model(tiny)
    B = M.build_model(tiny, M.PerturbationSpec.block(4, [0, 2], 0.5, 1000))  # layer 0 differs: real deviations
    t = M.make_synthetic_dataset(100, 1, 512, tiny.vocab_size)[0]
    prod = M.full_prefill(A, t)
    sel = M.token_selective_prefill(B, t, prod.kv, 0.15)
    P = len(t) - 1
    chosen = np.flatnonzero(np.any(sel.kv.k[0, :, :P] != prod.kv.k[0, :, :P], axis=(0, 2)))
    out.update(toy_tokens=toks, tiny_tokens=t, tiny_r15_logits=sel.logits, tiny_r15_selected=chosen,
               tiny_r15_kv_digest=_kv_digest(sel.kv))
    np.savez_compressed(OUT / "selective.npz", **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["config", "sched", "store", "engine", "profile", "selective", "adapt"]
    if "config" in which:
        config_and_hash_fixtures()
    if "sched" in which:
        sched_fixtures()
    if "store" in which:
        store_fixtures()
    if "engine" in which:
        engine_fixtures()
    if "profile" in which:
        profile_fixtures()
    if "selective" in which:
        selective_fixtures()
    if "adapt" in which:
        adapt_fixtures()
    print("wrote", sorted(p.name for p in OUT.iterdir() if p.suffix in (".npz", ".json")))
