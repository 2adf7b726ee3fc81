"""Host-side mirrors of the reference boundary, pinned to golden fixtures (CPU only).

* recompute-layer sets: RecomputeConfig normal form (model.py:155-211)
* selection: build_frontier / select_* / profile artifact (profiler.py:109-413)
* planner semantics: plan / estimate_ttft / CostModel (sched.py:54-281)
* store: context_hash, serving-mode filter, store_prefill / fetch_context_caches,
  snapshot index (store.py:55-395)

Every fixture under tests/golden/ was produced by the real reference
(tests/golden/make_golden.py); results must match bit-exactly.
"""

import json

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from oracle import crosskv_oracle as O

import paper_2411_02820_b200 as P
from paper_2411_02820_b200 import planner as S
from paper_2411_02820_b200 import selection as SEL
from paper_2411_02820_b200 import store as ST


@pytest.fixture(scope="module")
def cfg_hash():
    return json.loads((GOLDEN / "config_hash.json").read_text())


def test_recompute_config_normal_forms(cfg_hash):
    for case in cfg_hash["normal_forms"]:
        rc = P.RecomputeConfig(case["in"])
        assert [list(g) for g in rc.groups] == case["groups"]
        try:
            rc.validate_for(case["L"])
            valid = True
        except ValueError:
            valid = False
        assert valid == case["valid"]
        assert list(rc.transition_layers) == case["transition"]
        assert list(rc.reused_layers(case["L"])) == case["reused"]
        assert rc.recomputed_layer_count == case["k"]


def test_context_hash_golden(cfg_hash):
    for h in cfg_hash["hashes"]:
        t = np.random.default_rng(h["tokens_seed"]).integers(0, 128256, size=h["n"])
        assert ST.context_hash(t).digest == h["digest"]
        assert ST.context_hash(torch.from_numpy(t)).digest == h["digest"]
    with pytest.raises(ValueError):
        ST.context_hash([-1, 2])


def test_model_ident_matches_reference():
    st = json.loads((GOLDEN / "store.json").read_text())
    toy = P.ModelConfig(8, 64, 4, 2, 16, 128, 256, 128, 7)
    assert P.model_ident(toy, None) == st["ident_base"]
    assert P.model_ident(toy, P.PerturbationSpec.block(8, [4, 5], 1.0, 1000)) == st["ident_var"]


# ---------------------------------------------------------------------------
# selection
# ---------------------------------------------------------------------------


@pytest.fixture(scope="module")
def sel_fx():
    return json.loads((GOLDEN / "selection.json").read_text())


def test_config1_selection_from_reference_profile(sel_fx, tmp_path):
    art = SEL.load_profile(GOLDEN / "tiny_profile.json")
    fr = art.frontier
    assert [[e.k, e.quality, [list(g) for g in e.config.groups]] for e in fr.entries] == sel_fx["frontier"]
    assert fr.baseline_quality == sel_fx["baseline_quality"]
    assert [list(g) for g in SEL.select_by_quality_floor(fr).groups] == sel_fx["floor_default"] == [[2, 3]]
    for d, want in sel_fx["floor"].items():
        assert [list(g) for g in SEL.select_by_quality_floor(fr, float(d)).groups] == want
    for b, want in sel_fx["budget"].items():
        assert [list(g) for g in SEL.select_by_layer_budget(fr, int(b)).groups] == want
    # re-saving is byte-identical (deterministic artifact, test_profiler.py byte-determinism)
    out = tmp_path / "p.json"
    SEL.save_profile(art, out)
    assert out.read_text() == (GOLDEN / "tiny_profile.json").read_text()
    assert SEL.recompute_config_from_profile(GOLDEN / "tiny_profile.json").groups == ((2, 3),)


def test_frontier_random_cases(sel_fx):
    for case in sel_fx["random_cases"]:
        L, g = case["n_layers"], case["granularity"]
        assert len(SEL.enumerate_groups(L, g)) == case["n_configs"]
        pts = [SEL.ProfilePoint(P.RecomputeConfig([(a, b)]), b - a + 1, q) for a, b, q in case["points"]]
        res = case["result"]
        if "error" in res:
            with pytest.raises(ValueError):
                SEL.build_frontier(pts)
            continue
        fr = SEL.build_frontier(pts)
        assert [[e.k, e.quality, list(e.config.groups[0])] for e in fr.entries] == res["entries"]
        for d, want in res["floor"].items():
            assert [list(x) for x in SEL.select_by_quality_floor(fr, float(d)).groups] == want
        for b, want in res["budget"].items():
            assert [list(x) for x in SEL.select_by_layer_budget(fr, int(b)).groups] == want


def test_enumerate_groups_counts():
    assert len(SEL.enumerate_groups(8, 2)) == 10
    assert len(SEL.enumerate_groups(32, 2)) == 136
    with pytest.raises(ValueError):
        SEL.enumerate_groups(4, 0)


def test_load_profile_schema_errors(tmp_path):
    doc = json.loads((GOLDEN / "tiny_profile.json").read_text())
    for field, mutate in [("version", lambda d: d.update(version=2)),
                          ("pair.n_heads", lambda d: d["pair"].pop("n_heads")),
                          ("points[0]", lambda d: d["points"][0].update(quality=1.5)),
                          ("frontier", lambda d: d["frontier"].reverse())]:
        bad = json.loads(json.dumps(doc))
        mutate(bad)
        p = tmp_path / "bad.json"
        p.write_text(json.dumps(bad))
        with pytest.raises(P.SchemaError) as err:
            SEL.load_profile(p)
        assert err.value.field == field


# ---------------------------------------------------------------------------
# planner semantics
# ---------------------------------------------------------------------------


@pytest.fixture(scope="module")
def sched_fx():
    return json.loads((GOLDEN / "sched.json").read_text())


def _dump(tl):
    return {"events": [[e.request, e.resource, e.label, e.start, e.end] for e in tl.events],
            "ttft": tl.ttft, "ready": tl.ready}


def test_demo_scenario_golden(sched_fx):
    cost, reqs = S.demo_scenario()
    totals = {}
    for s in S.STRATEGIES:
        tl = S.plan(s, reqs, cost)
        assert _dump(tl) == sched_fx["demo"][s]
        totals[s] = tl.total_ttft
    assert totals == {"naive": 47, "reuse_only": 30, "pipelined": 17}


def test_random_scenarios_golden(sched_fx):
    for case in sched_fx["random"]:
        bw, kvb, eb, lct, at, unit = case["cost"]
        cost = S.CostModel.unit() if unit else S.CostModel(bw, kvb, eb, lct, at)
        reqs = [S.ScheduledRequest(i, a, m, P.RecomputeConfig(g), L) for i, a, m, g, L in case["requests"]]
        for s in S.STRATEGIES:
            got = _dump(S.plan(s, reqs, cost))
            want = case["plans"][s]
            assert got["events"] == want["events"]
            assert got["ttft"] == want["ttft"] and got["ready"] == want["ready"]
        for r in reqs:
            assert S.estimate_ttft(r, cost) == S.plan("pipelined", [r], cost).ttft[r.id]


def test_cost_from_model_golden(sched_fx):
    cfg = P.ModelConfig(32, 4096, 32, 8, 128, 14336, 128256, 32768, 0)
    c = S.CostModel.from_model(cfg, 8191, 770e9, 1e-9)
    assert [c.link_bandwidth, c.kv_layer_bytes, c.e_layer_bytes, c.layer_compute_time, c.anchor_time,
            c.unit_mode] == sched_fx["cost_from_model_8b"]
    m = S.CostModel.from_measured(cfg, 8191, 770.0, 2.3, 1.9)
    assert m.kv_layer_bytes == 2 * 8 * 128 * 2 * 8191 and m.e_layer_bytes == 4096 * 4 * 8191


def test_plan_rejects_bad_requests():
    cost, (a, b) = S.demo_scenario()
    with pytest.raises(ValueError):
        S.plan("pipelined", [b, a], cost)
    with pytest.raises(ValueError):
        S.plan("pipelined", [a, a], cost)
    with pytest.raises(ValueError):
        S.plan("eager", [a], cost)


# ---------------------------------------------------------------------------
# store (CPU tensors: the store logic is device-agnostic; f32 payloads give
# the reference's byte counts exactly, bf16 payloads half of them)
# ---------------------------------------------------------------------------


TOY = O.Dims(8, 64, 4, 2, 16, 128, 256, 128, 7)


@pytest.fixture(scope="module")
def toy_prefill():
    w = O.make_weights(TOY)
    toks = O.synthetic_tokens(42, 1, 40, 256)[0]
    k, v, e, logits = O.full_prefill(w, toks)
    kv = P.LayerKV(torch.from_numpy(k), torch.from_numpy(v))
    ecs = tuple(P.ECache(l, torch.from_numpy(e[l])) for l in sorted(e))
    return toks, P.PrefillResult(kv, ecs, torch.from_numpy(logits), torch.zeros(1, dtype=torch.int32))


@pytest.mark.parametrize("dtype,scale", [(torch.float32, 1), (torch.bfloat16, 2)])
def test_store_serving_filter_and_fetch(toy_prefill, dtype, scale):
    fx = json.loads((GOLDEN / "store.json").read_text())
    toks, pf = toy_prefill
    pf = P.PrefillResult(P.LayerKV(pf.kv.k.to(dtype), pf.kv.v.to(dtype)),
                         tuple(P.ECache(e.layer, e.hidden.to(dtype)) for e in pf.e_caches), pf.logits, pf.token_dev)
    ident = fx["ident_base"]
    for groups in ([(0, 1), (4, 5)], [(4, 5)], [], [(0, 7)], [(3, 3), (6, 7)]):
        want = fx[str(groups)]
        rc = P.RecomputeConfig(groups)
        st = ST.CacheStore(mode="serving", transition_layers=rc.transition_layers)
        assert ST.store_prefill(st, ident, toks, pf) * scale == want["total"]
        assert sorted(k.layer for k in st.keys() if k.kind == "kv") == want["kv_layers"]
        assert sorted(k.layer for k in st.keys() if k.kind == "e") == want["e_layers"]
        kv, e_map = ST.fetch_context_caches(st, ident, toks, rc, 8)
        assert sorted(e_map) == want["fetched_e"]
        assert (None if kv is None else kv.positions) == want["kv_positions"]
        if kv is not None:
            dense = kv.dense()
            for l in range(8):
                if l in rc.layer_set():
                    assert not dense.k[l].any()
                else:
                    assert torch.equal(dense.k[l], pf.kv.k[l]) and torch.equal(dense.v[l], pf.kv.v[l])


def test_fetch_misses_in_reference_order(toy_prefill):
    toks, pf = toy_prefill
    st = ST.CacheStore(mode="serving", transition_layers=(4,))
    ST.store_prefill(st, "m", toks, pf)
    with pytest.raises(P.CacheMissError) as err:
        ST.fetch_context_caches(st, "other", toks, P.RecomputeConfig([(4, 5)]), 8)
    assert (err.value.layer, err.value.kind) == (0, "kv")
    with pytest.raises(P.CacheMissError) as err:
        ST.fetch_context_caches(st, "m", toks, P.RecomputeConfig([(3, 5)]), 8)
    assert (err.value.layer, err.value.kind) == (3, "e")


def test_store_capacity_lru_and_immutability(toy_prefill):
    toks, pf = toy_prefill
    ctx = ST.context_hash(toks)
    sl = [ST.KVSlice(pf.kv.k[l], pf.kv.v[l]) for l in range(3)]
    size = sl[0].nbytes
    st = ST.CacheStore(capacity_bytes=2 * size)
    st.store(ST.CacheKey(ctx, "m", 0, "kv"), sl[0])
    st.store(ST.CacheKey(ctx, "m", 1, "kv"), sl[1])
    assert st.fetch(ST.CacheKey(ctx, "m", 0, "kv")) is not None  # touch 0 -> 1 is LRU
    st.store(ST.CacheKey(ctx, "m", 2, "kv"), sl[2])
    assert ST.CacheKey(ctx, "m", 1, "kv") not in st and ST.CacheKey(ctx, "m", 0, "kv") in st
    assert st.total_bytes == 2 * size
    with pytest.raises(P.CapacityError):
        ST.CacheStore(capacity_bytes=size - 1).store(ST.CacheKey(ctx, "m", 0, "kv"), sl[0])
    # the default store copies: mutating the producer buffer does not reach the store
    src = sl[0].k.clone()
    st2 = ST.CacheStore()
    st2.store(ST.CacheKey(ctx, "m", 0, "kv"), ST.KVSlice(src, sl[0].v))
    src.zero_()
    assert torch.equal(st2.fetch(ST.CacheKey(ctx, "m", 0, "kv")).k, sl[0].k)
    with pytest.raises(ValueError):
        st2.store(ST.CacheKey(ctx, "m", 3, "e"), pf.e_caches[2])
    assert st2.fetch(ST.CacheKey(ctx, "m", 5, "kv")) is None


def test_snapshot_index_matches_reference(toy_prefill, tmp_path):
    fx = json.loads((GOLDEN / "store.json").read_text())
    toks, pf = toy_prefill
    cfg = P.ModelConfig(8, 64, 4, 2, 16, 128, 256, 128, 7)
    st = ST.CacheStore(mode="serving", transition_layers=(4,), config=cfg)
    ST.store_prefill(st, fx["ident_base"], toks, pf)
    st.save_snapshot(tmp_path)
    idx = json.loads((tmp_path / "index.json").read_text())
    assert idx["entries"] == fx["snapshot_index"]["entries"]
    back = ST.CacheStore.load_snapshot(tmp_path, cfg, device="cpu", dtype=torch.float32)
    for key in st.keys():
        a, b = st.fetch(key), back.fetch(key)
        if key.kind == "kv":
            assert torch.equal(a.k, b.k) and torch.equal(a.v, b.v)
        else:
            assert torch.equal(a.hidden, b.hidden)
    idx["version"] = 9
    (tmp_path / "index.json").write_text(json.dumps(idx))
    with pytest.raises(P.SchemaError):
        ST.CacheStore.load_snapshot(tmp_path, cfg, device="cpu")


def test_adapt_config_golden():
    """SLO-adaptive choice over the Pareto frontier (sim.py:171-202): same
    decision as the reference on 80 random frontiers / policies / backlogs."""
    doc = json.loads((GOLDEN / "adapt.json").read_text())
    largest_pick = 0
    for case in doc["cases"]:
        L = case["L"]
        pts = [SEL.ProfilePoint(P.RecomputeConfig(p["groups"]), p["k"], p["quality"]) for p in case["points"]]
        fr = SEL.build_frontier(pts)
        bw, kvb, eb, lct, at, unit = case["cost"]
        cost = S.CostModel.unit() if unit else S.CostModel(link_bandwidth=bw, kv_layer_bytes=kvb, e_layer_bytes=eb,
                                                           layer_compute_time=lct, anchor_time=at)
        slo, qmin, on = case["policy"]
        req = S.ScheduledRequest("r0", 0.0, "m0", P.RecomputeConfig.full(L), L)
        dec = S.adapt_config(case["queue_depth"], req, fr, S.SloPolicy(slo, qmin, on), cost)
        want = case["decision"]
        assert [list(g) for g in dec.config.groups] == want["groups"]
        assert (dec.k, dec.quality, dec.slo_feasible) == (want["k"], want["quality"], want["slo_feasible"])
        largest_pick += dec.k > min(e.k for e in fr.entries if e.quality >= qmin) if any(
            e.quality >= qmin for e in fr.entries) else 0
    assert largest_pick > 0  # the idle path that trades latency for quality is exercised
    with pytest.raises(ValueError):
        S.SloPolicy(0.0, 0.5)
    with pytest.raises(ValueError):
        S.SloPolicy(1.0, 1.5)
