"""Pin the CPU oracle against the reference's golden vectors (CPU only).

The fixtures under tests/golden/ were produced by importing the real
reference (tests/golden/make_golden.py); these tests run everywhere.  The
``reference``-marked tests additionally compare live against the imported
reference and only run in the build container.
"""

import json

import numpy as np
import pytest

from oracle import crosskv_oracle as O
from conftest import GOLDEN

TOY = O.Dims(8, 64, 4, 2, 16, 128, 256, 128, 7)
TINY = O.Dims(4, 256, 4, 1, 64, 1024, 4096, 1024, 7)
MID = O.Dims(2, 1024, 8, 2, 128, 2816, 8192, 1024, 11)


@pytest.fixture(scope="module")
def toy_fx():
    return np.load(GOLDEN / "toy_engine.npz")


@pytest.fixture(scope="module")
def toy_base():
    return O.make_weights(TOY)


def test_weights_bitwise_match_reference_streams(toy_fx, toy_base):
    # model.py:251-253 / 300 / 314: same PCG64 streams -> bitwise-equal tensors
    assert np.array_equal(toy_base["embed"][3], toy_fx["embed_row3"])
    assert np.array_equal(toy_base["layers"][0]["wq"], toy_fx["wq0"])
    recv = O.make_weights(TOY, O.block_eps(8, [4, 5], 1.0), noise_seed=1000)
    assert np.array_equal(recv["layers"][5]["w2"], toy_fx["w2_5_recv"])
    assert np.array_equal(recv["layers"][3]["w1"], toy_base["layers"][3]["w1"])


def test_full_prefill_matches_reference(toy_fx, toy_base):
    k, v, e, logits = O.full_prefill(toy_base, toy_fx["tokens"])
    assert np.abs(logits - toy_fx["full_logits"]).max() <= 1e-5
    assert np.abs(k - toy_fx["full_k"]).max() <= 1e-5
    assert np.abs(v - toy_fx["full_v"]).max() <= 1e-5
    assert np.abs(e[2] - toy_fx["e2"]).max() <= 1e-5
    # layer-0 E is the embedding rows (test_model.py:127-132)
    assert np.array_equal(e[0], toy_base["embed"][toy_fx["tokens"][:-1]])


def test_golden_decode_known_answer(toy_fx, toy_base):
    # The reference's own known-answer vector (pkg/tests/test_model.py:23-26).
    golden = json.loads((GOLDEN / "config_hash.json").read_text())["golden_decode"]
    k, v, _, logits = O.full_prefill(toy_base, toy_fx["tokens"])
    toks = O.decode_greedy(toy_base, k, v, logits, 32)
    assert toks.tolist() == golden == toy_fx["decode32"].tolist()


def test_partial_prefill_matches_reference(toy_fx, toy_base):
    recv = O.make_weights(TOY, O.block_eps(8, [4, 5], 1.0), noise_seed=1000)
    k, v, e, _ = O.full_prefill(toy_base, toy_fx["tokens"])
    pk, pv, logits = O.partial_prefill(recv, toy_fx["tokens"], [(4, 5)], k, v, e)
    assert np.abs(logits - toy_fx["part45_logits"]).max() <= 1e-5
    assert np.abs(pk - toy_fx["part45_k"]).max() <= 1e-5
    assert np.abs(pv - toy_fx["part45_v"]).max() <= 1e-5
    # reused layers are exact copies of the sender window (model.py:602-603)
    P = len(toy_fx["tokens"]) - 1
    assert np.array_equal(pk[0, :, :P], k[0, :, :P])


def test_recompute_all_bitwise_equals_full(toy_fx, toy_base):
    k1, v1, _, l1 = O.full_prefill(toy_base, toy_fx["tokens"])
    k2, v2, l2 = O.partial_prefill(toy_base, toy_fx["tokens"], [(0, 7)], None, None, {})
    assert np.array_equal(l1, l2) and np.array_equal(k1, k2) and np.array_equal(v1, v2)


@pytest.mark.parametrize("groups", [[], [(2, 3)], [(0, 4)], [(1, 2), (5, 6)], [(0, 0), (7, 7)]])
def test_identity_reuse(toy_fx, toy_base, groups):
    k, v, e, logits = O.full_prefill(toy_base, toy_fx["tokens"])
    _, _, l2 = O.partial_prefill(toy_base, toy_fx["tokens"], groups, k, v, e)
    assert np.abs(l2 - logits).max() <= 1e-5
    assert O.first_token(l2) == O.first_token(logits)


def test_cache_miss_order(toy_fx, toy_base):
    k, v, e, _ = O.full_prefill(toy_base, toy_fx["tokens"])
    with pytest.raises(O.CacheMiss) as err:
        O.partial_prefill(toy_base, toy_fx["tokens"], [(0, 3)], None, None, {})
    assert (err.value.layer, err.value.kind) == (4, "kv")
    with pytest.raises(O.CacheMiss) as err:
        O.partial_prefill(toy_base, toy_fx["tokens"], [(4, 5)], k, v, {})
    assert (err.value.layer, err.value.kind) == (4, "e")


def test_tiny_config1_matches_reference():
    fx = np.load(GOLDEN / "tiny_prefix0.npz")
    A = O.make_weights(TINY)
    B = O.make_weights(TINY, O.block_eps(4, [2], 0.5), noise_seed=1000)
    k, v, e, lp = O.full_prefill(A, fx["tokens"])
    assert np.abs(lp - fx["prod_logits"]).max() <= 1e-4
    ck, cv, lc = O.partial_prefill(B, fx["tokens"], [(2, 3)], k, v, e)
    assert np.abs(lc - fx["cons_logits"]).max() <= 1e-4
    assert O.first_token(lc) == O.first_token(fx["cons_logits"])
    dig = np.stack([ck.astype(np.float64).sum(axis=(1, 2, 3)), np.abs(ck.astype(np.float64)).sum(axis=(1, 2, 3)),
                    cv.astype(np.float64).sum(axis=(1, 2, 3)), np.abs(cv.astype(np.float64)).sum(axis=(1, 2, 3))], 1)
    np.testing.assert_allclose(dig, fx["cons_kv_digest"], rtol=1e-5, atol=1e-2)
    assert np.abs(ck[:, :, -1] - fx["cons_k_anchor"]).max() <= 1e-5


def test_mid_head128_matches_reference():
    fx = np.load(GOLDEN / "mid_engine.npz")
    A = O.make_weights(MID)
    B = O.make_weights(MID, O.block_eps(2, [1], 0.5), noise_seed=77)
    k, v, e, lp = O.full_prefill(A, fx["tokens"])
    assert np.abs(lp - fx["prod_logits"]).max() <= 1e-4
    _, _, lc = O.partial_prefill(B, fx["tokens"], [(1, 1)], k, v, e)
    assert np.abs(lc - fx["cons_logits"]).max() <= 1e-4


def test_context_digest_golden():
    doc = json.loads((GOLDEN / "config_hash.json").read_text())
    for h in doc["hashes"]:
        t = np.random.default_rng(h["tokens_seed"]).integers(0, 128256, size=h["n"])
        assert O.context_digest(t) == h["digest"]


def test_normal_groups_golden():
    doc = json.loads((GOLDEN / "config_hash.json").read_text())
    for case in doc["normal_forms"]:
        assert [list(g) for g in O.normal_groups(case["in"])] == case["groups"]


def test_bf16_round_matches_torch():
    torch = pytest.importorskip("torch")
    x = np.random.default_rng(0).standard_normal(100_000).astype(np.float32) * 37
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float32).numpy()
    assert np.array_equal(O.bf16_round(x), ref)


@pytest.mark.reference
def test_live_against_reference_hypothesis_configs(crosskv_ref):
    M = crosskv_ref
    cfg = M.ModelConfig(*[getattr(TOY, f) for f in TOY.__dataclass_fields__])
    base = M.build_model(cfg)
    recv = M.build_model(cfg, M.PerturbationSpec.block(8, [2, 6], 0.7, 3))
    ob = O.make_weights(TOY)
    orr = O.make_weights(TOY, O.block_eps(8, [2, 6], 0.7), noise_seed=3)
    rng = np.random.default_rng(11)
    for trial in range(6):
        toks = M.make_synthetic_dataset(int(rng.integers(0, 9999)), 1, int(rng.integers(2, 60)), 256)[0]
        groups = O.normal_groups([sorted(rng.integers(0, 8, size=2).tolist()) for _ in range(int(rng.integers(0, 3)))])
        full = M.full_prefill(base, toks)
        ref = M.partial_prefill(recv, toks, M.RecomputeConfig(groups), full.kv, full.e_map())
        k, v, e, _ = O.full_prefill(ob, toks)
        _, _, lg = O.partial_prefill(orr, toks, groups, k, v, e)
        assert np.abs(lg - ref.logits).max() <= 1e-5, (trial, groups)


# ---------------------------------------------------------------------------
# token-selective baseline (model.py:682-743), pinned to selective.npz
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("ratio", [0.25, 1.0])
def test_token_selective_toy_matches_reference(toy_base, ratio):
    fx = np.load(GOLDEN / "selective.npz")
    recv = O.make_weights(TOY, O.block_eps(8, [4, 5], 1.0), noise_seed=1000)
    k, v, _, _ = O.full_prefill(toy_base, fx["toy_tokens"])
    sk, sv, logits, sel = O.token_selective_prefill(recv, fx["toy_tokens"], k, v, ratio)
    tag = f"toy_r{int(ratio * 100)}"
    assert np.abs(logits - fx[tag + "_logits"]).max() <= 1e-5
    assert np.abs(sk - fx[tag + "_k"]).max() <= 1e-5
    assert np.abs(sv - fx[tag + "_v"]).max() <= 1e-5
    assert len(sel) == int(np.ceil(ratio * (len(fx["toy_tokens"]) - 1)))


def test_token_selective_tiny_matches_reference():
    fx = np.load(GOLDEN / "selective.npz")
    A = O.make_weights(TINY)
    B = O.make_weights(TINY, O.block_eps(4, [0, 2], 0.5), noise_seed=1000)
    t = fx["tiny_tokens"]
    k, v, _, _ = O.full_prefill(A, t)
    sk, sv, logits, sel = O.token_selective_prefill(B, t, k, v, 0.15)
    assert np.array_equal(sel, fx["tiny_r15_selected"])
    assert np.abs(logits - fx["tiny_r15_logits"]).max() <= 1e-4
    dig = np.stack([sk.astype(np.float64).sum(axis=(1, 2, 3)), np.abs(sk.astype(np.float64)).sum(axis=(1, 2, 3)),
                    sv.astype(np.float64).sum(axis=(1, 2, 3)), np.abs(sv.astype(np.float64)).sum(axis=(1, 2, 3))], 1)
    np.testing.assert_allclose(dig, fx["tiny_r15_kv_digest"], rtol=1e-5, atol=1e-2)


def test_token_selective_selection_ties_and_misses(toy_base):
    dev = np.array([1.0, 3.0, 3.0, 0.5, 3.0, 2.0], dtype=np.float32)
    assert O.select_positions(dev, 0.5).tolist() == [1, 2, 4]
    assert O.select_positions(dev, 0.3).tolist() == [1, 2]          # ceil(1.8) = 2: ties to the lowest
    assert O.select_positions(np.zeros(5, np.float32), 0.4).tolist() == [0, 1]
    toks = O.synthetic_tokens(42, 1, 40, 256)[0]
    k, v, _, _ = O.full_prefill(toy_base, toks)
    with pytest.raises(O.CacheMiss) as e:
        O.token_selective_prefill(toy_base, toks, k[:5], v[:5], 0.5)
    assert e.value.layer == 5
    with pytest.raises(O.CacheMiss) as e:
        O.token_selective_prefill(toy_base, toks, k[:, :, :10], v[:, :, :10], 0.5)
    assert e.value.layer == 0
    with pytest.raises(ValueError):
        O.token_selective_prefill(toy_base, toks, k, v, 0.0)


def test_make_variant_equals_make_weights():
    """make_variant (shared base tensors) draws the same noise streams as
    make_weights with eps (model.py:315-320): bit-identical weights."""
    dims = O.Dims(4, 256, 4, 1, 64, 1024, 4096, 1024, 7)
    base = O.make_weights(dims)
    eps = O.block_eps(4, [1, 3], 0.25)
    want = O.make_weights(dims, eps, noise_seed=55)
    got = O.make_variant(base, eps, 55)
    assert np.array_equal(got["embed"], want["embed"]) and np.array_equal(got["unembed"], want["unembed"])
    for lw_w, lw_g in zip(want["layers"], got["layers"]):
        for name in O.LAYER_SLOTS:
            assert np.array_equal(lw_w[name], lw_g[name]), name


def test_einsum_attention_matches_blocked():
    """attend_einsum (the reference's einsum restatement, timed by bench.py)
    equals the blocked-BLAS attend to float32 rounding."""
    rng = np.random.default_rng(0)
    q = rng.standard_normal((70, 8, 64), dtype=np.float32)
    k = rng.standard_normal((2, 70, 64), dtype=np.float32)
    v = rng.standard_normal((2, 70, 64), dtype=np.float32)
    pos = np.arange(70)
    a = O.attend(q, k, v, pos)
    b = O.attend_einsum(q, k, v, pos[None, :] <= pos[:, None])
    assert np.abs(a - b).max() < 1e-5


@pytest.mark.reference
def test_einsum_attention_matches_reference(crosskv_ref):
    m = crosskv_ref
    cfg = m.ModelConfig(1, 512, 8, 2, 64, 1024, 4096, 128, 0)
    rng = np.random.default_rng(1)
    q = rng.standard_normal((60, 8, 64), dtype=np.float32)
    k = rng.standard_normal((2, 60, 64), dtype=np.float32)
    v = rng.standard_normal((2, 60, 64), dtype=np.float32)
    allowed = np.tril(np.ones((60, 60), dtype=bool))
    assert np.array_equal(m._masked_attention(q, k, v, allowed, cfg), O.attend_einsum(q, k, v, allowed))
