"""End-to-end parity of the B200 path against the CPU oracle (through the C ABI).

Inputs: the reference's seeded weights (same PCG64 streams, pinned in
test_oracle.py) and synthetic prefixes.  Tolerances:

* reused-KV placement: bit-exact (bf16 copy of the producer export);
* recomputed KV: rel-L2 <= 2e-2 vs the fp32 oracle;
* first-token logits: max|dlogit| <= 0.1 and rel-L2 <= 3e-2 vs the fp32
  oracle, and rel-L2 <= 1e-2 vs the bf16-faithful oracle (same rounding points);
* greedy first-token agreement reported over 16 prefixes.
"""

import numpy as np
import pytest
import torch

from oracle import crosskv_oracle as O

pytestmark = pytest.mark.gpu

TINY = (4, 256, 4, 1, 64, 1024, 4096, 1024, 7)
MID = (2, 1024, 8, 2, 128, 2816, 8192, 1024, 11)


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.fixture(scope="module")
def pkg():
    import paper_2411_02820_b200 as P
    return P


def _pair(pkg, dims, pert_layers, eps, seed):
    cfg = pkg.ModelConfig(*dims)
    spec = pkg.PerturbationSpec.block(cfg.n_layers, pert_layers, eps, seed)
    A = pkg.build_model(cfg)
    B = pkg.build_model(cfg, spec)
    od = O.Dims(*dims)
    oA = O.make_weights(od)
    oB = O.make_weights(od, O.block_eps(cfg.n_layers, pert_layers, eps), noise_seed=seed)
    return cfg, A, B, oA, oB


@pytest.fixture(scope="module")
def tiny(pkg):
    return _pair(pkg, TINY, [2], 0.5, 1000)


def _host(t):
    return t.float().cpu().numpy()


def test_config1_partial_prefill_parity(pkg, tiny):
    cfg, A, B, oA, oB = tiny
    toks = O.synthetic_tokens(100, 1, 512, 4096)[0]
    rc = pkg.RecomputeConfig([(2, 3)])
    prod = pkg.full_prefill(A, toks)
    cons = pkg.partial_prefill(B, toks, rc, prod.kv, prod.e_map())
    torch.cuda.synchronize()
    P = len(toks) - 1
    # --- producer export vs oracle
    k, v, e, lp = O.full_prefill(oA, toks)
    assert rel(_host(prod.kv.k), k) < 2e-2 and rel(_host(prod.kv.v), v) < 2e-2
    assert rel(_host(prod.e_map()[2].hidden), e[2]) < 1e-2
    assert prod.e_map()[2].hidden.dtype == torch.float32
    assert np.array_equal(_host(prod.e_map()[0].hidden), O.bf16_round(oA["embed"][toks[:P]]))
    assert np.abs(_host(prod.logits) - lp).max() < 0.1
    # --- consumer
    ck, cv, lc = O.partial_prefill(oB, toks, [(2, 3)], k, v, e)
    dense = cons.kv.dense()
    gk, gv = _host(dense.k), _host(dense.v)
    # reused layers: bit-exact copy of the producer's bf16 export (model.py:602-603)
    for l in (0, 1):
        assert torch.equal(dense.k[l, :, :P], prod.kv.k[l, :, :P])
        assert torch.equal(dense.v[l, :, :P], prod.kv.v[l, :, :P])
    for l in (2, 3):
        assert rel(gk[l, :, :P], ck[l, :, :P]) < 2e-2, l
        assert rel(gv[l, :, :P], cv[l, :, :P]) < 2e-2, l
    assert rel(gk[:, :, P], ck[:, :, P]) < 3e-2  # anchor K at every layer
    logits = _host(cons.logits)
    assert np.abs(logits - lc).max() < 0.1
    assert rel(logits, lc) < 3e-2
    assert cons.token == int(np.argmax(logits))
    # bf16-faithful mirror: same rounding points as the kernels
    bA, bB = O.round_weights_bf16(oA), O.round_weights_bf16(oB)
    fk, fv, fe, _ = O.full_prefill(bA, toks, act=O.bf16_round)  # E exported exactly (f32)
    _, _, lf = O.partial_prefill(bB, toks, [(2, 3)], O.bf16_round(fk), O.bf16_round(fv), fe, act=O.bf16_round)
    assert rel(logits, lf) < 1e-2


def test_first_token_agreement_16_prefixes(pkg, tiny):
    cfg, A, B, oA, oB = tiny
    from conftest import GOLDEN
    gold = np.load(GOLDEN / "tiny_16prefixes.npz")
    rc = pkg.RecomputeConfig([(2, 3)])
    agree_ref, agree_recv = 0, 0
    for i in range(16):
        toks = O.synthetic_tokens(100 + i, 1, 512, 4096)[0]
        prod = pkg.full_prefill(A, toks, e_layers=rc.transition_layers)
        cons = pkg.partial_prefill(B, toks, rc, prod.kv, prod.e_map())
        tok = cons.token
        agree_ref += tok == int(gold["first_partial"][i])      # reference partial prefill
        agree_recv += tok == int(gold["first_recv_full"][i])   # receiver's own full prefill
        assert np.abs(_host(cons.logits) - gold["logits_partial"][i]).max() < 0.1
    print(f"first-token agreement: vs reference partial {agree_ref}/16, vs receiver full {agree_recv}/16")
    assert agree_ref >= 15 and agree_recv >= 15


def test_mid_head128_parity(pkg):
    cfg, A, B, oA, oB = _pair(pkg, MID, [1], 0.5, 77)
    toks = O.synthetic_tokens(9, 1, 384, 8192)[0]
    prod = pkg.full_prefill(A, toks)
    cons = pkg.partial_prefill(B, toks, pkg.RecomputeConfig([(1, 1)]), prod.kv, prod.e_map())
    torch.cuda.synchronize()
    k, v, e, lp = O.full_prefill(oA, toks)
    _, _, lc = O.partial_prefill(oB, toks, [(1, 1)], k, v, e)
    assert rel(_host(prod.logits), lp) < 3e-2
    assert rel(_host(cons.logits), lc) < 3e-2
    assert np.abs(_host(cons.logits) - lc).max() < 0.1


@pytest.mark.parametrize("groups", [[], [(0, 3)], [(1, 2)], [(0, 0), (3, 3)], [(3, 3)]])
def test_identity_reuse(pkg, tiny, groups):
    cfg, A, B, oA, oB = tiny
    toks = O.synthetic_tokens(7, 1, 300, 4096)[0]
    full = pkg.full_prefill(A, toks)
    mixed = pkg.partial_prefill(A, toks, pkg.RecomputeConfig(groups), full.kv, full.e_map())
    torch.cuda.synchronize()
    lf, lm = _host(full.logits), _host(mixed.logits)
    # same model, different batching/rounding of the recomputed layers
    assert np.abs(lf - lm).max() < 0.1
    assert mixed.token == full.token


def test_errors_in_reference_order(pkg, tiny):
    cfg, A, B, oA, oB = tiny
    toks = O.synthetic_tokens(8, 1, 64, 4096)[0]
    full = pkg.full_prefill(A, toks)
    with pytest.raises(pkg.CacheMissError) as err:
        pkg.partial_prefill(B, toks, pkg.RecomputeConfig([(1, 2)]), None)
    assert (err.value.layer, err.value.kind) == (0, "kv")
    with pytest.raises(pkg.CacheMissError) as err:
        pkg.partial_prefill(B, toks, pkg.RecomputeConfig([(2, 3)]), full.kv, {})
    assert (err.value.layer, err.value.kind) == (2, "e")
    with pytest.raises(pkg.DegenerateInputError):
        pkg.partial_prefill(B, [5], pkg.RecomputeConfig.full(4), None)
    with pytest.raises(ValueError):
        pkg.partial_prefill(B, toks, pkg.RecomputeConfig([(2, 9)]), full.kv, full.e_map())
    short = pkg.full_prefill(A, toks[:10])
    with pytest.raises(pkg.CacheMissError) as err:
        pkg.partial_prefill(B, toks, pkg.RecomputeConfig([(2, 3)]), short.kv, full.e_map())
    assert (err.value.layer, err.value.kind) == (0, "kv")


def test_recompute_all_equals_full_prefill(pkg, tiny):
    cfg, A, B, oA, oB = tiny
    toks = O.synthetic_tokens(3, 1, 200, 4096)[0]
    full = pkg.full_prefill(B, toks)
    mixed = pkg.partial_prefill(B, toks, pkg.RecomputeConfig.full(4), None)
    torch.cuda.synchronize()
    assert np.abs(_host(full.logits) - _host(mixed.logits)).max() < 0.1
    d = mixed.kv.dense()
    assert rel(_host(d.k), _host(full.kv.k)) < 1e-2


def test_two_stream_pipeline_matches_single_stream(pkg, tiny):
    cfg, A, B, oA, oB = tiny
    toks = O.synthetic_tokens(11, 1, 512, 4096)[0]
    prod = pkg.full_prefill(A, toks)
    rc = pkg.RecomputeConfig([(2, 3)])
    one = pkg.partial_prefill(B, toks, rc, prod.kv, prod.e_map())
    side = torch.cuda.Stream()
    two = pkg.partial_prefill(B, toks, rc, prod.kv, prod.e_map(), copy_stream=side)
    torch.cuda.synchronize()
    assert torch.equal(one.logits, two.logits)
    assert torch.equal(one.kv.dense().k, two.kv.dense().k)


def test_paged_cache_with_shuffled_pages(pkg, tiny):
    cfg, A, B, oA, oB = tiny
    toks = O.synthetic_tokens(12, 1, 700, 4096)[0]
    prod = pkg.full_prefill(A, toks)
    rc = pkg.RecomputeConfig([(2, 3)])
    ref = pkg.partial_prefill(B, toks, rc, prod.kv, prod.e_map())
    cache = pkg.PagedKV.allocate(cfg, len(toks), "cuda", spare_pages=7, shuffle_seed=3)
    got = pkg.partial_prefill(B, toks, rc, prod.kv, prod.e_map(), out=cache)
    torch.cuda.synchronize()
    assert torch.equal(ref.logits, got.logits)
    assert torch.equal(ref.kv.dense().v, got.kv.dense().v)


@pytest.mark.parametrize("n", [2, 3, 65, 1024])
def test_edge_lengths(pkg, tiny, n):
    """Shortest window (n = 2: one reused position + the anchor), page boundaries,
    and n = max_seq (model.py:425-437 bounds)."""
    cfg, A, B, oA, oB = tiny
    toks = O.synthetic_tokens(50 + n, 1, n, 4096)[0]
    prod = pkg.full_prefill(A, toks)
    cons = pkg.partial_prefill(B, toks, pkg.RecomputeConfig([(2, 3)]), prod.kv, prod.e_map())
    torch.cuda.synchronize()
    k, v, e, lp = O.full_prefill(oA, toks)
    _, _, lc = O.partial_prefill(oB, toks, [(2, 3)], k, v, e)
    assert np.abs(_host(prod.logits) - lp).max() < 0.1
    assert np.abs(_host(cons.logits) - lc).max() < 0.1
    d = cons.kv.dense()
    assert torch.equal(d.k[:2, :, :n - 1], prod.kv.k[:2, :, :n - 1])
    with pytest.raises(ValueError):
        pkg.partial_prefill(B, O.synthetic_tokens(1, 1, 1025, 4096)[0], pkg.RecomputeConfig([(2, 3)]), prod.kv,
                            prod.e_map())


def test_multiple_groups_and_layer0_group(pkg, tiny):
    cfg, A, B, oA, oB = tiny
    toks = O.synthetic_tokens(61, 1, 257, 4096)[0]
    groups = [(0, 0), (2, 2)]
    prod = pkg.full_prefill(A, toks)
    cons = pkg.partial_prefill(B, toks, pkg.RecomputeConfig(groups), prod.kv, prod.e_map())
    torch.cuda.synchronize()
    k, v, e, _ = O.full_prefill(oA, toks)
    ck, cv, lc = O.partial_prefill(oB, toks, groups, k, v, e)
    assert np.abs(_host(cons.logits) - lc).max() < 0.1
    d = cons.kv.dense()
    P_ = len(toks) - 1
    for l in (1, 3):
        assert torch.equal(d.k[l, :, :P_], prod.kv.k[l, :, :P_])
    for l in (0, 2):
        assert rel(_host(d.k)[l, :, :P_], ck[l, :, :P_]) < 2e-2


def _random_case(i):
    """Seeded random (n, recompute groups) on TINY: the reference's identity /
    partial properties over configs its hypothesis test draws (test_model.py:298-314)."""
    rng = np.random.default_rng(4242 + i)
    n = int(rng.choice([2, 3, 64, 65, 127, 300, 511, 700, 1024]))
    L = TINY[0]
    groups = []
    for _ in range(int(rng.integers(0, 3))):
        a = int(rng.integers(0, L))
        b = int(rng.integers(a, L))
        groups.append((a, b))
    return n, groups


@pytest.mark.parametrize("case", range(10))
def test_random_configs_vs_oracle(pkg, tiny, case):
    cfg, A, B, oA, oB = tiny
    n, groups = _random_case(case)
    toks = O.synthetic_tokens(300 + case, 1, n, 4096)[0]
    rc = pkg.RecomputeConfig(groups)
    prod = pkg.full_prefill(A, toks)
    cons = pkg.partial_prefill(B, toks, rc, prod.kv, prod.e_map())
    torch.cuda.synchronize()
    P = n - 1
    k, v, e, _ = O.full_prefill(oA, toks)
    ck, cv, lc = O.partial_prefill(oB, toks, [tuple(g) for g in rc.groups], k, v, e)
    dense = cons.kv.dense()
    gk, gv = _host(dense.k), _host(dense.v)
    recomputed = set(rc.layer_set())
    for l in range(cfg.n_layers):
        if l in recomputed:
            if P >= 16:  # rel-L2 over a handful of values is dominated by bf16 rounding
                assert rel(gk[l, :, :P], ck[l, :, :P]) < 2e-2, (l, n, groups)
                assert rel(gv[l, :, :P], cv[l, :, :P]) < 2e-2, (l, n, groups)
        else:
            assert torch.equal(dense.k[l, :, :P], prod.kv.k[l, :, :P]), (l, n, groups)
            assert torch.equal(dense.v[l, :, :P], prod.kv.v[l, :, :P]), (l, n, groups)
    logits = _host(cons.logits)
    assert np.isfinite(logits).all()
    assert np.abs(logits - lc).max() < 0.1, (n, groups)
    assert rel(logits, lc) < 3e-2, (n, groups)
    assert cons.token == int(np.argmax(logits))


@pytest.fixture(scope="module")
def mid(pkg):
    return _pair(pkg, MID, [1], 0.5, 77)


@pytest.mark.parametrize("n,groups", [(129, [(0, 0)]), (257, [(1, 1)]), (640, [(0, 1)]), (1000, [])])
def test_mid_configs_vs_oracle(pkg, mid, n, groups):
    """Head dim 128, GQA 4, CTA-pair GEMMs and the tcgen05 FA at ragged lengths."""
    cfg, A, B, oA, oB = mid
    toks = O.synthetic_tokens(50 + n, 1, n, 8192)[0]
    prod = pkg.full_prefill(A, toks)
    cons = pkg.partial_prefill(B, toks, pkg.RecomputeConfig(groups), prod.kv, prod.e_map())
    torch.cuda.synchronize()
    P = n - 1
    k, v, e, _ = O.full_prefill(oA, toks)
    ck, cv, lc = O.partial_prefill(oB, toks, groups, k, v, e)
    dense = cons.kv.dense()
    recomputed = set(pkg.RecomputeConfig(groups).layer_set())
    for l in range(cfg.n_layers):
        if l in recomputed:
            assert rel(_host(dense.k[l, :, :P]), ck[l, :, :P]) < 2e-2, l
            assert rel(_host(dense.v[l, :, :P]), cv[l, :, :P]) < 2e-2, l
        else:
            assert torch.equal(dense.k[l, :, :P], prod.kv.k[l, :, :P]), l
            assert torch.equal(dense.v[l, :, :P], prod.kv.v[l, :, :P]), l
    logits = _host(cons.logits)
    assert np.abs(logits - lc).max() < 0.1 and rel(logits, lc) < 3e-2
    assert cons.token == int(np.argmax(logits))
