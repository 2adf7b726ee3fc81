"""Numerical parity at the headline dimensions (Llama-3-8B shapes), not only
self-consistency (VERDICT r1 "8B-dims numerical parity").

(a) Truncated 8B model vs the CPU ORACLE (SURVEY §7.2 phase 3, §8c: "8B-truncated
    (L = 1-2, n <= 2048) vs oracle"): L = 2 at full 8B width (d 4096, H 32,
    KVH 8, D 128, d_ff 14336, V 128256), n = 2048, the reference's seeded
    weights (oracle.make_weights == weights.reference_weights, pinned in
    test_oracle.py), B = A + block noise.  Run through the persistent
    co-resident anchor on two streams, the per-launch anchor on two streams,
    and a single stream: all three bit-identical, each within tolerance of the
    fp32 oracle (and of the bf16-faithful oracle) -- model.py:574-638.
(b) Full BASELINE config 2 (L = 32, n = 8192, k = 6) vs a GPU fp32 MIRROR of
    the block math on the same bf16 weights (tests/fp32_mirror.py):
    the producer's 32 window layers teacher-forced (each layer's K/V and output
    from the exported E of its input), the producer's anchor + logits, and the
    consumer partial prefill end to end (recompute [26, 31] from E(26) +
    32-layer anchor over the mixed cache) through both anchor shapes.
(c) A lossy 8B pair whose quality measurement can fail: B = A + small noise on
    EVERY layer + large noise on the recomputed block.  As the reference's
    test_model.py:190-194 (recompute beats full reuse), the partial prefill is
    closer to B's own full prefill than full reuse is, and its greedy
    agreement over a 32-token horizon (agreement_score, model.py:810-831) is at
    least full reuse's.

Tolerances (as test_gpu_parity): reused K/V bit-exact;
recomputed K/V rel-L2 <= 2e-2; anchor K/V rel-L2 <= 3e-2; logits
max|d| <= 0.1 and rel-L2 <= 3e-2 vs fp32; rel-L2 <= 1e-2 vs the bf16-faithful
oracle; residual-stream outputs (E of the next layer) rel-L2 <= 1e-2.
"""

import numpy as np
import pytest
import torch

from fp32_mirror import Mirror, rel
from oracle import crosskv_oracle as O

pytestmark = pytest.mark.gpu

V8 = 128256
TRUNC = (2, 4096, 32, 8, 128, 14336, V8, 2048, 21)  # ModelConfig / oracle Dims field order
SHAPE = dict(n_layers=32, d_model=4096, n_heads=32, n_kv_heads=8, head_dim=128, d_ff=14336, vocab_size=V8)
N = 8192
K = 6


def _np(t):
    return t.float().cpu().numpy()


def _nrel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


# ---------------------------------------------------------------------------
# (a) truncated 8B vs the CPU oracle
# ---------------------------------------------------------------------------


@pytest.fixture(scope="module")
def trunc():
    import paper_2411_02820_b200 as P
    from paper_2411_02820_b200.weights import from_host
    od = O.Dims(*TRUNC)
    oA = O.make_weights(od)
    oB = O.make_variant(oA, O.block_eps(2, [1], 0.5), 77)
    cfg = P.ModelConfig(*TRUNC)
    A = from_host(cfg, oA, "trunc8b-A")
    B = from_host(cfg, oB, "trunc8b-B")
    toks = O.synthetic_tokens(5, 1, 2048, V8)[0]
    k, v, e, lp = O.full_prefill(oA, toks)
    return P, cfg, A, B, oA, oB, toks, (k, v, e, lp)


def _consumer_runs(P, B, toks, rc, prod):
    from paper_2411_02820_b200 import _lib
    out = {}
    for shape in ("persistent", "launch"):
        with _lib.anchor_shape(shape):
            out[shape] = P.partial_prefill(B, toks, rc, prod.kv, prod.e_map(), copy_stream=torch.cuda.Stream())
            torch.cuda.synchronize()
    out["single"] = P.partial_prefill(B, toks, rc, prod.kv, prod.e_map())
    torch.cuda.synchronize()
    return out


def test_trunc8b_producer_vs_oracle(trunc):
    P, cfg, A, B, oA, oB, toks, (k, v, e, lp) = trunc
    prod = P.full_prefill(A, toks)
    torch.cuda.synchronize()
    Pn = len(toks) - 1
    assert _nrel(_np(prod.kv.k), k) < 2e-2 and _nrel(_np(prod.kv.v), v) < 2e-2
    assert _nrel(_np(prod.e_map()[1].hidden), e[1]) < 1e-2
    assert np.array_equal(_np(prod.e_map()[0].hidden), O.bf16_round(oA["embed"][toks[:Pn]]))
    lg = _np(prod.logits)
    assert np.abs(lg - lp).max() < 0.1 and _nrel(lg, lp) < 3e-2


@pytest.mark.parametrize("groups", [[(1, 1)], [(0, 0)]])
def test_trunc8b_consumer_vs_oracle(trunc, groups):
    P, cfg, A, B, oA, oB, toks, (k, v, e, lp) = trunc
    rc = P.RecomputeConfig(groups)
    prod = P.full_prefill(A, toks, e_layers=rc.transition_layers)
    runs = _consumer_runs(P, B, toks, rc, prod)
    # every anchor shape / stream order: the same arithmetic, the same bits
    ref = runs["single"]
    for name, r in runs.items():
        assert torch.equal(r.logits, ref.logits), name
        dr, d0 = r.kv.dense(), ref.kv.dense()
        assert torch.equal(dr.k, d0.k) and torch.equal(dr.v, d0.v), name
    ck, cv, lc = O.partial_prefill(oB, toks, groups, k, v, e)
    Pn = len(toks) - 1
    dense = ref.kv.dense()
    gk, gv = _np(dense.k), _np(dense.v)
    cov = {l for a, b in groups for l in range(a, b + 1)}
    for l in range(2):
        if l in cov:
            assert _nrel(gk[l, :, :Pn], ck[l, :, :Pn]) < 2e-2, l
            assert _nrel(gv[l, :, :Pn], cv[l, :, :Pn]) < 2e-2, l
        else:  # reused: the producer export's bits (model.py:602-603)
            assert torch.equal(dense.k[l, :, :Pn], prod.kv.k[l, :, :Pn])
            assert torch.equal(dense.v[l, :, :Pn], prod.kv.v[l, :, :Pn])
    assert _nrel(gk[:, :, Pn], ck[:, :, Pn]) < 3e-2 and _nrel(gv[:, :, Pn], cv[:, :, Pn]) < 3e-2
    lg = _np(ref.logits)
    assert np.abs(lg - lc).max() < 0.1, np.abs(lg - lc).max()
    assert _nrel(lg, lc) < 3e-2
    assert ref.token == int(np.argmax(lg))
    print(f"trunc 8B {groups}: max|dlogit| {np.abs(lg - lc).max():.3e} rel {_nrel(lg, lc):.3e}, "
          f"oracle argmax {int(np.argmax(lc))} gpu {ref.token}")


def test_trunc8b_consumer_vs_bf16_faithful_oracle(trunc):
    P, cfg, A, B, oA, oB, toks, _ = trunc
    rc = P.RecomputeConfig([(1, 1)])
    prod = P.full_prefill(A, toks, e_layers=rc.transition_layers)
    cons = P.partial_prefill(B, toks, rc, prod.kv, prod.e_map(), copy_stream=torch.cuda.Stream())
    torch.cuda.synchronize()
    bA, bB = O.round_weights_bf16(oA), O.round_weights_bf16(oB)
    fk, fv, fe, _ = O.full_prefill(bA, toks, act=O.bf16_round)  # E exported exactly (f32)
    _, _, lf = O.partial_prefill(bB, toks, [(1, 1)], O.bf16_round(fk), O.bf16_round(fv), fe, act=O.bf16_round)
    assert _nrel(_np(cons.logits), lf) < 1e-2


# ---------------------------------------------------------------------------
# (b) full config 2 vs the GPU fp32 mirror
# ---------------------------------------------------------------------------


@pytest.fixture(scope="module")
def cfg2():
    import paper_2411_02820_b200 as P
    cfg = P.ModelConfig(max_seq=N + 64, base_seed=0, **SHAPE)
    A = P.random_model(cfg, seed=11)
    B = P.random_model(cfg, seed=12, base=A, perturb_layers=range(32 - K, 32), eps=0.5)
    ids = np.random.default_rng(3).integers(0, cfg.vocab_size, size=N, dtype=np.int64)
    tok = torch.from_numpy(ids).cuda()
    prod = P.full_prefill(A, ids, tokens_dev=tok, copy_stream=torch.cuda.Stream())  # E at every layer
    torch.cuda.synchronize()
    return P, cfg, A, B, ids, tok, prod


def test_config2_producer_layers_vs_fp32_mirror(cfg2):
    """Each of the 32 window layers at n = 8192, teacher-forced from the
    exported E of its input: K/V into the export and the layer's output (the
    next layer's E) against fp32; then the producer's anchor pass over its own
    export and the logits."""
    P, cfg, A, B, ids, tok, prod = cfg2
    m = Mirror(A)
    Pn = N - 1
    e = prod.e_map()
    win = torch.arange(Pn, device="cuda")
    worst = [0.0, 0.0]
    for l in range(32):
        h, k, v = m.block(e[l].hidden, l, win, kv_only=(l == 31))
        rk = rel(prod.kv.k[l, :, :Pn].float().permute(1, 0, 2), k)
        rv = rel(prod.kv.v[l, :, :Pn].float().permute(1, 0, 2), v)
        assert rk < 2e-2 and rv < 2e-2, (l, rk, rv)
        worst[0] = max(worst[0], rk, rv)
        if h is not None:
            rh = rel(e[l + 1].hidden, h)
            assert rh < 1e-2, (l, rh)
            worst[1] = max(worst[1], rh)
        del h, k, v
    # anchor row over the producer's own K/V (model.py:627-637)
    ha = A.embed[tok[Pn:]].float()
    pos = torch.tensor([Pn], device="cuda")
    for l in range(32):
        kc = prod.kv.k[l, :, :Pn].float().permute(1, 0, 2)
        vc = prod.kv.v[l, :, :Pn].float().permute(1, 0, 2)
        ha, ko, vo = m.block(ha, l, pos, kc, vc)
        assert rel(prod.kv.k[l, :, Pn].float(), ko[0]) < 3e-2, l
    lm = m.logits(ha[0])
    d = (prod.logits - lm).abs().max().item()
    assert d < 0.1 and rel(prod.logits, lm) < 3e-2, d
    print(f"config 2 producer: worst layer K/V rel {worst[0]:.2e}, E rel {worst[1]:.2e}, "
          f"max|dlogit| {d:.3e}, logits rel {rel(prod.logits, lm):.3e}")


def test_config2_consumer_vs_fp32_mirror(cfg2):
    """The headline consumer step (recompute [26, 31] from E(26), 26 reused
    layers, anchor over the mixed cache) end to end against fp32, through the
    persistent co-resident anchor (two streams, the bench's shape) and the
    per-launch anchor: bit-identical to each other."""
    P, cfg, A, B, ids, tok, prod = cfg2
    from paper_2411_02820_b200 import _lib
    rc = P.RecomputeConfig([(32 - K, 31)])
    e_map = {26: prod.e_map()[26]}
    runs = {}
    for shape in ("persistent", "launch"):
        with _lib.anchor_shape(shape):
            runs[shape] = P.partial_prefill(B, ids, rc, prod.kv, e_map, copy_stream=torch.cuda.Stream(),
                                            tokens_dev=tok)
            torch.cuda.synchronize()
    assert torch.equal(runs["persistent"].logits, runs["launch"].logits)
    cons = runs["persistent"]
    m = Mirror(B)
    Km, Vm, lm = m.mixed(tok, rc.groups, prod.kv, {26: e_map[26].hidden})
    Pn = N - 1
    dense = cons.kv.dense()
    for l in range(32):
        gk = dense.k[l].float().permute(1, 0, 2)
        gv = dense.v[l].float().permute(1, 0, 2)
        if l < 32 - K:
            assert torch.equal(dense.k[l, :, :Pn], prod.kv.k[l, :, :Pn])
            assert torch.equal(dense.v[l, :, :Pn], prod.kv.v[l, :, :Pn])
        else:
            assert rel(gk[:Pn], Km[l][:Pn]) < 2e-2 and rel(gv[:Pn], Vm[l][:Pn]) < 2e-2, l
        assert rel(gk[Pn], Km[l][Pn]) < 3e-2 and rel(gv[Pn], Vm[l][Pn]) < 3e-2, l
    d = (cons.logits - lm).abs().max().item()
    r = rel(cons.logits, lm)
    assert d < 0.1 and r < 3e-2, (d, r)
    assert dense.k.shape[2] >= N and cons.token == int(cons.logits.argmax())
    print(f"config 2 consumer: max|dlogit| {d:.3e} rel {r:.3e}; argmax gpu {cons.token} fp32 {int(lm.argmax())}")


# ---------------------------------------------------------------------------
# (c) a lossy 8B pair: the quality measurement can fail
# ---------------------------------------------------------------------------


def test_lossy_pair_recompute_beats_full_reuse(cfg2):
    P, cfg, A, B0, ids, tok, prod = cfg2
    from paper_2411_02820_b200.quality import agreement_score
    n = 2048  # quality at a shorter prefix keeps the 4 decodes quick
    ids_q = ids[:n]
    lossy = P.random_model(cfg, seed=31, base=A, perturb_layers=range(32), eps=0.03)
    lossy = P.random_model(cfg, seed=32, base=lossy, perturb_layers=range(32 - K, 32), eps=0.5)
    rc = P.RecomputeConfig([(32 - K, 31)])
    exp = P.full_prefill(A, ids_q, e_layers=rc.transition_layers)
    own = P.full_prefill(lossy, ids_q, e_layers=())
    mixed = P.partial_prefill(lossy, ids_q, rc, exp.kv, exp.e_map())
    reuse = P.partial_prefill(lossy, ids_q, P.RecomputeConfig.none(), exp.kv, {})
    torch.cuda.synchronize()
    d_mixed, d_reuse = rel(mixed.logits, own.logits), rel(reuse.logits, own.logits)
    assert d_mixed < d_reuse, (d_mixed, d_reuse)
    covered = agreement_score(A, lossy, ids_q, rc, horizon=32)
    full_reuse = agreement_score(A, lossy, ids_q, P.RecomputeConfig.none(), horizon=32)
    print(f"lossy 8B pair (n={n}): logits rel vs own prefill: recompute {d_mixed:.3e}, full reuse {d_reuse:.3e}; "
          f"agreement@32 recompute {covered.score:.3f} (first divergence {covered.first_divergence}), "
          f"full reuse {full_reuse.score:.3f}")
    assert covered.score >= full_reuse.score
    assert 0.0 <= covered.score <= 1.0
