"""Batched requests (BASELINE config 4) and batched greedy decode on the B200.

A consumer's batch of requests runs the recompute request by request and ONE
batched anchor pass (every layer's weights streamed once for all rows).  Each
row's arithmetic is the single-request pass's, so the batch must equal its
requests run one by one through ``partial_prefill`` -- logits, greedy token
and every cache byte -- and a batched decode must equal per-sequence decodes.
Shapes: TINY (the GEMVs take the per-row path, the attention the batched
kernel), a d=2048 shape where every GEMV is the batched TMA kernel, and a
d_ff=14336 shape whose W2 rows do not all fit one launch (split 4 + 2).
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

SHAPES = {
    "tiny": dict(n_layers=4, d_model=256, n_heads=4, n_kv_heads=1, head_dim=64, d_ff=1024, vocab_size=4096,
                 max_seq=1024, base_seed=7),
    "wide": dict(n_layers=3, d_model=2048, n_heads=16, n_kv_heads=4, head_dim=128, d_ff=4096, vocab_size=16384,
                 max_seq=2048, base_seed=5),
    "longk": dict(n_layers=2, d_model=2048, n_heads=16, n_kv_heads=4, head_dim=128, d_ff=14336, vocab_size=8192,
                  max_seq=2048, base_seed=9),
}
LENGTHS = [300, 257, 512, 129, 64, 700, 2, 411]


def _pair(P, name):
    cfg = P.ModelConfig(**SHAPES[name])
    A = P.random_model(cfg, seed=11)
    B = P.random_model(cfg, seed=12, base=A, perturb_layers=range(cfg.n_layers - 2, cfg.n_layers), eps=0.5)
    return cfg, A, B


@pytest.mark.parametrize("name,nb,groups", [("tiny", 4, [(2, 3)]), ("tiny", 3, [(1, 1), (3, 3)]),
                                            ("tiny", 2, [(0, 3)]), ("tiny", 2, []),
                                            ("wide", 4, [(1, 2)]), ("wide", 8, [(2, 2)]),
                                            ("longk", 6, [(1, 1)])])
def test_batch_equals_one_by_one(name, nb, groups):
    import paper_2411_02820_b200 as P
    cfg, A, B = _pair(P, name)
    rng = np.random.default_rng(31 + nb)
    toks = [rng.integers(0, cfg.vocab_size, size=LENGTHS[b], dtype=np.int64) for b in range(nb)]
    rc = P.RecomputeConfig(groups)
    prods = [P.full_prefill(A, t, e_layers=rc.transition_layers) for t in toks]
    kvs = [p.kv for p in prods] if rc.reused_layers(cfg.n_layers) else [None] * nb
    got = P.partial_prefill_batch(B, toks, rc, kvs, [p.e_map() for p in prods], copy_stream=torch.cuda.Stream())
    ref = [P.partial_prefill(B, t, rc, kv, p.e_map()) for t, kv, p in zip(toks, kvs, prods)]
    torch.cuda.synchronize()
    for b in range(nb):
        assert torch.equal(got[b].logits, ref[b].logits), b
        assert got[b].token == ref[b].token
        gd, rd = got[b].kv.dense(), ref[b].kv.dense()
        assert torch.equal(gd.k, rd.k) and torch.equal(gd.v, rd.v), b


@pytest.mark.parametrize("name,nb", [("tiny", 3), ("wide", 5)])
def test_batched_decode_equals_per_sequence(name, nb):
    import paper_2411_02820_b200 as P
    from paper_2411_02820_b200.quality import decode_greedy, decode_greedy_batch
    cfg, A, _ = _pair(P, name)
    rng = np.random.default_rng(5)
    steps = 12
    toks = [rng.integers(0, cfg.vocab_size, size=LENGTHS[b] + 3, dtype=np.int64) for b in range(nb)]
    caches, lasts = [], []
    for t in toks:
        kv = P.LayerKV.empty(cfg, len(t) + steps)
        lasts.append(P.full_prefill(A, t, e_layers=[], out=kv))
        caches.append(kv)
    # per-sequence decode on copies of the caches (decode appends K/V)
    copies = [P.LayerKV(c.k.clone(), c.v.clone()) for c in caches]
    one = [decode_greedy(A, c, last, steps, positions=len(t)) for c, last, t in zip(copies, lasts, toks)]
    got = decode_greedy_batch(A, caches, lasts, steps, [len(t) for t in toks])
    for b in range(nb):
        assert np.array_equal(got[b], one[b]), b
        assert torch.equal(caches[b].k, copies[b].k) and torch.equal(caches[b].v, copies[b].v)


def test_batch_errors_name_the_request():
    import paper_2411_02820_b200 as P
    cfg, A, B = _pair(P, "tiny")
    rng = np.random.default_rng(3)
    toks = [rng.integers(0, cfg.vocab_size, size=n, dtype=np.int64) for n in (100, 120, 90)]
    rc = P.RecomputeConfig([(2, 3)])
    prods = [P.full_prefill(A, t, e_layers=rc.transition_layers) for t in toks]
    # request 1's export is too short for its window: KV miss at the first reused layer
    kvs = [prods[0].kv, prods[2].kv, prods[2].kv]
    with pytest.raises(P.CacheMissError) as e:
        P.partial_prefill_batch(B, toks, rc, kvs, [p.e_map() for p in prods])
    assert (e.value.layer, e.value.kind) == (0, "kv") and "request 1" in str(e.value)
    # request 2 lacks its E at the transition layer
    es = [prods[0].e_map(), prods[1].e_map(), {}]
    with pytest.raises(P.CacheMissError) as e:
        P.partial_prefill_batch(B, toks, rc, [p.kv for p in prods], es)
    assert (e.value.layer, e.value.kind) == (2, "e")
    with pytest.raises(ValueError):
        P.partial_prefill_batch(B, toks + [np.array([0, cfg.vocab_size])], rc, [p.kv for p in prods] + [None],
                                [p.e_map() for p in prods] + [None])
    with pytest.raises(P.DegenerateInputError):
        P.partial_prefill_batch(B, [toks[0], np.array([1])], rc, [prods[0].kv, prods[0].kv])


def test_captured_batch_replays_and_guards_contexts():
    """CapturedPartialPrefillBatch: one graph replay per batch equals the eager
    batch bit for bit; a request whose tokens are not its slot's context raises
    CacheMissError instead of reusing another context's KV."""
    import paper_2411_02820_b200 as P
    cfg, A, B = _pair(P, "tiny")
    rng = np.random.default_rng(17)
    toks = [rng.integers(0, cfg.vocab_size, size=n, dtype=np.int64) for n in (300, 180, 257)]
    rc = P.RecomputeConfig([(2, 3)])
    prods = [P.full_prefill(A, t, e_layers=rc.transition_layers) for t in toks]
    cap = P.CapturedPartialPrefillBatch(B, [len(t) for t in toks], rc, [p.kv for p in prods],
                                        [p.e_map() for p in prods])
    got = [r.logits.clone() for r in cap.run(toks)]
    ref = P.partial_prefill_batch(B, toks, rc, [p.kv for p in prods], [p.e_map() for p in prods])
    torch.cuda.synchronize()
    for b in range(3):
        assert torch.equal(got[b], ref[b].logits), b
    swapped = [toks[0], toks[1], rng.integers(0, cfg.vocab_size, size=257, dtype=np.int64)]  # not slot 2's context
    with pytest.raises(P.CacheMissError):
        cap.run(swapped)
    with pytest.raises(ValueError):
        cap.run(toks[:2])
