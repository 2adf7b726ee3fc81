"""Safety of the fused call and the serving form (VERDICT r1 "make the fused
call safe").

* A fused consumer call (persistent co-resident anchor) beside another
  stream's work -- a producer prefill with its per-launch kernels on the
  default stream -- gives bit-identical results (was tools/concurrency_check.py;
  the hazard it caught: a stand-alone kernel that does not fit beside one
  anchor CTA per SM starves the fused call's GEMMs).
* Two fused calls in flight at once on different stream pairs: the second
  runs the per-launch anchor (one persistent anchor per GPU), no hang, same
  bits (ds_fused_fallbacks counts the fallback).
* CapturedPartialPrefill serves only the context its export holds: another
  context raises CacheMissError, as the reference's fetch_context_caches does
  for a context it does not hold (store.py:351-395), instead of silently
  reusing the wrong KV.
* A captured graph owns its workspace: an eager call on the same stream that
  needs a larger workspace cannot free the graph's scratch.
* token-selective count in double precision: ceil(0.1 * 10) == 1, as the
  reference's math.ceil(ratio * window) (model.py:715).
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

SHAPE = dict(n_layers=32, d_model=4096, n_heads=32, n_kv_heads=8, head_dim=128, d_ff=14336, vocab_size=128256)
TINY = (4, 256, 4, 1, 64, 1024, 4096, 1024, 7)


@pytest.fixture(scope="module")
def big():
    import paper_2411_02820_b200 as P
    n = 16384
    cfg = P.ModelConfig(max_seq=n, base_seed=0, **SHAPE)
    A = P.random_model(cfg, seed=1)
    B = P.random_model(cfg, seed=2, base=A, perturb_layers=range(26, 32))
    ids = np.random.default_rng(3).integers(0, cfg.vocab_size, size=n, dtype=np.int64)
    tok = torch.from_numpy(ids).cuda()
    return P, cfg, A, B, ids, tok


@pytest.mark.timeout(600)
def test_fused_call_beside_producer_prefill(big):
    P, cfg, A, B, ids, tok = big
    s, side = torch.cuda.Stream(), torch.cuda.Stream()
    ref = P.full_prefill(B, ids, e_layers=(), stream=s, copy_stream=side, tokens_dev=tok)
    torch.cuda.synchronize()  # the outputs are written on stream s
    want = ref.logits.clone()
    for _ in range(2):
        P.full_prefill(A, ids, e_layers=(29,), tokens_dev=tok)  # default stream, not synchronised
        got = P.full_prefill(B, ids, e_layers=(), stream=s, copy_stream=side, tokens_dev=tok)
        torch.cuda.synchronize()
        assert torch.equal(got.logits, want), "results differ under concurrency"


@pytest.mark.timeout(600)
def test_two_fused_calls_in_flight(big):
    P, cfg, A, B, ids, tok = big
    from paper_2411_02820_b200 import _lib
    lib = _lib.lib()
    rc = P.RecomputeConfig([(26, 31)])
    n = 8192
    ids8, tok8 = ids[:n], tok[:n]
    prod = P.full_prefill(A, ids8, e_layers=rc.transition_layers, tokens_dev=tok8)
    torch.cuda.synchronize()
    streams = [(torch.cuda.Stream(), torch.cuda.Stream()) for _ in range(2)]
    caches = [P.PagedKV.allocate(cfg, n) for _ in streams]

    def call(i):
        s, x = streams[i]
        return P.partial_prefill(B, ids8, rc, prod.kv, prod.e_map(), stream=s, copy_stream=x, tokens_dev=tok8,
                                 out=caches[i])

    for i in (1, 0):  # warm: workspaces and outputs allocated, nothing in flight afterwards
        serial = call(i)
        torch.cuda.synchronize()
    serial = serial.logits.clone()
    before = lib.ds_fused_fallbacks()
    outs = [call(0), call(1)]  # the second is enqueued while the first (16 ms of GPU work) runs
    torch.cuda.synchronize()
    assert lib.ds_fused_fallbacks() == before + 1  # the second call ran the per-launch anchor
    for o in outs:
        assert torch.equal(o.logits, serial)
    # the same stream pair again: ordered behind the previous call, fused shape kept
    call(1)
    call(1)
    torch.cuda.synchronize()
    assert lib.ds_fused_fallbacks() == before + 1


@pytest.fixture(scope="module")
def tiny():
    import paper_2411_02820_b200 as P
    cfg = P.ModelConfig(*TINY)
    A = P.build_model(cfg)
    B = P.build_model(cfg, P.PerturbationSpec.block(4, [2], 0.5, 1000))
    return P, cfg, A, B


def test_captured_rejects_another_context(tiny):
    P, cfg, A, B = tiny
    rc = P.RecomputeConfig([(2, 3)])
    rng = np.random.default_rng(5)
    t1, t2 = (rng.integers(0, cfg.vocab_size, size=200, dtype=np.int64) for _ in range(2))
    prod = P.full_prefill(A, t1, e_layers=rc.transition_layers)
    assert prod.kv.context == P.context_hash(t1).digest
    cap = P.CapturedPartialPrefill(B, 200, rc, prod.kv, prod.e_map())
    ok = cap.run(t1).logits.clone()
    with pytest.raises(P.CacheMissError) as ei:
        cap.run(t2)
    assert ei.value.layer == 0 and ei.value.kind == "kv"
    torch.cuda.synchronize()
    assert torch.equal(cap.run(t1).logits, ok)
    # an export without a context tag needs context=; a wrong context= is refused
    bare = P.LayerKV(prod.kv.k, prod.kv.v)
    with pytest.raises(ValueError):
        P.CapturedPartialPrefill(B, 200, rc, bare, prod.e_map())
    with pytest.raises(ValueError):
        P.CapturedPartialPrefill(B, 200, rc, prod.kv, prod.e_map(), context=t2)
    cap2 = P.CapturedPartialPrefill(B, 200, rc, bare, prod.e_map(), context=t1)
    assert torch.equal(cap2.run(t1).logits, ok)
    # recompute-all reads no export: any context
    full = P.CapturedPartialPrefill(B, 200, P.RecomputeConfig.full(4), None)
    full.run(t2)
    torch.cuda.synchronize()


def test_captured_workspace_survives_eager_growth(tiny):
    P, cfg, A, B = tiny
    rc = P.RecomputeConfig([(2, 3)])
    t1 = np.random.default_rng(6).integers(0, cfg.vocab_size, size=200, dtype=np.int64)
    prod = P.full_prefill(A, t1, e_layers=rc.transition_layers)
    s, x = torch.cuda.Stream(), torch.cuda.Stream()
    cap = P.CapturedPartialPrefill(B, 200, rc, prod.kv, prod.e_map(), stream=s, copy_stream=x)
    ok = cap.run(t1).logits.clone()
    # eager calls on the graph's streams with a larger n grow the shared workspace
    t_big = np.random.default_rng(7).integers(0, cfg.vocab_size, size=1000, dtype=np.int64)
    with torch.cuda.stream(s):
        P.full_prefill(A, t_big, e_layers=(), stream=s, copy_stream=x)
        scratch = torch.full((1 << 22,), 7, dtype=torch.int32, device="cuda")  # likely lands on freed blocks
    torch.cuda.synchronize()
    for _ in range(3):
        assert torch.equal(cap.run(t1).logits, ok)
    del scratch


def test_token_selective_count_in_double(tiny):
    import math
    P, cfg, A, B = tiny
    for ratio, n in ((0.1, 11), (0.15, 21), (0.2, 6), (0.3, 11)):
        ids = np.random.default_rng(n).integers(0, cfg.vocab_size, size=n, dtype=np.int64)
        prod = P.full_prefill(A, ids, e_layers=())
        r = P.token_selective_prefill(B, ids, prod.kv, ratio)
        torch.cuda.synchronize()
        assert r.n_selected == math.ceil(ratio * (n - 1)), (ratio, n)
