"""Layer-pipelined scheduler and the store boundary on the B200 (through the C ABI).

The pipelined run issues the same kernels as the fused ds_partial_prefill,
split across a link stream and a compute stream, so results must be
bit-identical; fetching the sender caches from the HBM store (per-layer
pointer table, no dense assembly) must not change a bit either.
"""

import numpy as np
import pytest
import torch

from oracle import crosskv_oracle as O

pytestmark = pytest.mark.gpu

TINY = (4, 256, 4, 1, 64, 1024, 4096, 1024, 7)


@pytest.fixture(scope="module")
def pair():
    import paper_2411_02820_b200 as P
    cfg = P.ModelConfig(*TINY)
    A = P.build_model(cfg)
    B = P.build_model(cfg, P.PerturbationSpec.block(4, [2], 0.5, 1000))
    return P, cfg, A, B


@pytest.mark.parametrize("groups", [[(2, 3)], [(1, 1), (3, 3)], [], [(0, 1)], [(0, 3)]])
def test_pipeline_matches_fused_call(pair, groups):
    P, cfg, A, B = pair
    from paper_2411_02820_b200.pipeline import ConsumerPipeline
    toks = O.synthetic_tokens(21, 1, 333, 4096)[0]
    rc = P.RecomputeConfig(groups)
    prod = P.full_prefill(A, toks)
    fused = P.partial_prefill(B, toks, rc, prod.kv, prod.e_map())
    pipe = ConsumerPipeline(B, batch_kv_jobs=2)
    got = pipe.run(toks, rc, prod.kv, prod.e_map(), timing=True)
    torch.cuda.synchronize()
    assert torch.equal(fused.logits, got.logits)
    assert torch.equal(fused.kv.dense().k, got.kv.dense().k)
    assert torch.equal(fused.kv.dense().v, got.kv.dense().v)
    t = pipe.stage_times()
    assert t.ttft_ms > 0 and t.compute[-1][0] == "anchor"
    # link order = planner order: E first, then KV ascending
    labels = [lab for lab, _, _ in t.link]
    n_e = len(rc.transition_layers)
    assert all(l.startswith("E-") for l in labels[:n_e]) and all(l.startswith("KV-") for l in labels[n_e:])


def test_store_fetch_then_pipeline(pair):
    P, cfg, A, B = pair
    from paper_2411_02820_b200.pipeline import ConsumerPipeline
    toks = O.synthetic_tokens(22, 1, 512, 4096)[0]
    rc = P.RecomputeConfig([(2, 3)])
    prod = P.full_prefill(A, toks)
    st = P.CacheStore(mode="serving", transition_layers=rc.transition_layers, config=cfg)
    total = P.store_prefill(st, A.ident, toks, prod)
    assert total == 4 * cfg.kv_bytes_per_position_bf16 * len(toks) + cfg.e_bytes_per_position_stored * (len(toks) - 1)
    kv, e_map = P.fetch_context_caches(st, A.ident, toks, rc, cfg.n_layers)
    assert sorted(e_map) == [2] and kv.layers[2] is None and kv.layers[3] is None
    ref = P.partial_prefill(B, toks, rc, prod.kv, prod.e_map())
    via_store = P.partial_prefill(B, toks, rc, kv, e_map)
    piped = ConsumerPipeline(B).run(toks, rc, kv, e_map)
    torch.cuda.synchronize()
    assert torch.equal(ref.logits, via_store.logits) and torch.equal(ref.logits, piped.logits)
    P_ = len(toks) - 1
    d = via_store.kv.dense()
    for l in (0, 1):  # bit-exact placement of the stored slices
        assert torch.equal(d.k[l, :, :P_], prod.kv.k[l, :, :P_]) and torch.equal(d.v[l, :, :P_], prod.kv.v[l, :, :P_])
    # a store without the needed layer -> CacheMissError(kv) in ascending order
    with pytest.raises(P.CacheMissError) as err:
        P.fetch_context_caches(st, "nobody", toks, rc, cfg.n_layers)
    assert (err.value.layer, err.value.kind) == (0, "kv")


def test_pipeline_errors_in_reference_order(pair):
    P, cfg, A, B = pair
    from paper_2411_02820_b200.pipeline import ConsumerPipeline
    toks = O.synthetic_tokens(23, 1, 64, 4096)[0]
    prod = P.full_prefill(A, toks)
    pipe = ConsumerPipeline(B)
    with pytest.raises(P.CacheMissError) as err:
        pipe.run(toks, P.RecomputeConfig([(1, 2)]), None)
    assert (err.value.layer, err.value.kind) == (0, "kv")
    with pytest.raises(P.CacheMissError) as err:
        pipe.run(toks, P.RecomputeConfig([(2, 3)]), prod.kv, {})
    assert (err.value.layer, err.value.kind) == (2, "e")
    with pytest.raises(P.DegenerateInputError):
        pipe.run([3], P.RecomputeConfig.full(4), None)


def test_recompute_group_and_anchor_entry_points(pair):
    """ds_recompute_group + ds_anchor compose to ds_partial_prefill's result."""
    import ctypes as C
    P, cfg, A, B = pair
    from paper_2411_02820_b200 import _lib as L
    from paper_2411_02820_b200.engine import _workspace
    toks = O.synthetic_tokens(24, 1, 200, 4096)[0]
    n = len(toks)
    full = P.partial_prefill(B, toks, P.RecomputeConfig.full(4), None)
    cache = P.PagedKV.allocate(cfg, n)
    dst = cache.desc()
    tok = torch.from_numpy(toks).cuda()
    ws = _workspace(B, n)
    s = torch.cuda.current_stream().cuda_stream
    lib = L.lib()
    L.check(lib.ds_recompute_group(C.byref(B.desc()), tok.data_ptr(), n, 0, 3, None, 0, C.byref(dst),
                                   ws.data_ptr(), ws.numel(), s))
    logits = torch.empty(cfg.vocab_size, device="cuda")
    t = torch.empty(1, dtype=torch.int32, device="cuda")
    L.check(lib.ds_anchor(C.byref(B.desc()), tok.data_ptr(), n, C.byref(dst), logits.data_ptr(), t.data_ptr(),
                          ws.data_ptr(), ws.numel(), s))
    torch.cuda.synchronize()
    assert torch.equal(logits, full.logits)
    rc = lib.ds_recompute_group(C.byref(B.desc()), tok.data_ptr(), n, 2, 3, None, 0, C.byref(dst), ws.data_ptr(),
                                ws.numel(), s)
    assert rc == L.DS_ERR_CACHE_MISS


def test_captured_partial_prefill_matches_eager():
    """CapturedPartialPrefill (one CUDA-graph replay per request) gives the eager
    call's logits bit for bit, request after request; a graph per exported
    context serves that context's requests, and tokens are re-validated."""
    import numpy as np
    import paper_2411_02820_b200 as P
    from oracle import crosskv_oracle as O
    cfg = P.ModelConfig(4, 256, 4, 1, 64, 1024, 4096, 1024, 7)
    A = P.build_model(cfg, device="cuda")
    B = P.build_model(cfg, P.PerturbationSpec.block(4, [2], 0.5, 1000), device="cuda")
    rc = P.RecomputeConfig([(2, 3)])
    toks = [O.synthetic_tokens(300 + i, 1, 200, cfg.vocab_size)[0] for i in range(2)]
    for t in toks:  # one export (and one captured graph) per shared context
        prod = P.full_prefill(A, t, e_layers=rc.transition_layers)
        cap = P.CapturedPartialPrefill(B, 200, rc, prod.kv, prod.e_map())
        for _ in range(2):
            got = cap.run(t).logits.clone()
            ref = P.partial_prefill(B, t, rc, prod.kv, prod.e_map(), copy_stream=torch.cuda.Stream()).logits
            torch.cuda.synchronize()
            assert torch.equal(got, ref)
    with pytest.raises(ValueError):
        cap.run(np.full(200, cfg.vocab_size, dtype=np.int64))
    with pytest.raises(ValueError):
        cap.run(toks[0][:100])
