"""The persistent co-resident anchor on shapes other than the 8B headline.

At n = 4096 with two of eight layers recomputed (k * P >= 800 * L) the
two-stream call runs the persistent anchor beside the recompute; the
single-stream call runs the per-launch anchor kernels.  Both use the same
device functions, so logits and caches must agree bit for bit -- for the
ungated and SwiGLU MLPs, GQA ratios 4 and 8, and head_dim 128 and 64.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

N = 4096
SHAPES = [
    dict(n_layers=8, d_model=1024, n_heads=8, n_kv_heads=2, head_dim=128, d_ff=2816, vocab_size=4096),
    dict(n_layers=8, d_model=1024, n_heads=8, n_kv_heads=1, head_dim=128, d_ff=2816, vocab_size=4096,
         mlp_kind="swiglu"),
    dict(n_layers=8, d_model=1024, n_heads=16, n_kv_heads=4, head_dim=64, d_ff=2816, vocab_size=4096),
]


@pytest.mark.parametrize("shape", SHAPES, ids=["ungated-r4-d128", "swiglu-r8-d128", "ungated-r4-d64"])
def test_persistent_anchor_matches_per_launch(shape):
    import paper_2411_02820_b200 as P
    cfg = P.ModelConfig(max_seq=N + 64, base_seed=0, **shape)
    A = P.random_model(cfg, seed=5)
    B = P.random_model(cfg, seed=6, base=A, perturb_layers=range(6, 8), eps=0.5)
    ids = np.random.default_rng(9).integers(0, cfg.vocab_size, size=N, dtype=np.int64)
    rc = P.RecomputeConfig([(6, 7)])
    prod = P.full_prefill(A, ids, e_layers=rc.transition_layers)
    one = P.partial_prefill(B, ids, rc, prod.kv, prod.e_map())
    two = P.partial_prefill(B, ids, rc, prod.kv, prod.e_map(), copy_stream=torch.cuda.Stream())
    torch.cuda.synchronize()
    assert torch.isfinite(one.logits).all()
    assert torch.equal(one.logits, two.logits)
    d1, d2 = one.kv.dense(), two.kv.dense()
    assert torch.equal(d1.k, d2.k) and torch.equal(d1.v, d2.v)
    # reused layers placed bit-exactly by the anchor's fused copy
    assert torch.equal(d2.k[:6, :, :N - 1], prod.kv.k[:6, :, :N - 1])
    # recompute-all through the persistent path == the full prefill (same structure)
    full = P.full_prefill(B, ids, e_layers=(), copy_stream=torch.cuda.Stream())
    mixed = P.partial_prefill(B, ids, P.RecomputeConfig.full(8), None, copy_stream=torch.cuda.Stream())
    torch.cuda.synchronize()
    assert torch.equal(full.logits, mixed.logits)


@pytest.mark.parametrize("groups", [[(0, 1), (5, 6)], [(2, 3), (6, 7)]], ids=["from-embeddings", "two-transitions"])
def test_persistent_anchor_multi_group(groups):
    """Several recompute groups (one seeded from the embeddings, one ending before
    the last layer): the persistent anchor waits on each group's layers and the
    results equal the single-stream order bit for bit."""
    import paper_2411_02820_b200 as P
    cfg = P.ModelConfig(max_seq=N + 64, base_seed=0, **SHAPES[0])
    A = P.random_model(cfg, seed=7)
    B = P.random_model(cfg, seed=8, base=A, perturb_layers=[l for a, b in groups for l in range(a, b + 1)], eps=0.5)
    ids = np.random.default_rng(11).integers(0, cfg.vocab_size, size=N, dtype=np.int64)
    rc = P.RecomputeConfig(groups)
    prod = P.full_prefill(A, ids, e_layers=rc.transition_layers)
    one = P.partial_prefill(B, ids, rc, prod.kv, prod.e_map())
    two = P.partial_prefill(B, ids, rc, prod.kv, prod.e_map(), copy_stream=torch.cuda.Stream())
    torch.cuda.synchronize()
    assert torch.equal(one.logits, two.logits)
    d1, d2 = one.kv.dense(), two.kv.dense()
    assert torch.equal(d1.k, d2.k) and torch.equal(d1.v, d2.v)
    reused = [l for l in range(8) if not any(a <= l <= b for a, b in groups)]
    for l in reused:
        assert torch.equal(d2.k[l, :, :N - 1], prod.kv.k[l, :, :N - 1])


@pytest.mark.parametrize("shape", [
    dict(n_layers=8, d_model=1024, n_heads=8, n_kv_heads=8, head_dim=128, d_ff=2816, vocab_size=4096),
    dict(n_layers=8, d_model=1024, n_heads=16, n_kv_heads=8, head_dim=64, d_ff=2816, vocab_size=4096),
], ids=["r1-d128", "r2-d64"])
def test_per_launch_attention_ragged(shape):
    """GQA ratios 1 and 2 at a prompt length that is not a multiple of the
    32-key ring piece (n = 3001): the per-launch anchor (TMA-staged split-KV
    attention, single stream) equals the persistent kernel (two streams) bit
    for bit, including the reused layers it bulk-stores into the cache."""
    import paper_2411_02820_b200 as P
    n = 3001
    cfg = P.ModelConfig(max_seq=n + 64, base_seed=0, **shape)
    A = P.random_model(cfg, seed=15)
    B = P.random_model(cfg, seed=16, base=A, perturb_layers=range(5, 8), eps=0.5)
    ids = np.random.default_rng(19).integers(0, cfg.vocab_size, size=n, dtype=np.int64)
    rc = P.RecomputeConfig([(5, 7)])
    prod = P.full_prefill(A, ids, e_layers=rc.transition_layers)
    one = P.partial_prefill(B, ids, rc, prod.kv, prod.e_map())
    two = P.partial_prefill(B, ids, rc, prod.kv, prod.e_map(), copy_stream=torch.cuda.Stream())
    torch.cuda.synchronize()
    assert torch.isfinite(one.logits).all()
    assert torch.equal(one.logits, two.logits)
    d1, d2 = one.kv.dense(), two.kv.dense()
    assert torch.equal(d1.k, d2.k) and torch.equal(d1.v, d2.v)
    assert torch.equal(d1.k[:5, :, :n - 1], prod.kv.k[:5, :, :n - 1])
    assert torch.equal(d1.v[:5, :, :n - 1], prod.kv.v[:5, :, :n - 1])
