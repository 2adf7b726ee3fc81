"""Per-kernel parity on the B200 (through the C ABI).

GEMM / RMSNorm / attention are floating point: compared with a PyTorch fp32
reference of the same op on the same bf16 inputs, tolerances stated inline.
KV ingest is a copy: compared bit-exactly.
"""

import math

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    from paper_2411_02820_b200 import ops as O
    return O


def _rel(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-12)).item()


@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (256, 256, 128), (511, 384, 256), (300, 1024, 1024),
                                   (1000, 4096, 4096), (8191, 256, 512), (64, 2816, 1024)])
def test_gemm_store_bf16(ops, M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    a = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    b = (torch.randn(N, K, device="cuda", generator=g) / math.sqrt(K)).bfloat16()
    ref = a.float() @ b.float().T
    out = ops.gemm(a, b)
    torch.cuda.synchronize()
    # bf16 output rounding (2^-8 relative) dominates; accumulation is fp32
    assert _rel(out, ref) < 5e-3
    assert (out.float() - ref).abs().max().item() < 0.05 * ref.abs().max().item()


@pytest.mark.parametrize("M,N,K", [(256, 512, 1024), (777, 4096, 4096), (512, 256, 14336)])
def test_gemm_resid_and_silu(ops, M, N, K):
    from paper_2411_02820_b200 import _lib as L
    g = torch.Generator(device="cuda").manual_seed(1)
    a = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    b = (torch.randn(N, K, device="cuda", generator=g) / math.sqrt(K)).bfloat16()
    h = torch.randn(M, N, device="cuda", generator=g)
    acc = a.float() @ b.float().T
    out = ops.gemm(a, b, mode=L.EPI_RESID_F32, resid=h)
    torch.cuda.synchronize()
    # fp32 out: only accumulation-order differences (tolerance 3e-5 relative at K=14336)
    assert _rel(out, h + acc) < 3e-5
    h2 = h.clone()
    ops.gemm(a, b, mode=L.EPI_RESID_F32, resid=h2, out=h2)  # in place, as the layer uses it
    torch.cuda.synchronize()
    assert _rel(h2, h + acc) < 3e-5
    s = ops.gemm(a, b, mode=L.EPI_SILU_BF16)
    torch.cuda.synchronize()
    assert _rel(s, torch.nn.functional.silu(acc)) < 5e-3


def test_rmsnorm(ops):
    g = torch.Generator(device="cuda").manual_seed(2)
    x = torch.randn(300, 4096, device="cuda", generator=g) * 3
    gain = torch.rand(4096, device="cuda", generator=g) + 0.5
    ref = x / torch.sqrt((x * x).mean(-1, keepdim=True) + 1e-6) * gain
    out = ops.rmsnorm(x, gain)
    torch.cuda.synchronize()
    assert _rel(out, ref) < 3e-3
    table = torch.randn(1000, 4096, device="cuda", generator=g).bfloat16()
    ids = torch.randint(0, 1000, (77,), device="cuda", generator=g)
    cf = torch.empty(77, 4096, device="cuda")
    cb = torch.empty(77, 4096, device="cuda", dtype=torch.bfloat16)
    out = ops.rmsnorm(table, gain, gather=ids, copy_f32=cf, copy_bf16=cb)
    torch.cuda.synchronize()
    rows = table[ids].float()
    assert torch.equal(cf, rows) and torch.equal(cb, table[ids])
    assert _rel(out, rows / torch.sqrt((rows * rows).mean(-1, keepdim=True) + 1e-6) * gain) < 3e-3


def _ref_attention(q, k, v, q_pos0, H, G, D):
    # q [n, H*D]; k/v [G, S, D] (dense positions 0..S-1); causal by absolute position
    n = q.shape[0]
    R = H // G
    qh = q.float().view(n, H, D).transpose(0, 1)                  # [H, n, D]
    kk = k.float().repeat_interleave(R, dim=0)                     # [H, S, D]
    vv = v.float().repeat_interleave(R, dim=0)
    s = qh @ kk.transpose(1, 2) / math.sqrt(D)
    qp = torch.arange(n, device=q.device)[:, None] + q_pos0
    kp = torch.arange(k.shape[1], device=q.device)[None, :]
    s = s.masked_fill(kp > qp, float("-inf"))
    return (torch.softmax(s, -1) @ vv).transpose(0, 1).reshape(n, H * D)


@pytest.mark.parametrize("n,H,G,D", [(511, 4, 1, 64), (1000, 8, 2, 128), (64, 4, 4, 128), (2049, 32, 8, 128),
                                     (1, 4, 1, 64), (257, 8, 8, 128), (8191, 32, 8, 128)])
def test_attention_prefill_paged(ops, n, H, G, D):
    g = torch.Generator(device="cuda").manual_seed(n + H)
    pages = (n + 63) // 64
    perm = torch.randperm(pages + 3, device="cuda", generator=g)[:pages].to(torch.int32)
    kc = torch.randn(1, pages + 3, G, 64, D, device="cuda", generator=g).bfloat16()
    vc = torch.randn(1, pages + 3, G, 64, D, device="cuda", generator=g).bfloat16()
    # poison positions >= n (never valid keys) with NaN: must not leak
    dense_k = kc[0][perm.long()].permute(1, 0, 2, 3).reshape(G, pages * 64, D)[:, :n]
    dense_v = vc[0][perm.long()].permute(1, 0, 2, 3).reshape(G, pages * 64, D)[:, :n]
    if n % 64:
        last = perm[-1].long()
        kc[0, last, :, n % 64:] = float("nan")
        vc[0, last, :, n % 64:] = float("nan")
    q = torch.randn(n, H * D, device="cuda", generator=g).bfloat16()
    desc = ops.paged_kv_desc(kc, vc, perm, n)
    out = ops.attention_prefill(q, desc, 0, H, G, D)
    torch.cuda.synchronize()
    ref = _ref_attention(q, dense_k, dense_v, 0, H, G, D)
    assert torch.isfinite(out.float()).all()
    # bf16 P and bf16 output: ~1e-2 relative
    assert _rel(out, ref) < 1.5e-2


def test_kv_ingest_bit_exact(ops):
    g = torch.Generator(device="cuda").manual_seed(5)
    Lyr, G, n, D = 6, 2, 1000, 128
    P = n - 1
    src_k = torch.randn(Lyr, G, n, D, device="cuda", generator=g).bfloat16()
    src_v = torch.randn(Lyr, G, n, D, device="cuda", generator=g).bfloat16()
    pages = (n + 63) // 64
    table = torch.randperm(pages + 5, device="cuda", generator=g)[:pages].to(torch.int32)
    dk = torch.zeros(Lyr, pages + 5, G, 64, D, device="cuda", dtype=torch.bfloat16)
    dv = torch.zeros_like(dk)
    reused = [0, 2, 3, 5]
    ops.kv_ingest(ops.dense_kv_desc(src_k, src_v), ops.paged_kv_desc(dk, dv, table, n), reused, P, G, D)
    torch.cuda.synchronize()
    got_k = dk[:, table.long()].permute(0, 2, 1, 3, 4).reshape(Lyr, G, pages * 64, D)
    got_v = dv[:, table.long()].permute(0, 2, 1, 3, 4).reshape(Lyr, G, pages * 64, D)
    for l in range(Lyr):
        if l in reused:
            assert torch.equal(got_k[l, :, :P], src_k[l, :, :P])
            assert torch.equal(got_v[l, :, :P], src_v[l, :, :P])
            assert (got_k[l, :, P:] == 0).all()  # the anchor position is never copied (model.py:602)
        else:
            assert (got_k[l] == 0).all()


@pytest.mark.parametrize("n,q_pos0,D", [(300, 100, 128), (129, 1000, 64), (640, 64, 128)])
def test_attention_prefill_query_offset(ops, n, q_pos0, D):
    """Queries at positions q_pos0.. over a cache holding q_pos0 + n keys."""
    H, G = 8, 2
    g = torch.Generator(device="cuda").manual_seed(n + q_pos0)
    total = q_pos0 + n
    k = torch.randn(1, G, total, D, device="cuda", generator=g).bfloat16()
    v = torch.randn(1, G, total, D, device="cuda", generator=g).bfloat16()
    q = torch.randn(n, H * D, device="cuda", generator=g).bfloat16()
    out = ops.attention_prefill(q, ops.dense_kv_desc(k, v), 0, H, G, D, q_pos0=q_pos0)
    torch.cuda.synchronize()
    ref = _ref_attention(q, k[0], v[0], q_pos0, H, G, D)
    assert _rel(out, ref) < 1.5e-2


def test_kv_ingest_peer_kernel_bit_exact():
    """The peer-source ingest kernel (used when the producer export lives on
    another GPU) forced on one GPU through its debug switch: same placement."""
    import os
    import subprocess
    import sys
    code = (
        "import torch, sys; sys.path.insert(0, '.');"
        "from paper_2411_02820_b200 import ops;"
        "g = torch.Generator(device='cuda').manual_seed(5);"
        "Lyr, G, n, D = 4, 2, 700, 128; P = n - 1;"
        "sk = torch.randn(Lyr, G, n, D, device='cuda', generator=g).bfloat16();"
        "sv = torch.randn(Lyr, G, n, D, device='cuda', generator=g).bfloat16();"
        "pages = (n + 63) // 64;"
        "t = torch.randperm(pages + 3, device='cuda', generator=g)[:pages].to(torch.int32);"
        "dk = torch.zeros(Lyr, pages + 3, G, 64, D, device='cuda', dtype=torch.bfloat16); dv = torch.zeros_like(dk);"
        "ops.kv_ingest(ops.dense_kv_desc(sk, sv), ops.paged_kv_desc(dk, dv, t, n), [0, 3], P, G, D);"
        "torch.cuda.synchronize();"
        "gk = dk[:, t.long()].permute(0, 2, 1, 3, 4).reshape(Lyr, G, pages * 64, D);"
        "gv = dv[:, t.long()].permute(0, 2, 1, 3, 4).reshape(Lyr, G, pages * 64, D);"
        "ok = all(torch.equal(gk[l, :, :P], sk[l, :, :P]) and torch.equal(gv[l, :, :P], sv[l, :, :P]) for l in (0, 3));"
        "ok = ok and bool((gk[1] == 0).all()) and bool((gk[0, :, P:] == 0).all());"
        "print('OK' if ok else 'BAD')")
    from conftest import ROOT
    env = dict(os.environ, DS_INGEST_PEER_KERNEL="1")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert r.stdout.strip().endswith("OK"), r.stdout + r.stderr
