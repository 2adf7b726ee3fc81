"""SwiGLU MLP variant (Llama-3's gated MLP, the second row of
config 2).  The reference block is ungated, so there is no CPU oracle for this
variant: it is checked against a plain PyTorch fp32 mirror of the same block
math (model.py:466-566 with the MLP replaced by silu(x Wg) * (x Wu) @ W2) on
the same bf16-rounded weights.  Tolerances as test_gpu_parity.
"""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

DIMS = dict(n_layers=2, d_model=1024, n_heads=8, n_kv_heads=2, head_dim=128, d_ff=2816, vocab_size=8192,
            max_seq=1024, base_seed=5)


def _host_weights(seed, pert=0.0):
    rng = np.random.default_rng(seed)
    d, f, L = DIMS["d_model"], DIMS["d_ff"], DIMS["n_layers"]
    qd = DIMS["n_heads"] * DIMS["head_dim"]
    kvd = DIMS["n_kv_heads"] * DIMS["head_dim"]

    def m(r, c, std):
        return (rng.standard_normal((r, c)) * std).astype(np.float32)

    base = np.random.default_rng(1)
    out = {"embed": (base.standard_normal((DIMS["vocab_size"], d))).astype(np.float32),
           "unembed": (base.standard_normal((d, DIMS["vocab_size"])) / math.sqrt(d)).astype(np.float32),
           "g_final": np.ones(d, np.float32), "layers": []}
    for l in range(L):
        b = np.random.default_rng([2, l])
        lw = {"wq": (b.standard_normal((d, qd)) / math.sqrt(d)).astype(np.float32),
              "wk": (b.standard_normal((d, kvd)) / math.sqrt(d)).astype(np.float32),
              "wv": (b.standard_normal((d, kvd)) / math.sqrt(d)).astype(np.float32),
              "wo": (b.standard_normal((qd, d)) / math.sqrt(d)).astype(np.float32),
              "wg": (b.standard_normal((d, f)) / math.sqrt(d)).astype(np.float32),
              "wu": (b.standard_normal((d, f)) / math.sqrt(d)).astype(np.float32),
              "w2": (b.standard_normal((f, d)) / math.sqrt(f)).astype(np.float32),
              "g_attn": np.ones(d, np.float32), "g_mlp": np.ones(d, np.float32)}
        if pert and l == 1:
            for k in ("wq", "wk", "wv", "wo", "wg", "wu", "w2"):
                lw[k] = lw[k] + m(*lw[k].shape, pert * float(np.sqrt(np.mean(lw[k] ** 2))))
        out["layers"].append(lw)
    return out


def _bf(x):
    return torch.from_numpy(x).cuda().bfloat16().float()


class Mirror:
    """fp32 torch restatement of the block math on bf16-rounded weights."""

    def __init__(self, host):
        from paper_2411_02820_b200.weights import rope_tables
        self.h = host
        self.embed, self.unembed = _bf(host["embed"]), _bf(host["unembed"])
        self.layers = [{k: _bf(v) for k, v in lw.items()} for lw in host["layers"]]
        cos, sin = rope_tables(DIMS["head_dim"], DIMS["max_seq"])
        self.cos, self.sin = torch.from_numpy(cos).cuda(), torch.from_numpy(sin).cuda()

    @staticmethod
    def rms(x, g):
        return x / torch.sqrt((x * x).mean(-1, keepdim=True) + 1e-6) * g

    def rope(self, x, pos):
        half = x.shape[-1] // 2
        c, s = self.cos[pos][:, None, :], self.sin[pos][:, None, :]
        lo, hi = x[..., :half], x[..., half:]
        return torch.cat([lo * c - hi * s, lo * s + hi * c], -1)

    def block(self, h, lw, pos, kctx=None, vctx=None):
        H, G, D = DIMS["n_heads"], DIMS["n_kv_heads"], DIMS["head_dim"]
        T = h.shape[0]
        a = self.rms(h, lw["g_attn"])
        q = self.rope((a @ lw["wq"]).view(T, H, D), pos)
        k = self.rope((a @ lw["wk"]).view(T, G, D), pos)
        v = (a @ lw["wv"]).view(T, G, D)
        ks = k if kctx is None else torch.cat([kctx, k], 0)
        vs = v if vctx is None else torch.cat([vctx, v], 0)
        kk = ks.repeat_interleave(H // G, 1).transpose(0, 1)
        vv = vs.repeat_interleave(H // G, 1).transpose(0, 1)
        sc = q.transpose(0, 1) @ kk.transpose(1, 2) / math.sqrt(D)
        kp = torch.arange(ks.shape[0], device=h.device)[None, :]
        sc = sc.masked_fill(kp > pos[:, None], float("-inf"))
        o = (torch.softmax(sc, -1) @ vv).transpose(0, 1).reshape(T, H * D)
        x = h + o @ lw["wo"]
        m = self.rms(x, lw["g_mlp"])
        return x + (torch.nn.functional.silu(m @ lw["wg"]) * (m @ lw["wu"])) @ lw["w2"], k, v

    def mixed(self, ids, groups, sk=None, sv=None, se=None):
        L_ = DIMS["n_layers"]
        n = len(ids)
        P = n - 1
        cov = {l for a, b in groups for l in range(a, b + 1)}
        K, V, E = [None] * L_, [None] * L_, {}
        for l in range(L_):
            if l not in cov:
                K[l], V[l] = sk[l][:P], sv[l][:P]
        win = torch.arange(P, device="cuda")
        for a, b in groups:
            h = self.embed[torch.from_numpy(ids[:P]).cuda()] if a == 0 else se[a]
            for l in range(a, b + 1):
                E[l] = h
                h, K[l], V[l] = self.block(h, self.layers[l], win)
        ha = self.embed[int(ids[P])][None]
        pos = torch.tensor([P], device="cuda")
        Kf, Vf = [], []
        for l in range(L_):
            ha, ko, vo = self.block(ha, self.layers[l], pos, K[l], V[l])
            Kf.append(torch.cat([K[l], ko], 0))
            Vf.append(torch.cat([V[l], vo], 0))
        return Kf, Vf, E, (self.rms(ha[0], _bf(self.h["g_final"])) @ self.unembed)


@pytest.fixture(scope="module")
def models():
    import paper_2411_02820_b200 as P
    from paper_2411_02820_b200.weights import from_host
    cfg = P.ModelConfig(**DIMS, mlp_kind="swiglu")
    hA, hB = _host_weights(1), _host_weights(1, pert=0.5)
    return P, cfg, from_host(cfg, hA, "swA"), from_host(cfg, hB, "swB"), Mirror(hA), Mirror(hB)


def test_swiglu_gemm_epilogue():
    from paper_2411_02820_b200 import _lib as L, ops
    from paper_2411_02820_b200.weights import interleave_gate_up
    g = torch.Generator(device="cuda").manual_seed(3)
    M, K, F = 300, 1024, 512
    a = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    wg = (torch.randn(F, K, device="cuda", generator=g) / math.sqrt(K)).bfloat16()
    wu = (torch.randn(F, K, device="cuda", generator=g) / math.sqrt(K)).bfloat16()
    w = torch.from_numpy(interleave_gate_up(wg.float().cpu().numpy(), wu.float().cpu().numpy())).cuda().bfloat16()
    out = torch.empty(M, F, device="cuda", dtype=torch.bfloat16)
    ops.gemm(a, w, mode=L.EPI_SWIGLU_BF16, out=out)
    torch.cuda.synchronize()
    ref = torch.nn.functional.silu(a.float() @ wg.float().T) * (a.float() @ wu.float().T)
    assert ((out.float() - ref).norm() / ref.norm()).item() < 1e-2


def test_swiglu_full_and_partial_prefill(models):
    P, cfg, A, B, mA, mB = models
    ids = np.random.default_rng(9).integers(0, DIMS["vocab_size"], size=300, dtype=np.int64)
    prod = P.full_prefill(A, ids)
    cons = P.partial_prefill(B, ids, P.RecomputeConfig([(1, 1)]), prod.kv, prod.e_map())
    torch.cuda.synchronize()
    rk, rv, re, rl = mA.mixed(ids, [(0, 1)])
    lp = prod.logits
    assert (lp - rl).abs().max().item() < 0.1 and ((lp - rl).norm() / rl.norm()).item() < 3e-2
    sk = [prod.kv.k[l].float().transpose(0, 1) for l in range(2)]
    sv = [prod.kv.v[l].float().transpose(0, 1) for l in range(2)]
    se = {1: prod.e_map()[1].hidden.float()}
    _, _, _, cl = mB.mixed(ids, [(1, 1)], sk, sv, se)
    lc = cons.logits
    assert (lc - cl).abs().max().item() < 0.1 and ((lc - cl).norm() / cl.norm()).item() < 3e-2
    d = cons.kv.dense()
    assert torch.equal(d.k[0, :, :299], prod.kv.k[0, :, :299])  # reused layer: bit-exact
