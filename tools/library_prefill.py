"""Full prefill of the same model on library kernels -- the "cuBLAS + flash
attention" comparison point SURVEY 8(d) asks for next to our own full prefill.

Same block math (model.py:536-566, ungated or SwiGLU MLP), same bf16 weights
and f32 residual stream: GEMMs are torch.matmul (cuBLAS), attention is
flash_attn.flash_attn_func (causal) when it runs on this GPU, else
torch.nn.functional.scaled_dot_product_attention (causal; cuDNN / flash
backends), RMSNorm / RoPE / SiLU are torch elementwise ops.  A baseline only:
nothing on the product path calls this.

    library_full_prefill(model, tokens_dev) -> (logits [V] f32, attention_impl)
"""

from __future__ import annotations

import torch
import torch.nn.functional as F


def _attention():
    try:
        from flash_attn import flash_attn_func
        q = torch.randn(1, 64, 4, 128, device="cuda", dtype=torch.bfloat16)
        flash_attn_func(q, q, q, causal=True)
        torch.cuda.synchronize()
        return "flash_attn " + __import__("flash_attn").__version__, \
            lambda q, k, v: flash_attn_func(q[None], k[None], v[None], causal=True)[0]
    except Exception:  # no kernel for this GPU in the wheel
        def sdpa(q, k, v):
            R = q.shape[1] // k.shape[1]
            out = F.scaled_dot_product_attention(q.transpose(0, 1)[None], k.transpose(0, 1)[None],
                                                 v.transpose(0, 1)[None], is_causal=True, enable_gqa=R > 1)
            return out[0].transpose(0, 1)
        return "torch sdpa (causal)", sdpa


def _rms(x, g):
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + 1e-6) * g


def _rope(x, cos, sin):
    half = x.shape[-1] // 2
    x1, x2 = x[..., :half].float(), x[..., half:].float()
    c, s = cos[:, None, :], sin[:, None, :]
    return torch.cat([x1 * c - x2 * s, x1 * s + x2 * c], dim=-1).to(torch.bfloat16)


def make(model):
    """Returns (fn(tokens_dev) -> logits, attention_impl)."""
    cfg = model.config
    H, G, D, d, f = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.d_model, cfg.d_ff
    impl, attn = _attention()
    swiglu = cfg.mlp_kind == "swiglu"

    def run(tokens_dev):
        n = tokens_dev.shape[0]
        cos, sin = model.rope_cos[:n], model.rope_sin[:n]
        h = model.embed[tokens_dev].float()
        for lw in model.layers:
            a = _rms(h, lw["g_attn"]).to(torch.bfloat16)
            qkv = a @ lw["wqkv"].t()
            q = _rope(qkv[:, :H * D].view(n, H, D), cos, sin)
            k = _rope(qkv[:, H * D:(H + G) * D].view(n, G, D), cos, sin)
            v = qkv[:, (H + G) * D:].reshape(n, G, D)
            o = attn(q, k, v).reshape(n, H * D)
            h = h + (o @ lw["wo"].t()).float()
            a = _rms(h, lw["g_mlp"]).to(torch.bfloat16)
            up = a @ lw["w1"].t()
            if swiglu:  # gate / up interleaved in blocks of 16 rows (weights.interleave_gate_up)
                blk = up.view(n, -1, 2, 16)
                u = (F.silu(blk[:, :, 0].float()) * blk[:, :, 1].float()).reshape(n, f).to(torch.bfloat16)
            else:
                u = F.silu(up.float()).to(torch.bfloat16)
            h = h + (u @ lw["w2"].t()).float()
        x = _rms(h[-1:], model.g_final).to(torch.bfloat16)
        return (x @ model.unembed_t.t()).float()[0]

    return run, impl
