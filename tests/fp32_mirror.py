"""GPU fp32 mirror of the reference block math -- TEST INFRASTRUCTURE ONLY.

Where the CPU oracle is infeasible (8B dims at n = 8192: 213 s per layer,
SURVEY §8c), parity is checked against this plain PyTorch fp32 restatement
of the reference's block (model.py:466-566, Appendix A of SURVEY.md), run on
the SAME bf16 weights the kernels read (device layout of weights.py: Q/K/V
concatenated K-major, W1/W2 K-major; SwiGLU gate/up interleaved in blocks
of 16).  Every matmul is a full-precision fp32 cuBLAS SGEMM (TF32 off).
Nothing in the package imports this module.
"""

from __future__ import annotations

import math

import torch


def _fp32_matmuls():
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    torch.set_float32_matmul_precision("highest")


class Mirror:
    """fp32 forward of one device model (``ModelWeights``)."""

    def __init__(self, model, q_chunk: int = 1024):
        _fp32_matmuls()
        self.m = model
        c = model.config
        self.H, self.G, self.D, self.d, self.f = c.n_heads, c.n_kv_heads, c.head_dim, c.d_model, c.d_ff
        self.swiglu = c.mlp_kind == "swiglu"
        self.q_chunk = q_chunk

    # ---- pieces (model.py line refs in SURVEY Appendix A)
    @staticmethod
    def rms(x, g):  # model.py:466-468
        return x / torch.sqrt((x * x).mean(-1, keepdim=True) + 1e-6) * g

    def rope(self, x, pos):  # model.py:475-488 (tables in f64 -> f32, weights.rope_tables)
        half = x.shape[-1] // 2
        c = self.m.rope_cos[pos][:, None, :]
        s = self.m.rope_sin[pos][:, None, :]
        lo, hi = x[..., :half], x[..., half:]
        return torch.cat([lo * c - hi * s, lo * s + hi * c], -1)

    def attend(self, q, ks, vs, pos):
        """q [T,H,D] at absolute positions pos; ks/vs [S,G,D] at 0..S-1; key j
        visible iff j <= pos[t]; head h reads kv head h // (H/G) (model.py:491-519)."""
        T = q.shape[0]
        R = self.H // self.G
        kk = ks.permute(1, 0, 2)  # [G,S,D]
        vv = vs.permute(1, 0, 2)
        kp = torch.arange(ks.shape[0], device=q.device)
        out = torch.empty(T, self.H, self.D, device=q.device, dtype=torch.float32)
        scale = 1.0 / math.sqrt(self.D)
        for t0 in range(0, T, self.q_chunk):
            t1 = min(T, t0 + self.q_chunk)
            qc = q[t0:t1].view(t1 - t0, self.G, R, self.D).permute(1, 0, 2, 3).reshape(self.G, -1, self.D)
            s = torch.bmm(qc, kk.transpose(1, 2)) * scale  # [G, c*R, S]
            s = s.view(self.G, t1 - t0, R, -1)
            s = s.masked_fill(kp[None, None, None, :] > pos[t0:t1][None, :, None, None], float("-inf"))
            w = torch.softmax(s, -1).view(self.G, -1, ks.shape[0])
            o = torch.bmm(w, vv).view(self.G, t1 - t0, R, self.D).permute(1, 0, 2, 3)
            out[t0:t1] = o.reshape(t1 - t0, self.H, self.D)
        return out.reshape(T, self.H * self.D)

    def mlp(self, m, lw):  # model.py:532-533 (ungated) / SwiGLU row
        w1 = lw["w1"].float()
        if self.swiglu:
            blk = w1.view(self.f // 16, 2, 16, self.d)
            z = torch.nn.functional.silu(m @ blk[:, 0].reshape(self.f, self.d).T) * (m @ blk[:, 1].reshape(self.f, self.d).T)
        else:
            z = torch.nn.functional.silu(m @ w1.T)
        del w1
        return z @ lw["w2"].float().T

    def block(self, h, l, pos, kctx=None, vctx=None, kv_only=False):
        """One pre-norm block (model.py:536-562).  h [T,d] f32; kctx/vctx [S,G,D]
        (the context the rows attend over besides themselves).  Returns
        (h_out | None, k [T,G,D] post-RoPE, v [T,G,D])."""
        lw = self.m.layers[l]
        T = h.shape[0]
        HD, KD = self.H * self.D, self.G * self.D
        a = self.rms(h, lw["g_attn"])
        wqkv = lw["wqkv"].float()
        k = self.rope((a @ wqkv[HD:HD + KD].T).view(T, self.G, self.D), pos)
        v = (a @ wqkv[HD + KD:].T).view(T, self.G, self.D)
        if kv_only:
            return None, k, v
        q = self.rope((a @ wqkv[:HD].T).view(T, self.H, self.D), pos)
        del wqkv
        ks = k if kctx is None else torch.cat([kctx, k], 0)
        vs = v if vctx is None else torch.cat([vctx, v], 0)
        o = self.attend(q, ks, vs, pos)
        x = h + o @ lw["wo"].float().T
        return x + self.mlp(self.rms(x, lw["g_mlp"]), lw), k, v

    def logits(self, h_row):  # model.py:565-566
        return self.rms(h_row, self.m.g_final) @ self.m.unembed_t.float().T

    # ---- the consumer partial prefill (model.py:574-638)
    def mixed(self, ids, groups, sender_kv=None, sender_e=None):
        """ids: int64 device tensor [n]; groups: normal-form ranges; sender_kv:
        LayerKV (bf16 [L,G,n,D]) for the reused layers; sender_e: {a: [P,d] f32}.
        Returns (K list [n,G,D] per layer, V list, logits [V])."""
        L_ = self.m.config.n_layers
        n = ids.shape[0]
        P = n - 1
        cov = {l for a, b in groups for l in range(a, b + 1)}
        K, V = [None] * L_, [None] * L_
        for l in range(L_):
            if l not in cov:
                K[l] = sender_kv.k[l, :, :P].float().permute(1, 0, 2)
                V[l] = sender_kv.v[l, :, :P].float().permute(1, 0, 2)
        win = torch.arange(P, device=ids.device)
        for a, b in groups:
            h = self.m.embed[ids[:P]].float() if a == 0 else sender_e[a][:P].float()
            for l in range(a, b + 1):
                h, K[l], V[l] = self.block(h, l, win, kv_only=(l == b))
        ha = self.m.embed[ids[P:P + 1]].float()
        pos = torch.tensor([P], device=ids.device)
        Kf, Vf = [], []
        for l in range(L_):
            ha, ko, vo = self.block(ha, l, pos, K[l], V[l])
            Kf.append(torch.cat([K[l], ko], 0))
            Vf.append(torch.cat([V[l], vo], 0))
        return Kf, Vf, self.logits(ha[0])


def rel(a, b) -> float:
    a, b = a.double(), b.double()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))
