"""Time the recompute GEMM shapes alone (CUDA events, median of 10): QKV (+RoPE
into the cache), o-proj (+f32 residual), W1 (+SiLU), W2 (+residual), M = 8191.

    python tools/gemm_bench.py        (DS_GEMM_BN=128 forces 128-wide N tiles)
"""
import math
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_02820_b200 import _lib as L, ops  # noqa: E402


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


M, d, F = 8191, 4096, 14336
x = torch.randn(M, d, device="cuda").bfloat16()
u = torch.randn(M, F, device="cuda").bfloat16()
h = torch.randn(M, d, device="cuda")
for name, a, N, K, mode in [("qkv(store)", x, 6144, d, L.EPI_STORE_BF16), ("o-proj(resid)", x, d, d, L.EPI_RESID_F32),
                            ("w1(silu)", x, F, d, L.EPI_SILU_BF16), ("w2(resid)", u, d, F, L.EPI_RESID_F32)]:
    w = (torch.randn(N, K, device="cuda") / math.sqrt(K)).bfloat16()
    out = h if mode == L.EPI_RESID_F32 else torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ms = t(lambda: ops.gemm(a, w, mode=mode, resid=h if mode == L.EPI_RESID_F32 else None, out=out))
    print(f"{name:14s} N={N:5d} K={K:5d}: {ms:.4f} ms  {2 * M * N * K / ms / 1e9:.1f} TFLOP/s")
