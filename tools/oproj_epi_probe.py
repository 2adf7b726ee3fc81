"""o-proj shape (M=8191, N=K=4096) under each epilogue: is the f32 residual
epilogue what holds the K=4096 GEMM below the long-K ones?

    python tools/oproj_epi_probe.py
"""
import math
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_02820_b200 import _lib as L, ops  # noqa: E402


def t(fn, reps=20):
    for _ in range(3):
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
h = torch.randn(M, d, device="cuda")
for K in (4096, 8192, 14336):
    a = torch.randn(M, K, device="cuda").bfloat16()
    w = (torch.randn(d, K, device="cuda") / math.sqrt(K)).bfloat16()
    for name, mode in [("store_bf16", L.EPI_STORE_BF16), ("store_f32", L.EPI_STORE_F32), ("resid_f32", L.EPI_RESID_F32)]:
        out = h if mode == L.EPI_RESID_F32 else torch.empty(M, d, device="cuda",
                                                          dtype=torch.float32 if mode == L.EPI_STORE_F32 else torch.bfloat16)
        ms = t(lambda: ops.gemm(a, w, mode=mode, resid=h if mode == L.EPI_RESID_F32 else None, out=out))
        print(f"K={K:5d} {name:11s}: {ms:.4f} ms  {2 * M * d * K / ms / 1e9:.1f} TFLOP/s", flush=True)
